set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/r2f_gpu_all.log
(cd abtree/r1 && SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 8) > gpurun_out/ab_r1.txt 2>&1
SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 8 > gpurun_out/ab_new.txt 2>&1
timeout 1500 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2f_bench_c4.json 2> gpurun_out/r2f_bench_c4.err
(cd abtree/r1 && timeout 1500 python bench.py --scene c4 --steps 30 --warmup 10 --no-e2e --no-cpu-baseline) > gpurun_out/r2f_bench_c4_r1.json 2>&1
