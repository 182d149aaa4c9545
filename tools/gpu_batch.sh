set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_coupled.py tests/test_gpu_lbm.py -q -rf -x -k "terrain or boundaries or powder_3d or dune or fused or avalanche" 2>&1 | tail -3 > gpurun_out/r2o_tests.log
MLBM_FUSE_L0=1 python -m pytest tests/test_gpu_coupled.py -q -rf -x -k "column or sandstorm or snow or terrain" 2>&1 | tail -3 >> gpurun_out/r2o_tests.log
for i in 1 2; do
(cd abtree/prev && SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 16) > gpurun_out/ab_prev_$i.txt 2>&1
SCENE=AVALANCHE_C4 WARM=8 timeout 900 python tools/kernel_probe.py 16 > gpurun_out/ab_new_$i.txt 2>&1
done
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2o_bench.json 2>/dev/null
