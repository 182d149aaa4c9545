set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf 2>&1 | tail -5 > gpurun_out/r2q_tests.log
SCENE=AVALANCHE_C4 WARM=8 STEPS=12 python tools/rebuild_probe.py > gpurun_out/r2q_rebuild.txt 2>&1
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r2q_bench.json 2>/dev/null
