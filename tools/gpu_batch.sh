mkdir -p gpurun_out
python -m pytest tests -m gpu -q -rf 2>&1 | tail -5 > gpurun_out/r2s_tests.log
SCENE=AVALANCHE_C4 WARM=8 STEPS=12 python tools/rebuild_probe.py > gpurun_out/r2s_rebuild.txt 2>&1
SCENE=AVALANCHE_C4 MLBM_ADAPT_TIMESTAMPS=1 python tools/adapt_bench.py > gpurun_out/r2s_adapt.txt 2>&1
