timeout 900 python -m pytest tests/test_gpu_coupled.py -m gpu -x -q 2>&1 | tail -2
for sw in 1 0 1 0; do MLBM_LATEST_SWAP=$sw MLBM_STEP_TIMES=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/sw$sw.json 2> gpurun_out/sw$sw.err; python -c "
import json;d=json.loads(open('gpurun_out/sw$sw.json').read().strip().splitlines()[-1]);g=d['graph'];print('swap $sw', d['ms_per_step'], g['step_ms'], g['step_graph_captures'], g['rebuild_graph_captures'], g['topology_changes'])"; done
