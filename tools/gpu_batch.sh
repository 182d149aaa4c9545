set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_lbm.py -q -rA 2>&1 | tail -30 > gpurun_out/r2a_lbm.log
python -m pytest tests/test_gpu_gate_b.py -q -s -rA 2>&1 | tail -40 > gpurun_out/r2a_gateb.log
python -m pytest tests/test_gpu_coupled.py -q -rA -k "powder_over or checkpoint or powder_box or column_3d_two" 2>&1 | tail -20 > gpurun_out/r2a_coupled.log
timeout 900 python tools/gate_b_drift.py 20 column,sandstorm,sand_collapse_2d > gpurun_out/r2a_drift.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_lbm.py -q -x > gpurun_out/r2a_memcheck.txt 2>&1
tail -5 gpurun_out/*.log
