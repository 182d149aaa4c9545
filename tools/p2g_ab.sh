# A/B of the P2G kernel between variants/v_old and variants/v_new on C4
# (tools/p2g_variant.py: isolated mode-5 launches), raster agreement, then the
# GPU suites that exercise P2G with the in-tree library
mkdir -p gpurun_out
for v in v_old v_new v_old v_new; do MLBM_LIB=variants/$v/libmlbm_b200.so timeout 300 python tools/p2g_variant.py $v 2>&1 | tail -1; done
python tools/p2g_variant_cmp.py v_old v_new
timeout 600 python -m pytest tests/test_gpu_coupled.py tests/test_gpu_gate_b.py tests/test_gpu_seams.py -x -q -m gpu 2>&1 | tail -3
SCENE=AVALANCHE_C4 WARM=8 timeout 400 python tools/kernel_probe.py 6 2>&1 | head -12
