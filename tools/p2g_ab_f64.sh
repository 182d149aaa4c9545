# P2G fp32 variants (variants/v_old, variants/v_new) against the fp64 P2G of
# their own warmed C4 state (tools/p2g_variant.py with F64REF=1)
mkdir -p gpurun_out
for v in v_old v_new; do MLBM_LIB=variants/$v/libmlbm_b200.so F64REF=1 timeout 300 python tools/p2g_variant.py $v 2>&1 | tail -2; done
