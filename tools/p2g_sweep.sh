# isolated C4 P2G (mode 5) timing of several library builds under variants/
for v in ${VARS:-v_old v_new}; do MLBM_LIB=variants/$v/libmlbm_b200.so timeout 300 python tools/p2g_variant.py $v 2>&1 | tail -1; done
