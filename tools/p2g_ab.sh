mkdir -p gpurun_out
for v in v_old v_s9 v_s8 v_u8; do MLBM_LIB=variants/$v/libmlbm_b200.so timeout 300 python tools/p2g_variant.py $v 2>&1 | tail -1; done
python tools/p2g_variant_cmp.py v_old v_s9 v_s8 v_u8
for v in v_old v_s8; do
MLBM_LIB=variants/$v/libmlbm_b200.so WARM=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_p2g_cell" -c 1 -o /tmp/p2g_$v -f python tools/p2g_variant.py ncu_$v > /dev/null 2>&1
ncu -i /tmp/p2g_$v.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__registers_per_thread,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio > gpurun_out/p2g_raw_$v.csv 2>&1
python tools/src_hot.py /tmp/p2g_$v.ncu-rep k_p2g_cell 45 > gpurun_out/p2g_src_$v.txt 2>&1
done
