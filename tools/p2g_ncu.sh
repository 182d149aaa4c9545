# ncu (full set, source view) of one isolated P2G launch on C4 for each library
# variant under variants/: raw metrics and per-line hot spots
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__registers_per_thread,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,lts__t_sectors_op_red.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_global_red.sum
for v in ${VARS:-v_old v_new}; do
MLBM_LIB=variants/$v/libmlbm_b200.so WARM=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_p2g_cell" --launch-skip 4 -c 1 -o /tmp/p2g_$v -f python tools/p2g_variant.py ncu_$v > /dev/null 2>&1
ncu -i /tmp/p2g_$v.ncu-rep --page raw --csv --metrics $M > gpurun_out/p2g_raw_$v.csv 2>&1
python tools/src_hot.py /tmp/p2g_$v.ncu-rep k_p2g_cell 45 > gpurun_out/p2g_src_$v.txt 2>&1
done
