mkdir -p gpurun_out
for t in abtree/old .; do
 (cd $t && SCENE=AVALANCHE_C4 WARM=8 timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_stress_cell2|k_surface_need|k_g2p|k_p2g_cell2" -c 8 --csv python tools/kernel_probe.py 2) > gpurun_out/ab2_$(basename $t).csv 2>&1
done
