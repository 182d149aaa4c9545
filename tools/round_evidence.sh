#!/bin/bash
# Round evidence for profiles/ (run under gpurun, 1 GPU): bench lines for C4
# (default), C2, C3, C5 and C1, then — each only after its plain command
# exited 0 — an ncu launch list of a short C4 bench and ncu --set full
# captures of the top kernels on C4 and C2.   R=r2 bash tools/round_evidence.sh
R=${R:-r2}
mkdir -p gpurun_out
python bench.py > gpurun_out/${R}_bench_c4.json 2> gpurun_out/${R}_bench_c4.err; echo "bench c4 rc=$?"
python bench.py --scene c2 --steps 60 --warmup 20 > gpurun_out/${R}_bench_c2.json 2> gpurun_out/${R}_bench_c2.err; echo "bench c2 rc=$?"
python bench.py --scene c3 --steps 30 --warmup 10 --no-cpu-baseline > gpurun_out/${R}_bench_c3.json 2> gpurun_out/${R}_bench_c3.err; echo "bench c3 rc=$?"
python bench.py --scene c5 --steps 30 --warmup 10 --no-cpu-baseline > gpurun_out/${R}_bench_c5.json 2> gpurun_out/${R}_bench_c5.err; echo "bench c5 rc=$?"
python bench.py --scene c1 --steps 60 --warmup 10 > gpurun_out/${R}_bench_c1.json 2> gpurun_out/${R}_bench_c1.err; echo "bench c1 rc=$?"
CMD="python bench.py --steps 10 --warmup 4 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/${R}_plain.log 2>&1 && \
MLBM_PROFILE_TIMED=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --profile-from-start off --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launches.log 2>&1
echo "launch list rc=$?"
CMD3="python tools/kernel_probe.py 1"
SCENE=AVALANCHE_C4 WARM=4 $CMD3 > gpurun_out/${R}_plain3.log 2>&1 && \
SCENE=AVALANCHE_C4 WARM=4 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"level_kernel|k_p2g_cell2|k_g2p|k_stress_cell2|k_powder_advect|k_exchange|k_adapt_pass|k_classify|downward_kernel" -c 10 \
    -o gpurun_out/${R}_full_c4 -f $CMD3 > gpurun_out/${R}_ncu_full_c4.log 2>&1
echo "full set c4 rc=$?"
python tools/full_summary.py gpurun_out/${R}_full_c4.ncu-rep gpurun_out/${R}_full_summary_c4.txt gpurun_out/${R}_dram_traffic_c4.json > /dev/null 2>&1
for k in k_p2g_cell2 "level_kernel<(int)3, float, (int)1>" k_g2p k_stress_cell2 k_exchange; do python tools/src_hot.py gpurun_out/${R}_full_c4.ncu-rep "$k" 40; done > gpurun_out/${R}_src_hot_c4.txt 2>&1
CMD2="python tools/kernel_probe.py 2"
SCENE=COLUMN_3D_C2 $CMD2 > gpurun_out/${R}_plain2.log 2>&1 && \
SCENE=COLUMN_3D_C2 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"level_kernel|k_p2g_cell2|k_g2p|k_adapt_pass|k_exchange|downward_kernel" -c 12 \
    -o gpurun_out/${R}_full_c2 -f $CMD2 > gpurun_out/${R}_ncu_full_c2.log 2>&1
echo "full set c2 rc=$?"
python tools/full_summary.py gpurun_out/${R}_full_c2.ncu-rep gpurun_out/${R}_full_summary_c2.txt gpurun_out/${R}_dram_traffic_c2.json > /dev/null 2>&1
# the reports stay on the box (gpurun copies back at most 64 MiB)
rm -f gpurun_out/${R}_full_c4.ncu-rep gpurun_out/${R}_full_c2.ncu-rep
du -sh gpurun_out
python tools/launch_summary.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_launch_summary.txt 2>&1
