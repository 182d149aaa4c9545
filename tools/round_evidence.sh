#!/bin/bash
# Bench line + ncu launch list + ncu --set full of the top kernels, for profiles/.
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?"
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"level_kernel|k_p2g_cell|k_g2p|k_adapt_pass|k_exchange" -s 20 -c 8 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "profile rc=$?"
