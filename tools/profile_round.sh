#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench + full sets of the
# top kernels.  Run under gpurun (1 GPU).  Plain run first (ncu rule).
set -x
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
python tools/pcie_bw.py > gpurun_out/pcie.log 2>&1
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"level_kernel|k_p2g_smem|k_g2p" -s 6 -c 6 -o gpurun_out/prof_top $CMD > gpurun_out/ncu_full.log 2>&1
echo "profile rc=$?"
