#!/bin/bash
# ncu --set full on selected kernels (regex $1), 1 launch each after warm-up
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-20} -c ${3:-3} -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full profile rc=$?"
