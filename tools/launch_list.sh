# ncu launch list (kernel durations) of the timed steps of a short C4 bench: R=tag bash tools/launch_list.sh
R=${R:-tmpd}
CMD="python bench.py --steps 10 --warmup 4 --no-cpu-baseline --no-e2e"
MLBM_PROFILE_TIMED=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --profile-from-start off --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launches.log 2>&1
python tools/launch_summary.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_launch_summary.txt 2>&1
