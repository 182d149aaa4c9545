# ncu --set full with source of the two particle kernels on C4 (1 launch each)
mkdir -p gpurun_out
export SCENE=AVALANCHE_C4 WARM=4
python tools/kernel_probe.py 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_p2g_cell2|k_g2p" -c 2 -o gpurun_out/prof_c4 -f python tools/kernel_probe.py 1 > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?"
ls -la gpurun_out/prof_c4.ncu-rep
