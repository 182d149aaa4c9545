# ncu --set full (source view) of the powder-phase kernels on C4 (one eager step
# after WARM steps): surface flags, stress raster, diffusion, advection
mkdir -p gpurun_out
SCENE=AVALANCHE_C4 WARM=4 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"k_surface_need|k_powder_diffuse|k_powder_advect_tile|k_stress_cell2" -c 4 \
    -o /tmp/powder -f python tools/kernel_probe.py 1 > gpurun_out/ncu_powder.log 2>&1
python tools/full_summary.py /tmp/powder.ncu-rep gpurun_out/powder_summary.txt /dev/null > /dev/null 2>&1
for k in k_surface_need k_powder_diffuse k_powder_advect_tile k_stress_cell2; do python tools/src_hot.py /tmp/powder.ncu-rep "$k" 25; done > gpurun_out/powder_src.txt 2>&1
