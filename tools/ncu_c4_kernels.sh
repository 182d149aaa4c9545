#!/bin/bash
# ncu --set full of the top C4 kernels, one capture each (the 4th launch of
# the kernel: past the scene build and the first steps), summaries + DRAM
# traffic per launch for bench.py's roofline.   R=r2 bash tools/ncu_c4_kernels.sh
R=${R:-r2}
mkdir -p gpurun_out
export SCENE=AVALANCHE_C4 WARM=4
python tools/kernel_probe.py 1 > gpurun_out/${R}_k_plain.log 2>&1 || exit 1
for k in k_p2g_cell2 k_g2p level_kernel k_exchange k_stress_cell2 k_powder_advect k_adapt_pass k_classify downward_kernel k_gather_particles; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 \
      -o gpurun_out/${R}_k_$k -f python tools/kernel_probe.py 1 > gpurun_out/${R}_k_$k.log 2>&1
  echo "$k rc=$?"
done
python - <<'PY'
import glob, json, os, subprocess
R = os.environ.get("R", "r2")
traffic, lines = {}, []
for rep in sorted(glob.glob(f"gpurun_out/{R}_k_*.ncu-rep")):
    out_txt = rep.replace(".ncu-rep", "_summary.txt")
    out_js = rep.replace(".ncu-rep", "_traffic.json")
    subprocess.run(["python", "tools/full_summary.py", rep, out_txt, out_js], capture_output=True)
    try:
        traffic.update(json.load(open(out_js)))
        lines.append(open(out_txt).read())
    except OSError:
        pass
json.dump(traffic, open(f"gpurun_out/{R}_dram_traffic_c4.json", "w"), indent=1)
open(f"gpurun_out/{R}_full_summary_c4.txt", "w").write("\n".join(lines))
PY
for k in k_p2g_cell2 k_g2p k_exchange k_stress_cell2; do python tools/src_hot.py gpurun_out/${R}_k_$k.ncu-rep "$k" 40; done > gpurun_out/${R}_src_hot_c4.txt 2>&1
python tools/src_hot.py gpurun_out/${R}_k_level_kernel.ncu-rep "level_kernel" 40 >> gpurun_out/${R}_src_hot_c4.txt 2>&1
rm -f gpurun_out/${R}_k_*.ncu-rep
