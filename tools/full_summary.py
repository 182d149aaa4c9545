"""Summarise an ncu --set full report (one block per profiled launch) and
write the per-kernel DRAM traffic (read + write bytes per launch) as JSON.
python tools/full_summary.py REP OUT_TXT OUT_TRAFFIC_JSON"""
import csv, io, json, subprocess, sys, collections
rep, out_txt, out_json = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}
ki = h.index("Kernel Name")
lines = ["# ncu --set full --clock-control none (tools/round_evidence.sh), eager pass "
         "(tools/kernel_probe.py), one block per launch", ""]
traffic = collections.defaultdict(list)
for r in rows[2:]:
    name = r[ki]
    lines.append("----")
    lines.append("%-78s %s" % ("Kernel Name", name[:90]))
    vals = {}
    for k in keys:
        if k in h:
            i = h.index(k)
            lines.append("%-78s %s %s" % (k, r[i], u[i]))
            vals[k] = (r[i], u[i])
    try:
        rb = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * scale.get(vals["dram__bytes_read.sum"][1], 1)
        wb = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * scale.get(vals["dram__bytes_write.sum"][1], 1)
        short = name.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        traffic[short].append(rb + wb)
    except (KeyError, ValueError):
        pass
open(out_txt, "w").write("\n".join(lines) + "\n")
json.dump({k: {"bytes_per_launch": sum(v) / len(v), "launches": len(v)} for k, v in traffic.items()},
          open(out_json, "w"), indent=1)
print(open(out_json).read())
