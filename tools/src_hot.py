"""Per-CUDA-source-line instruction / stall-sample totals from an ncu report
(--print-source cuda,sass).  python tools/src_hot.py REP KERNEL_SUBSTR [top]"""
import csv, io, subprocess, sys, collections
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
path = func = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1]; continue
    if r[0] == "Function Name":
        func = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or func is None or kname not in func:
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    ei = hdr.index("Instructions Executed"); wi = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        e = float(r[ei] or 0); w = float(r[wi] or 0)
    except (ValueError, IndexError):
        continue
    a = agg[(path.split("/")[-1], line)]
    a[0] += e; a[1] += w; a[2] = r[1][:90]
te = sum(v[0] for v in agg.values()); tw = sum(v[1] for v in agg.values())
print("total warp instr %.0f samples %.0f" % (te, tw))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print("%-14s %5d  instr %5.1f%%  samples %5.1f%%  %s" % (k[0], k[1], 100 * v[0] / te, 100 * v[1] / tw, v[2]))
