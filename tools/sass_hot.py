"""Hot SASS ranges of one kernel in an ncu report: python tools/sass_hot.py REP KERNEL_SUBSTR [top]"""
import csv, subprocess, sys, io
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks = []
cur = None
for x in rows:
    if x and x[0] == "Kernel Name":
        cur = (x[1], [])
        blocks.append(cur)
        continue
    if cur is not None:
        cur[1].append(x)
for name, b in blocks:
    if kname not in name:
        continue
    h = b[0]
    si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    body = [x for x in b[1:] if len(x) > max(si, wi, ei)]
    tot = sum(float(x[wi]) for x in body)
    ins = sum(float(x[ei]) for x in body)
    print(name[:100], "samples", tot, "warp instr", ins, "sass lines", len(body))
    # coarse histogram over 32-instruction windows
    win = 32
    hist = []
    for i in range(0, len(body), win):
        s = sum(float(x[wi]) for x in body[i:i + win])
        e = sum(float(x[ei]) for x in body[i:i + win])
        hist.append((s, e, i))
    for s, e, i in sorted(hist, reverse=True)[:top // 2]:
        ops = {}
        for x in body[i:i + win]:
            op = x[si].split()[0] if not x[si].strip().startswith("@") else x[si].split()[1]
            ops[op] = ops.get(op, 0) + 1
        print("win %5d samples %6.0f (%.1f%%) instr %10.0f ops %s" % (
            i, s, 100 * s / tot, e, sorted(ops.items(), key=lambda kv: -kv[1])[:6]))
    break
