"""Critical-path view of graph-replayed steps (torch.profiler / CUPTI kernel
timestamps): per step the wall span from the first kernel start to the last
kernel end, the busy time of the union of all kernel intervals, the idle gaps,
and per stream the kernel time.  python tools/timeline.py [warm] [steps]
(SCENE env as the probes; default C4)"""
import json, os, sys, tempfile, collections
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
sc = os.environ.get("SCENE", "AVALANCHE_C4")
scd = S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "t.npy")) if sc == "AVALANCHE_C4" else getattr(S, sc)
sim = build_scene(validate_scene(scd))
warm = int(sys.argv[1]) if len(sys.argv) > 1 else 12
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
for _ in range(warm):
    sim.step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
marks = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(n):
        torch.cuda.synchronize()
        marks.append(sim.topology_changes)
        sim.step()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy") and "dur" in e]
# framework (aten) kernels: which host op launched them
ops = {e.get("args", {}).get("External id"): e["name"] for e in ev if e.get("cat") == "cpu_op"}
for e in ks:
    if "at::" in e["name"]:
        print("framework kernel %s <- host op %s" % (e["name"][:60], ops.get(e.get("args", {}).get("External id"))))
ks.sort(key=lambda e: e["ts"])
# split into steps at host synchronisations: gaps > 200 us between kernels
steps, cur = [], [ks[0]]
for e in ks[1:]:
    if e["ts"] - max(x["ts"] + x["dur"] for x in cur[-50:]) > 200:
        steps.append(cur); cur = [e]
    else:
        cur.append(e)
steps.append(cur)
for si, st in enumerate(steps):
    t0 = st[0]["ts"]; t1 = max(e["ts"] + e["dur"] for e in st)
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in st)
    busy, a, b = 0.0, iv[0][0], iv[0][1]
    gaps = []
    for s_, e_ in iv[1:]:
        if s_ > b:
            busy += b - a; gaps.append((s_ - b, a)); a, b = s_, e_
        else:
            b = max(b, e_)
    busy += b - a
    per_stream = collections.defaultdict(float)
    for e in st:
        per_stream[e.get("tid")] += e["dur"]
    tot = sum(e["dur"] for e in st)
    print("step %d: %d kernels, span %.3f ms, busy %.3f ms, idle %.3f ms, kernel sum %.3f ms, streams %s"
          % (si, len(st), (t1 - t0) / 1e3, busy / 1e3, (t1 - t0 - busy) / 1e3, tot / 1e3,
             {k: round(v / 1e3, 3) for k, v in per_stream.items()}))
    if si == len(steps) // 2:
        agg = collections.defaultdict(lambda: [0, 0.0])
        for e in st:
            nm = e["name"].replace("void ", "").split("(")[0].split("<")[0]
            agg[nm][0] += 1
            agg[nm][1] += e["dur"]
        print("  every kernel / copy / memset of this step (name, count, total us):")
        for nm, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            print("    %-44s %4d %10.1f" % (nm, c, t))
        # the exposed (not overlapped) time of each kernel name on the busy timeline
        print("  largest idle gaps (us):", sorted([round(g, 1) for g, _ in gaps], reverse=True)[:8])
        seq = []
        for e in st:
            seq.append((e["ts"] - t0, e["dur"], e.get("tid"), e["name"][:60]))
        for r in seq:
            if r[1] > 40:
                print("   %9.1f +%8.1f  [%s] %s" % r)
