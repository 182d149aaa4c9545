"""Where the time of a topology change goes: the rebuild body run eagerly with
per-C-call CUDA events (C2 scene), plus torch-side copies bracketed by hand."""
import sys, time, collections
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200 import _lib as L
from paper_2603_14982_b200.harness import build_scene, validate_scene
import os
_sc = os.environ.get("SCENE", "COLUMN_3D_C2")
if _sc == "AVALANCHE_C4":
    import tempfile
    _scd = S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "terrain.npy"))
else:
    _scd = getattr(S, _sc)
sim = build_scene(validate_scene(_scd))
if os.environ.get("SCENE") == "CLOUD_3D_C5":
    S.cloud_velocities(sim)
for _ in range(int(os.environ.get("WARM", "30"))):
    sim.step()
# force every later rebuild to run eagerly, traced
orig = sim._run_rebuild
acc = collections.defaultdict(float)
cnt = collections.Counter()
walls = []
def traced(fn, key):
    torch.cuda.synchronize()
    L.TRACE.records.clear()
    L.TRACE.enabled = True
    t = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    sim._rb_seen = set(); sim._rb_graphs = {}
    orig(fn, key)
    e1.record()
    torch.cuda.synchronize()
    walls.append(((time.perf_counter() - t) * 1e3, e0.elapsed_time(e1)))
    L.TRACE.enabled = False
    row = []
    for name, a, b, r, args in L.TRACE.records:
        acc[name] += a.elapsed_time(b) * 1e3
        cnt[name] += 1
        row.append((name, a.elapsed_time(b) * 1e3))
    per.append((key, row))
sim._run_rebuild = traced
per = []
for _ in range(int(os.environ.get("STEPS", "60"))):
    sim.step()
n = len(walls)
print("rebuilds", n)
print("wall ms (host) mean %.3f, device span ms mean %.3f" % (
    sum(w[0] for w in walls) / n, sum(w[1] for w in walls) / n))
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print("%-24s calls/rebuild %5.1f  us/rebuild %8.1f" % (k, cnt[k] / n, v / n))

for key, row in per[:4]:
    print("rebuild key", key)
    for name, us in row:
        print("   %-24s %8.1f us" % (name, us))
