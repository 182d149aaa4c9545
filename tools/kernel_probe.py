"""Per-C-call device time of the C2 step (eager pass, CUDA events around every
library call; L2 warm).  python tools/kernel_probe.py [steps]"""
import sys, collections
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
for _ in range(int(os.environ.get("WARM", "12"))):
    sim.step()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
sim.use_graphs = False
torch.cuda.synchronize()
# ncu --profile-from-start off captures only the probed steps (not the scene
# build's initial adapt pass or the warm-up)
torch.cuda.cudart().cudaProfilerStart()
L.TRACE.start()
for _ in range(n):
    sim.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
recs = L.TRACE.stop()
acc = collections.defaultdict(float)
cnt = collections.Counter()
for r in recs:
    name = r[0]
    if name == "mlbm_level_step":
        a = r[4]
        try:
            lvl = a[0]._obj.level
        except AttributeError:
            lvl = -1
        name += "[mode %s, L%d]" % (a[4], lvl)
    acc[name] += r[1].elapsed_time(r[2]) * 1e3
    cnt[name] += 1
tot = sum(acc.values())
print("steps", n, "sum of calls us/step %.1f" % (tot / n))
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print("%-34s calls/step %5.2f  us/call %7.1f  us/step %7.1f" % (k, cnt[k] / n, v / cnt[k], v / n))
