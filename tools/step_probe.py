"""Per-step wall time of the C2 coupled step with topology-change / capture flags."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rows = []
for i in range(n):
    c0, t0c = sim.graph_captures, sim.topology_changes
    torch.cuda.synchronize(); t = time.perf_counter()
    sim.step()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) * 1e3
    rows.append((i, dt, sim.graph_captures - c0, sim.topology_changes - t0c,
                 [sim.topology.n_tiles(l) for l in range(sim.topology.levels)]))
for r in rows:
    print("step %3d %8.3f ms capture=%d change=%d tiles=%s" % r)
import numpy as np
dts = np.array([r[1] for r in rows])
ch = np.array([r[3] for r in rows]) > 0
cp = np.array([r[2] for r in rows]) > 0
print("captures %d rebuild eager %d replays %d" % (sim.graph_captures, sim.rebuild_eager, sim.rebuild_replays)); print("mean %.3f ms, steps with change %d (mean %.3f ms), no-change no-capture mean %.3f ms" % (
    dts.mean(), ch.sum(), dts[ch].mean() if ch.any() else 0, dts[~ch & ~cp].mean()))
