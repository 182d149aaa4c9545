"""Wall-clock split of C2 topology-change steps (graph path): host bookkeeping
in GridAdaptor.finish / _prepare, the rebuild-graph replay and the eager
diagnostics row.  python tools/change_timing.py [steps]"""
import sys, os, time, collections
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
from paper_2603_14982_b200 import coupling as CP, adapt as AD
sim = build_scene(validate_scene(getattr(S, os.environ.get("SCENE", "COLUMN_3D_C2"))))
acc = collections.defaultdict(float)
cnt = collections.Counter()

def wrap(obj, name, key):
    f = getattr(obj, name)
    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        acc[key] += time.perf_counter() - t
        cnt[key] += 1
        return r
    setattr(obj, name, g)

wrap(sim.adaptor, "finish", "adaptor.finish (incl. prepare + replay + diag)")
wrap(sim.adaptor, "_prepare", "adaptor._prepare (host part)")
wrap(sim, "_run_rebuild", "_run_rebuild (replay + diag)")
wrap(sim, "_record_diagnostics", "_record_diagnostics (launches)")
wrap(sim.grid, "sync_topology", "grid.sync_topology")
wrap(sim.solver, "_refresh_tables", "solver._refresh_tables")
import torch.cuda.graphs as TG
_orig_replay = TG.CUDAGraph.replay
def _replay(self):
    t = time.perf_counter()
    _orig_replay(self)
    acc["CUDAGraph.replay (all graphs)"] += time.perf_counter() - t
    cnt["CUDAGraph.replay (all graphs)"] += 1
TG.CUDAGraph.replay = _replay
for _ in range(30):
    sim.step()
torch.cuda.synchronize()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
acc.clear(); cnt.clear()
c0 = sim.topology_changes
t0 = time.perf_counter()
for _ in range(n):
    sim.step()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
ch = sim.topology_changes - c0
print(f"steps {n} changes {ch} wall {1e3 * wall / n:.3f} ms/step")
for k, v in acc.items():
    print(f"{k:52s} calls {cnt[k]:4d}  {1e6 * v / max(cnt[k], 1):8.1f} us/call")
