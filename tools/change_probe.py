"""Split the cost of topology-changing steps (C2, graph path): host time in
_finish_graph_step (status parse + adaptor bookkeeping + rebuild launch) and
device time of the rebuild graph (events around _run_rebuild)."""
import sys, time, collections
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
import os
sim = build_scene(validate_scene(getattr(S, os.environ.get("SCENE", "COLUMN_3D_C2"))))
if os.environ.get("SCENE") == "CLOUD_3D_C5":
    S.cloud_velocities(sim)
for _ in range(40):
    sim.step()
orig_finish = sim._finish_graph_step
orig_rb = sim._run_rebuild
host, dev = [], []
def fin(adapt_now):
    t = time.perf_counter()
    orig_finish(adapt_now)
    host.append((time.perf_counter() - t) * 1e3)
def rb(fn, key):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    t = time.perf_counter()
    orig_rb(fn, key)
    th = (time.perf_counter() - t) * 1e3
    e1.record()
    dev.append((e0, e1, th))
sim._finish_graph_step = fin
sim._run_rebuild = rb
walls = []
for _ in range(80):
    torch.cuda.synchronize(); t = time.perf_counter()
    c0 = sim.topology_changes
    sim.step()
    torch.cuda.synchronize()
    walls.append(((time.perf_counter() - t) * 1e3, sim.topology_changes - c0))
torch.cuda.synchronize()
ch = [w for w, c in walls if c]
nc = [w for w, c in walls if not c]
print("steps: change %d mean %.3f ms, no-change %d mean %.3f ms" % (len(ch), sum(ch) / max(len(ch), 1), len(nc), sum(nc) / len(nc)))
print("finish host ms (all steps) mean %.3f, max %.3f" % (sum(host) / len(host), max(host)))
if dev:
    print("rebuild: n %d, device ms mean %.3f, host launch ms mean %.3f, eager %d replays %d" % (
        len(dev), sum(a.elapsed_time(b) for a, b, _ in dev) / len(dev), sum(t for _, _, t in dev) / len(dev),
        sim.rebuild_eager, sim.rebuild_replays))
