"""Per-step wall time of C4 steps and which rebuild path each took (eager
first sight, capture on second sight, replay): python tools/rebuild_paths.py [steps]"""
import os, sys, time, tempfile
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
sim = build_scene(validate_scene(S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "t.npy"))))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for i in range(n):
    e0, c0, r0 = sim.rebuild_eager, sim.graph_captures, sim.rebuild_replays
    torch.cuda.synchronize()
    t = time.perf_counter()
    sim.step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) * 1e3
    print("step %3d %7.2f ms  eager %d capture %d replay %d" % (
        i, dt, sim.rebuild_eager - e0, sim.graph_captures - c0, sim.rebuild_replays - r0), flush=True)
