"""cProfile of the host side of C2 steps (graph path): where the Python time
goes on topology-change steps.  python tools/host_profile.py [steps]"""
import cProfile, pstats, sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
sim = build_scene(validate_scene(getattr(S, os.environ.get("SCENE", "COLUMN_3D_C2"))))
for _ in range(30):
    sim.step()
torch.cuda.synchronize()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
c0 = sim.topology_changes
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    sim.step()
torch.cuda.synchronize()
pr.disable()
print("steps", n, "changes", sim.topology_changes - c0, "captures", sim.graph_captures)
pstats.Stats(pr).sort_stats(os.environ.get("SORT", "cumulative")).print_stats(int(os.environ.get("TOP", "35")))
