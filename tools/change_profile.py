"""Kernel table (torch.profiler / CUPTI) of C4 steps that change the topology:
python tools/change_profile.py [warm] [steps]  (SCENE env as the probes)"""
import os, sys, tempfile
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
sc = os.environ.get("SCENE", "AVALANCHE_C4")
scd = S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "t.npy")) if sc == "AVALANCHE_C4" else getattr(S, sc)
sim = build_scene(validate_scene(scd))
warm = int(sys.argv[1]) if len(sys.argv) > 1 else 22
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
for _ in range(warm):
    sim.step()
torch.cuda.synchronize()
c0 = sim.topology_changes
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(n):
        sim.step()
    torch.cuda.synchronize()
print("steps", n, "topology changes", sim.topology_changes - c0)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=70))
