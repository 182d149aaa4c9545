"""Time the particle sort (keys, counting sort, row gather) on the C4 state
after WARM steps: python tools/sort_probe.py [reps]"""
import os, sys, tempfile
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
sim = build_scene(validate_scene(S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "t.npy"))))
for _ in range(int(os.environ.get("WARM", "4"))):
    sim.step()
torch.cuda.synchronize()
ts = []
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    sim._sort_into_scratch()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("particle sort ms:", " ".join("%.3f" % t for t in ts))
