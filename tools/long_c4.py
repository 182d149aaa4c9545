"""Long C4 run (robustness): N coupled steps on one B200, wall time per
block of steps, topology changes, captures, particle mass, diagnostics.
python tools/long_c4.py [steps]"""
import os, sys, time, tempfile
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
sim = build_scene(validate_scene(S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "t.npy"))))
m0 = float(sim.particles.m.double().sum().item())
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
blk = 50
t = time.perf_counter()
for i in range(1, n + 1):
    sim.step()
    if i % blk == 0:
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / blk
        t = time.perf_counter()
        row = sim.diagnostics[-1]
        print(f"step {i:4d}: {1e3 * dt:7.2f} ms/step  changes {sim.topology_changes:4d}  captures "
              f"{sim.graph_captures:3d}  tiles {[sim.topology.n_tiles(l) for l in range(sim.topology.levels)]}"
              f"  sum_phi {row.sum_phi:.3e}  eps_min {row.eps_min:.3f}", flush=True)
m1 = float(sim.particles.m.double().sum().item())
print("mass drift", abs(m1 - m0) / m0, "violations", sim.last_report.violations if sim.last_report else None)
