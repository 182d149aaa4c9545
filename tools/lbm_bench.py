"""Level-kernel microbenchmark on a built scene: times mlbm_level_step for
every level and mode 0 (fused) / 1 (stream) / 2 (collide+bc) with CUDA events
(L2 warm, 20 reps, median), reports live cells and achieved algorithmic GB/s.
SCENE=SANDSTORM_3D_C3 python tools/lbm_bench.py"""
import os, sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200 import _lib as L
from paper_2603_14982_b200.harness import build_scene, validate_scene
_sc = os.environ.get("SCENE", "SANDSTORM_3D_C3")
if _sc == "AVALANCHE_C4":
    import tempfile
    _scd = S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "terrain.npy"))
else:
    _scd = getattr(S, _sc)
sim = build_scene(validate_scene(_scd))
for _ in range(4):
    sim.step()
torch.cuda.synchronize()
solver = sim.solver
topo = sim.topology
d = topo.d
NM = 1 + d + d * (d + 1) // 2
s = 4 if sim.dtype == torch.float32 else 8
T = 4 ** d
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for l in range(topo.levels):
    cells = topo.n_tiles(l) * T
    for mode in (0, 1, 2):
        r, w = solver.roles(l)
        src, dst = solver.arrays(r, l), solver.arrays(w, l)
        for cold in (False, True):
            ts = []
            for _ in range(20):
                if cold:
                    flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                solver._level_call(l, src, dst, mode)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            t = ts[len(ts) // 2]
            nb = cells * (2 * NM * s if mode < 2 else (2 * NM + d + 1) * s)
            print("L%d mode %d %s cells %8d  %8.1f us  %7.1f GB/s  %6.1f Mcell/ms" % (
                l, mode, "cold" if cold else "warm", cells, t, nb / t / 1e3, cells / t / 1e3))
solver.raise_pending()
