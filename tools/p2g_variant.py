"""One P2G library variant (MLBM_LIB) on the C4 particle state after WARM
steps: P2G mode 5 timed in isolation (CUDA events, 20 reps) and its raster
rows saved for a cross-variant comparison.
python tools/p2g_variant.py TAG   (SCENE / WARM env as the probes)"""
import os, sys, tempfile
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200 import _lib as L
from paper_2603_14982_b200.harness import build_scene, validate_scene
tag = sys.argv[1]
sc = os.environ.get("SCENE", "AVALANCHE_C4")
scd = S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "t.npy")) if sc == "AVALANCHE_C4" else getattr(S, sc)
torch.manual_seed(0)
sim = build_scene(validate_scene(scd))
for _ in range(int(os.environ.get("WARM", "4"))):
    sim.step()
torch.cuda.synchronize()
lib = L.lib()
s = L.stream_handle()
p, grid, mat = sim.particles, sim.grid, sim.material
lv0 = grid.level0()
n = len(p)
ps = p.pd.stride(0)
NACC = grid.R["nacc"]
ts = []
for rep in range(20):
    grid.clear()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    L.check(lib.mlbm_p2g(L.C.byref(lv0), n, L.ptr(p.xd), L.ptr(p.pd), ps, mat.lam, mat.mu, mat.alpha,
                         L.ptr(grid.ras), grid.ras.stride(0), 0, 5, L.ptr(grid._err), s), "p2g")
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print("%s: p2g mode 5 on %d particles: median %.1f us  min %.1f us" % (tag, n, ts[len(ts) // 2], ts[0]))
os.makedirs("/tmp/p2gvar", exist_ok=True)
torch.save(grid.ras[:NACC].cpu(), "/tmp/p2gvar/%s.pt" % tag)
