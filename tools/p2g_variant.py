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
if os.environ.get("F64REF"):
    # fp64 raster of the same (fp32) particle state: the yardstick for the
    # rounding of the fp32 variants (tools/p2g_variant_cmp.py f64 v_old v_new)
    p64 = p.pd.double()
    ras64 = torch.zeros(grid.ras.shape, dtype=torch.float64, device=grid.ras.device)
    L.check(lib.mlbm_p2g(L.C.byref(lv0), n, L.ptr(p.xd), L.ptr(p64), p64.stride(0), mat.lam, mat.mu,
                         mat.alpha, L.ptr(ras64), ras64.stride(0), 1, 0, L.ptr(grid._err), s), "p2g f64")
    torch.cuda.synchronize()
    # the warm-up steps ran this variant's P2G: its state is its own, so the
    # yardstick is saved per variant
    ref = ras64[:NACC].cpu()
    mine = grid.ras[:NACC].double().cpu()
    rel = [float((mine[q] - ref[q]).norm() / ref[q].norm().clamp_min(1e-300)) for q in range(NACC)]
    print("%s vs fp64 P2G of the same state, rel L2 per row: %s" % (tag, " ".join("%.1e" % r for r in rel)))
