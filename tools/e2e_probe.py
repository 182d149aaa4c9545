"""Probe the e2e leg: graph step alone vs with host<->device particle copies."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
sim = build_scene(validate_scene(S.COLUMN_3D_C2))
for _ in range(3):
    sim.step()
torch.cuda.synchronize()
p = sim.particles
hx = torch.empty_like(p.xd, device="cpu").pin_memory()
hp = torch.empty_like(p.pd, device="cpu").pin_memory()
hx.copy_(p.xd); hp.copy_(p.pd); torch.cuda.synchronize()
def timeit(fn, n=10):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e3
print("step only ms", timeit(sim.step))
print("h2d only ms", timeit(lambda: (p.xd.copy_(hx, non_blocking=True), p.pd.copy_(hp, non_blocking=True))))
print("d2h only ms", timeit(lambda: (hx.copy_(p.xd, non_blocking=True), hp.copy_(p.pd, non_blocking=True))))
def full():
    p.xd.copy_(hx, non_blocking=True); p.pd.copy_(hp, non_blocking=True)
    sim.step()
    hx.copy_(p.xd, non_blocking=True); hp.copy_(p.pd, non_blocking=True)
print("full ms", timeit(full), "captures", sim.graph_captures, "changes", sim.topology_changes)
import time as _t
for i in range(5):
    t0=_t.perf_counter(); p.xd.copy_(hx, non_blocking=True); p.pd.copy_(hp, non_blocking=True); torch.cuda.synchronize(); t1=_t.perf_counter()
    sim.step(); torch.cuda.synchronize(); t2=_t.perf_counter()
    hx.copy_(p.xd, non_blocking=True); hp.copy_(p.pd, non_blocking=True); torch.cuda.synchronize(); t3=_t.perf_counter()
    print("phase ms h2d %.3f step %.3f d2h %.3f captures %d changes %d" % ((t1-t0)*1e3,(t2-t1)*1e3,(t3-t2)*1e3, sim.graph_captures, sim.topology_changes))
