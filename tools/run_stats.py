"""Run-length statistics of the sorted particle storage (runs of equal P2G
stencil base floor(x - 0.5), split at 32-particle warp chunks) on a scene
after WARM steps: python tools/run_stats.py [warm...]"""
import os, sys, tempfile
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
sc = os.environ.get("SCENE", "AVALANCHE_C4")
scd = S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "t.npy")) if sc == "AVALANCHE_C4" else getattr(S, sc)
sim = build_scene(validate_scene(scd))
done = 0
for w in [int(a) for a in sys.argv[1:]] or [0, 1, 4, 15, 16, 17]:
    while done < w:
        sim.step(); done += 1
    torch.cuda.synchronize()
    x = sim.particles.xd
    b = torch.floor(x - 0.5).to(torch.int64)
    key = (b[0] * 4096 + b[1]) * 4096 + b[2]
    n = key.numel()
    brk = torch.ones(n, dtype=torch.bool, device=key.device)
    brk[1:] = key[1:] != key[:-1]
    brk[::32] = True
    nr = int(brk.sum())
    cell = torch.floor(x).to(torch.int64)
    ck = (cell[0] * 4096 + cell[1]) * 4096 + cell[2]
    cbrk = torch.ones(n, dtype=torch.bool, device=key.device)
    cbrk[1:] = ck[1:] != ck[:-1]
    print("step %3d: %d particles, %d runs (mean run %.2f); cell-runs mean %.2f; distinct bases %d"
          % (done, n, nr, n / nr, n / int(cbrk.sum()), int(torch.unique(key).numel())), flush=True)
