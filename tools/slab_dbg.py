import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2603_14982_b200 as B
from paper_2603_14982_b200.slab_lbm import SlabLBM, exchange_local
from paper_2603_14982_b200.harness.config import taylor_green_fn
d, cells, world, dtype = 3, (48, 16, 16), 2, torch.float64
lp = B.LevelParams(1, 0.8)
init = taylor_green_fn(0.05, cells[1], lp.nu(0), lp.taus, d)
whole = SlabLBM(cells, 0, 1, 0.8, dtype=dtype, init=init)
slabs = [SlabLBM(cells, r, world, 0.8, dtype=dtype, init=init) for r in range(world)]
for sl in slabs: print("rank", sl.rank, "x0", sl.x0, "first", sl.first, "owned", sl.n_owned, "col", sl.col, "left", sl.left, "right", sl.right)
for step in range(3):
    whole.step()
    for sl in slabs: ws = sl.step_local()
    exchange_local(slabs, ws)
    torch.cuda.synchronize()
    wi = whole.solver.last_roles(0)[1]
    coords, ref = whole.owned_cells(wi, "ux")
    key = {tuple(c): v for c, v in zip(coords.tolist(), ref)}
    for sl in slabs:
        c2, got = sl.owned_cells(sl.solver.last_roles(0)[1], "ux")
        want = np.array([key[tuple(c)] for c in c2.tolist()])
        bad = np.nonzero(got != want)[0]
        print("step", step, "rank", sl.rank, "ndiff", len(bad), "maxdiff", np.abs(got - want).max(), "x of diffs", sorted(set(c2[bad][:, 0].tolist()))[:10])
