"""Slab decomposition of the single-level LBM on one GPU:
N slab objects in one process exchange their ghost tile columns by device
copies (the same column mapping as the NCCL path) and must reproduce the
single-domain run bit for bit (fp64 and fp32), periodic Taylor-Green, 2 and 3
slabs, 2D and 3D."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
B = pytest.importorskip("paper_2603_14982_b200")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _tg(d, n, tau0):
    from paper_2603_14982_b200.harness.config import taylor_green_fn
    lp = B.LevelParams(1, tau0)
    return taylor_green_fn(0.05, n, lp.nu(0), lp.taus, d)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("d,cells,world", [(3, (48, 16, 16), 2), (3, (48, 16, 16), 3), (2, (64, 32), 2)])
def test_slabs_equal_single_domain(d, cells, world, dtype):
    _need_gpu()
    from paper_2603_14982_b200.slab_lbm import SlabLBM, exchange_local
    tau0 = 0.8
    init = _tg(d, cells[1], tau0)
    whole = SlabLBM(cells, 0, 1, tau0, dtype=dtype, init=init)
    slabs = [SlabLBM(cells, r, world, tau0, dtype=dtype, init=init) for r in range(world)]
    for _ in range(12):
        whole.step()
        ws = None
        for sl in slabs:
            ws = sl.step_local()
        exchange_local(slabs, ws)
    torch.cuda.synchronize()
    wi = whole.solver.last_roles(0)[1]
    from paper_2603_14982_b200.sparse_grid import moment_names
    for name in moment_names(d):
        coords, ref = whole.owned_cells(wi, name)
        key = {tuple(c): v for c, v in zip(coords.tolist(), ref)}
        for sl in slabs:
            c2, got = sl.owned_cells(sl.solver.last_roles(0)[1], name)
            want = np.array([key[tuple(c)] for c in c2.tolist()])
            assert np.array_equal(got, want), (name, sl.rank)
