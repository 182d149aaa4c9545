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


@pytest.mark.parametrize("d,cells,levels,world", [(3, (64, 16, 16), 2, 2), (3, (64, 32, 16), 3, 2),
                                                  (2, (128, 64), 3, 3)])
def test_multilevel_slabs_equal_single_domain(d, cells, levels, world):
    """Static refined hierarchy whose fine region straddles the cuts: every
    level's owned cells equal the single-domain run bit for bit (fp64)."""
    _need_gpu()
    from paper_2603_14982_b200.slab_lbm import (SlabMultiLevel, exchange_levels_local,
                                                run_cycle_slabs)
    from paper_2603_14982_b200.sparse_grid import moment_names
    tau0 = 0.8
    # global hierarchy: static refinement of a box across the middle of x
    gt = B.Topology.uniform(cells, levels)
    pair = B.PingPongPair(gt)
    ad = B.GridAdaptor(gt, B.LevelParams(levels, tau0))
    t0 = gt.tiles_dims(0)
    mask = np.zeros(t0, dtype=bool)
    mid = t0[0] // 2
    sl = (slice(mid - 3, mid + 3), slice(t0[1] // 4, t0[1] // 2)) + ((slice(0, t0[2] // 2),) if d == 3 else ())
    mask[sl] = True
    for _ in range(3):
        ad.update(B.RefineDriver(static_tiles=mask, levels=levels), pair)
    tiles = gt.tile_set()
    lp = B.LevelParams(levels, tau0)
    from paper_2603_14982_b200.harness.config import taylor_green_fn
    init = taylor_green_fn(0.04, cells[1], lp.nu(0), lp.taus, d)
    whole = SlabMultiLevel(cells, levels, tiles, 0, 1, tau0, init=init)
    slabs = [SlabMultiLevel(cells, levels, tiles, r, world, tau0, init=init) for r in range(world)]
    noop = lambda s, l, t: None                                          # noqa: E731
    sched = whole.solver._schedule
    for i in range(2 * len(sched)):
        run_cycle_slabs([whole], sched[i % len(sched)], noop)
        run_cycle_slabs(slabs, sched[i % len(sched)], exchange_levels_local)
    torch.cuda.synchronize()
    for l in range(levels):
        wi = whole.solver.last_roles(l)[1]
        for name in moment_names(d):
            coords, ref = whole.owned_cells(wi, l, name)
            key = {tuple(c): v for c, v in zip(coords.tolist(), ref)}
            for s in slabs:
                c2, got = s.owned_cells(s.solver.last_roles(l)[1], l, name)
                want = np.array([key[tuple(c)] for c in c2.tolist()])
                assert np.array_equal(got, want), (l, name, s.rank, np.abs(got - want).max())
