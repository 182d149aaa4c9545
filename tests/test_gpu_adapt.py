"""Device block maintenance vs the reference (golden adapt walk) and the
oracle (3D random walks): tile sets, int16 streaks, created / deleted
counts bit-exact after every update; surviving tiles keep their cells
bitwise (test_adapt.py:118-147)."""
import os

import numpy as np
import pytest
import torch

from oracle import adapt as OA
from oracle import grid as OG
from oracle import lbm as OL

pytestmark = pytest.mark.gpu
B = pytest.importorskip("paper_2603_14982_b200")
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def tiles_of(topo):
    return np.array(sorted(topo.tile_set()), dtype=np.int64).reshape(-1, 2 + topo.d)


@pytest.mark.parametrize("fused,path", [(True, "bits"), (True, "coop"), (False, "ops")])
def test_adapt_walk_matches_reference_golden(fused, path, monkeypatch):
    """fused: the one-launch pass, byte cooperative grid (coop, default) or
    bit-packed single CTA (bits, opt-in); unfused: one launch per bitmap op."""
    _need_gpu()
    monkeypatch.setenv("MLBM_ADAPT_PATH", path)
    g = np.load(os.path.join(GOLD, "adapt_walk.npz"))
    topo = B.Topology.uniform((64, 64), 3)
    pair = B.PingPongPair(topo)
    ad = B.GridAdaptor(topo, B.LevelParams(3, 0.8))
    ad.fused = fused
    for step in range(60):
        rep = ad.update(B.RefineDriver(positions=g[f"pos{step}"], levels=3), pair)
        assert np.array_equal(tiles_of(topo), g[f"tiles{step}"]), step
        for l, st in enumerate(ad.streak):
            assert np.array_equal(st, g[f"streak{step}_{l}"]), (step, l)
        assert list(rep.created) == list(g[f"created{step}"])
        assert list(rep.deleted) == list(g[f"deleted{step}"])
        assert rep.violations == []


@pytest.mark.parametrize("path,grid", [("bits", None), ("coop", None), ("coop", "296"),
                                       ("coop", "37")])
def test_adapt_3d_random_walk_vs_oracle(path, grid, monkeypatch):
    """grid: the cooperative pass with 2 CTAs per SM (the large-grid launch
    shape C4 uses) and with fewer CTAs than SMs (several tiles per thread)."""
    _need_gpu()
    monkeypatch.setenv("MLBM_ADAPT_PATH", path)
    if grid:
        monkeypatch.setenv("MLBM_ADAPT_GRID", grid)
    rng = np.random.default_rng(11)
    cells, levels = (64, 32, 32), 3
    otopo = OG.Topology.uniform(cells, levels)
    opair = OG.PingPongPair(otopo)
    oad = OA.GridAdaptor(otopo, OL.LevelParams(levels, 0.8))
    dtopo = B.Topology.uniform(cells, levels)
    dpair = B.PingPongPair(dtopo)
    dad = B.GridAdaptor(dtopo, B.LevelParams(levels, 0.8))
    pos = rng.random((4, 3)) * np.array(cells) * 0.8 + 2
    for step in range(40):
        pos = np.clip(pos + rng.normal(0, 2.0, pos.shape), 0.5, np.array(cells) - 0.5)
        orep = oad.update(OA.RefineDriver(pos, None, levels), opair)
        drep = dad.update(B.RefineDriver(positions=pos, levels=levels), dpair)
        assert dtopo.tile_set() == otopo.tile_set(), step
        for a, b in zip(dad.streak, oad.streak):
            assert np.array_equal(a, b), step
        assert list(drep.created) == list(orep.created)
        assert list(drep.deleted) == list(orep.deleted)
        assert drep.noop == orep.noop


def test_surviving_cells_keep_values_bitwise():
    _need_gpu()
    topo = B.Topology.uniform((64, 64), 3)
    pair = B.PingPongPair(topo)
    ad = B.GridAdaptor(topo, B.LevelParams(3, 0.8))
    ad.update(B.RefineDriver(positions=np.array([[10.5, 13.2]]), levels=3), pair)
    rng = np.random.default_rng(1)
    lv = pair.trees[0].levels[1]
    lv["sxy"] = rng.random(lv.data.shape[1])
    snap = {tuple(c): lv["sxy"][i * 16:(i + 1) * 16].cpu().numpy().copy()
            for i, c in enumerate(topo.tile_coords(1))}
    ad.update(B.RefineDriver(positions=np.array([[10.5, 13.2], [51.0, 49.0]]), levels=3), pair)
    lv2 = pair.trees[0].levels[1]
    hit = 0
    for i, c in enumerate(topo.tile_coords(1)):
        if tuple(c) in snap:
            assert np.array_equal(lv2["sxy"][i * 16:(i + 1) * 16].cpu().numpy(), snap[tuple(c)])
            hit += 1
    assert hit > 0


def test_particle_outside_domain_raises():
    _need_gpu()
    topo = B.Topology.uniform((64, 64), 3)
    pair = B.PingPongPair(topo)
    ad = B.GridAdaptor(topo, B.LevelParams(3, 0.8))
    with pytest.raises(ValueError):
        ad.update(B.RefineDriver(positions=np.array([[70.0, 3.0]]), levels=3), pair)


@pytest.mark.parametrize("path", ["bits", "coop"])
@pytest.mark.parametrize("dim", [2, 3])
def test_invariant_violations_reported_fused_and_unfused(dim, path, monkeypatch):
    """A tile set with a leaf whose ring is incomplete and a finest tile
    covered twice: the fused pass and the per-op pass report the same
    coverage / ring / particle counts (adapt.py:374-389, reported not
    raised), and a consistent tile set reports none."""
    _need_gpu()
    monkeypatch.setenv("MLBM_ADAPT_PATH", path)
    cells = (64, 64) if dim == 2 else (32, 32, 32)
    topo = B.Topology.uniform(cells, 2)
    pair = B.PingPongPair(topo)
    ad = B.GridAdaptor(topo, B.LevelParams(2, 0.8))
    ctr = np.array(cells, dtype=float) / 2 + 0.3
    drv = B.RefineDriver(positions=ctr[None, :], levels=2)
    for _ in range(3):
        ad.update(drv, pair)
    ok = topo.tile_set()
    # drop one border tile next to a leaf at level 0 and add a stray leaf at level 0
    lvl0 = sorted(t for t in ok if t[0] == 0)
    border = [t for t in lvl0 if t[-1] == 1][0]
    stray = (0,) + tuple(0 for _ in range(dim)) + (0,)
    bad = (set(ok) - {border}) | {stray}
    Lv = topo.levels
    counts = {}
    for fused in (True, False):
        topo.set_tile_set(sorted(bad))
        ad.fused = fused
        ad.plan_device(drv)
        counts[fused] = ad._status[Lv:Lv + 3].cpu().numpy().tolist()
    assert counts[True] == counts[False], counts
    assert counts[True][0] > 0 and counts[True][1] > 0, counts
    topo.set_tile_set(sorted(ok))
    ad.fused = True
    ad.plan_device(drv)
    assert ad._status[Lv:Lv + 3].cpu().numpy().tolist() == [0, 0, 0]


def test_adapt_windows_bit_identical_to_full_grid():
    """The G2P-seeded adapt pass works inside per-level tile windows
    (mlbm_adapt_pass `win`): a churning 3D cloud in a domain much larger than
    the cloud runs identically with the windows and over the whole grids —
    tile sets and int16 streaks bitwise after every step, fields and
    particles to the fp64 atomic-order noise — and the level-0 window stays
    smaller than the grid."""
    import scenes as S
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sc = S.scene(S.CLOUD_3D_SMALL)
    sc["domain"]["cells"] = [256, 96, 64]
    sc["domain"]["levels"] = 3
    # no periodic axis (a periodic axis keeps its whole extent)
    sc["boundaries"] = {"x_min": "outlet", "x_max": "outlet", "y_min": "wall", "y_max": "wall",
                        "z_min": "outlet", "z_max": "outlet"}
    sims = []
    for windows in (True, False):
        sim = build_scene(validate_scene(sc))
        sim.adaptor.windows = windows
        rng = np.random.default_rng(5)
        sim.particles.v = rng.normal(0, 0.1, (len(sim.particles), 3)).clip(-0.45, 0.45)
        sims.append(sim)
    changes = 0
    for s in range(16):
        for sim in sims:
            sim.step()
        a, b = sims
        assert a.topology.tile_set() == b.topology.tile_set(), f"step {s}"
        for x, y in zip(a.adaptor._streak, b.adaptor._streak):
            assert torch.equal(x, y), f"streaks, step {s}"
        changes = a.topology_changes
    assert changes > 0
    a, b = sims
    # fields and particles: equal up to the fp64 atomic summation order of P2G
    for l in range(a.topology.levels):
        for t in range(2):
            x = a.pair.trees[t].levels[l].data[:, :a.topology.cell_count(l)]
            y = b.pair.trees[t].levels[l].data[:, :b.topology.cell_count(l)]
            assert (x - y).abs().max().item() <= 1e-9
    assert (a.particles.xd - b.particles.xd).abs().max().item() <= 1e-9
    assert (a.particles.pd - b.particles.pd).abs().max().item() <= 1e-9
    # the windows were in use and narrower than the level-0 tile grid
    w = a.adaptor._win.view(2, a.topology.levels, 6).cpu().numpy()
    g0 = a.topology.tile_grid(0)
    ext = w[0, 0, 3:] - w[0, 0, :3] + 1
    assert a.adaptor._win_key is not None
    assert int(np.prod(ext)) < int(np.prod(g0))
