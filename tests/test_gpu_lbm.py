"""GPU parity of the LBM level kernels, transfers and schedule against the
oracle (fp64: <= 1e-12 abs; fp32 shifted form: <= 1e-5 relative L2).

Cases mirror the reference tests: one-step pull-streaming golden
(test_solver.py:206-254), Taylor-Green decay, static multi-level refinement
(test_solver.py:279-371), boundaries (test_solver.py:374-456), in 2D and 3D.
"""
import numpy as np
import pytest
import torch

from helpers import central_mask, compare_levels, oracle_static_refined, rel_l2
from oracle import grid as OG
from oracle import lbm as OL

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2603_14982_b200")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def smooth_fields(d, seed=0, amp=0.04):
    """Deterministic, coordinate-keyed non-trivial moment fields."""
    rng = np.random.default_rng(seed)
    k = rng.uniform(0.2, 0.9, size=(12, d))
    ph = rng.uniform(0, 6.28, size=12)
    ax = "xyz"[:d]

    def fn(pos, level):
        def w(i):
            return np.sin(pos @ k[i] + ph[i])
        out = {"rho": 1.0 + 0.02 * w(0)}
        for a in range(d):
            out["u" + ax[a]] = amp * w(1 + a)
        j = 4
        for a in range(d):
            for b in range(a, d):
                out["s" + ax[a] + ax[b]] = out["u" + ax[a]] * out["u" + ax[b]] + 0.004 * w(j % 12)
                j += 1
        return out
    return fn


def build_pair(otopo, dtype, fn, spec=None, gravity=None, tau0=0.8, h3=None,
               upward="coincident"):
    d = otopo.d
    ospec = spec or OL.BoundarySpec(d=d)
    params = dict(levels=otopo.levels, gravity=gravity or (0.0,) * d, upward_mode=upward)
    if h3 is not None:
        params["h3_xyz"] = h3
    opair = OG.PingPongPair(otopo)
    osv = OL.Solver(otopo, opair, OL.SolverParams(**params), OL.LevelParams(otopo.levels, tau0),
                    ospec)
    OL.set_fields(otopo, opair, fn)

    dtopo = B.Topology(otopo.finest, otopo.levels, otopo.periodic)
    dtopo.set_tile_set(otopo.tile_set())
    dpair = B.PingPongPair(dtopo, dtype)
    dspec = B.BoundarySpec(faces={k: (B.LogInlet(v.u0, v.beta, v.y0)
                                     if isinstance(v, OL.LogInlet) else v)
                                  for k, v in ospec.faces.items()},
                           solid_boxes=list(ospec.solid_boxes), heightmap=ospec.heightmap, dim=d)
    dparams = B.SolverParams(**params)
    dsv = B.MultiLevelSolver(dtopo, dpair, dparams, B.LevelParams(otopo.levels, tau0), dspec)
    for l in range(otopo.levels):
        if not dtopo.n_tiles(l):
            continue
        pos = dtopo.cell_coords(l) * float(1 << l)
        vals = fn(pos, l)
        for t in range(2):
            for nm, v in vals.items():
                dpair.trees[t].levels[l][nm] = v
    return osv, dsv


def moments(d):
    return OG.moment_names(d)


def last(sv, l):
    return sv.arrays(sv.last_roles(l)[1], l)


@pytest.mark.parametrize("d", [2, 3])
def test_one_step_single_level_fp64(d):
    _need_gpu()
    cells = (16,) * d
    otopo = OG.Topology.uniform(cells, 1)
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 3), tau0=0.73)
    osv.advance_bounce()
    dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(d))
    assert max(w.values()) <= 1e-14, w


@pytest.mark.parametrize("d", [2, 3])
def test_taylor_green_many_steps_fp64(d):
    _need_gpu()
    cells = (32, 32) if d == 2 else (16, 16, 8)
    otopo = OG.Topology.uniform(cells, 1)
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 5), tau0=0.8)
    for _ in range(50):
        osv.advance_bounce()
        dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(d))
    assert max(w.values()) <= 1e-12, w


@pytest.mark.parametrize("d,levels", [(2, 2), (2, 3), (3, 2)])
def test_static_multilevel_fp64(d, levels):
    _need_gpu()
    cells = (64, 64) if d == 2 else (32, 32, 32)
    otopo = oracle_static_refined(cells, levels, central_mask(cells, pad=8 if d == 2 else 4))
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 7), tau0=0.8)
    assert dsv.topology.tile_set() == otopo.tile_set()
    for _ in range(6):
        osv.advance_bounce()
        dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(d) + ["eps", "phi"])
    assert max(w.values()) <= 1e-12, w


def test_upward_average_mode_fp64():
    _need_gpu()
    cells = (64, 64)
    otopo = oracle_static_refined(cells, 2, central_mask(cells, pad=8))
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(2, 9), upward="average")
    for _ in range(4):
        osv.advance_bounce()
        dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(2))
    assert max(w.values()) <= 1e-12, w


@pytest.mark.parametrize("d", [2, 3])
def test_boundaries_fp64(d):
    _need_gpu()
    if d == 2:
        cells = (32, 32)
        faces = {"x_min": OL.LogInlet(0.04, 0.35, 6.0), "x_max": "outlet",
                 "y_min": "wall", "y_max": "outlet"}
        boxes = [(10.0, 0.0, 14.0, 5.0)]
    else:
        cells = (32, 16, 16)
        faces = {"x_min": OL.LogInlet(0.04, 0.35, 3.0), "x_max": "outlet",
                 "y_min": "wall", "y_max": "outlet", "z_min": "periodic", "z_max": "periodic"}
        boxes = [(10.0, 0.0, 2.0, 14.0, 5.0, 9.0)]
    spec = OL.BoundarySpec(d=d, faces=faces, solid_boxes=boxes)
    otopo = OG.Topology.uniform(cells, 1, spec.periodic_axes())
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 11), spec=spec,
                          gravity=(0.0, -1e-4) + ((0.0,) if d == 3 else ()))
    for _ in range(20):
        osv.advance_bounce()
        dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(d))
    assert max(w.values()) <= 1e-12, w


@pytest.mark.parametrize("d", [2, 3])
def test_fp32_shifted_rel_l2(d):
    """Gate B: fp32 device vs fp64 oracle, <= 1e-5 relative L2 after 100 steps."""
    _need_gpu()
    cells = (64, 64) if d == 2 else (32, 32, 16)
    otopo = OG.Topology.uniform(cells, 1)
    osv, dsv = build_pair(otopo, torch.float32, smooth_fields(d, 13, amp=0.03), tau0=0.8)
    for _ in range(100):
        osv.advance_bounce()
        dsv.advance_bounce()
    names = moments(d)
    for nm in names:
        r = rel_l2(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l), [nm])
        assert r <= 1e-5, (nm, r)
