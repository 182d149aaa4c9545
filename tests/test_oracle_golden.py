"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference
package itself (tests/golden/make_golden.py).  Every 2D path of the oracle
must reproduce them: topology and streaks bit-exact, fields / particles to
1e-12 (fp64 reduction order is the only freedom).
"""
import os

import numpy as np
import pytest

import scenes as S
from oracle import adapt as OA
from oracle import grid as OG
from oracle import lbm as OL
from oracle import scene as OS

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def tiles_of(topo):
    return np.array(sorted(topo.tile_set()), dtype=np.int64).reshape(-1, 2 + topo.d)


def fields_vs_gold(topo, arrays_fn, g, tol):
    names = OG.field_names(2)
    worst = 0.0
    for l in range(topo.levels):
        cc = topo.cell_coords(l)
        if not len(cc):
            continue
        order = np.lexsort(cc.T[::-1])
        assert np.array_equal(cc[order], g[f"L{l}_coords"])
        a = arrays_fn(l)
        for nm in names:
            worst = max(worst, float(np.abs(np.asarray(a[nm])[order] - g[f"L{l}_{nm}"]).max()))
    assert worst <= tol, worst
    return worst


def validated(scene):
    pytest.importorskip("torch")
    from paper_2603_14982_b200.harness.config import validate_scene
    return validate_scene(scene)


def test_one_step_golden():
    g = load("one_step_16")
    topo = OG.Topology.uniform((16, 16), 1)
    pair = OG.PingPongPair(topo)
    sv = OL.Solver(topo, pair, OL.SolverParams(levels=1), OL.LevelParams(1, float(g["tau"])))
    cc = topo.cell_coords(0)
    for tree in pair.trees:
        for nm in ("rho", "ux", "uy", "sxx", "sxy", "syy"):
            tree.levels[0][nm][:] = g[f"in_{nm}"][cc[:, 0], cc[:, 1]]
    sv.advance_bounce()
    fields_vs_gold(topo, lambda l: sv.arrays(sv.last_roles(l)[1], l), g, 1e-15)


@pytest.mark.parametrize("levels", [2, 3])
def test_refined_taylor_green_golden(levels):
    g = load(f"tg_refined_L{levels}")
    cells = (64, 64)
    t = [c // 4 for c in cells]
    static = np.zeros(t, dtype=bool)
    static[t[0] // 4: 3 * t[0] // 4, t[1] // 4: 3 * t[1] // 4] = True
    topo = OG.Topology.uniform(cells, levels)
    pair = OG.PingPongPair(topo)
    lp = OL.LevelParams(levels, 0.8)
    OA.GridAdaptor(topo, lp).update(OA.RefineDriver(np.zeros((0, 2)), static, levels), pair)
    assert np.array_equal(tiles_of(topo), g["tiles"])
    sv = OL.Solver(topo, pair, OL.SolverParams(levels=levels), lp)
    fn = OS.taylor_green_fn(0.05, 64, lp.nu(0), lp.taus, 2)
    OL.set_fields(topo, pair, fn)
    for _ in range(8):
        sv.advance_bounce()
    fields_vs_gold(topo, lambda l: sv.arrays(sv.last_roles(l)[1], l), g, 1e-13)


def test_adapt_walk_golden():
    g = load("adapt_walk")
    topo = OG.Topology.uniform((64, 64), 3)
    pair = OG.PingPongPair(topo)
    ad = OA.GridAdaptor(topo, OL.LevelParams(3, 0.8))
    for step in range(60):
        rep = ad.update(OA.RefineDriver(g[f"pos{step}"], None, 3), pair)
        assert np.array_equal(tiles_of(topo), g[f"tiles{step}"]), step
        for l in range(3):
            assert np.array_equal(ad.streak[l], g[f"streak{step}_{l}"]), (step, l)
        assert list(rep.created) == list(g[f"created{step}"])
        assert list(rep.deleted) == list(g[f"deleted{step}"])
        assert rep.violations == []


@pytest.mark.parametrize("name,scene,steps,vseed", [
    ("taylor_green_2d", S.TAYLOR_GREEN_2D, 20, None),
    ("sand_collapse_2d", S.SAND_COLLAPSE_2D, 20, None),
    ("powder_box_2d", S.POWDER_BOX_2D, 20, None),
    ("dune_2d", S.DUNE_2D, 20, None),
    ("cloud_2d", S.CLOUD_2D, 25, 4),
    ("dune_2d_cadence2_literal", S.DUNE_2D_CADENCE2_LITERAL, 20, None),
    ("powder_box_2d_literal", S.POWDER_BOX_2D_LITERAL, 20, None),
])
def test_scene_golden(name, scene, steps, vseed):
    g = load(name)
    cfg = validated(scene)
    sim = OS.build_scene(cfg.raw)
    if vseed is not None:
        rng = np.random.default_rng(vseed)
        sim.p.v[:] = rng.normal(0, 0.08, sim.p.v.shape).clip(-0.45, 0.45)
    for _ in range(steps):
        sim.step()
    assert np.array_equal(tiles_of(sim.topo), g["tiles"])
    assert list(sim.solver.k) == list(g["k"])
    sv = sim.solver
    fields_vs_gold(sim.topo, lambda l: sv.arrays(sv.last_roles(l)[1] if sv.k[l] else 0, l),
                   g, 1e-11)
    if "px" in g:
        assert np.abs(sim.p.x - g["px"]).max() <= 1e-11
        assert np.abs(sim.p.v - g["pv"]).max() <= 1e-12
        assert np.abs(sim.p.F - g["pF"]).max() <= 1e-11
        assert np.abs(sim.p.vol_corr - g["pvc"]).max() <= 1e-11
    if sim.adaptor is not None:
        for l, st in enumerate(sim.adaptor.streak):
            assert np.array_equal(st, g[f"streak{l}"])
    row = sim.diagnostics[-1]
    assert np.allclose(row["fluid_mom"], g["diag_fluid_mom"], rtol=1e-10, atol=1e-12)
    assert abs(row["sum_phi"] - float(g["diag_sum_phi"])) <= 1e-10 * max(1, abs(float(g["diag_sum_phi"])))
