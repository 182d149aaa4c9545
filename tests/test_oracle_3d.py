"""Pins for the 3D oracle (the reference cannot run 3D, lattice.py:77-79).

(i) exact z-extrusion reduction: a z-invariant 3D state under D3Q27 evolves
    exactly like the 2D oracle (which tests/test_oracle_golden.py pins to the
    reference) — LBM single/multi-level and elastic MPM;
(ii) the reference's own property tests restated in 3D.
"""
import itertools

import numpy as np
import pytest

from oracle import adapt as OA
from oracle import grid as OG
from oracle import lattice as OLat
from oracle import lbm as OL
from oracle import mpm as OM


def rand_fields_2d(nx, ny, seed):
    rng = np.random.default_rng(seed)
    g = {"rho": 1.0 + 0.05 * rng.random((nx, ny)),
         "ux": 0.06 * (rng.random((nx, ny)) - 0.5),
         "uy": 0.06 * (rng.random((nx, ny)) - 0.5)}
    g["sxx"] = g["ux"] ** 2 + 0.01 * rng.random((nx, ny))
    g["sxy"] = g["ux"] * g["uy"] + 0.01 * rng.random((nx, ny))
    g["syy"] = g["uy"] ** 2 + 0.01 * rng.random((nx, ny))
    return g


def load_grid(topo, pair, level, g2d, scale=1):
    cc = topo.cell_coords(level)
    vals = {nm: v[cc[:, 0], cc[:, 1]] for nm, v in g2d.items()}
    if topo.d == 3:
        z = np.zeros(len(cc))
        vals.update({"uz": z, "sxz": z, "syz": z, "szz": z})
    for tree in pair.trees:
        for nm, v in vals.items():
            tree.levels[level][nm][:] = v


@pytest.mark.parametrize("steps", [1, 5])
def test_lbm_extrusion_single_level(steps):
    n, nz = 16, 4
    g = rand_fields_2d(n, n, 3)
    out = {}
    for d, cells in ((2, (n, n)), (3, (n, n, nz))):
        topo = OG.Topology.uniform(cells, 1)
        pair = OG.PingPongPair(topo)
        sv = OL.Solver(topo, pair, OL.SolverParams(levels=1), OL.LevelParams(1, 0.73))
        load_grid(topo, pair, 0, g)
        for _ in range(steps):
            sv.advance_bounce()
        a = sv.arrays(sv.last_roles(0)[1], 0)
        cc = topo.cell_coords(0)
        out[d] = (cc, a)
    cc2, a2 = out[2]
    cc3, a3 = out[3]
    m2 = {tuple(c): i for i, c in enumerate(cc2)}
    idx = np.array([m2[(c[0], c[1])] for c in cc3])
    for nm in OG.moment_names(2):
        assert np.abs(a3[nm] - a2[nm][idx]).max() <= 1e-14, nm
    for nm in ("uz", "sxz", "syz", "szz"):
        assert np.abs(a3[nm]).max() <= 1e-15, nm


def test_lbm_extrusion_multilevel():
    levels = 2
    cells2, nz = (64, 64), 8
    t0 = (16, 16)
    st2 = np.zeros(t0, dtype=bool)
    st2[4:12, 4:12] = True
    st3 = np.repeat(st2[:, :, None], nz // 4, axis=2)
    res = {}
    for d, cells, st in ((2, cells2, st2), (3, cells2 + (nz,), st3)):
        topo = OG.Topology.uniform(cells, levels)
        pair = OG.PingPongPair(topo)
        lp = OL.LevelParams(levels, 0.8)
        OA.GridAdaptor(topo, lp).update(OA.RefineDriver(np.zeros((0, d)), st, levels), pair)
        sv = OL.Solver(topo, pair, OL.SolverParams(levels=levels), lp)
        for l in range(levels):
            g = rand_fields_2d(64 >> l, 64 >> l, 10 + l)
            load_grid(topo, pair, l, g)
        for _ in range(4):
            sv.advance_bounce()
        res[d] = (topo, sv)
    t2, s2 = res[2]
    t3, s3 = res[3]
    # topology is the z-extrusion of the 2D one
    ts2 = t2.tile_set()
    ts3 = t3.tile_set()
    assert {(e[0], e[1], e[2], e[4]) for e in ts3} == ts2
    for l in range(levels):
        a2 = s2.arrays(s2.last_roles(l)[1], l)
        a3 = s3.arrays(s3.last_roles(l)[1], l)
        m2 = {tuple(c): i for i, c in enumerate(t2.cell_coords(l))}
        idx = np.array([m2[(c[0], c[1])] for c in t3.cell_coords(l)])
        for nm in OG.moment_names(2):
            assert np.abs(a3[nm] - a2[nm][idx]).max() <= 1e-13, (l, nm)


def test_mpm_elastic_extrusion():
    rng = np.random.default_rng(8)
    n2, nz = 60, 4
    x2 = rng.random((n2, 2)) * 16 + 8
    v2 = rng.normal(0, 0.03, (n2, 2))
    C2 = rng.normal(0, 0.01, (n2, 2, 2))
    F2 = np.tile(np.eye(2), (n2, 1, 1)) + rng.normal(0, 0.01, (n2, 2, 2))
    mat = OM.SandMaterial(E=0.05)
    t2 = OG.Topology.uniform((32, 32), 1)
    p2 = OM.Particles(n2, 2)
    p2.x, p2.v, p2.C, p2.F = x2.copy(), v2.copy(), C2.copy(), F2.copy()
    p2.m[:] = 0.7
    p2.V0[:] = 0.25
    OM.mpm_step(p2, OM.MpmGrid(t2), 1.0, (0.0, -1e-3), mat, plastic=False)
    t3 = OG.Topology.uniform((32, 32, nz), 1)
    p3 = OM.Particles(n2 * nz, 3)
    for k in range(nz):
        sl = slice(k * n2, (k + 1) * n2)
        p3.x[sl, :2] = x2
        p3.x[sl, 2] = 0.3 + k
        p3.v[sl, :2] = v2
        p3.C[sl, :2, :2] = C2
        p3.F[sl, :2, :2] = F2
    p3.m[:] = 0.7
    p3.V0[:] = 0.25
    OM.mpm_step(p3, OM.MpmGrid(t3), 1.0, (0.0, -1e-3, 0.0), mat, plastic=False)
    for k in range(nz):
        sl = slice(k * n2, (k + 1) * n2)
        assert np.abs(p3.x[sl, :2] - p2.x).max() <= 1e-13
        assert np.abs(p3.v[sl, :2] - p2.v).max() <= 1e-14
        assert np.abs(p3.F[sl, :2, :2] - p2.F).max() <= 1e-13
        assert np.abs(p3.v[sl, 2]).max() <= 1e-15


def test_d3q27_tables():
    lat = OLat.d3q27()
    assert lat.q == 27 and abs(lat.w.sum() - 1.0) <= 1e-15
    assert np.array_equal(lat.c[lat.opp], -lat.c)
    # isotropy: sum w c_a c_b = cs2 delta
    m2 = np.einsum("i,ia,ib->ab", lat.w, lat.c, lat.c)
    assert np.allclose(m2, OLat.CS2 * np.eye(3), atol=1e-15)


@pytest.mark.parametrize("d", [2, 3])
def test_moment_round_trip(d):
    """Reconstruct -> moments returns the stored (rho, u, S) (test_lattice.py:144-155)."""
    lat = OLat.lattice_for(d)
    rng = np.random.default_rng(1)
    n = 200
    rho = 1.0 + 0.1 * (rng.random(n) - 0.5)
    u = [0.1 * (rng.random(n) - 0.5) for _ in range(d)]
    s = {p: u[p[0]] * u[p[1]] + 0.01 * (rng.random(n) - 0.5) for p in OLat.s_pairs(d)}
    fs = [OLat.reconstruct_dir(lat, i, rho, u, s) for i in range(lat.q)]
    r2, m, pi = OLat.moments_from_f(lat, fs)
    assert np.abs(r2 - rho).max() <= 1e-14
    for a in range(d):
        assert np.abs(m[a] / r2 - u[a]).max() <= 1e-14
    for p in OLat.s_pairs(d):
        assert np.abs(pi[p] / r2 - s[p]).max() <= 1e-14


def test_third_order_moment_d3q27():
    """D3Q27 reproduces the Hermite third moments it reconstructs (xyz too)."""
    lat = OLat.d3q27()
    rng = np.random.default_rng(2)
    rho = np.array([1.02])
    u = [np.array([v]) for v in 0.05 * (rng.random(3) - 0.5)]
    s = {p: u[p[0]] * u[p[1]] + 0.003 * (rng.random(1) - 0.5) for p in OLat.s_pairs(3)}
    fs = np.array([OLat.reconstruct_dir(lat, i, rho, u, s)[0] for i in range(27)])
    c = lat.c.astype(float)
    for k, t in enumerate(OLat.h3_triples(3)):
        a3 = sum(OLat.h3(c[i], t) * fs[i] for i in range(27))
        norm = OLat.CS6 if len(set(t)) == 3 else 2.0 * OLat.CS6   # sum_i w_i H_t(c_i)^2
        want = rho[0] * OLat.gamma(t, u, s)[0] * lat.h3coef[k] * norm
        assert abs(a3 - want) <= 1e-15
        # with the Hermite coefficient every component reproduces rho * Gamma
        assert abs(a3 - rho[0] * OLat.gamma(t, u, s)[0]) <= 1e-15


def test_mass_conserved_periodic_3d():
    topo = OG.Topology.uniform((8, 8, 8), 1)
    pair = OG.PingPongPair(topo)
    sv = OL.Solver(topo, pair, OL.SolverParams(levels=1), OL.LevelParams(1, 0.8))
    pos = topo.cell_coords(0).astype(float)
    k = 2 * np.pi / 8
    OL.set_fields(topo, pair, lambda p, l: {"rho": 1 + 0.01 * np.sin(k * p[:, 2]),
                                             "ux": 0.03 * np.sin(k * p[:, 1]),
                                             "uz": 0.02 * np.cos(k * p[:, 0])})
    m0 = pair.trees[0].levels[0]["rho"].sum()
    for _ in range(40):
        sv.advance_bounce()
    m1 = sv.arrays(sv.last_roles(0)[1], 0)["rho"].sum()
    assert abs(m1 - m0) / m0 <= 1e-13
    del pos


def test_rescale_round_trip_3d():
    rng = np.random.default_rng(0)
    u = [0.1 * (rng.random(1000) - 0.5) for _ in range(3)]
    s = {p: u[p[0]] * u[p[1]] + 0.01 * (rng.random(1000) - 0.5) for p in OLat.s_pairs(3)}
    up = OL.rescale_s(s, u, OL.kappa_up(0.8, 0.65, "derived"))
    back = OL.rescale_s(up, u, OL.kappa_down(0.8, 0.65, "derived"))
    assert max(np.abs(back[p] - s[p]).max() for p in s) <= 1e-15


def test_adapt_3d_settles_to_brute_force():
    rng = np.random.default_rng(5)
    cells = (32, 32, 32)
    levels = 3
    topo = OG.Topology.uniform(cells, levels)
    pair = OG.PingPongPair(topo)
    ad = OA.GridAdaptor(topo, OL.LevelParams(levels, 0.8))
    pos = rng.random((2, 3)) * 28 + 2
    unchanged, checked = 0, 0
    for _ in range(30):
        if rng.random() < 0.6:
            pos = np.clip(pos + rng.normal(0, 2.0, pos.shape), 0.5, 31.5)
            unchanged = 0
        else:
            unchanged += 1
        rep = ad.update(OA.RefineDriver(pos, None, levels), pair)
        assert rep.violations == []
        if unchanged >= 2:
            checked += 1
            assert topo.tile_set() == OA.brute_force_grid(OA.RefineDriver(pos, None, levels),
                                                          cells, levels)
    assert checked > 0


def test_brute_force_3d_one_particle():
    d = OA.RefineDriver(np.array([[10.5, 13.2, 13.9]]), None, 3)
    ref = OA.brute_force_grid(d, (64, 64, 64), 3)
    lvl0 = {e[1:4] for e in ref if e[0] == 0}
    assert lvl0 == set(itertools.product(range(0, 6), range(0, 6), range(0, 6)))
    topo = OG.Topology((64, 64, 64), 3)
    OA.apply_tile_set(topo, ref)
    topo.validate_coverage()
    topo.validate_two_tile_overlap()
