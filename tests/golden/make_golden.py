"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the builder container (needs /root/reference/pkg/src on the path):

    python tests/golden/make_golden.py

Each fixture stores, after N reference steps of a scene, the tile set, the
streak bitmaps (when an adaptor exists), every field of every level keyed by
cell coordinates (sorted lexicographically, so slot order never matters) and
the particle state.  The fixtures travel to the GPU box; the reference does
not.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(HERE))

from mlbm import sparse_grid as RG  # noqa: E402
from mlbm.harness import config as RCF  # noqa: E402
from mlbm.harness import cases as RC  # noqa: E402
from mlbm.harness.reference import uniform_solver  # noqa: E402
from mlbm.lattice import CS2, D2Q9, reconstruct_fields  # noqa: E402

import scenes as S  # noqa: E402


def dump_sim_state(topo, arrays_fn, levels):
    out = {}
    ts = sorted(topo.tile_set())
    out["tiles"] = np.array(ts, dtype=np.int64).reshape(-1, 4)
    for l in range(levels):
        cc = topo.cell_coords(l)
        if not len(cc):
            out[f"L{l}_coords"] = np.zeros((0, 2), dtype=np.int64)
            continue
        order = np.lexsort(cc.T[::-1])
        out[f"L{l}_coords"] = cc[order]
        a = arrays_fn(l)
        for nm in RG.FIELD_NAMES:
            out[f"L{l}_{nm}"] = np.asarray(a[nm])[order]
    return out


def scene_fixture(name, scene, steps, velocity_seed=None):
    cfg = RCF.validate_scene(scene)
    sim = RCF.build_scene(cfg)
    if velocity_seed is not None:
        rng = np.random.default_rng(velocity_seed)
        sim.particles.v[:] = rng.normal(0, 0.08, sim.particles.v.shape).clip(-0.45, 0.45)
    for _ in range(steps):
        sim.step()
    sv = sim.solver
    L = sim.topology.levels
    out = dump_sim_state(sim.topology,
                         lambda l: sv.arrays(sv.last_roles(l)[1] if sv.k[l] else 0, l), L)
    out["k"] = np.array(sv.k)
    if len(sim.particles):
        p = sim.particles
        out.update(px=p.x, pv=p.v, pC=p.C, pF=p.F, pvc=p.vol_corr)
    if sim.adaptor is not None:
        for l, st in enumerate(sim.adaptor.streak):
            out[f"streak{l}"] = st
    row = sim.diagnostics[-1]
    out["diag_fluid_mom"] = np.array(row.fluid_mom)
    out["diag_sediment_mom"] = np.array(row.sediment_mom)
    out["diag_sum_phi"] = np.array(row.sum_phi)
    out["diag_eps_min"] = np.array(row.eps_min)
    out["steps"] = np.array(steps)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "saved", {k: v.shape for k, v in out.items() if k.startswith("L0_rho")})


def one_step_golden():
    """Random 16^2 state, one stream+collide (test_solver.py:206-254 inputs)."""
    nx = ny = 16
    topo, pair, solver = uniform_solver((nx, ny), 0.73)
    rng = np.random.default_rng(3)
    g = {"rho": 1.0 + 0.05 * rng.random((nx, ny)),
         "ux": 0.06 * (rng.random((nx, ny)) - 0.5),
         "uy": 0.06 * (rng.random((nx, ny)) - 0.5)}
    g["sxx"] = g["ux"] * g["ux"] + 0.01 * rng.random((nx, ny))
    g["sxy"] = g["ux"] * g["uy"] + 0.01 * rng.random((nx, ny))
    g["syy"] = g["uy"] * g["uy"] + 0.01 * rng.random((nx, ny))
    cc = topo.cell_coords(0)
    for tree in pair.trees:
        for nm, v in g.items():
            tree.levels[0][nm][:] = v[cc[:, 0], cc[:, 1]]
    solver.advance_bounce()
    out = dump_sim_state(topo, lambda l: solver.arrays(solver.last_roles(l)[1], l), 1)
    out.update({f"in_{k}": v for k, v in g.items()})
    out["tau"] = np.array(0.73)
    np.savez_compressed(os.path.join(HERE, "one_step_16.npz"), **out)
    print("one_step_16 saved")


def multilevel_tg(levels):
    topo, pair, solver = RC.refined_multilevel((64, 64), levels, 0.8)
    nu = solver.level_params.nu(0)
    fn, _ = RC.taylor_green_fields(0.05, 64, nu, solver.level_params.taus)
    RC.set_fields(topo, pair, lambda px, py, l: fn(px, py, l))
    for _ in range(8):
        solver.advance_bounce()
    out = dump_sim_state(topo, lambda l: solver.arrays(solver.last_roles(l)[1], l), levels)
    np.savez_compressed(os.path.join(HERE, f"tg_refined_L{levels}.npz"), **out)
    print(f"tg_refined_L{levels} saved")


def adapt_walk():
    """Random particle walk through GridAdaptor.update: tile set + streaks per
    update (the fuzz of cases.py:371-411 / test_adapt.py:118-147)."""
    from mlbm.adapt import GridAdaptor, RefineDriver
    from mlbm.solver import LevelParams
    from mlbm.sparse_grid import PingPongPair, Topology
    rng = np.random.default_rng(0)
    topo = Topology.uniform((64, 64), levels=3)
    pair = PingPongPair(topo)
    ad = GridAdaptor(topo, LevelParams(3, 0.8))
    pos = rng.random((3, 2)) * 60 + 2
    out = {}
    for step in range(60):
        if rng.random() < 0.6:
            pos = np.clip(pos + rng.normal(0, 2.0, pos.shape), 0.5, 63.5)
        rep = ad.update(RefineDriver(positions=pos, levels=3), pair)
        out[f"pos{step}"] = pos.copy()
        out[f"tiles{step}"] = np.array(sorted(topo.tile_set()), dtype=np.int64).reshape(-1, 4)
        for l in range(3):
            out[f"streak{step}_{l}"] = ad.streak[l].copy()
        out[f"created{step}"] = np.array(rep.created)
        out[f"deleted{step}"] = np.array(rep.deleted)
    np.savez_compressed(os.path.join(HERE, "adapt_walk.npz"), **out)
    print("adapt_walk saved")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "variants":
        scene_fixture("dune_2d_cadence2_literal", S.DUNE_2D_CADENCE2_LITERAL, 20)
        scene_fixture("powder_box_2d_literal", S.POWDER_BOX_2D_LITERAL, 20)
        sys.exit(0)
    one_step_golden()
    multilevel_tg(2)
    multilevel_tg(3)
    adapt_walk()
    scene_fixture("taylor_green_2d", S.TAYLOR_GREEN_2D, 20)
    scene_fixture("sand_collapse_2d", S.SAND_COLLAPSE_2D, 20)
    scene_fixture("powder_box_2d", S.POWDER_BOX_2D, 20)
    scene_fixture("dune_2d", S.DUNE_2D, 20)
    scene_fixture("cloud_2d", S.CLOUD_2D, 25, velocity_seed=4)
    scene_fixture("dune_2d_cadence2_literal", S.DUNE_2D_CADENCE2_LITERAL, 20)
    scene_fixture("powder_box_2d_literal", S.POWDER_BOX_2D_LITERAL, 20)
