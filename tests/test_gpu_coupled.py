"""GPU parity of the full coupled step (LBM levels + exchange + MPM + powder +
block maintenance) against the oracle, 2D and 3D, fp64.

Gate A: integer topology bit-exact after every step
(tile sets and streaks), fields / particles within 1e-9 absolute (the
only difference is fp64 atomic summation order in P2G).
"""
import numpy as np
import pytest
import torch

import scenes as S
from oracle import scene as OS

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2603_14982_b200")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def build_both(scene_dict):
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    cfg = validate_scene(scene_dict)
    dsim = build_scene(cfg)
    osim = OS.build_scene(cfg.raw, heightmap=cfg.heightmap())
    return osim, dsim


def field_diff(osim, dsim):
    worst = 0.0
    d = dsim.d
    names = B.field_names(d)
    for l in range(dsim.topology.levels):
        ot, dt = osim.topo, dsim.topology
        if not dt.n_tiles(l):
            continue
        ow = osim.solver.last_roles(l)[1] if osim.solver.k[l] else 0
        dw = dsim.solver.last_roles(l)[1] if dsim.solver.k[l] else 0
        assert ow == dw ^ dsim.solver.flip[l]   # the device may have swapped the trees
        oa = osim.solver.arrays(ow, l)
        da = dsim.solver.arrays(dw, l)
        dmap = {tuple(c): i for i, c in enumerate(dt.cell_coords(l))}
        perm = np.array([dmap[tuple(c)] for c in ot.cell_coords(l)])
        for nm in names:
            worst = max(worst, float(np.abs(da[nm].cpu().numpy()[perm] - oa[nm]).max()))
    return worst


def particle_diff(osim, dsim):
    if not len(osim.p):
        return 0.0
    dx = np.abs(dsim.particles.x.cpu().numpy() - osim.p.x).max()
    dv = np.abs(dsim.particles.v.cpu().numpy() - osim.p.v).max()
    dF = np.abs(dsim.particles.F.cpu().numpy() - osim.p.F).max()
    return float(max(dx, dv, dF))


def set_level0_field(osim, dsim, name, fn):
    """Write fn(coords) into field `name` of level 0 in both trees of both
    sims (coordinate-keyed: the device stores cells in its own slot order)."""
    oc = osim.topo.cell_coords(0).astype(float)
    dc = dsim.topology.cell_coords(0).astype(float)
    for t in range(2):
        osim.solver.arrays(t, 0)[name][:] = fn(oc)
        dsim.solver.arrays(t, 0)[name] = fn(dc)


def run_and_compare(scene_dict, steps, tol=1e-9, check_streaks=True, prepare=None):
    _need_gpu()
    osim, dsim = build_both(scene_dict)
    if prepare is not None:
        prepare(osim, dsim)
    assert dsim.topology.tile_set() == osim.topo.tile_set()
    for s in range(steps):
        osim.step()
        dsim.step()
        assert dsim.topology.tile_set() == osim.topo.tile_set(), f"tile sets differ at step {s}"
        if check_streaks and osim.adaptor is not None:
            for l, (a, b) in enumerate(zip(dsim.adaptor.streak, osim.adaptor.streak)):
                assert np.array_equal(a, b), f"streaks differ at step {s} level {l}"
    fd = field_diff(osim, dsim)
    pd = particle_diff(osim, dsim)
    assert fd <= tol, f"fields differ by {fd}"
    assert pd <= tol, f"particles differ by {pd}"
    od = osim.diagnostics[-1]
    dd = dsim.diagnostics[-1]
    assert np.allclose(dd.fluid_mom, od["fluid_mom"], rtol=1e-9, atol=1e-12)
    assert np.allclose(dd.sediment_mom, od["sediment_mom"], rtol=1e-9, atol=1e-12)
    assert len(dd.drag_impulse) == len(od["drag_impulse"]) == dsim.d
    assert np.allclose(dd.drag_impulse, od["drag_impulse"], rtol=1e-9, atol=1e-12), (dd.drag_impulse, od["drag_impulse"])
    assert dd.tiles == od["tiles"]
    assert abs(dd.sum_phi - od["sum_phi"]) <= 1e-9 * max(1.0, abs(od["sum_phi"]))
    assert abs(dd.eps_min - od["eps_min"]) <= 1e-12
    return osim, dsim


def test_taylor_green_scene_2d():
    run_and_compare(S.TAYLOR_GREEN_2D, 10)


def test_sand_collapse_2d():
    run_and_compare(S.SAND_COLLAPSE_2D, 15)


def test_powder_box_2d():
    run_and_compare(S.POWDER_BOX_2D, 15)


def test_dune_2d_three_levels():
    run_and_compare(S.DUNE_2D, 12)


def test_dune_2d_cadence2_paper_literal():
    """mpm_cadence = 2 (the held hook on odd steps, coupling.py:454-465), the
    paper-literal S rescale and average upward transfer (solver.py:41-52,
    543-548) on three levels with adaptation: gate A (the oracle is pinned to
    the reference on this scene by tests/golden/dune_2d_cadence2_literal.npz)."""
    run_and_compare(S.DUNE_2D_CADENCE2_LITERAL, 12)


@pytest.mark.parametrize("latest_only", [False, True])
def test_cadence2_churn_3d(latest_only):
    """Held hook with topology changes between MPM steps in 3D, with the
    single-tree level-0 rebuild requested (it must fall back to both trees
    when mpm_cadence > 1)."""
    sc = S.scene(S.CLOUD_3D_SMALL, runtime__mpm_cadence=2)
    _need_gpu()
    osim, dsim = build_both(sc)
    if latest_only:
        dsim.latest_only_min_cells = 0
    rng = np.random.default_rng(23)
    v = rng.normal(0, 0.08, (len(osim.p), 3)).clip(-0.45, 0.45)
    osim.p.v[:] = v
    dsim.particles.v = v
    changes = 0
    for s in range(12):
        osim.step()
        dsim.step()
        assert dsim.topology.tile_set() == osim.topo.tile_set(), f"step {s}"
        if not osim.last_report.noop:
            changes += 1
    assert changes > 0
    assert field_diff(osim, dsim) <= 1e-9
    assert particle_diff(osim, dsim) <= 1e-9


def test_powder_box_2d_paper_literal_sign():
    run_and_compare(S.POWDER_BOX_2D_LITERAL, 12)


def test_h3_xyz_paper_literal_3d():
    """fluid.h3_xyz = paper_literal (PAPER.md's uniform 1/(2 cs^6) on Gamma_xyz)."""
    run_and_compare(S.scene(S.DUNE_3D_SMALL, fluid__h3_xyz="paper_literal"), 4)


@pytest.mark.parametrize("latest_only", [False, True])
def test_cloud_2d_block_churn(latest_only):
    """Per-step block churn; latest_only forces the single-tree level-0
    rebuild (on by default only for level 0s of >= 4M cells)."""
    sc = S.scene(S.CLOUD_2D)
    osim, dsim = build_both(sc)
    if latest_only:
        dsim.latest_only_min_cells = 0
    rng = np.random.default_rng(4)
    n = len(osim.p)
    v = rng.normal(0, 0.08, (n, 2)).clip(-0.45, 0.45)
    osim.p.v[:] = v
    dsim.particles.v = v
    changes = 0
    for s in range(25):
        osim.step()
        dsim.step()
        assert dsim.topology.tile_set() == osim.topo.tile_set(), f"step {s}"
        for a, b in zip(dsim.adaptor.streak, osim.adaptor.streak):
            assert np.array_equal(a, b)
        if not osim.last_report.noop:
            changes += 1
    assert changes > 0
    assert field_diff(osim, dsim) <= 1e-9
    assert particle_diff(osim, dsim) <= 1e-9


def test_column_3d_two_levels():
    run_and_compare(S.COLUMN_3D_SMALL, 8)


def test_cloud_3d_churn_latest_only_rebuild():
    """3D dispersed cloud with topology changes through the graph path and the
    single-tree level-0 rebuild forced on: gate A against the oracle."""
    _need_gpu()
    osim, dsim = build_both(S.scene(S.CLOUD_3D_SMALL))
    dsim.latest_only_min_cells = 0
    rng = np.random.default_rng(21)
    v = rng.normal(0, 0.08, (len(osim.p), 3)).clip(-0.45, 0.45)
    osim.p.v[:] = v
    dsim.particles.v = v
    changes = 0
    for s in range(12):
        osim.step()
        dsim.step()
        assert dsim.topology.tile_set() == osim.topo.tile_set(), f"step {s}"
        if not osim.last_report.noop:
            changes += 1
    assert changes > 0
    assert field_diff(osim, dsim) <= 1e-9
    assert particle_diff(osim, dsim) <= 1e-9


def test_fp32_dense_column_mode5():
    """Dense sampling (8 per cell) selects the 4-round P2G blocks (mode 5):
    gate B against the fp64 oracle after 15 steps."""
    _need_gpu()
    sc = S.scene(S.COLUMN_3D_SMALL, runtime__dtype="f32", particles__per_cell=8)
    osim, dsim = build_both(sc)
    assert dsim.p2g_mode == 5
    for _ in range(15):
        osim.step()
        dsim.step()
    assert dsim.topology.tile_set() == osim.topo.tile_set()
    x = dsim.particles.x.cpu().numpy()
    v = dsim.particles.v.double().cpu().numpy()
    rx = np.linalg.norm(x - osim.p.x) / np.linalg.norm(osim.p.x)
    rv = np.linalg.norm(v - osim.p.v) / max(np.linalg.norm(osim.p.v), 1e-30)
    assert rx <= 1e-5, rx
    assert rv <= 1e-4, rv


def test_dune_3d_inlet_outlet():
    run_and_compare(S.DUNE_3D_SMALL, 6)


def test_sandstorm_3d_three_levels():
    """C3 at test size: three levels, log inlet, outlets, z periodic, fp64."""
    run_and_compare(S.SANDSTORM_3D_SMALL, 6)


def test_fp32_sandstorm_3d_three_levels():
    """Gate B on the three-level path: fp32 device vs fp64 oracle."""
    _need_gpu()
    sc = S.scene(S.SANDSTORM_3D_SMALL, runtime__dtype="f32")
    osim, dsim = build_both(sc)
    for _ in range(10):
        osim.step()
        dsim.step()
        assert dsim.topology.tile_set() == osim.topo.tile_set()
    x = dsim.particles.x.cpu().numpy()
    v = dsim.particles.v.double().cpu().numpy()
    rx = np.linalg.norm(x - osim.p.x) / np.linalg.norm(osim.p.x)
    rv = np.linalg.norm(v - osim.p.v) / max(np.linalg.norm(osim.p.v), 1e-30)
    assert rx <= 1e-5, rx
    assert rv <= 1e-4, rv


def test_powder_3d_solids():
    run_and_compare(S.POWDER_3D_SMALL, 6)


@pytest.mark.parametrize("d", [2, 3])
def test_powder_over_sand_exchange_fp64(d):
    """A powder fraction of O(1e-2) over the sand (eta > phi > 0): the
    exchange's neighbour eps for grad eps must use the raw eta, not eta_eff
    written by another thread (coupling.py:127,159-182); gate A."""
    sc = S.scene(S.POWDER_BOX_2D if d == 2 else S.POWDER_3D_SMALL)

    def phi0(c):
        return 0.03 * (1.0 + np.sin(0.37 * c[:, 0] + 0.21 * c[:, 1])) * (c[:, 1] < 24)

    run_and_compare(sc, 6, prepare=lambda o, dd: set_level0_field(o, dd, "phi", phi0))


def test_fp32_column_3d_short():
    """Gate B on the coupled path: fp32 device vs fp64 oracle after 20 steps."""
    _need_gpu()
    sc = S.scene(S.COLUMN_3D_SMALL, runtime__dtype="f32")
    osim, dsim = build_both(sc)
    for _ in range(20):
        osim.step()
        dsim.step()
    assert dsim.topology.tile_set() == osim.topo.tile_set()
    x = dsim.particles.x.cpu().numpy()
    v = dsim.particles.v.double().cpu().numpy()
    rx = np.linalg.norm(x - osim.p.x) / np.linalg.norm(osim.p.x)
    rv = np.linalg.norm(v - osim.p.v) / max(np.linalg.norm(osim.p.v), 1e-30)
    assert rx <= 1e-5, rx
    assert rv <= 1e-4, rv


def test_avalanche_terrain_3d_small(tmp_path):
    """Config 4 ingredients at test size: two levels, a terrain heightmap under
    a granular slab (solids near the refined region), outlets, powder on —
    gate A against the oracle (tile sets, streaks, fields, particles)."""
    hf = S.terrain_heightfield((32, 32, 32), str(tmp_path / "terrain.npy"))
    sc = {"domain": {"cells": [32, 32, 32], "levels": 2},
          "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -1e-4, 0.0]},
          "boundaries": {"x_min": "outlet", "x_max": "outlet", "y_min": "wall",
                         "y_max": "outlet", "z_min": "outlet", "z_max": "outlet",
                         "heightfield": hf},
          "materials": {"density_ratio": 40.0, "E": 0.08},
          "particles": {"blocks": [[8.0, 4.0, 8.0, 24.0, 8.0, 24.0]], "per_cell": 2},
          "powder": {"enabled": True, "entrain": 0.02, "diffusion": 0.05},
          "runtime": {"seed": 7}}
    run_and_compare(sc, 6)


def test_fp32_powder_3d_short():
    """Gate B with powder + entrainment (the fp32 stress raster in the P2G
    layout and the shared-corner RK3 backtrace): fp32 device vs fp64 oracle."""
    _need_gpu()
    sc = S.scene(S.POWDER_3D_SMALL, runtime__dtype="f32")
    osim, dsim = build_both(sc)
    for _ in range(12):
        osim.step()
        dsim.step()
    assert dsim.topology.tile_set() == osim.topo.tile_set()
    x = dsim.particles.x.cpu().numpy()
    rx = np.linalg.norm(x - osim.p.x) / np.linalg.norm(osim.p.x)
    assert rx <= 1e-5, rx
    ow = osim.solver.last_roles(0)[1] if osim.solver.k[0] else 0
    dw = dsim.solver.last_roles(0)[1] if dsim.solver.k[0] else 0
    oa = osim.solver.arrays(ow, 0)["phi"]
    da = dsim.solver.arrays(dw, 0)["phi"].double().cpu().numpy()
    dmap = {tuple(c): i for i, c in enumerate(dsim.topology.cell_coords(0))}
    perm = np.array([dmap[tuple(c)] for c in osim.topo.cell_coords(0)])
    # phi is a volume fraction; in this small scene the entrainment source is
    # driven by near-zero stresses (phi ~ 1e-12 after 12 steps, fp32 round-off
    # level), so the gate is absolute: within 1e-9 of the fp64 oracle
    assert np.abs(oa).max() > 0.0
    assert np.abs(da[perm] - oa).max() <= 1e-9


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_powder_entrainment_stressed_column(dtype):
    """Entrainment from a collapsing (stressed) column: fp64 gate A on phi
    (<= 1e-9 relative L2); fp32 (surface-restricted stress raster in the P2G
    layout) within 5e-3 relative L2 of the fp64 oracle: phi ~ 1e-8 here and
    the source's surface / eta thresholds amplify fp32 round-off."""
    _need_gpu()
    sc = S.scene(S.COLUMN_3D_SMALL, runtime__dtype=dtype, powder__enabled=True,
                 powder__entrain=0.02)
    osim, dsim = build_both(sc)
    for _ in range(20):
        osim.step()
        dsim.step()
    assert dsim.topology.tile_set() == osim.topo.tile_set()
    ow = osim.solver.last_roles(0)[1] if osim.solver.k[0] else 0
    dw = dsim.solver.last_roles(0)[1] if dsim.solver.k[0] else 0
    oa = osim.solver.arrays(ow, 0)["phi"]
    da = dsim.solver.arrays(dw, 0)["phi"].double().cpu().numpy()
    dmap = {tuple(c): i for i, c in enumerate(dsim.topology.cell_coords(0))}
    perm = np.array([dmap[tuple(c)] for c in osim.topo.cell_coords(0)])
    assert np.abs(oa).max() > 0.0
    rel = np.linalg.norm(da[perm] - oa) / np.linalg.norm(oa)
    assert rel <= (1e-9 if dtype == "f64" else 5e-3), rel


def test_stress_raster_fp32_kernels_agree():
    """The fp32 stress raster in the P2G layout (per-warp node boxes) equals
    the per-particle atomic kernel within fp32 summation order."""
    _need_gpu()
    import os
    from paper_2603_14982_b200 import _lib as L
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    # a collapsing column with powder on: the particles deform within a few
    # steps (the powder box stays at F = I to fp32 precision for long)
    sim = build_scene(validate_scene(S.scene(S.COLUMN_3D_SMALL, runtime__dtype="f32",
                                             powder__enabled=True, powder__entrain=0.02)))
    for _ in range(40):
        sim.step()
        dF = (sim.particles.F.double() - torch.eye(3, dtype=torch.float64, device="cuda")).abs().max()
        if dF.item() > 1e-3:
            break
    lib, s = L.lib(), L.stream_handle()
    p, grid, mat = sim.particles, sim.grid, sim.material
    lv0 = grid.level0()
    R = grid.R
    out = []
    for atomic in (True, False):
        if atomic:
            os.environ["MLBM_STRESS_ATOMIC"] = "1"
        try:
            grid.ras[R["sig"]:R["etae"]].zero_()
            L.check(lib.mlbm_stress_raster(L.C.byref(lv0), len(p), L.ptr(p.xd), L.ptr(p.pd),
                                           p.pd.stride(0), mat.lam, mat.mu, mat.alpha,
                                           L.ptr(grid.ras), grid.ras.stride(0), 0,
                                           L.ptr(grid._err), s), "stress_raster")
            torch.cuda.synchronize()
        finally:
            os.environ.pop("MLBM_STRESS_ATOMIC", None)
        out.append(grid.ras[R["sig"]:R["etae"], :grid._live()].double().clone())
    # the surface-restricted raster (the production call) equals the full one
    # at every entrainment surface cell
    surf = torch.zeros(grid.ras.shape[1], dtype=torch.float32, device="cuda")
    grid.ras[R["sig"]:R["etae"]].zero_()
    L.check(lib.mlbm_stress_raster_surface(L.C.byref(lv0), len(p), L.ptr(p.xd), L.ptr(p.pd),
                                           p.pd.stride(0), mat.lam, mat.mu, mat.alpha,
                                           L.ptr(grid.ras), grid.ras.stride(0),
                                           float(sim.powder.eta_surface), L.ptr(surf), 0,
                                           L.ptr(grid._err), s), "stress_raster_surface")
    torch.cuda.synchronize()
    restricted = grid.ras[R["sig"]:R["etae"], :grid._live()].double().clone()
    grid.raise_pending()
    scale = out[0].abs().amax(dim=1, keepdim=True).clamp_min(1e-30)
    assert out[0].abs().max().item() > 0.0
    assert ((out[1] - out[0]).abs() / scale).max().item() <= 1e-5
    m = surf[:grid._live()] == 2.0          # the entrainment surface cells
    assert int(m.sum().item()) > 0
    assert int((surf[:grid._live()] == 1.0).sum().item()) > 0
    assert ((restricted[:, m] - out[0][:, m]).abs() / scale).max().item() <= 1e-5


@pytest.mark.parametrize("dtype,scene", [("f32", "column"), ("f64", "column"),
                                         ("f32", "cloud"), ("f32", "cloud_unsorted")])
def test_p2g_modes_agree(dtype, scene):
    """Every P2G variant (atomic, block smem, warp registers, cell lanes,
    per-warp box copies) rasterises the same particle set: fp64 within
    summation-order noise, fp32 within 1e-5 of the row maximum.  The dense
    column fits the block node boxes; the 1-per-cell cloud overflows them
    (per-warp boxes), and unsorted it overflows those too (global atomics)."""
    _need_gpu()
    from paper_2603_14982_b200 import _lib as L
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    base = S.COLUMN_3D_SMALL if scene == "column" else S.CLOUD_3D_SMALL
    sim = build_scene(validate_scene(S.scene(base, runtime__dtype=dtype)))
    for _ in range(3):
        sim.step()
    lib, s = L.lib(), L.stream_handle()
    p, grid, mat = sim.particles, sim.grid, sim.material
    lv0 = grid.level0()
    n, ps = len(p), p.pd.stride(0)
    dcode = 1 if dtype == "f64" else 0
    xa, pa, ida, ws = p.scratch()
    L.check(lib.mlbm_particle_sort(L.C.byref(lv0), n, L.ptr(p.xd), L.ptr(p.pd), L.ptr(p.pid), ps,
                                   L.ptr(xa), L.ptr(pa), L.ptr(ida), dcode, L.ptr(ws), ws.numel(),
                                   s), "sort")
    if scene == "cloud_unsorted":
        perm = torch.randperm(n, generator=torch.Generator().manual_seed(3)).cuda()
        xa[:, :n] = xa[:, :n][:, perm].clone()
        pa[:, :n] = pa[:, :n][:, perm].clone()
    nacc = grid.R["nacc"]
    out = []
    for mode in range(6):
        grid.clear()
        L.check(lib.mlbm_p2g(L.C.byref(lv0), n, L.ptr(xa), L.ptr(pa), ps, mat.lam, mat.mu,
                             mat.alpha, L.ptr(grid.ras), grid.ras.stride(0), dcode, mode,
                             L.ptr(grid._err), s), "p2g")
        out.append(grid.ras[:nacc, :grid._live()].double().clone())
    grid.raise_pending()
    scale = out[0].abs().amax(dim=1, keepdim=True).clamp_min(1e-300)
    tol = 1e-12 if dtype == "f64" else 1e-5
    for mode in range(1, 6):
        assert ((out[mode] - out[0]).abs() / scale).max().item() <= tol, mode


def test_host_mirror_round_trip_matches_resident_run():
    """host_io.HostMirror (host-owned particle state, chunked two-stream
    transfers) gives the same trajectory as the device-resident run."""
    _need_gpu()
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    from paper_2603_14982_b200.host_io import HostMirror
    cfg = validate_scene(S.scene(S.COLUMN_3D_SMALL, runtime__dtype="f32"))
    a = build_scene(cfg)
    b = build_scene(cfg)
    m = HostMirror([b.particles.xd, b.particles.pd], chunks=5)
    for _ in range(4):
        a.step()
        m.upload()
        b.step()
        m.download()
    m.synchronize()
    torch.cuda.synchronize()
    # the host copies are exactly the device state after the last download
    assert torch.equal(m.host[0], b.particles.xd.cpu())
    assert torch.equal(m.host[1], b.particles.pd.cpu())
    # and the trajectory matches the resident run up to fp32 atomic order
    ra = a.particles.xd.cpu().numpy()
    rb = m.host[0].numpy()
    assert np.linalg.norm(ra - rb) / np.linalg.norm(ra) <= 1e-6
    # an upload after host-side edits lands on the device unchanged
    m.host[1][0].mul_(2.0)
    m.upload()
    torch.cuda.synchronize()
    assert torch.equal(b.particles.pd.cpu(), m.host[1])


def test_c2_fp32_long_run_stable():
    """The bench workload (C2, fp32, graph path) for 400 steps: no device
    error, dozens of topology changes through the rebuild graph with few
    captures, particle mass conserved, invariants clean."""
    _need_gpu()
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    sim = build_scene(validate_scene(S.COLUMN_3D_C2))
    m0 = float(sim.particles.m.double().sum().item())
    for _ in range(400):
        sim.step()
    assert sim.topology_changes >= 20
    assert sim.graph_captures <= 16
    assert abs(float(sim.particles.m.double().sum().item()) - m0) <= 1e-6 * m0
    assert sim.last_report is not None and sim.last_report.violations == []
    row = sim.diagnostics[-1]
    assert np.all(np.isfinite(row.fluid_mom)) and np.all(np.isfinite(row.sediment_mom))


def test_frame_outputs_match_reference_frame():
    """write_frame from device buffers after 3 steps of the 2D dune scene
    reads back to the reference's own frame files (the outputs fixture)
    within fp64 summation noise; the particle dump and 'stored' map match
    exactly in structure."""
    _need_gpu()
    import os
    import tempfile
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    from paper_2603_14982_b200.harness import outputs as O
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                             "outputs_dune_2d.npz"))
    sc = S.scene(S.DUNE_2D, runtime__mpm_cadence=1)
    sc.setdefault("outputs", {}).update({"fields": True, "particles": True, "quicklook": True})
    cfg = validate_scene(sc)
    sim = build_scene(cfg)
    for _ in range(3):
        sim.step()
    with tempfile.TemporaryDirectory() as d:
        O.write_frame(d, 7, sim, cfg)
        for l in range(int(g["levels"])):
            back = O.read_vtk_level(os.path.join(d, f"frame_00007_l{l}.vtk"))
            assert np.array_equal(back["stored"], g[f"L{l}_stored"]), l
            for nm in ("rho", "ux", "uy", "eps", "phi"):
                assert np.abs(back[nm] - g[f"L{l}_{nm}"]).max() <= 1e-10, (l, nm)
        x, v, m = O.read_particles(os.path.join(d, "frame_00007_particles.bin"))
        assert np.abs(x - g["px"]).max() <= 1e-10 and np.abs(v - g["pv"]).max() <= 1e-10
        assert np.array_equal(m, g["pm"])
        assert os.path.getsize(os.path.join(d, "frame_00007_speed.ppm")) == \
            len(g["file_frame_00007_speed.ppm"])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("swap", [False, True])
def test_checkpoint_resume_continues_the_run(dtype, swap, tmp_path):
    """Run, checkpoint, run on; a fresh simulation loaded from the checkpoint
    continues identically (topology and streaks exact, fields / particles to
    atomic-order noise) through topology changes."""
    _need_gpu()
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    from paper_2603_14982_b200.harness.checkpoint import load_checkpoint, save_checkpoint
    sc = S.scene(S.CLOUD_3D_SMALL, runtime__dtype=dtype)

    def fresh():
        sim = build_scene(validate_scene(sc))
        x = sim.particles.x.cpu().numpy()
        v = np.zeros_like(x)
        v[:, 0] = np.where(x[:, 0] < 48.0, 0.3, -0.3)
        sim.particles.v = v
        if swap:
            # latest-only level-0 rebuild with swapped trees (the C4 path)
            sim.latest_only_min_cells = 0
        return sim

    a = fresh()
    flipped = False
    for _ in range(6):
        a.step()
        flipped |= a.solver.flip[0] == 1
    path = str(tmp_path / "ck.pt")
    save_checkpoint(path, a)
    for _ in range(8):
        a.step()
        flipped |= a.solver.flip[0] == 1
    assert flipped == swap
    b = fresh()
    load_checkpoint(path, b)
    for _ in range(8):
        b.step()
    assert a.topology_changes > 0
    assert b.topology.tile_set() == a.topology.tile_set()
    for sa, sb in zip(a.adaptor.streak, b.adaptor.streak):
        assert np.array_equal(sa, sb)
    tol = 1e-10 if dtype == "f64" else 1e-4
    assert np.abs(b.particles.x.cpu().numpy() - a.particles.x.cpu().numpy()).max() <= tol
    assert np.abs(b.particles.v.double().cpu().numpy() - a.particles.v.double().cpu().numpy()).max() <= tol
    wi = a.solver.last_roles(0)[1]
    for nm in ("rho", "ux", "uy", "uz"):
        da = a.solver.arrays(wi, 0)[nm].double().cpu().numpy()
        db = b.solver.arrays(b.solver.last_roles(0)[1], 0)[nm].double().cpu().numpy()
        assert np.abs(da - db).max() <= tol, nm


@pytest.mark.parametrize("scene", ["snow_3d", "snow_2d"])
def test_snow_nacc_fp64(scene):
    """The paper's snow (NACC + softening law) in G2P against
    the oracle's restatement (parity unpinned: the reference has no snow):
    gate A on fields and particles, the hardening state (vol_corr row) per
    particle, and both hardening branches reached (cracked and softening)."""
    sc = S.SNOW_3D_SMALL if scene == "snow_3d" else S.SNOW_2D
    osim, dsim = run_and_compare(sc, 10)
    from oracle import mpm as OM
    qd = dsim.particles.vol_corr.double().cpu().numpy()
    assert np.abs(qd - osim.p.vol_corr).max() <= 1e-9
    _, cracked = OM.nacc_state_decode(osim.p.vol_corr)
    assert cracked.any() and (~cracked).any()


def test_incremental_classification_matches_full():
    """The rebuild's incremental classification (clean tiles copied by warps,
    the dirty ones classified by a persistent grid over their list) leaves
    the same flags, masks and tile flags as classifying every tile anew."""
    _need_gpu()
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    from paper_2603_14982_b200.solver import build_tables
    sim = build_scene(validate_scene(S.scene(S.CLOUD_3D_SMALL)))
    x = sim.particles.x.cpu().numpy()
    v = np.zeros_like(x)
    v[:, 0] = np.where(x[:, 0] < 48.0, 0.3, -0.3)
    sim.particles.v = v
    topo, solver = sim.topology, sim.solver
    T = 4 ** topo.d
    checked = 0
    for _ in range(10):
        c0 = sim.topology_changes
        sim.step()
        if sim.topology_changes == c0:
            continue
        torch.cuda.synchronize()
        err = torch.zeros_like(solver._err)
        full = build_tables(topo, solver._bc, solver._solid, err)
        for l in range(topo.levels):
            n = topo.n_tiles(l)
            if not n:
                continue
            inc = solver._tables[l]
            for nm in ("cell_flags", "dir_masks"):
                assert torch.equal(getattr(inc, nm)[:n * T], getattr(full[l], nm)[:n * T]), (l, nm)
            assert torch.equal(inc.tile_flags[:n], full[l].tile_flags[:n]), l
        checked += 1
    assert checked > 0


def test_entrainment_surface_flags_match_numpy():
    """The entrainment-surface flags of the fp32 stress raster (per-tile
    shared-memory window): 2 on every surface cell (0 < eta < eta_surface with
    an absent or empty face neighbour), 1 on the other stored cells of its 3^3
    neighbourhood, 0 elsewhere — against a dense NumPy restatement."""
    _need_gpu()
    from paper_2603_14982_b200 import _lib as L
    sc = S.scene(S.POWDER_3D_SMALL, runtime__dtype="f32")
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    sim = build_scene(validate_scene(sc))
    for _ in range(3):
        sim.step()
    torch.cuda.synchronize()
    topo, grid, p = sim.topology, sim.grid, sim.particles
    lv0 = grid.level0()
    cells = np.asarray(topo.cell_coords(0))
    n0 = len(cells)
    surf = torch.zeros(n0 + 64, dtype=torch.float32, device="cuda")
    eta_s = float(sim.powder.eta_surface)
    L.check(L.lib().mlbm_stress_raster_surface(
        L.C.byref(lv0), len(p), L.ptr(p.xd), L.ptr(p.pd), p.pd.stride(0), sim.material.lam,
        sim.material.mu, sim.material.alpha, L.ptr(grid.ras), grid.ras.stride(0), eta_s,
        L.ptr(surf), 0, L.ptr(grid._err), L.stream_handle()), "stress_raster_surface")
    got = surf[:n0].cpu().numpy()
    eta = grid.ras[grid.R["etae"]][:n0].double().cpu().numpy()
    dims = topo.finest_cells
    per = topo.periodic3()
    idx = -np.ones(dims, dtype=np.int64)
    idx[cells[:, 0], cells[:, 1], cells[:, 2]] = np.arange(n0)
    want = np.zeros(n0)
    for i in np.nonzero((eta > 0) & (eta < eta_s))[0]:
        c = cells[i]
        empty = False
        for a in range(3):
            for sgn in (1, -1):
                q = c.copy()
                q[a] += sgn
                if per[a]:
                    q[a] %= dims[a]
                elif q[a] < 0 or q[a] >= dims[a]:
                    q = c                       # a domain face clamps to the cell itself
                j = idx[tuple(q)]
                if j < 0 or eta[j] < 1e-3:
                    empty = True
        if not empty:
            continue
        for o in np.ndindex(3, 3, 3):
            q = c + np.array(o) - 1
            ok = True
            for a in range(3):
                if per[a]:
                    q[a] %= dims[a]
                elif q[a] < 0 or q[a] >= dims[a]:
                    ok = False
            if not ok or idx[tuple(q)] < 0:
                continue
            j = idx[tuple(q)]
            want[j] = max(want[j], 2.0 if o == (1, 1, 1) else 1.0)
    assert (want == 2).any()
    assert np.array_equal(got, want)
