"""The reference's standalone per-kernel seams on the device, each against
the oracle function it replaces (fp64, coordinate-keyed):

  granular.stencil               granular.py:137-178
  coupling.rasterize_fractions   coupling.py:96-131
  coupling.difelice_drag         coupling.py:134-156
  CoupledSim._limit_drag         coupling.py:379-401
  coupling.grad_eps              coupling.py:159-182
  coupling.mixture_force         coupling.py:185-197
  coupling.powder_step           coupling.py:230-272
"""
import numpy as np
import pytest
import torch

import scenes as S
from oracle import coupling as OC
from oracle import mpm as OM
from oracle import scene as OS

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2603_14982_b200")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module", params=[2, 3])
def sims(request):
    _need_gpu()
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    sc = S.SAND_COLLAPSE_2D if request.param == 2 else S.COLUMN_3D_SMALL
    cfg = validate_scene(sc)
    dsim = build_scene(cfg)
    osim = OS.build_scene(cfg.raw, heightmap=cfg.heightmap())
    for _ in range(3):
        osim.step()
        dsim.step()
    assert dsim.topology.tile_set() == osim.topo.tile_set()
    oc = osim.topo.cell_coords(0)
    dc = dsim.topology.cell_coords(0)
    dmap = {tuple(c): i for i, c in enumerate(dc)}
    perm = np.array([dmap[tuple(c)] for c in oc])       # oracle cell -> device cell
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))                    # device cell -> oracle cell
    return osim, dsim, perm, inv


def field(coords, k, amp, off=0.0):
    return off + amp * np.sin(coords.astype(float) @ np.asarray(k)[:coords.shape[1]])


def dev(v, inv):
    """oracle-ordered values -> device-ordered tensor"""
    return torch.as_tensor(np.asarray(v)[inv], dtype=torch.float64, device="cuda")


def back(t, perm):
    """device tensor (n[, d]) -> oracle order numpy"""
    return t.double().cpu().numpy()[perm]


def test_stencil(sims):
    osim, dsim, perm, inv = sims
    d = dsim.d
    x = osim.p.x
    oidx, ow, og, odp = OM.stencil(x, osim.topo)
    out = B.granular.stencil(x, dsim.topology)
    idx, w = out[0].cpu().numpy(), out[1].cpu().numpy()
    g = np.stack([t.cpu().numpy() for t in out[2:2 + d]], axis=-1)
    dp = np.stack([t.cpu().numpy() for t in out[2 + d:]], axis=-1)
    oc = osim.topo.cell_coords(0)
    dc = dsim.topology.cell_coords(0)
    assert np.array_equal(dc[idx], oc[oidx])
    assert np.abs(w - ow).max() <= 1e-15
    assert np.abs(g - og).max() <= 1e-15
    assert np.abs(dp - odp).max() <= 1e-12


def test_stencil_outside_raises(sims):
    _, dsim, _, _ = sims
    d = dsim.d
    far = np.full((1, d), 0.2)       # the stencil leaves a walled domain
    with pytest.raises(B.TopologyError):
        B.granular.stencil(far, dsim.topology)


def test_fraction_drag_force_chain(sims):
    osim, dsim, perm, inv = sims
    from paper_2603_14982_b200 import coupling as DC
    d = dsim.d
    oc = osim.topo.cell_coords(0)
    n = len(oc)
    phi = np.abs(field(oc, [0.31, 0.17, 0.23], 0.05))
    rho = field(oc, [0.11, 0.29, 0.07], 0.01, 1.0)
    u = np.stack([field(oc, [0.2 + 0.1 * a, 0.13, 0.3 - 0.05 * a], 0.03) for a in range(d)], 1)
    eps_min, nu, dp = 0.5, 0.1, 0.8
    of = OC.rasterize_fractions(osim.p, osim.topo, phi, eps_min)
    df = DC.rasterize_fractions(dsim.particles, dsim.topology, dev(phi, inv), eps_min)
    for nm, o, dd in (("eps", of.eps, df.eps), ("eta", of.eta, df.eta), ("area", of.area, df.area),
                      ("mass", of.mass, df.mass), ("v", of.v, df.v)):
        assert np.abs(back(dd, perm) - o).max() <= 1e-12, nm
    ofs = OC.difelice_drag(of, rho, u, nu, OC.DragParams(), dp)
    dfs = DC.difelice_drag(df, dev(rho, inv), *[dev(u[:, a], inv) for a in range(2)], nu,
                           DC.DragParams(), dp, uz=dev(u[:, 2], inv) if d == 3 else None)
    assert np.abs(ofs).max() > 0
    assert np.abs(back(dfs, perm) - ofs).max() <= 1e-12 * max(1.0, np.abs(ofs).max())
    assert np.abs(back(df.rel, perm) - of.rel).max() <= 1e-14
    OC.limit_drag(of, rho, u, 1.0)
    DC.limit_drag(df, dev(rho, inv), *[dev(u[:, a], inv) for a in range(2)], 1.0,
                  uz=dev(u[:, 2], inv) if d == 3 else None)
    assert np.abs(back(df.fs, perm) - of.fs).max() <= 1e-12 * max(1.0, np.abs(of.fs).max())
    g = (0.0, -1e-4, 0.0)[:d]
    ofor = OC.mixture_force(of, rho, osim.topo, g, 1.0)
    dfor = DC.mixture_force(df, dev(rho, inv), dsim.topology, g, 1.0)
    assert np.abs(back(dfor, perm) - ofor).max() <= 1e-13
    assert np.abs(back(df.grad_term, perm) - of.grad_term).max() <= 1e-13
    eps2 = field(oc, [0.4, 0.27, 0.19], 0.2, 0.7)
    assert np.abs(back(DC.grad_eps(dev(eps2, inv), dsim.topology), perm)
                  - OC.grad_eps(eps2, osim.topo)).max() <= 1e-15
    assert n == dsim.topology.cell_count(0)


@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_powder_step(sims, sign):
    osim, dsim, perm, inv = sims
    from paper_2603_14982_b200 import coupling as DC
    d = dsim.d
    oc = osim.topo.cell_coords(0)
    phi = np.abs(field(oc, [0.21, 0.33, 0.12], 0.1))
    u = [field(oc, [0.05 + 0.07 * a, 0.19, 0.11], 0.4) for a in range(d)]
    src = np.abs(field(oc, [0.5, 0.1, 0.3], 1e-3))
    prm = OC.PowderParams(diffusion=0.05, sign=sign)
    o = OC.powder_step(phi, u, osim.topo, prm, 1.0, source=src)
    dd = DC.powder_step(dev(phi, inv), dev(u[0], inv), dev(u[1], inv), dsim.topology,
                        DC.PowderParams(diffusion=0.05, sign=sign), 1.0, source=dev(src, inv),
                        uz=dev(u[2], inv) if d == 3 else None)
    assert np.abs(back(dd, perm) - o).max() <= 1e-13


@pytest.mark.parametrize("d", [2, 3])
def test_fp32_diagnostics_match_torch_reductions(d):
    """The fp32 diagnostics kernels (4 cells / particles per thread, 16-byte
    row loads) against torch reductions of the same device state: fluid
    momentum, sum phi and eps min over the leaf cells of every level; sediment
    momentum and the drag-force sum over level 0."""
    _need_gpu()
    from paper_2603_14982_b200 import _lib as L
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    sc = S.scene(S.SAND_COLLAPSE_2D if d == 2 else S.COLUMN_3D_SMALL)
    sc.setdefault("runtime", {})["dtype"] = "f32"
    sim = build_scene(validate_scene(sc))
    for _ in range(3):
        sim.step()
    torch.cuda.synchronize()
    solver, lib = sim.solver, L.lib()
    out = torch.zeros(3 * d + 2, dtype=torch.float64, device="cuda")
    names = B.field_names(d)
    ref_mom = np.zeros(d)
    ref_phi, ref_emin = 0.0, 1.0
    for l in range(sim.topology.levels):
        n = sim.topology.cell_count(l)
        if not n:
            continue
        lw = solver.last_roles(l)[1] if solver.k[l] else 0
        a = solver.arrays(lw, l)
        vol = float((1 << d) ** l)
        out[:d + 2].zero_()
        out[d + 1] = 1.0
        L.check(lib.mlbm_diag_level(L.C.byref(solver._structs[l]), L.fields(a.data), vol, 0,
                                    L.ptr(out[:d + 2]), L.stream_handle()), "diag_level")
        torch.cuda.synchronize()
        leaf = (solver._tables[l].cell_flags[:n] & 64) != 0
        data = a.data[:, :n].double()
        rho = 1.0 + data[names.index("rho")]          # row 0 holds rho - 1
        for k in range(d):
            m = float((vol * rho * data[1 + k])[leaf].sum().item())
            assert abs(out[k].item() - m) <= 1e-9 * max(1.0, abs(m)) + 1e-12
            ref_mom[k] += m
        phi = float((vol * data[names.index("phi")])[leaf].sum().item())
        assert abs(out[d].item() - phi) <= 1e-9 * max(1.0, abs(phi)) + 1e-12
        emin = float(data[names.index("eps")][leaf].min().item()) if bool(leaf.any()) else 1.0
        assert out[d + 1].item() == pytest.approx(min(emin, 1.0), abs=0)
    # particles: sum m v over particles, sum fs over the level-0 cells
    p, g = sim.particles, sim.grid
    out.zero_()
    n0 = sim.topology.capacity_cells(0)
    L.check(lib.mlbm_diag_particles(d, len(p), L.ptr(p.pd), p.pd.stride(0), L.ptr(g.ras),
                                    g.ras.stride(0), n0, L.ptr(sim.topology.dcounts[0]), 0,
                                    L.ptr(out[d + 2:]), L.stream_handle()), "diag_particles")
    torch.cuda.synchronize()
    R = p.R
    mv = (p.pd[R["m"]].double() * p.pd[R["v"]:R["v"] + d].double()).sum(dim=1)
    fs = g.ras[g.R["fs"]:g.R["fs"] + d, :sim.topology.cell_count(0)].double().sum(dim=1)
    for k in range(d):
        assert abs(out[d + 2 + k].item() - mv[k].item()) <= 1e-9 * max(1.0, abs(mv[k].item())) + 1e-12
        assert abs(out[2 * d + 2 + k].item() - fs[k].item()) <= 1e-9 * max(1.0, abs(fs[k].item())) + 1e-12
