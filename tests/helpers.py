"""Shared test helpers: matched oracle / device scenes and coordinate-keyed
comparisons (slot order is never compared)."""
import numpy as np

from oracle import adapt as OA
from oracle import grid as OG
from oracle import lbm as OL


def oracle_static_refined(cells, levels, static, tau0=0.8, periodic=None):
    topo = OG.Topology(cells, levels, periodic)
    d = len(cells)
    drv = OA.RefineDriver(np.zeros((0, d)), static, levels)
    OA.apply_tile_set(topo, OA.brute_force_grid(drv, cells, levels, topo.periodic))
    return topo


def central_mask(cells, pad=4):
    t = [c // 4 for c in cells]
    m = np.zeros(t, dtype=bool)
    m[tuple(slice(n // pad, (pad - 1) * n // pad) for n in t)] = True
    return m


def keyed(coords, values):
    """dict coords -> row of values (values: list of 1-D arrays)."""
    v = np.stack(values, axis=1)
    return {tuple(c): v[i] for i, c in enumerate(coords)}


def compare_levels(otopo, oarr_fn, dtopo, darr_fn, names, levels=None):
    """max |device - oracle| per field over matching coordinates (all levels)."""
    levels = range(otopo.levels) if levels is None else levels
    worst = {nm: 0.0 for nm in names}
    for l in levels:
        oc = otopo.cell_coords(l)
        dc = dtopo.cell_coords(l)
        assert len(oc) == len(dc), f"level {l} cell counts differ"
        if not len(oc):
            continue
        oa = oarr_fn(l)
        da = darr_fn(l)
        # order device values by oracle coordinates
        dmap = {tuple(c): i for i, c in enumerate(dc)}
        perm = np.array([dmap[tuple(c)] for c in oc], dtype=np.int64)
        for nm in names:
            dv = np.asarray(da[nm].detach().cpu().numpy() if hasattr(da[nm], "detach") else da[nm])
            diff = np.abs(dv[perm] - np.asarray(oa[nm]))
            worst[nm] = max(worst[nm], float(diff.max()))
    return worst


def rel_l2(otopo, oarr_fn, dtopo, darr_fn, names, levels=None):
    levels = range(otopo.levels) if levels is None else levels
    num = den = 0.0
    for l in levels:
        oc = otopo.cell_coords(l)
        dc = dtopo.cell_coords(l)
        if not len(oc):
            continue
        oa, da = oarr_fn(l), darr_fn(l)
        dmap = {tuple(c): i for i, c in enumerate(dc)}
        perm = np.array([dmap[tuple(c)] for c in oc], dtype=np.int64)
        for nm in names:
            dv = da[nm].detach().cpu().numpy()[perm]
            ov = np.asarray(oa[nm])
            num += float(((dv - ov) ** 2).sum())
            den += float((ov ** 2).sum())
    return np.sqrt(num / max(den, 1e-300))


def _keyed_perm(otopo, dtopo, l):
    dmap = {tuple(c): i for i, c in enumerate(dtopo.cell_coords(l))}
    return np.array([dmap[tuple(c)] for c in otopo.cell_coords(l)], dtype=np.int64)


def gate_b_metrics(osim, dsim, ox0, dx0):
    """North-star gate B quantities (BASELINE.json): relative L2 of the
    density deviation drho = rho - 1, the velocity u and the second-order
    moment S over every stored cell of every level, and of the particle
    velocity v and displacement x - x0, device vs oracle.

    ``ox0``/``dx0`` are the initial positions (oracle, device original order)."""
    d = dsim.d
    ax = "xyz"[:d]
    groups = {"drho": ["rho"], "u": ["u" + a for a in ax],
              "S": ["s" + ax[a] + ax[b] for a in range(d) for b in range(a, d)]}
    acc = {g: [0.0, 0.0] for g in groups}
    for l in range(dsim.topology.levels):
        if not dsim.topology.n_tiles(l):
            continue
        ow = osim.solver.last_roles(l)[1] if osim.solver.k[l] else 0
        dw = dsim.solver.last_roles(l)[1] if dsim.solver.k[l] else 0
        oa = osim.solver.arrays(ow, l)
        da = dsim.solver.arrays(dw, l)
        perm = _keyed_perm(osim.topo, dsim.topology, l)
        for g, names in groups.items():
            for nm in names:
                ov = np.asarray(oa[nm], dtype=np.float64)
                if g == "drho":
                    # the device stores drho directly (row 0): no 1 + drho rounding
                    dv = da.data[0, :len(perm)].double().cpu().numpy()[perm]
                    ov = ov - 1.0
                else:
                    dv = da[nm].double().cpu().numpy()[perm]
                acc[g][0] += float(((dv - ov) ** 2).sum())
                acc[g][1] += float((ov ** 2).sum())
    out = {g: float(np.sqrt(n / max(dd, 1e-300))) for g, (n, dd) in acc.items()}
    if len(osim.p):
        v = dsim.particles.v.double().cpu().numpy()
        out["v"] = float(np.linalg.norm(v - osim.p.v) / max(np.linalg.norm(osim.p.v), 1e-300))
        ddisp = dsim.particles.x.cpu().numpy() - dx0
        odisp = osim.p.x - ox0
        out["x-x0"] = float(np.linalg.norm(ddisp - odisp) / max(np.linalg.norm(odisp), 1e-300))
    return out
