"""Scene assembly for the oracle (restates harness/config.py:150-166,293-353).

Consumes an already-validated scene dict (the product's
``paper_2603_14982_b200.harness.config`` or the reference's
``validate_scene`` produce the same ``raw`` layout), in 2D or 3D.  A 3D scene
has 3 extents, 6 faces (z_min/z_max), 6-tuple boxes (lo..., hi...) and an
optional 2D heightmap over (x, z).
"""
from __future__ import annotations

import numpy as np

from . import mpm
from .adapt import GridAdaptor, RefineDriver
from .coupling import CoupledSim, DragParams, PowderParams
from .grid import TILE, PingPongPair, Topology
from .lbm import (BoundarySpec, LevelParams, LogInlet, Solver, SolverParams,
                  face_names, set_fields)
from .lattice import CS2, H3_XYZ_HERMITE, H3_XYZ_PAPER


def boundary_spec(raw, d, heightmap=None):
    b = raw["boundaries"]
    faces = {}
    for f in face_names(d):
        v = b.get(f, "periodic")
        if isinstance(v, dict):
            faces[f] = LogInlet(float(v["u0"]), float(v["beta"]), float(v["y0"]))
        else:
            faces[f] = v
    boxes = [tuple(float(c) for c in box) for box in b.get("solid_boxes", [])]
    return BoundarySpec(d=d, faces=faces, solid_boxes=boxes,
                        heightmap=heightmap)


def material(raw):
    m = raw["materials"]
    u = raw["units"]
    stress = u["rho"] * (u["dx"] / u["dt"]) ** 2
    if m.get("model", "sand") == "snow":
        return mpm.SnowMaterial(E=m["E"] / stress, nu=m["nu"], M=m["nacc_M"],
                                beta=m["nacc_beta"], xi=m["nacc_xi"],
                                alpha_soft=m["nacc_alpha"], q_init=m["nacc_q0"],
                                floor_friction=m["floor_friction"],
                                friction_deg=m["friction_angle_deg"])
    return mpm.SandMaterial(E=m["E"] / stress, nu=m["nu"],
                            friction_deg=m["friction_angle_deg"],
                            floor_friction=m["floor_friction"])


def gravity_lattice(raw):
    u = raw["units"]
    return tuple(g * u["dt"] ** 2 / u["dx"] for g in raw["fluid"]["gravity"])


def taylor_green_fn(u0, n, nu, taus, d):
    """cases.py:54-77 (3D: z-extruded vortex in the x-y plane)."""
    k = 2.0 * np.pi / n

    def fn(pos, level):
        px, py = pos[:, 0], pos[:, 1]
        ux = -u0 * np.cos(k * px) * np.sin(k * py)
        uy = u0 * np.sin(k * px) * np.cos(k * py)
        p = -0.25 * u0 * u0 * (np.cos(2 * k * px) + np.cos(2 * k * py))
        tau = taus[level]
        sc = float(1 << level)
        dxux = u0 * k * np.sin(k * px) * np.sin(k * py)
        dyux = -u0 * k * np.cos(k * px) * np.cos(k * py)
        dxuy = u0 * k * np.cos(k * px) * np.cos(k * py)
        out = {"rho": 1.0 + p / CS2, "ux": ux, "uy": uy,
               "sxx": ux * ux - CS2 * tau * sc * 2.0 * dxux,
               "sxy": ux * uy - CS2 * tau * sc * (dyux + dxuy),
               "syy": uy * uy + CS2 * tau * sc * 2.0 * dxux}
        if d == 3:
            z = np.zeros_like(px)
            out.update({"uz": z, "sxz": z, "syz": z, "szz": z})
        return out
    return fn


def build_scene(raw, heightmap=None):
    d = len(raw["domain"]["cells"])
    cells = tuple(int(c) for c in raw["domain"]["cells"])
    L = int(raw["domain"]["levels"])
    spec = boundary_spec(raw, d, heightmap)
    topo = Topology.uniform(cells, L, spec.periodic_axes())
    pair = PingPongPair(topo)
    rng = np.random.default_rng(np.random.Philox(raw["runtime"]["seed"]))
    parts = None
    if raw["particles"]["blocks"]:
        dens = raw["materials"]["density_ratio"] * raw["fluid"]["rho0"]
        parts = mpm.sample_blocks(
            [tuple(float(v) for v in b) for b in raw["particles"]["blocks"]],
            raw["particles"]["per_cell"], dens, rng, d=d)
        if raw["materials"].get("model", "sand") == "snow":
            parts.vol_corr[:] = raw["materials"]["nacc_q0"]
    static = None
    if raw["adapt"]["static_boxes"]:
        static = np.zeros(topo.tiles_dims(0), dtype=bool)
        for box in raw["adapt"]["static_boxes"]:
            sl = tuple(slice(int(box[a]) // TILE,
                             (int(box[d + a]) + TILE - 1) // TILE)
                       for a in range(d))
            static[sl] = True
    fl = raw["fluid"]
    params = SolverParams(levels=L, rho0=fl["rho0"],
                          gravity=gravity_lattice(raw), eps_min=fl["eps_min"],
                          mpm_cadence=raw["runtime"]["mpm_cadence"],
                          rescale_convention=fl["rescale_convention"],
                          upward_mode=fl["upward_mode"],
                          h3_xyz=H3_XYZ_PAPER if fl.get("h3_xyz") ==
                          "paper_literal" else H3_XYZ_HERMITE)
    lp = LevelParams(L, fl["tau0"])
    adaptor = None
    if L > 1:
        adaptor = GridAdaptor(topo, lp, params.rescale_convention)
        adaptor.update(RefineDriver(parts.x if parts is not None
                                    else np.zeros((0, d)), static, L), pair)
    sv = Solver(topo, pair, params, lp, spec)
    powder = None
    pw = raw["powder"]
    if pw["enabled"]:
        powder = PowderParams(entrain=pw["entrain"], diffusion=pw["diffusion"],
                              sign=1.0 if pw["sign"] == "stable" else -1.0)
    sim = CoupledSim(sv, parts, material(raw),
                     sediment_gravity=np.asarray(gravity_lattice(raw)),
                     drag=DragParams(), powder=powder, adaptor=adaptor,
                     static_tiles=static, unit_dt=raw["units"]["dt"])
    if fl["init"] == "taylor_green":
        fn = taylor_green_fn(fl["init_u0"], cells[0], lp.nu(0), lp.taus, d)
        set_fields(topo, pair, fn)
    return sim
