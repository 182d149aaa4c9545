"""Frame outputs from device buffers (drop-in for
``pkg/src/mlbm/harness/outputs.py``).

Same files, same bytes as the reference writers for 2D scenes (checked
against fixtures the reference wrote, ``tests/golden/outputs_dune_2d.npz``):

  frame_NNNNN_lL.vtk         legacy ASCII structured points per level:
                             rho, eps, phi, stored (0 absent / 1 border /
                             2 leaf) and the velocity vectors, "%.17g"
  frame_NNNNN_particles.bin  "GLBMPART", version, count + little-endian
                             float64 records (x, y, vx, vy, m); 3D scenes
                             write version 2 records (x, y, z, vx, vy, vz, m)
  frame_NNNNN_speed.ppm / _parts.ppm   8-bit quicklooks (3D: the mid-z slice)
  CSV: per-frame particle summary, streamed diagnostics rows

Each level's fields are scattered into a dense grid on the device and come
to the host in one copy per frame; nothing is read back per cell.
"""
from __future__ import annotations

import os
import struct

import numpy as np
import torch

PARTICLE_MAGIC = b"GLBMPART"
_HDR = struct.Struct("<8sII")
_VERSION_2D, _VERSION_3D = 1, 2


# -- dense grids from device state ------------------------------------------------
def dense_level(topology, arrays, level, names):
    """{name: dense (nx, ny[, nz]) numpy grid} (absent cells 0) plus 'stored'."""
    d = topology.d
    dims = topology.cells_dims(level)
    n = topology.cell_count(level)
    dev = topology.device
    out = {}
    coords = torch.as_tensor(topology.cell_coords(level), device=dev) if n else None
    flat = None
    if n:
        flat = coords[:, 0]
        for a in range(1, d):
            flat = flat * dims[a] + coords[:, a]
    total = int(np.prod(dims))
    stack = torch.zeros((len(names) + 1, total), dtype=torch.float64, device=dev)
    if n:
        for i, nm in enumerate(names):
            stack[i, flat] = arrays[nm].double()
        kinds = torch.as_tensor(topology.tile_kinds(level), device=dev).repeat_interleave(4 ** d)
        stack[len(names), flat] = torch.where(kinds == 0, 2.0, 1.0).double()
    host = stack.cpu().numpy()
    for i, nm in enumerate(list(names) + ["stored"]):
        out[nm] = host[i].reshape(dims)
    return out


# -- VTK ------------------------------------------------------------------------------
def _rows(grid):
    """Text rows of a dense grid, x fastest (VTK order): one row per (y[, z])."""
    g = grid if grid.ndim == 3 else grid[:, :, None]
    lines = []
    for z in range(g.shape[2]):
        for y in range(g.shape[1]):
            lines.append(" ".join(np.char.mod("%.17g", g[:, y, z])))
    return lines


def vtk_text(level, dims, spacing, scalars, velocity):
    d = len(dims)
    nz = dims[2] if d == 3 else 1
    head = ["# vtk DataFile Version 3.0", f"fields level {level}", "ASCII",
            "DATASET STRUCTURED_POINTS", f"DIMENSIONS {dims[0]} {dims[1]} {nz}",
            "ORIGIN 0 0 0",
            f"SPACING {spacing} {spacing} {spacing if d == 3 else 1}",
            f"POINT_DATA {int(np.prod(dims))}"]
    body = []
    for name, grid in scalars:
        body.append(f"SCALARS {name} double 1")
        body.append("LOOKUP_TABLE default")
        body.extend(_rows(grid))
    body.append("VECTORS velocity double")
    comps = [v if v.ndim == 3 else v[:, :, None] for v in velocity]
    for z in range(comps[0].shape[2]):
        for y in range(comps[0].shape[1]):
            cols = [np.char.mod("%.17g", c[:, y, z]) for c in comps]
            if d == 2:
                cols.append(np.full(dims[0], "0.0"))
            trip = np.char.add(np.char.add(np.char.add(cols[0], " "), np.char.add(cols[1], " ")),
                               cols[2])
            body.append(" ".join(trip))
    return "\n".join(head + body) + "\n"


def write_vtk_level(path, topology, arrays, level):
    d = topology.d
    ax = "xyz"[:d]
    g = dense_level(topology, arrays, level, ["rho"] + ["u" + a for a in ax] + ["eps", "phi"])
    text = vtk_text(level, topology.cells_dims(level), float(1 << level),
                    [("rho", g["rho"]), ("eps", g["eps"]), ("phi", g["phi"]),
                     ("stored", g["stored"])],
                    [g["u" + a] for a in ax])
    with open(path, "w") as fh:
        fh.write(text)


def read_vtk_level(path):
    """Parse a level file back into {name: dense grid} (+ 'ux', 'uy'[, 'uz'])."""
    with open(path) as fh:
        lines = fh.read().splitlines()
    dims = None
    out = {}
    i = 0
    while i < len(lines):
        ln = lines[i]
        if ln.startswith("DIMENSIONS"):
            dims = tuple(int(v) for v in ln.split()[1:4])
        elif ln.startswith("SCALARS"):
            name = ln.split()[1]
            nrow = dims[1] * dims[2]
            vals = np.array([[float(v) for v in lines[i + 2 + r].split()] for r in range(nrow)])
            out[name] = vals.reshape(dims[2], dims[1], dims[0]).transpose(2, 1, 0).squeeze(-1) \
                if dims[2] == 1 else vals.reshape(dims[2], dims[1], dims[0]).transpose(2, 1, 0)
            i += 1 + nrow
        elif ln.startswith("VECTORS"):
            nrow = dims[1] * dims[2]
            vals = np.array([[float(v) for v in lines[i + 1 + r].split()] for r in range(nrow)])
            vals = vals.reshape(dims[2], dims[1], dims[0], 3).transpose(2, 1, 0, 3)
            for k, a in enumerate("xyz"):
                g = vals[..., k]
                out["u" + a] = g[..., 0] if dims[2] == 1 else g
            if dims[2] == 1:
                del out["uz"]
            i += nrow
        i += 1
    return out


# -- particles ------------------------------------------------------------------------
def write_particles(path, particles):
    x = particles.x.cpu().numpy()
    v = particles.v.double().cpu().numpy()
    m = particles.m.double().cpu().numpy()
    d = x.shape[1]
    rec = np.column_stack([x, v, m]).astype("<f8")
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(PARTICLE_MAGIC, _VERSION_2D if d == 2 else _VERSION_3D, len(m)))
        fh.write(rec.tobytes())


def read_particles(path):
    """(x, v, m) of a dump (version 1: 2D, version 2: 3D)."""
    raw = open(path, "rb").read()
    magic, version, count = _HDR.unpack_from(raw, 0)
    if magic != PARTICLE_MAGIC:
        raise ValueError(f"not a particle dump: bad magic {magic!r}")
    if version not in (_VERSION_2D, _VERSION_3D):
        raise ValueError(f"unsupported particle dump version {version}")
    d = 2 if version == _VERSION_2D else 3
    rec = np.frombuffer(raw, dtype="<f8", offset=_HDR.size, count=count * (2 * d + 1))
    rec = rec.reshape(count, 2 * d + 1)
    return rec[:, :d].copy(), rec[:, d:2 * d].copy(), rec[:, 2 * d].copy()


def particle_summary_csv(path, rows):
    with open(path, "w") as fh:
        fh.write("frame,count,kinetic_energy,max_speed\n")
        for frame, count, ke, vmax in rows:
            fh.write(f"{frame},{count},{ke!r},{vmax!r}\n")


# -- quicklooks ----------------------------------------------------------------------
def _ramp():
    t = np.linspace(0.0, 1.0, 256)
    rgb = np.stack([np.clip(2.0 * t, 0, 1), np.clip(1.0 - 2.0 * np.abs(t - 0.5), 0, 1),
                    np.clip(2.0 * (1.0 - t), 0, 1)], axis=1)
    return (rgb * 255).astype(np.uint8)


def write_ppm(path, values, vmax):
    """8-bit binary PPM of an (nx, ny) field, blue -> white -> red, y up."""
    idx = np.clip(values / max(vmax, 1e-300) * 255.0, 0, 255).astype(np.uint8)
    img = _ramp()[idx]
    nx, ny = values.shape
    with open(path, "wb") as fh:
        fh.write(f"P6\n{nx} {ny}\n255\n".encode())
        fh.write(np.ascontiguousarray(img.transpose(1, 0, 2)[::-1]).tobytes())


def _slice(grid):
    return grid if grid.ndim == 2 else grid[:, :, grid.shape[2] // 2]


def quicklook_speed(path, topology, arrays, vmax=0.1):
    ax = "xyz"[:topology.d]
    g = dense_level(topology, arrays, 0, ["u" + a for a in ax])
    speed = np.sqrt(sum(g["u" + a] ** 2 for a in ax)) if topology.d == 3 else \
        np.hypot(g["ux"], g["uy"])
    write_ppm(path, _slice(speed), vmax)


def quicklook_particles(path, topology, particles, vmax=8.0):
    dims = topology.cells_dims(0)
    dens = np.zeros(dims)
    if len(particles):
        c = np.floor(particles.x.cpu().numpy()).astype(np.int64)
        idx = tuple(c[:, a].clip(0, dims[a] - 1) for a in range(topology.d))
        np.add.at(dens, idx, 1.0)
    write_ppm(path, _slice(dens), vmax)


class DiagnosticsWriter:
    """Streams DiagRow rows to CSV (3D adds the z components)."""

    def __init__(self, path, levels, d=2):
        self.d = d
        self._fh = open(path, "w")
        ax = "xyz"[:d]
        cols = (["step", "t_phys"] + [f"fluid_mom_{a}" for a in ax] + [f"sed_mom_{a}" for a in ax]
                + [f"drag_imp_{a}" for a in ax] + ["sum_phi"]
                + [f"tiles_l{i}" for i in range(levels)] + ["eps_min"])
        self._fh.write(",".join(cols) + "\n")

    def write(self, row):
        vals = ([str(row.step), repr(row.t_phys)] + [repr(v) for v in row.fluid_mom]
                + [repr(v) for v in row.sediment_mom] + [repr(v) for v in row.drag_impulse]
                + [repr(row.sum_phi)] + [str(t) for t in row.tiles] + [repr(row.eps_min)])
        self._fh.write(",".join(vals) + "\n")

    def close(self):
        self._fh.close()


def write_frame(directory, frame, sim, cfg):
    """Every configured output of one frame (config ``outputs`` table)."""
    os.makedirs(directory, exist_ok=True)
    opt = cfg.raw["outputs"]
    solver, topo = sim.solver, sim.topology
    torch.cuda.synchronize()
    stem = os.path.join(directory, f"frame_{frame:05d}")
    if opt["fields"]:
        for level in range(topo.levels):
            if not topo.n_tiles(level):
                continue
            w = solver.last_roles(level)[1] if solver.k[level] else 0
            write_vtk_level(f"{stem}_l{level}.vtk", topo, solver.arrays(w, level), level)
    if opt["particles"] and len(sim.particles):
        write_particles(f"{stem}_particles.bin", sim.particles)
    if opt["quicklook"]:
        w = solver.last_roles(0)[1] if solver.k[0] else 0
        quicklook_speed(f"{stem}_speed.ppm", topo, solver.arrays(w, 0))
        quicklook_particles(f"{stem}_parts.ppm", topo, sim.particles)
