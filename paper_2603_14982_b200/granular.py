"""MPM sand on the B200 (drop-in for ``pkg/src/mlbm/granular.py``).

Particle state is device-resident structure-of-arrays: positions as float64
rows ``xd[d, n]`` and the run-dtype rows ``pd = [v(d), C(d*d), F(d*d), m, V0,
vol_corr]`` (27 reals per particle in 3D).  The step is three kernels:

  p2g   (granular.py:137-178 stencil, 260-279 Kirchhoff, 282-310 scatter)
  grid  (granular.py:313-341 grid_update; fused into the coupled exchange)
  g2p   (granular.py:344-412 gather, advect, SVD, Drucker-Prager)

There is no particle sort in the reference; scatter order is irrelevant to
the float tolerance.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .solver import BoundarySpec, build_tables
from .sparse_grid import DEFAULT_DTYPE, TILE, Topology, TopologyError, dtype_code


@dataclass
class SandMaterial:
    """granular.py:22-38."""
    E: float = 3.5e5
    nu: float = 0.3
    friction_deg: float = 30.0
    floor_friction: float = 0.5

    def __post_init__(self):
        self.lam = self.E * self.nu / ((1 + self.nu) * (1 - 2 * self.nu))
        self.mu = self.E / (2 * (1 + self.nu))
        sf = np.sin(np.radians(self.friction_deg))
        self.alpha = float(np.sqrt(2.0 / 3.0) * 2.0 * sf / (3.0 - sf))

    def wave_speed(self, density: float) -> float:
        return float(np.sqrt((self.lam + 2 * self.mu) / density))

    def snow_struct(self):
        return None


@dataclass
class SnowMaterial:
    """The paper's snow: Non-Associated Cam Clay (Wolper et
    al. 2019) on the sand's Hencky elasticity with the modified hardening law
    dq/dt = -alpha_soft q0' until q first reaches 0 (the particle cracks, its
    cohesion becomes 0), +q0' after.  Absent from the reference:
    oracle/mpm.py:nacc_return_map is the specification (parity unpinned).
    The hardening state rides in the vol_corr row (q >= 0, or -(q + 1) once
    cracked); particles start at q_init."""
    E: float = 3.5e5
    nu: float = 0.3
    M: float = 1.85
    beta: float = 0.3
    xi: float = 1.0
    alpha_soft: float = 0.5
    q_init: float = 0.05
    floor_friction: float = 0.5
    friction_deg: float = 30.0

    def __post_init__(self):
        self.lam = self.E * self.nu / ((1 + self.nu) * (1 - 2 * self.nu))
        self.mu = self.E / (2 * (1 + self.nu))
        self.alpha = 0.0

    def wave_speed(self, density: float) -> float:
        return float(np.sqrt((self.lam + 2 * self.mu) / density))

    def snow_struct(self):
        s = L.Snow()
        s.M, s.beta, s.xi, s.alpha_soft = self.M, self.beta, self.xi, self.alpha_soft
        return s


def snow_arg(mat):
    """mlbm_g2p's snow parameter block (NULL: Drucker-Prager sand)."""
    s = mat.snow_struct() if hasattr(mat, "snow_struct") else None
    if s is None:
        return None
    mat._snow_c = s                 # keep the struct alive for the call
    return L.C.byref(s)


def prow(d):
    """Run-dtype particle rows: v, C, F, m, V0, vol_corr and the Kirchhoff
    stress tau(F) (symmetric, kept current by G2P; mlbm_particle_stress)."""
    return {"v": 0, "C": d, "F": d + d * d, "m": d + 2 * d * d, "V0": d + 2 * d * d + 1,
            "vc": d + 2 * d * d + 2, "tau": d + 2 * d * d + 3,
            "n": d + 2 * d * d + 3 + d * (d + 1) // 2}


class Particles:
    """SoA particle state in HBM (granular.py:41-63)."""

    def __init__(self, n: int, d: int = 2, dtype=None, device=None):
        self.d = d
        self.dtype = dtype or DEFAULT_DTYPE
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.R = prow(d)
        self.xd = torch.zeros((d, n), dtype=torch.float64, device=self.device)
        self.pd = torch.zeros((self.R["n"], n), dtype=self.dtype, device=self.device)
        for a in range(d):
            self.pd[self.R["F"] + a * d + a] = 1.0
        self.pd[self.R["m"]] = 1.0
        self.pd[self.R["V0"]] = 1.0
        # storage order may be permuted by the per-step sort (coupling); pid
        # maps storage index -> original (reference) particle index
        self.pid = torch.arange(n, dtype=torch.int32, device=self.device)
        self.permuted = False
        self._scratch = None
        # the tau rows hold the Kirchhoff stress of F for the material they
        # were computed with (None: stale, recomputed before the next P2G)
        self.stress_mat = None

    @classmethod
    def wrap(cls, xd, pd, pid, dtype):
        """Particles over existing device views (x [d, n], rows [R, n] sharing
        one row stride, ids [n]) — capacity buffers of the slab migration."""
        p = cls.__new__(cls)
        p.d = xd.shape[0]
        p.dtype = dtype
        p.device = xd.device
        p.R = prow(p.d)
        assert xd.stride(0) == pd.stride(0), "x and rows must share the row stride"
        p.xd, p.pd, p.pid = xd, pd, pid
        p.permuted = False
        p._scratch = None
        p.stress_mat = None
        return p

    def ensure_stress(self, mat):
        """(Re)compute the tau rows from F when F changed outside G2P or the
        material differs (mlbm_particle_stress); G2P keeps them current."""
        key = (float(mat.lam), float(mat.mu))
        if self.stress_mat == key or not len(self):
            return
        L.check(L.lib().mlbm_particle_stress(self.d, len(self), L.ptr(self.pd), self.pd.stride(0),
                                             mat.lam, mat.mu, mat.alpha, dtype_code(self.dtype),
                                             L.stream_handle()), "particle_stress")
        self.stress_mat = key

    def scratch(self, n_slots=0):
        """Sort targets + sort workspace (allocated once; regrown when the
        level-0 slot capacity ``n_slots`` grows), with the storage's row
        stride (the kernels take one stride for both)."""
        need = int(L.lib().mlbm_sort_ws_bytes(max(len(self), 1), int(n_slots)))
        if self._scratch is not None and self._scratch[3].numel() < need:
            self._scratch = (*self._scratch[:3], torch.empty(int(need * 1.25), dtype=torch.uint8,
                                                             device=self.device))
        if self._scratch is None:
            n = len(self)
            cap = self.pd.stride(0)
            ws = torch.empty(int(need * 1.25), dtype=torch.uint8, device=self.device)
            self._scratch = (torch.empty((self.d, cap), dtype=torch.float64, device=self.device)[:, :n],
                             torch.empty((self.pd.shape[0], cap), dtype=self.dtype,
                                         device=self.device)[:, :n],
                             torch.empty(cap, dtype=torch.int32, device=self.device)[:n], ws)
        return self._scratch

    def _orig(self, t):
        """Rows [k, n] in storage order -> rows in original particle order."""
        if not self.permuted:
            return t
        out = torch.empty_like(t)
        out[:, self.pid.long()] = t
        return out

    def _store(self, rows, val):
        """Write rows given in original particle order into storage order."""
        if self.permuted:
            val = val[:, self.pid.long()]
        rows.copy_(val)

    def __len__(self):
        return self.xd.shape[1]

    def _rows(self, name, k):
        return self.pd[self.R[name]:self.R[name] + k]

    # reference-style (n, ...) views / setters -----------------------------------
    @property
    def x(self):
        return self._orig(self.xd).t()

    @x.setter
    def x(self, v):
        self._store(self.xd, torch.as_tensor(np.asarray(v) if not torch.is_tensor(v) else v,
                                             dtype=torch.float64,
                                             device=self.device).reshape(-1, self.d).t())

    @property
    def v(self):
        return self._orig(self._rows("v", self.d)).t()

    @v.setter
    def v(self, val):
        self._store(self._rows("v", self.d), self._as(val).reshape(-1, self.d).t())

    @property
    def C(self):
        return self._orig(self._rows("C", self.d * self.d)).t().reshape(-1, self.d, self.d)

    @C.setter
    def C(self, val):
        self._store(self._rows("C", self.d * self.d), self._as(val).reshape(-1, self.d * self.d).t())

    @property
    def F(self):
        return self._orig(self._rows("F", self.d * self.d)).t().reshape(-1, self.d, self.d)

    @F.setter
    def F(self, val):
        self.stress_mat = None
        self._store(self._rows("F", self.d * self.d), self._as(val).reshape(-1, self.d * self.d).t())

    def _row(self, name):
        return self._orig(self.pd[self.R[name]:self.R[name] + 1])[0]

    def _set_row(self, name, val):
        self._store(self.pd[self.R[name]:self.R[name] + 1], self._as(val).reshape(1, -1))

    @property
    def m(self):
        return self._row("m")

    @m.setter
    def m(self, val):
        self._set_row("m", val)

    @property
    def V0(self):
        return self._row("V0")

    @V0.setter
    def V0(self, val):
        self._set_row("V0", val)

    @property
    def vol_corr(self):
        return self._row("vc")

    @vol_corr.setter
    def vol_corr(self, val):
        self._set_row("vc", val)

    def _as(self, v):
        return torch.as_tensor(v if torch.is_tensor(v) else np.asarray(v), dtype=self.dtype,
                               device=self.device)

    def total_mass(self) -> float:
        return float(self.m.double().sum())

    def momentum(self):
        return (self.m.double()[:, None] * self.v.double()).sum(dim=0).cpu().numpy()

    def kinetic_energy(self) -> float:
        return float(0.5 * (self.m.double() * (self.v.double() ** 2).sum(dim=1)).sum())

    @classmethod
    def from_host(cls, x, v=None, C=None, F=None, m=None, V0=None, vol_corr=None,
                  dtype=None, device=None):
        x = np.asarray(x, dtype=float)
        p = cls(len(x), x.shape[1], dtype, device)
        p.x = x
        for name, val in (("v", v), ("C", C), ("F", F), ("m", m), ("V0", V0),
                          ("vol_corr", vol_corr)):
            if val is not None:
                setattr(p, name, val)
        return p


def sample_blocks(blocks, per_cell: int, density: float, rng, d: int = None,
                  dtype=None, device=None) -> Particles:
    """Jittered uniform sampling (granular.py:66-80); the host RNG stream is
    the reference's, so the same seed gives the same particles."""
    d = d or len(blocks[0]) // 2
    counts = []
    for b in blocks:
        vol = 1.0
        for a in range(d):
            vol *= b[d + a] - b[a]
        counts.append(int(round(vol * per_cell)))
    x = np.zeros((sum(counts), d))
    at = 0
    for b, cnt in zip(blocks, counts):
        u = rng.random((cnt, d))
        for a in range(d):
            x[at:at + cnt, a] = b[a] + u[:, a] * (b[d + a] - b[a])
        at += cnt
    n = len(x)
    p = Particles(n, d, dtype, device)
    p.x = x
    p.V0 = np.full(n, 1.0 / per_cell)
    p.m = np.full(n, density / per_cell)
    return p


def raster_rows(d):
    NS = d * (d + 1) // 2
    return {"mass": 0, "mom": 1, "fint": 1 + d, "eta": 1 + 2 * d, "area": 2 + 2 * d,
            "vmom": 3 + 2 * d, "vel": 3 + 3 * d, "fs": 3 + 4 * d, "eps": 3 + 5 * d,
            "grad": 4 + 5 * d, "rel": 4 + 6 * d, "sig": 4 + 7 * d, "etae": 4 + 7 * d + NS,
            "n": 5 + 7 * d + NS,
            "nacc": 3 + 3 * d}


class MpmGrid:
    """Level-0 node rows (granular.py:83-130) in one [rows, n0] device block."""

    def __init__(self, topology: Topology, boundaries: BoundarySpec | None = None,
                 dtype=None, tables=None):
        self.topology = topology
        self.d = topology.d
        self.boundaries = boundaries or BoundarySpec(dim=self.d)
        self.dtype = dtype or DEFAULT_DTYPE
        self.R = raster_rows(self.d)
        self._version = -1
        self._err = torch.zeros(L.ERR_INTS, dtype=torch.int32, device=topology.device)
        self._tables_fn = tables
        self.counters = torch.zeros(2, dtype=torch.int32, device=topology.device)
        self.sync_topology()

    def sync_topology(self):
        """Raster rows at the level-0 capacity (re-allocated only when the
        capacity grows, so captured graphs keep their pointers)."""
        if self._version == self.topology.cap_version:
            return
        n = self.topology.capacity_cells(0)
        self.ras = torch.zeros((self.R["n"], n), dtype=self.dtype, device=self.topology.device)
        self._version = self.topology.cap_version
        self._lv0 = None

    def level0(self):
        """Level-0 C struct with cell flags (sticky solids)."""
        if self._lv0 is None or self._lv0_ver != self.topology.version:
            self.sync_topology()
            if self._tables_fn is not None:
                t0 = self._tables_fn()
            else:
                bc = self.boundaries.bc_struct(1.0)
                solid = self.boundaries.solid_struct(self.d, self.topology.device)
                self._own_tables = build_tables(self.topology, bc, solid, self._err)
                t0 = self._own_tables[0]
            self._t0 = t0
            self._lv0 = self.topology.level_struct(0, t0)
            self._lv0_ver = self.topology.version
        return self._lv0

    def rows(self, name, k=1):
        return self.ras[self.R[name]:self.R[name] + k]

    def _live(self):
        return self.topology.cell_count(0)

    @property
    def mass(self):
        return self.ras[self.R["mass"], :self._live()]

    @property
    def mom(self):
        return self.rows("mom", self.d)[:, :self._live()].t()

    @property
    def f_int(self):
        return self.rows("fint", self.d)[:, :self._live()].t()

    @property
    def vel(self):
        return self.rows("vel", self.d)[:, :self._live()].t()

    @property
    def drag(self):
        return self.rows("fs", self.d)[:, :self._live()].t()

    def clear(self):
        L.zero(self.ras[:self.R["nacc"]])

    def raise_pending(self):
        e = self._err.cpu().numpy()
        if e[0]:
            self._err.zero_()
            raise TopologyError(f"particle stencil node ({e[3]},{e[4]},{e[5]}) not stored at "
                                f"the finest level / outside the domain")


def _faces(boundaries):
    out = (L.C.c_int32 * 6)()
    for i, f in enumerate(("x_min", "x_max", "y_min", "y_max", "z_min", "z_max")):
        out[i] = 1 if boundaries.faces.get(f) == "wall" else 0
    return out


def _d3(v, d):
    t = (L.C.c_double * 3)()
    for a in range(min(3, len(v))):
        t[a] = float(v[a])
    return t


def stencil(positions, topology: Topology):
    """granular.py:137-178 on the device: quadratic B-spline stencil over the
    level-0 node map.  ``positions`` is a Particles object or an (n, d) array.
    Returns (idx, w, g_x, g_y[, g_z], dpos_x, dpos_y[, dpos_z]), each (n, 3^d)
    in the reference's node order (x offset fastest); idx are level-0 cell
    indices of this topology.  A node outside a non-periodic domain or not
    stored at level 0 raises TopologyError (granular.py:160-173)."""
    d = topology.d
    if isinstance(positions, Particles):
        xd = positions.xd
    else:
        xd = torch.as_tensor(np.asarray(positions, dtype=np.float64) if not torch.is_tensor(positions)
                             else positions, dtype=torch.float64,
                             device=topology.device).reshape(-1, d).t().contiguous()
    n = xd.shape[1]
    K = 3 ** d
    dev = topology.device
    idx = torch.empty((K, n), dtype=torch.int32, device=dev)
    w = torch.empty((K, n), dtype=torch.float64, device=dev)
    g = torch.empty((d, K, n), dtype=torch.float64, device=dev)
    dp = torch.empty((d, K, n), dtype=torch.float64, device=dev)
    err = torch.zeros(L.ERR_INTS, dtype=torch.int32, device=dev)
    if n:
        lv0 = topology.level_struct(0)
        L.check(L.lib().mlbm_stencil(L.C.byref(lv0), n, L.ptr(xd), xd.stride(0), L.ptr(idx),
                                     L.ptr(w), L.ptr(g), L.ptr(dp), n, 1, L.ptr(err),
                                     L.stream_handle()), "stencil")
        e = err.cpu().numpy()
        if e[0]:
            raise TopologyError(f"particle stencil node near ({e[3]},{e[4]},{e[5]}) not stored at "
                                f"the finest level / outside the domain")
    return (idx.t().long(), w.t()) + tuple(g[a].t() for a in range(d)) + \
        tuple(dp[a].t() for a in range(d))


def p2g(particles: Particles, grid: MpmGrid, mat: SandMaterial, st=None):
    grid.sync_topology()
    grid.clear()
    if not len(particles):
        return
    particles.ensure_stress(mat)
    lv0 = grid.level0()
    L.check(L.lib().mlbm_p2g(L.C.byref(lv0), len(particles), L.ptr(particles.xd),
                             L.ptr(particles.pd), particles.pd.stride(0), mat.lam, mat.mu,
                             mat.alpha, L.ptr(grid.ras), grid.ras.stride(0),
                             dtype_code(grid.dtype), 0, L.ptr(grid._err), L.stream_handle()), "p2g")


def grid_update(grid: MpmGrid, dt: float, gravity, drag=None, floor_friction: float = 0.5):
    """granular.py:313-341: drag (n, d) lands in the FS rows first."""
    fs = grid.rows("fs", grid.d)
    fs.zero_()
    if drag is not None:
        n = grid._live()
        fs[:, :n].copy_(torch.as_tensor(drag, dtype=grid.dtype, device=grid.ras.device)
                        .reshape(-1, grid.d).t())
    lv0 = grid.level0()
    z = (L.C.c_double * 3)()
    empty = L.Fields(0, 0)
    L.check(L.lib().mlbm_exchange(L.C.byref(lv0), empty, empty, empty, empty, L.ptr(grid.ras),
                                  grid.ras.stride(0), 0.3, 1.0, 1.0, 0.01, float(dt), 1.0, z,
                                  _d3(gravity, grid.d), _faces(grid.boundaries),
                                  float(floor_friction), 0, dtype_code(grid.dtype),
                                  L.stream_handle()), "grid_update")


def g2p(particles: Particles, grid: MpmGrid, dt: float, mat: SandMaterial,
        plastic: bool = True, st=None) -> int:
    if not len(particles):
        return 0
    lv0 = grid.level0()
    grid.counters.zero_()
    L.check(L.lib().mlbm_g2p(L.C.byref(lv0), len(particles), L.ptr(particles.xd),
                             L.ptr(particles.xd), L.ptr(particles.pd), L.ptr(particles.pd),
                             L.ptr(None), L.ptr(None), particles.pd.stride(0), mat.lam, mat.mu,
                             mat.alpha, snow_arg(mat), L.ptr(grid.ras), grid.ras.stride(0), float(dt),
                             1 if plastic else 0, dtype_code(grid.dtype), L.ptr(grid.counters),
                             L.ptr(None), L.ptr(None), L.ptr(None),
                             L.ptr(grid._err), L.stream_handle()), "g2p")
    grid.raise_pending()
    return int(grid.counters[0].item())


def mpm_step(particles: Particles, grid: MpmGrid, dt: float, gravity, mat: SandMaterial,
             drag=None, plastic: bool = True, st=None) -> int:
    """One explicit MPM step (granular.py:415-425)."""
    grid.sync_topology()
    p2g(particles, grid, mat)
    grid_update(grid, dt, gravity, drag=drag, floor_friction=mat.floor_friction)
    return g2p(particles, grid, dt, mat, plastic=plastic)


def cfl_check(particles: Particles, dt: float) -> bool:
    if not len(particles):
        return True
    return float(particles.v.abs().max()) * dt < 0.5
