"""Two-way fluid-sediment coupling and the coupled step on the B200
(drop-in for ``pkg/src/mlbm/coupling.py``).

One finest cycle (CoupledSim.step, coupling.py:448-481) issues:

  coarser levels (Alg. 1 prelude)          mlbm_downward / mlbm_level_step / mlbm_upward
  level-0 stream (bare moments)            mlbm_level_step(mode=1)
  exchange: P2G + fractions               mlbm_p2g            coupling.py:96-131, granular.py:282-310
            eps, drag, limiter, grad eps,
            mixture force -> both trees,
            MPM grid update               mlbm_exchange       coupling.py:134-197, 379-446
            G2P + plasticity              mlbm_g2p            granular.py:344-412
  level-0 collide + boundaries             mlbm_level_step(mode=2, force/tau from fields)
  powder transport (+ entrainment)         mlbm_stress_raster, mlbm_powder
  block maintenance                        GridAdaptor.update (adapt.py)
  diagnostics                              mlbm_diag_level / mlbm_diag_particles

By default the whole step is replayed as a CUDA graph (one per cycle /
buffer-parity key, recaptured after each topology change) followed by ONE
device->host copy of the error records, adapt flags and diagnostics row; the
host only runs the rebuild when a level's tile set changed.
"""
from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np
import torch

from . import _lib as L
from .adapt import GridAdaptor, RefineDriver
from .granular import MpmGrid, Particles, SandMaterial, SnowMaterial, _d3, _faces, snow_arg
from .solver import FIELD_FORCE, FIELD_TAU, MultiLevelSolver
from .sparse_grid import dtype_code


@dataclass
class UnitScale:
    """coupling.py:26-56."""
    dx: float = 1.0
    dt: float = 1.0
    rho: float = 1.0

    def __post_init__(self):
        if self.dx <= 0 or self.dt <= 0 or self.rho <= 0:
            raise ValueError("unit scales must be positive")

    @property
    def C(self) -> float:
        return self.rho * self.dx / self.dt ** 2

    def velocity_to_lattice(self, v):
        return v * self.dt / self.dx

    def accel_to_lattice(self, a):
        return a * self.dt ** 2 / self.dx

    def force_density_to_lattice(self, f):
        return f / self.C

    def stress_to_lattice(self, s):
        return s / (self.rho * (self.dx / self.dt) ** 2)

    def time_to_lattice(self, t):
        return t / self.dt


@dataclass
class DragParams:
    d_p: float | None = None
    re_min: float = 0.01


@dataclass
class PowderParams:
    entrain: float = 0.0
    diffusion: float = 0.05
    sign: float = 1.0
    eta_surface: float = 0.6

    def check_stability(self, dt: float = 1.0):
        if self.sign > 0 and self.diffusion * dt > 0.25:
            raise ValueError(f"diffusion number D*dt={self.diffusion * dt} exceeds 0.25")


@dataclass
class DiagRow:
    step: int
    t_phys: float
    fluid_mom: tuple
    sediment_mom: tuple
    drag_impulse: tuple
    sum_phi: float
    tiles: tuple
    eps_min: float


def particle_diameter(V0, d):
    if d == 2:
        return 2.0 * np.sqrt(V0 / np.pi)
    return 2.0 * (3.0 * V0 / (4.0 * np.pi)) ** (1.0 / 3.0)


class CouplingFields:
    """Device views of the last exchange (coupling.py:80-93)."""

    def __init__(self, grid: MpmGrid, tree_level0=None):
        d = grid.d
        self.grid = grid
        self.d = d
        n = grid._live()
        r = grid.ras[:, :n]
        R = grid.R
        self.eps = r[R["eps"]]
        self.eta = r[R["etae"]]          # eta_eff (coupling.py:127)
        self.v = r[R["vmom"]:R["vmom"] + d].t()
        self.area = r[R["area"]]
        self.mass = r[R["mass"]]
        self.fs = r[R["fs"]:R["fs"] + d].t()
        self.grad_term = r[R["grad"]:R["grad"] + d].t()
        self.rel = r[R["rel"]:R["rel"] + d].t()
        self.force = None
        if tree_level0 is not None:
            base = tree_level0.index["f" + "x"]
            self.force = tree_level0.data[base:base + d, :n].t()


# -- the reference's standalone coupling functions (coupling.py:96-322) -------------
# Each is one mlbm_coupling_op pass over the level-0 raster of a MpmGrid (the
# fused CoupledSim step runs the same device functions inside mlbm_exchange).
# Arrays are level-0 cell vectors in this topology's cell order (device tensors
# or host arrays); results are device tensors.

def _seam_grid(topology, dtype=None):
    """A level-0 raster for the standalone seams: faces follow the topology's
    periodicity (non-periodic faces as outlets: no solids, no wall bands)."""
    from .solver import BoundarySpec
    faces = {}
    for a, ax in enumerate("xyz"[:topology.d]):
        kind = "periodic" if topology.periodic[a] else "outlet"
        faces[ax + "_min"] = faces[ax + "_max"] = kind
    return MpmGrid(topology, BoundarySpec(faces=faces, dim=topology.d), dtype=dtype)


def _cell_vec(v, grid, n):
    t = torch.as_tensor(v if torch.is_tensor(v) else np.asarray(v, dtype=np.float64),
                        dtype=grid.dtype, device=grid.ras.device).reshape(-1)
    if t.numel() != n:
        raise ValueError(f"expected {n} level-0 cell values, got {t.numel()}")
    return t.contiguous()


def _cell_rows(vs, grid, n):
    return torch.stack([_cell_vec(v, grid, n) for v in vs]).contiguous()


def _couple(grid, op, a0=None, u=None, out=None, eps_min=0.3, nu=1.0, d_p=1.0, re_min=0.01,
            dt=1.0, rho0=1.0, g=(0.0, 0.0, 0.0)):
    lv0 = grid.level0()
    L.check(L.lib().mlbm_coupling_op(
        L.C.byref(lv0), op, L.ptr(grid.ras), grid.ras.stride(0), L.ptr(a0),
        L.ptr(u), u.stride(0) if u is not None else 0, L.ptr(out),
        out.stride(0) if out is not None else 0, float(eps_min), float(nu), float(d_p),
        float(re_min), float(dt), float(rho0), _d3(g, grid.d), dtype_code(grid.dtype),
        L.stream_handle()), "coupling_op")


def rasterize_fractions(particles: Particles, topology, phi, eps_min: float,
                        drag: "DragParams" = None, st=None, grid: MpmGrid | None = None):
    """coupling.py:96-131: B-spline rasterisation of the sediment fraction,
    mass, cell velocity and cross-section area (the P2G scatter), then
    eps = clip(1 - eta_eff - phi, eps_min, 1).  Returns CouplingFields views of
    the grid raster (``grid`` defaults to a fresh MpmGrid of the topology)."""
    grid = grid or _seam_grid(topology, particles.dtype)
    grid.sync_topology()
    grid.clear()
    n = topology.cell_count(0)
    if len(particles):
        lv0 = grid.level0()
        # zero elastic moduli: the stress rows stay zero, the rest is the P2G scatter
        L.check(L.lib().mlbm_p2g(L.C.byref(lv0), len(particles), L.ptr(particles.xd),
                                 L.ptr(particles.pd), particles.pd.stride(0), 0.0, 0.0, 0.0,
                                 L.ptr(grid.ras), grid.ras.stride(0), dtype_code(grid.dtype), 0,
                                 L.ptr(grid._err), L.stream_handle()), "p2g")
        grid.raise_pending()
    _couple(grid, L.COUPLE_FRACTIONS, a0=_cell_vec(phi, grid, n), eps_min=eps_min)
    return CouplingFields(grid)


def difelice_drag(fields: CouplingFields, rho, ux, uy, nu: float, params: "DragParams",
                  d_p: float, uz=None):
    """coupling.py:134-156: Di Felice drag on the sediment per cell (fields.fs,
    fields.rel); the fluid receives -fs.  3D passes ``uz``."""
    grid = fields.grid
    n = grid._live()
    u = _cell_rows([ux, uy] + ([uz] if grid.d == 3 else []), grid, n)
    _couple(grid, L.COUPLE_DRAG, a0=_cell_vec(rho, grid, n), u=u, nu=nu, d_p=d_p,
            re_min=params.re_min)
    return fields.fs


def limit_drag(fields: CouplingFields, rho, ux, uy, dt: float, uz=None):
    """CoupledSim._limit_drag (coupling.py:379-401) on fields.fs, in place."""
    grid = fields.grid
    n = grid._live()
    u = _cell_rows([ux, uy] + ([uz] if grid.d == 3 else []), grid, n)
    _couple(grid, L.COUPLE_LIMIT, a0=_cell_vec(rho, grid, n), u=u, dt=dt)


def grad_eps(eps, topology, grid: MpmGrid | None = None):
    """coupling.py:159-182: central differences on level 0 (a missing
    neighbour counts as the cell itself); returns (n, d)."""
    grid = grid or _seam_grid(topology)
    n = topology.cell_count(0)
    e = _cell_vec(eps, grid, n)
    out = torch.empty((grid.d, n), dtype=grid.dtype, device=grid.ras.device)
    _couple(grid, L.COUPLE_GRAD_EPS, a0=e, out=out)
    return out.t()


def mixture_force(fields: CouplingFields, rho, topology, gravity, rho0: float = 1.0):
    """coupling.py:185-197: ((rho - rho0)/eps) grad eps + rho g - fs; sets
    fields.grad_term and fields.force, returns the force (n, d)."""
    grid = fields.grid
    n = grid._live()
    out = torch.empty((grid.d, n), dtype=grid.dtype, device=grid.ras.device)
    _couple(grid, L.COUPLE_MIXTURE_FORCE, a0=_cell_vec(rho, grid, n), out=out, rho0=rho0,
            g=tuple(gravity))
    fields.force = out.t()
    return fields.force


def powder_step(phi, ux, uy, topology, params: "PowderParams", dt: float, source=None, uz=None):
    """coupling.py:230-272: RK3 semi-Lagrangian advection with multilinear
    sampling, forward-Euler diffusion (params.sign), then + dt * source.
    Returns the new phi (n,) as a device tensor."""
    from .sparse_grid import field_names, fresh_block
    params.check_stability(dt)
    d = topology.d
    n = topology.cell_count(0)
    cap = topology.capacity_cells(0)
    dt_ = torch.float64 if (torch.is_tensor(phi) and phi.dtype == torch.float64) or \
        not torch.is_tensor(phi) else phi.dtype
    names = field_names(d)
    src = fresh_block(d, cap, dt_, topology.device)
    dst = fresh_block(d, cap, dt_, topology.device)

    def put(block, row, v):
        t = torch.as_tensor(v if torch.is_tensor(v) else np.asarray(v, dtype=np.float64),
                            dtype=dt_, device=topology.device).reshape(-1)
        block[row, :n].copy_(t)
    put(src, names.index("phi"), phi)
    for a, v in enumerate([ux, uy] + ([uz] if d == 3 else [])):
        put(dst, 1 + a, v)
    srcv = None
    if source is not None:
        srcv = torch.zeros(cap, dtype=dt_, device=topology.device)
        srcv[:n].copy_(torch.as_tensor(source if torch.is_tensor(source) else
                                       np.asarray(source, dtype=np.float64), dtype=dt_).reshape(-1))
    tmp = torch.empty(cap, dtype=dt_, device=topology.device)
    lv0 = topology.level_struct(0)
    L.check(L.lib().mlbm_powder_step(L.C.byref(lv0), L.fields(src), L.fields(dst), L.ptr(tmp),
                                     float(params.diffusion), float(params.sign), float(dt),
                                     L.ptr(srcv), dtype_code(dt_), L.stream_handle()),
            "powder_step")
    return dst[names.index("phi"), :n].clone()


class CoupledSim:
    """Owns the solver, the granular phase and the exchange (coupling.py:337-538)."""

    def __init__(self, solver: MultiLevelSolver, particles: Particles | None,
                 material: SandMaterial | None = None, sediment_gravity=None,
                 drag: DragParams | None = None, powder: PowderParams | None = None,
                 adaptor: GridAdaptor | None = None, static_tiles=None,
                 unit_scale: UnitScale | None = None):
        self.solver = solver
        self.topology = solver.topology
        self.d = self.topology.d
        self.pair = solver.pair
        self.dtype = solver.dtype
        self.particles = particles if particles is not None else \
            Particles(0, self.d, self.dtype, self.topology.device)
        self.material = material or SandMaterial()
        self.drag_params = drag or DragParams()
        self.powder = powder
        self.adaptor = adaptor
        self.static_tiles = static_tiles
        self.unit_scale = unit_scale or UnitScale()
        g = sediment_gravity if sediment_gravity is not None else solver.params.gravity
        self.sediment_gravity = np.asarray(g, dtype=float)
        self.grid = MpmGrid(self.topology, solver.boundaries, self.dtype,
                            tables=lambda: solver.tables(0))
        self.cadence = solver.params.mpm_cadence
        self.step_count = 0
        self.threads = 1
        self.clamped_particles = 0
        self.last_fields = None
        self._diag_rows = []
        self._tmp = None
        self.last_report = None
        # [fluid momentum d][sum phi][eps min][sediment momentum d][drag impulse d]
        self._diag_buf = torch.zeros(3 * self.d + 2, dtype=torch.float64,
                                     device=self.topology.device)
        # CUDA-graph step: one graph per (cycle, buffer parities,
        # exchange kind), recaptured after every topology change
        # one int32 block holding every device status word of the step (error
        # records, counters, adapt flags) -> a single D2H copy per step
        ne = L.ERR_INTS
        nst = 3 * self.topology.levels + 4 if adaptor is not None else 0
        self._sblock = torch.zeros(2 * ne + 2 + nst + (ne if adaptor is not None else 0),
                                   dtype=torch.int32, device=self.topology.device)
        self._sblock[:ne].copy_(solver._err)
        solver._err = self._sblock[:ne]
        self.grid._err = self._sblock[ne:2 * ne]
        self._counters = self._sblock[2 * ne:2 * ne + 2]
        if adaptor is not None:
            adaptor._status = self._sblock[2 * ne + 2:2 * ne + 2 + nst]
            adaptor._err = self._sblock[2 * ne + 2 + nst:]
        self.use_graphs = True
        self.sort_particles = True
        # particles move < 1 cell/step: re-sort every few steps (P2G / G2P only
        # need same-cell particles to be mostly adjacent)
        self.sort_every = int(os.environ.get("MLBM_SORT_EVERY", "16"))
        self._sort_now = True
        self._use_sorted = self._sort_ahead = self._sorted_ahead = False
        self.overlap_diag = os.environ.get("MLBM_OVERLAP_DIAG", "1") != "0"
        self._fork_pdiag = self._pdiag_forked = False
        # graphs of this many upcoming steps are captured whenever capacities
        # change (first step included), so steady stepping only replays: two
        # sort periods + 1, so the keys of the first sorted steps (which
        # differ from the unsorted start) are among them (a 35 ms capture
        # otherwise lands on step 16)
        self.precapture_steps = int(os.environ.get("MLBM_PRECAPTURE", str(2 * self.sort_every + 1))) or None
        # a rebuild key runs eagerly this many times before its graph is
        # captured (a capture costs a few ms of host time)
        self.rebuild_capture_after = int(os.environ.get("MLBM_REBUILD_CAPTURE_AFTER", "1"))
        self.latest_only_rebuild = os.environ.get("MLBM_LATEST_ONLY_REBUILD", "1") != "0"
        self.latest_only_min_cells = 1 << 22
        # MLBM_FUSE_L0=1: the level-0 coupled phase as P2G -> ONE stream +
        # exchange + collide kernel -> G2P.  Measured on C4 it is no faster
        # than the three kernels (the exchange's neighbour gathers lose the
        # separate kernel's occupancy: 1.97 vs 1.88 ms per step; graph step
        # 23.0 vs 22.1 ms), so the separate kernels stay the default.
        self.fuse_level0 = os.environ.get("MLBM_FUSE_L0", "0") == "1"
        self.p2g_mode = 4          # sorted input: 1 block smem, 2 warp registers, 3 cell lanes,
                                   # 4 cell lanes + per-warp box copies (fp32; fp64 runs mode 3),
                                   # 5 = 4 with two rounds of particles per block
        if particles is not None and len(particles) and self.dtype == torch.float32:
            # dense sampling (>= 8 particles per cell, V0 = 1 / per_cell): two
            # rounds per block share one node box (-8 % P2G time on C3 / C4)
            v0 = float(particles.V0.double().mean().item())
            if v0 > 0.0 and 1.0 / v0 >= 7.5:
                self.p2g_mode = 5
        self._graphs = {}
        self._graph_ver = None
        self._pool = None
        self.graph_replays = 0
        self.graph_captures = 0
        self.step_graph_captures = self.rebuild_graph_captures = 0
        self.topology_changes = 0
        self.rebuild_eager = 0
        self.rebuild_replays = 0
        self._pending_row = None
        if self.drag_params.d_p is None and len(self.particles):
            self.drag_params.d_p = float(particle_diameter(float(self.particles.V0.double().mean()),
                                                           self.d))
        if self.powder is not None:
            self.powder.check_stability(1.0)

    @property
    def coupling_active(self) -> bool:
        return len(self.particles) > 0

    @property
    def cfl_flags(self):
        return int(self._cfl)

    # -- exchange ------------------------------------------------------------------
    def _exchange(self, solver):
        """The coupling hook (coupling.py:403-446) as three launches between
        the level-0 stream and collide: P2G, the exchange, G2P."""
        self._p2g_phase(solver)
        self._exchange_kernel(solver)
        self._g2p_phase(solver)
        return FIELD_FORCE, FIELD_TAU

    def _p2g_phase(self, solver):
        grid = self.grid
        grid.sync_topology()
        p = self.particles
        mat = self.material
        lv0 = grid.level0()
        grid.clear()
        n = len(p)
        ps = p.pd.stride(0)
        if self.sort_particles and n and (self._sort_now or self._use_sorted):
            xa, pa, ida, ws = p.scratch()
            if not self._use_sorted:          # else sorted at the end of the last step
                self._sort_into_scratch()
            src_x, src_p, src_id, smem = xa, pa, ida, self.p2g_mode
            p.permuted = True
        else:
            src_x, src_p, src_id = p.xd, p.pd, None
            smem = self.p2g_mode if (self.sort_particles and p.permuted) else 0
        self._p2g_src = (src_x, src_p, src_id)
        L.check(L.lib().mlbm_p2g(L.C.byref(lv0), n, L.ptr(src_x), L.ptr(src_p), ps,
                                 mat.lam, mat.mu, mat.alpha, L.ptr(grid.ras), grid.ras.stride(0),
                                 dtype_code(self.dtype), smem, L.ptr(grid._err),
                                 L.stream_handle()), "p2g")
        solver.launches += 1

    def _exchange_args(self, solver):
        sp = solver.params
        return (float(sp.eps_min), float(solver.level_params.nu(0)),
                float(self.drag_params.d_p or 1.0), float(self.drag_params.re_min),
                float(self.cadence), float(sp.rho0), _d3(sp.gravity, self.d),
                _d3(self.sediment_gravity, self.d), _faces(solver.boundaries),
                float(self.material.floor_friction))

    def _exchange_kernel(self, solver):
        r, w = solver.roles(0)
        grid = self.grid
        L.check(L.lib().mlbm_exchange(L.C.byref(grid.level0()), L.fields(solver.arrays(w, 0).data),
                                      L.fields(solver.arrays(r, 0).data),
                                      L.fields(self.pair.trees[0].levels[0].data),
                                      L.fields(self.pair.trees[1].levels[0].data),
                                      L.ptr(grid.ras), grid.ras.stride(0),
                                      *self._exchange_args(solver), 1, dtype_code(self.dtype),
                                      L.stream_handle()), "exchange")
        solver.launches += 1

    def _level0_coupled(self, solver):
        """Level-0 stream + exchange + collide + boundaries in ONE kernel
        (mlbm_level0_coupled, level_kernel mode 5): the exchange of each cell
        runs on its bare post-stream moments in registers."""
        r, w = solver.roles(0)
        grid = self.grid
        solver._refresh_tables()
        cp = solver._collide_struct(0, force_mode=1, tau_mode=1)
        L.check(L.lib().mlbm_level0_coupled(
            L.C.byref(solver._structs[0]), L.fields(solver.arrays(r, 0).data),
            L.fields(solver.arrays(w, 0).data), L.fields(self.pair.trees[0].levels[0].data),
            L.fields(self.pair.trees[1].levels[0].data), dtype_code(self.dtype), L.C.byref(cp),
            L.C.byref(solver._bc), L.ptr(grid.ras), grid.ras.stride(0), *self._exchange_args(solver),
            L.ptr(solver._err), L.stream_handle()), "level0_coupled")
        solver.launches += 1

    def _g2p_phase(self, solver):
        grid = self.grid
        p = self.particles
        mat = self.material
        src_x, src_p, src_id = self._p2g_src
        seeds = self._g2p_seeds()
        ad = self.adaptor
        L.check(L.lib().mlbm_g2p(L.C.byref(grid.level0()), len(p), L.ptr(src_x), L.ptr(p.xd),
                                 L.ptr(src_p), L.ptr(p.pd), L.ptr(src_id),
                                 L.ptr(p.pid) if src_id is not None else L.ptr(None),
                                 p.pd.stride(0), mat.lam, mat.mu, mat.alpha, snow_arg(mat),
                                 L.ptr(grid.ras), grid.ras.stride(0), float(self.cadence), 1,
                                 dtype_code(self.dtype), L.ptr(self._counters),
                                 L.ptr(ad._seeds if seeds else None),
                                 L.ptr(self.topology.lv[0].kind if seeds else None),
                                 L.ptr(ad.ext_count if seeds else None),
                                 L.ptr(grid._err), L.stream_handle()), "g2p")
        solver.launches += 1
        self.last_fields = CouplingFields(grid, self.pair.trees[0].levels[0])
        if self._fork_pdiag:
            # graph step: the particle part of the diagnostics row (sum m v of
            # the new velocities, sum fs of this exchange) reads only what G2P
            # and the exchange wrote: it runs on the side stream concurrently
            # with the collide, the stress raster and the powder transport
            # (joined before the step's status copy)
            main = torch.cuda.current_stream()
            side = self._side_stream()
            fork = torch.cuda.Event()
            fork.record(main)
            side.wait_event(fork)
            with torch.cuda.stream(side):
                self._record_diagnostics(fluid=False)
            self._pdiag_forked = True

    def _hook(self):
        """The coupling hook for run_cycle: fused (P2G -> one level-0 kernel
        -> G2P) unless fuse_level0 is off."""
        return _CoupledHook(self) if self.fuse_level0 else self._exchange

    def _sort_into_scratch(self):
        """Radix sort of the particle rows by (level-0 tile slot, cell) into
        the scratch buffers (no reference counterpart; ordering only)."""
        p = self.particles
        lv0 = self.grid.level0()
        xa, pa, ida, ws = p.scratch(lv0.n_tiles)
        L.check(L.lib().mlbm_particle_sort(L.C.byref(lv0), len(p), L.ptr(p.xd), L.ptr(p.pd),
                                           L.ptr(p.pid), p.pd.stride(0), L.ptr(xa), L.ptr(pa),
                                           L.ptr(ida), dtype_code(self.dtype), L.ptr(ws),
                                           ws.numel(), L.stream_handle()), "particle_sort")
        self.solver.launches += 1

    @staticmethod
    def _held(solver):
        return FIELD_FORCE, FIELD_TAU

    def step(self):
        """One finest cycle of the coupled pipeline (coupling.py:448-481)."""
        solver = self.solver
        schedule = solver._schedule
        ci = solver.k[0] % len(schedule)
        is_mpm = self.coupling_active and (self.step_count % self.cadence == 0)
        adapt_now = self.adaptor is not None and self.coupling_active and \
            self.step_count % self.cadence == 0
        if self.particles is not None and (is_mpm or self.powder is not None):
            # P2G / the entrainment raster read the particles' stress rows
            self.particles.ensure_stress(self.material)
        if self.use_graphs and torch.cuda.is_available():
            self._step_graph(ci, is_mpm, adapt_now)
        else:
            self._step_eager(ci, is_mpm, adapt_now)
        self.step_count += 1

    # -- eager path (host checks after every phase) --------------------------------
    def _step_eager(self, ci, is_mpm, adapt_now):
        solver = self.solver
        self._sort_now = (self.step_count % self.sort_every) == 0
        self._use_sorted = False
        self._sort_ahead = self._sorted_ahead = False
        cycle = solver._schedule[ci]
        if is_mpm:
            solver.run_cycle(cycle, hook=self._hook())
        elif self.coupling_active:
            solver.run_cycle(cycle, hook=self._held)
        else:
            solver.run_cycle(cycle)
        if self.coupling_active and is_mpm:
            self.grid.raise_pending()
        if self.powder is not None:
            self._powder_cycle(is_mpm)
        # the particle part on the raster of this step's exchange (before the
        # rebuild renumbers the level-0 slots), the fluid part after the adapt;
        # a step without MPM keeps the last MPM step's particle part (the
        # particles and the last exchange's fields are unchanged)
        if is_mpm:
            self._record_diagnostics(fluid=False)
        if adapt_now:
            driver = self._driver()
            self.last_report = self.adaptor.update(driver, self.pair)
            if not self.last_report.noop:
                self.topology_changes += 1
            self.grid.sync_topology()
        self._record_diagnostics(particles=False)
        self._push_diag_row(self._diag_buf.cpu().numpy())

    def _g2p_seeds(self):
        """G2P writes the next adapt pass's seed tiles (fused cooperative pass
        only; the bit-packed and per-op paths seed from the positions)."""
        return (self.adaptor is not None and self.adaptor.fused and len(self.particles) > 0
                and not os.environ.get("MLBM_ADAPT_PATH", "").startswith("b"))

    def _driver(self):
        return RefineDriver(positions_soa=self.particles.xd, static_tiles=self.static_tiles,
                            levels=self.topology.levels, g2p_seeds=self._g2p_seeds())

    # -- graph path: all kernels of the step replayed as one CUDA graph, one
    #    device->host status copy, host work only when the topology changes --
    def _device_step(self, ci, is_mpm, adapt_now):
        solver = self.solver
        cycle = solver._schedule[ci]
        check = solver.check_errors
        solver.check_errors = False
        self._fork_pdiag = self.overlap_diag
        self._pdiag_forked = False
        try:
            if is_mpm:
                solver.run_cycle(cycle, hook=self._hook())
            elif self.coupling_active:
                solver.run_cycle(cycle, hook=self._held)
            else:
                solver.run_cycle(cycle)
        finally:
            solver.check_errors = check
            self._fork_pdiag = False
        if self.powder is not None:
            self._powder_cycle(is_mpm)
        # particles: already recorded on the side stream after G2P; a step
        # without MPM keeps the last MPM step's particle part (particles and
        # the last exchange's drag unchanged — recomputing it would read a
        # raster the rebuild may have renumbered)
        pdiag = is_mpm and not self._pdiag_forked
        if adapt_now and self.overlap_diag:
            # the diagnostics reductions read only fields and particles: they
            # run on a side stream concurrently with the latency-bound adapt
            # pass (both captured into the same graph, joined before the copy)
            main = torch.cuda.current_stream()
            side = self._side_stream()
            fork = torch.cuda.Event()
            fork.record(main)
            side.wait_event(fork)
            with torch.cuda.stream(side):
                self._record_diagnostics(particles=pdiag)
                if self._sort_ahead:
                    self._sort_into_scratch()
            self.adaptor.plan_device(self._driver())
            join = torch.cuda.Event()
            join.record(side)
            main.wait_event(join)
        else:
            if adapt_now:
                self.adaptor.plan_device(self._driver())
            if self._pdiag_forked:
                join = torch.cuda.Event()
                join.record(self._side_stream())
                torch.cuda.current_stream().wait_event(join)
            self._record_diagnostics(particles=pdiag)
        self._host_i32.copy_(self._sblock, non_blocking=True)
        self._host_f64.copy_(self._diag_buf, non_blocking=True)

    def _side_stream(self):
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.topology.device)
        return self._side

    def _ensure_host_status(self, adapt_now=None):
        if getattr(self, "_host_i32", None) is None:
            self._host_i32 = torch.zeros(self._sblock.numel(), dtype=torch.int32).pin_memory()
            self._host_f64 = torch.zeros(self._diag_buf.numel(), dtype=torch.float64).pin_memory()

    def _sort_flags(self, step, sorted_ahead, is_mpm, adapt_now):
        """(use_sorted, sort_now, sort_ahead) of a step.  Particle sort: every
        sort_every steps; with the diagnostics overlap it runs at the end of
        the previous step beside the adapt pass (it only reads the particle
        rows the pass reads) and this step's P2G takes the sorted scratch."""
        use_sorted = sorted_ahead
        sort_now = (step % self.sort_every) == 0 and not use_sorted
        sort_ahead = bool(self.overlap_diag and adapt_now and is_mpm and self.cadence == 1
                          and self.sort_particles and len(self.particles)
                          and (step + 1) % self.sort_every == 0)
        return use_sorted, sort_now, sort_ahead

    def _step_kinds(self, step):
        is_mpm = self.coupling_active and (step % self.cadence == 0)
        adapt_now = self.adaptor is not None and self.coupling_active and step % self.cadence == 0
        return is_mpm, adapt_now

    def _capture(self, key, ci, is_mpm, adapt_now, k, bounce, flags):
        """Capture the step graph of one key with the host state (level
        counters, bounce, sort flags) that step will have; restores it."""
        solver = self.solver
        if self._pool is None:
            self._pool = torch.cuda.graph_pool_handle()
        saved = (list(solver.k), self.pair.bounce, self._use_sorted, self._sort_now,
                 self._sort_ahead, self.last_fields)
        solver.k[:] = k
        self.pair.bounce = bounce
        self._use_sorted, self._sort_now, self._sort_ahead = flags
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        n0 = L.TRACE.launches
        tracing = L.TRACE.enabled
        L.TRACE.enabled = False
        try:
            with torch.cuda.graph(g, pool=self._pool):
                self._device_step(ci, is_mpm, adapt_now)
        finally:
            L.TRACE.enabled = tracing
        nk = L.TRACE.launches - n0
        L.TRACE.launches = n0          # captured, not executed
        dk = [a - b for a, b in zip(solver.k, k)]
        db = self.pair.bounce - bounce
        entry = (g, dk, db, self.last_fields, nk)
        (k0, self.pair.bounce, self._use_sorted, self._sort_now, self._sort_ahead,
         self.last_fields) = saved
        solver.k[:] = k0
        self._graphs[key] = entry
        self.graph_captures += 1
        self.step_graph_captures += 1
        return entry

    def _key(self, ci, k, is_mpm, adapt_now, flags, lf_set):
        use_sorted, sort_now, sort_ahead = flags
        return (ci, tuple((v + f) & 1 for v, f in zip(k, self.solver.flip)), is_mpm, adapt_now,
                sort_now, use_sorted, sort_ahead,
                self.powder is not None and is_mpm and lf_set)

    def _precapture(self, n):
        """Capture the graphs of the next ``n`` steps now (host state
        predicted from each graph's level-counter increments), so steady
        stepping replays only — re-run whenever capacities change."""
        solver = self.solver
        f0 = solver.flip[0]
        # a latest-only rebuild swaps level 0's trees: the graphs of both
        # placements are captured up front
        swaps = self.adaptor is not None and self.adaptor.latest_swap and self._latest_only()
        try:
            for f in ((f0, 1 - f0) if swaps else (f0,)):
                solver.flip[0] = f
                self._precapture_run(n)
        finally:
            solver.flip[0] = f0

    def _precapture_run(self, n):
        schedule = self.solver._schedule
        k = list(self.solver.k)
        b = self.pair.bounce
        sa = self._sorted_ahead
        lf = self.last_fields is not None
        for j in range(n):
            step = self.step_count + j
            ci = k[0] % len(schedule)
            is_mpm, adapt_now = self._step_kinds(step)
            flags = self._sort_flags(step, sa, is_mpm, adapt_now)
            key = self._key(ci, k, is_mpm, adapt_now, flags, lf)
            entry = self._graphs.get(key)
            if entry is None:
                entry = self._capture(key, ci, is_mpm, adapt_now, k, b, flags)
            k = [a + d for a, d in zip(k, entry[1])]
            b += entry[2]
            sa = flags[2]
            lf = lf or is_mpm

    def _step_graph(self, ci, is_mpm, adapt_now):
        solver = self.solver
        topo = self.topology
        gver = (topo.cap_version, tuple(topo.n_tiles(l) > 0 for l in range(topo.levels)))
        fresh = self._graph_ver != gver
        if fresh:
            self._graphs.clear()
            self._pool = None          # graphs of the old capacities freed with their pool
            self._graph_ver = gver
        # persistent buffers (and the side stream) are created outside any capture
        self._side_stream()
        if self.sort_particles and len(self.particles):
            self.particles.scratch(self.grid.level0().n_tiles)
        if self.powder is not None:
            self._powder_tmp()
        # refresh host-side tables / rasters before capture (may sync)
        solver._refresh_tables()
        self.grid.sync_topology()
        self.grid.level0()
        self._ensure_host_status(adapt_now)
        if self.adaptor is not None and self.adaptor.fused:
            self.adaptor.prepare_windows(self.static_tiles)   # syncs: never inside a capture
        if fresh and self.precapture_steps:
            self._precapture(self.precapture_steps)
        flags = self._sort_flags(self.step_count, self._sorted_ahead, is_mpm, adapt_now)
        self._use_sorted, self._sort_now, self._sort_ahead = flags
        key = self._key(ci, solver.k, is_mpm, adapt_now, flags, self.last_fields is not None)
        entry = self._graphs.get(key)
        if entry is None:
            entry = self._capture(key, ci, is_mpm, adapt_now, list(solver.k), self.pair.bounce,
                                  flags)
        g, dk, db, lf, nk = entry
        g.replay()
        self._sorted_ahead = self._sort_ahead
        L.TRACE.launches += nk
        self.graph_replays += 1
        for l, v in enumerate(dk):
            solver.k[l] += v
        self.pair.bounce += db
        if is_mpm:
            self.last_fields = lf
        torch.cuda.current_stream().synchronize()
        self._finish_graph_step(adapt_now)

    def _finish_graph_step(self, adapt_now):
        self._resolve_pending_diag()
        h = self._host_i32.numpy().astype(np.int64)
        ne = L.ERR_INTS
        serr, gerr = h[:ne], h[ne:2 * ne]
        diag = self._host_f64.numpy().copy()
        if serr[0]:
            self.solver._err.copy_(torch.as_tensor(serr, dtype=torch.int32))
            self.solver.raise_pending()
        if gerr[0]:
            self.grid._err.copy_(torch.as_tensor(gerr, dtype=torch.int32))
            self.grid.raise_pending()
        if adapt_now:
            nst = 3 * self.topology.levels + 4
            status = h[2 * ne + 2:2 * ne + 2 + nst]
            err = h[2 * ne + 2 + nst:]
            # level 0 steps once per finest cycle: of its two trees only the one
            # read next carries state (the other is rewritten by the next
            # stream / exchange before any read), so a rebuild migrates that one
            self.last_report = self.adaptor.finish(self._driver(), self.pair, status, err,
                                                   check_after=False,
                                                   device_runner=self._run_rebuild,
                                                   latest_only=self._latest_only())
            if not self.last_report.noop:
                # the rebuild graph re-takes this step's diagnostics on the new
                # topology (coupling.py:481) into a second pinned buffer; the row
                # is completed at the next synchronisation point
                self.topology_changes += 1
                self._push_diag_row(None)
                return
        self._push_diag_row(diag)

    def _latest_only(self):
        # it halves the level-0 migration but doubles the rebuild-graph keys
        # (the tree is part of the key): worth it only for large level 0s
        if not self.latest_only_rebuild or self.topology.capacity_cells(0) < self.latest_only_min_cells:
            return None
        # with mpm_cadence > 1 the held hook (coupling.py:460-465) reads the
        # force / eps rows of the write tree on the non-MPM steps: that tree
        # must migrate too
        if self.cadence > 1:
            return None
        return {0: self.solver.roles(0)[0]}

    def _run_rebuild(self, device_fn, key):
        """Device half of a topology change + the table rebuild as one CUDA
        graph per (capacities, rebuilt levels) — run eagerly the first time a
        key is seen (so every buffer it needs is allocated outside capture),
        captured and replayed after; then the diagnostics row of the step on
        the new topology (coupling.py:481) into a second pinned buffer."""
        solver = self.solver
        topo = self.topology
        self.grid.sync_topology()
        if getattr(self, "_host_rb", None) is None:
            self._host_rb = torch.zeros(self._diag_buf.numel(), dtype=torch.float64).pin_memory()
        full = (topo.cap_version, key, tuple(topo.n_tiles(l) > 0 for l in range(topo.levels)))
        if getattr(self, "_rb_ver", None) != topo.cap_version:
            self._rb_graphs, self._rb_seen, self._rb_ver = {}, set(), topo.cap_version
            self._rb_seen_n = {}

        # tables of the changed levels and of their neighbours (interfaces)
        changed = key[0] if key and isinstance(key[0], tuple) else key
        affected = sorted({m for l in changed for m in (l - 1, l, l + 1) if 0 <= m < topo.levels})

        def body():
            device_fn()
            solver._refresh_tables(only=affected)

        g = self._rb_graphs.get(full)
        seen = self._rb_seen_n.get(full, 0) if isinstance(getattr(self, "_rb_seen_n", None), dict) else 0
        if g is None and seen < self.rebuild_capture_after:
            # eager (the first time: every buffer allocated outside capture)
            self._rb_seen_n = getattr(self, "_rb_seen_n", None) or {}
            self._rb_seen_n[full] = seen + 1
            self._rb_seen.add(full)
            body()
            self.rebuild_eager += 1
        else:
            if g is None:
                if self._pool is None:
                    self._pool = torch.cuda.graph_pool_handle()
                g = torch.cuda.CUDAGraph()
                n0 = L.TRACE.launches
                tracing = L.TRACE.enabled
                L.TRACE.enabled = False
                try:
                    with torch.cuda.graph(g, pool=self._pool):
                        body()
                finally:
                    L.TRACE.enabled = tracing
                g.nk = L.TRACE.launches - n0
                L.TRACE.launches = n0
                self._rb_graphs[full] = g
                self.graph_captures += 1
                self.rebuild_graph_captures += 1
            g.replay()
            L.TRACE.launches += g.nk
            solver._tables_version = topo.version
            self.rebuild_replays += 1
        if self.adaptor.latest_swap:
            # latest-only levels now hold their latest values in the other tree
            for l, _ in (key[1] if key and isinstance(key[0], tuple) else ()):
                solver.flip[l] ^= 1
        # the step graph left this step's particle diagnostics in the buffer
        self._record_diagnostics(particles=False)
        self._host_rb.copy_(self._diag_buf, non_blocking=True)

    def _resolve_pending_diag(self):
        """Complete a diagnostics row whose values a rebuild graph is still
        copying (call after a stream synchronisation)."""
        if self._pending_row is not None:
            i = self._pending_row
            self._pending_row = None
            self._diag_rows[i] = self._make_diag_row(self._host_rb.numpy(),
                                                     *self._diag_rows[i])

    def _powder_tmp(self):
        n0 = self.topology.capacity_cells(0)
        if self._tmp is None or self._tmp.numel() != n0:
            self._tmp = torch.empty(n0, dtype=self.dtype, device=self.topology.device)
            # per-tile powder activity (the advection skips tiles with no phi
            # within reach)
            self._tile_ws = torch.empty(2 * self.topology.lv[0].cap, dtype=torch.uint8,
                                        device=self.topology.device)
        return self._tmp

    def _powder_cycle(self, is_mpm):
        solver = self.solver
        r, w = solver.last_roles(0)
        grid = self.grid
        lib = L.lib()
        s = L.stream_handle()
        dcode = dtype_code(self.dtype)
        self._powder_tmp()
        src = is_mpm and self.last_fields is not None and self.powder.entrain > 0.0 \
            and len(self.particles) > 0
        if src:
            R = grid.R
            L.zero(grid.ras[R["sig"]:R["etae"]])
            p = self.particles
            lv0 = grid.level0()
            # the raster is only read at entrainment surface cells: fp32 runs
            # restrict it to them (surface flags in the powder scratch, which
            # the advection overwrites afterwards); fp64 runs rasterise fully
            L.check(lib.mlbm_stress_raster_surface(
                L.C.byref(lv0), len(p), L.ptr(p.xd), L.ptr(p.pd), p.pd.stride(0),
                self.material.lam, self.material.mu, self.material.alpha, L.ptr(grid.ras),
                grid.ras.stride(0), float(self.powder.eta_surface), L.ptr(self._tmp), dcode,
                L.ptr(grid._err), s), "stress_raster")
            self._powder_stress_done()
        lv0 = solver._structs[0]
        pw = self.powder
        L.check(lib.mlbm_powder(L.C.byref(lv0), L.fields(solver.arrays(r, 0).data),
                                L.fields(solver.arrays(w, 0).data), L.ptr(grid.ras),
                                grid.ras.stride(0), L.ptr(self._tmp), L.ptr(self._tile_ws),
                                float(pw.diffusion),
                                float(pw.sign), 1.0, float(pw.entrain), float(pw.eta_surface),
                                1 if src else 0, dcode, s), "powder")
        self._powder_done()

    def _powder_stress_done(self):
        """Hook after the entrainment stress raster (the slab step sums the
        ghost-node stress of its neighbours here)."""

    def _powder_done(self):
        """Hook after the powder transport (the slab step refreshes the ghost
        columns of phi here)."""

    # -- diagnostics -------------------------------------------------------------------
    def _record_diagnostics(self, fluid=True, particles=True):
        """Device reductions of coupling.py:500-531 into a persistent buffer.
        The fluid part (leaf-weighted momentum, sum phi, eps min) depends on
        the topology; the particle part (momentum, drag impulse of the last
        exchange) does not — after a rebuild only the fluid part is retaken."""
        solver = self.solver
        d = self.d
        lib = L.lib()
        s = L.stream_handle()
        dcode = dtype_code(self.dtype)
        out = self._diag_buf
        if fluid:
            L.zero(out[:d + 2])
            L.fill(out[d + 1:d + 2], 1.0)
        if particles:
            L.zero(out[d + 2:])
        for l in range(self.topology.levels if fluid else 0):
            if not self.topology.n_tiles(l):
                continue
            lw = solver.last_roles(l)[1] if solver.k[l] else 0
            a = solver.arrays(lw, l)
            L.check(lib.mlbm_diag_level(L.C.byref(solver._structs[l]), L.fields(a.data),
                                        float((1 << d) ** l), dcode, L.ptr(out[:d + 2]), s),
                    "diag_level")
        if not particles:
            return
        p = self.particles
        g = self.grid
        n0 = self.topology.capacity_cells(0) if self.last_fields is not None else 0
        L.check(lib.mlbm_diag_particles(d, len(p), L.ptr(p.pd), p.pd.stride(0), L.ptr(g.ras),
                                        g.ras.stride(0), n0, L.ptr(self.topology.dcounts[0]),
                                        dcode, L.ptr(out[d + 2:]), s),
                "diag_particles")

    def _make_diag_row(self, o, step, tiles):
        d = self.d
        return DiagRow(
            step=step, t_phys=step * self.unit_scale.dt,
            fluid_mom=tuple(float(v) for v in o[:d]),
            sediment_mom=tuple(float(v) for v in o[d + 2:2 * d + 2]),
            drag_impulse=tuple(float(-v) for v in o[2 * d + 2:3 * d + 2]),
            sum_phi=float(o[d]),
            tiles=tiles,
            eps_min=float(o[d + 1]))

    def _push_diag_row(self, o):
        """Append this step's row; ``o is None``: values pending in the
        rebuild buffer (completed by ``_resolve_pending_diag``)."""
        step = self.step_count + 1
        tiles = tuple(self.topology.n_tiles(l) for l in range(self.topology.levels))
        if o is None:
            self._pending_row = len(self._diag_rows)
            self._diag_rows.append((step, tiles))
        else:
            self._diag_rows.append(self._make_diag_row(o, step, tiles))

    @property
    def diagnostics(self):
        if self._pending_row is not None:
            torch.cuda.current_stream().synchronize()
            self._resolve_pending_diag()
        return self._diag_rows

    def fluid_momentum(self):
        rows = self.diagnostics
        if not rows:
            self._record_diagnostics()
            o = self._diag_buf.cpu().numpy()
            return np.array(o[:self.d])
        return np.array(rows[-1].fluid_mom)

    @property
    def _cfl(self):
        return int(self._counters[1].item())


class _CoupledHook:
    """run_cycle hook of a coupled MPM step: called as a plain hook it runs the
    exchange between stream and collide (coupling.py:403-446); run_cycle uses
    its fused form — pre (P2G), one level-0 stream + exchange + collide kernel,
    post (G2P)."""

    def __init__(self, sim):
        self.sim = sim

    def __call__(self, solver):
        return self.sim._exchange(solver)

    def pre(self, solver):
        self.sim._p2g_phase(solver)

    def level0(self, solver):
        self.sim._level0_coupled(solver)

    def post(self, solver):
        self.sim._g2p_phase(solver)
