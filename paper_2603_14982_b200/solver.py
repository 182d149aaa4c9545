"""Multi-level moment-space LBM on the B200 (drop-in for solver.py).

Class / method names, arguments and error behaviour follow
``pkg/src/mlbm/solver.py``; every data-parallel kernel runs as hand-written
sm_100a CUDA through the C ABI (``include/mlbm_b200.h``):

  ======================================  =============================================
  reference seam                          B200 kernel
  ======================================  =============================================
  stream_kernel      solver.py:336-381    mlbm_level_step(mode=1)
  collide_kernel     solver.py:394-453    mlbm_level_step(mode=3)
  boundary_kernel    solver.py:460-481    mlbm_level_step(mode=4)
  stream_collide     solver.py:483-488    mlbm_level_step(mode=0)   fused, one pass
  downward_kernel    solver.py:501-526    mlbm_downward
  upward_kernel      solver.py:536-560    mlbm_upward
  _LevelTables       solver.py:177-274    mlbm_classify_level + mlbm_build_interface
  ======================================  =============================================

The schedule (Alg. 1 linearisation, buffer roles) is the reference's
(solver.py:564-649) issued from the host; divergence is detected on the
device and raised as DivergenceError after the cycle.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .lattice import CS2, H3_XYZ_HERMITE, H3_XYZ_PAPER, DivergenceError
from .sparse_grid import (TILE, LevelFields, PingPongPair, Topology, TopologyError,
                          buffer_roles, dtype_code, field_names)

RESCALE_DERIVED = "derived"
RESCALE_PAPER_LITERAL = "paper_literal"


def rescale_tau(tau_l: float, k: int) -> float:
    """Relaxation time k levels coarser (solver.py:34-36)."""
    return tau_l / 2.0 ** k + (2.0 ** k - 1.0) / 2.0 ** (k + 1)


def _kappa_up(tau_l, tau_lp1, convention):
    if convention == RESCALE_DERIVED:
        return 2.0 * tau_lp1 / tau_l
    if convention == RESCALE_PAPER_LITERAL:
        return tau_lp1 / (2.0 * tau_l)
    raise ValueError(f"unknown rescale convention {convention!r}")


def _kappa_down(tau_l, tau_lp1, convention):
    if convention == RESCALE_DERIVED:
        return tau_l / (2.0 * tau_lp1)
    if convention == RESCALE_PAPER_LITERAL:
        return 2.0 * tau_lp1 / tau_l
    raise ValueError(f"unknown rescale convention {convention!r}")


def _seq(u):
    u = np.asarray(u, dtype=float)
    d = u.shape[-1]
    return np.stack([u[..., a] * u[..., b] for a in range(d) for b in range(a, d)], axis=-1)


def rescale_s_up(s, u, tau_l, tau_lp1, convention=RESCALE_DERIVED):
    """Fine -> coarse S rescale (solver.py:55-59); host helper."""
    eq = _seq(u)
    return _kappa_up(tau_l, tau_lp1, convention) * (np.asarray(s, float) - eq) + eq


def rescale_s_down(s, u, tau_l, tau_lp1, convention=RESCALE_DERIVED):
    eq = _seq(u)
    return _kappa_down(tau_l, tau_lp1, convention) * (np.asarray(s, float) - eq) + eq


@dataclass
class LevelParams:
    """Per-level lattice scales (solver.py:70-91)."""
    levels: int
    tau0: float
    taus: list = field(default_factory=list)

    def __post_init__(self):
        if self.tau0 <= 0.5:
            raise ValueError(f"tau0 must exceed 1/2, got {self.tau0}")
        self.taus = [rescale_tau(self.tau0, l) for l in range(self.levels)]

    def dx(self, level):
        return float(1 << level)

    def dt(self, level):
        return float(1 << level)

    def nu(self, level):
        return CS2 * (self.taus[level] - 0.5)


@dataclass
class SolverParams:
    """solver.py:93-111 plus the 3D Hermite xyz coefficient."""
    levels: int
    rho0: float = 1.0
    gravity: tuple = (0.0, 0.0)
    eps_min: float = 0.3
    mpm_cadence: int = 1
    rescale_convention: str = RESCALE_DERIVED
    upward_mode: str = "coincident"
    h3_xyz: float = H3_XYZ_HERMITE

    def __post_init__(self):
        if self.levels < 1:
            raise ValueError("levels must be >= 1")
        if not 0.0 < self.eps_min < 1.0:
            raise ValueError("eps_min must lie in (0, 1)")
        if self.mpm_cadence < 1:
            raise ValueError("mpm_cadence must be >= 1")
        if self.upward_mode not in ("coincident", "average"):
            raise ValueError("upward_mode must be 'coincident' or 'average'")


FACES = ("x_min", "x_max", "y_min", "y_max", "z_min", "z_max")
_FACE_KIND = {"periodic": 0, "wall": 1, "outlet": 2}


def faces_for(d):
    return FACES[:2 * d]


@dataclass
class LogInlet:
    u0: float
    beta: float
    y0: float


@dataclass
class BoundarySpec:
    """Per-face condition + static solids (solver.py:121-156).

    ``solid_boxes`` are (lo..., hi...) in finest cells (2D: (x0, y0, x1, y1)
    exactly as the reference); ``heightmap`` (finest x[, z]) marks cells whose
    corner y lies below h as solid (config.py:161-165's heightfield).
    """
    faces: dict = None
    solid_boxes: list = field(default_factory=list)
    heightmap: np.ndarray | None = None
    dim: int = 2

    def __post_init__(self):
        if self.faces is None:
            self.faces = {f: "periodic" for f in faces_for(self.dim)}
        else:
            if any(k in self.faces for k in ("z_min", "z_max")):
                self.dim = 3
            for f in faces_for(self.dim):
                self.faces.setdefault(f, "periodic")

    def validate(self, finest_cells):
        d = len(finest_cells)
        for a in "xyz"[:d]:
            pa = self.faces[a + "_min"] == "periodic"
            pb = self.faces[a + "_max"] == "periodic"
            if pa != pb:
                raise ValueError(f"faces {a}_min/{a}_max must both be periodic or neither")
        for face, cond in self.faces.items():
            if isinstance(cond, LogInlet):
                if face != "x_min":
                    raise ValueError("log inlet is supported on the x_min face")
                if not 0 <= cond.y0 < finest_cells[1]:
                    raise ValueError("log inlet y0 outside the domain height")
            elif cond not in ("periodic", "wall", "outlet"):
                raise ValueError(f"unknown boundary condition {cond!r} on {face}")
        if len(self.solid_boxes) > 16:
            raise ValueError("at most 16 solid boxes (use a heightmap)")

    def periodic_axes(self, d=None):
        d = d or self.dim
        return tuple(self.faces[a + "_min"] == "periodic" for a in "xyz"[:d])

    def bc_struct(self, rho0):
        bc = L.BC()
        for i, f in enumerate(FACES):
            cond = self.faces.get(f, "periodic")
            if isinstance(cond, LogInlet):
                bc.face[i] = 3
                bc.inlet_u0, bc.inlet_beta, bc.inlet_y0 = cond.u0, cond.beta, cond.y0
            else:
                bc.face[i] = _FACE_KIND[cond]
        bc.rho0 = rho0
        return bc

    def solid_struct(self, d, device):
        s = L.Solid()
        s.n_boxes = len(self.solid_boxes)
        for b, box in enumerate(self.solid_boxes):
            for a in range(d):
                s.boxes[b][a] = float(box[a])
                s.boxes[b][3 + a] = float(box[d + a])
        self._hm = None
        if self.heightmap is not None:
            hm = np.asarray(self.heightmap, dtype=np.float32)
            if hm.ndim == 1:
                hm = hm[:, None]
            self._hm = torch.as_tensor(hm, device=device).contiguous()
            s.heightmap = self._hm.data_ptr()
            s.hm_dims[0] = hm.shape[0]
            s.hm_dims[1] = hm.shape[1]
        return s


class _LevelTables:
    """Device classification of one level (solver.py:177-274)."""

    def __init__(self, n_cells, n_tiles, device):
        self.cell_flags = L.zeros(n_cells, torch.uint8, device)
        self.dir_masks = L.zeros(n_cells, torch.int64, device)
        self.tile_flags = L.zeros(n_tiles, torch.uint8, device)
        self.down = None   # (targets, src, n)
        self.up = None

    def active_mask(self):
        return (self.cell_flags & 1).bool()


def build_tables(topo: Topology, bc, solid, err, tables=None, only=None):
    """Classify every level (flags, bounce-back masks, interface stencils) on
    the device (solver.py:177-274 + sparse_grid.py:468-544).  Buffers are
    (re)allocated only when a level's capacity changed; counts of I^d / I^u go
    to ``topo.dcounts[l, 2:4]``.  No host synchronisation: violations land in
    ``err`` and are raised by the caller's next status check.  ``only``
    restricts the classification and interface builds to a set of levels
    (those whose own or adjacent kind grids changed); the others keep theirs."""
    lib = L.lib()
    s = L.stream_handle()
    T = TILE ** topo.d
    tables = dict(tables or {})
    fresh = set()                       # levels whose tables are (re)allocated here

    def fresh_ok(t, l):
        return l not in fresh
    if not hasattr(topo, "_dirty"):
        topo._dirty, topo._dirty_changed = None, set()
    hier = topo.hier_struct()
    NC = 1 << topo.d
    scratch = torch.zeros((topo.levels, 2), dtype=torch.int32, device=topo.device) \
        if not hasattr(topo, "_cls_counts") else topo._cls_counts
    topo._cls_counts = scratch
    for l in range(topo.levels):
        cap = topo.lv[l].cap
        t = tables.get(l)
        if t is None or t.cap != cap:
            t = _LevelTables(cap * T, cap, topo.device)
            t.cap = cap
            t.down = (L.zeros(cap * T, torch.int32, topo.device),
                      L.full((cap * T, NC), -1, torch.int32, topo.device), cap * T)
            t.up = (L.zeros(cap * T, torch.int32, topo.device),
                    L.full((cap * T, NC), -1, torch.int32, topo.device), cap * T)
            tables[l] = t
            fresh.add(l)
        if not cap or (only is not None and l not in only):
            continue
        lvs = topo.level_struct(l)
        # incremental after a topology change (adapt._prepare left the dirty
        # maps): tiles with no kind change within one tile at any level copy
        # their classification from the old arrays
        dirty = (topo._dirty or {}).get(l) if only is not None and fresh_ok(t, l) else None
        prev = (None,) * 4
        if dirty is not None:
            if getattr(t, "prev", None) is None or t.prev[0].numel() != t.cell_flags.numel():
                t.prev = (torch.empty_like(t.cell_flags), torch.empty_like(t.dir_masks),
                          torch.empty_like(t.tile_flags))
            for a, b in zip(t.prev, (t.cell_flags, t.dir_masks, t.tile_flags)):
                L.copy(a, b)
            old_slot = topo.lv[l].old_slot if l in topo._dirty_changed else None
            prev = (old_slot,) + t.prev
            if getattr(t, "cls_work", None) is None or t.cls_work.numel() < cap + 1:
                t.cls_work = L.zeros(cap + 1, torch.int32, topo.device)
        work = t.cls_work if dirty is not None else None
        L.check(lib.mlbm_classify_level(L.C.byref(lvs), L.C.byref(hier), L.C.byref(bc),
                                        L.C.byref(solid), L.ptr(t.cell_flags),
                                        L.ptr(t.dir_masks), L.ptr(t.tile_flags),
                                        L.ptr(scratch[l]), L.ptr(err), L.ptr(dirty),
                                        *[L.ptr(x) for x in prev], L.ptr(work), s), "classify_level")
    for l, t in tables.items():
        if not topo.lv[l].cap or (only is not None and l not in only):
            continue
        for which, other in ((0, l + 1), (1, l - 1)):
            cnt = topo.dcounts[l, 2 + which:3 + which]
            if other < 0 or other >= topo.levels or not topo.lv[other].cap:
                L.zero(cnt)                  # cudaMemsetAsync: no framework kernel in the graph
                continue
            tg, src, _ = t.down if which == 0 else t.up
            ws = topo.workspace(topo.capacity_cells(l))
            lv_a = topo.level_struct(l, t)
            lv_b = topo.level_struct(other, tables[other])
            L.check(lib.mlbm_build_interface(L.C.byref(lv_a), L.C.byref(lv_b), which,
                                             L.ptr(tg), L.ptr(src), L.ptr(cnt), L.ptr(err),
                                             L.ptr(ws), ws.numel(), s), "build_interface")
    topo._dirty, topo._dirty_changed = None, set()       # consumed
    return tables


class MultiLevelSolver:
    """Owns the kernels and the recursion schedule (solver.py:277-612)."""

    def __init__(self, topology: Topology, pair: PingPongPair, params: SolverParams,
                 level_params: LevelParams, boundaries: BoundarySpec | None = None):
        if params.levels != topology.levels:
            raise ValueError("params.levels must match the topology")
        self.topology = topology
        self.d = topology.d
        self.pair = pair
        self.params = params
        if len(params.gravity) < self.d:
            params.gravity = tuple(params.gravity) + (0.0,) * (self.d - len(params.gravity))
        self.level_params = level_params
        self.boundaries = boundaries or BoundarySpec(dim=self.d)
        self.boundaries.validate(topology.finest_cells)
        self.dtype = pair.dtype
        self.dcode = dtype_code(self.dtype)
        self.k = [0] * topology.levels
        # per level: 1 when the level's two trees swapped places (a latest-only
        # rebuild migrated the latest tree into the other one's storage)
        self.flip = [0] * topology.levels
        self._tables_version = -1
        self._tables = {}
        self.check_errors = True
        self._err = torch.zeros(L.ERR_INTS, dtype=torch.int32, device=topology.device)
        self._bc = self.boundaries.bc_struct(params.rho0)
        self._solid = self.boundaries.solid_struct(self.d, topology.device)
        self._near_maps = []
        if self._solid.n_boxes or self._solid.heightmap:
            # the geometry is static: its near-solid tile maps once per level
            for l in range(topology.levels):
                nm = torch.zeros(int(np.prod(topology.tile_grid(l))), dtype=torch.uint8,
                                 device=topology.device)
                L.check(L.lib().mlbm_solid_near(L.C.byref(topology.level_struct(l)),
                                                L.C.byref(self._solid), L.ptr(nm),
                                                L.stream_handle()), "solid_near")
                self._near_maps.append(nm)
                self._solid.near[l] = nm.data_ptr()
        self._schedule = build_schedule(topology.levels)
        self.launches = 0
        self._refresh_tables()

    # -- tables -----------------------------------------------------------------
    def _refresh_tables(self, only=None):
        topo = self.topology
        if self._tables_version == topo.version:
            return
        if only is not None and (self._tables is None or
                                 any(l not in self._tables for l in range(topo.levels))):
            only = None
        self._tables = build_tables(topo, self._bc, self._solid, self._err, self._tables, only)
        self._tables_version = topo.version
        if getattr(self, "_structs_cap", None) != topo.cap_version:
            self._structs = {l: topo.level_struct(l, t) for l, t in self._tables.items()}
            self._structs_cap = topo.cap_version

    def _raise_topology(self, msg):
        raise TopologyError(msg)

    def tables(self, level):
        self._refresh_tables()
        return self._tables[level]

    @property
    def interfaces(self):
        self._refresh_tables()
        return self._tables

    def arrays(self, tree_idx, level) -> LevelFields:
        return self.pair.trees[tree_idx].levels[level]

    def roles(self, level):
        return buffer_roles(level, (self.k[level] + self.flip[level]) & 1)

    def last_roles(self, level):
        return buffer_roles(level, (self.k[level] - 1 + self.flip[level]) & 1)

    # -- kernels ----------------------------------------------------------------
    def _collide_struct(self, level, force_mode=0, tau_mode=0, tau=None, tau_ptr=None):
        cp = L.Collide()
        cp.tau = float(self.level_params.taus[level] if tau is None else tau)
        g = tuple(self.params.gravity) + (0.0,) * 3
        for a in range(3):
            cp.gravity[a] = float(g[a])
        cp.h3_xyz = float(self.params.h3_xyz)
        cp.force_mode = force_mode
        cp.tau_mode = tau_mode
        cp.tau0 = float(self.level_params.taus[0])
        cp.tau_ptr = tau_ptr.data_ptr() if tau_ptr is not None else 0
        return cp

    def _level_call(self, level, src, dst, mode, cp=None):
        if self.topology.lv[level].cap == 0:
            return
        self._refresh_tables()
        lvs = self._structs[level]
        cp = cp or self._collide_struct(level)
        L.check(L.lib().mlbm_level_step(L.C.byref(lvs), L.fields(_data(src)), L.fields(_data(dst)),
                                        self.dcode, mode, L.C.byref(cp), L.C.byref(self._bc),
                                        L.ptr(self._err), L.stream_handle()), "level_step")
        self.launches += 1

    def stream_kernel(self, level, src_a, dst):
        self._level_call(level, src_a, dst, 1)

    def collide_kernel(self, level, src_a, dst, force=None, tau_eff=None):
        cp = self._resolve_force_tau(level, dst, force, tau_eff)
        self._level_call(level, src_a, dst, 3, cp)

    def boundary_kernel(self, level, dst):
        self._level_call(level, dst, dst, 4)

    def _resolve_force_tau(self, level, dst, force, tau_eff):
        force_mode, tau_mode, tau, tau_ptr = 0, 0, None, None
        if force is FIELD_FORCE:
            force_mode = 1
        elif force is not None:
            dd = _data(dst)
            base = field_names(self.d).index("fx")
            for a in range(self.d):
                fa = torch.as_tensor(force[a], dtype=self.dtype, device=dd.device).reshape(-1)
                dd[base + a, :fa.numel()].copy_(fa)
            force_mode = 1
        if tau_eff is FIELD_TAU:
            tau_mode = 1
        elif tau_eff is not None:
            if np.ndim(tau_eff) == 0 and not torch.is_tensor(tau_eff):
                tau = float(tau_eff)
            else:
                self._tau_buf = torch.as_tensor(tau_eff, dtype=self.dtype,
                                                device=_data(dst).device).contiguous()
                tau_mode, tau_ptr = 2, self._tau_buf
        return self._collide_struct(level, force_mode, tau_mode, tau, tau_ptr)

    def stream(self, level):
        r, w = self.roles(level)
        self.stream_kernel(level, self.arrays(r, level), self.arrays(w, level))

    def collide(self, level, force=None, tau_eff=None):
        r, w = self.roles(level)
        self.collide_kernel(level, self.arrays(r, level), self.arrays(w, level), force, tau_eff)

    def apply_boundaries(self, level):
        _, w = self.roles(level)
        self.boundary_kernel(level, self.arrays(w, level))

    def collide_and_boundaries(self, level, force=None, tau_eff=None):
        """collide + apply_boundaries in one pass (mode 2)."""
        r, w = self.roles(level)
        cp = self._resolve_force_tau(level, self.arrays(w, level), force, tau_eff)
        self._level_call(level, self.arrays(r, level), self.arrays(w, level), 2, cp)

    def stream_collide(self, level, force=None, tau_eff=None):
        """One full step at a level, fused into a single kernel (mode 0)."""
        r, w = self.roles(level)
        if force is None and tau_eff is None:
            self._level_call(level, self.arrays(r, level), self.arrays(w, level), 0)
        else:
            self.stream(level)
            self.collide_and_boundaries(level, force, tau_eff)
        self.k[level] += 1

    # -- cross-level transfers -----------------------------------------------------
    def downward_transfer(self, level, step):
        coarse = level + 1
        old_t, new_t = self.last_roles(coarse)
        r, _ = self.roles(level)
        self.downward_kernel(level, step, self.arrays(old_t, coarse),
                             self.arrays(new_t, coarse), self.arrays(r, level))

    def downward_kernel(self, level, step, olda, newa, dst):
        self._refresh_tables()
        t = self._tables.get(level)
        if t is None or not self.topology.lv[level].cap or level + 1 >= self.topology.levels:
            return
        tg, src, n = t.down
        kap = _kappa_down(self.level_params.taus[level], self.level_params.taus[level + 1],
                          self.params.rescale_convention)
        L.check(L.lib().mlbm_downward(self.d, n, L.ptr(self.topology.dcounts[level, 2:3]),
                                      L.ptr(tg), L.ptr(src),
                                      L.ptr(self.topology.lv[level].tile_xyz),
                                      L.fields(_data(olda)), L.fields(_data(newa)),
                                      L.fields(_data(dst)), self.dcode, int(step), kap,
                                      L.stream_handle()), "downward")
        self.launches += 1

    def upward_transfer(self, level):
        coarse = level + 1
        _, fine_w = self.last_roles(level)
        _, coarse_w = self.last_roles(coarse)
        self.upward_kernel(level, self.arrays(fine_w, level), self.arrays(coarse_w, coarse))

    def upward_kernel(self, level, fine, dst):
        self._refresh_tables()
        t = self._tables.get(level + 1)
        if t is None or not self.topology.lv[level + 1].cap or not self.topology.lv[level].cap:
            return
        tg, src, n = t.up
        kap = _kappa_up(self.level_params.taus[level], self.level_params.taus[level + 1],
                        self.params.rescale_convention)
        avg = 1 if self.params.upward_mode == "average" else 0
        L.check(L.lib().mlbm_upward(self.d, n, L.ptr(self.topology.dcounts[level + 1, 3:4]),
                                    L.ptr(tg), L.ptr(src), L.fields(_data(fine)),
                                    L.fields(_data(dst)), self.dcode, avg, kap,
                                    L.stream_handle()), "upward")
        self.launches += 1

    # -- schedule -------------------------------------------------------------------
    def run_cycle(self, cycle, hook=None):
        """One finest cycle (solver.py:564-595)."""
        self._refresh_tables()
        for kind, level, s in cycle["pre"]:
            if kind == "down":
                self.downward_transfer(level, s)
            elif kind == "sc":
                self.stream_collide(level)
            elif kind == "up":
                self.upward_transfer(level)
        s0 = cycle["s0"]
        if self.topology.levels > 1:
            self.downward_transfer(0, s0)
        if hook is None:
            r, w = self.roles(0)
            self._level_call(0, self.arrays(r, 0), self.arrays(w, 0), 0)
        elif hasattr(hook, "level0"):
            # fused coupled step: P2G needs no stream output, the exchange of a
            # cell only its own bare moments: pre -> one level-0 kernel -> post
            hook.pre(self)
            hook.level0(self)
            hook.post(self)
        else:
            self.stream(0)
            out = hook(self)
            force, tau_eff = (None, None) if out is None else out
            self.collide_and_boundaries(0, force, tau_eff)
        self.k[0] += 1
        if self.topology.levels > 1 and s0 == 2:
            self.upward_transfer(0)
        if cycle["last"]:
            self.pair.bounce += 1
        if self.check_errors:
            self.raise_pending()

    def raise_pending(self):
        """Raise DivergenceError / TopologyError recorded on the device."""
        err = self._err.cpu().numpy()
        if err[0] == 0:
            return
        self._err.zero_()
        code, level, count = int(err[0]), int(err[1]), int(err[2])
        cells = [tuple(int(v) for v in err[3 + 3 * i: 3 + 3 * i + self.d])
                 for i in range(min(count, 5))]
        if code == 1:
            raise DivergenceError(f"level {level}: non-physical density after streaming",
                                  level=level, cells=cells)
        if code == 2:
            raise DivergenceError(f"level {level}: non-finite velocity after collision",
                                  level=level, cells=cells)
        raise TopologyError(f"device error code {code} at level {level} cells {cells}")

    def advance_bounce(self, hook=None):
        for cycle in self._schedule:
            self.run_cycle(cycle, hook=hook)

    def run_finest_steps(self, n: int, hook=None):
        per = len(self._schedule)
        i = self.k[0] % per
        for _ in range(n):
            self.run_cycle(self._schedule[i], hook=hook)
            i = (i + 1) % per

    def cycles_per_bounce(self) -> int:
        return len(self._schedule)


class _Sentinel:
    def __init__(self, name):
        self.name = name

    def __repr__(self):
        return self.name


FIELD_FORCE = _Sentinel("FIELD_FORCE")   # hook result: use the f fields of the write tree
FIELD_TAU = _Sentinel("FIELD_TAU")       # hook result: tau = tau0 * eps of the write tree


def _data(a):
    return a.data if isinstance(a, LevelFields) else a


def build_schedule(levels: int):
    """Linearised Alg. 1 recursion (solver.py:615-649)."""
    ops = []

    def rec(level, s):
        if level < levels - 1:
            ops.append(("down", level, s))
        ops.append(("sc", level, s))
        if level < levels - 1 and s == 2:
            ops.append(("up", level, s))
        if level > 0:
            rec(level - 1, 1)
            rec(level - 1, 2)

    rec(levels - 1, 1)
    cycles, pre = [], []
    for kind, level, s in ops:
        if level == 0 and kind in ("down", "up"):
            continue
        if level == 0 and kind == "sc":
            cycles.append({"pre": pre, "s0": s, "last": False})
            pre = []
        else:
            pre.append((kind, level, s))
    cycles[-1]["last"] = True
    return cycles
