"""Kernel-level binding for the reference's own solver class.

A maintainer who keeps the reference's host code (``mlbm.solver.MultiLevelSolver``
with NumPy field dicts) and swaps only its data-parallel kernels subclasses it and
forwards the five kernel seams to :class:`B200Kernels`:

    class MultiLevelSolverB200(mlbm.solver.MultiLevelSolver):
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            self.b200 = B200Kernels(self, divergence_error=mlbm.lattice.DivergenceError)
        def stream_kernel(self, level, src_a, dst):    self.b200.stream_kernel(level, src_a, dst)
        def collide_kernel(self, level, src_a, dst, force=None, tau_eff=None):
            self.b200.collide_kernel(level, src_a, dst, force, tau_eff)
        def boundary_kernel(self, level, dst):         self.b200.boundary_kernel(level, dst)
        def downward_kernel(self, level, step, olda, newa, dst):
            self.b200.downward_kernel(level, step, olda, newa, dst)
        def upward_kernel(self, level, fine, dst):     self.b200.upward_kernel(level, fine, dst)

Every seam keeps the reference's signature and semantics (solver.py:336-560): the
arguments are the caller's NumPy dicts (``rho, ux, uy, sxx, sxy, syy, eps, fx, fy,
phi`` in the caller's cell order), outputs are written into them in place, and a
non-physical state raises ``divergence_error(msg, level=, cells=)`` like
solver.py:398-406,447-453.  The kernels themselves are the sm_100a launches of
``mlbm_level_step`` (modes 1 / 3 / 4), ``mlbm_downward`` and ``mlbm_upward``
through the C ABI; the dicts are staged through device buffers around each call
(this seam is the reference's per-kernel granularity — the fused, device-resident
path is ``MultiLevelSolver`` of this package).

The device topology mirrors ``ref.topology.tile_set()`` and is re-synchronised when
``ref.topology.version`` changes (adapt).  Works with any object exposing the
reference's solver attributes (``topology``, ``boundaries``, ``params``,
``level_params``), e.g. the NumPy oracle's ``Solver`` in the GPU tests.
"""
from __future__ import annotations

import numpy as np
import torch

from .lattice import DivergenceError
from .solver import BoundarySpec, LevelParams, LogInlet, MultiLevelSolver, SolverParams
from .sparse_grid import LevelFields, PingPongPair, Topology, field_names, fresh_block


def _finest(topo):
    for name in ("finest_cells", "finest"):
        if hasattr(topo, name):
            return tuple(int(c) for c in getattr(topo, name))
    raise AttributeError("topology exposes neither finest_cells nor finest")


def _device_boundaries(spec, d):
    faces = {}
    for face, cond in spec.faces.items():
        if hasattr(cond, "u0") and hasattr(cond, "beta"):
            faces[face] = LogInlet(float(cond.u0), float(cond.beta), float(cond.y0))
        else:
            faces[face] = cond
    return BoundarySpec(faces=faces, solid_boxes=[tuple(b) for b in spec.solid_boxes],
                        heightmap=getattr(spec, "heightmap", None), dim=d)


class B200Kernels:
    """The five kernel seams of ``ref`` (a reference-API solver) on the B200."""

    def __init__(self, ref, divergence_error=DivergenceError):
        self.ref = ref
        self.divergence_error = divergence_error
        rt = ref.topology
        self.finest = _finest(rt)
        self.d = len(self.finest)
        self.levels = int(rt.levels)
        p = ref.params
        sp = dict(levels=self.levels, rho0=float(p.rho0), gravity=tuple(p.gravity),
                  eps_min=float(p.eps_min), mpm_cadence=int(p.mpm_cadence),
                  rescale_convention=p.rescale_convention, upward_mode=p.upward_mode)
        if hasattr(p, "h3_xyz"):
            sp["h3_xyz"] = float(p.h3_xyz)
        self.topo = Topology(self.finest, self.levels, tuple(rt.periodic))
        self.topo.set_tile_set(rt.tile_set())
        # fp64 like the reference: untouched cells round-trip exactly
        self.pair = PingPongPair(self.topo, torch.float64)
        self.sv = MultiLevelSolver(self.topo, self.pair, SolverParams(**sp),
                                   LevelParams(self.levels, float(ref.level_params.tau0)),
                                   _device_boundaries(ref.boundaries, self.d))
        self.names = field_names(self.d)
        # what stream / collide / boundary write (the f rows are inputs only)
        self.written = tuple(nm for nm in self.names if not (nm[0] == 'f' and len(nm) == 2))
        self._version = getattr(rt, "version", None)
        self._perm = {}
        self._bufs = {}

    # -- topology / staging ------------------------------------------------------
    def _sync(self):
        v = getattr(self.ref.topology, "version", None)
        if v is not None and v != self._version:
            self.topo.set_tile_set(self.ref.topology.tile_set())
            self.pair.ensure_capacity()
            self.sv._refresh_tables()
            self._version = v
            self._perm.clear()
            self._bufs.clear()

    def _perm_of(self, level):
        """Device cell index of each reference cell (None: identical order)."""
        if level not in self._perm:
            rc = np.asarray(self.ref.topology.cell_coords(level))
            dc = self.topo.cell_coords(level)
            if len(rc) != len(dc):
                raise RuntimeError(f"level {level}: device and reference cell counts differ")
            if np.array_equal(rc, dc):
                self._perm[level] = None
            else:
                dmap = {tuple(c): i for i, c in enumerate(dc)}
                self._perm[level] = torch.as_tensor(
                    np.array([dmap[tuple(c)] for c in rc], dtype=np.int64), device=self.topo.device)
        return self._perm[level]

    def _buf(self, level, slot):
        key = (level, slot)
        if key not in self._bufs:
            blk = fresh_block(self.d, self.topo.capacity_cells(level), self.pair.dtype,
                              self.topo.device)
            self._bufs[key] = LevelFields(self.d, blk,
                                          live=(lambda l=level: self.topo.cell_count(l)))
        return self._bufs[key]

    def _to_dev(self, level, host):
        v = torch.as_tensor(np.asarray(host, dtype=np.float64), device=self.topo.device)
        perm = self._perm_of(level)
        if perm is None:
            return v
        out = torch.empty_like(v)
        out[perm] = v
        return out

    def _up(self, level, arrays, slot):
        lf = self._buf(level, slot)
        n = self.topo.cell_count(level)
        for i, nm in enumerate(self.names):
            if nm in arrays:
                v = self._to_dev(level, arrays[nm])
                lf.data[i, :n].copy_(v - 1.0 if i == 0 else v)
        return lf

    def _down(self, level, lf, arrays, names=None):
        n = self.topo.cell_count(level)
        perm = self._perm_of(level)
        for i, nm in enumerate(self.names):
            if nm not in arrays or (names is not None and nm not in names):
                continue
            v = lf.data[i, :n]
            if perm is not None:
                v = v[perm]
            v = v.double().cpu().numpy()
            arrays[nm][:] = v + 1.0 if i == 0 else v

    def _raise(self):
        try:
            self.sv.raise_pending()
        except DivergenceError as e:
            if self.divergence_error is DivergenceError:
                raise
            raise self.divergence_error(str(e), level=e.level, cells=e.cells) from None

    # -- the reference's kernel seams (solver.py:336-560) ---------------------------
    def stream_kernel(self, level, src_a, dst):
        """solver.py:336-381 → mlbm_level_step(mode=1)."""
        if not len(dst["rho"]):
            return
        self._sync()
        s, w = self._up(level, src_a, 0), self._buf(level, 1)
        self.sv.stream_kernel(level, s, w)
        self._down(level, w, dst, names=self.written)

    def collide_kernel(self, level, src_a, dst, force=None, tau_eff=None):
        """solver.py:394-453 → mlbm_level_step(mode=3); force = (f_x, f_y[, f_z])
        per-cell arrays or None (gravity), tau_eff a scalar, a per-cell array or None."""
        if not len(dst["rho"]):
            return
        self._sync()
        s, w = self._up(level, src_a, 0), self._up(level, dst, 1)
        f = None if force is None else tuple(self._to_dev(level, fa) for fa in force)
        t = tau_eff
        if tau_eff is not None and np.ndim(tau_eff) > 0:
            t = self._to_dev(level, tau_eff)
        self.sv.collide_kernel(level, s, w, f, t)
        self._raise()
        self._down(level, w, dst, names=self.written)

    def boundary_kernel(self, level, dst):
        """solver.py:460-481 → mlbm_level_step(mode=4)."""
        if not len(dst["rho"]):
            return
        self._sync()
        w = self._up(level, dst, 1)
        self.sv.boundary_kernel(level, w)
        self._down(level, w, dst)

    def downward_kernel(self, level, step, olda, newa, dst):
        """solver.py:501-526 → mlbm_downward (writes the I^d targets of dst)."""
        self._sync()
        c = level + 1
        if c >= self.levels or not self.topo.cell_count(level):
            return
        o, nw = self._up(c, olda, 0), self._up(c, newa, 1)
        w = self._up(level, dst, 2)
        self.sv.downward_kernel(level, step, o, nw, w)
        self._down(level, w, dst)

    def upward_kernel(self, level, fine, dst):
        """solver.py:536-560 → mlbm_upward (writes the I^u targets of dst)."""
        self._sync()
        c = level + 1
        if c >= self.levels or not self.topo.cell_count(level):
            return
        f = self._up(level, fine, 0)
        w = self._up(c, dst, 2)
        self.sv.upward_kernel(level, f, w)
        self._down(c, w, dst)
