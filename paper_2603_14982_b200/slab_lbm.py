"""Slab-decomposed single-level HOME-LBM over several ranks.

The finest-level domain is cut along x into slabs on tile-column bounds
(`parallel_slabs.SlabPartition`).  Each rank keeps a local tile box = its own
columns plus one ghost tile column on every side that has a neighbour rank
(or wraps periodically).  Tiles are stored in sorted (x, y, z) slot order, so
the left ghost column, the owned columns and the right ghost column are three
contiguous slot ranges: the level step runs over the owned range only
(`mlbm_level_t.first`), reads its x-neighbours' moments from the ghost
columns exactly like from any other neighbour tile, and after every step the
owned edge columns of the write tree are sent to the neighbours' ghost
columns (one send + one receive per side, NCCL point-to-point over NVLink on
the device path, ``torch.distributed`` batch P2P).  A slab run is therefore
bit-identical to the single-domain run (tests/test_gpu_slab.py).

Scope: single-level scenes (configs[0], C1).  The multi-level coupled path
additionally needs the interface stencils, the particle migration and the
seed OR-reduction across slabs (host logic in ``parallel_slabs.py``).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .parallel_slabs import SlabPartition
from .solver import BoundarySpec, LevelParams, MultiLevelSolver, SolverParams, H3_XYZ_HERMITE
from .sparse_grid import PingPongPair, Topology, TILE, moment_names


class SlabLBM:
    """One rank's slab of a single-level periodic-in-(y, z) LBM domain."""

    def __init__(self, global_cells, rank, world, tau0, dtype=torch.float32,
                 periodic=(True, True, True), init=None, device=None):
        self.global_cells = tuple(int(v) for v in global_cells)
        self.d = len(self.global_cells)
        self.rank, self.world = rank, world
        self.part = SlabPartition(self.global_cells, 1, world, periodic_x=bool(periodic[0]))
        x0, x1 = self.part.slab(rank)
        left, right = self.part.neighbors(rank)
        self.left = left if world > 1 else None
        self.right = right if world > 1 else None
        self.gl = 1 if self.left is not None else 0          # ghost columns
        self.gr = 1 if self.right is not None else 0
        self.x0 = x0 - TILE * self.gl                        # local box origin (finest cells)
        local = (x1 - x0 + TILE * (self.gl + self.gr),) + self.global_cells[1:]
        per_local = ((bool(periodic[0]) and world == 1),) + tuple(bool(p) for p in periodic[1:self.d])
        self.topology = Topology.uniform(local, 1, periodic=per_local, device=device)
        self.pair = PingPongPair(self.topology, dtype)
        self.params = SolverParams(levels=1, h3_xyz=H3_XYZ_HERMITE)
        self.level_params = LevelParams(1, tau0)
        faces = {}
        for a, ax in enumerate("xyz"[:self.d]):
            kind = "periodic" if per_local[a] else "wall"   # ghost sides: never stepped
            faces[ax + "_min"] = faces[ax + "_max"] = kind
        self.solver = MultiLevelSolver(self.topology, self.pair, self.params, self.level_params,
                                       BoundarySpec(faces=faces, dim=self.d))
        t = self.topology.tiles_dims(0)
        self.col = int(np.prod(t[1:]))                       # tiles per x column
        self.n_owned = (t[0] - self.gl - self.gr) * self.col
        self.first = self.gl * self.col
        self.nm = len(moment_names(self.d))
        if init is not None:
            self.set_fields(init)
        # owned-range level struct (counts = NULL: n_tiles is the exact end)
        self._lv = None
        cols = self.col * TILE ** self.d
        self._send = [torch.empty((self.nm, cols), dtype=dtype, device=self.topology.device)
                      for _ in range(2)]
        self._recv = [torch.empty_like(b) for b in self._send]

    # -- fields -------------------------------------------------------------------
    def set_fields(self, fn):
        """fn(pos (n, d) in GLOBAL finest units, level) -> {name: values}."""
        pos = self.topology.cell_coords(0).astype(float)
        pos[:, 0] = np.mod(pos[:, 0] + self.x0, self.global_cells[0])   # ghosts wrap
        vals = fn(pos, 0)
        for tree in self.pair.trees:
            for nm, v in vals.items():
                tree.levels[0][nm] = v

    def owned_cells(self, tree_idx, name):
        """Host copy of one field over the owned cells, with their global coords."""
        a = self.pair.trees[tree_idx].levels[0]
        T = TILE ** self.d
        lo, hi = self.first * T, (self.first + self.n_owned) * T
        coords = self.topology.cell_coords(0)[lo:hi].copy()
        coords[:, 0] += self.x0
        return coords, a[name].cpu().numpy()[lo:hi]

    # -- step -----------------------------------------------------------------------
    def _level_struct(self):
        if self._lv is None:
            self.solver._refresh_tables()
            st = self.topology.level_struct(0, self.solver._tables[0])
            lv = L.Level.from_buffer_copy(st)
            lv.counts = None
            lv.first = self.first
            lv.n_tiles = self.first + self.n_owned
            self._lv = lv
        return self._lv

    def step_local(self):
        """Fused stream + collide over the owned tiles (solver.py:483-488)."""
        s = self.solver
        r, w = s.roles(0)
        cp = s._collide_struct(0)
        L.check(L.lib().mlbm_level_step(L.C.byref(self._level_struct()),
                                        L.fields(s.arrays(r, 0).data),
                                        L.fields(s.arrays(w, 0).data), s.dcode, 0,
                                        L.C.byref(cp), L.C.byref(s._bc), L.ptr(s._err),
                                        L.stream_handle()), "level_step")
        s.k[0] += 1
        return w

    def edge_columns(self, tree_idx):
        """(first owned column, last owned column) views [nm, col cells]."""
        a = self.pair.trees[tree_idx].levels[0].data
        T = TILE ** self.d
        c = self.col * T
        lo = self.first * T
        hi = (self.first + self.n_owned) * T
        return a[:self.nm, lo:lo + c], a[:self.nm, hi - c:hi]

    def ghost_columns(self, tree_idx):
        """(left ghost, right ghost) views or None."""
        a = self.pair.trees[tree_idx].levels[0].data
        T = TILE ** self.d
        c = self.col * T
        left = a[:self.nm, 0:c] if self.gl else None
        hi = (self.first + self.n_owned) * T
        right = a[:self.nm, hi:hi + c] if self.gr else None
        return left, right

    def exchange(self, tree_idx):
        """Owned edge columns -> neighbours' ghost columns (P2P, both sides)."""
        if self.world == 1:
            return
        lo_col, hi_col = self.edge_columns(tree_idx)
        gl, gr = self.ghost_columns(tree_idx)
        exchange_columns(lo_col, hi_col, gl, gr, self.left, self.right, self._send, self._recv)

    def step(self):
        w = self.step_local()
        self.exchange(w)


def exchange_columns(lo_col, hi_col, ghost_l, ghost_r, left, right, send, recv):
    """Batch P2P of one slab's edge columns (backend-agnostic: NCCL on CUDA
    tensors, gloo on CPU tensors).  Posting order (send right, send left,
    recv left, recv right) matches the messages pairwise even when
    left == right (two ranks, periodic x)."""
    send[0].copy_(lo_col)
    send[1].copy_(hi_col)
    ops = []
    if right is not None:
        ops.append(dist.P2POp(dist.isend, send[1], right))
    if left is not None:
        ops.append(dist.P2POp(dist.isend, send[0], left))
    if left is not None:
        ops.append(dist.P2POp(dist.irecv, recv[0], left))
    if right is not None:
        ops.append(dist.P2POp(dist.irecv, recv[1], right))
    if ops:
        for q in dist.batch_isend_irecv(ops):
            q.wait()
    if ghost_l is not None:
        ghost_l.copy_(recv[0])
    if ghost_r is not None:
        ghost_r.copy_(recv[1])


def exchange_local(slabs, tree_idx):
    """Single-process stand-in for the P2P exchange between slab objects that
    live in one process (tests): device copies, same column mapping."""
    world = len(slabs)
    for r, sl in enumerate(slabs):
        lo_col, hi_col = sl.edge_columns(tree_idx)
        if sl.right is not None:
            dst = slabs[sl.right].ghost_columns(tree_idx)[0]
            dst.copy_(hi_col)
        if sl.left is not None:
            dst = slabs[sl.left].ghost_columns(tree_idx)[1]
            dst.copy_(lo_col)
    assert world == len(slabs)
