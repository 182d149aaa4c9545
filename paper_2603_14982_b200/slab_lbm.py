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
    L.pack_cols(lo_col, send[0])
    L.pack_cols(hi_col, send[1])
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
        L.unpack_cols(recv[0], ghost_l)
    if ghost_r is not None:
        L.unpack_cols(recv[1], ghost_r)


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


# ---------------------------------------------------------------------------------
# Multi-level slabs (static hierarchy): SURVEY.md §8(e) collective (i) for every
# level of the Alg. 1 recursion.

class SlabMultiLevel:
    """One rank's slab of a static multi-level LBM hierarchy.

    The global tile set is cropped to the slab plus a ghost region one
    coarsest tile wide on every side with a neighbour (2^(L-1-l) tile columns
    at level l), shifted to a local box whose x faces are walls (ghost tiles
    are never stepped).  Level steps run over the owned slot range of each
    level; after every level step the owned edge columns of the level's write
    tree are sent to the neighbours' ghost columns, so interface fills that
    read coarse cells across the cut and the next pulls see the owners'
    values.  Downward / upward transfers run on every target of the local box
    (those in the ghost region recompute the owners' values from the same
    inputs or are overwritten before use)."""

    def __init__(self, global_cells, levels, global_tiles, rank, world, tau0,
                 dtype=torch.float64, periodic=(True, True, True), init=None, device=None,
                 params=None, level_params=None, faces=None, solver_cls=None):
        self.global_cells = tuple(int(v) for v in global_cells)
        self.d = len(self.global_cells)
        self.levels = levels
        self.rank, self.world = rank, world
        self.part = SlabPartition(self.global_cells, levels, world, periodic_x=bool(periodic[0]))
        x0, x1 = self.part.slab(rank)
        left, right = self.part.neighbors(rank)
        self.left = left if world > 1 else None
        self.right = right if world > 1 else None
        cw = self.part.coarse_width                       # finest cells of one coarsest tile
        self.gl = cw if self.left is not None else 0
        self.gr = cw if self.right is not None else 0
        self.x0 = x0 - self.gl
        local = (x1 - x0 + self.gl + self.gr,) + self.global_cells[1:]
        per_local = ((bool(periodic[0]) and world == 1),) + tuple(bool(p) for p in periodic[1:self.d])
        self.topology = Topology(local, levels, periodic=per_local, device=device)
        gx = self.global_cells[0]
        tiles = set()
        for e in global_tiles:
            l, c = e[0], list(e[1:-1])
            tw = TILE << l
            for wrap in ((0, -gx, gx) if periodic[0] else (0,)):
                lx = c[0] * tw + wrap - self.x0             # local finest x of the tile origin
                if 0 <= lx < local[0]:
                    tiles.add((l, lx // tw) + tuple(c[1:]) + (e[-1],))
        self.topology.set_tile_set(sorted(tiles))
        self.pair = PingPongPair(self.topology, dtype)
        self.params = params or SolverParams(levels=levels, h3_xyz=H3_XYZ_HERMITE)
        self.level_params = level_params or LevelParams(levels, tau0)
        lf = {}
        for a, ax in enumerate("xyz"[:self.d]):
            kind = "periodic" if per_local[a] else "wall"
            lf[ax + "_min"] = lf[ax + "_max"] = kind
        if faces is not None:
            # the scene's faces; x sides facing a neighbour rank become walls of
            # the local box (their ghost cells are never stepped)
            lf = dict(faces)
            if world > 1:
                if self.left is not None or lf.get("x_min") == "periodic":
                    lf["x_min"] = "wall"
                if self.right is not None or lf.get("x_max") == "periodic":
                    lf["x_max"] = "wall"
        self.faces = lf
        cls = solver_cls or MultiLevelSolver
        self.solver = cls(self.topology, self.pair, self.params, self.level_params,
                          BoundarySpec(faces=lf, dim=self.d))
        self.solver.check_errors = False
        self.local_cells = local
        self.compute_ranges()
        if init is not None:
            self.set_fields(init)
        self._lv = {}

    def compute_ranges(self):
        """Per level: owned slot range and the slot ranges of the edge / ghost
        columns (slots are x-major, so each is contiguous); re-run after a
        topology change."""
        local = self.local_cells
        self.ranges = []
        for l in range(self.levels):
            xs = self.topology.tile_coords(l)[:, 0] if self.topology.n_tiles(l) else np.zeros(0, int)
            wl = (self.gl // (TILE << l), self.gr // (TILE << l))
            ncol = local[0] // (TILE << l)
            cnt = lambda lo, hi: int(((xs >= lo) & (xs < hi)).sum())      # noqa: E731
            a = cnt(0, wl[0])
            b = a + cnt(wl[0], ncol - wl[1])
            self.ranges.append({
                "ghost_l": (0, a), "owned": (a, b), "ghost_r": (b, len(xs)),
                "edge_l": (a, a + cnt(wl[0], 2 * wl[0])) if wl[0] else (a, a),
                "edge_r": (b - cnt(ncol - 2 * wl[1], ncol - wl[1]), b) if wl[1] else (b, b)})
        self._lv = {}

    def set_fields(self, fn):
        for l in range(self.levels):
            if not self.topology.n_tiles(l):
                continue
            pos = self.topology.cell_coords(l).astype(float) * float(1 << l)
            pos[:, 0] = np.mod(pos[:, 0] + self.x0, self.global_cells[0])
            vals = fn(pos, l)
            for tree in self.pair.trees:
                for nm, v in vals.items():
                    tree.levels[l][nm] = v

    def _owned_struct(self, level):
        if level not in self._lv:
            s = self.solver
            s._refresh_tables()
            lv = L.Level.from_buffer_copy(s._structs[level])
            lv.counts = None
            a, b = self.ranges[level]["owned"]
            lv.first = a
            lv.n_tiles = b
            self._lv[level] = lv
        return self._lv[level]

    def step_level(self, level):
        """Fused stream + collide of the owned tiles of one level; returns
        the write tree index."""
        s = self.solver
        r, w = s.roles(level)
        a, b = self.ranges[level]["owned"]
        if b > a:
            cp = s._collide_struct(level)
            L.check(L.lib().mlbm_level_step(L.C.byref(self._owned_struct(level)),
                                            L.fields(s.arrays(r, level).data),
                                            L.fields(s.arrays(w, level).data), s.dcode, 0,
                                            L.C.byref(cp), L.C.byref(s._bc), L.ptr(s._err),
                                            L.stream_handle()), "level_step")
        s.k[level] += 1
        return w

    def cells(self, level, rng):
        T = TILE ** self.d
        return rng[0] * T, rng[1] * T

    def owned_cells(self, tree_idx, level, name):
        a = self.pair.trees[tree_idx].levels[level]
        lo, hi = self.cells(level, self.ranges[level]["owned"])
        coords = self.topology.cell_coords(level)[lo:hi].copy()
        coords[:, 0] = np.mod(coords[:, 0] + (self.x0 >> level), self.global_cells[0] >> level)
        return coords, a[name].cpu().numpy()[lo:hi]


def run_cycle_slabs(slabs, cycle, exchange):
    """One finest cycle of the Alg. 1 schedule (solver.py:564-595) on slab
    objects in lockstep; ``exchange(slabs, level, tree)`` after every level
    step (device copies in one process, or P2P between processes)."""
    s0 = slabs[0]
    L_ = s0.levels
    for kind, level, s in cycle["pre"]:
        if kind == "down":
            for sl in slabs:
                sl.solver.downward_transfer(level, s)
        elif kind == "sc":
            w = None
            for sl in slabs:
                w = sl.step_level(level)
            exchange(slabs, level, w)
        elif kind == "up":
            for sl in slabs:
                sl.solver.upward_transfer(level)
    if L_ > 1:
        for sl in slabs:
            sl.solver.downward_transfer(0, cycle["s0"])
    w = None
    for sl in slabs:
        w = sl.step_level(0)
    exchange(slabs, 0, w)
    if L_ > 1 and cycle["s0"] == 2:
        for sl in slabs:
            sl.solver.upward_transfer(0)
    if cycle["last"]:
        for sl in slabs:
            sl.pair.bounce += 1


def exchange_levels_local(slabs, level, tree_idx):
    """Single-process stand-in for the per-level P2P: owned edge columns of
    ``level`` (write tree) -> the neighbours' ghost columns."""
    nm = len(moment_names(slabs[0].d))
    for sl in slabs:
        a = sl.pair.trees[tree_idx].levels[level].data
        for side, nb_idx in (("edge_r", sl.right), ("edge_l", sl.left)):
            if nb_idx is None:
                continue
            nb = slabs[nb_idx]
            g = "ghost_l" if side == "edge_r" else "ghost_r"
            lo, hi = sl.cells(level, sl.ranges[level][side])
            glo, ghi = nb.cells(level, nb.ranges[level][g])
            assert hi - lo == ghi - glo, (level, side, hi - lo, ghi - glo)
            nb.pair.trees[tree_idx].levels[level].data[:nm, glo:ghi].copy_(a[:nm, lo:hi])


def exchange_levels_p2p(slabs, level, tree_idx):
    """The per-level exchange between processes (one slab per rank): batch
    P2P of the owned edge columns into the neighbours' ghost columns
    (NCCL over NVLink for CUDA tensors)."""
    (sl,) = slabs
    if sl.world == 1:
        return
    nm = len(moment_names(sl.d))
    a = sl.pair.trees[tree_idx].levels[level].data
    r = sl.ranges[level]
    lo_l, hi_l = sl.cells(level, r["edge_l"])
    lo_r, hi_r = sl.cells(level, r["edge_r"])
    glo_l, ghi_l = sl.cells(level, r["ghost_l"])
    glo_r, ghi_r = sl.cells(level, r["ghost_r"])
    edge_l = a[:nm, lo_l:hi_l]
    edge_r = a[:nm, lo_r:hi_r]
    ghost_l = a[:nm, glo_l:ghi_l] if sl.left is not None else None
    ghost_r = a[:nm, glo_r:ghi_r] if sl.right is not None else None
    key = (level, edge_l.shape[1], edge_r.shape[1],
           0 if ghost_l is None else ghost_l.shape[1], 0 if ghost_r is None else ghost_r.shape[1])
    bufs = getattr(sl, "_p2p_bufs", {})
    if key not in bufs:
        mk = lambda n: torch.empty((nm, n), dtype=a.dtype, device=a.device)     # noqa: E731
        bufs[key] = ([mk(edge_l.shape[1]), mk(edge_r.shape[1])],
                     [mk(key[3]), mk(key[4])])
        sl._p2p_bufs = bufs
    send, recv = bufs[key]
    exchange_columns(edge_l, edge_r, ghost_l, ghost_r, sl.left, sl.right, send, recv)
