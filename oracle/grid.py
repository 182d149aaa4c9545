"""Sparse tile hierarchy, field trees and interface sets (oracle).

Restates ``pkg/src/mlbm/sparse_grid.py`` for d = 2, 3:
  * 4^d tiles, within-tile cell index lx + 4 ly (+ 16 lz)   sparse_grid.py:17-18,219-239
  * canonical (sorted-coords) slot order                      sparse_grid.py:183-200
  * cell maps / coords / leaf rasters / owner grid            sparse_grid.py:210-282
  * coverage + two-tile-ring validation                        sparse_grid.py:304-337
  * Chebyshev dilation (separable shift-or)                    sparse_grid.py:340-363
  * field trees (rho = eps = 1 defaults) and buffer roles      sparse_grid.py:369-405
  * interface sets I^d (2-cell rim) / I^u (1-cell rim)         sparse_grid.py:439-544
Tiles are kept as a sorted (n, d) coordinate array per level plus kinds, so
comparisons against the device path key on coordinates, never slots.
"""
from __future__ import annotations

import itertools

import numpy as np

from .lattice import s_names

TILE = 4
LEAF = 0
BORDER = 1


class TopologyError(RuntimeError):
    pass


class DivergenceError(RuntimeError):
    def __init__(self, message, level=None, cells=None):
        super().__init__(message)
        self.level = level
        self.cells = cells


def field_names(d):
    """2D order equals sparse_grid.py:29; 3D extends it."""
    ax = "xyz"[:d]
    return (["rho"] + ["u" + a for a in ax] + s_names(d) + ["eps"]
            + ["f" + a for a in ax] + ["phi"])


def moment_names(d):
    ax = "xyz"[:d]
    return ["rho"] + ["u" + a for a in ax] + s_names(d)


def cells_per_tile(d):
    return TILE ** d


def local_offsets(d):
    """(T^d, d) local coords in within-tile index order lx + 4ly + 16lz."""
    n = TILE ** d
    idx = np.arange(n)
    return np.stack([(idx // TILE ** a) % TILE for a in range(d)], axis=1)


def shift_or(mask, axis, wrap):
    out = mask.copy()
    n = mask.shape[axis]
    if n > 1:
        sl = [slice(None)] * mask.ndim

        def S(s):
            sl2 = list(sl)
            sl2[axis] = s
            return tuple(sl2)
        out[S(slice(1, None))] |= mask[S(slice(None, -1))]
        out[S(slice(None, -1))] |= mask[S(slice(1, None))]
        if wrap:
            out[S(slice(0, 1))] |= mask[S(slice(n - 1, n))]
            out[S(slice(n - 1, n))] |= mask[S(slice(0, 1))]
    return out


def dilate(mask, steps, periodic):
    """Chebyshev dilation by ``steps`` (sparse_grid.py:358-363)."""
    out = mask.copy()
    for _ in range(steps):
        for a in range(mask.ndim):
            out = shift_or(out, a, periodic[a])
    return out


def group_any(mask):
    """Parent bitmap: any over each 2^d child group (adapt.py:84-87)."""
    d = mask.ndim
    shp = []
    for n in mask.shape:
        shp += [n // 2, 2]
    return mask.reshape(shp).any(axis=tuple(range(1, 2 * d, 2)))


def group_all(mask):
    d = mask.ndim
    shp = []
    for n in mask.shape:
        shp += [n // 2, 2]
    return mask.reshape(shp).all(axis=tuple(range(1, 2 * d, 2)))


def upsample2(mask):
    out = mask
    for a in range(mask.ndim):
        out = np.repeat(out, 2, axis=a)
    return out


class Topology:
    """Per-level sorted tile lists over a fixed box (sparse_grid.py:125-337)."""

    def __init__(self, finest_cells, levels, periodic=None):
        self.d = len(finest_cells)
        self.finest = tuple(int(v) for v in finest_cells)
        if levels < 1:
            raise ValueError("levels must be >= 1")
        step = TILE * (1 << (levels - 1))
        if any(v % step for v in self.finest):
            raise ValueError(f"extents must be divisible by {step}")
        self.levels = levels
        self.periodic = tuple(bool(p) for p in
                              (periodic if periodic is not None
                               else (True,) * self.d))
        self.tiles = [np.zeros((0, self.d), dtype=np.int64)
                      for _ in range(levels)]
        self.kinds = [np.zeros(0, dtype=np.int8) for _ in range(levels)]
        self.version = 0
        self._cache = {}

    @classmethod
    def uniform(cls, finest_cells, levels=1, periodic=None):
        t = cls(finest_cells, levels, periodic)
        top = levels - 1
        dims = t.tiles_dims(top)
        coords = np.array(list(itertools.product(*[range(n) for n in dims])),
                          dtype=np.int64).reshape(-1, t.d)
        t.set_level(top, coords, np.zeros(len(coords), dtype=np.int8))
        t.bump()
        return t

    # geometry -------------------------------------------------------------
    def cells_dims(self, level):
        return tuple(v >> level for v in self.finest)

    def tiles_dims(self, level):
        return tuple(v // TILE for v in self.cells_dims(level))

    def n_tiles(self, level):
        return len(self.tiles[level])

    def cell_count(self, level):
        return self.n_tiles(level) * TILE ** self.d

    def bump(self):
        self.version += 1
        self._cache.clear()

    def set_level(self, level, coords, kinds):
        """Store tiles in canonical sorted order (sparse_grid.py:183-200);
        returns old slot per new slot (-1 = fresh)."""
        coords = np.asarray(coords, dtype=np.int64).reshape(-1, self.d)
        kinds = np.asarray(kinds, dtype=np.int8)
        order = np.lexsort(coords.T[::-1]) if len(coords) else \
            np.zeros(0, dtype=np.int64)
        coords = coords[order]
        kinds = kinds[order]
        old_map = self.tile_map(level)
        old = old_map[tuple(coords.T)] if len(coords) else \
            np.zeros(0, dtype=np.int64)
        self.tiles[level] = coords
        self.kinds[level] = kinds
        self._cache.clear()
        return old

    def tile_set(self):
        out = set()
        for l in range(self.levels):
            for c, k in zip(self.tiles[l], self.kinds[l]):
                out.add((l,) + tuple(int(v) for v in c) + (int(k),))
        return out

    # cached rasters ---------------------------------------------------------
    def _cached(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    def tile_map(self, level):
        def build():
            m = np.full(self.tiles_dims(level), -1, dtype=np.int64)
            if len(self.tiles[level]):
                m[tuple(self.tiles[level].T)] = np.arange(len(self.tiles[level]))
            return m
        return self._cached(("tmap", level), build)

    def tile_bitmap(self, level, kind=None):
        def build():
            m = np.zeros(self.tiles_dims(level), dtype=bool)
            sel = np.ones(len(self.tiles[level]), dtype=bool) if kind is None \
                else self.kinds[level] == kind
            if sel.any():
                m[tuple(self.tiles[level][sel].T)] = True
            return m
        return self._cached(("tbm", level, kind), build)

    def cell_coords(self, level):
        def build():
            off = local_offsets(self.d)
            t = self.tiles[level]
            return (t[:, None, :] * TILE + off[None]).reshape(-1, self.d)
        return self._cached(("coords", level), build)

    def cell_map(self, level):
        def build():
            m = np.full(self.cells_dims(level), -1, dtype=np.int64)
            cc = self.cell_coords(level)
            if len(cc):
                m[tuple(cc.T)] = np.arange(len(cc))
            return m
        return self._cached(("cmap", level), build)

    def leaf_cells(self, level):
        def build():
            return upsample_tiles(self.tile_bitmap(level, LEAF), self.d)
        return self._cached(("leaf", level), build)

    def leaf_flat(self, level):
        """Per stored cell: inside a leaf tile."""
        return np.repeat(self.kinds[level] == LEAF, TILE ** self.d)

    def owner_grid(self, level):
        """sparse_grid.py:255-282: coarsest first, finer overwrite; sample
        the cell's corner."""
        def build():
            dims = self.cells_dims(level)
            owner = np.full(dims, -1, dtype=np.int64)
            grids = np.meshgrid(*[np.arange(n) for n in dims], indexing="ij")
            for lp in range(self.levels - 1, -1, -1):
                leaf = self.leaf_cells(lp)
                if not leaf.any():
                    continue
                if lp >= level:
                    idx = tuple(g >> (lp - level) for g in grids)
                else:
                    idx = tuple(g << (level - lp) for g in grids)
                owner[leaf[idx]] = lp
            return owner
        return self._cached(("owner", level), build)

    # validation -------------------------------------------------------------
    def validate_coverage(self):
        count = np.zeros(self.finest, dtype=np.int64)
        for l in range(self.levels):
            leaf = self.leaf_cells(l)
            if not leaf.any():
                continue
            up = leaf.astype(np.int64)
            for a in range(self.d):
                up = np.repeat(up, 1 << l, axis=a)
            count += up
        if not np.all(count == 1):
            bad = np.argwhere(count != 1)
            raise TopologyError(f"leaf coverage violated at {len(bad)} cells")

    def validate_two_tile_overlap(self):
        for l in range(self.levels):
            leaf = self.tile_bitmap(l, LEAF)
            if not leaf.any():
                continue
            present = self.tile_bitmap(l)
            missing = dilate(leaf, 2, self.periodic) & ~present
            if missing.any():
                raise TopologyError(f"level {l}: ring tile missing")


def upsample_tiles(bitmap, d):
    out = bitmap
    for a in range(d):
        out = np.repeat(out, TILE, axis=a)
    return out


# -- field storage -------------------------------------------------------------

class FieldTree:
    def __init__(self, topo: Topology):
        self.levels = []
        for l in range(topo.levels):
            self.levels.append(fresh_arrays(topo.d, topo.cell_count(l)))


def fresh_arrays(d, n):
    arr = {nm: np.zeros(n) for nm in field_names(d)}
    arr["rho"][:] = 1.0
    arr["eps"][:] = 1.0
    return arr


class PingPongPair:
    def __init__(self, topo: Topology):
        self.trees = (FieldTree(topo), FieldTree(topo))
        self.bounce = 0


def buffer_roles(level, parity):
    """sparse_grid.py:396-405."""
    return (0, 1) if (level + parity) % 2 == 0 else (1, 0)


# -- interface sets ------------------------------------------------------------

def interp_stencil(cells, coarse_map, periodic, ratio_log2=1):
    """2^d multilinear stencil (sparse_grid.py:439-465); corner k uses
    offset bit a of k along axis a."""
    d = cells.shape[1]
    dims = coarse_map.shape
    base = cells >> ratio_log2
    frac = (cells & ((1 << ratio_log2) - 1)) / float(1 << ratio_log2)
    n = len(cells)
    idx = np.empty((n, 1 << d), dtype=np.int64)
    w = np.empty((n, 1 << d))
    for k in range(1 << d):
        cc = []
        wk = np.ones(n)
        for a in range(d):
            o = (k >> a) & 1
            ca = base[:, a] + o
            ca = ca % dims[a] if periodic[a] else ca.clip(0, dims[a] - 1)
            cc.append(ca)
            wk = wk * (frac[:, a] if o else 1.0 - frac[:, a])
        idx[:, k] = coarse_map[tuple(cc)]
        w[:, k] = wk
    return idx, w


class Interfaces:
    def __init__(self):
        self.downs = {}     # level -> (targets, src, w)
        self.ups = {}       # coarse level -> (targets, src, src_all)


def classify_interfaces(topo: Topology) -> Interfaces:
    """sparse_grid.py:468-544."""
    sets = Interfaces()
    d = topo.d
    for l in range(topo.levels):
        if topo.n_tiles(l) == 0:
            continue
        cmap = topo.cell_map(l)
        occ = cmap >= 0
        gap = ~occ
        if not gap.any():
            continue
        owner = topo.owner_grid(l)
        if (gap & (owner == l)).any():
            raise TopologyError(f"level {l}: leaf-owned cell not stored")
        gap_coarse = gap & (owner > l)
        gap_fine = gap & (owner >= 0) & (owner < l)
        id_mask = occ & dilate(gap_coarse, 2, topo.periodic)
        iu_mask = occ & dilate(gap_fine, 1, topo.periodic)
        if (id_mask & iu_mask).any():
            raise TopologyError(f"level {l}: downward and upward rims overlap")
        if id_mask.any():
            if l == topo.levels - 1:
                raise TopologyError("top level cannot have a downward rim")
            cells = np.argwhere(id_mask)
            idx, w = interp_stencil(cells, topo.cell_map(l + 1), topo.periodic)
            if ((w > 0) & (idx < 0)).any():
                raise TopologyError(f"I^d level {l} lacks coarse sources")
            sets.downs[l] = (cmap[tuple(cells.T)], idx, w)
        if iu_mask.any():
            if l == 0:
                raise TopologyError("level 0 cannot have an upward rim")
            cells = np.argwhere(iu_mask)
            fmap = topo.cell_map(l - 1)
            src = fmap[tuple((cells * 2).T)]
            if (src < 0).any():
                raise TopologyError(f"I^u level {l} lacks coincident source")
            fdims = topo.cells_dims(l - 1)
            src_all = np.empty((len(cells), 1 << d), dtype=np.int64)
            for k in range(1 << d):
                cc = []
                for a in range(d):
                    o = (k >> a) & 1
                    ca = cells[:, a] * 2 + o
                    ca = ca % fdims[a] if topo.periodic[a] else \
                        ca.clip(0, fdims[a] - 1)
                    cc.append(ca)
                src_all[:, k] = fmap[tuple(cc)]
            sets.ups[l] = (cmap[tuple(cells.T)], src, src_all)
    return sets
