"""Device-resident sparse tile hierarchy and ping-pong field storage.

Mirrors ``pkg/src/mlbm/sparse_grid.py`` (Topology / FieldTree /
PingPongPair / buffer_roles, :125-405) for d = 2 or 3, but every table lives
in HBM and is built by the sm_100a kernels of ``csrc/topology.cu``:

* per level a dense uint8 *kind grid* over the tile grid (0 absent, 1 leaf,
  2 border) is the source of truth; compaction into sorted slots
  (``mlbm_compact_tiles``) reproduces the reference's canonical
  ``sorted(coords)`` slot order (sparse_grid.py:191) bit-exactly;
* the dense ``tile_map`` (tile -> slot) is the block hash;
* ``nbr`` holds the 3^d neighbour slots per tile.

Host-side views (``tile_set``, ``cell_coords``, ``cell_map`` ...) copy to the
host on demand for tests and inspection; the step never calls them.
"""
from __future__ import annotations

from collections.abc import MutableMapping

import numpy as np
import torch

from . import _lib as L

TILE = 4
LEAF = 0            # reference kind values (sparse_grid.py:20-21)
BORDER = 1
KIND_NAMES = {LEAF: "leaf", BORDER: "border"}
DEV_LEAF = 1        # device kind-grid values
DEV_BORDER = 2

DEFAULT_DTYPE = torch.float64


class TopologyError(RuntimeError):
    """A structural invariant was violated (sparse_grid.py:33-34)."""


def field_names(d):
    ax = "xyz"[:d]
    s = ["s" + ax[a] + ax[b] for a in range(d) for b in range(a, d)]
    return ["rho"] + ["u" + a for a in ax] + s + ["eps"] + ["f" + a for a in ax] + ["phi"]


def moment_names(d):
    return field_names(d)[:1 + d + d * (d + 1) // 2]


def cells_per_tile(d):
    return TILE ** d


def n_nbr(d):
    return 3 ** d


def buffer_roles(level: int, bounce: int):
    """(read, write) tree indices (sparse_grid.py:396-405)."""
    return (0, 1) if (level + bounce) % 2 == 0 else (1, 0)


def _device():
    return torch.device("cuda", torch.cuda.current_device())


class LevelTopo:
    """Device tables of one level, allocated at a capacity (tiles) so that
    pointers stay fixed across topology changes; the live count is in
    ``Topology.dcounts`` (device) and ``n_tiles`` (host mirror)."""

    def __init__(self, d, grid_dims, device):
        self.d = d
        self.grid = tuple(grid_dims)                      # tile grid (3 axes)
        self.grid_n = int(np.prod(self.grid))
        self.kind = torch.zeros(self.grid_n, dtype=torch.uint8, device=device)
        self.tile_map = torch.full((self.grid_n,), -1, dtype=torch.int32, device=device)
        self.tile_map_new = torch.full((self.grid_n,), -1, dtype=torch.int32, device=device)
        self.n_tiles = 0
        self.cap = 0
        self.created = 0
        self.device = device
        self._alloc(0)

    def _alloc(self, cap):
        dev = self.device
        old = (getattr(self, "tile_xyz", None), getattr(self, "tile_kind", None),
               getattr(self, "nbr", None), getattr(self, "old_slot", None))
        # library memsets / fills: a capacity growth inside the timed steps
        # launches no framework kernel
        self.tile_xyz = L.zeros((cap, 3), torch.int32, dev)
        self.tile_kind = L.zeros(cap, torch.uint8, dev)
        self.nbr = L.full((cap, n_nbr(self.d)), -1, torch.int32, dev)
        self.old_slot = L.full((cap,), -1, torch.int32, dev)
        if old[0] is not None and self.cap:
            k = min(self.cap, cap)
            self.tile_xyz[:k].copy_(old[0][:k])
            self.tile_kind[:k].copy_(old[1][:k])
            self.nbr[:k].copy_(old[2][:k])
            self.old_slot[:k].copy_(old[3][:k])
        self.cap = cap


def capacity_for(n, grid_n, T):
    """Tile capacity of a level: 1.5x the need (at least +256) rounded to 256
    tiles, capped by the tile grid.  Kernels launch over the capacity and exit
    past the live count, so headroom costs empty blocks; growth bumps
    ``cap_version`` (the step graphs are re-captured)."""
    return min(grid_n, ((max(int(1.5 * n), n + 256) + 255) // 256) * 256)


class Topology:
    """Tile tables for all levels over a fixed box (sparse_grid.py:125-337)."""

    def __init__(self, finest_cells, levels: int, periodic=None, device=None):
        self.d = len(finest_cells)
        if self.d not in (2, 3):
            raise ValueError("2 or 3 extents expected")
        self.finest_cells = tuple(int(v) for v in finest_cells)
        if levels < 1:
            raise ValueError("levels must be >= 1")
        if levels > L.MAX_LEVELS:
            raise ValueError(f"at most {L.MAX_LEVELS} levels")
        step = TILE * (1 << (levels - 1))
        if any(v % step for v in self.finest_cells):
            raise ValueError(
                f"finest cells {self.finest_cells} must be divisible by {step} "
                f"(tile size x 2^(levels-1))")
        self.levels = levels
        self.periodic = tuple(bool(p) for p in
                              (periodic if periodic is not None else (True,) * self.d))
        self.device = device or _device()
        L.lib()
        self.lv = [LevelTopo(self.d, self.tile_grid(l), self.device)
                   for l in range(levels)]
        self.version = 0
        self.cap_version = 0
        # device counts per level: [live tiles, fresh tiles, |I^d|, |I^u|]
        self.dcounts = torch.zeros((levels, 4), dtype=torch.int32, device=self.device)
        self._ws = torch.zeros(0, dtype=torch.uint8, device=self.device)
        self._host_cache = {}

    # -- geometry -------------------------------------------------------------
    def cells_dims(self, level):
        return tuple(v >> level for v in self.finest_cells)

    def tiles_dims(self, level):
        return tuple(v // TILE for v in self.cells_dims(level))

    def tile_grid(self, level):
        t = self.tiles_dims(level)
        return t + (1,) * (3 - self.d)

    def cell_grid(self, level):
        c = self.cells_dims(level)
        return c + (1,) * (3 - self.d)

    def n_tiles(self, level):
        return self.lv[level].n_tiles

    def cell_count(self, level):
        return self.lv[level].n_tiles * TILE ** self.d

    def periodic3(self):
        return tuple(int(p) for p in self.periodic) + (0,) * (3 - self.d)

    @classmethod
    def uniform(cls, finest_cells, levels: int = 1, periodic=None, device=None):
        """All-leaf coverage at the coarsest level (sparse_grid.py:167-177)."""
        topo = cls(finest_cells, levels, periodic, device)
        top = levels - 1
        kinds = {top: torch.full_like(topo.lv[top].kind, DEV_LEAF)}
        topo.rebuild(kinds)
        return topo

    def set_tile_set(self, tiles):
        """Load an explicit tile set {(level, *coords, kind)} with reference
        kinds (LEAF = 0, BORDER = 1) into every level (host upload; the
        apply_reference_topology helper of adapt.py:474-481)."""
        kinds = {}
        for l in range(self.levels):
            kinds[l] = np.zeros(self.tile_grid(l), dtype=np.uint8)
        for e in tiles:
            l, c, k = e[0], tuple(e[1:-1]) + (0,) * (3 - self.d), e[-1]
            kinds[l][c] = DEV_LEAF if k == LEAF else DEV_BORDER
        self.rebuild({l: torch.as_tensor(k.reshape(-1), device=self.device)
                      for l, k in kinds.items()})

    def workspace(self, n):
        need = int(L.lib().mlbm_ws_bytes(int(n)))
        if self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    # -- rebuild ----------------------------------------------------------------
    def ensure_capacity(self, level, n):
        """Grow a level's tile arrays to hold n tiles (keeps content)."""
        lt = self.lv[level]
        if n <= lt.cap:
            return False
        lt._alloc(capacity_for(n, lt.grid_n, TILE ** self.d))
        self.cap_version += 1
        return True

    def compact(self, level, kind):
        """Sorted-slot compaction of a new kind grid into ``tile_map_new``,
        ``tile_xyz``, ``tile_kind``, ``old_slot`` and ``dcounts[level, 0:2]``
        (sparse_grid.py:183-200).  No host synchronisation."""
        lt = self.lv[level]
        ws = self.workspace(lt.grid_n)
        tiles = (L.C.c_int32 * 3)(*self.tile_grid(level))
        L.check(L.lib().mlbm_compact_tiles(self.d, tiles, L.ptr(kind), L.ptr(lt.tile_map),
                                           L.ptr(lt.tile_map_new), L.ptr(lt.tile_xyz),
                                           L.ptr(lt.tile_kind), L.ptr(lt.old_slot), lt.cap,
                                           L.ptr(self.dcounts[level]), L.ptr(ws), ws.numel(),
                                           L.stream_handle()), "compact_tiles")

    def build_neighbors(self, level, new_map=True):
        lt = self.lv[level]
        if not lt.cap:
            return
        st = self.level_struct(level)
        if new_map:
            st.tile_map = lt.tile_map_new.data_ptr()
        L.check(L.lib().mlbm_build_neighbors(L.C.byref(st), L.ptr(lt.nbr), L.stream_handle()),
                "build_neighbors")

    def commit_device(self, kinds: dict):
        """Make the compacted maps / kinds current (device copies only)."""
        for level, kind in kinds.items():
            lt = self.lv[level]
            lt.tile_map.copy_(lt.tile_map_new)
            if kind.data_ptr() != lt.kind.data_ptr():
                lt.kind.copy_(kind)

    def commit_host(self, counts: dict):
        """Host mirrors take the known new counts; bumps the topology version."""
        for level, n in counts.items():
            self.lv[level].n_tiles = int(n)
        self.bump()

    def commit(self, kinds: dict, counts: dict):
        self.commit_device(kinds)
        self.commit_host(counts)

    def rebuild(self, kinds: dict):
        """Replace the kind grids of the given levels (host-driven path used
        at construction and by ``set_tile_set``; counts read back)."""
        counts = {l: int((k != 0).sum().item()) for l, k in kinds.items()}
        self.host_rebuilds = getattr(self, "host_rebuilds", 0) + 1   # GridAdaptor windows reset
        for l, n in counts.items():
            self.ensure_capacity(l, n)
        for l, k in kinds.items():
            self.compact(l, k)
        for l in kinds:
            self.build_neighbors(l, new_map=True)
        created = self.dcounts[:, 1].cpu().numpy()
        for l in kinds:
            self.lv[l].created = int(created[l])
        self.commit(kinds, counts)

    def bump(self):
        self.version += 1
        self._host_cache.clear()

    # -- C structs --------------------------------------------------------------
    def level_struct(self, level, tables=None):
        lt = self.lv[level]
        st = L.Level()
        st.dim = self.d
        st.level = level
        for a, v in enumerate(self.cell_grid(level)):
            st.cells[a] = v
        for a, v in enumerate(self.tile_grid(level)):
            st.tiles[a] = v
        for a, v in enumerate(self.periodic3()):
            st.periodic[a] = v
        st.n_tiles = lt.cap                   # launch capacity; live count on device
        st.tile_map = lt.tile_map.data_ptr()
        st.tile_xyz = lt.tile_xyz.data_ptr() if lt.cap else 0
        st.nbr = lt.nbr.data_ptr() if lt.cap else 0
        st.counts = self.dcounts[level].data_ptr()
        if tables is not None and lt.cap:
            st.cell_flags = tables.cell_flags.data_ptr()
            st.dir_masks = tables.dir_masks.data_ptr()
            st.tile_flags = tables.tile_flags.data_ptr()
        return st

    def capacity_cells(self, level):
        return self.lv[level].cap * TILE ** self.d

    def hier_struct(self, pair=None):
        h = L.Hier()
        h.dim = self.d
        h.levels = self.levels
        for a in range(3):
            h.finest[a] = self.finest_cells[a] if a < self.d else 4
            h.periodic[a] = self.periodic3()[a]
        for l in range(self.levels):
            h.kind[l] = self.lv[l].kind.data_ptr()
            h.tile_map[l] = self.lv[l].tile_map.data_ptr()
            h.n_tiles[l] = self.lv[l].n_tiles
            if pair is not None:
                for t in range(2):
                    a = pair.trees[t].levels[l].data
                    h.fields[t][l] = a.data_ptr() if a.numel() else 0
                    h.stride[l] = a.stride(0) if a.numel() else 0
        return h

    # -- host views (tests / inspection) -----------------------------------------
    def _host(self, key, fn):
        if key not in self._host_cache:
            self._host_cache[key] = fn()
        return self._host_cache[key]

    def tile_coords(self, level):
        n = self.lv[level].n_tiles
        return self._host(("xyz", level),
                          lambda: self.lv[level].tile_xyz[:n, :self.d].cpu().numpy()
                          .astype(np.int64))

    def tile_kinds(self, level):
        """Reference kind values (LEAF = 0, BORDER = 1) per slot."""
        n = self.lv[level].n_tiles
        return self._host(("kind", level),
                          lambda: self.lv[level].tile_kind[:n].cpu().numpy().astype(np.int64) - 1)

    def kind_grid(self, level):
        return self._host(("kgrid", level),
                          lambda: self.lv[level].kind.cpu().numpy().reshape(
                              self.tile_grid(level))[(...,) if self.d == 3 else (..., 0)])

    def tile_set(self) -> set:
        out = set()
        for l in range(self.levels):
            for c, k in zip(self.tile_coords(l), self.tile_kinds(l)):
                out.add((l,) + tuple(int(v) for v in c) + (int(k),))
        return out

    def dump_text(self) -> str:
        lines = []
        for l in range(self.levels):
            for c, k in zip(self.tile_coords(l), self.tile_kinds(l)):
                lines.append(f"{l} " + " ".join(str(int(v)) for v in c) + f" {KIND_NAMES[int(k)]}")
        return "\n".join(lines) + ("\n" if lines else "")

    def cell_coords(self, level):
        def build():
            t = self.tile_coords(level)
            n = TILE ** self.d
            idx = np.arange(n)
            off = np.stack([(idx // TILE ** a) % TILE for a in range(self.d)], axis=1)
            return (t[:, None, :] * TILE + off[None]).reshape(-1, self.d)
        return self._host(("coords", level), build)

    def cell_map(self, level):
        def build():
            m = np.full(self.cells_dims(level), -1, dtype=np.int64)
            cc = self.cell_coords(level)
            if len(cc):
                m[tuple(cc.T)] = np.arange(len(cc))
            return m
        return self._host(("cmap", level), build)

    def leaf_flat(self, level):
        return np.repeat(self.tile_kinds(level) == LEAF, TILE ** self.d)

    def leaf_cells(self, level):
        def build():
            g = self.kind_grid(level) == DEV_LEAF
            for a in range(self.d):
                g = np.repeat(g, TILE, axis=a)
            return g
        return self._host(("leaf", level), build)


# -- field storage -------------------------------------------------------------

class LevelFields(MutableMapping):
    """Name -> 1-D device view of one level's SoA block ``data[nf, n]``.

    Storage keeps drho = rho - 1 in row 0 (the shifted form); ``self["rho"]``
    returns a fresh 1 + drho tensor and ``self["rho"] = v`` stores v - 1.
    Every other name is a live view (in-place writes land in HBM).
    """

    def __init__(self, d, data, live=None):
        self.d = d
        self.data = data                 # [nf, capacity cells]
        self.live = live                 # callable -> live cell count (None: all)
        self.names = field_names(d)
        self.index = {nm: i for i, nm in enumerate(self.names)}

    def n(self):
        return self.data.shape[1] if self.live is None else self.live()

    def __getitem__(self, name):
        i = self.index[name]
        n = self.n()
        if i == 0:
            return 1.0 + self.data[0, :n]
        return self.data[i, :n]

    def __setitem__(self, name, value):
        i = self.index[name]
        n = self.n()
        v = torch.as_tensor(value, dtype=self.data.dtype, device=self.data.device)
        if i == 0:
            self.data[0, :n].copy_(v - 1.0)
        else:
            self.data[i, :n].copy_(v)

    def __delitem__(self, name):
        raise TypeError("fields are fixed")

    def __iter__(self):
        return iter(self.names)

    def __len__(self):
        return len(self.names)

    def numpy(self):
        out = {nm: self[nm].detach().cpu().numpy() for nm in self.names}
        return out

    def __len_cells__(self):
        return self.data.shape[1]


def fresh_block(d, n, dtype, device):
    data = L.zeros((len(field_names(d)), n), dtype, device)
    if data.is_cuda:
        L.fill(data[field_names(d).index("eps")], 1.0)
    else:
        data[field_names(d).index("eps")] = 1.0
    return data


class FieldTree:
    """Per-level SoA blocks over the stored tiles (sparse_grid.py:369-382),
    allocated at the level capacity."""

    def __init__(self, topology: Topology, dtype=None):
        dtype = dtype or DEFAULT_DTYPE
        self.levels = [LevelFields(topology.d,
                                   fresh_block(topology.d, topology.capacity_cells(l), dtype,
                                               topology.device),
                                   live=(lambda l=l: topology.cell_count(l)))
                       for l in range(topology.levels)]

    def nbytes(self):
        return sum(lv.data.numel() * lv.data.element_size() for lv in self.levels)


class PingPongPair:
    """Two field trees with identical topology plus the bounce counter.
    ``scratch[l]`` is the migration target of a level (same capacity)."""

    def __init__(self, topology: Topology, dtype=None):
        self.dtype = dtype or DEFAULT_DTYPE
        self.topology = topology
        self.trees = (FieldTree(topology, self.dtype), FieldTree(topology, self.dtype))
        self.scratch = {}
        self.bounce = 0

    def ensure_capacity(self):
        """Grow field blocks to the topology capacity (content kept)."""
        topo = self.topology
        for l in range(topo.levels):
            cap = topo.capacity_cells(l)
            for tree in self.trees:
                lf = tree.levels[l]
                if lf.data.shape[1] < cap:
                    nb = fresh_block(topo.d, cap, self.dtype, topo.device)
                    k = lf.data.shape[1]
                    nb[:, :k].copy_(lf.data)
                    lf.data = nb

    def scratch_blocks(self, level):
        cap = self.topology.capacity_cells(level)
        sb = self.scratch.get(level)
        if sb is None or sb[0].shape[1] != cap:
            sb = tuple(fresh_block(self.topology.d, cap, self.dtype, self.topology.device)
                       for _ in range(2))
            self.scratch[level] = sb
        return sb

    def nbytes(self):
        return self.trees[0].nbytes() + self.trees[1].nbytes()


def dtype_code(dtype):
    if dtype == torch.float32:
        return 0
    if dtype == torch.float64:
        return 1
    raise ValueError(f"unsupported dtype {dtype}")
