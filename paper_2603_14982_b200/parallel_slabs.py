"""Spatial slab decomposition for the multi-GPU path.

The reference is single-process (``coupling.py:364-365``: ``threads`` is
recorded, unused).  The B200 build splits the domain into slabs along x, one
per rank, cut on the coarsest tile width ``4 * 2**(levels-1)`` so that every
level's tiles — and the downward / upward stencils, which stay within a
coarse tile — live on one rank.  Per finest cycle the ranks exchange:

  (i)   before each level step, a one-tile-column halo of the read tree on both
        x faces (the pull stencil has radius 1, ``solver.py:239-253``);
  (ii)  after P2G, ghost-node partial sums two cells deep;
  (iii) after G2P, the particles whose x left the slab (CFL < 1 cell/step, so
        only nearest neighbours);
  (iv)  for block maintenance, a bitwise-OR all-reduce of the level-0 seed
        bitmap, after which every rank evaluates the global bitmaps
        redundantly (bit-exact by construction) and materialises its slab.

This module holds the backend-agnostic host logic (index arithmetic, routing,
collective calls through ``torch.distributed``).  It is exercised with the
gloo backend at world size 2 on CPU (``tests/test_dist_cpu.py``); the device
path passes CUDA tensors to the same calls over NCCL.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

TILE = 4


@dataclass(frozen=True)
class SlabPartition:
    finest_cells: tuple
    levels: int
    world: int
    periodic_x: bool = True

    def __post_init__(self):
        w = self.coarse_width
        nx = self.finest_cells[0]
        if nx % w:
            raise ValueError(f"x extent {nx} not divisible by the coarse tile width {w}")
        if nx // w < self.world:
            raise ValueError(f"{nx // w} coarse tile columns cannot feed {self.world} ranks")

    @property
    def coarse_width(self):
        return TILE * (1 << (self.levels - 1))

    def cuts(self):
        """Finest-cell x cuts [x_0 = 0, ..., x_world = nx] on coarse-tile bounds."""
        w = self.coarse_width
        ncol = self.finest_cells[0] // w
        base, extra = divmod(ncol, self.world)
        cols = [base + (1 if r < extra else 0) for r in range(self.world)]
        return [0] + list(np.cumsum(cols) * w)

    def slab(self, rank):
        c = self.cuts()
        return c[rank], c[rank + 1]

    def tile_columns(self, rank, level):
        """Owned level-``level`` tile x-columns [c0, c1)."""
        x0, x1 = self.slab(rank)
        tw = TILE << level
        return x0 // tw, x1 // tw

    def halo_columns(self, rank, level):
        """Tile columns read from the neighbours before a level step: one
        column on each side (wrapped when periodic, absent at a wall)."""
        c0, c1 = self.tile_columns(rank, level)
        ntx = (self.finest_cells[0] >> level) // TILE
        left, right = c0 - 1, c1
        if self.periodic_x:
            left %= ntx
            right %= ntx
        else:
            left = left if left >= 0 else None
            right = right if right < ntx else None
        return left, right

    def neighbors(self, rank):
        """(left, right) neighbour ranks (None at a non-periodic wall)."""
        lft, rgt = rank - 1, rank + 1
        if self.periodic_x:
            return lft % self.world, rgt % self.world
        return (lft if lft >= 0 else None), (rgt if rgt < self.world else None)

    def owner(self, x):
        """Rank owning finest-unit x positions (array)."""
        x = np.asarray(x, dtype=float)
        nx = self.finest_cells[0]
        if self.periodic_x:
            x = np.mod(x, nx)
        c = np.asarray(self.cuts()[1:-1], dtype=float)
        return np.searchsorted(c, x, side="right").astype(np.int64)

    def ghost_node_columns(self, rank):
        """Level-0 node x-ranges written by this rank's particles but owned by
        the neighbours: 2 nodes below x0 (base = floor(x - 1/2) >= x0 - 1
        for x >= x0 ... the quadratic stencil reaches x0 - 1) and 2 above
        x1 - 1 (stencil base + 2 <= x1 + 1)."""
        x0, x1 = self.slab(rank)
        return (x0 - 2, x0), (x1, x1 + 2)


def route_particles(part: SlabPartition, rank: int, x: np.ndarray):
    """Indices of local particles per destination rank (after G2P)."""
    own = part.owner(x[:, 0])
    out = {}
    for r in np.unique(own):
        if int(r) != rank:
            out[int(r)] = np.nonzero(own == r)[0]
    return out, np.nonzero(own == rank)[0]


def _sendrecv(send_to, send_t, recv_from, recv_like):
    """Paired point-to-point exchange with one neighbour (isend + irecv)."""
    reqs = []
    recv = torch.empty_like(recv_like)
    if send_to is not None:
        reqs.append(dist.isend(send_t.contiguous(), send_to))
    if recv_from is not None:
        reqs.append(dist.irecv(recv, recv_from))
    for q in reqs:
        q.wait()
    return recv if recv_from is not None else None


def exchange_halo_x(part: SlabPartition, rank: int, slab: torch.Tensor, depth: int):
    """Face halo along x of a dense slab block ``[nf, nx_local, ...]``:
    returns ``[nf, depth + nx_local + depth, ...]`` with the neighbours'
    edge layers (the read-tree halo of exchange (i); ``depth`` = 4 cells =
    one tile column).  Wall sides are padded by edge replication."""
    left, right = part.neighbors(rank)
    lo_edge = slab[:, :depth]
    hi_edge = slab[:, -depth:]
    # send my low edge to the left, receive the right neighbour's low edge
    from_right = _sendrecv(left, lo_edge, right, hi_edge)
    from_left = _sendrecv(right, hi_edge, left, lo_edge)
    if from_left is None:
        from_left = lo_edge[:, :1].expand_as(lo_edge).clone()
    if from_right is None:
        from_right = hi_edge[:, -1:].expand_as(hi_edge).clone()
    return torch.cat([from_left, slab, from_right], dim=1)


def reduce_ghost_nodes(part: SlabPartition, rank: int, acc: torch.Tensor, depth: int = 2):
    """Exchange (ii): ``acc`` is ``[rows, depth + nx_local + depth, ...]`` of
    P2G partial sums including the ghost node layers; the ghost layers are
    sent to their owners and added to their interior edges.  Returns the
    interior ``[rows, nx_local, ...]``."""
    left, right = part.neighbors(rank)
    lo_ghost = acc[:, :depth]
    hi_ghost = acc[:, -depth:]
    interior = acc[:, depth:-depth].clone()
    from_right = _sendrecv(left, lo_ghost, right, hi_ghost)   # right's low ghosts
    from_left = _sendrecv(right, hi_ghost, left, lo_ghost)    # left's high ghosts
    if from_right is not None:
        interior[:, -depth:] += from_right
    if from_left is not None:
        interior[:, :depth] += from_left
    return interior


def migrate_particles(part: SlabPartition, rank: int, x: torch.Tensor, state: torch.Tensor):
    """Exchange (iii): send particles that left the slab to the neighbour
    owning them (count, then payload), receive the arrivals.  ``x``: [n, d]
    float64 positions, ``state``: [n, k] per-particle rows (float64 here;
    the device path sends the run-dtype rows)."""
    dest, keep = route_particles(part, rank, x.cpu().numpy())
    left, right = part.neighbors(rank)
    bad = [r for r in dest if r not in (left, right)]
    if bad:
        raise RuntimeError(f"particles jumped past the nearest slab (to ranks {bad})")
    d, k = x.shape[1], state.shape[1]
    out_x, out_s = [x[keep]], [state[keep]]
    empty = np.zeros(0, dtype=np.int64)
    sent = set()
    for send_to, recv_from in ((left, right), (right, left)):
        idx = empty
        if send_to is not None and send_to not in sent:
            idx = dest.get(send_to, empty)
            sent.add(send_to)
        cnt = torch.tensor([len(idx)], dtype=torch.int64)
        rcnt = _sendrecv(send_to, cnt, recv_from, cnt)
        n_in = int(rcnt.item()) if rcnt is not None else 0
        payload = torch.cat([x[idx], state[idx].to(x.dtype)], dim=1)
        got = _sendrecv(send_to if len(idx) else None, payload,
                        recv_from if n_in else None,
                        torch.zeros((n_in, d + k), dtype=x.dtype))
        if got is not None:
            out_x.append(got[:, :d])
            out_s.append(got[:, d:].to(state.dtype))
    return torch.cat(out_x), torch.cat(out_s)


def allreduce_seeds(seeds: torch.Tensor):
    """Exchange (iv): bitwise OR of uint8 seed bitmaps (MAX on {0, 1})."""
    t = seeds.to(torch.uint8)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t
