"""Slab decomposition of the coupled multi-level step over a static hierarchy
(SURVEY.md §8(e) collectives (i), (ii), (iii), (v)).

Each rank owns an x-slab (cut on the coarsest tile width) and keeps a local
box = slab + one coarsest tile of ghost region per neighbour side
(``slab_lbm.SlabMultiLevel``).  A local ``CoupledSim`` runs the reference's
coupled cycle (coupling.py:448-481) with the same kernels, plus:

  (i)   after every level-l stream / step / collide, the owned edge columns of
        the level's write tree go to the neighbours' ghost columns;
  (ii)  after P2G, the accumulator rows (mass, momentum, internal force, eta,
        area, sum w m v) of the ghost region are added into the owners' edge
        columns, and the completed edge rows are copied back into the ghost
        region — so the exchange kernel (drag, grad eps, grid update) computes
        the ghost cells near the cut exactly as their owner does, and G2P of
        particles near the cut gathers correct grid velocities;
  (iii) after the step, particles whose x left the slab move to the
        neighbour (count, then payload);
  (v)   the diagnostics row is reduced over ranks (sums; eps min).

  (iv)  block maintenance: every rank keeps the global kind grids and adapt
        state and runs the adapt pass redundantly on the uint8 OR (MAX) of the
        ranks' seed tiles, then rebuilds its local box;

``ThreadExchanger`` runs the ranks as threads of one process on one GPU
(tests); ``P2PExchanger`` is the torch.distributed (NCCL) version.
"""
from __future__ import annotations

import threading

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .adapt import GridAdaptor, RefineDriver
from .coupling import CoupledSim
from .granular import Particles, _d3, _faces, snow_arg
from .slab_lbm import SlabMultiLevel, exchange_columns
from .solver import FIELD_FORCE, FIELD_TAU, MultiLevelSolver
from .sparse_grid import TILE, Topology, dtype_code, moment_names


class ThreadExchanger:
    """Rank threads of one process: a shared mailbox and a barrier."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.box = {}

    def _post(self, rank, key, val):
        self.box[(rank, key)] = val

    def _sync(self):
        torch.cuda.synchronize()
        self.barrier.wait()

    def columns(self, sl, edge_l, edge_r, ghost_l, ghost_r):
        self._post(sl.rank, "cols", (edge_l.clone(), edge_r.clone()))
        self._sync()
        if ghost_l is not None:
            ghost_l.copy_(self.box[(sl.left, "cols")][1])
        if ghost_r is not None:
            ghost_r.copy_(self.box[(sl.right, "cols")][0])
        self._sync()

    def ghost_reduce(self, sl, ghost_l, ghost_r, edge_l, edge_r):
        self._post(sl.rank, "ghost", (None if ghost_l is None else ghost_l.clone(),
                                       None if ghost_r is None else ghost_r.clone()))
        self._sync()
        if sl.left is not None:
            edge_l.add_(self.box[(sl.left, "ghost")][1])
        if sl.right is not None:
            edge_r.add_(self.box[(sl.right, "ghost")][0])
        self._sync()

    def particles(self, sl, to_left, to_right):
        self._post(sl.rank, "parts", (to_left, to_right))
        self._sync()
        got = []
        if sl.left is not None:
            got.append(self.box[(sl.left, "parts")][1])
        if sl.right is not None and sl.right != sl.left:
            got.append(self.box[(sl.right, "parts")][0])
        elif sl.right is not None:
            got.append(self.box[(sl.right, "parts")][0])
        self._sync()
        return got

    def migrate_counts(self, sl, n_left, n_right):
        """(iii) counts: my leavers per side -> arrivals (from left, from right)."""
        self._post(sl.rank, "mcnt", (n_left, n_right))
        self._sync()
        ml = self.box[(sl.left, "mcnt")][1] if sl.left is not None else 0
        mr = self.box[(sl.right, "mcnt")][0] if sl.right is not None else 0
        self._sync()
        return ml, mr

    def migrate_payload(self, sl, send_l, send_r, recv_l, recv_r):
        """(iii) payloads: one contiguous byte message per direction."""
        self._post(sl.rank, "mpay", (send_l, send_r))
        self._sync()
        if sl.left is not None and recv_l is not None and recv_l.numel():
            recv_l.copy_(self.box[(sl.left, "mpay")][1])
        if sl.right is not None and recv_r is not None and recv_r.numel():
            recv_r.copy_(self.box[(sl.right, "mpay")][0])
        self._sync()

    def allreduce(self, sl, t, op):
        self._post(sl.rank, "red", t.clone())
        self._sync()
        vals = [self.box[(r, "red")] for r in range(self.world)]
        out = vals[0].clone()
        for v in vals[1:]:
            out = (torch.minimum(out, v) if op == "min" else
                   torch.maximum(out, v) if op == "max" else out + v)
        t.copy_(out)
        self._sync()


class P2PExchanger:
    """torch.distributed point-to-point / all-reduce (NCCL between GPUs).
    With a gloo process group (CPU transport) CUDA tensors are staged through
    host memory, so the same multi-process code path runs on one GPU."""

    def __init__(self):
        self._bufs = {}
        self.stage = dist.is_initialized() and dist.get_backend() == "gloo"

    def _h(self, t):
        return t.cpu() if (self.stage and t is not None and t.is_cuda) else t

    def columns(self, sl, edge_l, edge_r, ghost_l, ghost_r):
        if self.stage:
            gl = self._h(ghost_l).clone() if ghost_l is not None else None
            gr = self._h(ghost_r).clone() if ghost_r is not None else None
            send = [torch.empty_like(self._h(edge_l)), torch.empty_like(self._h(edge_r))]
            recv = [torch.empty_like(gl if gl is not None else send[0]),
                    torch.empty_like(gr if gr is not None else send[1])]
            exchange_columns(self._h(edge_l), self._h(edge_r), gl, gr, sl.left, sl.right, send, recv)
            if ghost_l is not None:
                ghost_l.copy_(gl)
            if ghost_r is not None:
                ghost_r.copy_(gr)
            return
        key = ("c", edge_l.shape, edge_r.shape)
        if key not in self._bufs:
            self._bufs[key] = ([torch.empty_like(edge_l), torch.empty_like(edge_r)],
                               [torch.empty_like(ghost_l) if ghost_l is not None else torch.empty_like(edge_l),
                                torch.empty_like(ghost_r) if ghost_r is not None else torch.empty_like(edge_r)])
        send, recv = self._bufs[key]
        exchange_columns(edge_l, edge_r, ghost_l, ghost_r, sl.left, sl.right, send, recv)

    def ghost_reduce(self, sl, ghost_l, ghost_r, edge_l, edge_r):
        # send my ghost sums to their owners, receive theirs for my edges
        recv_l = torch.empty_like(self._h(edge_l)) if sl.left is not None else None
        recv_r = torch.empty_like(self._h(edge_r)) if sl.right is not None else None

        def packed(v):
            h = self._h(v)
            return L.pack_cols(h, torch.empty(h.shape, dtype=h.dtype, device=h.device))
        ops = []
        if sl.right is not None:
            ops.append(dist.P2POp(dist.isend, packed(ghost_r), sl.right))
        if sl.left is not None:
            ops.append(dist.P2POp(dist.isend, packed(ghost_l), sl.left))
        if sl.left is not None:
            ops.append(dist.P2POp(dist.irecv, recv_l, sl.left))
        if sl.right is not None:
            ops.append(dist.P2POp(dist.irecv, recv_r, sl.right))
        for q in dist.batch_isend_irecv(ops):
            q.wait()
        if recv_l is not None:
            L.unpack_cols(recv_l.to(edge_l.device), edge_l, add=True)
        if recv_r is not None:
            L.unpack_cols(recv_r.to(edge_r.device), edge_r, add=True)

    def particles(self, sl, to_left, to_right):
        dev = to_left.device
        to_left, to_right = self._h(to_left), self._h(to_right)
        got = []
        for send_to, payload, recv_from in ((sl.right, to_right, sl.left), (sl.left, to_left, sl.right)):
            n_out = torch.tensor([payload.shape[1] if payload is not None else 0], dtype=torch.int64,
                                 device=payload.device if payload is not None else "cuda")
            n_in = torch.zeros_like(n_out)
            ops = []
            if send_to is not None:
                ops.append(dist.P2POp(dist.isend, n_out, send_to))
            if recv_from is not None:
                ops.append(dist.P2POp(dist.irecv, n_in, recv_from))
            for q in dist.batch_isend_irecv(ops):
                q.wait()
            rows = payload.shape[0]
            buf = torch.empty((rows, int(n_in.item())), dtype=payload.dtype, device=payload.device)
            ops = []
            if send_to is not None and payload.shape[1]:
                ops.append(dist.P2POp(dist.isend, payload.contiguous(), send_to))
            if recv_from is not None and buf.shape[1]:
                ops.append(dist.P2POp(dist.irecv, buf, recv_from))
            if ops:
                for q in dist.batch_isend_irecv(ops):
                    q.wait()
            got.append(buf.to(dev))
        return got

    def migrate_counts(self, sl, n_left, n_right):
        """(iii) counts (two phases: to the right / from the left, then to
        the left / from the right — pairs up even when left == right)."""
        dev = "cpu" if self.stage else "cuda"
        got = []
        for send_to, cnt, recv_from in ((sl.right, n_right, sl.left), (sl.left, n_left, sl.right)):
            out = torch.tensor([cnt], dtype=torch.int64, device=dev)
            inn = torch.zeros(1, dtype=torch.int64, device=dev)
            ops = []
            if send_to is not None:
                ops.append(dist.P2POp(dist.isend, out, send_to))
            if recv_from is not None:
                ops.append(dist.P2POp(dist.irecv, inn, recv_from))
            for q in dist.batch_isend_irecv(ops):
                q.wait()
            got.append(int(inn.item()) if recv_from is not None else 0)
        return got[0], got[1]

    def migrate_payload(self, sl, send_l, send_r, recv_l, recv_r):
        """(iii) payloads: one contiguous byte message per direction, same
        two-phase order as migrate_counts."""
        for send_to, buf, recv_from, rbuf in ((sl.right, send_r, sl.left, recv_l),
                                              (sl.left, send_l, sl.right, recv_r)):
            ops = []
            hb = self._h(buf) if buf is not None else None
            hr = None
            if rbuf is not None and rbuf.numel():
                hr = torch.empty(rbuf.shape, dtype=rbuf.dtype, device="cpu") if self.stage else rbuf
            if send_to is not None and hb is not None and hb.numel():
                ops.append(dist.P2POp(dist.isend, hb, send_to))
            if recv_from is not None and hr is not None:
                ops.append(dist.P2POp(dist.irecv, hr, recv_from))
            if ops:
                for q in dist.batch_isend_irecv(ops):
                    q.wait()
            if hr is not None and hr is not rbuf:
                rbuf.copy_(hr)

    def allreduce(self, sl, t, op):
        h = self._h(t)
        dist.all_reduce(h, op={"min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}.get(
            op, dist.ReduceOp.SUM))
        if h is not t:
            t.copy_(h)


class _SlabSolver(MultiLevelSolver):
    """Level steps over the owned slot range; (i) after every write."""

    slab = None

    def _level_call(self, level, src, dst, mode, cp=None):
        sl = self.slab
        if self.topology.lv[level].cap == 0:
            return
        self._refresh_tables()
        a, b = sl.ranges[level]["owned"]
        if b > a:
            cp = cp or self._collide_struct(level)
            L.check(L.lib().mlbm_level_step(L.C.byref(sl._owned_struct(level)),
                                            L.fields(dst_data(src)), L.fields(dst_data(dst)),
                                            self.dcode, mode, L.C.byref(cp), L.C.byref(self._bc),
                                            L.ptr(self._err), L.stream_handle()), "level_step")
        self.launches += 1
        sl.owner.exchange_level(level, dst)


def dst_data(a):
    return a.data if hasattr(a, "data") and not torch.is_tensor(a) else a


class SlabCoupled(CoupledSim):
    """One rank of the slab-decomposed coupled step (static hierarchy)."""

    def __init__(self, ref: CoupledSim, rank: int, world: int, exchanger):
        self.rank, self.world, self.xch = rank, world, exchanger
        topo = ref.topology
        d = topo.d
        per = tuple(bool(p) for p in topo.periodic) + (True,) * (3 - d)
        faces = dict(ref.solver.boundaries.faces)
        self.sl = SlabMultiLevel(topo.finest_cells, topo.levels, topo.tile_set(), rank, world,
                                 ref.solver.level_params.tau0, dtype=ref.dtype, periodic=per,
                                 params=ref.solver.params, level_params=ref.solver.level_params,
                                 faces=faces, solver_cls=_SlabSolver)
        sl = self.sl
        sl.owner = self
        sl.solver.slab = sl
        # fields of the reference state, by coordinates, into both local trees
        for l in range(topo.levels):
            if not sl.topology.n_tiles(l):
                continue
            gkey = {tuple(c): i for i, c in enumerate(topo.cell_coords(l).tolist())}
            lc = sl.topology.cell_coords(l).copy()
            lc[:, 0] = np.mod(lc[:, 0] + (sl.x0 >> l), topo.finest_cells[0] >> l)
            idx = torch.as_tensor([gkey[tuple(c)] for c in lc.tolist()], device=topo.device)
            nloc = sl.topology.cell_count(l)
            for t in range(2):
                sl.pair.trees[t].levels[l].data[:, :nloc].copy_(
                    ref.pair.trees[t].levels[l].data[:, :topo.cell_count(l)][:, idx])
        x0, x1 = sl.part.slab(rank)
        self.x_lo, self.x_hi = x0, x1
        p = ref.particles
        gx = p.x.cpu().numpy()
        own = (sl.part.owner(gx[:, 0]) == rank)
        part = self._make_particles(ref, torch.as_tensor(np.nonzero(own)[0], device=topo.device))
        super().__init__(sl.solver, part, ref.material, sediment_gravity=ref.sediment_gravity,
                         drag=ref.drag_params, powder=ref.powder, adaptor=None,
                         unit_scale=ref.unit_scale)
        self.drag_params.d_p = ref.drag_params.d_p
        self._global_active = len(ref.particles) > 0
        self.use_graphs = False
        self.sort_particles = True
        # (iv) block maintenance: every rank keeps the GLOBAL kind grids and
        # adapt state and runs the pass redundantly on OR-reduced seeds; the
        # new global kinds are cropped to the local box and the local
        # topology is rebuilt / migrated with the same kernels
        self.gad = None
        if ref.adaptor is not None:
            self.gtopo = Topology(topo.finest_cells, topo.levels, periodic=topo.periodic)
            self.gtopo.set_tile_set(sorted(topo.tile_set()))
            self.gad = GridAdaptor(self.gtopo, ref.solver.level_params,
                                   ref.adaptor.rescale_convention)
            for a, b in zip(self.gad._streak, ref.adaptor._streak):
                a.copy_(b)
            self.lad = GridAdaptor(sl.topology, ref.solver.level_params,
                                   ref.adaptor.rescale_convention)
            self.static_global = ref.static_tiles
        self.step_count = ref.step_count
        self.solver.k[:] = list(ref.solver.k)
        self.pair.bounce = ref.pair.bounce

    @property
    def coupling_active(self) -> bool:
        # every rank runs the hook when the global particle set is non-empty
        # (the exchanges inside it pair up across ranks)
        return getattr(self, "_global_active", len(self.particles) > 0)

    # -- particles ----------------------------------------------------------------
    def _make_particles(self, ref, idx):
        p = ref.particles
        n = int(idx.numel())
        out = Particles(n, p.d, p.dtype, p.device)
        gx = p._orig(p.xd)[:, idx]
        gx[0] -= self.sl.x0
        out.xd.copy_(gx)
        out.pd.copy_(p._orig(p.pd)[:, idx])
        out.pid.copy_(idx.to(torch.int32))
        return out

    def _local_x_range(self):
        return self.x_lo - self.sl.x0, self.x_hi - self.sl.x0

    # -- (i) per-level ghost columns ----------------------------------------------------
    def exchange_level(self, level, dst, rows=None):
        """(i) owned edge columns -> the neighbours' ghost columns (rows: a row
        slice of the SoA block, default the moments)."""
        sl = self.sl
        if self.world == 1:
            return
        rows = rows or slice(0, len(moment_names(sl.d)))
        a = dst_data(dst)
        r = sl.ranges[level]
        lo_l, hi_l = sl.cells(level, r["edge_l"])
        lo_r, hi_r = sl.cells(level, r["edge_r"])
        glo_l, ghi_l = sl.cells(level, r["ghost_l"])
        glo_r, ghi_r = sl.cells(level, r["ghost_r"])
        self.xch.columns(sl, a[rows, lo_l:hi_l], a[rows, lo_r:hi_r],
                         a[rows, glo_l:ghi_l] if sl.left is not None else None,
                         a[rows, glo_r:ghi_r] if sl.right is not None else None)

    # -- powder across the cut -------------------------------------------------------------
    def _ghost_rows_reduce(self, r0, r1):
        """(ii) for raster rows [r0, r1): ghost-node partial sums to the owners,
        completed edge rows back into the ghost region."""
        if self.world == 1:
            return
        sl, ras = self.sl, self.grid.ras
        rr = sl.ranges[0]
        lo_l, hi_l = sl.cells(0, rr["edge_l"])
        lo_r, hi_r = sl.cells(0, rr["edge_r"])
        glo_l, ghi_l = sl.cells(0, rr["ghost_l"])
        glo_r, ghi_r = sl.cells(0, rr["ghost_r"])
        gl = ras[r0:r1, glo_l:ghi_l] if sl.left is not None else None
        gr = ras[r0:r1, glo_r:ghi_r] if sl.right is not None else None
        el, er = ras[r0:r1, lo_l:hi_l], ras[r0:r1, lo_r:hi_r]
        self.xch.ghost_reduce(sl, gl, gr, el, er)
        self.xch.columns(sl, el, er, gl, gr)

    def _powder_stress_done(self):
        # the entrainment stress raster of surface cells near the cut needs the
        # neighbour's particles: sum the SIG rows like the P2G rows
        R = self.grid.R
        self._ghost_rows_reduce(R["sig"], R["etae"])

    def _powder_done(self):
        # the next backtrace and exchange read phi in the ghost columns
        _, w = self.solver.last_roles(0)
        phi = self.pair.trees[w].levels[0].index["phi"]
        self.exchange_level(0, self.pair.trees[w].levels[0], rows=slice(phi, phi + 1))

    # -- the coupling hook with (ii) ------------------------------------------------------
    def _exchange(self, solver):
        r, w = solver.roles(0)
        grid = self.grid
        grid.sync_topology()
        p = self.particles
        lib = L.lib()
        s = L.stream_handle()
        dcode = dtype_code(self.dtype)
        mat = self.material
        lv0 = grid.level0()
        grid.clear()
        n = len(p)
        ps = p.pd.stride(0)
        # particles sorted by (tile slot, cell) every sort_every steps (the
        # migration keeps the kept particles' order; arrivals append at the end),
        # so P2G runs the per-warp node-box modes like the single domain
        src_x, src_p, src_id, smem = p.xd, p.pd, None, 0
        if n and self.sort_particles:
            if self.step_count % self.sort_every == 0 or not p.permuted:
                self._sort_into_scratch()
                xa, pa, ida, _ = p.scratch()
                src_x, src_p, src_id = xa, pa, ida
                p.permuted = True
            smem = self.p2g_mode
        if n:
            L.check(lib.mlbm_p2g(L.C.byref(lv0), n, L.ptr(src_x), L.ptr(src_p), ps, mat.lam, mat.mu,
                                 mat.alpha, L.ptr(grid.ras), grid.ras.stride(0), dcode, smem,
                                 L.ptr(grid._err), s), "p2g")
        if self.world > 1:
            sl = self.sl
            nacc = grid.R["nacc"]
            rr = sl.ranges[0]
            lo_l, hi_l = sl.cells(0, rr["edge_l"])
            lo_r, hi_r = sl.cells(0, rr["edge_r"])
            glo_l, ghi_l = sl.cells(0, rr["ghost_l"])
            glo_r, ghi_r = sl.cells(0, rr["ghost_r"])
            ras = grid.ras
            gl = ras[:nacc, glo_l:ghi_l] if sl.left is not None else None
            gr = ras[:nacc, glo_r:ghi_r] if sl.right is not None else None
            el, er = ras[:nacc, lo_l:hi_l], ras[:nacc, lo_r:hi_r]
            self.xch.ghost_reduce(sl, gl, gr, el, er)            # (ii) sums to owners
            self.xch.columns(sl, el, er, gl, gr)                 # completed rows back
        sp = solver.params
        L.check(lib.mlbm_exchange(L.C.byref(lv0), L.fields(solver.arrays(w, 0).data),
                                  L.fields(solver.arrays(r, 0).data),
                                  L.fields(self.pair.trees[0].levels[0].data),
                                  L.fields(self.pair.trees[1].levels[0].data),
                                  L.ptr(grid.ras), grid.ras.stride(0), float(sp.eps_min),
                                  float(solver.level_params.nu(0)),
                                  float(self.drag_params.d_p or 1.0), float(self.drag_params.re_min),
                                  float(self.cadence), float(sp.rho0), _d3(sp.gravity, self.d),
                                  _d3(self.sediment_gravity, self.d), _faces(solver.boundaries),
                                  float(mat.floor_friction), 1, dcode, s), "exchange")
        if n:
            L.check(lib.mlbm_g2p(L.C.byref(lv0), n, L.ptr(src_x), L.ptr(p.xd), L.ptr(src_p),
                                 L.ptr(p.pd), L.ptr(src_id),
                                 L.ptr(p.pid) if src_id is not None else L.ptr(None), ps, mat.lam,
                                 mat.mu,
                                 mat.alpha, snow_arg(mat), L.ptr(grid.ras), grid.ras.stride(0),
                                 float(self.cadence), 1, dcode, L.ptr(self._counters),
                                 L.ptr(None), L.ptr(None), L.ptr(None),
                                 L.ptr(grid._err), s), "g2p")
        from .coupling import CouplingFields
        self.last_fields = CouplingFields(grid, self.pair.trees[0].levels[0])
        return FIELD_FORCE, FIELD_TAU

    # -- (iii) migration, (v) diagnostics ----------------------------------------------
    def _migrate(self):
        """(iii) particles whose x left the slab: a stable on-device partition
        (mlbm_migrate_count / mlbm_migrate_pack: warp ballots + block scan),
        one count exchange, one contiguous message per direction, arrivals
        appended after the kept particles (mlbm_migrate_unpack) in a second
        capacity-sized particle buffer set (no per-step reallocation)."""
        if self.world == 1:
            return
        p = self.particles
        sl = self.sl
        lib, s = L.lib(), L.stream_handle()
        n, d, R = len(p), p.d, p.pd.shape[0]
        dc = dtype_code(p.dtype)
        es = p.pd.element_size()
        lo, hi = self._local_x_range()
        gx = float(sl.global_cells[0])
        hl, hr = int(sl.left is not None), int(sl.right is not None)
        ws = self._mig_buf("ws", int(lib.mlbm_migrate_ws_bytes(max(n, 1))))
        cnt = self._mig_buf("cnt", 12)[:12].view(torch.int32)
        L.check(lib.mlbm_migrate_count(n, L.ptr(p.xd), float(lo), float(hi), hl, hr, L.ptr(cnt),
                                       L.ptr(ws), ws.numel(), s), "migrate_count")
        nk, nl, nr = (int(v) for v in cnt.cpu().tolist())
        ml, mr = self.xch.migrate_counts(sl, nl, nr)
        total = nk + ml + mr
        # the other buffer set of capacity >= total receives keep + arrivals
        cur = getattr(self, "_mig_set", 0)
        tgt = self._mig_set_bufs(1 - cur, total, d, R, p.dtype)
        cap = tgt[0].shape[1]
        msg = lambda m: m * (8 * d + es * R + 4)                   # noqa: E731
        send_l = self._mig_buf("sl", msg(nl))[:msg(nl)]
        send_r = self._mig_buf("sr", msg(nr))[:msg(nr)]
        recv_l = self._mig_buf("rl", msg(ml))[:msg(ml)]
        recv_r = self._mig_buf("rr", msg(mr))[:msg(mr)]

        def parts(buf, m):
            b = buf.data_ptr()
            return (L.C.c_void_p(b), L.C.c_void_p(b + 8 * d * m),
                    L.C.c_void_p(b + 8 * d * m + es * R * m))
        xl, pl, il = parts(send_l, nl)
        xr, pr, ir = parts(send_r, nr)
        L.check(lib.mlbm_migrate_pack(d, n, L.ptr(p.xd), L.ptr(p.pd), L.ptr(p.pid), p.pd.stride(0), R,
                                      dc, float(lo), float(hi), float(sl.x0), gx, hl, hr,
                                      L.ptr(tgt[0]), L.ptr(tgt[1]), L.ptr(tgt[2]), cap,
                                      xl, pl, il, nl, xr, pr, ir, nr, L.ptr(ws), ws.numel(), s),
                "migrate_pack")
        self.xch.migrate_payload(sl, send_l, send_r, recv_l, recv_r)
        at = nk
        for buf, m in ((recv_l, ml), (recv_r, mr)):
            if m:
                xi, pi, ii = parts(buf, m)
                L.check(lib.mlbm_migrate_unpack(d, m, xi, pi, ii, m, R, dc, float(sl.x0), gx,
                                                float(sl.topology.finest_cells[0]), L.ptr(tgt[0]),
                                                L.ptr(tgt[1]), L.ptr(tgt[2]), cap, at, s),
                        "migrate_unpack")
                at += m
        self._mig_set = 1 - cur
        np_ = Particles.wrap(tgt[0][:, :total], tgt[1][:, :total], tgt[2][:total], p.dtype)
        np_.stress_mat = p.stress_mat          # the tau rows travel with the particles
        np_.permuted = p.permuted
        np_._scratch = self._mig_scratch(1 - cur, total, d, R, p.dtype, cap)
        self.particles = np_

    def _mig_buf(self, key, nbytes):
        """Persistent byte buffers, grown geometrically."""
        bufs = self.__dict__.setdefault("_mig_bufs", {})
        b = bufs.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(int(nbytes * 1.25), 64), dtype=torch.uint8, device=self.pair.trees[0]
                            .levels[0].data.device)
            bufs[key] = b
        return b

    def _mig_scratch(self, which, n, d, R, dtype, cap):
        """Sort scratch of buffer set `which`: same row stride as the set."""
        scr = self.__dict__.setdefault("_mig_scr", [None, None])
        st = scr[which]
        lib = L.lib()
        slots = self.topology.lv[0].cap
        if st is None or st[0].shape[1] != cap or st[3].numel() < lib.mlbm_sort_ws_bytes(cap, slots):
            dev = self.pair.trees[0].levels[0].data.device
            st = (torch.empty((d, cap), dtype=torch.float64, device=dev),
                  torch.empty((R, cap), dtype=dtype, device=dev),
                  torch.empty(cap, dtype=torch.int32, device=dev),
                  torch.empty(int(lib.mlbm_sort_ws_bytes(cap, slots) * 1.25), dtype=torch.uint8,
                              device=dev))
            scr[which] = st
        return st[0][:, :n], st[1][:, :n], st[2][:n], st[3]

    def _mig_set_bufs(self, which, need, d, R, dtype):
        """Particle buffer set `which` (x, rows, ids) with capacity >= need."""
        sets = self.__dict__.setdefault("_mig_sets", [None, None])
        st = sets[which]
        if st is None or st[0].shape[1] < need:
            cap = max(int(need * 1.25) + 1024, 1024)
            dev = self.pair.trees[0].levels[0].data.device
            st = (torch.empty((d, cap), dtype=torch.float64, device=dev),
                  torch.empty((R, cap), dtype=dtype, device=dev),
                  torch.empty(cap, dtype=torch.int32, device=dev))
            sets[which] = st
        return st

    def _record_diagnostics(self):
        solver = self.solver
        d = self.d
        sl = self.sl
        lib = L.lib()
        s = L.stream_handle()
        dcode = dtype_code(self.dtype)
        out = self._diag_buf
        out.zero_()
        out[d + 1:d + 2].fill_(1.0)
        for l in range(self.topology.levels):
            a, b = sl.ranges[l]["owned"]
            if b <= a:
                continue
            lw = solver.last_roles(l)[1] if solver.k[l] else 0
            arr = solver.arrays(lw, l)
            st = L.Level.from_buffer_copy(solver._structs[l])
            st.counts = None
            st.first = a
            st.n_tiles = b
            L.check(lib.mlbm_diag_level(L.C.byref(st), L.fields(arr.data),
                                        float((1 << d) ** l), dcode, L.ptr(out[:d + 2]), s),
                    "diag_level")
        p = self.particles
        g = self.grid
        a, b = sl.cells(0, sl.ranges[0]["owned"])
        n0 = (b - a) if self.last_fields is not None else 0
        ras = g.ras[:, a:]
        L.check(lib.mlbm_diag_particles(d, len(p), L.ptr(p.pd), p.pd.stride(0), L.ptr(ras),
                                        g.ras.stride(0), n0, L.ptr(None), dcode,
                                        L.ptr(out[d + 2:]), s), "diag_particles")
        if self.world > 1:
            emin = out[d + 1:d + 2].clone()
            out[d + 1] = 0.0
            self.xch.allreduce(sl, out, "sum")
            self.xch.allreduce(sl, emin, "min")
            out[d + 1:d + 2].copy_(emin)

    def _step_eager(self, ci, is_mpm, adapt_now):
        """coupling.py:448-481 on the slab: cycle (with (i)/(ii) inside),
        migration (iii), global block maintenance (iv), reduced diagnostics (v)."""
        solver = self.solver
        if self.particles is not None:
            self.particles.ensure_stress(self.material)
        cycle = solver._schedule[ci]
        if is_mpm:
            solver.run_cycle(cycle, hook=self._exchange)
        elif self.coupling_active:
            solver.run_cycle(cycle, hook=self._held)
        else:
            solver.run_cycle(cycle)
        if self.coupling_active and is_mpm:
            self.grid.raise_pending()
        if self.powder is not None:
            self._powder_cycle(is_mpm)
        self._migrate()
        if self.gad is not None and self.coupling_active and self.step_count % self.cadence == 0:
            self._adapt()
        self._record_diagnostics()
        self._push_diag_row(self._diag_buf.cpu().numpy())

    # -- (iv) block maintenance -----------------------------------------------------
    def _adapt(self):
        gad, gtopo, sl = self.gad, self.gtopo, self.sl
        lib = L.lib()
        s = L.stream_handle()
        d = self.d
        p = self.particles
        seeds = gad._seeds
        L.zero(seeds)
        if len(p):
            gx = p.xd.clone()
            gx[0] = torch.remainder(gx[0] + sl.x0, sl.global_cells[0])
            t0 = (L.C.c_int32 * 3)(*gtopo.tile_grid(0))
            L.check(lib.mlbm_seed_tiles(d, len(p), L.ptr(gx), gx.stride(0), 1, t0,
                                        L.ptr(seeds), L.ptr(gad._err), s), "seed_tiles")
        if self.world > 1:
            self.xch.allreduce(sl, seeds, "max")          # (iv) uint8 OR of the seed tiles
        gad._seeds_dirty = False
        # the fused pass with no particles: seeds are preset, cleared at its end
        gad.plan_device(RefineDriver(static_tiles=self.static_global, levels=gtopo.levels))
        status = gad._status.cpu().numpy()
        Lv = gtopo.levels
        changed = [l for l in range(Lv) if status[l]]
        if not changed:
            return
        self.topology_changes += 1
        # global kinds (no fields on the global topology)
        gtopo.rebuild({l: gad._new[l].clone() for l in changed})
        # crop to the local box (ghosts wrap periodically) and rebuild locally
        lt = sl.topology
        lchanged, counts, fresh = [], [0] * Lv, [0] * Lv
        for l in range(Lv):
            g = gtopo.tile_grid(l)
            tw = TILE << l
            cols = (torch.arange(lt.tile_grid(l)[0], device=lt.device) + sl.x0 // tw) % g[0]
            new = gtopo.lv[l].kind.view(g)[cols].reshape(-1)
            old = lt.lv[l].kind
            self.lad._new[l].copy_(new)
            if not torch.equal(new, old):
                lchanged.append(l)
            nz = new != 0
            counts[l] = int(nz.sum().item())
            fresh[l] = int((nz & (old == 0)).sum().item())
        if lchanged:
            self.lad._prepare(lchanged, self.pair, counts, [1] * Lv)()
            self.solver._refresh_tables()
            self.grid.sync_topology()
            sl.compute_ranges()
        # fresh ghost tiles hold locally initialised values: refresh both trees'
        # ghost columns from the owners (every rank: the global change is common)
        for l in range(Lv):
            for t in range(2):
                self.exchange_level(l, self.pair.trees[t].levels[l])

    # -- gather for tests ---------------------------------------------------------------
    def owned_particles(self):
        """(pid, global x, v) of the owned particles."""
        p = self.particles
        x = p.xd.t().clone()
        x[:, 0] += self.sl.x0
        x[:, 0] = torch.remainder(x[:, 0], self.sl.global_cells[0])
        v = p.pd[p.R["v"]:p.R["v"] + p.d].t()
        return p.pid.cpu().numpy(), x.cpu().numpy(), v.double().cpu().numpy()
