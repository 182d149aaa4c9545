"""GPU block maintenance (drop-in for ``pkg/src/mlbm/adapt.py``).

``GridAdaptor.update(driver, pair)`` runs the reference's bitmap algorithm
(adapt.py:54-230) as dense uint8 tile-grid kernels on the device:

  seeds (particle tiles + static mask)          mlbm_seed_tiles       adapt.py:54-65
  desired cumulative coverage                   mlbm_bitmap_op/dilate adapt.py:77-105
  current cumulative coverage                   mlbm_bitmap_op        adapt.py:108-121
  hysteresis (int16 streaks, sibling groups,
    2-ring guard)                               mlbm_effective_level  adapt.py:152-182
  leaf/border plan + no-op test                 mlbm_plan_level       adapt.py:184-225
  rebuild (sorted slots) + bitwise migration    mlbm_compact_tiles,
                                                mlbm_migrate_level    adapt.py:232-286
  new-cell initialisation + S rescale chain     mlbm_init_new_cells   adapt.py:288-372
  invariants                                    mlbm_check_*          adapt.py:374-389

One small device->host copy per update returns the changed flags and
violation counts; a topology change adds the two copies of the rebuild.
The tile sets, streaks and surviving-tile bits are identical to the
reference's by construction (integer work only).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .sparse_grid import (DEV_BORDER, DEV_LEAF, TILE, LevelFields, PingPongPair, Topology,
                          dtype_code, fresh_block)
from .solver import LevelParams

PAD_TILES = 2


@dataclass
class RefineDriver:
    """Inputs of the level-selection function (adapt.py:42-65).

    ``positions``: (n, d) array / tensor in finest units, or a float64
    device tensor laid out [d, n] (``positions_soa``) as the particle state
    keeps it.
    """
    positions: object = None
    static_tiles: np.ndarray | None = None
    levels: int = 1
    positions_soa: object = None
    # the seed tiles of this update were written by mlbm_g2p of the same step
    # (CoupledSim with a fused adaptor): the fused pass reads no positions
    g2p_seeds: bool = False

    def device_positions(self, d, device):
        if self.positions_soa is not None:
            return self.positions_soa
        if self.positions is None:
            return None
        x = torch.as_tensor(self.positions, dtype=torch.float64, device=device)
        if x.numel() == 0:
            return None
        return x.reshape(-1, d).t().contiguous()

    def seed_tiles(self, tiles_dims):
        """Host reference of the seeds (test helper, adapt.py:54-65)."""
        seeds = np.zeros(tiles_dims, dtype=bool)
        if self.positions is not None and len(self.positions):
            pos = np.asarray(self.positions.cpu() if torch.is_tensor(self.positions)
                             else self.positions)
            t = np.floor(pos).astype(np.int64) // TILE
            if (t < 0).any() or any((t[:, a] >= tiles_dims[a]).any()
                                    for a in range(len(tiles_dims))):
                raise ValueError("particle outside the domain bounding box")
            seeds[tuple(t.T)] = True
        if self.static_tiles is not None:
            seeds |= self.static_tiles
        return seeds


@dataclass
class AdaptReport:
    created: list = field(default_factory=list)
    deleted: list = field(default_factory=list)
    noop: bool = True
    violations: list = field(default_factory=list)

    def total_created(self):
        return int(sum(self.created)) if self.created else 0

    def total_deleted(self):
        return int(sum(self.deleted)) if self.deleted else 0


def _i3(v):
    return (L.C.c_int32 * 3)(*v)


class GridAdaptor:
    """Incremental topology maintenance with coarsening hysteresis."""

    def __init__(self, topology: Topology, level_params: LevelParams,
                 rescale_convention: str = "derived"):
        self.topology = topology
        self.level_params = level_params
        self.rescale_convention = rescale_convention
        dev = topology.device
        self._grids = [topology.tile_grid(l) for l in range(topology.levels)]
        n = [int(np.prod(g)) for g in self._grids]
        z = lambda k: torch.zeros(k, dtype=torch.uint8, device=dev)   # noqa: E731
        self._streak = [torch.zeros(k, dtype=torch.int16, device=dev) for k in n]
        self._des = [z(k) for k in n]
        self._cur = [z(k) for k in n]
        self._eff = [z(k) for k in n]
        self._par = [z(k) for k in n]
        self._guard = [z(k) for k in n]
        self._own = [z(k) for k in n]
        self._stor = [z(k) for k in n]
        self._tmp = [z(k) for k in n]
        self._new = [z(k) for k in n]
        # incremental classification after a rebuild: changed-tile lists and
        # the dirty maps the classification reads
        self._chg_list = [torch.zeros(k, dtype=torch.int32, device=dev) for k in n]
        self._chg_n = torch.zeros(len(n), dtype=torch.int32, device=dev)
        self._dirty = [z(k) for k in n]
        self._seeds = z(n[0])
        # [changed L][violations 3][pad][new tile counts L][fresh tile counts L]
        self._status = torch.zeros(3 * topology.levels + 4, dtype=torch.int32, device=dev)
        self._err = torch.zeros(L.ERR_INTS, dtype=torch.int32, device=dev)
        self._taus = torch.tensor(level_params.taus, dtype=torch.float64, device=dev)
        self._static_key = None
        self._static_dev = None
        self._bar = torch.zeros(2, dtype=torch.int32, device=dev)
        self.fused = True          # one cooperative launch per pass (csrc/adapt.cu)
        # seeds written by G2P (CoupledSim): the next fused pass reads no positions
        # and takes G2P's count of particles outside level-0 leaves from here
        self.ext_count = torch.zeros(1, dtype=torch.int32, device=dev)
        self.launches = 0
        # tile windows of the G2P-seeded fused pass ([2][levels][6] int32, see
        # mlbm_adapt_pass): valid for the key (host rebuilds, static mask) they
        # were derived under; any other pass invalidates them
        self.windows = os.environ.get("MLBM_ADAPT_WINDOWS", "1") != "0"
        # latest-only levels: migrate into the other tree and swap the roles
        # (one pass over the level) instead of scratch + copy back (two)
        self.latest_swap = os.environ.get("MLBM_LATEST_SWAP", "1") != "0"
        self._win = torch.zeros(2 * topology.levels * 6, dtype=torch.int32, device=dev)
        self._win_key = None

    @property
    def streak(self):
        """Host copy of the int16 streak bitmaps (adapt.py:147-148)."""
        d = self.topology.d
        out = []
        for l, g in enumerate(self._grids):
            a = self._streak[l].cpu().numpy().reshape(g)
            out.append(a if d == 3 else a[..., 0])
        return out

    # -- bitmap helpers ------------------------------------------------------------
    def _op(self, op, level, src, dst):
        L.check(L.lib().mlbm_bitmap_op(op, self.topology.d, _i3(self._grids[level]),
                                       L.ptr(src), L.ptr(dst), L.stream_handle()), "bitmap_op")
        self.launches += 1

    def _parents_into(self, level_child, src, dst):
        self._op(1, level_child, src, dst)

    def _dilate(self, level, src, dst):
        topo = self.topology
        L.check(L.lib().mlbm_dilate(topo.d, _i3(self._grids[level]), _i3(topo.periodic3()),
                                    PAD_TILES, L.ptr(src), L.ptr(dst), L.ptr(self._tmp[level]),
                                    L.stream_handle()), "dilate")
        self.launches += 1

    def _static(self, static):
        if static is None:
            return None
        key = (id(static), static.shape)
        if self._static_key != key:
            a = np.asarray(static, dtype=np.uint8)
            if a.ndim == 2:
                a = a[..., None]
            self._static_dev = torch.as_tensor(a.reshape(-1), device=self.topology.device)
            self._static_key = key
        return self._static_dev

    # -- update ----------------------------------------------------------------------
    def update(self, driver: RefineDriver, pair: PingPongPair) -> AdaptReport:
        """One adaptation pass (adapt.py:198-230)."""
        self.plan_device(driver)
        status = self._status.cpu().numpy()
        err = self._err.cpu().numpy()
        return self.finish(driver, pair, status, err)

    def status_tensors(self):
        """Device tensors whose host copies ``finish`` consumes."""
        return self._status, self._err

    def plan_device(self, driver: RefineDriver):
        """Every kernel of the pass that does not depend on its outcome: seeds,
        desired / current / effective coverage, plan and no-op flags
        (status[0:L]) and the invariants of the current topology
        (status[L:L+3]).  No host synchronisation (CUDA-graph capturable)."""
        if self.fused:
            return self._plan_fused(driver)
        self._win_key = None                        # the per-op pass writes whole grids
        if driver.g2p_seeds:
            L.zero(self.ext_count)     # the per-op pass seeds from the positions itself
        self._seeds_dirty = True
        topo = self.topology
        lib = L.lib()
        s = L.stream_handle()
        Lv = topo.levels
        self._status.zero_()
        seeds = self._seeds
        seeds.zero_()
        x = driver.device_positions(topo.d, topo.device)
        if x is not None and x.shape[1]:
            L.check(lib.mlbm_seed_tiles(topo.d, x.shape[1], L.ptr(x), x.stride(0), 1,
                                        _i3(self._grids[0]), L.ptr(seeds), L.ptr(self._err), s),
                    "seed_tiles")
        st = self._static(driver.static_tiles)
        if st is not None:
            self._op(2, 0, st, seeds)
        des, cur, eff = self._des, self._cur, self._eff
        if Lv == 1:
            des[0].fill_(1)
        else:
            self._op(0, 0, seeds, des[0])
            for l in range(1, Lv):
                self._parents_into(l - 1, des[l - 1], self._par[l])
                if l == Lv - 1:
                    des[l].fill_(1)
                else:
                    self._dilate(l, self._par[l], self._guard[l])
                    self._op(0, l, self._guard[l], des[l])
        for l in range(Lv):
            self._op(6, l, topo.lv[l].kind, cur[l])
            if l > 0:
                self._parents_into(l - 1, cur[l - 1], self._par[l])
                self._op(2, l, self._par[l], cur[l])
        for l in range(Lv):
            guard = par = None
            if l > 0:
                self._parents_into(l - 1, eff[l - 1], self._par[l])
                self._dilate(l, self._par[l], self._guard[l])
                guard, par = self._guard[l], self._par[l]
            L.check(lib.mlbm_effective_level(topo.d, _i3(self._grids[l]), L.ptr(des[l]),
                                             L.ptr(cur[l]), L.ptr(guard), L.ptr(par),
                                             L.ptr(self._streak[l]), L.ptr(eff[l]), s),
                    "effective_level")
            self.launches += 1
        if Lv > 1:
            eff[Lv - 1].fill_(1)
        for l in range(Lv):
            self._op(4, l, eff[l], self._own[l])
            if l > 0:
                self._parents_into(l - 1, eff[l - 1], self._par[l])
                self._op(3, l, self._par[l], self._own[l])
            self._dilate(l, self._own[l], self._stor[l])
            L.check(lib.mlbm_plan_level(self._own[l].numel(), L.ptr(self._own[l]),
                                        L.ptr(self._stor[l]), L.ptr(topo.lv[l].kind),
                                        L.ptr(self._new[l]), L.ptr(self._status[l:l + 1]), s),
                    "plan_level")
            self.launches += 1
            nz = self._new[l] != 0
            self._status[Lv + 4 + l] = nz.sum().to(torch.int32)
            self._status[2 * Lv + 4 + l] = (nz & (topo.lv[l].kind == 0)).sum().to(torch.int32)
        self._invariants_device(driver)

    def prepare_windows(self, static_tiles):
        """(Re)derive the pass windows from the current kinds when the topology
        was set from the host or the static mask changed (syncs; call outside
        graph capture).  Returns whether windows are in use."""
        if not self.windows:
            return False
        topo = self.topology
        self._static(static_tiles)
        key = (getattr(topo, "host_rebuilds", 0), self._static_key if static_tiles is not None else None)
        if self._win_key == key:
            return True
        Lv = topo.levels
        w = np.zeros((2, Lv, 6), dtype=np.int32)
        w[:, :, :3] = np.iinfo(np.int32).max
        w[:, :, 3:] = -np.iinfo(np.int32).max
        for l in range(Lv - 1):
            g = self._grids[l]
            nz = torch.nonzero(topo.lv[l].kind.view(*g))
            boxes = []
            if nz.shape[0]:
                boxes.append((nz.min(0).values.cpu().numpy(), nz.max(0).values.cpu().numpy()))
            if l == 0 and static_tiles is not None:
                st = np.nonzero(np.asarray(static_tiles).reshape(g))
                if st[0].size:
                    boxes.append((np.array([a.min() for a in st]), np.array([a.max() for a in st])))
            for lo, hi in boxes:
                w[1, l, :3] = np.minimum(w[1, l, :3], lo)
                w[1, l, 3:] = np.maximum(w[1, l, 3:], hi)
        self._win.copy_(torch.as_tensor(w.reshape(-1)))
        self._win_key = key
        return True

    def _plan_fused(self, driver):
        topo = self.topology
        if getattr(self, "_seeds_dirty", False):     # left set by the unfused path
            L.zero(self._seeds)
            self._seeds_dirty = False
        Lv = topo.levels
        arr = lambda ts: (L.C.c_void_p * Lv)(*[t.data_ptr() for t in ts])   # noqa: E731
        ext = self.ext_count if driver.g2p_seeds else None
        x = None if driver.g2p_seeds else driver.device_positions(topo.d, topo.device)
        st = self._static(driver.static_tiles)
        win = None
        if ext is not None and self.windows:
            if torch.cuda.is_current_stream_capturing():
                if self._win_key is not None:
                    win = self._win                 # prepared before the capture
            elif self.prepare_windows(driver.static_tiles):
                win = self._win
        if win is None:
            self._win_key = None                    # a full-grid pass: re-derive next time
        h = topo.hier_struct()
        L.zero(self._status)
        L.check(L.lib().mlbm_adapt_pass(L.C.byref(h), arr(self._des), arr(self._cur),
                                        arr(self._eff), arr(self._par), arr(self._own),
                                        arr(self._new), arr(self._stor), arr(self._streak),
                                        L.ptr(self._seeds),
                                        L.ptr(st), L.ptr(x), x.stride(0) if x is not None else 0,
                                        x.shape[1] if x is not None else 0,
                                        L.ptr(ext), L.ptr(win),
                                        L.ptr(self._status),
                                        L.ptr(self._err), L.ptr(self._bar), L.stream_handle()),
                "adapt_pass")
        self.launches += 1

    def finish(self, driver, pair, status, err, check_after=True, device_runner=None,
               latest_only=None):
        """Host half: raise on seed errors; when a level changed, rebuild and
        migrate on the device without host synchronisation (the new counts
        come from the adapt pass); build the report.  ``check_after`` re-runs
        the invariants on the new topology (one readback); the graph path
        skips it and the next pass reports them.  ``latest_only`` {level: tree}
        migrates / initialises only that tree of a level whose other tree is
        fully rewritten before it is read again (the coupled step's level 0).
        ``device_runner(fn, key)``
        (graph path) runs the device half ``fn`` — eagerly or as a replay of a
        graph cached under ``key`` — after the host bookkeeping is done."""
        topo = self.topology
        Lv = topo.levels
        rep = AdaptReport(created=[0] * Lv, deleted=[0] * Lv)
        if err[0]:
            self._err.zero_()
            raise ValueError("particle outside the domain bounding box")
        changed = [l for l in range(Lv) if status[l]]
        viol = status[Lv:Lv + 3]
        if changed:
            rep.noop = False
            new_counts = [int(v) for v in status[Lv + 4:2 * Lv + 4]]
            fresh = [int(v) for v in status[2 * Lv + 4:3 * Lv + 4]]
            for l in changed:
                rep.created[l] = fresh[l]
                rep.deleted[l] = topo.n_tiles(l) - (new_counts[l] - fresh[l])
            if device_runner is None:
                lo = {l: t for l, t in (latest_only or {}).items() if l in changed}
                self._prepare(changed, pair, new_counts, fresh, lo)()
            else:
                # graph path: the init kernel always runs (it finds no fresh tile
                # when there is none), so the rebuild graph's key is only the set
                # of changed levels
                lo = {l: t for l, t in (latest_only or {}).items() if l in changed}
                dev = self._prepare(changed, pair, new_counts, [1] * Lv, lo)
                device_runner(dev, (tuple(changed), tuple(sorted(lo.items()))))
            if check_after:
                self._invariants_device(driver)
                viol = self._status[Lv:Lv + 3].cpu().numpy()
            else:
                viol = (0, 0, 0)
        self._report_invariants(viol, rep)
        return rep

    def _prepare(self, changed, pair, new_counts, fresh, latest_only=None):
        """Rebuild + bitwise migration + new-cell init (adapt.py:232-372).
        Host part here (capacity growth, host counts, version bump); returns
        the device part — compaction into the spare tile map, neighbours,
        migration into the scratch blocks, initialisation from the old
        hierarchy, then scratch / maps / kinds become current — which launches
        only kernels and device copies on fixed pointers (graph-capturable)."""
        topo = self.topology
        grown = False
        for l in changed:
            grown |= topo.ensure_capacity(l, new_counts[l])
        if grown:
            pair.ensure_capacity()
        for l in changed:
            if not (self.latest_swap and l in (latest_only or {})):
                pair.scratch_blocks(l)
        old_h = topo.hier_struct(pair)           # old maps, old fields, old counts
        # latest-only levels migrate their latest tree t straight into the
        # other tree's storage (no scratch, no copy back; the caller swaps the
        # level's tree roles): the old hierarchy shows tree t in both places,
        # so a finer-level fallback of another level's init reads the latest
        # old-layout values, never the tree being rewritten
        swap = {l: t for l, t in (latest_only or {}).items() if self.latest_swap}
        for l, t in swap.items():
            old_h.fields[1 - t][l] = old_h.fields[t][l]
        topo.commit_host({l: new_counts[l] for l in changed})
        new_h = topo.hier_struct()
        d = topo.d
        dcode = dtype_code(pair.dtype)
        conv = 0 if self.rescale_convention == "derived" else 1
        init = {l: bool(fresh[l]) for l in changed}
        latest_only = latest_only or {}
        Lv = topo.levels
        # the classification that follows is incremental: it reads these dirty
        # maps (tiles within one tile of a kind change at any level)
        topo._dirty = {l: self._dirty[l] for l in range(Lv)}
        topo._dirty_changed = set(changed)

        def dirty_maps():
            # sparse: the changed tiles of each changed level (compacted), then
            # their one-tile neighbourhoods marked at every level
            for l in range(Lv):
                L.zero(self._dirty[l])
            h = topo.hier_struct()
            arr = (L.C.c_void_p * Lv)(*[t.data_ptr() for t in self._dirty])
            for l in changed:
                n = self._new[l].numel()
                ws = topo.workspace(n)
                L.check(L.lib().mlbm_changed_tiles(n, L.ptr(topo.lv[l].kind), L.ptr(self._new[l]),
                                                   L.ptr(self._chg_list[l]), L.ptr(self._chg_n[l:l + 1]),
                                                   L.ptr(ws), ws.numel(), L.stream_handle()),
                        "changed_tiles")
                L.check(L.lib().mlbm_mark_dirty(L.C.byref(h), l, L.ptr(self._chg_list[l]),
                                                L.ptr(self._chg_n[l:l + 1]), arr, L.stream_handle()),
                        "mark_dirty")

        def device():
            lib = L.lib()
            s = L.stream_handle()
            dirty_maps()
            for l in changed:
                topo.compact(l, self._new[l])
            for l in changed:
                topo.build_neighbors(l, new_map=True)
            for l in changed:
                lt = topo.lv[l]
                cnt = L.ptr(topo.dcounts[l])
                # trees to carry over: both, or only the one read next (the
                # other is rewritten before it is read; its stale cells stay)
                ts = (latest_only[l],) if l in latest_only else (0, 1)
                old = [L.fields(pair.trees[t].levels[l].data) for t in ts] + [L.fields(None)]
                if l in swap:
                    new = [L.fields(pair.trees[1 - swap[l]].levels[l].data), L.fields(None)]
                else:
                    sb = pair.scratch_blocks(l)
                    new = [L.fields(sb[t]) for t in ts] + [L.fields(None)]
                L.check(lib.mlbm_migrate_level(d, lt.cap, cnt, L.ptr(lt.old_slot), old[0], old[1],
                                               new[0], new[1], dcode, s), "migrate_level")
                if init[l]:
                    L.check(lib.mlbm_init_new_cells(L.C.byref(old_h), L.C.byref(new_h), l,
                                                    L.ptr(lt.tile_xyz), L.ptr(lt.old_slot),
                                                    lt.cap, cnt, new[0], new[1],
                                                    L.ptr(self._taus), conv,
                                                    dcode, L.ptr(self._status[Lv_slot(topo)]),
                                                    s), "init_new_cells")
                if l in swap:
                    continue
                L.check(lib.mlbm_copy_live_fields(d, lt.cap, cnt, new[0], new[1],
                                                  *[L.fields(pair.trees[t].levels[l].data)
                                                    for t in ts], *([L.fields(None)] if len(ts) == 1
                                                                    else []), dcode, s),
                        "copy_live_fields")
            topo.commit_device({l: self._new[l] for l in changed})
        return device

    def _invariants_device(self, driver):
        """Coverage, two-tile rings, particles in level-0 leaves
        (adapt.py:374-389) -> status[L:L+3]; reported, not raised."""
        topo = self.topology
        lib = L.lib()
        s = L.stream_handle()
        v = self._status[topo.levels:topo.levels + 3]
        v.zero_()
        h = topo.hier_struct()
        L.check(lib.mlbm_check_coverage(L.C.byref(h), L.ptr(v), s), "check_coverage")
        for l in range(topo.levels):
            self._op(6, l, topo.lv[l].kind, self._own[l])
            self._dilate(l, self._own[l], self._stor[l])
            L.check(lib.mlbm_count_ring_violations(self._stor[l].numel(), L.ptr(self._stor[l]),
                                                   L.ptr(topo.lv[l].kind), L.ptr(v), s),
                    "ring_violations")
        x = driver.device_positions(topo.d, topo.device)
        if x is not None and x.shape[1]:
            L.check(lib.mlbm_check_particles(topo.d, x.shape[1], L.ptr(x), x.stride(0), 1,
                                             _i3(self._grids[0]), L.ptr(topo.lv[0].kind),
                                             L.ptr(v), s), "check_particles")

    @staticmethod
    def _report_invariants(cnt, rep):
        if cnt[0]:
            rep.violations.append(("invariant", f"leaf coverage violated at {cnt[0]} tiles"))
        if cnt[1]:
            rep.violations.append(("invariant", f"{cnt[1]} ring tiles missing"))
        if cnt[2]:
            rep.violations.append(("particle not in level-0 leaf", int(cnt[2])))


def Lv_slot(topo):
    """status word receiving uninitialised-cell counts (the pad slot)"""
    return topo.levels + 3


def update_grid(adaptor: GridAdaptor, driver: RefineDriver, pair) -> AdaptReport:
    return adaptor.update(driver, pair)
