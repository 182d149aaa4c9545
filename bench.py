#!/usr/bin/env python
"""Benchmark of the coupled adaptive HOME-LBM <-> MPM step on B200.

Workload (default, BASELINE.json configs[3]): four-level
1536x768x384-effective avalanche with powder cloud over a terrain heightmap,
55,836,672 MPM particles, two-way coupling, powder entrainment, block
maintenance every step, fp32 device state (shifted density), on ONE B200
(--scene c2 / c3 / c5 / c1 select the other configs).  One bench "step" = one finest coupled
cycle ``CoupledSim.step()`` (coupling.py:448-481): coarser-level prelude,
level-0 stream, exchange + MPM, level-0 collide, adapt, diagnostics.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the CPU oracle
port of the same path instead (the reference is pure NumPy and 2D-only, see
DESIGN.md §1).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = ("effective MLUPS and MPM particles/s per coupled step at 1/2/4/8 B200; "
          "HBM GB/s vs peak")
UNIT = "effective MLUPS"
REF_TIMED_STEPS_CAP = 5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    # C4 (configs[3], the north-star avalanche) fits one B200: it is the
    # headline workload; c2 / c3 / c5 / c1 remain selectable
    ap.add_argument("--scene", default="c4", choices=["c2", "c3", "c4", "c5", "c1"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--slabs", action="store_true",
                    help="coupled slab decomposition (slab_coupled.py) even at N = 1 "
                         "(N > 1 always runs it unless --replicas)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: N independent full-scene replicas instead of slabs")
    return ap.parse_args()


_C4_DIR = None


def scene_dict(name, scale=1):
    import scenes as S
    if name == "c4":
        import tempfile
        global _C4_DIR
        _C4_DIR = _C4_DIR or tempfile.mkdtemp(prefix="mlbm_c4_")
        return S.avalanche_c4(os.path.join(_C4_DIR, f"terrain_s{scale}.npy"), scale=scale)
    return {"c2": S.COLUMN_3D_C2, "c3": S.SANDSTORM_3D_C3, "c5": S.CLOUD_3D_C5,
            "c1": S.TAYLOR_GREEN_3D_C1}[name]


def workload_name(name):
    return {"c2": "C2: two-level 128^3-effective 3D granular column collapse in air, 262,144 "
                  "MPM sand particles, two-way coupled, adapt every step",
            "c3": "C3: three-level 512x256x128-effective dune under log-law wind inflow, "
                  "4,194,304 MPM sand particles, two-way coupled, adapt every step",
            "c4": "C4: four-level 1536x768x384-effective snow avalanche with powder cloud over a "
                  "terrain heightmap, 55,836,672 MPM particles (NACC snow), two-way coupled, "
                  "powder entrainment, adapt every step, on ONE B200",
            "c5": "C5: dynamic-refinement stress, periodic 256^3, L = 3, 2,097,152 particles in a "
                  "dispersed cloud with Gaussian velocities (sigma 0.1), blocks activated / "
                  "retired every step",
            "c1": "C1: single-level 64^3 periodic Taylor-Green (D3Q27)"}[name]


# -- clocks -------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 6 and p[0].isdigit():
                    rows.append(p)
        os.unlink(self.f.name)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        sm = [int(r[0]) for r in rows]
        return {"sm_mhz": int(statistics.median(sm)), "sm_max_mhz": int(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


TRAFFIC_FILES = {"c2": "r2e_dram_traffic_c2.json", "c4": "r2e_dram_traffic_c4.json"}


def dram_traffic(scene):
    """Per-launch DRAM bytes of the top kernels from the committed ncu full-set
    capture of the same workload (profiles/r1_dram_traffic*.json,
    tools/full_summary.py); {} when no capture of this scene is committed."""
    fn = TRAFFIC_FILES.get(scene)
    if fn is None:
        return {}
    try:
        with open(os.path.join(ROOT, "profiles", fn)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# -- algorithmic bytes per kernel class ---------------------------------
def kernel_class(rec, d, s, live):
    """(class, algorithmic bytes, units) of one traced C-ABI call.  Kernels are
    launched over tile capacities; ``live(lv_struct)`` / ``live(ptr)`` give the
    live tile count of a level / the device count a pointer refers to."""
    name, _, _, _ = rec[:4]
    args = rec[4]
    NM = 1 + d + d * (d + 1) // 2
    T = 4 ** d
    if name == "mlbm_level_step":
        lv, mode = args[0]._obj, int(args[4])
        cells = live(lv) * T
        if mode == 0:
            return "level_step[fused]", cells * 2 * NM * s, cells
        if mode == 1:
            # the coupled level-0 stream also carries eps and phi to the write tree
            return "level_step[stream]", cells * (2 * NM + 4) * s, cells
        return "level_step[collide+bc]", cells * (2 * NM + d + 1) * s, cells
    if name == "mlbm_p2g":
        n = int(args[1])
        return "p2g", n * (8 * d + (2 * d + 2 * d * d + 2) * s), n
    if name == "mlbm_g2p":
        n = int(args[1])
        return "g2p", n * (16 * d + (d * d + 1) * s + (d + 2 * d * d + 1) * s), n
    if name == "mlbm_exchange":
        cells = live(args[0]._obj) * T
        return "exchange", cells * (17 + 25) * s, cells
    if name in ("mlbm_downward", "mlbm_upward"):
        # unique bytes: upward reads its 2^d fine sources (disjoint between
        # targets); downward targets share their 2^d coarse sources with their
        # neighbours (the gathers hit L2): about one coarse cell (old and new
        # trees) per fine target
        n = live(args[2])
        nc = 1 << d
        reads = nc if name == "mlbm_upward" else 2
        return "transfer", n * (reads + 1) * (NM + 2) * s, n
    if name.startswith("mlbm_diag"):
        return "diagnostics", 0, 0
    if name.startswith("mlbm_stress_raster") or name == "mlbm_powder":
        return "powder", 0, 0
    if name == "mlbm_adapt_pass":
        return "adapt_pass", 0, 0
    if name.startswith("mlbm_check_") or name in ("mlbm_count_ring_violations", "mlbm_bitmap_op",
                                                   "mlbm_dilate"):
        # re-checked after a rebuild only on the eager path (the graph path
        # leaves them to the next adapt pass): not part of the timed steps
        return "invariants (eager profile only)", 0, 0
    if name in ("mlbm_compact_tiles", "mlbm_build_neighbors", "mlbm_migrate_level",
                "mlbm_copy_live_fields", "mlbm_init_new_cells", "mlbm_classify_level",
                "mlbm_build_interface"):
        return "rebuild (topology changes)", 0, 0
    if name == "mlbm_particle_sort":
        n = int(args[1])
        return "particle_sort", n * 2 * (8 * d + (d + 2 * d * d + 3) * s + 4), n
    return "adapt/topology", 0, 0


def run_mine(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2603_14982_b200 import _lib as L
    from paper_2603_14982_b200.harness import build_scene, validate_scene

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = validate_scene(scene_dict(args.scene))
    sim = build_scene(cfg)
    if args.scene == "c5":
        import scenes as S
        S.cloud_velocities(sim)
    d = cfg.dim
    eff_cells = int(np.prod(cfg.cells))
    n_part = len(sim.particles)
    s = 4 if cfg.dtype == torch.float32 else 8

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        sim.step()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    # ---- timed region: device time per step (CUDA events), L2 flushed between steps
    # the scene / graph objects built so far are long-lived: frozen out of the
    # cyclic collector's scans (a full collection over them stalls the host
    # between graph launches for tens of ms; collection itself stays on)
    gc.collect()
    gc.freeze()
    clocks = Clocks(local_rank)
    launches0 = L.TRACE.launches
    caps0, chg0 = sim.graph_captures, sim.topology_changes
    cnt0 = {k: getattr(sim, k, 0) for k in ("step_graph_captures", "rebuild_graph_captures", "rebuild_eager")}
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    # MLBM_PROFILE_TIMED=1: the profiler range covers the timed steps only
    # (ncu --profile-from-start off: a launch list without the scene build)
    prof_timed = os.environ.get("MLBM_PROFILE_TIMED") == "1"
    if prof_timed:
        torch.cuda.cudart().cudaProfilerStart()
    ev = []
    for _ in range(args.steps):
        L.zero(flush)                      # L2 flush: a memset, not a kernel
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        sim.step()
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    if prof_timed:
        torch.cuda.cudart().cudaProfilerStop()
    barrier()
    clk = clocks.stop()
    launches = L.TRACE.launches - launches0
    graph_info = {"graph_replays_per_step": 1, "graph_captures": sim.graph_captures - caps0,
                  "topology_changes": sim.topology_changes - chg0}
    graph_info.update({k: getattr(sim, k, 0) - v for k, v in cnt0.items()})
    step_ms = [a.elapsed_time(b) for a, b in ev]
    if os.environ.get("MLBM_STEP_TIMES") == "1":
        graph_info["step_ms_all"] = [round(x, 2) for x in step_ms]
    graph_info["step_ms"] = {"min": round(min(step_ms), 3), "median": round(statistics.median(step_ms), 3),
                             "max": round(max(step_ms), 3)}
    t_ms = sum(step_ms)
    t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    ms_per_step = t_ms / args.steps
    value = world * eff_cells * args.steps / (t_ms * 1e-3) / 1e6
    pps = world * n_part * args.steps / (t_ms * 1e-3)

    # ---- e2e through the public API with host-owned particle state
    e2e = None
    if not args.no_e2e:
        from paper_2603_14982_b200.host_io import HostMirror
        p = sim.particles
        # host-owned particle state, pinned: positions and the reference's
        # particle rows (v, C, F, m, V0, vol_corr); the Kirchhoff stress rows
        # are a device cache of F (not reference state) and are recomputed from
        # the uploaded F on the device every step (mlbm_particle_stress)
        mirror = HostMirror([p.xd, p.pd[:p.R["tau"]]])
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        diag_bytes = 0
        for _ in range(args.steps):
            mirror.upload()                  # host -> device, chunked on a copy stream
            sim.particles.stress_mat = None  # tau(F) of the uploaded F
            sim.particles.ensure_stress(sim.material)
            sim.step()
            mirror.download()                # device -> host, overlaps the next upload
            row = sim.diagnostics[-1]        # D2H of the step's diagnostics row
            diag_bytes = 8 * (3 * d + 2)
        mirror.synchronize()
        e1.record()
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        te = float(te.item())
        nb = mirror.nbytes
        e2e = {"value": round(world * eff_cells * args.steps / (te * 1e-3) / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb + diag_bytes,
               "particles_per_s": round(world * n_part * args.steps / (te * 1e-3), 1),
               "ms_per_step": te / args.steps,
               "path": "CoupledSim.step() with the particle state owned by pinned host memory "
                       "(host_io.HostMirror: positions + the reference's rows v, C, F, m, V0, "
                       "vol_corr): uploaded before and read back after every step in row chunks "
                       "on two copy streams (download of step k overlaps upload of step k+1), "
                       "the stress cache tau(F) recomputed from the uploaded F on the device, "
                       "+ diagnostics row D2H"}
        del row

    # ---- per-kernel device times: an eager pass of the same steps with every
    #      C-ABI call bracketed by CUDA events on the launching stream
    sim.use_graphs = False
    kp = min(args.steps, 10)
    L.TRACE.start()
    ek0 = torch.cuda.Event(enable_timing=True)
    ek1 = torch.cuda.Event(enable_timing=True)
    ek0.record()
    for _ in range(kp):
        L.zero(flush)
        sim.step()
    ek1.record()
    torch.cuda.synchronize()
    recs = L.TRACE.stop()
    t_eager_ms = ek0.elapsed_time(ek1)
    sim.use_graphs = True
    classes = {}
    dc = sim.topology.dcounts.cpu().numpy()
    base = sim.topology.dcounts.data_ptr()
    by_ptr = {base + 4 * i: int(v) for i, v in enumerate(dc.reshape(-1))}

    def live(x):
        if isinstance(x, int):
            return by_ptr.get(x, 0)
        if hasattr(x, "value"):                     # ctypes c_void_p
            return by_ptr.get(x.value or 0, 0)
        return sim.topology.n_tiles(int(x.level))

    for r in recs:
        name, e0, e1, _ = r[:4]
        cls, nbytes, units = kernel_class(r, d, s, live)
        c = classes.setdefault(cls, {"ms": 0.0, "launches": 0, "bytes": 0.0})
        c["ms"] += e0.elapsed_time(e1)
        c["launches"] += 1
        c["bytes"] += nbytes
    peak, peak_kind = measured_peak()
    total_k = sum(c["ms"] for c in classes.values())
    for c in classes.values():
        c["ms_per_step"] = c["ms"] / kp
        c["share_of_graph_step"] = c["ms_per_step"] / ms_per_step if ms_per_step else 0.0
        c["achieved_gbs"] = c["bytes"] / (c["ms"] * 1e-3) / 1e9 if c["ms"] and c["bytes"] else None
    dom = max((k for k in classes if classes[k]["bytes"]), key=lambda k: classes[k]["ms"])

    traffic = dram_traffic(args.scene)

    def roof(k):
        c = classes[k]
        ach = c["achieved_gbs"]
        kern = {"p2g": "k_p2g_cell2", "g2p": "k_g2p", "exchange": "k_exchange",
                "transfer": "downward_kernel"}.get(k, "level_kernel" if k.startswith("level") else k)
        tr = traffic.get(kern)
        return {"kernel": k, "bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                "unit": "GB/s", "frac": round(ach / peak, 4), "peak_source": peak_kind,
                "bytes_per_launch": c["bytes"] / c["launches"],
                "avg_launch_us": 1e3 * c["ms"] / c["launches"],
                "traffic": tr["bytes_per_launch"] if tr else None,
                "traffic_source": ("profiles/" + TRAFFIC_FILES.get(args.scene, "") +
                                   ": dram__bytes_read.sum + dram__bytes_write.sum per launch of "
                                   + kern + " from one ncu --set full capture ("
                                   + args.scene.upper() + ")") if tr else None}

    lbm_keys = [k for k in classes if k.startswith("level_step")]
    lbm_bytes = sum(classes[k]["bytes"] for k in lbm_keys)
    lbm_ms = sum(classes[k]["ms"] for k in lbm_keys)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.scene)

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if s == 4 else "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.scene),
                   "effective_cells": eff_cells, "particles": n_part,
                   "levels": cfg.levels, "lattice": "D3Q27" if d == 3 else "D2Q9",
                   "stored_tiles": [sim.topology.n_tiles(l) for l in range(cfg.levels)],
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "flushed (256 MB write) between timed steps, outside the events"},
        "particles_per_s": round(pps, 1),
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": roof(dom),
        "roofline_lbm": {"kernel": "level_step (all modes)", "bound": "hbm",
                         "achieved": round(lbm_bytes / (lbm_ms * 1e-3) / 1e9, 1) if lbm_ms else None,
                         "peak": peak, "unit": "GB/s",
                         "frac": round(lbm_bytes / (lbm_ms * 1e-3) / 1e9 / peak, 4) if lbm_ms else None,
                         "share_of_graph_step": round(lbm_ms / kp / ms_per_step, 4)},
        "kernels": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv)
                        for kk, vv in v.items()} for k, v in sorted(classes.items())},
        "kernel_profile": {"steps": kp, "mode": "eager pass after the timed region, each C-ABI "
                                                 "call bracketed by CUDA events",
                           "kernel_ms_per_step": round(total_k / kp, 4),
                           "eager_ms_per_step": round(t_eager_ms / kp, 4)},
        "graph": graph_info,
        "topology_changes": graph_info["topology_changes"],
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)


def run_slab(args, rank, world, local_rank):
    """C1 (configs[0]) as a slab-decomposed single-level run: rank r owns a
    64^3 slab of a (64 N) x 64 x 64 periodic Taylor-Green domain (weak
    scaling); after every level step the owned edge tile columns go to the
    neighbours' ghost columns by NCCL point-to-point (slab_lbm.py)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2603_14982_b200 import _lib as L
    from paper_2603_14982_b200.harness.config import taylor_green_fn
    from paper_2603_14982_b200.slab_lbm import SlabLBM
    from paper_2603_14982_b200.solver import LevelParams

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n = 64
    cells = (n * world, n, n)
    tau0 = 0.8
    lp = LevelParams(1, tau0)
    sim = SlabLBM(cells, rank, world, tau0, dtype=torch.float32,
                  init=taylor_green_fn(0.05, n, lp.nu(0), lp.taus, 3), device=dev)
    owned = sim.n_owned * 64

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        sim.step()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    clocks = Clocks(local_rank)
    launches0 = L.TRACE.launches
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev, kev = [], []
    for _ in range(args.steps):
        L.zero(flush)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        w = sim.step_local()
        e1.record()
        sim.exchange(w)
        e2.record()
        ev.append((e0, e2))
        kev.append((e0, e1))
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = L.TRACE.launches - launches0
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    k_ms = sum(a.elapsed_time(b) for a, b in kev)
    t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    eff = world * n ** 3
    value = eff * args.steps / (t_ms * 1e-3) / 1e6
    # e2e: the moment state uploaded from pinned host memory and read back every step
    trees = sim.pair.trees
    host = [torch.empty_like(tr.levels[0].data, device="cpu").pin_memory() for tr in trees]
    for h, tr in zip(host, trees):
        h.copy_(tr.levels[0].data)
    torch.cuda.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    nb = 0
    for _ in range(args.steps):
        r, _w = sim.solver.roles(0)
        trees[r].levels[0].data.copy_(host[r], non_blocking=True)
        w = sim.step_local()
        sim.exchange(w)
        host[w].copy_(trees[w].levels[0].data, non_blocking=True)
        nb = trees[w].levels[0].data.numel() * trees[w].levels[0].data.element_size()
    e1.record()
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    te = float(te.item())
    peak, peak_kind = measured_peak()
    kbytes = owned * 2 * 10 * 4
    ach = kbytes * args.steps / (k_ms * 1e-3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.scene)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "C1 slabs: single-level periodic Taylor-Green, D3Q27, a 64^3 "
                                   "slab per GPU of a (64 N) x 64 x 64 domain, ghost tile columns "
                                   "exchanged by NCCL P2P every step",
                       "effective_cells": eff, "parallelism": f"slabs{world}",
                       "l2": "flushed (256 MB write) between timed steps, outside the events"},
            "e2e": {"value": round(eff * args.steps / (te * 1e-3) / 1e6, 3), "unit": UNIT,
                    "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
                    "path": "moment tree uploaded from / read back to pinned host memory every "
                            "step around SlabLBM.step"},
            "gpu_launches": launches,
            "roofline": {"kernel": "level_kernel mode 0 (owned tiles)", "bound": "hbm",
                         "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4), "peak_source": peak_kind,
                         "bytes_per_launch": kbytes, "traffic": None,
                         "avg_launch_us": round(1e3 * k_ms / args.steps, 2)},
            "exchange_ms_per_step": round((t_ms - k_ms) / args.steps, 4),
            "cpu_baseline": cpu, "clocks": clk}), flush=True)


def run_slabs_coupled(args, rank, world, local_rank):
    """The north-star decomposition: the chosen scene (C4 by
    default) split into N x-slabs cut on the coarsest tile width, one per GPU,
    coupled step with the slab collectives (i)-(v) over NCCL point-to-point
    (halo columns and ghost-node sums packed by mlbm_halo_pack, particles
    migrated by mlbm_migrate_count / pack / unpack, uint8 seed OR).  Strong
    scaling: the total work is the scene's."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2603_14982_b200 import _lib as L
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    from paper_2603_14982_b200.slab_coupled import P2PExchanger, SlabCoupled, ThreadExchanger

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    cfg = validate_scene(scene_dict(args.scene))
    ref = build_scene(cfg)           # the global scene, cropped to this rank's slab
    if args.scene == "c5":
        import scenes as S
        S.cloud_velocities(ref)
    ref.use_graphs = False
    xch = P2PExchanger() if world > 1 else ThreadExchanger(1)
    sim = SlabCoupled(ref, rank, world, xch)
    n_glob = len(ref.particles)
    del ref
    torch.cuda.empty_cache()
    eff = int(np.prod(cfg.cells))
    for _ in range(args.warmup):
        sim.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local_rank)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    l0 = L.TRACE.launches
    chg0 = sim.topology_changes
    e0.record()
    for _ in range(args.steps):
        sim.step()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    n_loc = torch.tensor([len(sim.particles)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(n_loc)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(eff * args.steps / (t_ms * 1e-3) / 1e6, 3),
            "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if cfg.dtype == torch.float32 else "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.scene) + f", split into {world} x-slab(s)",
                       "effective_cells": eff, "particles": int(n_loc.item()),
                       "particles_at_start": n_glob, "parallelism": f"slabs{world}",
                       "l2": "not flushed (slab step)"},
            "particles_per_s": round(float(n_loc.item()) * args.steps / (t_ms * 1e-3), 1),
            "e2e": None, "gpu_launches": L.TRACE.launches - l0, "clocks": clk,
            "topology_changes": sim.topology_changes - chg0}), flush=True)


# C4's full scene is ~55.8M particles: the CPU sample is the same scene with
# every extent divided by 4 (872,448 particles, ~50 s per oracle step)
CPU_SAMPLE_SCALE = {"c4": 4}


def oracle_sample(scene):
    """Bounded CPU sample of the same workload: the fp64 NumPy oracle port."""
    from oracle import scene as OS
    from paper_2603_14982_b200.harness.config import validate_scene
    cfg = validate_scene(scene_dict(scene, CPU_SAMPLE_SCALE.get(scene, 1)))
    return cfg, OS.build_scene(cfg.raw, heightmap=cfg.heightmap())


def sample_name(scene):
    k = CPU_SAMPLE_SCALE.get(scene)
    return (f"{scene.upper()} scene with every extent divided by {k}" if k else
            f"full {scene.upper()} scene")


def cpu_baseline(scene):
    import numpy as np
    cfg, sim = oracle_sample(scene)
    t0 = time.perf_counter()
    sim.step()
    dt = time.perf_counter() - t0
    eff = int(np.prod(cfg.cells))
    return {"value": round(eff / dt / 1e6, 4), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"1 coupled step of the {sample_name(scene)} in the fp64 NumPy oracle "
                      f"port (oracle/, single thread) after scene build: {dt:.2f} s",
            "particles_per_s": round(len(sim.p) / dt, 1)}


def run_reference(args, rank):
    """--impl reference: the CPU implementation of the path (oracle port; the
    reference itself is 2D-only NumPy and cannot run this 3D config)."""
    import numpy as np
    if rank != 0:
        return
    cfg, sim = oracle_sample(args.scene)
    eff = int(np.prod(cfg.cells))
    for _ in range(min(args.warmup, 1)):
        sim.step()
    k = min(args.steps, REF_TIMED_STEPS_CAP)
    t0 = time.perf_counter()
    for _ in range(k):
        sim.step()
    dt = time.perf_counter() - t0
    value = eff * k / dt / 1e6
    sample = (f"{k} coupled steps (of {args.steps} requested, capped to bound CPU time) of the "
              f"{sample_name(args.scene)} in the fp64 NumPy oracle port, 1 thread")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": k, "warmup": min(args.warmup, 1),
        "ms_per_step": round(1e3 * dt / k, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.scene), "effective_cells": eff,
                   "particles": len(sim.p)},
        "particles_per_s": round(len(sim.p) * k / dt, 1),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.scene == "c1":
            run_slab(args, rank, world, local_rank)
        elif args.slabs or (world > 1 and not args.replicas):
            run_slabs_coupled(args, rank, world, local_rank)
        else:
            run_mine(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
