"""Loader and ctypes bindings of the sm_100a C-ABI library (libmlbm_b200.so).

The library is built in-tree by :func:`build` (nvcc, ``-gencode
arch=compute_100a,code=sm_100a``) and loaded with ctypes; every product
kernel goes through these bindings.  There is no CPU fallback: if the
library is missing or no CUDA device is present, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBPATH = os.environ.get("MLBM_LIB") or os.path.join(HERE, "libmlbm_b200.so")
SOURCES = ["lbm.cu", "topology.cu", "mpm.cu", "adapt.cu", "adapt_bits.cu", "slab.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-Wno-deprecated-declarations",
              "-diag-suppress", "1444"]

MAX_LEVELS = 6


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def build(force=False, verbose=False, extra=(), out=None):
    """Compile every .cu into the in-tree shared library (objects cached).
    ``extra`` nvcc flags + ``out`` path build a tuning variant (tools/)."""
    objs = []
    libpath = out or LIBPATH
    bdir = os.path.join(os.path.dirname(out), "build") if out else os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    hdrs.append(os.path.join(INCLUDE, "mlbm_b200.h"))
    hmt = max(os.path.getmtime(h) for h in hdrs)
    procs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        op = os.path.join(bdir, src.replace(".cu", ".o"))
        objs.append(op)
        if (not force and os.path.exists(op) and os.path.getmtime(op) >=
                max(os.path.getmtime(sp), hmt)):
            continue
        cmd = [_nvcc()] + NVCC_FLAGS + list(extra) + ["-I", INCLUDE, "-c", sp, "-o", op]
        if verbose:
            print(" ".join(cmd))
        procs.append((cmd, subprocess.Popen(cmd)))
    for cmd, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    if (force or not os.path.exists(libpath) or
            os.path.getmtime(libpath) < max(os.path.getmtime(o) for o in objs)):
        cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
               "-o", libpath] + objs + ["-lcudart"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return libpath


# -- C structs (mirror include/mlbm_b200.h) ------------------------------------

class Snow(C.Structure):
    """mlbm_snow_t: NACC snow parameters (include/mlbm_b200.h)."""
    _fields_ = [("M", C.c_double), ("beta", C.c_double), ("xi", C.c_double),
                ("alpha_soft", C.c_double)]


class Level(C.Structure):
    _fields_ = [("dim", C.c_int32), ("level", C.c_int32),
                ("cells", C.c_int32 * 3), ("tiles", C.c_int32 * 3),
                ("periodic", C.c_int32 * 3), ("n_tiles", C.c_int32),
                ("tile_map", C.c_void_p), ("tile_xyz", C.c_void_p),
                ("nbr", C.c_void_p), ("cell_flags", C.c_void_p),
                ("dir_masks", C.c_void_p), ("tile_flags", C.c_void_p),
                ("counts", C.c_void_p), ("first", C.c_int32)]


class Fields(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("stride", C.c_int64)]


class BC(C.Structure):
    _fields_ = [("face", C.c_int32 * 6), ("inlet_u0", C.c_double),
                ("inlet_beta", C.c_double), ("inlet_y0", C.c_double),
                ("rho0", C.c_double)]


class Solid(C.Structure):
    _fields_ = [("n_boxes", C.c_int32), ("boxes", (C.c_double * 6) * 16),
                ("heightmap", C.c_void_p), ("hm_dims", C.c_int32 * 2),
                ("near", C.c_void_p * 6)]


class Collide(C.Structure):
    _fields_ = [("tau", C.c_double), ("gravity", C.c_double * 3),
                ("h3_xyz", C.c_double), ("force_mode", C.c_int32),
                ("tau_mode", C.c_int32), ("tau0", C.c_double),
                ("tau_ptr", C.c_void_p)]


class Hier(C.Structure):
    _fields_ = [("dim", C.c_int32), ("levels", C.c_int32),
                ("finest", C.c_int32 * 3), ("periodic", C.c_int32 * 3),
                ("kind", C.c_void_p * MAX_LEVELS),
                ("tile_map", C.c_void_p * MAX_LEVELS),
                ("fields", (C.c_void_p * MAX_LEVELS) * 2),
                ("stride", C.c_int64 * MAX_LEVELS),
                ("n_tiles", C.c_int32 * MAX_LEVELS)]


ERR_INTS = 19   # mlbm_error_t as int32 words
# mlbm_coupling_op operations (include/mlbm_b200.h)
COUPLE_FRACTIONS, COUPLE_DRAG, COUPLE_LIMIT, COUPLE_GRAD_EPS, COUPLE_MIXTURE_FORCE = range(5)

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double
_SIGS = {
    "mlbm_level_step": [C.POINTER(Level), Fields, Fields, I32, I32,
                        C.POINTER(Collide), C.POINTER(BC), P, P],
    "mlbm_downward": [I32, I32, P, P, P, P, Fields, Fields, Fields, I32, I32, D, P],
    "mlbm_upward": [I32, I32, P, P, P, Fields, Fields, I32, I32, D, P],
    "mlbm_ws_bytes": [I64],
    "mlbm_compact_tiles": [I32, P, P, P, P, P, P, P, I32, P, P, I64, P],
    "mlbm_build_neighbors": [C.POINTER(Level), P, P],
    "mlbm_classify_level": [C.POINTER(Level), C.POINTER(Hier), C.POINTER(BC),
                            C.POINTER(Solid), P, P, P, P, P, P, P, P, P, P, P, P],
    "mlbm_copy": [P, P, I64, P],
    "mlbm_changed_tiles": [I64, P, P, P, P, P, I64, P],
    "mlbm_mark_dirty": [C.POINTER(Hier), I32, P, P, P, P],
    "mlbm_build_interface": [C.POINTER(Level), C.POINTER(Level), I32, P, P, P, P,
                             P, I64, P],
    "mlbm_seed_tiles": [I32, I32, P, I64, I32, P, P, P, P],
    "mlbm_bitmap_op": [I32, I32, P, P, P, P],
    "mlbm_dilate": [I32, P, P, I32, P, P, P, P],
    "mlbm_effective_level": [I32, P, P, P, P, P, P, P, P],
    "mlbm_plan_level": [I32, P, P, P, P, P, P],
    "mlbm_check_coverage": [C.POINTER(Hier), P, P],
    "mlbm_count_ring_violations": [I64, P, P, P, P],
    "mlbm_check_particles": [I32, I32, P, I64, I32, P, P, P, P],
    "mlbm_copy_live_fields": [I32, I32, P, Fields, Fields, Fields, Fields, I32, P],
    "mlbm_migrate_level": [I32, I32, P, P, Fields, Fields, Fields, Fields, I32, P],
    "mlbm_init_new_cells": [C.POINTER(Hier), C.POINTER(Hier), I32, P, P, I32, P,
                            Fields, Fields, P, I32, I32, P, P],
    "mlbm_adapt_pass": [C.POINTER(Hier), P, P, P, P, P, P, P, P, P, P, P, I64, I32, P, P, P, P, P,
                        P],
    "mlbm_adapt_set_timestamps": [P],
    "mlbm_adapt_bits_set_timestamps": [P],
    "mlbm_raster_rows": [I32],
    "mlbm_particle_rows": [I32],
    "mlbm_p2g": [C.POINTER(Level), I32, P, P, I64, D, D, D, P, I64, I32, I32, P, P],
    "mlbm_sort_ws_bytes": [I64, I64],
    "mlbm_scan_ws_bytes": [I32],
    "mlbm_scan_i32": [I32, P, P, P, I64, P],
    "mlbm_particle_sort": [C.POINTER(Level), I32, P, P, P, I64, P, P, P, I32, P, I64, P],
    "mlbm_exchange": [C.POINTER(Level), Fields, Fields, Fields, Fields, P, I64,
                      D, D, D, D, D, D, P, P, P, D, I32, I32, P],
    "mlbm_level0_coupled": [C.POINTER(Level), Fields, Fields, Fields, Fields, I32,
                            C.POINTER(Collide), C.POINTER(BC), P, I64, D, D, D, D, D, D, P, P, P, D,
                            P, P],
    "mlbm_g2p": [C.POINTER(Level), I32, P, P, P, P, P, P, I64, D, D, D, C.POINTER(Snow), P,
                 I64, D, I32, I32, P, P, P, P, P, P],
    "mlbm_stress_raster": [C.POINTER(Level), I32, P, P, I64, D, D, D, P, I64,
                           I32, P, P],
    "mlbm_stress_raster_surface": [C.POINTER(Level), I32, P, P, I64, D, D, D, P, I64, D, P,
                                   I32, P, P],
    "mlbm_powder": [C.POINTER(Level), Fields, Fields, P, I64, P, P, D, D, D, D, D,
                    I32, I32, P],
    "mlbm_coupling_op": [C.POINTER(Level), I32, P, I64, P, P, I64, P, I64, D, D, D, D, D, D,
                         P, I32, P],
    "mlbm_halo_pack": [P, I64, I32, I64, I64, P, I32, P],
    "mlbm_halo_unpack": [P, P, I64, I32, I64, I64, I32, I32, P],
    "mlbm_migrate_ws_bytes": [I32],
    "mlbm_migrate_count": [I32, P, D, D, I32, I32, P, P, I64, P],
    "mlbm_migrate_pack": [I32, I32, P, P, P, I64, I32, I32, D, D, D, D, I32, I32, P, P, P, I64,
                          P, P, P, I64, P, P, P, I64, P, I64, P],
    "mlbm_migrate_unpack": [I32, I32, P, P, P, I64, I32, I32, D, D, D, P, P, P, I64, I32, P],
    "mlbm_memset": [P, I32, I64, P],
    "mlbm_fill": [P, I64, I32, D, P],
    "mlbm_solid_near": [C.POINTER(Level), C.POINTER(Solid), P, P],
    "mlbm_particle_stress": [I32, I32, P, I64, D, D, D, I32, P],
    "mlbm_stencil": [C.POINTER(Level), I32, P, I64, P, P, P, P, I64, I32, P, P],
    "mlbm_powder_step": [C.POINTER(Level), Fields, Fields, P, D, D, D, P, I32, P],
    "mlbm_diag_level": [C.POINTER(Level), Fields, D, I32, P, P],
    "mlbm_diag_particles": [I32, I32, P, I64, P, I64, I64, P, I32, P, P],
}
_RET64 = {"mlbm_ws_bytes", "mlbm_sort_ws_bytes", "mlbm_migrate_ws_bytes", "mlbm_scan_ws_bytes"}

_LIB = None


class KernelError(RuntimeError):
    pass


def load(path=LIBPATH):
    """Load the shared library and bind every exported symbol."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise KernelError(
            f"CUDA library {path} is missing: run __graft_entry__.build() "
            "(no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int64 if name in _RET64 else C.c_int
    _LIB = lib
    return lib


class _Tracer:
    """Counts kernel launches of the library and, when enabled, brackets each
    C-ABI call with CUDA events on the current stream (bench.py uses it to
    time kernels inside the timed region)."""

    def __init__(self):
        self.launches = 0
        self.enabled = False
        self.records = []

    def start(self):
        self.enabled = True
        self.records = []

    def stop(self):
        self.enabled = False
        return self.records


TRACE = _Tracer()


class _TracedLib:
    def __init__(self, lib):
        self._lib = lib
        self._cache = {}

    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        if not name.startswith("mlbm_") or name in _RET64 or name.endswith("_rows"):
            return fn

        def call(*args):
            if TRACE.enabled:
                import torch
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                r = fn(*args)
                e1.record()
                TRACE.records.append((name, e0, e1, r, args))
            else:
                r = fn(*args)
            if r > 0:
                TRACE.launches += r
            return r
        return call


_TRACED = None


def lib():
    """The bound library; raises if it cannot run kernels here."""
    global _TRACED
    import torch
    if not torch.cuda.is_available():
        raise KernelError("no CUDA device: the B200 path has no CPU fallback")
    if _TRACED is None:
        _TRACED = _TracedLib(load())
    return _TRACED


def check(status, what):
    if status < 0:
        raise KernelError(f"{what} failed with status {status}")


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def zero(t):
    """Zero a contiguous device tensor on the current stream (cudaMemsetAsync:
    no framework kernel inside captured graphs)."""
    if t is None or t.numel() == 0:
        return
    assert t.is_contiguous()
    check(lib().mlbm_memset(ptr(t), 0, t.numel() * t.element_size(), stream_handle()), "memset")


def pack_cols(view, buf):
    """Rows x columns view of a SoA block (unit column stride) -> contiguous
    buffer with the library's halo kernel (mlbm_halo_pack); CPU: copy."""
    if not view.is_cuda:
        buf.copy_(view)
        return buf
    assert view.stride(1) == 1 and buf.is_contiguous() and buf.numel() == view.numel()
    check(lib().mlbm_halo_pack(ptr(view), view.stride(0), view.shape[0], 0, view.shape[1], ptr(buf),
                               view.element_size(), stream_handle()), "halo_pack")
    return buf


def unpack_cols(buf, view, add=False):
    """Contiguous buffer -> rows x columns view (copy, or add: ghost-node sums)."""
    import torch
    if not view.is_cuda:
        if add:
            view.add_(buf.to(view.device))
        else:
            view.copy_(buf)
        return
    assert view.stride(1) == 1 and buf.is_contiguous() and buf.numel() == view.numel()
    dt = 1 if view.dtype == torch.float64 else 0
    check(lib().mlbm_halo_unpack(ptr(buf), ptr(view), view.stride(0), view.shape[0], 0, view.shape[1],
                                 dt, 1 if add else 0, stream_handle()), "halo_unpack")


def copy(dst, src):
    """Device-to-device copy of a whole contiguous tensor on the stream."""
    assert dst.is_contiguous() and src.is_contiguous() and dst.numel() == src.numel()
    check(lib().mlbm_copy(ptr(dst), ptr(src), src.numel() * src.element_size(), stream_handle()),
          "copy")


def zeros(shape, dtype, device):
    """A zeroed device tensor (cudaMemsetAsync; no framework kernel), torch
    elsewhere."""
    import torch
    if torch.device(device).type != "cuda":
        return torch.zeros(shape, dtype=dtype, device=device)
    t = torch.empty(shape, dtype=dtype, device=device)
    zero(t)
    return t


def full(shape, value, dtype, device):
    """A device tensor filled with ``value`` (library fill kernel; uint8,
    int32, float32, float64), torch elsewhere."""
    import torch
    if torch.device(device).type != "cuda":
        return torch.full(shape, value, dtype=dtype, device=device)
    t = torch.empty(shape, dtype=dtype, device=device)
    fill(t, value)
    return t


def fill(t, value):
    """Fill a contiguous device tensor with ``value`` (library kernel)."""
    import torch
    if t is None or t.numel() == 0:
        return
    assert t.is_contiguous()
    kind = {torch.uint8: 0, torch.int32: 1, torch.float32: 2, torch.float64: 3}[t.dtype]
    check(lib().mlbm_fill(ptr(t), t.numel(), kind, float(value), stream_handle()), "fill")


def stream_handle():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def fields(t):
    """Fields struct of a [nf, n] tensor (row stride)."""
    if t is None:
        return Fields(0, 0)
    return Fields(t.data_ptr(), t.stride(0))
