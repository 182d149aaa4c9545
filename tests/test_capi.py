"""The C-ABI library: builds for sm_100a, loads, and exports every symbol
declared in include/mlbm_b200.h (no kernel launches: CPU-only check)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mlbm_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t)\s+(mlbm_\w+)\s*\(", txt, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("mlbm_level_step", "mlbm_downward", "mlbm_upward", "mlbm_compact_tiles",
              "mlbm_classify_level", "mlbm_build_interface", "mlbm_effective_level",
              "mlbm_plan_level", "mlbm_migrate_level", "mlbm_init_new_cells", "mlbm_p2g",
              "mlbm_exchange", "mlbm_g2p", "mlbm_powder", "mlbm_diag_level"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    pytest.importorskip("torch")
    from paper_2603_14982_b200 import _lib
    if not os.path.exists(_lib.LIBPATH):
        _lib.build()
    lib = ctypes.CDLL(_lib.LIBPATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert missing == []
    # every declared symbol has a ctypes signature in the binding table
    unbound = [s for s in declared_symbols() if s not in _lib._SIGS]
    assert unbound == []


def test_library_is_sm100a():
    from paper_2603_14982_b200 import _lib
    if not os.path.exists(_lib.LIBPATH):
        pytest.skip("library not built")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIBPATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_14982_b200 import _lib
    with pytest.raises(_lib.KernelError):
        _lib.lib()


def test_pure_host_size_queries():
    from paper_2603_14982_b200 import _lib
    if not os.path.exists(_lib.LIBPATH):
        pytest.skip("library not built")
    lib = _lib.load()
    # the reference's 27 reals per particle in 3D (3 float64 positions + 24 rows)
    # plus the cached Kirchhoff stress (6 rows in 3D, 3 in 2D)
    assert lib.mlbm_particle_rows(3) == 24 + 6
    assert lib.mlbm_particle_rows(2) == 13 + 3
    assert lib.mlbm_raster_rows(3) == 4 + 7 * 3 + 6 + 1
    assert lib.mlbm_ws_bytes(1000) >= 4 * 1000          # flags + block sums of the scan
    assert lib.mlbm_sort_ws_bytes(1000, 50) > 3 * 4 * 1000
