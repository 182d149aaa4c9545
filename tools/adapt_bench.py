"""Time GridAdaptor.plan_device (fused cooperative pass) on the C2 scene."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
import os
_sc = os.environ.get("SCENE", "COLUMN_3D_C2")
if _sc == "AVALANCHE_C4":
    import tempfile
    _scd = S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "terrain.npy"))
else:
    _scd = getattr(S, _sc)
sim = build_scene(validate_scene(_scd))
for _ in range(3):
    sim.step()
ad = sim.adaptor
drv = sim._driver()
torch.cuda.synchronize()
for fused in (True, False):
    ad.fused = fused
    for _ in range(3):
        ad.plan_device(drv)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ad.plan_device(drv)
    e1.record(); torch.cuda.synchronize()
    print("fused" if fused else "separate", "plan_device us", 1e3 * e0.elapsed_time(e1) / 20)
import os, ctypes
from paper_2603_14982_b200 import _lib as L
if os.environ.get("MLBM_ADAPT_TIMESTAMPS"):
    ad.fused = True
    ad.plan_device(drv); torch.cuda.synchronize()
    lib = L.load()
    tsbuf = torch.zeros(64, dtype=torch.int64, device="cuda")     # caller-owned stamps
    lib.mlbm_adapt_set_timestamps(ctypes.c_void_p(tsbuf.data_ptr()))
    ad.plan_device(drv); torch.cuda.synchronize()
    lib.mlbm_adapt_set_timestamps(ctypes.c_void_p(0))
    ts = tsbuf.cpu().tolist()[:16]
    names = {0: "start", 2: "A+B seeds/invariants", 3: "C des0/cur1", 4: "D par/cur", 5: "E des[l]",
             6: "F eff0", 7: "G par(eff)", 8: "H eff[l]", 9: "top eff", 10: "I own", 11: "J storage/kinds"}
    prev = ts[0]
    for i in range(2, 12):
        if ts[i]:
            print("  %-22s %6.2f us" % (names[i], (ts[i] - prev) / 1e3))
            prev = ts[i]
    print("  total                  %6.2f us" % ((prev - ts[0]) / 1e3))
if os.environ.get("MLBM_ADAPT_TIMESTAMPS"):
    lib.mlbm_adapt_bits_ts_ptr.restype = ctypes.c_void_p
    ptr = lib.mlbm_adapt_bits_ts_ptr()
    if ptr:
        ad.plan_device(drv); torch.cuda.synchronize()
        buf = (ctypes.c_uint64 * 64)()
        cudart.cudaMemcpy(buf, ctypes.c_void_p(ptr), ctypes.c_size_t(64 * 8), 2)
        ts = [v for v in list(buf)[:40]]
        last = ts[0]
        out = []
        for k in range(1, 40):
            if ts[k]:
                out.append(round((ts[k] - last) / 1e3, 2))
                last = ts[k]
        print("bits phase deltas us:", out, "total", round((last - ts[0]) / 1e3, 2))
