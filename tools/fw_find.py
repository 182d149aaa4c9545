import os, sys, tempfile, json
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
import scenes as S
from paper_2603_14982_b200.harness import build_scene, validate_scene
scd = S.avalanche_c4(os.path.join(tempfile.mkdtemp(), "t.npy"))
sim = build_scene(validate_scene(scd))
for _ in range(6):
    sim.step()
torch.cuda.synchronize()
mode = sys.argv[1] if len(sys.argv) > 1 else "graph"
sim.use_graphs = mode == "graph"
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], with_stack=True) as prof:
    for _ in range(6):
        sim.step()
    torch.cuda.synchronize()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("aten::") and e.name not in ("aten::empty", "aten::empty_strided", "aten::view", "aten::as_strided", "aten::slice", "aten::select", "aten::lift_fresh", "aten::detach_", "aten::alias", "aten::_local_scalar_dense", "aten::item", "aten::resolve_conj", "aten::resolve_neg", "aten::numpy_T", "aten::t", "aten::transpose", "aten::expand", "aten::unsqueeze", "aten::reshape", "aten::_reshape_alias", "aten::to", "aten::_to_copy", "aten::pin_memory", "aten::_pin_memory", "aten::is_pinned", "aten::set_"):
        st = [f for f in (e.stack or []) if "paper_2603" in f or "bench" in f]
        print(e.name, st[:3])
