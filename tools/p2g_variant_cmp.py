"""Relative differences between the raster rows saved by tools/p2g_variant.py:
python tools/p2g_variant_cmp.py REF OTHER..."""
import sys
import torch
ref = torch.load("/tmp/p2gvar/%s.pt" % sys.argv[1]).double()
for t in sys.argv[2:]:
    o = torch.load("/tmp/p2gvar/%s.pt" % t).double()
    rel = [float((o[q] - ref[q]).norm() / ref[q].norm().clamp_min(1e-300)) for q in range(ref.shape[0])]
    print(t, "vs", sys.argv[1], "rel L2 per row:", " ".join("%.1e" % r for r in rel))
