import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import scenes as S
from oracle import scene as OS
from paper_2603_14982_b200.harness import build_scene, validate_scene
cfg = validate_scene(S.scene(S.POWDER_3D_SMALL, runtime__dtype=sys.argv[1]))
dsim = build_scene(cfg); osim = OS.build_scene(cfg.raw, heightmap=cfg.heightmap())
for st in range(12):
    osim.step(); dsim.step()
    ow = osim.solver.last_roles(0)[1] if osim.solver.k[0] else 0
    dw = dsim.solver.last_roles(0)[1] if dsim.solver.k[0] else 0
    oa = osim.solver.arrays(ow, 0)["phi"]
    da = dsim.solver.arrays(dw, 0)["phi"].double().cpu().numpy()
    dmap = {tuple(c): i for i, c in enumerate(dsim.topology.cell_coords(0))}
    perm = np.array([dmap[tuple(c)] for c in osim.topo.cell_coords(0)])
    n = np.linalg.norm(oa)
    print(st, "phi norm %.3e rel %.3e" % (n, np.linalg.norm(da[perm] - oa) / max(n, 1e-300)))
