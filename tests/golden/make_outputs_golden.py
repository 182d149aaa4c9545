"""Golden frame outputs written by the REFERENCE's own writers (outputs.py)
for a small 2D scene, stored with the exact inputs the writers saw, so the
B200 package's writers can be checked byte for byte without the reference.

    python tests/golden/make_outputs_golden.py      (builder container only)
"""
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

from mlbm.harness import config as RCF  # noqa: E402
from mlbm.harness import outputs as RO  # noqa: E402

import scenes as S  # noqa: E402


def main():
    sc = S.scene(S.DUNE_2D, runtime__mpm_cadence=1)
    sc.setdefault("outputs", {}).update({"fields": True, "particles": True, "quicklook": True,
                                          "diagnostics": True})
    cfg = RCF.validate_scene(sc)
    sim = RCF.build_scene(cfg)
    for _ in range(3):
        sim.step()
    out = {}
    with tempfile.TemporaryDirectory() as d:
        RO.write_frame(d, 7, sim, cfg)
        for fn in sorted(os.listdir(d)):
            with open(os.path.join(d, fn), "rb") as fh:
                out["file_" + fn] = np.frombuffer(fh.read(), dtype=np.uint8)
        rows = [(0, len(sim.particles), 1.25, 0.5), (1, 7, 0.1 + 0.2, 3.0)]
        p = os.path.join(d, "summary.csv")
        RO.particle_summary_csv(p, rows)
        out["file_summary.csv"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
        p = os.path.join(d, "diag.csv")
        w = RO.DiagnosticsWriter(p, sim.topology.levels)
        for r in sim.diagnostics:
            w.write(r)
        w.close()
        out["file_diag.csv"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
    # the writers' inputs: dense per-level grids (x-major) and the particles
    topo, sv = sim.topology, sim.solver
    out["levels"] = np.array(topo.levels)
    for l in range(topo.levels):
        nx, ny = topo.cells_dims(l)
        cmap = topo.cell_map(l)
        w = sv.last_roles(l)[1] if sv.k[l] else 0
        arr = sv.arrays(w, l)
        for nm in ("rho", "ux", "uy", "eps", "phi"):
            g = np.zeros((nx, ny))
            g[cmap >= 0] = np.asarray(arr[nm])[cmap[cmap >= 0]]
            out[f"L{l}_{nm}"] = g
        st = np.zeros((nx, ny))
        t = topo.tables[l]
        for slot, (tx, ty) in enumerate(t.coords):
            st[tx * 4:(tx + 1) * 4, ty * 4:(ty + 1) * 4] = 2.0 if t.kind[slot] == 0 else 1.0
        out[f"L{l}_stored"] = st
    out["px"] = np.asarray(sim.particles.x)
    out["pv"] = np.asarray(sim.particles.v)
    out["pm"] = np.asarray(sim.particles.m)
    out["diag"] = np.array([[r.step, r.t_phys, *r.fluid_mom, *r.sediment_mom, *r.drag_impulse,
                             r.sum_phi, *r.tiles, r.eps_min] for r in sim.diagnostics])
    np.savez_compressed(os.path.join(HERE, "outputs_dune_2d.npz"), **out)
    print("wrote outputs_dune_2d.npz:", sorted(k for k in out if k.startswith("file_")))


if __name__ == "__main__":
    main()
