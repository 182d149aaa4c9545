"""Frame writers vs files the REFERENCE's own writers produced
(tests/golden/outputs_dune_2d.npz, made by make_outputs_golden.py): the same
inputs give the same bytes (VTK levels, particle dump, PPM quicklooks, CSV)."""
import os
import tempfile
from types import SimpleNamespace

import numpy as np
import torch

from paper_2603_14982_b200.harness import outputs as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "outputs_dune_2d.npz")


def _g():
    return np.load(GOLD)


def _bytes(g, name):
    return g["file_" + name].tobytes()


def test_vtk_levels_byte_identical():
    g = _g()
    for l in range(int(g["levels"])):
        dims = g[f"L{l}_rho"].shape
        text = O.vtk_text(l, dims, float(1 << l),
                          [("rho", g[f"L{l}_rho"]), ("eps", g[f"L{l}_eps"]),
                           ("phi", g[f"L{l}_phi"]), ("stored", g[f"L{l}_stored"])],
                          [g[f"L{l}_ux"], g[f"L{l}_uy"]])
        assert text.encode() == _bytes(g, f"frame_00007_l{l}.vtk"), l


def test_vtk_round_trip():
    g = _g()
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "l0.vtk")
        with open(p, "wb") as fh:
            fh.write(_bytes(g, "frame_00007_l0.vtk"))
        back = O.read_vtk_level(p)
    assert np.array_equal(back["rho"], g["L0_rho"])
    assert np.array_equal(back["ux"], g["L0_ux"]) and np.array_equal(back["uy"], g["L0_uy"])


def test_particle_dump_and_quicklooks_byte_identical():
    g = _g()
    parts = SimpleNamespace(x=torch.as_tensor(g["px"]), v=torch.as_tensor(g["pv"]),
                            m=torch.as_tensor(g["pm"]))
    parts.__len__ = lambda: len(g["pm"])
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "p.bin")
        O.write_particles(p, parts)
        assert open(p, "rb").read() == _bytes(g, "frame_00007_particles.bin")
        x, v, m = O.read_particles(p)
        assert np.array_equal(x, g["px"]) and np.array_equal(v, g["pv"]) and np.array_equal(m, g["pm"])
        p = os.path.join(d, "s.ppm")
        O.write_ppm(p, np.hypot(g["L0_ux"], g["L0_uy"]), 0.1)
        assert open(p, "rb").read() == _bytes(g, "frame_00007_speed.ppm")
        dens = np.zeros(g["L0_rho"].shape)
        c = np.floor(g["px"]).astype(np.int64)
        np.add.at(dens, (c[:, 0].clip(0, dens.shape[0] - 1), c[:, 1].clip(0, dens.shape[1] - 1)), 1.0)
        p = os.path.join(d, "q.ppm")
        O.write_ppm(p, dens, 8.0)
        assert open(p, "rb").read() == _bytes(g, "frame_00007_parts.ppm")


def test_csv_writers_byte_identical():
    g = _g()
    L = int(g["levels"])
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "s.csv")
        O.particle_summary_csv(p, [(0, len(g["pm"]), 1.25, 0.5), (1, 7, 0.1 + 0.2, 3.0)])
        assert open(p, "rb").read() == _bytes(g, "summary.csv")
        p = os.path.join(d, "d.csv")
        w = O.DiagnosticsWriter(p, L)
        for r in g["diag"]:
            w.write(SimpleNamespace(step=int(r[0]), t_phys=float(r[1]),
                                    fluid_mom=(float(r[2]), float(r[3])),
                                    sediment_mom=(float(r[4]), float(r[5])),
                                    drag_impulse=(float(r[6]), float(r[7])), sum_phi=float(r[8]),
                                    tiles=tuple(int(t) for t in r[9:9 + L]),
                                    eps_min=float(r[9 + L])))
        w.close()
        assert open(p, "rb").read() == _bytes(g, "diag.csv")
