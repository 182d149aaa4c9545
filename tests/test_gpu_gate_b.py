"""Gate B of BASELINE.json's north star: the fp32 device path against the
fp64 oracle, <= 1e-5 relative L2 on the density deviation, velocity and
second-order moment fields of every level and on the particle velocities and
displacements, after N steps (SURVEY.md §8(d) gate B).

The fp32 path stores drho = rho - 1 and reconstructs g = f - w;
particle positions stay float64.  The drift curve over N = 1..20 is committed
under profiles/ (tools/gate_b_drift.py)."""
import numpy as np
import pytest
import torch

import scenes as S
from helpers import central_mask, gate_b_metrics, oracle_static_refined
from oracle import grid as OG
from oracle import scene as OS

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2603_14982_b200")

GATE_B = 1e-5


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def build_both(scene_dict):
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    cfg = validate_scene(scene_dict)
    return OS.build_scene(cfg.raw, heightmap=cfg.heightmap()), build_scene(cfg)


def run_gate_b(sc, steps):
    osim, dsim = build_both(sc)
    ox0 = osim.p.x.copy()
    dx0 = dsim.particles.x.cpu().numpy().copy()
    for s in range(steps):
        osim.step()
        dsim.step()
        assert dsim.topology.tile_set() == osim.topo.tile_set(), f"tile sets differ at step {s}"
    return gate_b_metrics(osim, dsim, ox0, dx0)


@pytest.mark.parametrize("name,steps", [("column", 20), ("sandstorm", 20), ("sand_collapse_2d", 20)])
def test_gate_b_coupled_fp32(name, steps):
    _need_gpu()
    sc = {"column": S.COLUMN_3D_SMALL, "sandstorm": S.SANDSTORM_3D_SMALL,
          "sand_collapse_2d": S.SAND_COLLAPSE_2D}[name]
    m = run_gate_b(S.scene(sc, runtime__dtype="f32"), steps)
    print(name, m)
    bad = {k: v for k, v in m.items() if not v <= GATE_B}
    assert not bad, (m, bad)


@pytest.mark.parametrize("levels", [2, 3])
def test_gate_b_multilevel_lbm_fp32(levels):
    """fp32 multi-level LBM (transfers, rescaling, sub-cycling) vs fp64."""
    _need_gpu()
    from test_gpu_lbm import build_pair, last, smooth_fields
    from helpers import rel_l2
    cells = (32, 32, 32)
    otopo = oracle_static_refined(cells, levels, central_mask(cells, pad=4))
    osv, dsv = build_pair(otopo, torch.float32, smooth_fields(3, 23, amp=0.03), tau0=0.8)
    for _ in range(100 >> (levels - 1)):
        osv.advance_bounce()
        dsv.advance_bounce()
    names = OG.moment_names(3)
    for nm in names:
        if nm == "rho":
            # relative to the deviation, not to rho ~ 1
            ol = {l: {"rho": np.asarray(last(osv, l)["rho"]) - 1.0} for l in range(levels)}
            dl = {l: {"rho": last(dsv, l).data[0, :dsv.topology.cell_count(l)]}
                  for l in range(levels)}
            r = rel_l2(otopo, lambda l: ol[l], dsv.topology, lambda l: dl[l], ["rho"])
        else:
            r = rel_l2(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l), [nm])
        assert r <= GATE_B, (nm, r)


def test_c2_full_size_gate_a_and_b():
    """BASELINE.json configs[1] at its bench size (128^3-effective, two
    levels, 262,144 particles): fp64 device at gate A (tile sets and streaks
    exact, fields / particles <= 1e-9) and the fp32 bench path at gate B
    (<= 1e-5 relative L2), both after 2 coupled steps against the oracle."""
    _need_gpu()
    from test_gpu_coupled import field_diff, particle_diff
    steps = 2
    o64, d64 = build_both(S.scene(S.COLUMN_3D_C2, runtime__dtype="f64"))
    _, d32 = build_both(S.scene(S.COLUMN_3D_C2, runtime__dtype="f32"))
    ox0 = o64.p.x.copy()
    dx0 = d32.particles.x.cpu().numpy().copy()
    for s in range(steps):
        o64.step()
        d64.step()
        d32.step()
        assert d64.topology.tile_set() == o64.topo.tile_set(), s
        assert d32.topology.tile_set() == o64.topo.tile_set(), s
        for a, b in zip(d64.adaptor.streak, o64.adaptor.streak):
            assert np.array_equal(a, b)
    assert field_diff(o64, d64) <= 1e-9
    assert particle_diff(o64, d64) <= 1e-9
    m = gate_b_metrics(o64, d32, ox0, dx0)
    print("c2", m)
    assert all(v <= GATE_B for v in m.values()), m


def test_gate_b_snow_fp32():
    """Gate B on the snow path (NACC in fp32 G2P) against the fp64 oracle."""
    _need_gpu()
    m = run_gate_b(S.scene(S.SNOW_3D_SMALL, runtime__dtype="f32"), 10)
    print("snow", m)
    assert all(v <= GATE_B for v in m.values()), m
