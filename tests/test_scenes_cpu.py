"""The bench scenes validate through the reference-schema builder and have the
sizes SURVEY.md §8(d) states (CPU only: no device work)."""
import numpy as np

import scenes as S
from paper_2603_14982_b200.harness.config import validate_scene


def _particles(cfg):
    p = cfg.raw["particles"]
    d = cfg.dim
    n = 0
    for b in p["blocks"]:
        vol = 1.0
        for a in range(d):
            vol *= b[d + a] - b[a]
        n += int(round(vol * p["per_cell"]))
    return n


def test_c4_avalanche_scene(tmp_path):
    cfg = validate_scene(S.avalanche_c4(str(tmp_path / "terrain.npy")))
    assert tuple(cfg.cells) == (1536, 768, 384) and cfg.levels == 4
    assert _particles(cfg) == 55_836_672
    hm = cfg.heightmap()
    assert hm.shape == (1536, 384)
    # a mountain flank: > 100 cells of relief under the slab ...
    assert hm[256:1280].max() - hm[256:1280].min() > 100.0
    # ... and no particle starts inside the terrain
    for b in cfg.raw["particles"]["blocks"]:
        assert b[1] > hm[int(b[0]):int(b[3])].max()
    assert cfg.raw["powder"]["enabled"]
    # the CPU sample: every extent divided by 4, coarsest tiles still whole
    small = validate_scene(S.avalanche_c4(str(tmp_path / "terrain4.npy"), scale=4))
    assert tuple(small.cells) == (384, 192, 96)
    assert all(c % (4 << (small.levels - 1)) == 0 for c in small.cells)


def test_bench_scene_sizes():
    assert _particles(validate_scene(S.COLUMN_3D_C2)) == 262_144
    assert _particles(validate_scene(S.SANDSTORM_3D_C3)) == 4_194_304
    assert _particles(validate_scene(S.CLOUD_3D_C5)) == 2_097_152
    assert tuple(validate_scene(S.TAYLOR_GREEN_3D_C1).cells) == (64, 64, 64)
    assert np.prod(validate_scene(S.SANDSTORM_3D_C3).cells) == 512 * 256 * 128
