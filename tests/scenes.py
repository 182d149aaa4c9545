"""Scene dicts used by the parity tests and the bench.

2D scenes restate the reference's shipped scenes (pkg/scenes/*.toml) and the
2D analogs of BASELINE.json configs; 3D scenes are the
configs at test / bench sizes."""
import copy

TAYLOR_GREEN_2D = {"domain": {"cells": [64, 64], "levels": 1},
                   "fluid": {"tau0": 0.8, "init": "taylor_green", "init_u0": 0.05}}

SAND_COLLAPSE_2D = {
    "domain": {"cells": [192, 64], "levels": 1},
    "fluid": {"tau0": 1.8, "gravity": [0.0, -1e-3]},
    "boundaries": {"x_min": "wall", "x_max": "wall", "y_min": "wall", "y_max": "wall"},
    "materials": {"density_ratio": 2.0, "E": 0.08, "nu": 0.3, "friction_angle_deg": 30.0,
                  "floor_friction": 0.5},
    "particles": {"blocks": [[84.0, 2.0, 108.0, 44.0]], "per_cell": 10},
    "runtime": {"seed": 11}}

DUNE_2D = {
    "domain": {"cells": [256, 128], "levels": 3},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, 0.0]},
    "boundaries": {"x_min": {"kind": "log_inlet", "u0": 0.04, "beta": 0.35, "y0": 6.0},
                   "x_max": "outlet", "y_min": "wall", "y_max": "outlet"},
    "materials": {"density_ratio": 40.0, "E": 0.08, "nu": 0.3, "friction_angle_deg": 30.0,
                  "floor_friction": 0.5},
    "particles": {"blocks": [[64.0, 2.5, 140.0, 10.0]], "per_cell": 4},
    "runtime": {"seed": 42, "mpm_cadence": 1}}

POWDER_BOX_2D = {
    "domain": {"cells": [64, 64], "levels": 1},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -5e-5]},
    "boundaries": {"x_min": "periodic", "x_max": "periodic", "y_min": "wall", "y_max": "wall"},
    "materials": {"density_ratio": 20.0, "E": 0.08},
    "particles": {"blocks": [[24.0, 6.0, 40.0, 22.0]], "per_cell": 4},
    "powder": {"enabled": True, "entrain": 0.02, "diffusion": 0.05},
    "runtime": {"seed": 3}}

# dispersed cloud forcing per-step block churn (config 5, 2D analog)
CLOUD_2D = {
    "domain": {"cells": [128, 128], "levels": 3},
    "fluid": {"tau0": 1.8, "eps_min": 0.5},
    "materials": {"density_ratio": 10.0, "E": 0.08},
    "particles": {"blocks": [[40.0, 40.0, 56.0, 56.0], [80.0, 70.0, 92.0, 86.0]], "per_cell": 1},
    "runtime": {"seed": 9}}

# reference behaviours the default scenes never reach: the held hook at
# mpm_cadence = 2 (coupling.py:454-465), the paper-literal S rescale
# (solver.py:41-52) and average upward transfer on three levels, and the
# paper-literal powder diffusion sign (coupling.py:262-267)
DUNE_2D_CADENCE2_LITERAL = copy.deepcopy(DUNE_2D)
DUNE_2D_CADENCE2_LITERAL["runtime"]["mpm_cadence"] = 2
DUNE_2D_CADENCE2_LITERAL["fluid"]["rescale_convention"] = "paper_literal"
DUNE_2D_CADENCE2_LITERAL["fluid"]["upward_mode"] = "average"

POWDER_BOX_2D_LITERAL = copy.deepcopy(POWDER_BOX_2D)
POWDER_BOX_2D_LITERAL["powder"]["sign"] = "paper_literal"
POWDER_BOX_2D_LITERAL["runtime"]["mpm_cadence"] = 2

# ---- 3D -------------------------------------------------------------------------
COLUMN_3D_SMALL = {     # config 2 at test size
    "domain": {"cells": [32, 32, 32], "levels": 2},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -1e-4, 0.0]},
    "boundaries": {"x_min": "wall", "x_max": "wall", "y_min": "wall", "y_max": "wall",
                   "z_min": "wall", "z_max": "wall"},
    "materials": {"density_ratio": 40.0, "E": 0.08},
    "particles": {"blocks": [[12.0, 2.0, 12.0, 20.0, 18.0, 20.0]], "per_cell": 2},
    "runtime": {"seed": 5}}

DUNE_3D_SMALL = {       # config 3 at test size
    "domain": {"cells": [64, 32, 16], "levels": 2},
    "fluid": {"tau0": 1.8, "eps_min": 0.5},
    "boundaries": {"x_min": {"kind": "log_inlet", "u0": 0.04, "beta": 0.35, "y0": 6.0},
                   "x_max": "outlet", "y_min": "wall", "y_max": "outlet",
                   "z_min": "periodic", "z_max": "periodic"},
    "materials": {"density_ratio": 40.0, "E": 0.08},
    "particles": {"blocks": [[16.0, 2.0, 0.0, 36.0, 8.0, 16.0]], "per_cell": 2},
    "runtime": {"seed": 42}}

SANDSTORM_3D_SMALL = {  # config 3 (C3) at test size: three levels, inflow, z periodic
    "domain": {"cells": [64, 32, 16], "levels": 3},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -1e-4, 0.0]},
    "boundaries": {"x_min": {"kind": "log_inlet", "u0": 0.05, "beta": 0.35, "y0": 6.0},
                   "x_max": "outlet", "y_min": "wall", "y_max": "outlet",
                   "z_min": "periodic", "z_max": "periodic"},
    "materials": {"density_ratio": 40.0, "E": 0.08, "nu": 0.3, "friction_angle_deg": 30.0,
                  "floor_friction": 0.5},
    "particles": {"blocks": [[16.0, 2.0, 0.0, 44.0, 7.0, 16.0]], "per_cell": 2},
    "runtime": {"seed": 9}}

# dispersed cloud forcing per-step block churn across slab cuts (config 5 at test size)
CLOUD_3D_SMALL = {
    "domain": {"cells": [96, 32, 32], "levels": 2},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -3e-4, 0.0]},
    "boundaries": {"y_min": "wall", "y_max": "wall"},
    "materials": {"density_ratio": 10.0, "E": 0.08},
    "particles": {"blocks": [[26.0, 12.0, 8.0, 38.0, 24.0, 24.0],
                             [58.0, 14.0, 10.0, 70.0, 26.0, 22.0]], "per_cell": 1},
    "runtime": {"seed": 13}}

POWDER_3D_SMALL = {     # config 4 ingredients at test size (powder on, solids)
    "domain": {"cells": [32, 32, 16], "levels": 1},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -5e-5, 0.0]},
    "boundaries": {"y_min": "wall", "y_max": "outlet",
                   "solid_boxes": [[0.0, 0.0, 0.0, 8.0, 3.0, 16.0]]},
    "materials": {"density_ratio": 20.0, "E": 0.08},
    "particles": {"blocks": [[12.0, 6.0, 4.0, 20.0, 14.0, 12.0]], "per_cell": 2},
    "powder": {"enabled": True, "entrain": 0.02, "diffusion": 0.05},
    "runtime": {"seed": 3}}

# the paper's snow (NACC + softening law; parity unpinned):
# a softened column under strong gravity cracks within a few steps, so both
# hardening branches run
SNOW_3D_SMALL = copy.deepcopy(COLUMN_3D_SMALL)
SNOW_3D_SMALL["fluid"]["gravity"] = [0.0, -1e-3, 0.0]
SNOW_3D_SMALL["materials"].update({"model": "snow", "nacc_q0": 0.002, "nacc_alpha": 2.0})

SNOW_2D = copy.deepcopy(SAND_COLLAPSE_2D)
SNOW_2D["materials"].update({"model": "snow", "nacc_q0": 0.002, "nacc_alpha": 2.0})

# BASELINE.json configs[1]: two-level 128^3-effective column collapse in air,
# 262,144 particles
COLUMN_3D_C2 = {
    "domain": {"cells": [128, 128, 128], "levels": 2},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -1e-4, 0.0]},
    "boundaries": {"x_min": "wall", "x_max": "wall", "y_min": "wall", "y_max": "wall",
                   "z_min": "wall", "z_max": "wall"},
    "materials": {"density_ratio": 40.0, "E": 0.08, "nu": 0.3, "friction_angle_deg": 30.0,
                  "floor_friction": 0.5},
    "particles": {"blocks": [[48.0, 4.0, 48.0, 80.0, 68.0, 80.0]], "per_cell": 4},
    "runtime": {"seed": 5, "dtype": "f32"}}

# BASELINE.json configs[2]: three-level 512x256x128-effective
# sand migration under a log-law wind inflow; dune block [96,352]x[2,18]x[0,128]
# at 8 per cell = 4,194,304 particles, seed 42
SANDSTORM_3D_C3 = {
    "domain": {"cells": [512, 256, 128], "levels": 3},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -1e-4, 0.0]},
    "boundaries": {"x_min": {"kind": "log_inlet", "u0": 0.04, "beta": 0.35, "y0": 6.0},
                   "x_max": "outlet", "y_min": "wall", "y_max": "outlet",
                   "z_min": "periodic", "z_max": "periodic"},
    "materials": {"density_ratio": 40.0, "E": 0.08, "nu": 0.3, "friction_angle_deg": 30.0,
                  "floor_friction": 0.5},
    "particles": {"blocks": [[96.0, 2.0, 0.0, 352.0, 18.0, 128.0]], "per_cell": 8},
    "runtime": {"seed": 42, "dtype": "f32"}}

# BASELINE.json configs[4]: dynamic-refinement stress — a
# dispersed cloud in a periodic 256^3 box, L = 3, 2,097,152 particles (a 128^3
# block at 1 per cell) with Gaussian velocities sigma 0.1 clipped at 0.45
# (set by cloud_velocities), density ratio 10
CLOUD_3D_C5 = {
    "domain": {"cells": [256, 256, 256], "levels": 3},
    "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, 0.0, 0.0]},
    "materials": {"density_ratio": 10.0, "E": 0.08},
    "particles": {"blocks": [[64.0, 64.0, 64.0, 192.0, 192.0, 192.0]], "per_cell": 1},
    "runtime": {"seed": 17, "dtype": "f32"}}


def cloud_velocities(sim, sigma=0.1, clip=0.45, seed=17):
    """C5 initial particle velocities: N(0, sigma^2) per component, clipped."""
    import numpy as np
    rng = np.random.default_rng(seed)
    v = np.clip(rng.normal(0.0, sigma, (len(sim.particles), sim.d)), -clip, clip)
    sim.particles.v = v


def terrain_heightfield(cells, path, base=1.0, amp=2.5):
    """Synthetic terrain under the C4 slab: heights in finest cells over
    (x, z), a ramp falling along +x with a cross-slope undulation; every height
    stays below the slab floor (y = 4), so no particle starts inside a solid.
    Deterministic, written as an .npy for ``boundaries.heightfield``."""
    import numpy as np
    nx, nz = cells[0], cells[2]
    x = (np.arange(nx) + 0.5) / nx
    z = (np.arange(nz) + 0.5) / nz
    h = base + amp * (0.6 * (1.0 - x)[:, None] + 0.4 * (0.5 + 0.5 * np.cos(2 * np.pi * z))[None, :])
    np.save(path, np.minimum(h, 3.5).astype(np.float64))
    return path


def slope_heightfield(cells, path, scale=1, h0=150.0, amp=3.0):
    """A mountain flank for C4: heights in finest cells over (x, z) falling
    along +x from ~h0 to ~1 (x^1.5 profile, span > 100 cells across the slab)
    with a cross-slope undulation of +-amp/2; ``scale`` divides the full-scene
    coordinates and heights (the CPU sample).  Written as an .npy."""
    import numpy as np
    nx, nz = cells[0], cells[2]
    xs = (np.arange(nx) + 0.5) * scale / 1536.0
    zs = (np.arange(nz) + 0.5) * scale / 384.0
    h = h0 * (1.0 - xs)[:, None] ** 1.5 + amp * (0.5 + 0.5 * np.cos(2 * np.pi * zs))[None, :] + 1.0
    np.save(path, (h / scale).astype(np.float64))
    return path


def avalanche_c4(heightfield_path, scale=1):
    """BASELINE.json configs[3]: four-level
    1536x768x384-effective snow avalanche with powder cloud on a mountain
    flank — a floor wall under a heightmap falling ~110 cells along x
    (solids), outlets elsewhere, g along -y, a snow slab 24 cells thick laid
    on the slope as 16 steps of 64 cells ([256, 1280) x [50, 334) in x, z; each
    step starts one cell above the highest terrain under it),
    1024 x 24 x 284 = 6,979,584 cells at 8 per cell = 55,836,672 particles of
    NACC snow with the paper's softening law (the reference
    has no snow model, so this part is parity-unpinned), powder entrainment on.
    ``scale`` > 1 divides every extent (the bounded CPU sample)."""
    import math
    import numpy as np
    s = float(scale)
    cells = [1536 // scale, 768 // scale, 384 // scale]
    slope_heightfield(cells, heightfield_path, scale)
    hm = np.load(heightfield_path)
    blocks = []
    for k in range(16):
        x0, x1 = (256.0 + 64.0 * k) / s, (256.0 + 64.0 * (k + 1)) / s
        top = float(hm[int(x0):int(math.ceil(x1)), :].max())
        y0 = math.ceil(top) + 1.0
        blocks.append([x0, y0, 50.0 / s, x1, y0 + 24.0 / s, 334.0 / s])
    return {
        "domain": {"cells": cells, "levels": 4},
        "fluid": {"tau0": 1.8, "eps_min": 0.5, "gravity": [0.0, -1e-4, 0.0]},
        "boundaries": {"x_min": "outlet", "x_max": "outlet", "y_min": "wall", "y_max": "outlet",
                       "z_min": "outlet", "z_max": "outlet",
                       "heightfield": heightfield_path},
        "materials": {"density_ratio": 40.0, "E": 0.08, "nu": 0.3, "friction_angle_deg": 30.0,
                      "floor_friction": 0.5, "model": "snow", "nacc_q0": 0.02,
                      "nacc_alpha": 0.5},
        "particles": {"blocks": blocks, "per_cell": 8},
        "powder": {"enabled": True, "entrain": 0.02, "diffusion": 0.05},
        "runtime": {"seed": 7, "dtype": "f32"}}


# configs[0]: single-level 64^3 periodic Taylor-Green
TAYLOR_GREEN_3D_C1 = {"domain": {"cells": [64, 64, 64], "levels": 1},
                      "fluid": {"tau0": 0.8, "init": "taylor_green", "init_u0": 0.05},
                      "runtime": {"dtype": "f32"}}


def scene(d, **over):
    s = copy.deepcopy(d)
    for k, v in over.items():
        tbl, key = k.split("__")
        s.setdefault(tbl, {})[key] = v
    return s
