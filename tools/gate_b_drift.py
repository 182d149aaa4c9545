"""Gate-B drift curve: fp32 device vs fp64 oracle, relative L2 of drho, u, S
(every level), particle v and x - x0 after each of N = 1..20 coupled steps.

  python tools/gate_b_drift.py [steps] > profiles/rN_gate_b_drift.txt
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import scenes as S  # noqa: E402
from helpers import gate_b_metrics  # noqa: E402
from oracle import scene as OS  # noqa: E402
from paper_2603_14982_b200.harness import build_scene, validate_scene  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["column", "sandstorm"]
    table = {"column": S.COLUMN_3D_SMALL, "sandstorm": S.SANDSTORM_3D_SMALL,
             "sand_collapse_2d": S.SAND_COLLAPSE_2D, "dune_2d": S.DUNE_2D}
    for name in names:
        cfg = validate_scene(S.scene(table[name], runtime__dtype="f32"))
        dsim = build_scene(cfg)
        osim = OS.build_scene(cfg.raw, heightmap=cfg.heightmap())
        ox0 = osim.p.x.copy()
        dx0 = dsim.particles.x.cpu().numpy().copy()
        print(f"# {name}: fp32 device vs fp64 oracle, relative L2 after N steps")
        print(f"{'N':>3} {'drho':>10} {'u':>10} {'S':>10} {'v':>10} {'x-x0':>10}")
        for n in range(1, steps + 1):
            osim.step()
            dsim.step()
            m = gate_b_metrics(osim, dsim, ox0, dx0)
            print(f"{n:>3} {m['drho']:10.3e} {m['u']:10.3e} {m['S']:10.3e} "
                  f"{m.get('v', 0):10.3e} {m.get('x-x0', 0):10.3e}", flush=True)


if __name__ == "__main__":
    main()
