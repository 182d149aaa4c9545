"""Multi-level moment-space LBM (oracle, fp64, d = 2 or 3).

Restates ``pkg/src/mlbm/solver.py``:
  * tau / S rescaling laws              solver.py:34-67, LevelParams :70-91
  * boundary spec + solid raster        solver.py:116-171 (3D: six faces, the
    log inlet stays on x_min with y vertical; an optional heightmap makes
    cells with corner y < h(x[, z]) solid, config.py:161-165's heightfield)
  * per-level gather / bounce-back tables solver.py:177-274
  * stream / collide / boundary kernels  solver.py:336-481
  * downward / upward transfers          solver.py:492-560
  * Alg. 1 linearised schedule, run_cycle solver.py:564-649
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .grid import (BORDER, LEAF, DivergenceError, PingPongPair, Topology,
                   TopologyError, buffer_roles, classify_interfaces,
                   field_names)
from .lattice import CS2, H3_XYZ_HERMITE, Lattice, h2, lattice_for, \
    moments_from_f, reconstruct_dir, s_pairs, s_names

RESCALE_DERIVED = "derived"
RESCALE_PAPER_LITERAL = "paper_literal"


def rescale_tau(tau, k):
    return tau / 2.0 ** k + (2.0 ** k - 1.0) / 2.0 ** (k + 1)


def kappa_up(tf, tc, conv):
    if conv == RESCALE_DERIVED:
        return 2.0 * tc / tf
    if conv == RESCALE_PAPER_LITERAL:
        return tc / (2.0 * tf)
    raise ValueError(conv)


def kappa_down(tf, tc, conv):
    if conv == RESCALE_DERIVED:
        return tf / (2.0 * tc)
    if conv == RESCALE_PAPER_LITERAL:
        return 2.0 * tc / tf
    raise ValueError(conv)


def rescale_s(s, u, kappa):
    """S' = kappa (S - uu) + uu over dict (a,b)->array (solver.py:55-67)."""
    out = {}
    for (a, b), v in s.items():
        eq = u[a] * u[b]
        out[(a, b)] = kappa * (v - eq) + eq
    return out


@dataclass
class LevelParams:
    levels: int
    tau0: float
    taus: list = field(default_factory=list)

    def __post_init__(self):
        if self.tau0 <= 0.5:
            raise ValueError("tau0 must exceed 1/2")
        self.taus = [rescale_tau(self.tau0, l) for l in range(self.levels)]

    def nu(self, level):
        return CS2 * (self.taus[level] - 0.5)


@dataclass
class SolverParams:
    levels: int
    rho0: float = 1.0
    gravity: tuple = None
    eps_min: float = 0.3
    mpm_cadence: int = 1
    rescale_convention: str = RESCALE_DERIVED
    upward_mode: str = "coincident"
    h3_xyz: float = H3_XYZ_HERMITE


@dataclass
class LogInlet:
    u0: float
    beta: float
    y0: float


def face_names(d):
    return [a + s for a in "xyz"[:d] for s in ("_min", "_max")]


@dataclass
class BoundarySpec:
    d: int = 2
    faces: dict = None
    solid_boxes: list = field(default_factory=list)   # (lo..., hi...)
    heightmap: np.ndarray | None = None               # finest (x[, z])

    def __post_init__(self):
        if self.faces is None:
            self.faces = {f: "periodic" for f in face_names(self.d)}

    def periodic_axes(self):
        return tuple(self.faces[a + "_min"] == "periodic"
                     for a in "xyz"[:self.d])


def solid_at(spec: BoundarySpec, g):
    """Solid test at finest-unit corner coords g: (n, d) (solver.py:159-171)."""
    out = np.zeros(len(g), dtype=bool)
    d = spec.d
    for box in spec.solid_boxes:
        lo, hi = box[:d], box[d:]
        m = np.ones(len(g), dtype=bool)
        for a in range(d):
            m &= (g[:, a] >= lo[a]) & (g[:, a] < hi[a])
        out |= m
    if spec.heightmap is not None:
        h = spec.heightmap
        if d == 2:
            hx = h[np.clip(g[:, 0], 0, len(h) - 1)]
        else:
            hx = h[np.clip(g[:, 0], 0, h.shape[0] - 1),
                   np.clip(g[:, 2], 0, h.shape[1] - 1)]
        out |= (hx > 0) & (g[:, 1] < hx)
    return out


class LevelTables:
    """solver.py:177-274, generic over d."""

    def __init__(self, topo: Topology, spec: BoundarySpec, sets, lat: Lattice,
                 level):
        d = topo.d
        cmap = topo.cell_map(level)
        dims = topo.cells_dims(level)
        coords = topo.cell_coords(level)
        n = len(coords)
        per = topo.periodic
        scale = 1 << level
        self.solid_flat = solid_at(spec, coords * scale)

        bc = np.zeros(n, dtype=bool)
        self.outlets = []
        self.inlet = None
        for face in face_names(d):
            cond = spec.faces[face]
            axis = "xyz".index(face[0])
            side = 0 if face.endswith("_min") else 1
            if isinstance(cond, str) and cond in ("periodic", "wall"):
                continue
            edge = 0 if side == 0 else dims[axis] - 1
            sel = coords[:, axis] == edge
            if not sel.any():
                continue
            cells = np.nonzero(sel)[0]
            bc[cells] = True
            inner_c = coords[cells].copy()
            inner_c[:, axis] += 1 if side == 0 else -1
            inner = cmap[tuple(inner_c.T)]
            if (inner < 0).any():
                raise TopologyError("boundary cell lacks inner neighbor")
            if cond == "outlet":
                self.outlets.append((cells, inner, axis,
                                     -1.0 if side == 0 else 1.0))
            else:
                ypos = coords[cells, 1].astype(float) * scale
                self.inlet = (cells, ypos, cond)

        ghost = np.zeros(n, dtype=bool)
        if level in sets.downs:
            ghost[sets.downs[level][0]] = True
        if level in sets.ups:
            ghost[sets.ups[level][0]] = True
        self.active = ~(ghost | bc | self.solid_flat)
        self.active_idx = np.nonzero(self.active)[0]
        self.inactive_idx = np.nonzero(~self.active)[0]

        q = lat.q
        self.src = np.empty((q, n), dtype=np.int64)
        self.bb = np.zeros((q, n), dtype=bool)
        for i in range(q):
            s = coords - lat.c[i][None, :]
            oob = np.zeros(n, dtype=bool)
            wallbb = np.zeros(n, dtype=bool)
            for a in range(d):
                if per[a]:
                    s[:, a] %= dims[a]
                else:
                    lo = s[:, a] < 0
                    hi = s[:, a] >= dims[a]
                    oob |= lo | hi
                    if spec.faces["xyz"[a] + "_min"] == "wall":
                        wallbb |= lo
                    if spec.faces["xyz"[a] + "_max"] == "wall":
                        wallbb |= hi
            s2 = np.stack([s[:, a].clip(0, dims[a] - 1) for a in range(d)], 1)
            flat = cmap[tuple(s2.T)]
            is_solid = solid_at(spec, s2 * scale)
            bb = (~oob & is_solid) | wallbb
            missing = oob | (flat < 0)
            self.bb[i] = bb
            self.src[i] = np.where(bb | missing, np.arange(n), flat)
            if (missing & ~bb & self.active).any():
                raise TopologyError(
                    f"active cell at level {level} has no source for dir {i}")
        self.coords = coords


class Solver:
    """MultiLevelSolver restated (solver.py:277-612)."""

    def __init__(self, topo: Topology, pair: PingPongPair,
                 params: SolverParams, lp: LevelParams,
                 spec: BoundarySpec | None = None):
        self.topo = topo
        self.d = topo.d
        self.pair = pair
        self.params = params
        if params.gravity is None:
            params.gravity = (0.0,) * self.d
        self.lp = lp
        self.spec = spec or BoundarySpec(d=self.d)
        self.lat = lattice_for(self.d, params.h3_xyz)
        self.k = [0] * topo.levels
        self._ver = -1
        self.schedule = build_schedule(topo.levels)
        self.refresh()

    def refresh(self):
        if self._ver == self.topo.version:
            return
        self.sets = classify_interfaces(self.topo)
        self.tables = {}
        for l in range(self.topo.levels):
            if self.topo.n_tiles(l):
                self.tables[l] = LevelTables(self.topo, self.spec, self.sets,
                                             self.lat, l)
        self._ver = self.topo.version

    def arrays(self, tree, level):
        return self.pair.trees[tree].levels[level]

    def roles(self, level):
        return buffer_roles(level, self.k[level] & 1)

    def last_roles(self, level):
        return buffer_roles(level, (self.k[level] - 1) & 1)

    # kernels ------------------------------------------------------------------
    def _unpack(self, a, idx=None):
        d = self.d
        ax = "xyz"[:d]
        g = (lambda v: v) if idx is None else (lambda v: v[idx])
        rho = g(a["rho"])
        u = [g(a["u" + x]) for x in ax]
        s = {p: g(a[nm]) for p, nm in zip(s_pairs(d), s_names(d))}
        return rho, u, s

    def stream_kernel(self, level, src_a, dst):
        if not len(dst["rho"]):
            return
        t = self.tables[level]
        lat = self.lat
        fs = []
        for i in range(lat.q):
            idx = t.src[i]
            rho, u, s = self._unpack(src_a, idx)
            fi = reconstruct_dir(lat, i, rho, u, s)
            if t.bb[i].any():
                sel = t.bb[i]
                rho2, u2, s2 = self._unpack(src_a, sel)
                fi = np.array(fi, dtype=float)
                fi[sel] = reconstruct_dir(lat, int(lat.opp[i]), rho2, u2, s2)
            fs.append(fi)
        rho, m, pi = moments_from_f(lat, fs)
        ax = "xyz"[:self.d]
        dst["rho"][:] = rho
        for a in range(self.d):
            dst["u" + ax[a]][:] = m[a]
        for p, nm in zip(s_pairs(self.d), s_names(self.d)):
            dst[nm][:] = pi[p]
        dst["eps"][:] = src_a["eps"]
        dst["phi"][:] = src_a["phi"]

    def collide_kernel(self, level, src_a, dst, force=None, tau_eff=None):
        if not len(dst["rho"]):
            return
        t = self.tables[level]
        d = self.d
        ax = "xyz"[:d]
        rho = dst["rho"]
        ra = rho[t.active_idx]
        if (~np.isfinite(ra) | (ra <= 0.0)).any():
            raise DivergenceError(f"level {level}: non-physical density",
                                  level=level)
        if force is None:
            sc = float(1 << level)
            F = [rho * (self.params.gravity[a] * sc) for a in range(d)]
        else:
            F = list(force)
        tau = self.lp.taus[level] if tau_eff is None else tau_eff
        inv_rho = 1.0 / rho
        us = [(dst["u" + ax[a]] + 0.5 * F[a]) * inv_rho for a in range(d)]
        inv_tau = 1.0 / tau
        fcoef = (2.0 * tau - 1.0) / (2.0 * tau) * inv_rho
        news = {}
        for (a, b), nm in zip(s_pairs(d), s_names(d)):
            ss = dst[nm] * inv_rho
            news[nm] = (1.0 - inv_tau) * ss + inv_tau * us[a] * us[b] \
                + fcoef * (F[a] * us[b] + F[b] * us[a])
        for a in range(d):
            dst["u" + ax[a]][:] = us[a] + 0.5 * F[a] * inv_rho
        for nm, v in news.items():
            dst[nm][:] = v
        idx = t.inactive_idx
        if idx.size:
            for nm in ["rho"] + ["u" + x for x in ax] + s_names(d) + \
                    ["eps", "phi"]:
                dst[nm][idx] = src_a[nm][idx]
        bad = np.zeros(len(t.active_idx), dtype=bool)
        for a in range(d):
            bad |= ~np.isfinite(dst["u" + ax[a]][t.active_idx])
        if bad.any():
            raise DivergenceError(f"level {level}: non-finite velocity",
                                  level=level)

    def boundary_kernel(self, level, dst):
        if not len(dst["rho"]):
            return
        t = self.tables[level]
        d = self.d
        ax = "xyz"[:d]
        names = ["rho"] + ["u" + x for x in ax] + s_names(d)
        for cells, inner, axis, sign in t.outlets:
            un = np.minimum(np.maximum(sign * dst["u" + ax[axis]][inner], 0.0),
                            1.0)
            for nm in names:
                v = dst[nm]
                v[cells] = v[cells] - un * (v[cells] - v[inner])
        if t.inlet is not None:
            cells, ypos, cond = t.inlet
            arg = 1.0 + cond.beta * (ypos - cond.y0)
            uxv = np.where(ypos >= cond.y0,
                           cond.u0 * np.log(np.maximum(arg, 1.0)), 0.0)
            dst["rho"][cells] = self.params.rho0
            dst["ux"][cells] = uxv
            for x in ax[1:]:
                dst["u" + x][cells] = 0.0
            for (a, b), nm in zip(s_pairs(d), s_names(d)):
                dst[nm][cells] = uxv * uxv if (a == 0 and b == 0) else 0.0

    def downward_kernel(self, level, step, olda, newa, dst):
        if level not in self.sets.downs:
            return
        tgt, src, w = self.sets.downs[level]
        src = src.clip(min=0)
        d = self.d
        ax = "xyz"[:d]
        vals = {}
        for nm in ["rho"] + ["u" + x for x in ax] + s_names(d) + ["eps", "phi"]:
            v = olda[nm][src]
            if step == 2:
                v = 0.5 * (v + newa[nm][src])
            vals[nm] = (v * w).sum(axis=1)
        kap = kappa_down(self.lp.taus[level], self.lp.taus[level + 1],
                         self.params.rescale_convention)
        u = [vals["u" + x] for x in ax]
        s = rescale_s({p: vals[nm] for p, nm in zip(s_pairs(d), s_names(d))},
                      u, kap)
        for nm in vals:
            dst[nm][tgt] = vals[nm]
        for p, nm in zip(s_pairs(d), s_names(d)):
            dst[nm][tgt] = s[p]

    def upward_kernel(self, level, fine, dst):
        coarse = level + 1
        if coarse not in self.sets.ups:
            return
        tgt, src, src_all = self.sets.ups[coarse]
        d = self.d
        ax = "xyz"[:d]
        if self.params.upward_mode == "average":
            def fetch(nm):
                return fine[nm][src_all].mean(axis=1)
        else:
            def fetch(nm):
                return fine[nm][src]
        u = [fetch("u" + x) for x in ax]
        kap = kappa_up(self.lp.taus[level], self.lp.taus[coarse],
                       self.params.rescale_convention)
        s = rescale_s({p: fetch(nm) for p, nm in zip(s_pairs(d), s_names(d))},
                      u, kap)
        dst["rho"][tgt] = fetch("rho")
        for a in range(d):
            dst["u" + ax[a]][tgt] = u[a]
        for p, nm in zip(s_pairs(d), s_names(d)):
            dst[nm][tgt] = s[p]
        dst["eps"][tgt] = fetch("eps")
        dst["phi"][tgt] = fetch("phi")

    # orchestration ------------------------------------------------------------
    def stream(self, level):
        r, w = self.roles(level)
        self.stream_kernel(level, self.arrays(r, level), self.arrays(w, level))

    def collide(self, level, force=None, tau_eff=None):
        r, w = self.roles(level)
        self.collide_kernel(level, self.arrays(r, level),
                            self.arrays(w, level), force, tau_eff)

    def apply_boundaries(self, level):
        _, w = self.roles(level)
        self.boundary_kernel(level, self.arrays(w, level))

    def stream_collide(self, level):
        self.stream(level)
        self.collide(level)
        self.apply_boundaries(level)
        self.k[level] += 1

    def downward_transfer(self, level, step):
        c = level + 1
        old_t, new_t = self.last_roles(c)
        r, _ = self.roles(level)
        self.downward_kernel(level, step, self.arrays(old_t, c),
                             self.arrays(new_t, c), self.arrays(r, level))

    def upward_transfer(self, level):
        c = level + 1
        _, fw = self.last_roles(level)
        _, cw = self.last_roles(c)
        self.upward_kernel(level, self.arrays(fw, level), self.arrays(cw, c))

    def run_cycle(self, cycle, hook=None):
        self.refresh()
        for kind, level, s in cycle["pre"]:
            if kind == "down":
                self.downward_transfer(level, s)
            elif kind == "sc":
                self.stream_collide(level)
            else:
                self.upward_transfer(level)
        s0 = cycle["s0"]
        if self.topo.levels > 1:
            self.downward_transfer(0, s0)
        self.stream(0)
        force, tau_eff = None, None
        if hook is not None:
            out = hook(self)
            if out is not None:
                force, tau_eff = out
        self.collide(0, force, tau_eff)
        self.apply_boundaries(0)
        self.k[0] += 1
        if self.topo.levels > 1 and s0 == 2:
            self.upward_transfer(0)
        if cycle["last"]:
            self.pair.bounce += 1

    def advance_bounce(self, hook=None):
        for cyc in self.schedule:
            self.run_cycle(cyc, hook)

    def run_finest_steps(self, n, hook=None):
        per = len(self.schedule)
        i = self.k[0] % per
        for _ in range(n):
            self.run_cycle(self.schedule[i], hook)
            i = (i + 1) % per


def build_schedule(levels):
    """Linearised Alg. 1 recursion (solver.py:615-649)."""
    ops = []

    def rec(level, s):
        if level < levels - 1:
            ops.append(("down", level, s))
        ops.append(("sc", level, s))
        if level < levels - 1 and s == 2:
            ops.append(("up", level, s))
        if level > 0:
            rec(level - 1, 1)
            rec(level - 1, 2)

    rec(levels - 1, 1)
    cycles, pre = [], []
    for kind, level, s in ops:
        if level == 0 and kind in ("down", "up"):
            continue
        if level == 0 and kind == "sc":
            cycles.append({"pre": pre, "s0": s, "last": False})
            pre = []
        else:
            pre.append((kind, level, s))
    cycles[-1]["last"] = True
    return cycles


def set_fields(topo, pair, fn):
    """cases.py:40-51: write fn(pos (n,d) finest units, level) into both trees."""
    for l in range(topo.levels):
        if not topo.n_tiles(l):
            continue
        pos = topo.cell_coords(l) * float(1 << l)
        vals = fn(pos, l)
        for tree in pair.trees:
            for nm, v in vals.items():
                tree.levels[l][nm][:] = v
