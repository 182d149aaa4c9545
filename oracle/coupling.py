"""Fluid-sediment exchange and the coupled step (oracle, d = 2 or 3).

Restates ``pkg/src/mlbm/coupling.py``:
  * rasterize_fractions (eta, mass, momentum, area; eps clamp) coupling.py:96-131
    (3D cross-section pi (3V/4pi)^(2/3); 2D 2 sqrt(V/pi))
  * Di Felice drag                                             coupling.py:134-156
  * grad eps (central, missing -> own) / mixture force          coupling.py:159-197
  * renormalised multilinear sampling                           coupling.py:200-227
  * powder transport (RK3 backtrace, (2d+1)-point Laplacian)    coupling.py:230-272
  * entrainment source                                           coupling.py:275-322
  * drag limiter, exchange, held hook, step, powder cycle,
    diagnostics                                                  coupling.py:337-538
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import mpm
from .adapt import RefineDriver
from .grid import Topology
from .lbm import Solver


@dataclass
class DragParams:
    d_p: float | None = None
    re_min: float = 0.01


@dataclass
class PowderParams:
    entrain: float = 0.0
    diffusion: float = 0.05
    sign: float = 1.0
    eta_surface: float = 0.6


class Fields:
    pass


def particle_area(V0, d):
    if d == 2:
        return 2.0 * np.sqrt(V0 / np.pi)
    return np.pi * (3.0 * V0 / (4.0 * np.pi)) ** (2.0 / 3.0)


def particle_diameter(V0, d):
    if d == 2:
        return 2.0 * np.sqrt(V0 / np.pi)
    return 2.0 * (3.0 * V0 / (4.0 * np.pi)) ** (1.0 / 3.0)


def rasterize_fractions(p, topo: Topology, phi, eps_min, st=None):
    d = topo.d
    n = topo.cell_count(0)
    eta = np.zeros(n)
    mass = np.zeros(n)
    mom = np.zeros((n, d))
    area = np.zeros(n)
    if len(p):
        idx, w, _, _ = st if st is not None else mpm.stencil(p.x, topo)
        flat = idx.ravel()
        eta += np.bincount(flat, weights=(w * p.V0[:, None]).ravel(),
                           minlength=n)
        wm = w * p.m[:, None]
        mass += np.bincount(flat, weights=wm.ravel(), minlength=n)
        for a in range(d):
            mom[:, a] += np.bincount(flat, weights=(wm * p.v[:, a:a + 1])
                                     .ravel(), minlength=n)
        ap = particle_area(p.V0, d)
        area += np.bincount(flat, weights=(w * ap[:, None]).ravel(),
                            minlength=n)
    massive = mass > 0
    v = np.zeros((n, d))
    v[massive] = mom[massive] / mass[massive, None]
    eta_eff = np.maximum(eta - phi, 0.0)
    f = Fields()
    f.eps = np.clip(1.0 - eta_eff - phi, eps_min, 1.0)
    f.eta = eta_eff
    f.v = v
    f.area = area
    f.mass = mass
    f.fs = np.zeros((n, d))
    f.force = np.zeros((n, d))
    f.grad_term = np.zeros((n, d))
    f.rel = None
    return f


def difelice_drag(f, rho, u, nu, params: DragParams, d_p):
    rel = u - f.v
    f.rel = rel
    speed = np.sqrt((rel ** 2).sum(axis=1)) if rel.shape[1] == 3 else \
        np.hypot(rel[:, 0], rel[:, 1])
    act = (f.area > 0) & (speed > 0)
    fs = np.zeros_like(rel)
    if act.any():
        eps = f.eps[act]
        sp = speed[act]
        re = np.maximum(eps * sp * d_p / nu, params.re_min)
        cd = (0.63 + 4.8 / np.sqrt(re)) ** 2
        chi = 3.7 - 0.65 * np.exp(-0.5 * (1.5 - np.log10(re)) ** 2)
        coef = 0.5 * cd * eps ** (-chi) * rho[act] * f.area[act] * sp
        fs[act] = coef[:, None] * rel[act]
    f.fs = fs
    return fs


def _norm(v):
    return np.sqrt((v ** 2).sum(axis=1)) if v.shape[1] == 3 else \
        np.hypot(v[:, 0], v[:, 1])


def limit_drag(f, rho, u, dt, beta_exact=0.5):
    mag = _norm(f.fs)
    hot = mag > 0
    if not hot.any():
        return
    wrel = _norm(u - f.v)[hot]
    inv_mass = 1.0 / rho[hot] + 1.0 / np.maximum(f.mass[hot], 1e-12)
    beta = mag[hot] * dt * inv_mass / np.maximum(wrel, 1e-14)
    over = np.maximum(beta - beta_exact, 0.0)
    real = np.minimum(beta, beta_exact) + over / (1.0 + over)
    f.fs[hot] *= (real / np.maximum(beta, 1e-14))[:, None]


def _axis_neighbor(topo, axis, sign):
    cmap = topo.cell_map(0)
    dims = topo.cells_dims(0)
    nb = topo.cell_coords(0).copy()
    nb[:, axis] += sign
    if topo.periodic[axis]:
        nb[:, axis] %= dims[axis]
    else:
        nb[:, axis] = nb[:, axis].clip(0, dims[axis] - 1)
    return cmap[tuple(nb.T)]


def grad_eps(eps, topo):
    own = np.arange(len(eps))
    out = np.empty((len(eps), topo.d))
    for a in range(topo.d):
        fp = _axis_neighbor(topo, a, 1)
        fm = _axis_neighbor(topo, a, -1)
        plus = eps[np.where(fp >= 0, fp, own)]
        minus = eps[np.where(fm >= 0, fm, own)]
        out[:, a] = 0.5 * (plus - minus)
    return out


def mixture_force(f, rho, topo, gravity, rho0=1.0):
    g = grad_eps(f.eps, topo)
    f.grad_term = ((rho - rho0) / f.eps)[:, None] * g
    force = f.grad_term.copy()
    for a in range(topo.d):
        force[:, a] += rho * gravity[a] - f.fs[:, a]
    f.force = force
    return force


def sample_linear(values, pos, topo):
    d = topo.d
    cmap = topo.cell_map(0)
    dims = topo.cells_dims(0)
    base = np.floor(pos).astype(np.int64)
    frac = pos - base
    acc = np.zeros(len(pos))
    ws = np.zeros(len(pos))
    for k in range(1 << d):
        cc = []
        w = np.ones(len(pos))
        for a in range(d):
            o = (k >> a) & 1
            ca = base[:, a] + o
            ca = ca % dims[a] if topo.periodic[a] else ca.clip(0, dims[a] - 1)
            cc.append(ca)
            w = w * (frac[:, a] if o else 1.0 - frac[:, a])
        flat = cmap[tuple(cc)]
        w = w * (flat >= 0)
        acc += w * values[flat.clip(min=0)]
        ws += w
    ok = ws > 0
    acc[ok] /= ws[ok]
    return acc


def powder_step(phi, u, topo, params: PowderParams, dt, source=None):
    d = topo.d
    coords = topo.cell_coords(0).astype(float)

    def vel(pos):
        return np.stack([sample_linear(u[a], pos, topo) for a in range(d)], 1)
    k1 = vel(coords)
    k2 = vel(coords - 0.5 * dt * k1)
    k3 = vel(coords - 0.75 * dt * k2)
    back = coords - dt * (2.0 * k1 + 3.0 * k2 + 4.0 * k3) / 9.0
    adv = sample_linear(phi, back, topo)
    own = np.arange(len(phi))
    lap = -2.0 * d * adv
    for a in range(d):
        for sgn in (1, -1):
            fl = _axis_neighbor(topo, a, sgn)
            lap += adv[np.where(fl >= 0, fl, own)]
    out = adv + params.sign * params.diffusion * dt * lap
    if source is not None:
        out = out + dt * source
    return out


def entrainment_rate(f, p, topo, mat, params: PowderParams):
    d = topo.d
    n = topo.cell_count(0)
    q = np.zeros(n)
    if params.entrain <= 0.0 or not len(p):
        return q
    tau = mpm.kirchhoff(p, mat)
    idx, w, _, _ = mpm.stencil(p.x, topo)
    wv = w * p.V0[:, None]
    flat = idx.ravel()
    sig = np.zeros((n, d, d))
    for a in range(d):
        for b in range(a, d):
            sig[:, a, b] = np.bincount(
                flat, weights=(wv * tau[:, a, b, None]).ravel(), minlength=n)
            sig[:, b, a] = sig[:, a, b]
    speed = _norm(f.v)
    eta = f.eta
    has_empty = np.zeros(n, dtype=bool)
    for a in range(d):
        for sgn in (1, -1):
            fl = _axis_neighbor(topo, a, sgn)
            has_empty |= (fl < 0) | (eta[fl.clip(min=0)] < 1e-3)
    surf = (eta > 0.0) & (eta < params.eta_surface) & has_empty & (speed > 0.0)
    if surf.any():
        v = f.v[surf]
        vsv = np.einsum("na,nab,nb->n", v, sig[surf], v)
        q[surf] = params.entrain * np.abs(vsv) / speed[surf]
    return q


class CoupledSim:
    def __init__(self, solver: Solver, particles, material=None,
                 sediment_gravity=None, drag=None, powder=None, adaptor=None,
                 static_tiles=None, unit_dt=1.0):
        self.solver = solver
        self.topo = solver.topo
        self.d = self.topo.d
        self.pair = solver.pair
        self.p = particles if particles is not None else \
            mpm.Particles(0, self.d)
        self.mat = material or mpm.SandMaterial()
        self.drag = drag or DragParams()
        self.powder = powder
        self.adaptor = adaptor
        self.static_tiles = static_tiles
        self.unit_dt = unit_dt
        self.g_s = np.asarray(sediment_gravity if sediment_gravity is not None
                              else solver.params.gravity, dtype=float)
        self.grid = mpm.MpmGrid(self.topo, solver.spec)
        self.cadence = solver.params.mpm_cadence
        self.step_count = 0
        self.diagnostics = []
        self.cfl_flags = 0
        self.clamped = 0
        self.last_fields = None
        if self.drag.d_p is None and len(self.p):
            self.drag.d_p = float(particle_diameter(self.p.V0.mean(), self.d))

    @property
    def coupling_active(self):
        return len(self.p) > 0

    def _exchange(self, sv):
        r, w = sv.roles(0)
        dst = sv.arrays(w, 0)
        src = sv.arrays(r, 0)
        ax = "xyz"[:self.d]
        rho = dst["rho"]
        u = np.stack([dst["u" + x] / rho for x in ax], axis=1)
        st = mpm.stencil(self.p.x, self.topo)
        f = rasterize_fractions(self.p, self.topo, src["phi"],
                                sv.params.eps_min, st=st)
        difelice_drag(f, rho, u, sv.lp.nu(0), self.drag, self.drag.d_p or 1.0)
        limit_drag(f, rho, u, float(self.cadence))
        mixture_force(f, rho, self.topo, sv.params.gravity, sv.params.rho0)
        self.last_fields = f
        for tree in self.pair.trees:
            arr = tree.levels[0]
            arr["eps"][:] = f.eps
            for a, x in enumerate(ax):
                arr["f" + x][:] = f.force[:, a]
        dt = float(self.cadence)
        self.grid.drag = f.fs
        self.clamped += mpm.mpm_step(self.p, self.grid, dt, self.g_s, self.mat,
                                     drag=f.fs, st=st)
        if not mpm.cfl_check(self.p, dt):
            self.cfl_flags += 1
        return [f.force[:, a] for a in range(self.d)], f.eps * sv.lp.taus[0]

    def step(self):
        sv = self.solver
        cyc = sv.schedule[sv.k[0] % len(sv.schedule)]
        is_mpm = self.coupling_active and self.step_count % self.cadence == 0
        if is_mpm:
            sv.run_cycle(cyc, hook=self._exchange)
        elif self.coupling_active:
            def held(s):
                _, w = s.roles(0)
                dst = s.arrays(w, 0)
                return ([dst["f" + x] for x in "xyz"[:self.d]],
                        dst["eps"] * s.lp.taus[0])
            sv.run_cycle(cyc, hook=held)
        else:
            sv.run_cycle(cyc)
        if self.powder is not None:
            self._powder_cycle(is_mpm)
        if self.adaptor is not None and self.coupling_active and \
                self.step_count % self.cadence == 0:
            drv = RefineDriver(positions=self.p.x,
                               static_tiles=self.static_tiles,
                               levels=self.topo.levels)
            self.last_report = self.adaptor.update(drv, self.pair)
            self.grid.sync()
        self.step_count += 1
        self._record()

    def _powder_cycle(self, is_mpm):
        sv = self.solver
        r, w = sv.last_roles(0)
        dst = sv.arrays(w, 0)
        src = sv.arrays(r, 0)
        source = None
        if is_mpm and self.last_fields is not None:
            source = entrainment_rate(self.last_fields, self.p, self.topo,
                                      self.mat, self.powder)
        dst["phi"][:] = powder_step(src["phi"],
                                    [dst["u" + x] for x in "xyz"[:self.d]],
                                    self.topo, self.powder, 1.0, source)

    def diag_row(self):
        sv = self.solver
        d = self.d
        fm = np.zeros(d)
        sum_phi = 0.0
        eps_min = 1.0
        for l in range(self.topo.levels):
            if not self.topo.n_tiles(l):
                continue
            lw = sv.last_roles(l)[1] if sv.k[l] else 0
            a = sv.arrays(lw, l)
            leaf = self.topo.leaf_flat(l)
            vol = float((1 << d) ** l)
            for i, x in enumerate("xyz"[:d]):
                fm[i] += vol * (a["rho"][leaf] * a["u" + x][leaf]).sum()
            sum_phi += vol * a["phi"][leaf].sum()
            if leaf.any():
                eps_min = min(eps_min, float(a["eps"][leaf].min()))
        drag = self.last_fields.fs.sum(axis=0) if self.last_fields is not None \
            else np.zeros(d)
        return dict(step=self.step_count,
                    t_phys=self.step_count * self.unit_dt,
                    fluid_mom=tuple(float(v) for v in fm),
                    sediment_mom=tuple(float(v) for v in self.p.momentum())
                    if len(self.p) else (0.0,) * d,
                    drag_impulse=tuple(float(-v) for v in drag),
                    sum_phi=float(sum_phi),
                    tiles=tuple(self.topo.n_tiles(l)
                                for l in range(self.topo.levels)),
                    eps_min=eps_min)

    def _record(self):
        self.diagnostics.append(self.diag_row())
