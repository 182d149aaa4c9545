"""MPM sand (oracle, d = 2 or 3).

Restates ``pkg/src/mlbm/granular.py``:
  * SandMaterial (lam, mu, alpha)          granular.py:22-38
  * Particles SoA, sample_blocks           granular.py:41-80
  * MpmGrid wall bands / sticky solids     granular.py:83-130
  * quadratic B-spline stencil (3^d nodes) granular.py:137-178
  * svd2 (2D closed form)                  granular.py:181-213; 3D uses a
    rotation-variant SVD (U, V proper rotations, sign on the last value)
  * Drucker-Prager return map (d-generic:
    e = eps + vc/d, (d lam + 2 mu)/(2 mu))  granular.py:216-241
  * Kirchhoff stress                       granular.py:260-279
  * p2g / grid_update / g2p / mpm_step     granular.py:282-425
  * SnowMaterial + nacc_return_map: the paper's snow, absent
    from the reference — PARITY UNPINNED, see nacc_return_map
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import Topology, TopologyError
from .lbm import BoundarySpec, face_names, solid_at


@dataclass
class SandMaterial:
    E: float = 3.5e5
    nu: float = 0.3
    friction_deg: float = 30.0
    floor_friction: float = 0.5

    def __post_init__(self):
        self.lam = self.E * self.nu / ((1 + self.nu) * (1 - 2 * self.nu))
        self.mu = self.E / (2 * (1 + self.nu))
        sf = np.sin(np.radians(self.friction_deg))
        self.alpha = np.sqrt(2.0 / 3.0) * 2.0 * sf / (3.0 - sf)


@dataclass
class SnowMaterial:
    """Snow for the avalanche scene: Non-Associated Cam
    Clay (Wolper et al. 2019) on the same Hencky elasticity as the sand, with
    the paper's modified hardening law.  Not in the reference:
    this restatement is the specification the device follows (parity
    unpinned).

    M: critical-state slope; beta: cohesion (tensile / compressive strength
    ratio); xi: hardening factor of p0 = kappa (1e-5 + sinh(xi max(q, 0)));
    alpha_soft: the paper's softening coefficient alpha; q_init: the initial
    (softened) hardening parameter q."""
    E: float = 3.5e5
    nu: float = 0.3
    M: float = 1.85
    beta: float = 0.3
    xi: float = 1.0
    alpha_soft: float = 0.5
    q_init: float = 0.05
    floor_friction: float = 0.5
    friction_deg: float = 30.0       # unused by NACC (kept for the scene schema)

    def __post_init__(self):
        self.lam = self.E * self.nu / ((1 + self.nu) * (1 - 2 * self.nu))
        self.mu = self.E / (2 * (1 + self.nu))
        self.alpha = 0.0

    def kappa(self, d):
        """Hencky bulk modulus: p = -kappa tr(e) with tau = 2 mu e + lam tr(e) I."""
        return self.lam + 2.0 * self.mu / d


def nacc_state_decode(qs):
    """The per-particle hardening state lives in the vol_corr row: qs >= 0 is
    the hardening parameter q of a particle that never reached q = 0; a
    particle that did (cracked, cohesion 0 from then on) stores -(q + 1)."""
    cracked = qs < 0.0
    return np.where(cracked, -qs - 1.0, qs), cracked


def nacc_return_map(e, qs, mat: SnowMaterial):
    """NACC return map in principal log-strain space (Hencky elasticity) with
    the softening law of PAPER.md:630-637.

    e: (n, d) trial log stretches; qs: (n,) hardening state (nacc_state_decode).
    p = -kappa tr(e), s = 2 mu dev(e), q_s = sqrt((6 - d)/2) |s|; yield
    y = (1 + 2 beta) q_s^2 + M^2 (p + beta p0)(p - p0) <= 0 (Wolper et al. 2019):
      p > p0          -> compressive tip  (p = p0, s = 0)
      p < -beta p0    -> tensile tip      (p = -beta p0, s = 0)
      y <= 0          -> elastic
      else            -> s scaled onto the surface at fixed p (non-associated)
    NACC's hardening increment of h = -log Jp is dh0 = log J_x - log J_trial,
    J_x the elastic volume on the surface: the tip in the tip cases, else the
    surface point on the line from (p_c = (1 - beta) p0 / 2, 0) to the trial
    state.  The paper's law: dq = -alpha_soft dh0 until q first reaches 0
    (the particle cracks, its cohesion beta becomes 0), dq = +dh0 after.
    Returns (e_new, qs_new)."""
    n, d = e.shape
    kappa = mat.kappa(d)
    mu = mat.mu
    q, cracked = nacc_state_decode(np.asarray(qs, dtype=float))
    beta = np.where(cracked, 0.0, mat.beta)
    p0 = kappa * (1e-5 + np.sinh(mat.xi * np.maximum(q, 0.0)))
    ev = e.sum(axis=1)
    eh = e - ev[:, None] / d
    sn = 2.0 * mu * np.sqrt((eh ** 2).sum(axis=1))
    cs = np.sqrt((6.0 - d) / 2.0)
    p_tr = -kappa * ev
    q_tr = cs * sn
    M2 = mat.M * mat.M
    yp = M2 * (p_tr + beta * p0) * (p_tr - p0)
    y = (1.0 + 2.0 * beta) * q_tr ** 2 + yp
    out = e.copy()
    dlogjp = np.zeros(n)
    c1 = p_tr > p0
    c2 = (~c1) & (p_tr < -beta * p0)
    c4 = (~c1) & (~c2) & (y > 1e-12 * np.maximum(p0 * p0 * M2, 1e-300))
    ev1 = -p0 / kappa
    out[c1] = (ev1[c1] / d)[:, None]
    dlogjp[c1] = ev[c1] - ev1[c1]
    ev2 = beta * p0 / kappa
    out[c2] = (ev2[c2] / d)[:, None]
    dlogjp[c2] = ev[c2] - ev2[c2]
    if c4.any():
        s_new = np.sqrt(np.maximum(-yp[c4], 0.0) / (1.0 + 2.0 * beta[c4])) / cs
        scale = np.where(sn[c4] > 0.0, s_new / np.where(sn[c4] > 0.0, sn[c4], 1.0), 0.0)
        out[c4] = eh[c4] * scale[:, None] + (ev[c4] / d)[:, None]
        # hardening: the surface point towards the ellipse centre
        pb, qb, b4, p04 = p_tr[c4], q_tr[c4], beta[c4], p0[c4]
        pc = (1.0 - b4) * p04 / 2.0
        d0, d1 = pc - pb, -qb
        nrm = np.sqrt(d0 * d0 + d1 * d1)
        nrm = np.where(nrm > 0.0, nrm, 1.0)
        d0, d1 = d0 / nrm, d1 / nrm
        A = M2 * d0 * d0 + (1.0 + 2.0 * b4) * d1 * d1
        B = M2 * d0 * (2.0 * pc - p04 + b4 * p04)
        C = M2 * (pc + b4 * p04) * (pc - p04)
        disc = np.sqrt(np.maximum(B * B - 4.0 * A * C, 0.0))
        A = np.where(A > 0.0, A, 1.0)
        l1 = (-B + disc) / (2.0 * A)
        l2 = (-B - disc) / (2.0 * A)
        p1 = pc + l1 * d0
        p2 = pc + l2 * d0
        px = np.where((pb - pc) * (p1 - pc) > 0.0, p1, p2)
        dlogjp[c4] = ev[c4] + px / kappa
    dh0 = -dlogjp
    qn = q + np.where(cracked, 1.0, -mat.alpha_soft) * dh0
    newly = (~cracked) & (qn <= 0.0)
    cr = cracked | newly
    qn = np.where(cr, np.maximum(qn, 0.0), qn)
    qn = np.where(newly, 0.0, qn)
    return out, np.where(cr, -qn - 1.0, qn)


def nacc_yield(e, qs, mat: SnowMaterial):
    """y(p, q_s) of nacc_return_map for states e (test helper)."""
    n, d = e.shape
    kappa = mat.kappa(d)
    q, cracked = nacc_state_decode(np.asarray(qs, dtype=float))
    beta = np.where(cracked, 0.0, mat.beta)
    p0 = kappa * (1e-5 + np.sinh(mat.xi * np.maximum(q, 0.0)))
    ev = e.sum(axis=1)
    eh = e - ev[:, None] / d
    q_s = np.sqrt((6.0 - d) / 2.0) * 2.0 * mat.mu * np.sqrt((eh ** 2).sum(axis=1))
    p = -kappa * ev
    return (1.0 + 2.0 * beta) * q_s ** 2 + mat.M ** 2 * (p + beta * p0) * (p - p0), p0


class Particles:
    def __init__(self, n, d=2):
        self.d = d
        self.x = np.zeros((n, d))
        self.v = np.zeros((n, d))
        self.C = np.zeros((n, d, d))
        self.F = np.tile(np.eye(d), (n, 1, 1))
        self.m = np.ones(n)
        self.V0 = np.ones(n)
        self.vol_corr = np.zeros(n)

    def __len__(self):
        return self.x.shape[0]

    def momentum(self):
        return (self.m[:, None] * self.v).sum(axis=0)

    def total_mass(self):
        return float(self.m.sum())

    def copy(self):
        p = Particles(len(self), self.d)
        for k in ("x", "v", "C", "F", "m", "V0", "vol_corr"):
            setattr(p, k, getattr(self, k).copy())
        return p


def sample_blocks(blocks, per_cell, density, rng, d=2):
    """granular.py:66-80; a block is (lo..., hi...)."""
    counts = []
    for b in blocks:
        vol = 1.0
        for a in range(d):
            vol *= b[d + a] - b[a]
        counts.append(int(round(vol * per_cell)))
    p = Particles(sum(counts), d)
    at = 0
    for b, cnt in zip(blocks, counts):
        u = rng.random((cnt, d))
        for a in range(d):
            p.x[at:at + cnt, a] = b[a] + u[:, a] * (b[d + a] - b[a])
        at += cnt
    p.V0[:] = 1.0 / per_cell
    p.m[:] = density / per_cell
    return p


class MpmGrid:
    def __init__(self, topo: Topology, spec: BoundarySpec | None = None):
        self.topo = topo
        self.spec = spec or BoundarySpec(d=topo.d)
        self._ver = -1
        self.sync()

    def sync(self):
        if self._ver == self.topo.version:
            return
        topo = self.topo
        d = topo.d
        n = topo.cell_count(0)
        self.mass = np.zeros(n)
        self.mom = np.zeros((n, d))
        self.f_int = np.zeros((n, d))
        self.drag = np.zeros((n, d))
        self.vel = np.zeros((n, d))
        coords = topo.cell_coords(0)
        dims = topo.cells_dims(0)
        self.wall_sets = []
        for face in face_names(d):
            if self.spec.faces.get(face) != "wall":
                continue
            axis = "xyz".index(face[0])
            sign = 1.0 if face.endswith("_min") else -1.0
            sel = coords[:, axis] <= 1 if sign > 0 else \
                coords[:, axis] >= dims[axis] - 2
            sel = np.nonzero(sel)[0]
            if sel.size:
                self.wall_sets.append((sel, axis, sign))
        self.sticky = np.nonzero(solid_at(self.spec, coords))[0]
        self._ver = topo.version

    def clear(self):
        self.mass[:] = 0
        self.mom[:] = 0
        self.f_int[:] = 0
        self.vel[:] = 0


def stencil(x, topo: Topology):
    """Returns idx, w, grad (n,K,d), dpos (n,K,d); K = 3^d, node k has
    offset (k // 3^a) % 3 along axis a (granular.py:133-178)."""
    d = topo.d
    dims = topo.cells_dims(0)
    cmap = topo.cell_map(0)
    base = np.floor(x - 0.5).astype(np.int64)
    f = x - base
    W = np.stack([0.5 * (1.5 - f) ** 2, 0.75 - (f - 1.0) ** 2,
                  0.5 * (f - 0.5) ** 2], axis=-1)          # (n, d, 3)
    dW = np.stack([f - 1.5, -2.0 * (f - 1.0), f - 0.5], axis=-1)
    K = 3 ** d
    offs = np.array([[(k // 3 ** a) % 3 for a in range(d)] for k in range(K)])
    node = base[:, None, :] + offs[None]                     # (n, K, d)
    for a in range(d):
        if topo.periodic[a]:
            node[:, :, a] %= dims[a]
        elif (node[:, :, a] < 0).any() or (node[:, :, a] >= dims[a]).any():
            raise TopologyError("particle stencil leaves the domain")
    idx = cmap[tuple(node.reshape(-1, d).T)].reshape(len(x), K)
    if (idx < 0).any():
        raise TopologyError("particle stencil node not stored at level 0")
    n = len(x)
    w = np.ones((n, K))
    grad = np.ones((n, K, d))
    for a in range(d):
        wa = W[:, a, :][:, offs[:, a]]
        dwa = dW[:, a, :][:, offs[:, a]]
        w = w * wa
        for b in range(d):
            grad[:, :, b] *= dwa if a == b else wa
    dpos = (base[:, None, :] + offs[None]) - x[:, None, :]
    return idx, w, grad, dpos


def svd2(F):
    a, b, c, d = F[:, 0, 0], F[:, 0, 1], F[:, 1, 0], F[:, 1, 1]
    e, f, g, h = 0.5 * (a + d), 0.5 * (a - d), 0.5 * (c + b), 0.5 * (c - b)
    q, r = np.hypot(e, h), np.hypot(f, g)
    a1, a2 = np.arctan2(g, f), np.arctan2(h, e)
    tu, tv = 0.5 * (a1 + a2), 0.5 * (a1 - a2)

    def rot(t):
        R = np.empty((len(t), 2, 2))
        R[:, 0, 0] = np.cos(t)
        R[:, 0, 1] = -np.sin(t)
        R[:, 1, 0] = np.sin(t)
        R[:, 1, 1] = np.cos(t)
        return R
    return rot(tu), np.stack([q + r, q - r], axis=1), rot(tv)


def svd3(F):
    U, s, Vt = np.linalg.svd(F)
    V = np.swapaxes(Vt, 1, 2).copy()
    s = s.copy()
    du = np.linalg.det(U) < 0
    U[du, :, 2] *= -1
    s[du, 2] *= -1
    dv = np.linalg.det(V) < 0
    V[dv, :, 2] *= -1
    s[dv, 2] *= -1
    return U, s, V


def svd(F):
    return svd2(F) if F.shape[1] == 2 else svd3(F)


def dp_return_map(eps, vc, mat: SandMaterial):
    d = eps.shape[1]
    e = eps + vc[:, None] / d
    tr = e.sum(axis=1)
    ehat = e - tr[:, None] / d
    norm = np.sqrt((ehat ** 2).sum(axis=1))
    dg = norm + ((d * mat.lam + 2.0 * mat.mu) / (2.0 * mat.mu)) * tr * mat.alpha
    tip = tr > 0.0
    shear = (~tip) & (norm > 0.0) & (dg > 0.0)
    out = e.copy()
    out[tip] = 0.0
    if shear.any():
        out[shear] = e[shear] - (dg[shear] / norm[shear])[:, None] * ehat[shear]
    return out, tr - out.sum(axis=1)


def kirchhoff(p: Particles, mat: SandMaterial):
    U, sig, _ = svd(p.F)
    eps = np.log(np.maximum(sig, 1e-12))
    tr = eps.sum(axis=1)
    tp = 2.0 * mat.mu * eps + mat.lam * tr[:, None]
    return np.einsum("nik,nk,njk->nij", U, tp, U)


def p2g(p: Particles, grid: MpmGrid, mat, st=None):
    grid.sync()
    grid.clear()
    if not len(p):
        return
    idx, w, grad, dpos = st if st is not None else stencil(p.x, grid.topo)
    d = p.d
    n = grid.mass.shape[0]
    tau = kirchhoff(p, mat)
    flat = idx.ravel()
    wm = w * p.m[:, None]
    grid.mass += np.bincount(flat, weights=wm.ravel(), minlength=n)
    for a in range(d):
        aff = p.v[:, a:a + 1] + np.einsum("nb,nkb->nk", p.C[:, a, :], dpos)
        grid.mom[:, a] += np.bincount(flat, weights=(wm * aff).ravel(),
                                      minlength=n)
        fa = np.einsum("nb,nkb->nk", p.V0[:, None] * tau[:, a, :], grad)
        grid.f_int[:, a] -= np.bincount(flat, weights=fa.ravel(), minlength=n)


def grid_update(grid: MpmGrid, dt, gravity, drag=None, floor_friction=0.5):
    massive = grid.mass > 0.0
    inv_m = np.zeros_like(grid.mass)
    inv_m[massive] = 1.0 / grid.mass[massive]
    force = grid.f_int.copy()
    if drag is not None:
        force += drag
    grid.vel = (grid.mom + dt * force) * inv_m[:, None]
    grid.vel[massive] += dt * np.asarray(gravity)[None, :]
    grid.vel[~massive] = 0.0
    d = grid.vel.shape[1]
    for sel, axis, sign in grid.wall_sets:
        v = grid.vel[sel]
        vn = sign * v[:, axis]
        into = vn < 0.0
        if not into.any():
            continue
        tang = [b for b in range(d) if b != axis]
        vt = v[into][:, tang]
        vtn = np.sqrt((vt ** 2).sum(axis=1)) if d == 3 else np.abs(vt[:, 0])
        scale = np.maximum(0.0, 1.0 - floor_friction * (-vn[into])
                           / np.maximum(vtn, 1e-14))
        vi = v[into]
        vi[:, axis] = 0.0
        vi[:, tang] = vt * scale[:, None]
        v[into] = vi
        grid.vel[sel] = v
    if grid.sticky.size:
        grid.vel[grid.sticky] = 0.0


def g2p(p: Particles, grid: MpmGrid, dt, mat, plastic=True, st=None):
    if not len(p):
        return 0
    idx, w, _, dpos = st if st is not None else stencil(p.x, grid.topo)
    d = p.d
    gv = grid.vel[idx]                                      # (n, K, d)
    wg = w[:, :, None] * gv
    p.v = wg.sum(axis=1)
    p.C = 4.0 * np.einsum("nka,nkb->nab", wg, dpos)
    p.x = p.x + dt * p.v
    dims = grid.topo.cells_dims(0)
    clamped = 0
    for a in range(d):
        if grid.topo.periodic[a]:
            p.x[:, a] %= dims[a]
        else:
            lo, hi = 2.0, dims[a] - 2.0
            clamped += int(((p.x[:, a] < lo) | (p.x[:, a] > hi)).sum())
            p.x[:, a] = p.x[:, a].clip(lo, hi)
    G = np.eye(d)[None] + dt * p.C
    p.F = np.einsum("nij,njk->nik", G, p.F)
    if plastic:
        U, sig, V = svd(p.F)
        sig = np.clip(sig, 0.05, 4.0)
        if isinstance(mat, SnowMaterial):
            eps_new, vc = nacc_return_map(np.log(sig), p.vol_corr, mat)
        else:
            eps_new, vc = dp_return_map(np.log(sig), p.vol_corr, mat)
        p.vol_corr = vc
        p.F = np.einsum("nik,nk,njk->nij", U, np.exp(eps_new), V)
    return clamped


def mpm_step(p, grid, dt, gravity, mat, drag=None, plastic=True, st=None):
    grid.sync()
    if st is None and len(p):
        st = stencil(p.x, grid.topo)
    p2g(p, grid, mat, st=st)
    grid_update(grid, dt, gravity, drag=drag, floor_friction=mat.floor_friction)
    return g2p(p, grid, dt, mat, plastic=plastic, st=st)


def cfl_check(p, dt):
    if not len(p):
        return True
    return float(np.abs(p.v).max()) * dt < 0.5
