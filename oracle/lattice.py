"""Lattice tables and moment algebra (oracle, fp64, d = 2 or 3).

Restates ``pkg/src/mlbm/lattice.py``:
  * D2Q9 tables            -> lattice.py:51-74 (same direction order)
  * Hermite reconstruction -> lattice.py:127-186 (``_gamma_terms``,
    ``reconstruct_fields``, ``reconstruct_direction``)
  * moment recovery        -> lattice.py:189-205
and extends them to D3Q27 with the third-order index set
{xxy, xyy, xxz, xzz, yzz, yyz, xyz} of PAPER.md:180-188.

The ``xyz`` coefficient is a choice the paper leaves open (PAPER.md prints
1/(2 cs^6) uniformly; the Hermite projection gives 1/cs^6 because xyz has six
orderings against three for xxy).  ``H3_XYZ_HERMITE`` is the default, and the
paper-literal value is selectable; on z-extruded states Gamma_xyz == 0 so the
2D reduction is independent of the choice.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

CS2 = 1.0 / 3.0
CS4 = CS2 * CS2
CS6 = CS4 * CS2

H3_XYZ_HERMITE = 1.0 / CS6
H3_XYZ_PAPER = 1.0 / (2.0 * CS6)

AXES = "xyz"


def s_pairs(d):
    """Independent second-moment components (a <= b), row-major."""
    return [(a, b) for a in range(d) for b in range(a, d)]


def s_names(d):
    return ["s" + AXES[a] + AXES[b] for a, b in s_pairs(d)]


def h3_triples(d):
    """Third-order Hermite index set (sorted index triples)."""
    if d == 2:
        return [(0, 0, 1), (0, 1, 1)]
    # xxy, xyy, xxz, xzz, yzz, yyz, xyz
    return [(0, 0, 1), (0, 1, 1), (0, 0, 2), (0, 2, 2), (1, 2, 2), (1, 1, 2),
            (0, 1, 2)]


@dataclass(frozen=True)
class Lattice:
    d: int
    q: int
    c: np.ndarray          # (q, d) int
    w: np.ndarray          # (q,)
    opp: np.ndarray        # (q,)
    h3coef: np.ndarray     # (n3,) coefficient per third-order component

    @property
    def n_s(self):
        return self.d * (self.d + 1) // 2


def d2q9() -> Lattice:
    # lattice.py:53-60 — rest, axis directions, diagonals
    c = np.array([[0, 0], [1, 0], [0, 1], [-1, 0], [0, -1],
                  [1, 1], [-1, 1], [-1, -1], [1, -1]], dtype=np.int64)
    w = np.array([4.0 / 9.0] + [1.0 / 9.0] * 4 + [1.0 / 36.0] * 4)
    opp = np.array([0, 3, 4, 1, 2, 7, 8, 5, 6], dtype=np.int64)
    return Lattice(2, 9, c, w, opp, np.full(2, 1.0 / (2.0 * CS6)))


def d3q27(h3_xyz=H3_XYZ_HERMITE) -> Lattice:
    """Tensor product of D1Q3 (w = 2/3, 1/6, 1/6); rest first, then
    opposite pairs adjacent (i, i+1) ordered face, edge, corner."""
    reps = []
    for v in itertools.product((1, 0, -1), repeat=3):
        v = np.array(v)
        if not v.any():
            continue
        # representative: first non-zero component positive
        if v[np.nonzero(v)[0][0]] > 0:
            reps.append(v)
    reps.sort(key=lambda v: (int(np.abs(v).sum()), [-x for x in v]))
    dirs = [np.zeros(3, dtype=np.int64)]
    for v in reps:
        dirs.append(v)
        dirs.append(-v)
    c = np.array(dirs, dtype=np.int64)
    w1 = {0: 2.0 / 3.0, 1: 1.0 / 6.0, -1: 1.0 / 6.0}
    w = np.array([w1[a] * w1[b] * w1[e] for a, b, e in c])
    opp = np.empty(27, dtype=np.int64)
    for i in range(27):
        opp[i] = [j for j in range(27) if (c[j] == -c[i]).all()][0]
    coef = np.full(7, 1.0 / (2.0 * CS6))
    coef[6] = h3_xyz
    return Lattice(3, 27, c, w, opp, coef)


def lattice_for(d, h3_xyz=H3_XYZ_HERMITE) -> Lattice:
    return d2q9() if d == 2 else d3q27(h3_xyz)


def h2(c, a, b):
    return c[a] * c[b] - (CS2 if a == b else 0.0)


def h3(c, t):
    """H3_{abc}(c) = c_a c_b c_g - cs2 (c_a d_bg + c_b d_ag + c_g d_ab)."""
    a, b, g = t
    v = c[a] * c[b] * c[g]
    v -= CS2 * ((c[a] if b == g else 0.0) + (c[b] if a == g else 0.0)
                + (c[g] if a == b else 0.0))
    return v


def gamma(t, u, s):
    """Gamma_abg = S_ab u_g + S_ag u_b + S_bg u_a - 2 u_a u_b u_g
    (lattice.py:127-131).  ``s`` maps (a<=b) -> array."""
    a, b, g = t

    def S(i, j):
        return s[(min(i, j), max(i, j))]
    return S(a, b) * u[g] + S(a, g) * u[b] + S(b, g) * u[a] \
        - 2.0 * u[a] * u[b] * u[g]


def reconstruct_dir(lat: Lattice, i, rho, u, s):
    """f_i from moments (lattice.py:170-186).  u: list of d arrays;
    s: dict (a,b)->array."""
    c = lat.c[i].astype(float)
    d = lat.d
    cu = sum(c[a] * u[a] for a in range(d)) / CS2
    a2 = 0.0
    for (a, b) in s_pairs(d):
        hv = h2(c, a, b)
        if hv != 0.0:
            a2 = a2 + (1.0 if a == b else 2.0) * hv * s[(a, b)]
    out = 1.0 + cu + a2 / (2.0 * CS4)
    a3 = 0.0
    for k, t in enumerate(h3_triples(d)):
        hv = h3(c, t)
        if hv != 0.0:
            a3 = a3 + lat.h3coef[k] * hv * gamma(t, u, s)
    out = out + a3
    return rho * lat.w[i] * out


def moments_from_f(lat: Lattice, fs):
    """Bare moments (rho*, sum c f, sum (cc - cs2 d) f) of a list of f_i
    (solver.py:362-371)."""
    d = lat.d
    rho = 0.0
    m = [0.0] * d
    pi = {p: 0.0 for p in s_pairs(d)}
    for i, f in enumerate(fs):
        c = lat.c[i].astype(float)
        rho = rho + f
        for a in range(d):
            if c[a]:
                m[a] = m[a] + c[a] * f
        for (a, b) in s_pairs(d):
            hv = h2(c, a, b)
            if hv != 0.0:
                pi[(a, b)] = pi[(a, b)] + hv * f
    return rho, m, pi
