"""Lattice constants and host-side moment helpers (lattice.py:1-216).

The device kernels carry their own compile-time D2Q9 / D3Q27 tables
(``csrc/common.cuh``); this module only holds what the host API exposes:
the sound speed, the Hermite xyz-coefficient choices for D3Q27 and the
DivergenceError type the solver raises (lattice.py:23-29).
"""
from __future__ import annotations

import numpy as np

CS2 = 1.0 / 3.0
CS4 = CS2 * CS2
CS6 = CS4 * CS2

# Gamma_xyz coefficient in the D3Q27 third-order reconstruction: the Hermite
# projection weights xyz by 6/3! = 1/cs^6; PAPER.md:180-188 prints 1/(2 cs^6).
H3_XYZ_HERMITE = 1.0 / CS6
H3_XYZ_PAPER = 1.0 / (2.0 * CS6)


class DivergenceError(RuntimeError):
    """A kernel produced a non-physical state (rho <= 0, NaN)."""

    def __init__(self, message, level=None, cells=None):
        super().__init__(message)
        self.level = level
        self.cells = cells


def seq(u):
    """Equilibrium second moment u (x) u as independent components
    (lattice.py:116-124), any d."""
    u = np.asarray(u, dtype=float)
    d = u.shape[-1]
    return np.stack([u[..., a] * u[..., b] for a in range(d) for b in range(a, d)], axis=-1)
