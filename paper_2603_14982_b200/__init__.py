"""B200-native hot path of arXiv 2603.14982's adaptive multi-level
HOME-LBM <-> MPM coupled solver.

Drop-in for the reference package's solver / scene API (``pkg/src/mlbm``):
same class and method names, device-resident state, hand-written sm_100a
kernels behind a C ABI (``include/mlbm_b200.h``).  No CPU fallback.
"""
from .lattice import CS2, DivergenceError, H3_XYZ_HERMITE, H3_XYZ_PAPER
from .sparse_grid import (BORDER, LEAF, TILE, FieldTree, PingPongPair, Topology,
                          TopologyError, buffer_roles, field_names)
from .solver import (BoundarySpec, LevelParams, LogInlet, MultiLevelSolver, SolverParams,
                     build_schedule, rescale_s_down, rescale_s_up, rescale_tau)
from .adapt import AdaptReport, GridAdaptor, RefineDriver, update_grid

__all__ = [
    "CS2", "DivergenceError", "H3_XYZ_HERMITE", "H3_XYZ_PAPER", "BORDER", "LEAF", "TILE",
    "FieldTree", "PingPongPair", "Topology", "TopologyError", "buffer_roles", "field_names",
    "BoundarySpec", "LevelParams", "LogInlet", "MultiLevelSolver", "SolverParams",
    "build_schedule", "rescale_s_down", "rescale_s_up", "rescale_tau", "AdaptReport",
    "GridAdaptor", "RefineDriver", "update_grid",
]
