"""GPU parity of the LBM level kernels, transfers and schedule against the
oracle (fp64: <= 1e-12 abs; fp32 shifted form: <= 1e-5 relative L2).

Cases mirror the reference tests: one-step pull-streaming golden
(test_solver.py:206-254), Taylor-Green decay, static multi-level refinement
(test_solver.py:279-371), boundaries (test_solver.py:374-456), in 2D and 3D.
"""
import numpy as np
import pytest
import torch

from helpers import central_mask, compare_levels, oracle_static_refined, rel_l2
from oracle import grid as OG
from oracle import lbm as OL

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_2603_14982_b200")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def smooth_fields(d, seed=0, amp=0.04):
    """Deterministic, coordinate-keyed non-trivial moment fields."""
    rng = np.random.default_rng(seed)
    k = rng.uniform(0.2, 0.9, size=(12, d))
    ph = rng.uniform(0, 6.28, size=12)
    ax = "xyz"[:d]

    def fn(pos, level):
        def w(i):
            return np.sin(pos @ k[i] + ph[i])
        out = {"rho": 1.0 + 0.02 * w(0)}
        for a in range(d):
            out["u" + ax[a]] = amp * w(1 + a)
        j = 4
        for a in range(d):
            for b in range(a, d):
                out["s" + ax[a] + ax[b]] = out["u" + ax[a]] * out["u" + ax[b]] + 0.004 * w(j % 12)
                j += 1
        return out
    return fn


def build_pair(otopo, dtype, fn, spec=None, gravity=None, tau0=0.8, h3=None,
               upward="coincident"):
    d = otopo.d
    ospec = spec or OL.BoundarySpec(d=d)
    params = dict(levels=otopo.levels, gravity=gravity or (0.0,) * d, upward_mode=upward)
    if h3 is not None:
        params["h3_xyz"] = h3
    opair = OG.PingPongPair(otopo)
    osv = OL.Solver(otopo, opair, OL.SolverParams(**params), OL.LevelParams(otopo.levels, tau0),
                    ospec)
    OL.set_fields(otopo, opair, fn)

    dtopo = B.Topology(otopo.finest, otopo.levels, otopo.periodic)
    dtopo.set_tile_set(otopo.tile_set())
    dpair = B.PingPongPair(dtopo, dtype)
    dspec = B.BoundarySpec(faces={k: (B.LogInlet(v.u0, v.beta, v.y0)
                                     if isinstance(v, OL.LogInlet) else v)
                                  for k, v in ospec.faces.items()},
                           solid_boxes=list(ospec.solid_boxes), heightmap=ospec.heightmap, dim=d)
    dparams = B.SolverParams(**params)
    dsv = B.MultiLevelSolver(dtopo, dpair, dparams, B.LevelParams(otopo.levels, tau0), dspec)
    for l in range(otopo.levels):
        if not dtopo.n_tiles(l):
            continue
        pos = dtopo.cell_coords(l) * float(1 << l)
        vals = fn(pos, l)
        for t in range(2):
            for nm, v in vals.items():
                dpair.trees[t].levels[l][nm] = v
    return osv, dsv


def moments(d):
    return OG.moment_names(d)


def last(sv, l):
    return sv.arrays(sv.last_roles(l)[1], l)


@pytest.mark.parametrize("d", [2, 3])
def test_one_step_single_level_fp64(d):
    _need_gpu()
    cells = (16,) * d
    otopo = OG.Topology.uniform(cells, 1)
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 3), tau0=0.73)
    osv.advance_bounce()
    dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(d))
    assert max(w.values()) <= 1e-14, w


@pytest.mark.parametrize("d", [2, 3])
def test_taylor_green_many_steps_fp64(d):
    _need_gpu()
    cells = (32, 32) if d == 2 else (16, 16, 8)
    otopo = OG.Topology.uniform(cells, 1)
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 5), tau0=0.8)
    for _ in range(50):
        osv.advance_bounce()
        dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(d))
    assert max(w.values()) <= 1e-12, w


@pytest.mark.parametrize("d,levels", [(2, 2), (2, 3), (3, 2)])
def test_static_multilevel_fp64(d, levels):
    _need_gpu()
    cells = (64, 64) if d == 2 else (32, 32, 32)
    otopo = oracle_static_refined(cells, levels, central_mask(cells, pad=8 if d == 2 else 4))
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 7), tau0=0.8)
    assert dsv.topology.tile_set() == otopo.tile_set()
    for _ in range(6):
        osv.advance_bounce()
        dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(d) + ["eps", "phi"])
    assert max(w.values()) <= 1e-12, w


def test_upward_average_mode_fp64():
    _need_gpu()
    cells = (64, 64)
    otopo = oracle_static_refined(cells, 2, central_mask(cells, pad=8))
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(2, 9), upward="average")
    for _ in range(4):
        osv.advance_bounce()
        dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(2))
    assert max(w.values()) <= 1e-12, w


@pytest.mark.parametrize("d", [2, 3])
def test_boundaries_fp64(d):
    _need_gpu()
    if d == 2:
        cells = (32, 32)
        faces = {"x_min": OL.LogInlet(0.04, 0.35, 6.0), "x_max": "outlet",
                 "y_min": "wall", "y_max": "outlet"}
        boxes = [(10.0, 0.0, 14.0, 5.0)]
    else:
        cells = (32, 16, 16)
        faces = {"x_min": OL.LogInlet(0.04, 0.35, 3.0), "x_max": "outlet",
                 "y_min": "wall", "y_max": "outlet", "z_min": "periodic", "z_max": "periodic"}
        boxes = [(10.0, 0.0, 2.0, 14.0, 5.0, 9.0)]
    spec = OL.BoundarySpec(d=d, faces=faces, solid_boxes=boxes)
    otopo = OG.Topology.uniform(cells, 1, spec.periodic_axes())
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 11), spec=spec,
                          gravity=(0.0, -1e-4) + ((0.0,) if d == 3 else ()))
    for _ in range(20):
        osv.advance_bounce()
        dsv.advance_bounce()
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l),
                       moments(d))
    assert max(w.values()) <= 1e-12, w


@pytest.mark.parametrize("d", [2, 3])
def test_fp32_shifted_rel_l2(d):
    """Gate B: fp32 device vs fp64 oracle, <= 1e-5 relative L2 after 100 steps."""
    _need_gpu()
    cells = (64, 64) if d == 2 else (32, 32, 16)
    otopo = OG.Topology.uniform(cells, 1)
    osv, dsv = build_pair(otopo, torch.float32, smooth_fields(d, 13, amp=0.03), tau0=0.8)
    for _ in range(100):
        osv.advance_bounce()
        dsv.advance_bounce()
    names = moments(d)
    for nm in names:
        r = rel_l2(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l), [nm])
        assert r <= 1e-5, (nm, r)


class DeviceNaive:
    """The reference's NaiveReference (harness/reference.py:31-106) over the
    device kernels: one dedicated (current, next) buffer pair per level (2L
    buffers outside the solver's ping-pong pair), each level step driven as
    stream_kernel -> collide_kernel -> boundary_kernel (reference.py:67-72)."""

    def __init__(self, dsv):
        from paper_2603_14982_b200.sparse_grid import LevelFields, fresh_block
        self.sv = dsv
        topo = dsv.topology
        self.buffers = []
        for l in range(topo.levels):
            pair = []
            for _ in range(2):
                blk = fresh_block(topo.d, topo.capacity_cells(l), dsv.dtype, topo.device)
                pair.append(LevelFields(topo.d, blk, live=(lambda l=l: topo.cell_count(l))))
            self.buffers.append(pair)
        self.k = [0] * topo.levels

    def load_from(self, trees_levels):
        for l, lf in enumerate(trees_levels):
            for b in self.buffers[l]:
                b.data.copy_(lf.data)

    def cur(self, l):
        return self.buffers[l][self.k[l] % 2]

    def nxt(self, l):
        return self.buffers[l][1 - self.k[l] % 2]

    def _sc(self, l):
        self.sv.stream_kernel(l, self.cur(l), self.nxt(l))
        self.sv.collide_kernel(l, self.cur(l), self.nxt(l))
        self.sv.boundary_kernel(l, self.nxt(l))
        self.k[l] += 1

    def _down(self, l, sub):
        c = l + 1
        kc = self.k[c]
        self.sv.downward_kernel(l, sub, self.buffers[c][(kc - 1) % 2], self.buffers[c][kc % 2],
                                self.cur(l))

    def _up(self, l):
        c = l + 1
        self.sv.upward_kernel(l, self.cur(l), self.buffers[c][self.k[c] % 2])

    def advance_bounce(self):
        levels = self.sv.topology.levels
        for cycle in self.sv._schedule:
            for kind, level, sub in cycle["pre"]:
                {"down": lambda: self._down(level, sub), "sc": lambda: self._sc(level),
                 "up": lambda: self._up(level)}[kind]()
            if levels > 1:
                self._down(0, cycle["s0"])
            self._sc(0)
            if levels > 1 and cycle["s0"] == 2:
                self._up(0)
        self.sv.raise_pending()


def _bc_spec(d, y0):
    if d == 2:
        faces = {"x_min": OL.LogInlet(0.04, 0.35, y0), "x_max": "outlet",
                 "y_min": "wall", "y_max": "outlet"}
    else:
        faces = {"x_min": OL.LogInlet(0.04, 0.35, y0), "x_max": "outlet",
                 "y_min": "wall", "y_max": "outlet", "z_min": "periodic", "z_max": "periodic"}
    return OL.BoundarySpec(d=d, faces=faces)


@pytest.mark.parametrize("d,levels", [(2, 3), (3, 2)])
def test_naive_reference_order_fp64(d, levels):
    """stream_kernel -> collide_kernel -> boundary_kernel on external 2L
    buffers (test_harness.py:119-146) reproduces the oracle's two-tree run,
    with outlets, a log inlet and a wall, across refinement interfaces."""
    _need_gpu()
    cells = (64, 64) if d == 2 else (32, 32, 32)
    spec = _bc_spec(d, 6.0 if d == 2 else 3.0)
    otopo = oracle_static_refined(cells, levels, central_mask(cells, pad=8 if d == 2 else 4),
                                  periodic=spec.periodic_axes())
    g = (0.0, -1e-5) + ((0.0,) if d == 3 else ())
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 17), spec=spec, gravity=g)
    naive = DeviceNaive(dsv)
    naive.load_from(dsv.pair.trees[0].levels)
    for _ in range(4):
        osv.advance_bounce()
        naive.advance_bounce()
    names = moments(d) + ["eps", "phi"]
    w = compare_levels(otopo, lambda l: last(osv, l), dsv.topology,
                       lambda l: naive.cur(l), names)
    assert max(w.values()) <= 1e-12, w
    # and the device's own fused two-tree run agrees with its per-kernel run
    for _ in range(4):
        dsv.advance_bounce()
    w2 = compare_levels(otopo, lambda l: last(osv, l), dsv.topology, lambda l: last(dsv, l), names)
    assert max(w2.values()) <= 1e-12, w2


@pytest.mark.parametrize("d", [2, 3])
def test_collide_kernel_force_and_tau_arrays_fp64(d):
    """collide_kernel with a per-cell force pair and a per-cell tau array
    (solver.py:410-418) and boundary_kernel alone, vs the oracle."""
    _need_gpu()
    cells = (32, 32) if d == 2 else (16, 16, 16)
    spec = _bc_spec(d, 3.0)
    otopo = OG.Topology.uniform(cells, 1, spec.periodic_axes())
    osv, dsv = build_pair(otopo, torch.float64, smooth_fields(d, 19), spec=spec)
    # the device stores cells in its own slot order: build the per-cell
    # arrays from coordinates so both sides see the same values
    rng = np.random.default_rng(4)
    kf = rng.uniform(0.1, 0.7, size=(d + 1, d))

    def per_cell(pos):
        F = [1e-4 * np.sin(pos @ kf[a]) for a in range(d)]
        tau = 0.8 + 0.3 * (1 + np.sin(pos @ kf[d]))
        return F, tau
    opos = otopo.cell_coords(0).astype(float)
    dpos = dsv.topology.cell_coords(0).astype(float)
    oF, otau = per_cell(opos)
    dF, dtau = per_cell(dpos)
    orr, ow = osv.roles(0)
    osv.stream_kernel(0, osv.arrays(orr, 0), osv.arrays(ow, 0))
    osv.collide_kernel(0, osv.arrays(orr, 0), osv.arrays(ow, 0), force=oF, tau_eff=otau)
    osv.boundary_kernel(0, osv.arrays(ow, 0))
    dr_, dw_ = dsv.roles(0)
    dsv.stream_kernel(0, dsv.arrays(dr_, 0), dsv.arrays(dw_, 0))
    dsv.collide_kernel(0, dsv.arrays(dr_, 0), dsv.arrays(dw_, 0), force=dF, tau_eff=dtau)
    dsv.boundary_kernel(0, dsv.arrays(dw_, 0))
    dsv.raise_pending()
    w = compare_levels(otopo, lambda l: osv.arrays(ow, l), dsv.topology,
                       lambda l: dsv.arrays(dw_, l), moments(d) + ["eps", "phi"])
    assert max(w.values()) <= 1e-13, w


def test_collide_kernel_reports_divergence():
    """Non-physical density after streaming raises DivergenceError with the
    cell coordinates (solver.py:398-406)."""
    _need_gpu()
    from paper_2603_14982_b200.lattice import DivergenceError
    otopo = OG.Topology.uniform((16, 16), 1)
    _, dsv = build_pair(otopo, torch.float64, smooth_fields(2, 1))
    r, w = dsv.roles(0)
    dsv.stream_kernel(0, dsv.arrays(r, 0), dsv.arrays(w, 0))
    dst = dsv.arrays(w, 0)
    rho = dst["rho"].clone()
    pos = dsv.topology.cell_coords(0)
    bad = int(np.nonzero((pos[:, 0] == 5) & (pos[:, 1] == 7))[0][0])
    rho[bad] = -1.0
    dst["rho"] = rho
    dsv.collide_kernel(0, dsv.arrays(r, 0), dst)
    with pytest.raises(DivergenceError) as ei:
        dsv.raise_pending()
    assert ei.value.level == 0 and (5, 7) in [tuple(c) for c in ei.value.cells]


def test_reference_subclass_binding_naive_order():
    """a reference-API solver class (the oracle's Solver,
    which has the reference's signatures — the reference itself does not
    travel to the GPU box) whose five kernel seams are forwarded to
    refbind.B200Kernels, driven in the NaiveReference order on NumPy dicts,
    reproduces the unmodified class on a three-level 2D run with an inlet,
    outlets and a wall; the divergence error type is the caller's."""
    _need_gpu()
    from paper_2603_14982_b200.refbind import B200Kernels

    class Boom(Exception):
        def __init__(self, msg, level=None, cells=None):
            super().__init__(msg)
            self.level, self.cells = level, cells

    class SolverB200(OL.Solver):
        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            # the reference's attribute names (the oracle abbreviates them)
            self.topology, self.level_params, self.boundaries = self.topo, self.lp, self.spec
            self.b200 = B200Kernels(self, divergence_error=Boom)

        def stream_kernel(self, level, src_a, dst):
            self.b200.stream_kernel(level, src_a, dst)

        def collide_kernel(self, level, src_a, dst, force=None, tau_eff=None):
            self.b200.collide_kernel(level, src_a, dst, force, tau_eff)

        def boundary_kernel(self, level, dst):
            self.b200.boundary_kernel(level, dst)

        def downward_kernel(self, level, step, olda, newa, dst):
            self.b200.downward_kernel(level, step, olda, newa, dst)

        def upward_kernel(self, level, fine, dst):
            self.b200.upward_kernel(level, fine, dst)

    cells, levels = (64, 64), 3
    spec = _bc_spec(2, 6.0)
    fn = smooth_fields(2, 29)
    runs = []
    for cls in (OL.Solver, SolverB200):
        otopo = oracle_static_refined(cells, levels, central_mask(cells, pad=8),
                                      periodic=spec.periodic_axes())
        pair = OG.PingPongPair(otopo)
        sv = cls(otopo, pair, OL.SolverParams(levels=levels, gravity=(0.0, -1e-5)),
                 OL.LevelParams(levels, 0.8), spec)
        OL.set_fields(otopo, pair, fn)
        for _ in range(3):
            sv.advance_bounce()
        runs.append((otopo, sv))
    (ot, a), (_, b) = runs
    names = moments(2) + ["eps", "phi"]
    worst = 0.0
    for l in range(levels):
        if not ot.cell_count(l):
            continue
        x, y = last(a, l), last(b, l)
        for nm in names:
            worst = max(worst, float(np.abs(np.asarray(x[nm]) - np.asarray(y[nm])).max()))
    assert worst <= 1e-12, worst
    # a non-physical density surfaces as the caller's exception type
    r, w = b.roles(0)
    dst = b.arrays(w, 0)
    b.stream_kernel(0, b.arrays(r, 0), dst)
    dst["rho"][5] = -1.0
    with pytest.raises(Boom):
        b.collide_kernel(0, b.arrays(r, 0), dst)
