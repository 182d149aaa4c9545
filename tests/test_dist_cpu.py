"""Multi-rank host logic of the slab decomposition with the
gloo backend, world size 2, on CPU: partition arithmetic, read-tree halo
exchange (a slab-parallel LBM step equals the single-domain step), P2G
ghost-node reduction, particle migration and the seed OR-allreduce."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import lattice as OLat
from paper_2603_14982_b200 import parallel_slabs as PS

WORLD = 2


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def dense_step(lat, f, tau):
    """Single-level periodic pull stream + BGK collide on a dense grid of
    moments f[name] (np.roll transcription, test_solver.py:229-247)."""
    d = lat.d
    ax = "xyz"[:d]
    sp = OLat.s_pairs(d)
    sn = OLat.s_names(d)
    rho, u, s = f["rho"], [f["u" + a] for a in ax], {p: f[n] for p, n in zip(sp, sn)}
    pulled = []
    for i in range(lat.q):
        fi = OLat.reconstruct_dir(lat, i, rho, u, s)
        pulled.append(np.roll(fi, tuple(int(v) for v in lat.c[i]), axis=tuple(range(d))))
    r2, m, pi = OLat.moments_from_f(lat, pulled)
    out = {"rho": r2}
    us = [m[a] / r2 for a in range(d)]
    for a in range(d):
        out["u" + ax[a]] = us[a]
    for (a, b), n in zip(sp, sn):
        out[n] = (1 - 1 / tau) * pi[(a, b)] / r2 + (1 / tau) * us[a] * us[b]
    return out


def random_fields(d, shape, seed):
    rng = np.random.default_rng(seed)
    ax = "xyz"[:d]
    f = {"rho": 1 + 0.02 * rng.random(shape)}
    for a in ax:
        f["u" + a] = 0.04 * (rng.random(shape) - 0.5)
    for (a, b), n in zip(OLat.s_pairs(d), OLat.s_names(d)):
        f[n] = f["u" + ax[a]] * f["u" + ax[b]] + 0.002 * rng.random(shape)
    return f


def _worker(rank, port, case, q, world=WORLD):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, case(rank)))
    finally:
        dist.destroy_process_group()


def run_world(case, world=WORLD):
    port = free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, case, q, world)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


# -- cases (module-level so spawn can pickle them) --------------------------------

def case_lbm_halo_2d(rank):
    return _lbm_halo(rank, 2, (64, 32))


def case_lbm_halo_3d(rank):
    return _lbm_halo(rank, 3, (32, 16, 8))


def _lbm_halo(rank, d, cells):
    lat = OLat.lattice_for(d)
    part = PS.SlabPartition(cells, 2, WORLD)
    g = random_fields(d, cells, 5)
    x0, x1 = part.slab(rank)
    names = list(g)
    loc = torch.as_tensor(np.stack([g[n][x0:x1] for n in names]))
    padded = PS.exchange_halo_x(part, rank, loc, depth=4).numpy()
    fields = {n: padded[i] for i, n in enumerate(names)}
    stepped = dense_step(lat, fields, 0.73)
    return {n: v[4:-4] for n, v in stepped.items()}


def case_ghost_nodes(rank):
    cells = (32, 8)
    part = PS.SlabPartition(cells, 1, WORLD)
    x0, x1 = part.slab(rank)
    rng = np.random.default_rng(7)
    xs = rng.random((400, 2)) * np.array(cells)
    mine = xs[part.owner(xs[:, 0]) == rank]
    acc = np.zeros((1, (x1 - x0) + 4, cells[1]))
    for x in mine:
        base = np.floor(x - 0.5).astype(int)
        f = x - base
        w = [np.array([0.5 * (1.5 - fa) ** 2, 0.75 - (fa - 1) ** 2, 0.5 * (fa - 0.5) ** 2]) for fa in f]
        for ox in range(3):
            for oy in range(3):
                nx = base[0] + ox - x0 + 2          # local index incl. 2 ghost layers
                ny = (base[1] + oy) % cells[1]
                acc[0, nx, ny] += w[0][ox] * w[1][oy]
    # periodic x at the global ends is handled by the neighbour wrap
    out = PS.reduce_ghost_nodes(part, rank, torch.as_tensor(acc), depth=2)
    return out.numpy()


def case_migrate(rank):
    cells = (64, 16)
    part = PS.SlabPartition(cells, 2, WORLD)
    rng = np.random.default_rng(11)
    xs = rng.random((300, 2)) * np.array(cells)
    ids = np.arange(300, dtype=float)
    own = part.owner(xs[:, 0]) == rank
    x = torch.as_tensor(xs[own])
    st = torch.as_tensor(ids[own][:, None])
    moved = x.clone()
    moved[:, 0] = torch.remainder(moved[:, 0] + torch.as_tensor(
        rng.normal(0, 3.0, len(xs))[own]), cells[0])
    nx, ns = PS.migrate_particles(part, rank, moved, st)
    assert (part.owner(nx[:, 0].numpy()) == rank).all()
    return np.concatenate([ns.numpy(), nx.numpy()], axis=1)


def case_seeds(rank):
    seeds = torch.zeros(16, dtype=torch.uint8)
    seeds[rank * 3: rank * 3 + 2] = 1
    seeds[10] = 1 if rank == 1 else 0
    return PS.allreduce_seeds(seeds).numpy()


def case_slab_columns(rank):
    """exchange_columns with 3 ranks, periodic: every rank's ghost columns
    receive its neighbours' edge columns (the device path's exact calls)."""
    from paper_2603_14982_b200.slab_lbm import exchange_columns
    world = dist.get_world_size()
    cols = torch.arange(4 * 6, dtype=torch.float64).reshape(4, 6) + 100 * rank
    lo, hi = cols[:, :3], cols[:, 3:]
    gl, gr = torch.zeros(4, 3, dtype=torch.float64), torch.zeros(4, 3, dtype=torch.float64)
    send = [torch.empty(4, 3, dtype=torch.float64) for _ in range(2)]
    recv = [torch.empty(4, 3, dtype=torch.float64) for _ in range(2)]
    exchange_columns(lo, hi, gl, gr, (rank - 1) % world, (rank + 1) % world, send, recv)
    return gl.numpy(), gr.numpy()


# -- tests --------------------------------------------------------------------------

def test_partition_arithmetic():
    p = PS.SlabPartition((1536, 768, 384), 4, 8)
    c = p.cuts()
    assert c[0] == 0 and c[-1] == 1536 and all(v % 32 == 0 for v in c)
    assert [c[i + 1] - c[i] for i in range(8)] == [192] * 8     # 6 coarse tiles each
    assert p.tile_columns(3, 0) == (144, 192) and p.tile_columns(3, 3) == (18, 24)
    assert p.halo_columns(0, 0) == (383, 48)
    assert p.neighbors(0) == (7, 1)
    assert list(p.owner([0.0, 191.9, 192.0, 1535.9, 1536.2])) == [0, 0, 1, 7, 0]
    q = PS.SlabPartition((128, 64), 2, 3, periodic_x=False)
    assert q.cuts() == [0, 48, 88, 128] and q.neighbors(0) == (None, 1)
    with pytest.raises(ValueError):
        PS.SlabPartition((40, 40), 3, 2)       # 40 not a multiple of 16
    with pytest.raises(ValueError):
        PS.SlabPartition((32, 32), 3, 4)       # 2 coarse columns for 4 ranks


@pytest.mark.parametrize("case,d,cells", [(case_lbm_halo_2d, 2, (64, 32)),
                                          (case_lbm_halo_3d, 3, (32, 16, 8))])
def test_slab_lbm_step_equals_single_domain(case, d, cells):
    out = run_world(case)
    ref = dense_step(OLat.lattice_for(d), random_fields(d, cells, 5), 0.73)
    part = PS.SlabPartition(cells, 2, WORLD)
    for n, v in ref.items():
        got = np.concatenate([out[r][n] for r in range(WORLD)], axis=0)
        assert np.abs(got - v).max() <= 1e-15, n
    assert part.cuts()[-1] == cells[0]


def test_ghost_node_reduction_equals_global_scatter():
    out = run_world(case_ghost_nodes)
    got = np.concatenate([out[r][0] for r in range(WORLD)], axis=0)
    cells = (32, 8)
    rng = np.random.default_rng(7)
    xs = rng.random((400, 2)) * np.array(cells)
    ref = np.zeros(cells)
    for x in xs:
        base = np.floor(x - 0.5).astype(int)
        f = x - base
        w = [np.array([0.5 * (1.5 - fa) ** 2, 0.75 - (fa - 1) ** 2, 0.5 * (fa - 0.5) ** 2]) for fa in f]
        for ox in range(3):
            for oy in range(3):
                ref[(base[0] + ox) % cells[0], (base[1] + oy) % cells[1]] += w[0][ox] * w[1][oy]
    assert np.abs(got - ref).max() <= 1e-12
    assert abs(got.sum() - 400.0) <= 1e-9


def test_particle_migration_conserves_and_routes():
    out = run_world(case_migrate)
    allp = np.concatenate([out[r] for r in range(WORLD)])
    assert sorted(allp[:, 0].astype(int).tolist()) == list(range(300))


def test_seed_or_allreduce():
    out = run_world(case_seeds)
    want = np.zeros(16, dtype=np.uint8)
    want[0:2] = 1
    want[3:5] = 1
    want[10] = 1
    for r in range(WORLD):
        assert np.array_equal(out[r], want)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_column_exchange(world):
    out = run_world(case_slab_columns, world)
    for r in range(world):
        gl, gr = out[r]
        lft, rgt = (r - 1) % world, (r + 1) % world
        base = np.arange(24, dtype=float).reshape(4, 6)
        assert np.array_equal(gl, (base + 100 * lft)[:, 3:]), r      # left neighbour's high edge
        assert np.array_equal(gr, (base + 100 * rgt)[:, :3]), r      # right neighbour's low edge


def case_p2p_exchanger(rank):
    """slab_coupled.P2PExchanger with gloo on CPU tensors: columns, ghost
    sums, particle payloads of ragged sizes, all-reduces."""
    from types import SimpleNamespace
    from paper_2603_14982_b200.slab_coupled import P2PExchanger
    world = dist.get_world_size()
    sl = SimpleNamespace(rank=rank, left=(rank - 1) % world, right=(rank + 1) % world)
    x = P2PExchanger()
    base = torch.arange(12, dtype=torch.float64).reshape(3, 4) + 100 * rank
    el, er = base[:, :2].clone(), base[:, 2:].clone()
    gl, gr = torch.zeros(3, 2, dtype=torch.float64), torch.zeros(3, 2, dtype=torch.float64)
    x.columns(sl, el, er, gl, gr)
    out = {"gl": gl.numpy().copy(), "gr": gr.numpy().copy()}
    ghost_l = torch.full((3, 2), 1.0 + rank, dtype=torch.float64)
    ghost_r = torch.full((3, 2), 10.0 + rank, dtype=torch.float64)
    e_l, e_r = torch.zeros(3, 2, dtype=torch.float64), torch.zeros(3, 2, dtype=torch.float64)
    x.ghost_reduce(sl, ghost_l, ghost_r, e_l, e_r)
    out["el"], out["er"] = e_l.numpy().copy(), e_r.numpy().copy()
    to_l = torch.full((5, rank + 1), -float(rank), dtype=torch.float64)
    to_r = torch.full((5, 2 * rank + 1), float(rank), dtype=torch.float64)
    got = x.particles(sl, to_l, to_r)
    out["got"] = [g.numpy().copy() for g in got]
    # the migration messages of SlabCoupled._migrate: counts, then one byte
    # buffer per direction
    ml, mr = x.migrate_counts(sl, rank + 1, 2 * rank + 1)
    out["mc"] = (ml, mr)
    rl, rr = torch.empty(ml, dtype=torch.uint8), torch.empty(mr, dtype=torch.uint8)
    x.migrate_payload(sl, torch.full((rank + 1,), rank, dtype=torch.uint8),
                      torch.full((2 * rank + 1,), 100 + rank, dtype=torch.uint8), rl, rr)
    out["rl"], out["rr"] = rl.numpy().copy(), rr.numpy().copy()
    t = torch.tensor([float(rank), 5.0 - rank], dtype=torch.float64)
    x.allreduce(sl, t, "sum")
    m = torch.tensor([float(rank)], dtype=torch.float64)
    x.allreduce(sl, m, "max")
    out["sum"], out["max"] = t.numpy().copy(), m.numpy().copy()
    return out


def test_p2p_exchanger_gloo():
    world = 3
    out = run_world(case_p2p_exchanger, world)
    for r in range(world):
        lft, rgt = (r - 1) % world, (r + 1) % world
        base = lambda k: np.arange(12, dtype=float).reshape(3, 4) + 100 * k   # noqa: E731
        o = out[r]
        assert np.array_equal(o["gl"], base(lft)[:, 2:])
        assert np.array_equal(o["gr"], base(rgt)[:, :2])
        assert np.all(o["el"] == 10.0 + lft) and np.all(o["er"] == 1.0 + rgt)
        # got[0]: from the left (its to_right payload), got[1]: from the right (its to_left)
        assert o["got"][0].shape == (5, 2 * lft + 1) and np.all(o["got"][0] == lft)
        assert o["got"][1].shape == (5, rgt + 1) and np.all(o["got"][1] == -rgt)
        assert np.array_equal(o["sum"], [0 + 1 + 2, 15 - 3]) and o["max"][0] == 2
        assert o["mc"] == (2 * lft + 1, rgt + 1)
        assert np.all(o["rl"] == 100 + lft) and len(o["rl"]) == 2 * lft + 1
        assert np.all(o["rr"] == rgt) and len(o["rr"]) == rgt + 1
