"""Slab decomposition of the coupled multi-level step (static hierarchy) on
one GPU: rank threads exchange ghost columns, P2G ghost sums, particles and
the diagnostics row through a barrier mailbox (the same calls the NCCL path
makes) and must reproduce the single-domain run: particles by id and owned
fields within fp64 atomic-order noise, diagnostics row likewise."""
import threading

import numpy as np
import pytest
import torch

import scenes as S

pytestmark = pytest.mark.gpu
B = pytest.importorskip("paper_2603_14982_b200")


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ref(scene, adapt):
    from paper_2603_14982_b200.harness import build_scene, validate_scene
    sim = build_scene(validate_scene(scene))
    if not adapt:
        sim.adaptor = None      # static hierarchy (the one built around the particles)
    sim.use_graphs = False
    sim.sort_particles = False
    return sim


@pytest.mark.parametrize("scene,world,steps,adapt", [
    (S.COLUMN_3D_SMALL, 2, 6, False), (S.SANDSTORM_3D_SMALL, 2, 6, False),
    (S.COLUMN_3D_SMALL, 2, 8, True), (S.SANDSTORM_3D_SMALL, 2, 8, True),
    (S.CLOUD_3D_SMALL, 3, 14, True),
    # powder transport + entrainment across the cut (stress raster ghost sums,
    # phi ghost columns), the column straddling it
    (S.scene(S.COLUMN_3D_SMALL, powder__enabled=True, powder__entrain=0.02), 2, 10, True)])
def test_coupled_slabs_equal_single_domain(scene, world, steps, adapt):
    _need_gpu()
    from paper_2603_14982_b200.slab_coupled import SlabCoupled, ThreadExchanger
    ref = _ref(scene, adapt)
    base = _ref(scene, adapt)          # identical initial state for the slabs
    if scene is S.CLOUD_3D_SMALL:
        # the two clouds drift towards each other at 0.3 cells/step: tiles are
        # created / retired every few steps and particles cross the cuts
        for sim in (ref, base):
            x = sim.particles.x.cpu().numpy()
            v = np.zeros_like(x)
            v[:, 0] = np.where(x[:, 0] < 48.0, 0.3, -0.3)
            sim.particles.v = v
    xch = ThreadExchanger(world)
    ranks = [SlabCoupled(base, r, world, xch) for r in range(world)]
    errs = []

    def run(sim):
        try:
            torch.cuda.set_device(0)
            for _ in range(steps):
                sim.step()
        except BaseException as e:      # noqa: BLE001
            errs.append(e)
            xch.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in ranks]
    for t in th:
        t.start()
    for _ in range(steps):
        ref.step()
    for t in th:
        t.join()
    assert not errs, errs
    torch.cuda.synchronize()
    # particles by id
    rx = ref.particles.x.cpu().numpy()
    rv = ref.particles.v.cpu().numpy()
    seen = 0
    for r in ranks:
        pid, x, v = r.owned_particles()
        seen += len(pid)
        assert np.abs(x - rx[pid]).max() <= 1e-10, r.rank
        assert np.abs(v - rv[pid]).max() <= 1e-10, r.rank
    assert seen == len(rx)
    # owned level-0 moments
    from paper_2603_14982_b200.sparse_grid import moment_names
    wi = ref.solver.last_roles(0)[1]
    ga = ref.solver.arrays(wi, 0)
    gkey = {tuple(c): i for i, c in enumerate(ref.topology.cell_coords(0).tolist())}
    names = moment_names(ref.d) + (["phi"] if ref.powder is not None else [])
    if ref.powder is not None:
        assert np.abs(ga["phi"].cpu().numpy()).max() > 0.0     # entrainment happened
    for r in ranks:
        for name in names:
            c2, got = r.sl.owned_cells(r.solver.last_roles(0)[1], 0, name)
            want = ga[name].cpu().numpy()[[gkey[tuple(c)] for c in c2.tolist()]]
            assert np.abs(got - want).max() <= 1e-10, (name, r.rank)
    if adapt:
        # block maintenance: every rank holds the same global hierarchy
        for r in ranks:
            assert r.gtopo.tile_set() == ref.topology.tile_set()
        if scene is S.CLOUD_3D_SMALL:      # the churn scene must exercise rebuilds
            assert ref.topology_changes > 0
    # diagnostics row (reduced over ranks)
    dr = ref.diagnostics[-1]
    for r in ranks:
        dd = r.diagnostics[-1]
        assert np.allclose(dd.fluid_mom, dr.fluid_mom, rtol=1e-9, atol=1e-12)
        assert np.allclose(dd.sediment_mom, dr.sediment_mom, rtol=1e-9, atol=1e-12)
        assert abs(dd.eps_min - dr.eps_min) <= 1e-12


def _mp_worker(rank, world, port, scene_name, steps, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import scenes as S2
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2603_14982_b200.slab_coupled import P2PExchanger, SlabCoupled
        base = _ref(getattr(S2, scene_name), True)
        sim = SlabCoupled(base, rank, world, P2PExchanger())
        for _ in range(steps):
            sim.step()
        pid, x, v = sim.owned_particles()
        d = sim.diagnostics[-1]
        q.put((rank, pid, x, v, tuple(d.fluid_mom), tuple(d.sediment_mom),
               sorted(sim.gtopo.tile_set())))
    finally:
        dist.destroy_process_group()


def test_coupled_slabs_two_processes_p2p():
    """The multi-process path (P2PExchanger over a torch.distributed group,
    here gloo with host staging so both processes share cuda:0) reproduces
    the single-domain run."""
    _need_gpu()
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world, steps = 2, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, "SANDSTORM_3D_SMALL", steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    ref = _ref(S.SANDSTORM_3D_SMALL, True)
    for _ in range(steps):
        ref.step()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rx = ref.particles.x.cpu().numpy()
    rv = ref.particles.v.cpu().numpy()
    seen = 0
    for rank, pid, x, v, fm, sm, tiles in out:
        seen += len(pid)
        assert np.abs(x - rx[pid]).max() <= 1e-10, rank
        assert np.abs(v - rv[pid]).max() <= 1e-10, rank
        assert np.allclose(fm, ref.diagnostics[-1].fluid_mom, rtol=1e-9, atol=1e-12)
        assert np.allclose(sm, ref.diagnostics[-1].sediment_mom, rtol=1e-9, atol=1e-12)
        assert set(tiles) == ref.topology.tile_set()
    assert seen == len(rx)
