"""Checkpoint / resume of a coupled simulation (the
reference has none).

A checkpoint holds everything the next step reads: the tile set of every
level (the sorted slot order is a function of it), both ping-pong trees of
every level, the level step counters and the buffer bounce, the step count,
the int16 hysteresis streaks, and the particle state in storage order with
its id map.  Rasters, tables and graphs are derived and rebuilt on load.
Resuming into a simulation built from the same scene continues the run.
"""
from __future__ import annotations

import torch

FORMAT = 1


def save_checkpoint(path, sim):
    torch.cuda.synchronize()
    topo, pair, solver = sim.topology, sim.pair, sim.solver
    L = topo.levels
    p = sim.particles
    state = {
        "format": FORMAT, "d": topo.d, "levels": L, "finest": tuple(topo.finest_cells),
        "dtype": str(pair.dtype),
        # (level, tile coords, kind) rows as one int64 tensor: the file holds only
        # tensors and plain containers, so it loads with weights_only=True
        "tiles": torch.tensor(sorted(topo.tile_set()), dtype=torch.int64).reshape(-1, 2 + topo.d),
        # logical tree order (a level whose trees swapped places is saved
        # unswapped), so a restored run starts with no swap
        "trees": [[pair.trees[t ^ solver.flip[l]].levels[l].data[:, :topo.cell_count(l)].cpu().clone()
                   for l in range(L)] for t in range(2)],
        "k": list(solver.k), "bounce": pair.bounce, "step_count": sim.step_count,
        "streaks": ([s.cpu().clone() for s in sim.adaptor._streak]
                    if sim.adaptor is not None else None),
        "particles": {"xd": p.xd.cpu().clone(), "pd": p.pd.cpu().clone(),
                      "pid": p.pid.cpu().clone(), "permuted": p.permuted,
                      "stress_valid": p.stress_mat is not None},
        "topology_changes": sim.topology_changes,
    }
    torch.save(state, path)


def load_checkpoint(path, sim):
    """Restore ``sim`` (built from the same scene) to the saved state."""
    st = torch.load(path, weights_only=True)
    topo, pair, solver = sim.topology, sim.pair, sim.solver
    if st.get("format") != FORMAT:
        raise ValueError(f"unsupported checkpoint format {st.get('format')}")
    if (st["d"], st["levels"], tuple(st["finest"])) != (topo.d, topo.levels, tuple(topo.finest_cells)):
        raise ValueError("checkpoint does not match this scene's domain / levels")
    if st["dtype"] != str(pair.dtype):
        raise ValueError(f"checkpoint dtype {st['dtype']} != {pair.dtype}")
    torch.cuda.synchronize()
    topo.set_tile_set({tuple(int(v) for v in row) for row in st["tiles"].tolist()})
    pair.ensure_capacity()
    for t in range(2):
        for l in range(topo.levels):
            src = st["trees"][t][l]
            pair.trees[t].levels[l].data[:, :src.shape[1]].copy_(src.to(topo.device))
    solver.k[:] = list(st["k"])
    solver.flip[:] = [0] * topo.levels
    pair.bounce = st["bounce"]
    sim.step_count = st["step_count"]
    sim.topology_changes = st.get("topology_changes", 0)
    if st["streaks"] is not None and sim.adaptor is not None:
        for a, b in zip(sim.adaptor._streak, st["streaks"]):
            a.copy_(b.to(a.device))
    ps = st["particles"]
    p = sim.particles
    if ps["xd"].shape != p.xd.shape or ps["pd"].shape != p.pd.shape:
        raise ValueError("checkpoint particle count / layout does not match")
    p.xd.copy_(ps["xd"].to(p.device))
    p.pd.copy_(ps["pd"].to(p.device))
    p.pid.copy_(ps["pid"].to(p.device))
    p.permuted = ps["permuted"]
    # the tau rows were saved with the state they describe
    p.stress_mat = ((float(sim.material.lam), float(sim.material.mu))
                    if ps.get("stress_valid") else None)
    # derived state: tables, rasters, captured graphs
    solver._tables_version = -1
    solver._refresh_tables()
    sim.grid.sync_topology()
    sim._graphs.clear()
    sim._graph_ver = None
    sim._pool = None
    sim._sorted_ahead = sim._sort_ahead = sim._use_sorted = False
    if hasattr(sim, "_rb_ver"):
        sim._rb_ver = None
    torch.cuda.synchronize()
