"""TEST INFRASTRUCTURE: the slab decomposition of paper_2105_04150_b200.slabs
driven on the CPU with the C oracle as each rank's "device".

Each rank runs one-step simulate() calls of the oracle on its LOCAL problem
(slabs.local_problem) and, between steps, sends the u, v, a of its owned
nodes that are ghosts on the neighbouring ranks through the same send maps
the GPU path hands to pd_ctx_connect (slabs.send_maps, with device row =
local id).  A one-step simulate is a restart (bitwise equal to continuing,
engine.cpp:393-396), and a ghost's drift/BC positions are computed from exact
copies of its owner's inputs, so the owned rows must come out bitwise equal
to the global run: this checks the partition, the local problems, the ghost
maps and the gather without a GPU."""
import numpy as np

from paper_2105_04150_b200 import slabs
from paper_2105_04150_b200.types import SimulateOptions


def emulate(oracle, bundle, state, options, comm):
    n = bundle.particles.size()
    N = int(state.connectivity.group_size)
    if bundle.model.needs_history() and np.asarray(state.bond_history).size != n * N:
        state.bond_history = np.zeros(n * N)
    ranges = slabs.partition(bundle.particles.coords, comm.world)
    parts = slabs.plan(bundle.particles.coords, state.connectivity.entries, N, comm.world, ranges)
    part = parts[comm.rank]
    bl, sl = slabs.local_problem(part, bundle, state)
    # device rows == local ids on the oracle
    mine = {}
    for key, owner in (("lo", part.lo), ("hi", part.hi)):
        loc = part.ghosts_of(owner, ranges) if owner >= 0 else np.zeros(0, np.int64)
        mine[key] = (part.local_ids[loc], loc.astype(np.int64))
    send_lo, send_hi = slabs.send_maps(part, ranges, comm.allgather(mine))
    nl = part.n_local
    ob, oe = part.own_begin, part.own_end
    for s in range(options.first_step, options.first_step + options.steps):
        oracle.simulate(bl, sl, SimulateOptions(1, 0, s, options.integrator, options.variant))
        # ghost exchange: rows for each neighbour
        out = {}
        for peer, smap in ((part.lo, send_lo), (part.hi, send_hi)):
            if peer < 0:
                continue
            idx = np.flatnonzero(smap[ob:oe] >= 0) + ob
            out[peer] = (smap[idx], sl.u.reshape(nl, 3)[idx].copy(),
                         sl.v.reshape(nl, 3)[idx].copy(), sl.a.reshape(nl, 3)[idx].copy())
        got = comm.allgather(out)
        for q in range(comm.world):
            if comm.rank in got[q]:
                rows, u, v, a = got[q][comm.rank]
                sl.u.reshape(nl, 3)[rows] = u
                sl.v.reshape(nl, 3)[rows] = v
                sl.a.reshape(nl, 3)[rows] = a
    # gather owned rows into the global state
    ids = part.local_ids
    ent = sl.connectivity.entries.reshape(nl, N)[ob:oe]
    gent = np.where(ent >= 0, ids[np.maximum(ent, 0)], -1).astype(np.int32)
    m = {"range": (part.g_begin, part.g_end), "u": sl.u.reshape(nl, 3)[ob:oe],
         "v": sl.v.reshape(nl, 3)[ob:oe], "a": sl.a.reshape(nl, 3)[ob:oe], "entries": gent,
         "n_neigh": sl.connectivity.n_neigh[ob:oe],
         "hist": np.asarray(sl.bond_history).reshape(nl, N)[ob:oe]
         if bundle.model.needs_history() else None}
    for g in comm.allgather(m):
        b, e = g["range"]
        state.u.reshape(n, 3)[b:e] = g["u"]
        state.v.reshape(n, 3)[b:e] = g["v"]
        state.a.reshape(n, 3)[b:e] = g["a"]
        state.connectivity.entries.reshape(n, N)[b:e] = g["entries"]
        state.connectivity.n_neigh[b:e] = g["n_neigh"]
        if g["hist"] is not None:
            state.bond_history.reshape(n, N)[b:e] = g["hist"]
    state.step = options.first_step + options.steps
    return parts
