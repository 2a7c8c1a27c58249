"""Multi-GPU z-slab decomposition of the time step.

The reference is single-process (`parallel_chunks`, src/parallel.cpp:42-75,
splits contiguous node ranges over threads of one host).  Here one process
(or one thread, for in-process ranks) drives one GPU; rank r owns a contiguous
range of the reference's node numbering.  On the reference's lattices
(grid_coordinates, geometry.cpp:25-38: x fastest, z slowest) that range is a
stack of whole z-planes, so its neighbours live only in the slabs above and
below.  Each rank holds a LOCAL model:

    local nodes = owned nodes + ghosts (every node an owned row references),
    numbered in ascending reference order, so the owned nodes are the
    contiguous range [own_begin, own_end) and every owned row keeps its slot
    order (the exact variants stay bitwise equal to one GPU).

Per time step the fused step kernel stores the new displacement of each owned
node that is a ghost elsewhere straight into the neighbour's u buffer (peer
memory over NVLink), and a one-thread sync kernel publishes the step to every
rank (csrc/pd_aux.cu slab_sync_kernel).  The host exchanges only the
pd_peer_handle records, once, through a `Comm`: torch.distributed (NCCL or
gloo) across processes, or `ThreadComm` for ranks that share one process.

Write steps (tip records, write hooks) and the final state are gathered on the
host: every rank contributes its owned rows and every rank receives the global
state (SPMD, like the reference's single process).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np

from .types import (BoundaryConditions, Corrections, ForceField, IntegratorKind, KernelVariant,
                    ModelBundle, NeighborList, ParticleSet, SimulateOptions, SimulateResult,
                    SimulationState, TipRecord)


# ---- communication -----------------------------------------------------------

class Comm:
    rank: int = 0
    world: int = 1

    def allgather(self, obj):  # pragma: no cover - interface
        raise NotImplementedError


class TorchComm(Comm):
    """torch.distributed all_gather_object over an initialised process group
    (NCCL between GPU processes, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allgather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


class ThreadComm(Comm):
    """Ranks that are threads of one process (several slabs on one GPU)."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.slots = [None] * world
            self.barrier = threading.Barrier(world)

    def __init__(self, shared: "ThreadComm._Shared", rank: int):
        self.shared = shared
        self.rank = rank
        self.world = shared.world

    @classmethod
    def group(cls, world: int) -> List["ThreadComm"]:
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def allgather(self, obj):
        sh = self.shared
        sh.slots[self.rank] = obj
        sh.barrier.wait()
        out = list(sh.slots)
        sh.barrier.wait()
        return out


# ---- partition ---------------------------------------------------------------

@dataclass
class SlabPart:
    rank: int
    world: int
    g_begin: int            # owned reference node ids [g_begin, g_end)
    g_end: int
    local_ids: np.ndarray   # reference ids of the local nodes, ascending (int64)
    own_begin: int          # owned range in the local numbering
    own_end: int
    lo: int                 # neighbour ranks (-1: none)
    hi: int

    @property
    def n_local(self) -> int:
        return int(self.local_ids.size)

    def ghosts_of(self, owner: int, ranges: Sequence[tuple]) -> np.ndarray:
        """Local ids of this part's ghosts owned by rank `owner`."""
        b, e = ranges[owner]
        ids = self.local_ids
        return np.flatnonzero((ids >= b) & (ids < e))


def partition(coords: np.ndarray, world: int) -> List[tuple]:
    """Contiguous reference-index ranges of near-equal size.  When the nodes
    are z-sorted (the lattice order) each cut is moved to the nearest start of
    a z-plane, so slabs are whole planes."""
    n = np.asarray(coords).size // 3
    if world < 1 or world > n:
        raise ValueError(f"slabs: cannot split {n} nodes over {world} ranks")
    z = np.asarray(coords, dtype=np.float64)[2::3]
    starts = None
    if n > 1 and np.all(np.diff(z) >= 0):
        starts = np.flatnonzero(np.diff(z) > 0) + 1
    cuts = [0]
    for r in range(1, world):
        c = int(round(r * n / world))
        if starts is not None and starts.size:
            k = int(np.argmin(np.abs(starts - c)))
            c = int(starts[k])
        if c <= cuts[-1]:
            raise ValueError("slabs: fewer z-planes than ranks")
        cuts.append(c)
    cuts.append(n)
    if cuts[-2] >= n:
        raise ValueError("slabs: fewer z-planes than ranks")
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def plan(coords: np.ndarray, entries: np.ndarray, group_size: int, world: int,
         ranges: Optional[List[tuple]] = None) -> List[SlabPart]:
    """Slab parts of every rank from the global rows.  Raises ValueError when a
    slab is thinner than the horizon (a row reaches past the next slab)."""
    n = np.asarray(coords).size // 3
    N = int(group_size)
    ent = np.asarray(entries, dtype=np.int32).reshape(n, N)
    ranges = ranges or partition(coords, world)
    parts = []
    for r, (b, e) in enumerate(ranges):
        rows = ent[b:e]
        cross = rows[(rows >= 0) & ((rows < b) | (rows >= e))]
        ghosts = np.unique(cross).astype(np.int64)
        lo = r - 1 if r > 0 else -1
        hi = r + 1 if r + 1 < world else -1
        ok_lo = (ghosts >= ranges[lo][0]) & (ghosts < ranges[lo][1]) if lo >= 0 else False
        ok_hi = (ghosts >= ranges[hi][0]) & (ghosts < ranges[hi][1]) if hi >= 0 else False
        if ghosts.size and not np.all(ok_lo | ok_hi):
            raise ValueError(f"slabs: rank {r}'s rows reach past its neighbouring slabs "
                             f"(slab thinner than the horizon); use fewer ranks")
        g_lo = ghosts[ghosts < b]
        g_hi = ghosts[ghosts >= e]
        local = np.concatenate([g_lo, np.arange(b, e, dtype=np.int64), g_hi])
        parts.append(SlabPart(r, world, b, e, local, int(g_lo.size), int(g_lo.size + e - b),
                              lo, hi))
    return parts


def local_problem(part: SlabPart, bundle: ModelBundle, state: SimulationState):
    """The rank's local ModelBundle / SimulationState (tips are handled on the
    host, so the local bundle has none)."""
    ids = part.local_ids
    n = bundle.particles.size()
    nl = ids.size
    N = int(state.connectivity.group_size)
    g2l = np.full(n, -1, np.int32)
    g2l[ids] = np.arange(nl, dtype=np.int32)
    ob, oe = part.own_begin, part.own_end
    gb, ge = part.g_begin, part.g_end

    def rows3(a):
        return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(n, 3)[ids]).ravel()

    p = bundle.particles
    particles = ParticleSet(rows3(p.coords), np.asarray(p.volume, np.float64)[ids].copy(),
                            np.asarray(p.density, np.float64)[ids].copy())
    fam = state.connectivity
    ent = np.asarray(fam.entries, np.int32).reshape(n, N)[gb:ge]
    loc = np.full((nl, N), -1, np.int32)
    live = ent >= 0
    own = loc[ob:oe]
    own[live] = g2l[ent[live]]
    n_neigh = np.zeros(nl, np.int32)
    n_neigh[ob:oe] = np.asarray(fam.n_neigh)[gb:ge]
    initial = np.zeros(nl, np.int32)
    initial[ob:oe] = np.asarray(fam.initial_n_neigh)[gb:ge]

    def slot_rows(a, fill, dtype):
        if a is None or np.asarray(a).size == 0:
            return None
        out = np.full((nl, N), fill, dtype)
        out[ob:oe] = np.asarray(a, dtype).reshape(n, N)[gb:ge]
        return out.ravel()

    bt = slot_rows(fam.bond_type, 0, np.uint8)
    conn = NeighborList(loc.ravel(), n_neigh, initial, N, float(fam.horizon), bt)
    hist = slot_rows(state.bond_history, 0.0, np.float64)
    st = SimulationState(rows3(state.u), rows3(state.v), rows3(state.a), int(state.step), conn,
                         hist if hist is not None else np.zeros(0))
    c = bundle.corrections
    nf = None if c.no_failure is None or np.asarray(c.no_failure).size == 0 else \
        np.asarray(c.no_failure, np.uint8)[ids].copy()
    corr = Corrections(slot_rows(c.lambda_, 1.0, np.float64), slot_rows(c.beta, 1.0, np.float64),
                       nf)
    bc = bundle.bc
    k3 = np.asarray(bc.kind, np.uint8).reshape(n, 3)[ids].ravel()
    lbc = BoundaryConditions(k3.copy(), rows3(bc.magnitude),
                             np.asarray(bc.ramp_id, np.uint8).reshape(n, 3)[ids].ravel().copy(),
                             list(bc.ramps), np.asarray(bc.no_failure, np.uint8)[ids].copy(), {})
    return ModelBundle(particles, bundle.model, corr, lbc, bundle.dt), st


def send_maps(part: SlabPart, ranges, ghost_rows_of_all) -> tuple:
    """send_lo / send_hi for pd_ctx_connect: for each local owned node the
    device row it occupies on rank lo / hi (-1 if it is not a ghost there).
    ghost_rows_of_all[q] = {"lo": (ref ids, rows), "hi": (ref ids, rows)}: rank
    q's ghosts owned by q-1 ("lo") and by q+1 ("hi") with their device rows."""
    nl = part.n_local
    out = []
    for side, peer, key in (("lo", part.lo, "hi"), ("hi", part.hi, "lo")):
        arr = np.full(nl, -1, np.int64)
        if peer >= 0:
            gids, rows = ghost_rows_of_all[peer][key]
            loc = np.searchsorted(part.local_ids, gids)
            if gids.size and not np.array_equal(part.local_ids[loc], gids):
                raise RuntimeError("slabs: ghost map mismatch between neighbouring ranks")
            arr[loc] = rows
        out.append(arr)
    return out[0], out[1]


# ---- the rank driver ------------------------------------------------------------

def _tip_records(bundle: ModelBundle, values: dict, step: int) -> dict:
    """record_tips (engine.cpp:349-370) from gathered per-node values, summed
    in set order with plain IEEE double adds (Python floats)."""
    out = {}
    for name in sorted(bundle.bc.tip_sets):
        nodes = bundle.bc.tip_sets[name]
        acc = [[0.0, 0.0, 0.0] for _ in range(5)]
        for i in nodes:
            row = values[int(i)]
            for f in range(5):
                for ax in range(3):
                    acc[f][ax] = acc[f][ax] + float(row[3 * f + ax])
        if len(nodes):
            inv = 1.0 / float(len(nodes))
            for f in range(3):
                acc[f] = [x * inv for x in acc[f]]
        out[name] = TipRecord(int(step), *[np.array(a) for a in acc])
    return out


class SlabRank:
    """One rank of a slab-decomposed simulation (one GPU)."""

    def __init__(self, comm: Comm, device: int = 0):
        from .engine import Context
        self.comm = comm
        self.ctx = Context(device)

    def setup(self, part: SlabPart, ranges, bundle_l: ModelBundle, state_l: SimulationState,
              variant) -> None:
        self.part = part
        self.ranges = ranges
        self.variant = variant
        ctx = self.ctx
        ctx.upload_part(bundle_l, state_l, variant, part.own_begin, part.own_end)
        handles = self.comm.allgather(ctx.export())
        mine = {}
        for key, owner in (("lo", part.lo), ("hi", part.hi)):
            if owner < 0:
                mine[key] = (np.zeros(0, np.int64), np.zeros(0, np.int64))
                continue
            loc = part.ghosts_of(owner, ranges)
            mine[key] = (part.local_ids[loc], ctx.internal_index(loc))
        allg = self.comm.allgather(mine)
        send_lo, send_hi = send_maps(part, ranges, allg)
        ctx.connect(part.rank, part.world, handles, part.lo, part.hi, send_lo, send_hi)
        # no rank may start spinning in a sync kernel before every rank has
        # loaded its kernels (pd_ctx_connect)
        self.comm.allgather(None)

    def run(self, steps: int, first_step: int, integrator, variant=None) -> None:
        self.ctx.run(steps, first_step, integrator, 0,
                     self.variant if variant is None else variant)

    def gather_state(self, state: SimulationState, with_forces: bool = False) -> Optional[ForceField]:
        """Every rank's owned rows into the global `state` (on every rank)."""
        from .types import make_state
        part = self.part
        nl = part.n_local
        N = self.ctx.N
        loc = make_state(NeighborList(np.full(nl * N, -1, np.int32), np.zeros(nl, np.int32),
                                      np.zeros(nl, np.int32), N), self.ctx.history)
        ff = ForceField() if with_forces else None
        self.ctx.download(loc, ff)
        ob, oe = part.own_begin, part.own_end
        ids = part.local_ids
        ent = loc.connectivity.entries.reshape(nl, N)[ob:oe]
        gent = np.where(ent >= 0, ids[np.maximum(ent, 0)], -1).astype(np.int32)
        mine = {"range": (part.g_begin, part.g_end),
                "u": loc.u.reshape(nl, 3)[ob:oe], "v": loc.v.reshape(nl, 3)[ob:oe],
                "a": loc.a.reshape(nl, 3)[ob:oe], "entries": gent,
                "n_neigh": loc.connectivity.n_neigh[ob:oe],
                "hist": loc.bond_history.reshape(nl, N)[ob:oe] if self.ctx.history else None,
                "step": loc.step}
        if ff is not None:
            mine["body"] = ff.body_force.reshape(nl, 3)[ob:oe]
            mine["ext"] = ff.external_force.reshape(nl, 3)[ob:oe]
        parts = self.comm.allgather(mine)
        n = state.size()
        out_ff = ForceField(np.zeros(3 * n), np.zeros(3 * n)) if with_forces else None
        U, V, A = (x.reshape(n, 3) for x in (state.u, state.v, state.a))
        E = state.connectivity.entries.reshape(n, N)
        H = state.bond_history.reshape(n, N) if self.ctx.history else None
        for m in parts:
            b, e = m["range"]
            U[b:e], V[b:e], A[b:e] = m["u"], m["v"], m["a"]
            E[b:e] = m["entries"]
            state.connectivity.n_neigh[b:e] = m["n_neigh"]
            if H is not None:
                H[b:e] = m["hist"]
            if out_ff is not None:
                out_ff.body_force.reshape(n, 3)[b:e] = m["body"]
                out_ff.external_force.reshape(n, 3)[b:e] = m["ext"]
        state.step = parts[0]["step"]
        return out_ff

    def gather_tip_values(self, bundle: ModelBundle) -> dict:
        part = self.part
        want = sorted({int(i) for s in bundle.bc.tip_sets.values() for i in s
                       if part.g_begin <= int(i) < part.g_end})
        g = np.array(want, dtype=np.int64)
        loc = np.searchsorted(part.local_ids, g)
        vals = self.ctx.node_values(loc)
        merged = {}
        for d in self.comm.allgather(dict(zip(want, vals))):
            merged.update(d)
        return merged

    def close(self) -> None:
        self.ctx.close()


def simulate_slabs(bundle: ModelBundle, state: SimulationState, options: SimulateOptions,
                   on_write: Optional[Callable[[SimulationState, ForceField], None]] = None,
                   comm: Optional[Comm] = None, device: int = 0) -> SimulateResult:
    """simulate() (engine.hpp:128-129) over comm.world GPUs, SPMD: every rank
    passes the same global bundle and state and gets the global result."""
    from .abi import PeridynRuntimeError
    comm = comm or TorchComm()
    if options.steps < 1:
        from .abi import InvalidArgument
        raise InvalidArgument("simulate: steps must be >= 1")
    n = bundle.particles.size()
    N = int(state.connectivity.group_size)
    if bundle.model.needs_history() and np.asarray(
            state.bond_history if state.bond_history is not None else []).size != n * N:
        state.bond_history = np.zeros(n * N)  # engine.cpp:382-384
    ranges = partition(bundle.particles.coords, comm.world)
    parts = plan(bundle.particles.coords, state.connectivity.entries, N, comm.world, ranges)
    part = parts[comm.rank]
    bundle_l, state_l = local_problem(part, bundle, state)
    rank = SlabRank(comm, device)
    result = SimulateResult({name: [] for name in sorted(bundle.bc.tip_sets)})
    try:
        rank.setup(part, ranges, bundle_l, state_l, options.variant)
        first, last = options.first_step, options.first_step + options.steps
        needs_writes = options.write_every > 0 and (on_write is not None or bundle.bc.tip_sets)
        s = first
        while s < last:
            nxt = last
            if needs_writes:
                w = (s // options.write_every + 1) * options.write_every
                nxt = min(last, w)
            try:
                # a run split at write steps is a restart, bitwise equal to an
                # uninterrupted run (engine.cpp:393-396; test_engine.cpp:443-470)
                rank.run(nxt - s, s, options.integrator)
            except PeridynRuntimeError:
                rank.gather_state(state)
                raise
            s = nxt
            if needs_writes and s % options.write_every == 0:
                if bundle.bc.tip_sets:
                    vals = rank.gather_tip_values(bundle)
                    for name, rec in _tip_records(bundle, vals, s).items():
                        result.tips[name].append(rec)
                if on_write is not None:
                    ff = rank.gather_state(state, with_forces=True)
                    on_write(state, ff)
        rank.gather_state(state)
    finally:
        rank.close()
    return result


def simulate_slabs_local(bundle: ModelBundle, state: SimulationState, options: SimulateOptions,
                         world: int, device: int = 0, on_write=None) -> SimulateResult:
    """`world` slab ranks as threads of this process on one device (testing the
    multi-GPU path on a single GPU: peer stores become same-device stores)."""
    comms = ThreadComm.group(world)
    results: List = [None] * world
    errors: List = [None] * world
    states = [state] + [SimulationState(state.u.copy(), state.v.copy(), state.a.copy(), state.step,
                                        state.connectivity.copy(),
                                        None if state.bond_history is None
                                        else np.array(state.bond_history, copy=True))
                        for _ in range(world - 1)]

    def body(r):
        hook = on_write if (r == 0 or on_write is None) else (lambda st, ff: None)
        try:
            results[r] = simulate_slabs(bundle, states[r], options, hook, comms[r], device)
        except BaseException as e:  # noqa: BLE001 - re-raised on the caller's thread
            errors[r] = e

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    return results[0]
