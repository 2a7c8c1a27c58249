#!/usr/bin/env python
"""Multi-GPU projection on one B200.

1. Rank-local step: for W = 2, 4, 8 z-slabs of the 216^3 bench lattice, the
   local model of an interior rank (its owned planes + 3 ghost planes per cut)
   is uploaded as a part and stepped alone (same kernel, same brick choice,
   ghost rows not integrated), timed with CUDA events on its stream.  Beside
   the full-lattice step T1 this gives the compute-only strong-scaling
   efficiency T1 / (W * T_rank).
2. Slab barrier: two thread-ranks on this one GPU step a tiny model through
   the real peer-store + slab_sync_kernel path; the per-step cost over the
   same model on one rank is the barrier's floor (NVLink adds its latency).

  python scripts/bench_slab_local.py [--size 216] [--steps 100] > out.json
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

HORIZON = 3.0


def local_lattice(size, z0, z1, g):
    """Owned planes [z0, z1) plus g ghost planes each side (clipped)."""
    import scenarios as S
    from paper_2105_04150_b200 import geometry, make_state
    from paper_2105_04150_b200.types import (BoundaryConditions, Corrections, DamageLaw,
                                             DamageModel, ModelBundle, ParticleSet)
    zl0, zl1 = max(0, z0 - g), min(size, z1 + g)
    grid = geometry.GridDesc((0.0, 0.0, float(zl0)), 1.0, (size, size, zl1 - zl0))
    coords = geometry.grid_coordinates(grid)
    nl = grid.node_count()
    particles = ParticleSet(coords, np.ones(nl), np.ones(nl), np.zeros(nl, np.uint16))
    bundle = ModelBundle(particles, DamageModel([DamageLaw.pmb(1.0, 1e6)]), Corrections(),
                         BoundaryConditions.none(nl), 1e-3)
    fam = geometry.build_family(coords, HORIZON, grid)
    state = make_state(fam, False)
    state.u = S.seed_displacements(coords)
    plane = size * size
    return bundle, state, (z0 - zl0) * plane, (z1 - zl0) * plane, fam


def time_part(bundle, state, ob, oe, variant, steps, warmup):
    import torch
    from paper_2105_04150_b200 import IntegratorKind, engine
    ctx = engine.Context(0)
    ctx.upload_part(bundle, state, variant, ob, oe)
    stream = torch.cuda.ExternalStream(ctx.stream())
    ctx.run(warmup, 0, IntegratorKind.velocity_verlet, 0, variant)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.run(steps, warmup, IntegratorKind.velocity_verlet, 0, variant)
    e1.record(stream)
    torch.cuda.synchronize()
    kernel = ctx.kernel()
    ctx.close()
    return e0.elapsed_time(e1) / steps, kernel


def barrier_cost(steps, counts=(16, 16, 24)):
    """us/step of the slab barrier: a small model (one kernel per step
    ~ latency-bound) stepped by 2 thread-ranks on this GPU (peer stores +
    slab_sync_kernel per step) against the same model on 1 rank; only the
    stepping of already connected ranks is timed (CUDA events + wall)."""
    import threading

    import torch

    import scenarios as S
    from paper_2105_04150_b200 import IntegratorKind, KernelVariant, engine, geometry, make_state
    from paper_2105_04150_b200 import slabs
    b, h, g = S.bench_lattice_bundle(counts)
    fam = geometry.build_family(b.particles.coords, h, g)
    st = make_state(fam, False)
    st.u = S.seed_displacements(b.particles.coords)
    variant = KernelVariant.bond_parallel
    out = {}
    # one rank
    ctx = engine.Context(0)
    ctx.upload(b, st, variant)
    ctx.run(10, 0, IntegratorKind.velocity_verlet, 0, variant)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.run(steps, 10, IntegratorKind.velocity_verlet, 0, variant)
    torch.cuda.synchronize()
    out[1] = (time.perf_counter() - t0) / steps
    ctx.close()
    # two thread-ranks
    world = 2
    comms = slabs.ThreadComm.group(world)
    ranges = slabs.partition(b.particles.coords, world)
    parts = slabs.plan(b.particles.coords, fam.entries, int(fam.group_size), world, ranges)
    ranks = [None] * world
    times = [0.0] * world

    def setup(r):
        bl, sl = slabs.local_problem(parts[r], b, st)
        ranks[r] = slabs.SlabRank(comms[r], 0)
        ranks[r].setup(parts[r], ranges, bl, sl, variant)
        ranks[r].run(10, 0, IntegratorKind.velocity_verlet)
        comms[r].allgather(None)
        t = time.perf_counter()
        ranks[r].run(steps, 10, IntegratorKind.velocity_verlet)
        torch.cuda.synchronize()
        times[r] = time.perf_counter() - t

    th = [threading.Thread(target=setup, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in ranks:
        r.close()
    out[2] = max(times) / steps
    return {"model": f"{counts[0]}x{counts[1]}x{counts[2]} lattice, exact variant, velocity-Verlet",
            "steps": steps, "us_per_step_1_rank": 1e6 * out[1],
            "us_per_step_2_thread_ranks": 1e6 * out[2],
            "barrier_us_per_step": 1e6 * (out[2] - out[1]),
            "note": "stepping of connected ranks only (wall clock around run() + synchronize); "
                    "both ranks share this one GPU, so their kernels also compete for it"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=216)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--variant", default="fast", choices=["fast", "exact"])
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--barrier-only", action="store_true")
    args = ap.parse_args()
    from paper_2105_04150_b200 import KernelVariant
    variant = KernelVariant.fast if args.variant == "fast" else KernelVariant.bond_parallel
    g = int(math.ceil(HORIZON))
    size = args.size
    if args.barrier_only:
        print(json.dumps({"barrier": barrier_cost(2000)}))
        return 0
    rows = []
    t1 = None
    for world in [int(w) for w in args.worlds.split(",")]:
        cuts = [int(round(r * size / world)) for r in range(world + 1)]
        r = world // 2 if world > 1 else 0
        z0, z1 = cuts[r], cuts[r + 1]
        bundle, state, ob, oe, fam = local_lattice(size, z0, z1, g)
        ms, kernel = time_part(bundle, state, ob, oe, variant, args.steps, args.warmup)
        live = int(fam.n_neigh[ob:oe].sum())
        if world == 1:
            t1 = ms
        row = {"world": world, "rank": r, "owned_planes": z1 - z0,
               "local_planes": z1 - z0 + (z0 - max(0, z0 - g)) + (min(size, z1 + g) - z1),
               "ms_per_step": ms, "kernel": kernel, "live_bonds_owned": live,
               "bond_evals_per_s": live / (ms / 1e3)}
        if t1 is not None:
            row["compute_efficiency"] = t1 / (world * ms)
        rows.append(row)
        print(json.dumps(row), file=sys.stderr)
        del bundle, state, fam
    out = {"lattice": f"{size}^3", "variant": args.variant, "ranks": rows,
           "barrier": barrier_cost(2000)}
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
