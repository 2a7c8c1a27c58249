#!/usr/bin/env python
"""Benchmark: explicit bond-based peridynamics time step on B200.

Workload (BASELINE.json configs[3], at N=1 the metric's 10M-node case): the
reference bench lattice (bench.cpp:76-104) -- cubic lattice 216^3 =
10,077,696 nodes, spacing 1, V = rho = 1, PMB c = 1, s_c = 1e6 (no breaking),
dt = 1e-3, horizon 3 (N = 128, 1,209,979,144 live directed bonds), seeded u,
velocity-Verlet.  One "step" = one simulate() time step (fused force + break +
reduce + kick + next drift), run device-resident through the C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--variant fast|exact]
  python bench.py --impl reference      # the reference CPU path on host cores

Prints ONE JSON line (rank 0).  Metric: live directed bond evaluations per
second (whole job), with ms/step, the HBM roofline of the fused step kernel,
an end-to-end number through the host-buffer simulate() call, the reference
CPU baseline and the SM clocks seen during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "bond evals/sec & ms/step at 1M/10M nodes; % of HBM peak; 1/2/4/8 GPU"
UNIT = "bond_evals/s"
HORIZON = 3.0


def algorithmic_bytes(n: int, N: int, live: int, r: int = 8) -> int:
    """4B + 2 ceil(nN/8) + n (7*3r + 2r)."""
    return 4 * live + 2 * ((n * N + 7) // 8) + n * (7 * 3 * r + 2 * r)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, flag in zip(names, f[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_traffic(key):
    """DRAM bytes per launch of the step kernel from the committed ncu capture
    (profiles/traffic.json, written from `ncu --set full`), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p))[key]["traffic_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def rebar_bond_types(counts, fam):
    """cfg5-style bond classes on the lattice (SURVEY 8(d) realisation of the RC
    beam): two rebar lines along x at (y, z) = (ny/4, nz/5) and (3ny/4, nz/5);
    type 1 = steel-steel (both ends on a rebar), 2 = interface (one end), 0 =
    concrete.  Only rebar rows and rows that reach a rebar node carry types."""
    nx, ny, nz = counts
    n, N = fam.node_count(), int(fam.group_size)
    ent = fam.entries.reshape(n, N)
    on = np.zeros(n, bool)
    for y in (ny // 4, (3 * ny) // 4):
        z = nz // 5
        on[np.arange(nx) + nx * (y + ny * z)] = True
    bt = np.zeros((n, N), np.uint8)
    rebar = np.flatnonzero(on)
    rows = ent[rebar]
    bt[rebar] = np.where(rows >= 0, np.where(on[np.maximum(rows, 0)], 1, 2), 0)
    near = np.unique(rows[rows >= 0])
    near = near[~on[near]]
    nrows = ent[near]
    bt[near] = np.where((nrows >= 0) & on[np.maximum(nrows, 0)], 2, 0)
    return bt.reshape(-1)


def build_workload(counts, law="pmb"):
    """The reference bench fixture; law "trilinear" is SURVEY 8(d)'s history
    variant trilinear(1, 1e-3, 2e-3, 1e6) (n-linear path, nothing breaks);
    "multi" is the cfg5 law set on the same lattice: trilinear concrete, PMB
    steel and bilinear interface selected per bond by type (rebar_bond_types)."""
    import scenarios as S
    from paper_2105_04150_b200 import geometry, make_state
    from paper_2105_04150_b200.types import DamageLaw
    bundle, h, g = S.bench_lattice_bundle(counts)
    if law == "trilinear":
        bundle.model.laws = [DamageLaw.trilinear(1.0, 1e-3, 2e-3, 1e6)]
    elif law == "multi":
        bundle.model.laws = [DamageLaw.trilinear(1.0, 1e-3, 2e-3, 1e6),
                             DamageLaw.pmb(7.0, 1e6),
                             DamageLaw.bilinear(3.0, 1e-3, 1e6)]
    fam = geometry.build_family(bundle.particles.coords, h, g)
    if law == "multi":
        fam.bond_type = rebar_bond_types(counts, fam)
    state = make_state(fam, bundle.model.needs_history())
    state.u = S.seed_displacements(bundle.particles.coords)
    return bundle, fam, state


def cpu_baseline(counts_full, steps=2):
    """The reference CPU path (oracle/_ref, built from /root/reference/proj/src)
    on a bounded sample of the workload: a z-slab of the full lattice."""
    sample = (counts_full[0], counts_full[1], min(counts_full[2], 24))
    threads = os.cpu_count() or 1
    try:
        from oracle.pyoracle import Reference
        ref = Reference(threads=threads)
        secs, live, build_s = ref.bench_lattice(sample, HORIZON, 1e6, steps, threads)
        kind = "reference"
    except OSError:
        import scenarios as S
        from oracle.pyoracle import COracle
        from paper_2105_04150_b200 import SimulateOptions, make_state
        orc = COracle(threads=threads)
        bundle, h, g = S.bench_lattice_bundle(sample)
        fam = orc.build_family(bundle.particles.coords, h, g.hint())
        st = make_state(fam, False)
        st.u = S.seed_displacements(bundle.particles.coords)
        t0 = time.perf_counter()
        orc.simulate(bundle, st, SimulateOptions(steps))
        secs = time.perf_counter() - t0
        live = int(fam.n_neigh.sum())
        kind = "port"
    n = sample[0] * sample[1] * sample[2]
    return {"value": live * steps / secs, "unit": UNIT, "cores": threads, "kind": kind,
            "ms_per_step": 1e3 * secs / steps,
            "sample": f"{sample[0]}x{sample[1]}x{sample[2]} = {n} nodes z-slab of the same "
                      f"lattice, {steps} velocity-Verlet steps of simulate(bond_parallel), "
                      f"{live} live bonds"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    counts = (args.size, args.size, args.size)
    steps_each = 2
    vals = []
    cb = None
    for _ in range(args.warmup + args.steps):
        cb = cpu_baseline(counts, steps_each)
        vals.append(cb["value"])
    timed = vals[args.warmup:]
    value = statistics.median(timed)
    n = counts[0] * counts[1] * counts[2]
    # the full workload's live bonds (interior rows of a 216^3 lattice), to
    # express the sample throughput as ms/step of the whole workload
    live_full = 1209979144 if counts == (216, 216, 216) else None
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": (1e3 * live_full / value) if live_full else None,
        "ms_per_step_note": "extrapolated from the sample's bond throughput to the full lattice",
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg4 lattice {args.size}^3 = {n} nodes, delta=3dx (N=128), "
                               "PMB, velocity-Verlet (reference CPU, bounded z-slab sample)",
                   "nodes": n},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


def _summary(args, value, ms_step, world, n, N, live, bytes_step, achieved, e2e, launches,
             clocks, cpu, variant_name, extra_config=None, layout=None):
    peak, peak_kind = measured_peaks()
    law_key = "" if getattr(args, "law", "pmb") == "pmb" else f"_{args.law}"
    traffic = (measured_traffic(f"{layout}_{args.size}_{variant_name}{law_key}")
               if world == 1 and layout else None)
    law = {"pmb": "PMB c=1 s_c=1e6",
           "trilinear": "trilinear(1, 1e-3, 2e-3, 1e6) with history",
           "multi": "cfg5 laws by bond type: trilinear concrete, PMB steel, bilinear interface, "
                    "two rebar lines, history"}[getattr(args, "law", "pmb")]
    cfg = {"workload": f"cfg4 lattice {args.size}^3 = {n} nodes, delta=3dx (N={N}), "
                       f"{law}, velocity-Verlet, dt=1e-3, seeded u"
                       + (f", {world} z-slabs" if world > 1 else ""),
           "nodes": n, "group_size": N, "live_bonds": live, "variant": variant_name,
           "l2": f"inputs larger than L2 ({bytes_step / 1e9:.2f} GB/step algorithmic)",
           "parallelism": f"z-slab x{world}" if world > 1 else "single GPU"}
    cfg.update(extra_config or {})
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if variant_name == "exact" else "f32 bond math / f64 state",
        "data": "synthetic", "config": cfg,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": None if traffic is None else traffic / 1e9,
                     "traffic_unit": "GB per launch (ncu dram__bytes_read+write)",
                     "peak_source": peak_kind, "bytes_per_step": bytes_step,
                     "note": "achieved = SURVEY 8(d) algorithmic bytes / device time; the "
                             "lattice kernel keeps connectivity implicit, so DRAM traffic is "
                             "below the algorithmic bytes and the kernel is issue-bound"},
        "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu,
    }


def run_single(args, variant, local):
    import torch
    from paper_2105_04150_b200 import IntegratorKind, SimulateOptions, engine, make_state
    counts = (args.size, args.size, args.size)
    t_setup = time.perf_counter()
    bundle, fam, state0 = build_workload(counts, args.law)
    n = bundle.particles.size()
    N = int(fam.group_size)
    live = int(fam.n_neigh.sum())
    setup_s = time.perf_counter() - t_setup

    ctx = engine.Context(local)
    ctx.upload(bundle, state0, variant)
    layout = ctx.layout()
    stream = torch.cuda.ExternalStream(ctx.stream())
    step = 0
    ctx.run(args.warmup, step, IntegratorKind.velocity_verlet, 0, variant)
    step += args.warmup
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        ctx.run(args.steps, step, IntegratorKind.velocity_verlet, 0, variant)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = ctx.launch_count() - launches0
    ms_total = ev0.elapsed_time(ev1)
    ms_step = ms_total / args.steps
    value = live * args.steps / (ms_total / 1e3)
    bytes_step = algorithmic_bytes(n, N, live)
    if args.law in ("trilinear", "multi"):  # + 2 h B history (h = 4: fp32 on the fast path)
        bytes_step += 2 * (4 if args.variant == "fast" else 8) * live
    if args.law == "multi":  # + B bond_type
        bytes_step += live
    achieved = bytes_step / (ms_step / 1e3) / 1e9
    ctx.close()
    del ctx

    # end to end: one simulate() call through the C ABI from host buffers
    st = make_state(fam, bundle.model.needs_history())
    st.u = state0.u.copy()
    e2e_steps = args.e2e_steps
    # bytes that cross PCIe: coords, u, v, a, V, rho, rows, counts in; u, v, a,
    # n_neigh and only the rows that changed (none without breaks) out
    h2d = (3 * n * 8 * 4 + 2 * n * 8 + n * N * 4 + 2 * n * 4)
    d2h = (3 * n * 8 * 3 + n * 4)
    # one untimed call first (driver/pinned-buffer first-use costs), then the timed one
    warm = make_state(fam, bundle.model.needs_history())
    warm.u = state0.u.copy()
    engine.simulate(bundle, warm, SimulateOptions(2, 0, 0, IntegratorKind.velocity_verlet, variant))
    del warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    engine.simulate(bundle, st, SimulateOptions(e2e_steps, 0, 0, IntegratorKind.velocity_verlet,
                                                variant))
    e2e_s = time.perf_counter() - t0
    e2e = {"value": live * e2e_steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps,
           "seconds": e2e_s,
           "how": f"one simulate() call via the C ABI, {e2e_steps} steps, host buffers "
                  "(upload + layout + run + download inside the timed region)"}
    cpu = None if args.no_cpu else cpu_baseline(counts)
    out = _summary(args, value, ms_step, 1, n, N, live, bytes_step, achieved, e2e, launches,
                   clk.summary(), cpu, args.variant,
                   {"setup_s": round(setup_s, 2), "layout": layout}, layout)
    print(json.dumps(out))
    return 0


def run_slabs(args, variant, rank, world, local):
    """Strong scaling of the same lattice over `world` GPUs: rank r owns a
    z-slab of whole planes and builds its local model (owned planes + 3 ghost
    planes per cut, built on its own GPU); ghost rows are pushed by the step
    kernel over NVLink (paper_2105_04150_b200.slabs)."""
    import math

    import torch
    import torch.distributed as dist
    from paper_2105_04150_b200 import IntegratorKind, geometry, make_state, slabs
    from paper_2105_04150_b200.types import (BoundaryConditions, Corrections, DamageLaw,
                                             DamageModel, ModelBundle, ParticleSet)
    import scenarios as S

    nx = ny = nz = args.size
    plane = nx * ny
    g = int(math.ceil(HORIZON))
    cuts = [int(round(r * nz / world)) for r in range(world + 1)]
    z0, z1 = cuts[rank], cuts[rank + 1]
    zl0, zl1 = max(0, z0 - g), min(nz, z1 + g)
    t_setup = time.perf_counter()
    grid = geometry.GridDesc((0.0, 0.0, float(zl0)), 1.0, (nx, ny, zl1 - zl0))
    coords = geometry.grid_coordinates(grid)
    nl = grid.node_count()
    particles = ParticleSet(coords, np.ones(nl), np.ones(nl), np.zeros(nl, np.uint16))
    bundle = ModelBundle(particles, DamageModel([DamageLaw.pmb(1.0, 1e6)]), Corrections(),
                         BoundaryConditions.none(nl), 1e-3)
    fam = geometry.build_family(coords, HORIZON, grid)
    state = make_state(fam, False)
    state.u = S.seed_displacements(coords)
    ob, oe = (z0 - zl0) * plane, (z1 - zl0) * plane
    part = slabs.SlabPart(rank, world, z0 * plane, z1 * plane,
                          np.arange(zl0 * plane, zl1 * plane, dtype=np.int64), ob, oe,
                          rank - 1 if rank > 0 else -1, rank + 1 if rank + 1 < world else -1)
    ranges = [(cuts[r] * plane, cuts[r + 1] * plane) for r in range(world)]
    comm = slabs.TorchComm()
    Ns = comm.allgather(int(fam.group_size))
    if len(set(Ns)) != 1:
        raise SystemExit(f"slab families disagree on the group size: {Ns}")
    live_own = int(fam.n_neigh[ob:oe].sum())
    setup_s = time.perf_counter() - t_setup

    red_dev = "cuda" if dist.get_backend() == "nccl" else "cpu"

    def timed_max(ms):
        t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # e2e through the rank-local public API: host buffers -> upload + connect
    # -> run -> owned rows back to host, max over ranks
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sr = slabs.SlabRank(comm, local)
    sr.setup(part, ranges, bundle, state, variant)
    sr.run(args.e2e_steps, 0, IntegratorKind.velocity_verlet)
    down = make_state(fam, False)
    sr.ctx.download(down)
    torch.cuda.synchronize()
    e2e_s = timed_max((time.perf_counter() - t0) * 1e3) / 1e3
    sr.close()

    sr = slabs.SlabRank(comm, local)
    sr.setup(part, ranges, bundle, state, variant)
    ctx = sr.ctx
    stream = torch.cuda.ExternalStream(ctx.stream())
    sr.run(args.warmup, 0, IntegratorKind.velocity_verlet)
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = ctx.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record(stream)
        sr.run(args.steps, args.warmup, IntegratorKind.velocity_verlet)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms_total = timed_max(ev0.elapsed_time(ev1))
    launches = ctx.launch_count() - launches0
    sr.close()
    tot = torch.tensor([live_own, launches], dtype=torch.int64, device=red_dev)
    dist.all_reduce(tot)
    live, launches = int(tot[0].item()), int(tot[1].item())
    n = nx * ny * nz
    N = Ns[0]
    ms_step = ms_total / args.steps
    value = live * args.steps / (ms_total / 1e3)
    bytes_step = algorithmic_bytes(n, N, live)
    achieved = bytes_step / (ms_step / 1e3) / 1e9
    halo_bytes = 2 * (world - 1) * g * plane * 32 * 2  # u pushed both ways per cut, per step
    e2e = {"value": live * args.e2e_steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": (nl * (24 * 3 + 16 + 24 + fam.group_size * 4)) // args.e2e_steps,
           "d2h_bytes_per_step": (nl * (24 * 3 + fam.group_size * 4 + 4)) // args.e2e_steps,
           "seconds": e2e_s,
           "how": f"per rank: host buffers -> upload_part + connect -> {args.e2e_steps} steps -> "
                  "download, max over ranks (bytes are rank 0's)"}
    clocks = comm.allgather(clk.summary())
    if rank == 0:
        out = _summary(args, value, ms_step, world, n, N, live, bytes_step, achieved, e2e,
                       launches, clocks[0], None, args.variant,
                       {"setup_s": round(setup_s, 2), "halo_bytes_per_step_nvlink": halo_bytes,
                        "clocks_all_ranks": clocks})
        print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="fast", choices=["exact", "fast"])
    ap.add_argument("--size", type=int, default=216)
    ap.add_argument("--e2e-steps", type=int, default=1000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--law", default="pmb", choices=["pmb", "trilinear", "multi"])
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    from paper_2105_04150_b200 import KernelVariant

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    variant = KernelVariant.fast if args.variant == "fast" else KernelVariant.bond_parallel
    if world == 1:
        return run_single(args, variant, local)
    import torch.distributed as dist
    if torch.cuda.device_count() >= world:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:  # several ranks share a GPU (a 1-GPU test box): gloo for the host plumbing
        dist.init_process_group("gloo")
    try:
        return run_slabs(args, variant, rank, world, local)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
