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
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML every ~2 ms on a thread (a 20-step region lasts ~22 ms), or
    nvidia-smi -lms 50 when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons)
        self.stop = threading.Event()
        self.proc = None
        self.source = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _nvml_sample(self, nv, h, mx):
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.samples.append((float(sm), float(mx),
                             {k for k, b in self.REASONS.items() if bits & b}))

    def _nvml_loop(self, nv, h, mx):
        while not self.stop.is_set():
            try:
                self._nvml_sample(nv, h, mx)
            except Exception:
                break
            self.live.set()
            time.sleep(0.002)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self._nv = (nv, h, mx)
            self.t = threading.Thread(target=self._nvml_loop, args=(nv, h, mx), daemon=True)
            self.source = "nvml"
            self.live = threading.Event()
            self.t.start()
            self.live.wait(timeout=1.0)  # the sampler is running before the timed region
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.source = "nvidia-smi"
            self.t = threading.Thread(target=self._smi_read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _smi_read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                self.samples.append((float(f[1]), float(f[2]),
                                     {n for n, fl in zip(names, f[5:9]) if fl.lower() == "active"}))
            except ValueError:
                continue

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if getattr(self, "t", None):
            self.t.join(timeout=5)

    def summary(self):
        sm = [x[0] for x in self.samples]
        reasons = set().union(*[x[2] for x in self.samples]) if self.samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(x[1] for x in self.samples) if self.samples else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


NCU_METRICS = ("dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
               "sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,"
               "sm__warps_active.avg.pct_of_peak_sustained_active")


def ncu_probe(args, kernel: str):
    """Measured DRAM traffic of the step kernel in THIS run's configuration:
    `ncu` profiles one warm launch of `kernel` in a child `bench.py --probe-run`
    (same workload, law and variant), reading dram__bytes_read/write.sum, the
    issue-slot utilisation and the warp instructions.  Profiler numbers are
    never the bench value; only the per-launch byte count and ratios are used.
    Returns a dict, or {"error": ...} when ncu is unavailable."""
    import csv
    import shutil
    import tempfile
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    base = kernel.split("<", 1)[0]
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "probe.csv")
        cmd = [ncu, "--metrics", NCU_METRICS, "--clock-control", "none", "-k", f"regex:^{base}$",
               "-s", "2", "-c", "1", "--csv", "--page", "raw", "--log-file", log,
               sys.executable, os.path.abspath(__file__), "--probe-run", "--size", str(args.size),
               "--law", args.law, "--variant", args.variant, "--mesh", args.mesh]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        except (OSError, subprocess.TimeoutExpired) as exc:
            return {"error": f"ncu probe failed: {exc}"}
        if not os.path.exists(log):
            return {"error": f"ncu probe rc={r.returncode}: {r.stderr[-300:]}"}
        rows = list(csv.reader(open(log)))
    hdr = next((i for i, row in enumerate(rows) if "dram__bytes_read.sum" in row), None)
    if hdr is None or len(rows) < hdr + 3:
        return {"error": "ncu probe: no kernel row"}
    head, units, vals = rows[hdr], rows[hdr + 1], rows[hdr + 2]

    def val(name, scale_units=True):
        v = float(vals[head.index(name)].replace(",", ""))
        u = units[head.index(name)].strip().lower()
        if scale_units:
            v *= {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-9,
                  "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(u, 1.0)
        return v
    name = vals[head.index("Kernel Name")] if "Kernel Name" in head else base
    return {"kernel": name[:120],
            "dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
            "dram_read_bytes": val("dram__bytes_read.sum"),
            "ncu_time_s": val("gpu__time_duration.sum"),
            "warp_instructions": val("sm__inst_executed.sum", False),
            "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active", False),
            "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active", False)}


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


LAWS = {
    "pmb": "PMB c=1 s_c=1e6 (no breaking)",
    "fracture": "PMB c=1 s_c=1e-5 (SURVEY 8(d) fracturing variant: ~12 % of the bonds break "
                "at step 1, breaks continue)",
    "trilinear": "trilinear(1, 1e-3, 2e-3, 1e6) with history",
    "multi": "cfg5 laws by bond type: trilinear concrete, PMB steel, bilinear interface, "
             "two rebar lines, history",
}
S_C = {"pmb": 1e6, "fracture": 1e-5, "trilinear": 1e6, "multi": 1e6}


MESHES = {
    "lattice": "cubic lattice (the reference bench fixture)",
    "jitter": "irregular mesh: the same lattice with every coordinate jittered by a seeded "
              "uniform +-0.2 spacing (rows of 90-150 neighbours; the general tile kernel)",
    "shuffled": "the jittered mesh with its nodes numbered in a seeded random order (no "
                "spatial coherence in the input numbering)",
}


def jitter_coords(coords, amp=0.2, seed=2105):
    rng = np.random.default_rng(seed)
    return coords + rng.uniform(-amp, amp, coords.shape)


def build_workload(counts, law="pmb", mesh="lattice"):
    """The reference bench fixture (bench.cpp:76-104); law "fracture" is SURVEY
    8(d)'s fracturing variant (PMB s_c = 1e-5), "trilinear" its history variant
    trilinear(1, 1e-3, 2e-3, 1e6) (n-linear path, nothing breaks); "multi" is
    the cfg5 law set on the same lattice: trilinear concrete, PMB steel and
    bilinear interface selected per bond by type (rebar_bond_types)."""
    import scenarios as S
    from paper_2105_04150_b200 import geometry, make_state
    from paper_2105_04150_b200.types import DamageLaw
    bundle, h, g = S.bench_lattice_bundle(counts, s_c=S_C[law])
    if mesh in ("jitter", "shuffled"):
        bundle.particles.coords = jitter_coords(bundle.particles.coords)
        g = None
    if mesh == "shuffled":
        order = np.random.default_rng(7).permutation(bundle.particles.size())
        bundle.particles.coords = bundle.particles.coords.reshape(-1, 3)[order].reshape(-1)
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


def reference_runs(counts, law, run_steps, threads):
    """The UNMODIFIED reference (oracle/_ref, compiled from
    /root/reference/proj/src) on the SAME workload: simulate(bond_parallel,
    velocity-Verlet) of the full lattice, one call per run continuing the
    state (bench.cpp:106-117).  Returns (seconds per run, live bonds, family
    build seconds), or None when the reference is not built or the law has no
    reference fixture here ("multi" needs the bond classes)."""
    if law == "multi":
        return None
    try:
        from oracle.pyoracle import Reference
        ref = Reference(threads=0)
    except OSError:
        return None
    return ref.bench_lattice_runs(counts, HORIZON, S_C[law], run_steps, threads,
                                  law=1 if law == "trilinear" else 0)


def split_runs(k: int):
    """K timed steps as runs of >= 3 steps (>= 3 runs when K >= 9)."""
    if k >= 9:
        return [k // 3, k // 3, k - 2 * (k // 3)]
    return [k]


def cpu_baseline(counts, law):
    """The reference CPU path on this box's host cores, on the same workload as
    the GPU line: one warm-up step, then the median of 3 runs of 3 steps on
    all cores (median of >= 3 runs of >= 3 steps)."""
    cores = host_cores()
    got = reference_runs(counts, law, [1, 3, 3, 3], [cores] * 4)
    if got is None:
        return None
    secs, live, build_s = got
    per = [t / 3 for t in secs[1:]]
    ms = 1e3 * statistics.median(per)
    n = counts[0] * counts[1] * counts[2]
    return {"value": live * 1e3 / ms, "unit": UNIT, "cores": cores, "kind": "reference",
            "ms_per_step": ms, "cpu": cpu_model(), "same_config": True,
            "runs_ms_per_step": [1e3 * x for x in per], "family_build_s": build_s,
            "sample": f"the full workload ({counts[0]}x{counts[1]}x{counts[2]} = {n} nodes, "
                      f"{live} live bonds at the start): simulate(bond_parallel, velocity-Verlet) "
                      f"of the unmodified reference, 1 warm-up step then the median of 3 runs x "
                      f"3 steps on {cores} threads"}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref)
    on the SAME configuration as our arm, all host cores, W warm-up steps
    then exactly K timed steps in runs of >= 3 steps; plus one 1-core run."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    counts = (args.size, args.size, args.size)
    cores = host_cores()
    timed = split_runs(args.steps)
    one = [args.ref_one_core_steps] if args.ref_one_core_steps > 0 else []
    got = reference_runs(counts, args.law, [args.warmup] + timed + one,
                         [cores] * (1 + len(timed)) + [1] * len(one))
    n = counts[0] * counts[1] * counts[2]
    if got is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no reference fixture for law {args.law} (oracle/_ref not built or "
                          "the law needs bond classes)"}))
        return 0
    secs, live, build_s = got
    runs = secs[1:1 + len(timed)]
    per_run = [t / k for t, k in zip(runs, timed)]
    ms = 1e3 * statistics.median(per_run)
    value = live * 1e3 / ms
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": sum(timed), "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"cfg4 lattice {args.size}^3 = {n} nodes, delta=3dx (N=128), "
                               f"{LAWS[args.law]}, velocity-Verlet, dt=1e-3, seeded u",
                   "nodes": n, "live_bonds": live, "law": args.law, "same_config": True},
        "runs": [{"steps": k, "seconds": t, "ms_per_step": 1e3 * t / k}
                 for k, t in zip(timed, runs)],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "cpu": cpu_model(), "family_build_s": build_s,
                         "sample": f"the full workload, {len(timed)} runs of {timed} steps, "
                                   "median ms/step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if one:
        t1 = secs[-1] / one[0]
        out["one_core"] = {"steps": one[0], "ms_per_step": 1e3 * t1, "value": live / t1,
                           "unit": UNIT}
    print(json.dumps(out))
    return 0


def _summary(args, value, ms_step, world, n, N, live, bytes_step, achieved, e2e, launches,
             clocks, cpu, variant_name, probe=None, extra_config=None):
    peak, peak_kind = measured_peaks()
    mesh = {"lattice": "lattice", "jitter": "jittered lattice (irregular mesh)",
            "shuffled": "jittered lattice, randomly numbered (irregular mesh)"}[args.mesh]
    cfg = {"workload": f"cfg4 {mesh} {args.size}^3 = {n} nodes, delta=3dx (N={N}), "
                       f"{LAWS[args.law]}, velocity-Verlet, dt=1e-3, seeded u"
                       + (f", {world} z-slabs" if world > 1 else ""),
           "nodes": n, "group_size": N, "live_bonds": live, "variant": variant_name,
           "law": args.law, "mesh": args.mesh,
           "l2": f"inputs larger than L2 ({bytes_step / 1e9:.2f} GB/step algorithmic)",
           "parallelism": f"z-slab x{world}" if world > 1 else "single GPU"}
    cfg.update(extra_config or {})
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None, "peak_source": peak_kind,
            "bytes_per_step": bytes_step,
            "note": "achieved = SURVEY 8(d) algorithmic bytes per step / device time per step"}
    if probe and "dram_bytes" in probe:
        dram_gbs = probe["dram_bytes"] / (ms_step / 1e3) / 1e9
        issue = probe["issue_active_pct"] / 100.0
        roof.update({
            "traffic": probe["dram_bytes"] / 1e9,
            "traffic_unit": "GB per launch, measured by ncu in this run "
                            "(dram__bytes_read.sum + dram__bytes_write.sum)",
            "dram_gbs": dram_gbs, "dram_frac": dram_gbs / peak, "issue_frac": issue,
            "occupancy": probe["warps_active_pct"] / 100.0,
            "thread_instructions_per_bond": 32.0 * probe["warp_instructions"] / max(live, 1),
        })
        # what actually limits the kernel: HBM when the measured DRAM rate is
        # near peak, the issue slots otherwise
        if roof["dram_frac"] < 0.6 and issue > 0.6:
            roof["bound"] = "issue"
            roof["note"] += ("; the kernel moves fewer DRAM bytes than the formula counts "
                             "(implicit / compact connectivity), so it is issue-bound: see "
                             "dram_frac and issue_frac")
    elif probe:
        roof["probe_error"] = probe.get("error")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if variant_name == "exact" else "f32 bond math / f64 state",
        "data": "synthetic", "config": cfg, "roofline": roof,
        "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu,
    }


def probe_run(args, variant):
    """--probe-run: the workload's upload and a few steps (ncu_probe's child)."""
    from paper_2105_04150_b200 import IntegratorKind, engine
    bundle, fam, state0 = build_workload((args.size,) * 3, args.law, args.mesh)
    ctx = engine.Context(0)
    ctx.upload(bundle, state0, variant)
    ctx.run(4, 0, IntegratorKind.velocity_verlet, 0, variant)
    ctx.close()
    return 0


def run_single(args, variant, local):
    import torch
    from paper_2105_04150_b200 import IntegratorKind, SimulateOptions, engine, make_state
    counts = (args.size, args.size, args.size)
    t_setup = time.perf_counter()
    bundle, fam, state0 = build_workload(counts, args.law, args.mesh)
    n = bundle.particles.size()
    N = int(fam.group_size)
    setup_s = time.perf_counter() - t_setup

    ctx = engine.Context(local)
    ctx.upload(bundle, state0, variant)
    layout = ctx.layout()
    stream = torch.cuda.ExternalStream(ctx.stream())
    step = 0
    ctx.run(args.warmup, step, IntegratorKind.velocity_verlet, 0, variant)
    step += args.warmup
    torch.cuda.synchronize()
    kernel = ctx.kernel()
    launches0 = ctx.launch_count()
    live0 = ctx.live_bonds()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        ctx.run(args.steps, step, IntegratorKind.velocity_verlet, 0, variant)
        ev1.record(stream)
        torch.cuda.synchronize()
    step += args.steps
    launches = ctx.launch_count() - launches0
    live1 = ctx.live_bonds()
    ms_total = ev0.elapsed_time(ev1)
    ms_step = ms_total / args.steps
    # live bonds fall while the fracturing variant breaks: count the mean of
    # the live bonds before and after the timed steps
    live = (live0 + live1) // 2
    value = live * args.steps / (ms_total / 1e3)
    bytes_step = algorithmic_bytes(n, N, live)
    if args.law in ("trilinear", "multi"):  # + 2 h B history (h = 4: fp32 on the fast path)
        bytes_step += 2 * (4 if args.variant == "fast" else 8) * live
    if args.law == "multi":  # + B bond_type
        bytes_step += live
    achieved = bytes_step / (ms_step / 1e3) / 1e9
    # the same kernel over a longer stretch, so the clock sampler sees it under
    # sustained load (reported beside the timed value, not instead of it)
    sustain = None
    if args.sustain_steps > 0:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk2:
            torch.cuda.synchronize()
            e0.record(stream)
            ctx.run(args.sustain_steps, step, IntegratorKind.velocity_verlet, 0, variant)
            e1.record(stream)
            torch.cuda.synchronize()
        sustain = {"steps": args.sustain_steps,
                   "ms_per_step": e0.elapsed_time(e1) / args.sustain_steps,
                   "clocks": clk2.summary()}
    ctx.close()
    del ctx

    # end to end: one simulate() call through the C ABI from host buffers
    st = make_state(fam, bundle.model.needs_history())
    st.u = state0.u.copy()
    e2e_steps = args.e2e_steps
    hist_b = 8 * n * N if bundle.model.needs_history() else 0
    # bytes that cross PCIe: coords, u, v, a, V, rho, rows, counts (+ bond
    # types, history) in; u, v, a, n_neigh (+ history) and only the rows that
    # changed out
    h2d = (3 * n * 8 * 4 + 2 * n * 8 + n * N * 4 + 2 * n * 4 + hist_b
           + (n * N if fam.bond_type is not None else 0))
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
    changed = int(np.count_nonzero(st.connectivity.n_neigh != fam.n_neigh))
    d2h = 3 * n * 8 * 3 + n * 4 + changed * N * 4 + hist_b
    live_e2e = (int(fam.n_neigh.sum()) + int(st.connectivity.n_neigh.sum())) // 2
    e2e = {"value": live_e2e * e2e_steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps,
           "seconds": e2e_s, "rows_changed": changed,
           "how": f"one simulate() call via the C ABI, {e2e_steps} steps, host buffers "
                  "(upload + layout + run + download inside the timed region)"}
    del st, fam, state0, bundle
    probe = None if args.no_probe else ncu_probe(args, kernel)
    # the reference fixture is the lattice: no CPU line for the jittered mesh
    cpu = None if args.no_cpu or args.mesh != "lattice" else cpu_baseline(counts, args.law)
    extra = {"setup_s": round(setup_s, 2), "layout": layout, "kernel": kernel,
             "live_bonds_timed": [live0, live1]}
    if sustain:
        extra["sustained"] = sustain
    out = _summary(args, value, ms_step, 1, n, N, live, bytes_step, achieved, e2e, launches,
                   clk.summary(), cpu, args.variant, probe, extra)
    if probe and "dram_bytes" in probe:
        out["ncu_probe"] = probe
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
                       launches, clocks[0], None, args.variant, None,
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
    ap.add_argument("--law", default="pmb", choices=sorted(LAWS))
    ap.add_argument("--mesh", default="lattice", choices=sorted(MESHES))
    ap.add_argument("--no-probe", action="store_true", help="skip the ncu DRAM-traffic probe")
    ap.add_argument("--sustain-steps", type=int, default=200,
                    help="extra untimed-for-value steps under the clock sampler")
    ap.add_argument("--ref-one-core-steps", type=int, default=3,
                    help="reference arm: steps of the extra 1-core run (0 = none)")
    ap.add_argument("--probe-run", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.probe_run:
        from paper_2105_04150_b200 import KernelVariant
        return probe_run(args, KernelVariant.fast if args.variant == "fast"
                         else KernelVariant.bond_parallel)

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
