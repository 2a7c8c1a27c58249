#!/usr/bin/env python
"""cfg5 at its stated scale on one B200: the reinforced-concrete beam of
PAPER.md:580-597 at dx = 1.6 mm (~31M nodes, tests/scenarios.rc_beam_setup):
three bond classes from a rule-table classifier, surface-correction factors,
trilinear concrete + linear steel + bilinear interface laws with history,
no-failure supports, quintic displacement loading, velocity-Verlet.

Every setup pass runs on the device (family, classifier, neighbourhood
volumes, lambda).  The fast variant (typed lattice kernel) is timed with
CUDA events over K steps after W warm-up steps; the exact variant (bitwise
path) over a few steps.  Parity at a downscale: tests/test_gpu_cfg5.py.

  python scripts/bench_cfg5.py [--dx 1.6] [--steps 100] [--exact-steps 3] > out.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dx", type=float, default=1.6, help="node spacing in mm")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--exact-steps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import scenarios as S
    from paper_2105_04150_b200 import IntegratorKind, KernelVariant, engine, geometry, make_state
    out = {"config": "cfg5 RC beam (PAPER.md:580-597)", "dx_mm": args.dx}
    t = time.perf_counter()
    b, g, delta, cls = S.rc_beam_setup(args.dx)
    out["setup_s"] = time.perf_counter() - t
    n = b.particles.size()
    out["nodes"] = n
    out["grid"] = list(g.counts)
    t = time.perf_counter()
    fam = geometry.build_family(b.particles.coords, delta, g)
    out["family_s"] = time.perf_counter() - t
    t = time.perf_counter()
    fam.bond_type = geometry.classify_bonds(b.particles.coords, fam, cls)
    out["classify_s"] = time.perf_counter() - t
    t = time.perf_counter()
    vol = b.particles.volume
    v0 = geometry.max_neighborhood_volume(vol, fam)
    b.corrections.lambda_ = geometry.surface_correction_factors(vol, fam, v0)
    out["lambda_s"] = time.perf_counter() - t
    out["group_size"] = int(fam.group_size)
    out["live_bonds"] = int(fam.n_neigh.sum())
    counts = np.zeros(3, np.int64)
    lo, hi = np.inf, -np.inf
    chunk = 1 << 26
    for a in range(0, fam.entries.size, chunk):  # bounded temporaries at 31M x 128
        live = fam.entries[a:a + chunk] >= 0
        counts += np.bincount(fam.bond_type[a:a + chunk][live], minlength=3)[:3]
        lam = b.corrections.lambda_[a:a + chunk][live]
        lo, hi = min(lo, float(lam.min())), max(hi, float(lam.max()))
    out["bonds_by_type"] = counts.tolist()
    out["lambda_range"] = [lo, hi]
    vv = IntegratorKind.velocity_verlet
    for variant, steps in ((KernelVariant.fast, args.steps), (KernelVariant.bond_parallel,
                                                             args.exact_steps)):
        if steps <= 0:
            continue
        st = make_state(fam, False)  # history: zeros allocated on the device
        ctx = engine.Context(0)
        t = time.perf_counter()
        ctx.upload(b, st, variant)
        torch.cuda.synchronize()
        up = time.perf_counter() - t
        stream = torch.cuda.ExternalStream(ctx.stream())
        ctx.run(args.warmup, 0, vv, 0, variant)
        torch.cuda.synchronize()
        free, total = torch.cuda.mem_get_info()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        live0 = ctx.live_bonds()
        e0.record(stream)
        ctx.run(steps, args.warmup, vv, 0, variant)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        live1 = ctx.live_bonds()
        row = {"kernel": ctx.kernel(), "layout": ctx.layout(), "upload_s": up, "steps": steps,
               "ms_per_step": ms, "bond_evals_per_s": 0.5 * (live0 + live1) / (ms / 1e3),
               "live_bonds_timed": [live0, live1], "device_memory_used_gb": (total - free) / 1e9}
        out[variant.name] = row
        print(json.dumps({variant.name: row}), file=sys.stderr)
        ctx.close()
        del ctx, st
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
