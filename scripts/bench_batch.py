"""The calibration / UQ outer loop: K independent cfg1-size
simulate() calls (3-point-bend beam, 50 x 14 x 14 = 9,800 nodes, PMB, Euler,
1000 steps) -- one at a time vs pd_simulate_batch on one GPU -- beside one
run of the reference CPU path (oracle/_ref, all host cores)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import scenarios as S  # noqa: E402
from paper_2105_04150_b200 import engine, geometry  # noqa: E402
from paper_2105_04150_b200.types import (IntegratorKind, KernelVariant, SimulateOptions,  # noqa: E402
                                         make_state)

K = int(os.environ.get("K", "16"))
STEPS = 1000


def models():
    out = []
    for k in range(K):
        b, h, g = S.beam_bundle()
        b.bc.magnitude[:] = b.bc.magnitude * (0.5 + 0.1 * k)  # a parameter sweep
        out.append((b, h, g))
    return out


def main():
    ms = models()
    fam = geometry.build_family(ms[0][0].particles.coords, ms[0][1], ms[0][2])
    live = int(fam.n_neigh.sum())
    res = {"workload": f"cfg1 beam 50x14x14 = {fam.node_count()} nodes, {live} live bonds, "
                       f"PMB, Euler, {STEPS} steps, K = {K} models (load sweep)"}
    for variant in (KernelVariant.fast, KernelVariant.bond_parallel):
        opts = [SimulateOptions(STEPS, 0, 0, IntegratorKind.euler, variant) for _ in ms]
        # warm-up
        engine.simulate(ms[0][0], make_state(fam, False), SimulateOptions(5, 0, 0,
                                                                         IntegratorKind.euler,
                                                                         variant))
        states = [make_state(fam, False) for _ in ms]
        t0 = time.perf_counter()
        for (b, h, g), st, o in zip(ms, states, opts):
            engine.simulate(b, st, o)
        seq = time.perf_counter() - t0
        states2 = [make_state(fam, False) for _ in ms]
        t0 = time.perf_counter()
        engine.simulate_batch([m[0] for m in ms], states2, opts)
        bat = time.perf_counter() - t0
        same = all(np.array_equal(a.u, b.u) for a, b in zip(states, states2))
        res[variant.name] = {"sequential_s": seq, "batch_s": bat,
                             "sequential_bond_evals_per_s": K * STEPS * live / seq,
                             "batch_bond_evals_per_s": K * STEPS * live / bat,
                             "batch_speedup": seq / bat, "batch_equals_sequential": same}
    try:
        from oracle.pyoracle import Reference
        ref = Reference(threads=os.cpu_count() or 1)
        b = ms[0][0]
        st = make_state(fam, False)
        t0 = time.perf_counter()
        ref.simulate(b, st, SimulateOptions(STEPS, 0, 0, IntegratorKind.euler))
        one = time.perf_counter() - t0
        res["reference_cpu"] = {"one_run_s": one, "cores": os.cpu_count(),
                                "bond_evals_per_s": STEPS * live / one}
    except OSError as e:
        res["reference_cpu"] = {"unavailable": str(e)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
