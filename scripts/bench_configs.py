"""BASELINE.json configs beside the reference CPU path, each as one simulate() call.

cfg1  3-point-bend beam 50 x 14 x 14 = 9,800 nodes, PMB, Euler, 1000 steps
cfg2  pre-cracked plate 100 x 100 x 10 = 100,000 nodes, bilinear, Euler-Cromer, 1000 steps
      (edge notch cut with break_initial_bonds, opposite edges pulled on a linear ramp)
cfg3  cubic lattice 100^3 = 1,000,000 nodes, PMB, velocity-Verlet, 1000 steps
      (the reference runs a 5-step sample; its time is scaled to 1000 steps)
cfg4 is bench.py's default line.  cfg5's law set (several laws chosen by bond type) is
`bench.py --law multi` on the cfg4 lattice.

GPU: the fast and exact variants of one simulate() call (host buffers in, state out), after
one untimed call.  Reference: the unmodified reference (oracle/_ref) on all host cores.
Writes one JSON object (stdout, and gpurun_out/r02_configs.json when --save is given;
profiles/r02_configs.json is a copy).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import scenarios as S  # noqa: E402
from oracle.pyoracle import COracle, Reference  # noqa: E402
from paper_2105_04150_b200 import engine, geometry  # noqa: E402
from paper_2105_04150_b200.types import (IntegratorKind, KernelVariant, SimulateOptions,  # noqa: E402
                                         make_state)


def cfg1():
    b, h, g = S.beam_bundle()
    fam = geometry.build_family(b.particles.coords, h, g)
    return "cfg1 beam 50x14x14, PMB, Euler", b, fam, IntegratorKind.euler, 1000, 1000


def cfg2():
    b, h, g, notch = S.notched_plate_bundle(100, 100, 10, 1000)
    fam = geometry.build_family(b.particles.coords, h, g)
    geometry.break_notch(fam, b.particles.coords, notch["axis"], notch["position"],
                         notch["sweep_axis"], notch["depth"])
    return ("cfg2 notched plate 100x100x10, bilinear, Euler-Cromer", b, fam,
            IntegratorKind.euler_cromer, 1000, 1000)


def cfg3():
    b, h, g = S.bench_lattice_bundle((100, 100, 100))
    fam = geometry.build_family(b.particles.coords, h, g)
    return "cfg3 lattice 100^3, PMB, velocity-Verlet", b, fam, IntegratorKind.velocity_verlet, 1000, 5


def run(backend, b, fam, integ, steps, variant):
    st = make_state(fam, b.model.needs_history())
    if b.bc.kind.sum() == 0:  # the bench lattice: seeded displacements
        st.u = S.seed_displacements(b.particles.coords)
    t0 = time.perf_counter()
    backend.simulate(b, st, SimulateOptions(steps, 0, 0, integ, variant))
    return time.perf_counter() - t0, st


def main():
    threads = os.cpu_count() or 1
    ref = Reference(threads=threads)
    out = {"host_cores": threads}
    for make in (cfg1, cfg2, cfg3):
        name, b, fam, integ, steps, ref_steps = make()
        live = int(fam.n_neigh.sum())
        row = {"nodes": fam.node_count(), "live_bonds": live, "steps": steps}
        for variant in (KernelVariant.fast, KernelVariant.bond_parallel):
            run(engine.backend(), b, fam, integ, 2, variant)  # warm-up
            secs, st = run(engine.backend(), b, fam, integ, steps, variant)
            row[f"gpu_{variant.name}_s"] = secs
            row[f"gpu_{variant.name}_bond_evals_per_s"] = live * steps / secs
            row[f"gpu_{variant.name}_broken"] = int(fam.n_neigh.sum() - st.connectivity.n_neigh.sum())
        secs, st = run(ref, b, fam, integ, ref_steps, KernelVariant.bond_parallel)
        row["reference_s"] = secs * steps / ref_steps
        row["reference_note"] = (f"{ref_steps} steps timed" +
                                 ("" if ref_steps == steps else f", scaled to {steps}"))
        row["reference_bond_evals_per_s"] = live * ref_steps / secs
        row["speedup_fast_vs_reference"] = row["reference_s"] / row["gpu_fast_s"]
        row["speedup_exact_vs_reference"] = row["reference_s"] / row["gpu_bond_parallel_s"]
        out[name] = row
        print(name, json.dumps(row), file=sys.stderr)
    print(json.dumps(out))
    if "--save" in sys.argv:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)  # merged back by gpurun
        with open(os.path.join(ROOT, "gpurun_out", "r02_configs.json"), "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
