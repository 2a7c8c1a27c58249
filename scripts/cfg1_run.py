"""cfg1 (the 9,800-node beam) as one simulate() call per variant: per-step
wall time of the device-resident loop (used with ncu to split the step into
kernel time and launch gaps)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import scenarios as S  # noqa: E402
from paper_2105_04150_b200 import engine, geometry  # noqa: E402
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, SimulateOptions, make_state  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
b, h, g = S.beam_bundle()
fam = geometry.build_family(b.particles.coords, h, g)
for variant in (KernelVariant.fast, KernelVariant.bond_parallel):
    for rep in range(2):
        st = make_state(fam, False)
        t0 = time.perf_counter()
        engine.simulate(b, st, SimulateOptions(steps, 0, 0, IntegratorKind.euler, variant))
        dt = time.perf_counter() - t0
    print(f"{variant.name}: {steps} steps {dt * 1e3:.1f} ms ({dt / steps * 1e6:.1f} us/step)")
