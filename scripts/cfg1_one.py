"""One cfg1 simulate() (beam 50x14x14, PMB, Euler) on the fast variant: wall time per call."""
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
for rep in range(3):
    st = make_state(fam, False)
    t0 = time.perf_counter()
    engine.simulate(b, st, SimulateOptions(steps, 0, 0, IntegratorKind.euler, KernelVariant.fast))
    print(f"cfg1 fast simulate {steps} steps: {1e3 * (time.perf_counter() - t0):.2f} ms")
