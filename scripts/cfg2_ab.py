"""cfg2 (the notched plate) as simulate() calls: per-phase host timings
(PD_TIMING=1) of the fast variant, to split a config's wall time."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import scenarios as S  # noqa: E402
from paper_2105_04150_b200 import engine, geometry  # noqa: E402
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, SimulateOptions, make_state  # noqa: E402

b, h, g, notch = S.notched_plate_bundle(100, 100, 10, 1000)
fam = geometry.build_family(b.particles.coords, h, g)
geometry.break_notch(fam, b.particles.coords, notch["axis"], notch["position"],
                     notch["sweep_axis"], notch["depth"])
for rep in range(3):
    st = make_state(fam, True)
    t0 = time.perf_counter()
    engine.simulate(b, st, SimulateOptions(1000, 0, 0, IntegratorKind.euler_cromer,
                                           KernelVariant.fast))
    print(f"simulate {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr)
