"""Host enqueue cost per step of ctx.run() on a tiny model: lattice fast path vs exact path."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import scenarios as S  # noqa: E402
from paper_2105_04150_b200 import engine, geometry  # noqa: E402
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, make_state  # noqa: E402

b, h, g = S.bench_lattice_bundle((16, 16, 16))
fam = geometry.build_family(b.particles.coords, h, g)
for variant in (KernelVariant.fast, KernelVariant.bond_parallel):
    ctx = engine.Context(0)
    st = make_state(fam, False)
    ctx.upload(b, st, variant)
    ctx.run(10, 0, IntegratorKind.euler, 0, variant)
    torch.cuda.synchronize()
    for n in (2000, 2000):
        t0 = time.perf_counter()
        ctx.run(n, 10, IntegratorKind.euler, 0, variant)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{variant.name} {ctx.layout()}: enqueue {1e6 * (t1 - t0) / n:.2f} us/step, "
              f"until idle {1e6 * (t2 - t0) / n:.2f} us/step")
    ctx.close()
