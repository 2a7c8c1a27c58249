"""cfg1 (the 9,800-node beam): per-step time of the device-resident loop.

For each variant: one simulate() call from host buffers (wall time), then the
resident context timed with CUDA events over the same 1000 Euler steps (the
persistent small-model launch for the fast variant unless PD_LAT_PERSIST=0).
Prints broken bonds and a displacement checksum so runs can be compared.

  python scripts/cfg1_run.py [steps] [--write-every W]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import scenarios as S  # noqa: E402
from paper_2105_04150_b200 import engine, geometry  # noqa: E402
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, SimulateOptions, make_state  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = int(args[0]) if args else 1000
we = int(sys.argv[sys.argv.index("--write-every") + 1]) if "--write-every" in sys.argv else 0
b, h, g = S.beam_bundle()
fam = geometry.build_family(b.particles.coords, h, g)
eu = IntegratorKind.euler
for variant in (KernelVariant.fast, KernelVariant.bond_parallel):
    for rep in range(2):
        st = make_state(fam, False)
        t0 = time.perf_counter()
        engine.simulate(b, st, SimulateOptions(steps, 0, 0, eu, variant))
        dt = time.perf_counter() - t0
    broken = int(fam.n_neigh.sum() - st.connectivity.n_neigh.sum())
    print(f"{variant.name}: simulate {steps} steps {dt * 1e3:.1f} ms ({dt / steps * 1e6:.1f} us/step), "
          f"{broken} broken, sum|u| {np.abs(st.u).sum():.12e}")
    import torch
    st = make_state(fam, False)
    ctx = engine.Context(0)
    ctx.upload(b, st, variant)
    stream = torch.cuda.ExternalStream(ctx.stream())
    ctx.run(steps, 0, eu, we, variant)  # warm
    torch.cuda.synchronize()
    ctx.close()
    st = make_state(fam, False)
    ctx = engine.Context(0)
    ctx.upload(b, st, variant)
    stream = torch.cuda.ExternalStream(ctx.stream())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.run(steps, 0, eu, we, variant)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ctx.download(st)
    broken = int(fam.n_neigh.sum() - st.connectivity.n_neigh.sum())
    print(f"{variant.name}: resident {steps} steps (write every {we}) {ms:.2f} ms "
          f"({ms / steps * 1e3:.2f} us/step), kernel {ctx.kernel()}, {broken} broken, "
          f"sum|u| {np.abs(st.u).sum():.12e}")
    ctx.close()
