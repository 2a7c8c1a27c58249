import os, sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import scenarios as S
from paper_2105_04150_b200 import engine, geometry
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, SimulateOptions, make_state, ForceField
def run(case, steps):
    if case == "multi":
        b, h, g = S.multimaterial_bundle((16, 8, 10))
        fam = geometry.build_family(b.particles.coords, h, g)
        fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    else:
        b, h, g, notch = S.notched_plate_bundle(32, 32, 4, 100)
        fam = geometry.build_family(b.particles.coords, h, g)
    out = {}
    for forced in (None, "general"):
        if forced: os.environ["PD_FAST_LAYOUT"] = forced
        else: os.environ.pop("PD_FAST_LAYOUT", None)
        ctx = engine.Context(0)
        st = make_state(fam, True)
        if SEED: st.u = S.seed_displacements(b.particles.coords) * 1.0
        ctx.upload(b, st, KernelVariant.fast)
        lay = ctx.layout()
        ctx.run(steps, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.fast)
        ctx.download(st)
        ctx.close()
        out[lay] = st
    a, t = out["lattice"], out["tiles"]
    for k in ("u", "v", "a", "bond_history"):
        x, y = getattr(a, k), getattr(t, k)
        d = np.abs(x - y); sc = np.max(np.abs(y)) + 1e-300
        idx = np.unravel_index(np.argmax(d), d.shape)
        print(case, steps, k, "maxdiff/scale", float(np.max(d) / sc), "finite", np.isfinite(x).all(), "at", idx, x.flat[np.argmax(d)], y.flat[np.argmax(d)])
    print("nneigh diff", int((a.connectivity.n_neigh != t.connectivity.n_neigh).sum()))
SEED = False
for case in ("plate", "multi"):
    for steps in (1, 2, 3, 4, 5, 6, 7):
        try:
            run(case, steps)
        except Exception as e:
            print(case, steps, "ERR", e)
