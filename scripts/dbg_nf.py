import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import scenarios as S
from oracle.pyoracle import COracle
from paper_2105_04150_b200 import engine
from paper_2105_04150_b200.types import *
o = COracle(threads=8)
b, h, g, notch = S.notched_plate_bundle(32, 32, 4, 100)
fam = o.build_family(b.particles.coords, h, g.hint())
n = b.particles.size()
rng = np.random.default_rng(0)
u = rng.normal(0, 0.05, 3*n)
for lawname, law in (("bilinear", b.model.laws[0]), ("pmb", DamageLaw.pmb(b.model.laws[0].stiffness, b.model.laws[0].breakpoints[0]))):
    for nf in (False, True):
        model = DamageModel([law])
        corr = Corrections(None, None, b.bc.no_failure.copy() if nf else None)
        outs = []
        for be, var in ((o, KernelVariant.bond_parallel), (engine.backend(), KernelVariant.fast)):
            st = make_state(fam, model.needs_history()); st.u = u.copy()
            f = ForceField(); f.resize(n)
            be.compute_forces(var, st, b.particles, model, corr, f)
            outs.append((f.body_force, st))
        ba = fam.n_neigh.sum() - outs[0][1].connectivity.n_neigh.sum()
        bb = fam.n_neigh.sum() - outs[1][1].connectivity.n_neigh.sum()
        d = outs[0][1].connectivity.entries != outs[1][1].connectivity.entries
        err = np.max(np.abs(outs[0][0]-outs[1][0]))/np.max(np.abs(outs[0][0]))
        print(lawname, "nf" if nf else "--", "broken oracle", ba, "fast", bb, "diff slots", d.sum(), "force err", err)
