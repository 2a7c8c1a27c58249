import sys, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import scenarios as S
from oracle.pyoracle import COracle
from paper_2105_04150_b200 import engine
from paper_2105_04150_b200.types import *
o = COracle(threads=8)
b, h, g, notch = S.notched_plate_bundle(32, 32, 4, 100)
fam = o.build_family(b.particles.coords, h, g.hint())
o.break_notch(fam, b.particles.coords, notch["axis"], notch["position"], notch["sweep_axis"], notch["depth"])
n = b.particles.size()
for integ in (IntegratorKind.euler_cromer, IntegratorKind.velocity_verlet):
  for nfon in (True, False):
    bb = b
    if not nfon:
        import copy; bb = copy.deepcopy(b); bb.bc.no_failure[:] = 0
    hist = {}
    for name, be, var in (("oracle", o, KernelVariant.bond_parallel), ("fast", engine.backend(), KernelVariant.fast)):
        st = make_state(fam, True)
        rec = []
        be.simulate(bb, st, SimulateOptions(100, 10, 0, integ, var), lambda s, f: rec.append((int(s.connectivity.n_neigh.sum()), float(np.abs(s.u).max()), float(np.abs(f.body_force).max()))))
        hist[name] = rec
    print(integ.name, "nf" if nfon else "--")
    for a, c in zip(hist["oracle"], hist["fast"]):
        print("   ", a, c)
