"""Generate the binary-container fixtures (tests/golden/*.pdst, *.pdnl) with
the UNMODIFIED reference's io::save_state / io::save_cache (io.cpp:416-505),
via oracle/_ref.  Run here, where /root/reference is mounted:

    python tests/golden/make_golden_io.py

state_trilinear.pdst  a fractured trilinear multi-material bar after 40
                      velocity-Verlet steps of the reference simulate(): u, v,
                      a, entries with breaks, counts, bond types, history
state_pmb.pdst        the PMB bench lattice (no history / bond types)
snap_trilinear.pdsnap write_snapshot(make_snapshot(...)) of the trilinear state
family.pdnl           a family cache with bond types, lambda and beta
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.pyoracle import Reference  # noqa: E402
from paper_2105_04150_b200.types import (IntegratorKind, SimulateOptions,  # noqa: E402
                                         make_state)
import scenarios as S  # noqa: E402


def trilinear_case(ref):
    b, h, g = S.multimaterial_bundle((7, 5, 6))
    fam = ref.build_family(b.particles.coords, 2.0, g.hint())
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    st = make_state(fam, True)
    ref.simulate(b, st, SimulateOptions(40, 0, 0, IntegratorKind.velocity_verlet))
    return b, fam, st


def main():
    ref = Reference(threads=1)
    b, fam, st = trilinear_case(ref)
    ref.save_state(st, os.path.join(HERE, "state_trilinear.pdst"))
    ref.write_snapshot(st, b.particles, os.path.join(HERE, "snap_trilinear.pdsnap"))
    bb, h, g = S.bench_lattice_bundle((6, 5, 4))
    fam2 = ref.build_family(bb.particles.coords, 2.0, g.hint())
    st2 = make_state(fam2, False)
    st2.u = S.seed_displacements(bb.particles.coords)
    st2.step = 7
    ref.save_state(st2, os.path.join(HERE, "state_pmb.pdst"))
    rng = np.random.default_rng(5)
    from paper_2105_04150_b200.types import Corrections
    corr = Corrections(rng.uniform(0.5, 1.5, fam.entries.size), rng.uniform(0.5, 1.0, fam.entries.size),
                       None)
    ref.save_cache(fam, corr, os.path.join(HERE, "family.pdnl"))
    print("broken bonds in the trilinear state:",
          int(fam.n_neigh.sum() - st.connectivity.n_neigh.sum()))


if __name__ == "__main__":
    main()
