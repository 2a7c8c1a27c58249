"""pd_simulate_batch: independent simulate() calls run concurrently on one GPU
(the calibration / UQ outer loop).  Every model's result must equal its own
one-at-a-time run: bitwise for the exact variant (against the oracle)."""
import numpy as np
import pytest

import scenarios as S
from golden_io import same_bits, tips_table
from paper_2105_04150_b200 import engine
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, SimulateOptions, make_state

pytestmark = pytest.mark.gpu


def _plate(oracle, pull):
    b, h, g, notch = S.notched_plate_bundle(20, 16, 6, 40, pull=pull)
    fam = oracle.build_family(b.particles.coords, h, g.hint())
    oracle.break_notch(fam, b.particles.coords, notch["axis"], notch["position"],
                       notch["sweep_axis"], notch["depth"])
    return b, fam


def test_batch_equals_individual_runs(oracle):
    cases = []
    for k, pull in enumerate((0.2, 0.4, 0.6, 0.8, 1.0, 1.2)):
        b, fam = _plate(oracle, pull)
        integ = list(IntegratorKind)[k % 3]
        cases.append((b, fam, SimulateOptions(60, 20, 0, integ, KernelVariant.bond_parallel)))
    states = [make_state(fam, b.model.needs_history()) for b, fam, _ in cases]
    res = engine.simulate_batch([c[0] for c in cases], states, [c[2] for c in cases], threads=3)
    for (b, fam, o), st, r in zip(cases, states, res):
        ref = make_state(fam, b.model.needs_history())
        rr = oracle.simulate(b, ref, o)
        for name in ("u", "v", "a"):
            assert same_bits(getattr(ref, name), getattr(st, name)), name
        assert np.array_equal(ref.connectivity.entries, st.connectivity.entries)
        assert same_bits(tips_table(rr), tips_table(r))
    assert sum(fam.n_neigh.sum() - st.connectivity.n_neigh.sum()
               for (b, fam, o), st in zip(cases, states)) > 0


def test_batch_reports_the_failing_model(oracle):
    b, fam = _plate(oracle, 0.4)
    bad = S.notched_plate_bundle(20, 16, 6, 40)[0]
    bad.dt = -1.0
    with pytest.raises(Exception, match="model 1"):
        engine.simulate_batch([b, bad], [make_state(fam, True), make_state(fam, True)],
                              [SimulateOptions(5), SimulateOptions(5)])
