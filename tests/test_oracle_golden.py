"""Pin the C oracle (oracle/pd_oracle.c) to the reference.

Every comparison is bitwise: the oracle restates the reference's operation
order and is compiled without FMA, so any difference is a restatement bug.
Golden fixtures come from the unmodified reference (tests/golden/make_golden.py);
where oracle/_ref is built (this container) the reference is also run live.
"""
import hashlib

import numpy as np
import pytest

import scenarios as S
from golden_io import random_case, same_bits, sim_case, tips_table
from paper_2105_04150_b200.abi import InvalidArgument, PeridynRuntimeError
from paper_2105_04150_b200.types import (ForceField, IntegratorKind, KernelVariant,
                                         SimulateOptions, make_state)

SIM_CASES = ["fracture", "trilinear", "plate", "beam", "multi", "lattice"]


def _seeds(d):
    return sorted({int(k[1:5]) for k in d.files if k.startswith("s")})


def test_random_forces_match_golden(oracle, golden):
    d = golden("random_forces")
    seeds = _seeds(d)
    assert len(seeds) >= 20
    for seed in seeds:
        for variant, tag in ((KernelVariant.bond_parallel, "bpr"), (KernelVariant.node_parallel, "node")):
            p, m, c, s = random_case(d, seed)
            f = ForceField()
            f.resize(p.size())
            oracle.compute_forces(variant, s, p, m, c, f)
            assert same_bits(f.body_force, d[f"s{seed}_{tag}_body"]), (seed, tag)
            assert np.array_equal(s.connectivity.entries, d[f"s{seed}_bpr_entries"]), (seed, tag)
            assert np.array_equal(s.connectivity.n_neigh, d[f"s{seed}_bpr_n_neigh"]), (seed, tag)
            assert same_bits(s.bond_history, d[f"s{seed}_bpr_history"]), (seed, tag)


def test_all_fifty_criterion_one_seeds_live(oracle, reference):
    """acceptance/main.cpp:46-70 seed set, oracle vs the compiled reference."""
    for seed in range(1000, 1050):
        for variant in (KernelVariant.bond_parallel, KernelVariant.node_parallel):
            outs = []
            for be in (reference, oracle):
                p, m, c, s = reference.random_config(seed)
                f = ForceField()
                f.resize(p.size())
                be.compute_forces(variant, s, p, m, c, f)
                outs.append((f.body_force, s.connectivity.entries, s.connectivity.n_neigh,
                             s.bond_history))
            for a, b in zip(*outs):
                assert same_bits(a, b), (seed, variant)


def _digest(st, forces):
    h = hashlib.sha256()
    for a in (st.u, st.v, st.a, st.connectivity.entries, st.connectivity.n_neigh,
              forces.body_force, forces.external_force):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("case", SIM_CASES)
def test_simulate_matches_golden(oracle, golden, case):
    d = golden("simulate")
    bundle, state, steps, we, first, integ = sim_case(d, case)
    digests = []
    res = oracle.simulate(bundle, state,
                          SimulateOptions(steps, we, first, IntegratorKind(integ),
                                          KernelVariant.bond_parallel),
                          lambda st, f: digests.append(_digest(st, f)))
    pre = case + "_out_"
    assert state.step == int(d[pre + "step"])
    for name in ("u", "v", "a"):
        assert same_bits(getattr(state, name), d[pre + name]), name
    assert np.array_equal(state.connectivity.entries, d[pre + "entries"])
    assert np.array_equal(state.connectivity.n_neigh, d[pre + "n_neigh"])
    if d[pre + "history"].size:
        assert same_bits(state.bond_history, d[pre + "history"])
    assert same_bits(tips_table(res), d[case + "_tips"])
    assert digests == list(d[case + "_hook_digests"])


def test_fracture_cases_actually_break(golden):
    d = golden("simulate")
    for case in ("fracture", "trilinear", "plate", "multi", "lattice"):
        assert d[case + "_n_neigh"].sum() > d[case + "_out_n_neigh"].sum(), case


def test_family_matches_golden(oracle, golden):
    d = golden("family")
    fam = oracle.build_family(d["random_coords"], 1.1)
    assert fam.group_size == int(d["random_group"])
    assert np.array_equal(fam.entries, d["random_entries"])
    from paper_2105_04150_b200.geometry import GridDesc, grid_coordinates
    g = GridDesc((0.0, 0.0, 0.0), 1.0, (10, 10, 10))
    fam = oracle.build_family(grid_coordinates(g), np.pi, g.hint())
    assert fam.group_size == int(d["grid_group"]) == 128
    assert np.array_equal(fam.entries, d["grid_entries"])
    assert fam.n_neigh.max() == 122  # acceptance criterion 7


def test_plane_cut_damage_matches_golden(oracle, golden):
    d = golden("family")
    from paper_2105_04150_b200.geometry import GridDesc, grid_coordinates
    g = GridDesc((0.0, 0.0, 0.0), 1.0, (20, 20, 20))
    gc = grid_coordinates(g)
    fam = oracle.build_family(gc, 3.0, g.hint())
    oracle.break_plane(fam, gc, 0, 9.5)
    assert np.array_equal(fam.entries, d["cut_entries"])
    assert np.array_equal(fam.n_neigh, d["cut_n_neigh"])
    assert same_bits(oracle.damage(fam), d["cut_phi"])


def test_ramps_match_golden(oracle, golden):
    t = golden("ramps")["table"]
    for kind, rise, target, step, sc, ra, ac in t:
        args = (int(kind), int(rise), float(target), int(step))
        assert same_bits(np.float64(oracle.ramp("scale", *args)), np.float64(sc))
        assert same_bits(np.float64(oracle.ramp("rate", *args)), np.float64(ra))
        assert same_bits(np.float64(oracle.ramp("accel", *args)), np.float64(ac))


def test_reduce_group_known_answers(oracle):
    """test_engine.cpp:14-40"""
    v = np.array([[1, 1, 1], [2, 2, 2], [3, 3, 3], [4, 4, 4]], dtype=np.float64)
    assert np.array_equal(oracle.reduce_group(v), [10, 10, 10])
    assert np.array_equal(oracle.reduce_group(np.zeros((64, 3))), [0, 0, 0])
    assert oracle.reduce_group(np.array([[5.0, 6.0, 7.0]]))[1] == 6
    rng = np.random.default_rng(3)
    r = rng.uniform(-1, 1, (128, 3))
    assert np.allclose(oracle.reduce_group(r), r.sum(axis=0), rtol=1e-13)
    with pytest.raises(InvalidArgument):
        oracle.reduce_group(np.zeros((3, 3)))


def test_error_behaviour_matches_reference(oracle, reference):
    """steps < 1, non-finite u with the step index, bad dt (engine.cpp:23-28, 335-341, 376-377)."""
    bundle, h, _ = S.small_fracture_bundle()
    fam = oracle.build_family(bundle.particles.coords, h)
    for be in (oracle, reference):
        st = make_state(fam, False)
        with pytest.raises(InvalidArgument, match="steps must be >= 1"):
            be.simulate(bundle, st, SimulateOptions(0))
        st = make_state(fam, False)
        st.u[5] = np.nan
        st.step = 77
        f = ForceField()
        f.resize(bundle.particles.size())
        with pytest.raises(PeridynRuntimeError, match="77"):
            be.compute_forces(KernelVariant.bond_parallel, st, bundle.particles, bundle.model,
                              bundle.corrections, f)
    # NaN injected mid-run: state at the throw is identical for both
    outs = []
    for be in (oracle, reference):
        st = make_state(fam, False)
        st.v[:] = 0.0
        st.v[7] = np.inf
        with pytest.raises(PeridynRuntimeError) as ei:
            be.simulate(bundle, st, SimulateOptions(5, 0, 10, IntegratorKind.velocity_verlet))
        outs.append((str(ei.value), st.u.copy(), st.v.copy(), st.a.copy(), st.step))
    assert outs[0][0] == outs[1][0]
    assert outs[0][4] == outs[1][4] == 10
    for a, b in zip(outs[0][1:4], outs[1][1:4]):
        assert same_bits(a, b)
