"""The reference's force-pass cases (test_engine.cpp:67-194) on the device,
for the exact variants (bitwise against the C oracle) and the fast variant
(the reference's own expectations), plus the degenerate shapes the reference
handles: one node, isolated nodes (empty rows), group size 1, a row of
padding only, and a model that breaks every bond in one pass."""
import numpy as np
import pytest

import scenarios as S
from paper_2105_04150_b200 import abi, engine, geometry
from paper_2105_04150_b200.types import (BoundaryConditions, Corrections, DamageLaw,
                                         DamageModel, ForceField, IntegratorKind, KernelVariant,
                                         ModelBundle, ParticleSet, SimulateOptions, make_state)

pytestmark = pytest.mark.gpu

VARIANTS = (KernelVariant.bond_parallel, KernelVariant.node_parallel, KernelVariant.fast)


def two_node(c=2.0, v1=1.0, v2=1.0, stretch=0.0):
    """TwoNode::make (test_engine.cpp:46-63)."""
    p = ParticleSet(np.array([0, 0, 0, 1, 0, 0], np.float64), np.array([v1, v2]), np.ones(2),
                    np.zeros(2, np.uint16))
    fam = geometry.build_family(p.coords, 1.5)
    st = make_state(fam, False)
    st.u[3] = stretch
    return p, DamageModel([DamageLaw.pmb(c, 0.5)]), st


def forces(n, ext=None):
    f = ForceField()
    f.resize(n)
    if ext is not None:
        f.external_force[:] = ext
    return f


def both(oracle, variant, p, model, st, corr=None):
    """compute_forces on the device and (exact variants) on the oracle."""
    corr = corr or Corrections()
    out = []
    bes = (engine.backend(), oracle) if variant != KernelVariant.fast else (engine.backend(),)
    for be in bes:
        s = make_state(st.connectivity, False)
        s.u = st.u.copy()
        s.step = st.step
        f = forces(p.size())
        be.compute_forces(variant, s, p, model, corr, f)
        out.append((s, f))
    if len(out) == 2:
        (a, fa), (b, fb) = out
        assert np.array_equal(fa.body_force.view(np.uint64), fb.body_force.view(np.uint64))
        assert np.array_equal(a.connectivity.entries, b.connectivity.entries)
        assert np.array_equal(a.connectivity.n_neigh, b.connectivity.n_neigh)
    return out[0]


@pytest.mark.parametrize("variant", VARIANTS)
def test_single_bond_force(oracle, variant):
    """test_engine.cpp:67-83"""
    c, v1, v2, s = 3.0, 1.5, 2.5, 0.01
    p, model, st = two_node(c, v1, v2, s)
    model = DamageModel([DamageLaw.pmb(c, 0.5)])
    _, f = both(oracle, variant, p, model, st)
    tol = 1e-13 if variant != KernelVariant.fast else 2e-5
    assert f.body_force[0] == pytest.approx(c * s * v2, rel=tol)
    assert f.body_force[1] == 0.0
    assert f.body_force[3] == pytest.approx(-c * s * v1, rel=tol)


@pytest.mark.parametrize("variant", VARIANTS)
def test_all_bonds_broken_gives_zero_force(oracle, variant):
    """test_engine.cpp:85-96: rows of padding only."""
    p, model, st = two_node(stretch=0.01)
    st.connectivity.entries[:] = -1
    st.connectivity.n_neigh[:] = 0
    _, f = both(oracle, variant, p, model, st)
    assert not f.body_force.any()


@pytest.mark.parametrize("variant", VARIANTS)
def test_zero_displacement_zero_force_keeps_external(oracle, variant):
    """test_engine.cpp:98-108: the external force array is preserved."""
    p, model, st = two_node()
    f = forces(2)
    f.external_force[1] = 7.0
    engine.backend().compute_forces(variant, st, p, model, Corrections(), f)
    assert not f.body_force.any()
    assert f.external_force[1] == 7.0


@pytest.mark.parametrize("variant", VARIANTS)
def test_break_is_fused_and_irreversible(oracle, variant):
    """test_engine.cpp:110-122"""
    p, model, st = two_node(stretch=0.6)  # beyond s_c = 0.5
    s, f = both(oracle, variant, p, model, st)
    assert list(s.connectivity.n_neigh) == [0, 0] and f.body_force[0] == 0.0
    s.u[3] = 0.0
    s2, _ = both(oracle, variant, p, model, s)
    assert list(s2.connectivity.n_neigh) == [0, 0]


@pytest.mark.parametrize("variant", VARIANTS)
def test_no_failure_nodes_keep_their_bonds(oracle, variant):
    """test_engine.cpp:124-136"""
    p, model, st = two_node(stretch=0.6)
    corr = Corrections(no_failure=np.array([1, 0], np.uint8))
    s, f = both(oracle, variant, p, model, st, corr)
    assert list(s.connectivity.n_neigh) == [1, 1]
    tol = 1e-12 if variant != KernelVariant.fast else 2e-5
    assert f.body_force[0] == pytest.approx(2 * 0.6 * 1, rel=tol)


@pytest.mark.parametrize("variant", VARIANTS)
def test_momentum_balance(oracle, variant):
    """test_engine.cpp:168-184: equal volumes, no corrections."""
    b, h, g = S.bench_lattice_bundle((11, 10, 9), s_c=1e6)
    fam = geometry.build_family(b.particles.coords, h, g)
    st = make_state(fam, False)
    st.u = S.seed_displacements(b.particles.coords) * 50.0
    f = forces(fam.node_count())
    engine.backend().compute_forces(variant, st, b.particles, b.model, Corrections(), f)
    terms = f.body_force.reshape(-1, 3)
    scale = np.abs(terms).sum()
    tol = 1e-10 if variant != KernelVariant.fast else 1e-5
    assert np.all(np.abs(terms.sum(0)) <= tol * scale)


@pytest.mark.parametrize("variant", VARIANTS)
def test_nonfinite_displacement_names_the_step(oracle, variant):
    """test_engine.cpp:186-194"""
    p, model, st = two_node(stretch=0.01)
    st.step = 77
    st.u[0] = np.nan
    with pytest.raises(abi.PeridynRuntimeError, match="77"):
        engine.backend().compute_forces(variant, st, p, model, Corrections(), forces(2))


@pytest.mark.parametrize("variant", VARIANTS)
def test_degenerate_models(oracle, variant):
    """One node (group size 1, an empty row), isolated nodes beside a bonded
    pair, through compute_forces and a 5-step simulate."""
    cases = [np.array([0, 0, 0], np.float64),                       # n = 1
             np.array([0, 0, 0, 1, 0, 0, 10, 0, 0, 20, 5, 0], np.float64)]  # isolated nodes
    for coords in cases:
        n = coords.size // 3
        p = ParticleSet(coords, np.ones(n), np.ones(n), np.zeros(n, np.uint16))
        fam = geometry.build_family(coords, 1.5)
        assert fam.group_size >= 1
        model = DamageModel([DamageLaw.pmb(2.0, 0.5)])
        st = make_state(fam, False)
        st.u = np.linspace(0, 1e-3, 3 * n)
        both(oracle, variant, p, model, st)
        bundle = ModelBundle(p, model, Corrections(), BoundaryConditions.none(n), 1e-3)
        outs = []
        bes = (engine.backend(), oracle) if variant != KernelVariant.fast else (engine.backend(),)
        for be in bes:
            s2 = make_state(fam, False)
            s2.u = st.u.copy()
            be.simulate(bundle, s2, SimulateOptions(5, 0, 0, IntegratorKind.velocity_verlet,
                                                    variant))
            outs.append(s2)
        if len(outs) == 2:
            assert np.array_equal(outs[0].u.view(np.uint64), outs[1].u.view(np.uint64))
        assert outs[0].step == 5
