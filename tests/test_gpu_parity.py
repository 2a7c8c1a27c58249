"""GPU parity: the CUDA path through the C ABI against the reference's golden
vectors and the C oracle.  The fp64 variants (bond_parallel, node_parallel)
must be BITWISE equal -- body forces, u/v/a, the broken-bond set (entries),
n_neigh, bond history, tips and the state every write hook sees."""
import hashlib

import numpy as np
import pytest

import scenarios as S
from golden_io import random_case, same_bits, sim_case, tips_table
from paper_2105_04150_b200 import abi, engine, geometry
from paper_2105_04150_b200.types import (ForceField, IntegratorKind, KernelVariant,
                                         SimulateOptions, make_state)

pytestmark = pytest.mark.gpu

EXACT = (KernelVariant.bond_parallel, KernelVariant.node_parallel)


def _digest(st, forces):
    h = hashlib.sha256()
    for a in (st.u, st.v, st.a, st.connectivity.entries, st.connectivity.n_neigh,
              forces.body_force, forces.external_force):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _assert_same_state(a, b):
    assert a.step == b.step
    for name in ("u", "v", "a"):
        assert same_bits(getattr(a, name), getattr(b, name)), name
    assert np.array_equal(a.connectivity.entries, b.connectivity.entries)
    assert np.array_equal(a.connectivity.n_neigh, b.connectivity.n_neigh)
    ha = a.bond_history if a.bond_history is not None else np.zeros(0)
    hb = b.bond_history if b.bond_history is not None else np.zeros(0)
    assert same_bits(np.asarray(ha, np.float64), np.asarray(hb, np.float64))


# ---- golden vectors from the reference ----------------------------------------

def test_gpu_random_forces_match_golden(golden):
    d = golden("random_forces")
    seeds = sorted({int(k[1:5]) for k in d.files if k.startswith("s")})
    for seed in seeds:
        for variant, tag in ((KernelVariant.bond_parallel, "bpr"), (KernelVariant.node_parallel, "node")):
            p, m, c, s = random_case(d, seed)
            f = ForceField()
            f.resize(p.size())
            engine.compute_forces(variant, s, p, m, c, f)
            assert same_bits(f.body_force, d[f"s{seed}_{tag}_body"]), (seed, tag)
            assert np.array_equal(s.connectivity.entries, d[f"s{seed}_bpr_entries"]), (seed, tag)
            assert np.array_equal(s.connectivity.n_neigh, d[f"s{seed}_bpr_n_neigh"]), (seed, tag)
            assert same_bits(s.bond_history, d[f"s{seed}_bpr_history"]), (seed, tag)


@pytest.mark.parametrize("case", ["fracture", "trilinear", "plate", "beam", "multi", "lattice"])
def test_gpu_simulate_matches_golden(golden, case):
    d = golden("simulate")
    bundle, state, steps, we, first, integ = sim_case(d, case)
    digests = []
    res = engine.simulate(bundle, state,
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


def test_gpu_family_matches_golden(golden):
    d = golden("family")
    fam = geometry.build_family(d["random_coords"], 1.1)
    assert fam.group_size == int(d["random_group"])
    assert np.array_equal(fam.entries, d["random_entries"])
    g = geometry.GridDesc((0.0, 0.0, 0.0), 1.0, (10, 10, 10))
    fam = geometry.build_family(geometry.grid_coordinates(g), np.pi, g)
    assert fam.group_size == 128 and fam.n_neigh.max() == 122
    assert np.array_equal(fam.entries, d["grid_entries"])


def test_gpu_damage_matches_golden(golden):
    d = golden("family")
    g = geometry.GridDesc((0.0, 0.0, 0.0), 1.0, (20, 20, 20))
    gc = geometry.grid_coordinates(g)
    fam = geometry.build_family(gc, 3.0, g)
    geometry.break_plane(fam, gc, 0, 9.5)
    assert np.array_equal(fam.entries, d["cut_entries"])
    assert same_bits(engine.local_damage(fam), d["cut_phi"])


# ---- wider coverage against the C oracle ----------------------------------------

@pytest.mark.parametrize("seed", range(30))
def test_gpu_random_configs_match_oracle(oracle, seed):
    """numpy analogue of make_random_config at up to 4000 nodes, both variants."""
    p, model, horizon, draws, rng = S.random_config_np(seed, (10, 4000) if seed % 3 == 0 else (10, 500))
    fam = oracle.build_family(p.coords, horizon)
    if fam.group_size > 1024:
        pytest.skip("group size beyond the supported 1024")
    corr, st0 = S.finish_random_config(p, model, fam, draws, rng)
    hist0 = np.abs(rng.normal(0, 0.02, fam.entries.size)) * (seed % 2)
    for variant in EXACT:
        outs = []
        for be in (oracle, engine.backend()):
            st = make_state(st0.connectivity, model.needs_history())
            st.u = st0.u.copy()
            if model.needs_history():
                st.bond_history = hist0.copy()
            f = ForceField()
            f.resize(p.size())
            be.compute_forces(variant, st, p, model, corr, f)
            outs.append((f, st))
        assert same_bits(outs[0][0].body_force, outs[1][0].body_force), variant
        _assert_same_state(outs[0][1], outs[1][1])


@pytest.mark.parametrize("horizon,group", [(5.2, 1024), (4.2, 512)])
def test_gpu_large_groups_match_oracle(oracle, horizon, group):
    """Families beyond 256 members (the reference allows any power of two,
    types.hpp:63-73): a lattice with a wide horizon, fracturing, both exact
    variants and the fast variant's tile path, 20 velocity-Verlet steps."""
    b, h, g = S.bench_lattice_bundle((14, 13, 12), s_c=2e-4, horizon=horizon)
    fam = oracle.build_family(b.particles.coords, horizon, g.hint())
    assert fam.group_size == group
    dev = geometry.build_family(b.particles.coords, horizon, g)
    assert np.array_equal(dev.entries, fam.entries)
    u0 = S.seed_displacements(b.particles.coords) * 30.0
    for variant in EXACT:
        outs = []
        for be in (oracle, engine.backend()):
            st = make_state(fam, False)
            st.u = u0.copy()
            be.simulate(b, st, SimulateOptions(20, 0, 0, IntegratorKind.velocity_verlet, variant))
            outs.append(st)
        _assert_same_state(outs[0], outs[1])
        assert int(fam.n_neigh.sum() - outs[1].connectivity.n_neigh.sum()) > 0
    st = make_state(fam, False)
    st.u = u0.copy()
    engine.simulate(b, st, SimulateOptions(20, 0, 0, IntegratorKind.velocity_verlet,
                                           KernelVariant.fast))
    scale = np.abs(outs[0].u).max()
    assert np.abs(st.u - outs[0].u).max() <= 5e-3 * scale


def _plate(oracle, nx=40, ny=40, nz=4, steps=120):
    b, h, g, notch = S.notched_plate_bundle(nx, ny, nz, steps)
    fam = oracle.build_family(b.particles.coords, h, g.hint())
    oracle.break_notch(fam, b.particles.coords, notch["axis"], notch["position"],
                       notch["sweep_axis"], notch["depth"])
    return b, fam


@pytest.mark.parametrize("integrator", list(IntegratorKind))
def test_gpu_simulate_integrators_match_oracle(oracle, integrator):
    b, fam = _plate(oracle, 32, 32, 4, 100)
    b.model.damping = 0.02
    outs = []
    for be in (oracle, engine.backend()):
        st = make_state(fam, b.model.needs_history())
        digests = []
        res = be.simulate(b, st, SimulateOptions(100, 20, 3, integrator),
                          lambda s, f: digests.append(_digest(s, f)))
        outs.append((st, tips_table(res), digests))
    _assert_same_state(outs[0][0], outs[1][0])
    assert same_bits(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]
    assert fam.n_neigh.sum() > outs[1][0].connectivity.n_neigh.sum()  # it fractured


def test_gpu_lattice_fracture_variant_matches_oracle(oracle):
    """The bench's fracturing variant (s_c = 1e-5) on 24^3 with the node variant too."""
    b, h, g = S.bench_lattice_bundle((24, 24, 24), s_c=1e-5)
    fam = geometry.build_family(b.particles.coords, h, g)
    assert np.array_equal(fam.entries, oracle.build_family(b.particles.coords, h, g.hint()).entries)
    for variant in EXACT:
        outs = []
        for be in (oracle, engine.backend()):
            st = make_state(fam, False)
            st.u = S.seed_displacements(b.particles.coords)
            be.simulate(b, st, SimulateOptions(30, 0, 0, IntegratorKind.velocity_verlet, variant))
            outs.append(st)
        _assert_same_state(*outs)
        broken = fam.n_neigh.sum() - outs[1].connectivity.n_neigh.sum()
        assert broken > 0.01 * fam.n_neigh.sum()


def test_gpu_trilinear_multimaterial_matches_oracle(oracle):
    b, h, g = S.multimaterial_bundle((16, 8, 8))
    fam = geometry.build_family(b.particles.coords, h, g)
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    b.corrections.beta = np.random.default_rng(1).uniform(0.7, 1.0, fam.entries.size)
    outs = []
    for be in (oracle, engine.backend()):
        st = make_state(fam, True)
        res = be.simulate(b, st, SimulateOptions(150, 25, 0, IntegratorKind.velocity_verlet))
        outs.append((st, tips_table(res)))
    _assert_same_state(outs[0][0], outs[1][0])
    assert same_bits(outs[0][1], outs[1][1])


def test_gpu_family_matches_oracle_random_points(oracle):
    rng = np.random.default_rng(11)
    for n, side, horizon in ((5000, 12.0, 1.3), (20000, 20.0, 1.9), (3000, 30.0, 0.8)):
        coords = rng.uniform(0, side, 3 * n)
        a = oracle.build_family(coords, horizon)
        b = geometry.build_family(coords, horizon)
        assert a.group_size == b.group_size
        assert np.array_equal(a.entries, b.entries)
        assert np.array_equal(a.n_neigh, b.n_neigh)


def test_gpu_coincident_nodes_rejected():
    coords = np.array([0, 0, 0, 1, 0, 0, 1, 0, 0], dtype=np.float64)
    with pytest.raises(abi.InvalidArgument, match="coincident"):
        geometry.build_family(coords, 1.5)


# ---- error semantics, restart, determinism ----------------------------------------

@pytest.mark.parametrize("integrator", list(IntegratorKind))
def test_gpu_nonfinite_midrun_matches_oracle(oracle, integrator):
    """A blow-up mid-run raises at the same step with the same state as the reference."""
    b, h, _ = S.small_fracture_bundle()
    fam = oracle.build_family(b.particles.coords, h)
    b.model.laws[0] = type(b.model.laws[0]).pmb(0.05, 1e9)
    b.bc.kind[:] = 0
    b.bc.kind[3 * 7] = 2  # force axis with an enormous load
    b.bc.magnitude[3 * 7] = 1.5e308
    outs = []
    for be in (oracle, engine.backend()):
        st = make_state(fam, False)
        with pytest.raises(abi.PeridynRuntimeError) as ei:
            be.simulate(b, st, SimulateOptions(120, 5, 2, integrator))
        outs.append((str(ei.value), st))
    assert outs[0][0] == outs[1][0]
    _assert_same_state(outs[0][1], outs[1][1])


def test_gpu_restart_is_bitwise(oracle):
    """test_engine.cpp:443-470 on the device."""
    b, h, _ = S.small_fracture_bundle()
    fam = oracle.build_family(b.particles.coords, h)
    whole = make_state(fam, False)
    r1 = engine.simulate(b, whole, SimulateOptions(120, 30))
    split = make_state(fam, False)
    engine.simulate(b, split, SimulateOptions(50, 30))
    r2 = engine.simulate(b, split, SimulateOptions(70, 30, 50))
    _assert_same_state(whole, split)
    assert r2.tips["pull"][0].step == 60
    assert r2.tips["pull"][-1].step == r1.tips["pull"][-1].step


def test_gpu_context_matches_one_shot(oracle):
    b, fam = _plate(oracle, 24, 24, 4, 60)
    st1 = make_state(fam, b.model.needs_history())
    engine.simulate(b, st1, SimulateOptions(60, 0, 0, IntegratorKind.euler_cromer))
    ctx = engine.Context()
    st2 = make_state(fam, b.model.needs_history())
    ctx.upload(b, st2)
    ctx.run(25, 0, IntegratorKind.euler_cromer)
    ctx.run(35, 25, IntegratorKind.euler_cromer)
    ctx.download(st2)
    _assert_same_state(st1, st2)
    phi = ctx.damage()
    assert same_bits(phi, oracle.damage(st1.connectivity))
    assert ctx.live_bonds() == int(st1.connectivity.n_neigh.sum())
    assert ctx.launch_count() > 60
    ctx.close()


def test_gpu_deterministic_repeat(oracle):
    b, fam = _plate(oracle, 32, 32, 4, 80)
    outs = []
    for _ in range(2):
        st = make_state(fam, b.model.needs_history())
        engine.simulate(b, st, SimulateOptions(80, 0, 0, IntegratorKind.euler_cromer))
        outs.append(st)
    _assert_same_state(*outs)


# ---- BASELINE cfg3 size: 1M nodes, bitwise against the oracle ------------------

def test_gpu_million_node_lattice_matches_oracle(oracle):
    b, h, g = S.bench_lattice_bundle((100, 100, 100))
    fam = geometry.build_family(b.particles.coords, h, g)
    assert fam.group_size == 128
    assert int(fam.n_neigh.sum()) == 117_844_248
    outs = []
    for be in (engine.backend(), oracle):
        st = make_state(fam, False)
        st.u = S.seed_displacements(b.particles.coords)
        be.simulate(b, st, SimulateOptions(3, 0, 0, IntegratorKind.velocity_verlet))
        outs.append(st)
    _assert_same_state(*outs)


def test_gpu_many_breakpoint_law_matches_oracle(oracle, reference):
    """A piecewise-linear softening law with 12 breakpoints (the reference
    allows any count, types.hpp:75-91): the exact variants run it bitwise
    against the C oracle and the reference; the fast variant, whose kernels
    keep 8-breakpoint tables, refuses it with a clear error."""
    from paper_2105_04150_b200.types import DamageLaw
    b, h, g = S.bench_lattice_bundle((12, 11, 10), s_c=1e6)
    bp = [2e-4 * (k + 1) for k in range(12)]
    c = 1.0
    f = [c * bp[0]] + [c * bp[0] * (1.0 - k / 11.0) for k in range(1, 12)]
    law = DamageLaw(c, bp, f)
    law.validate()
    b.model.laws = [law]
    fam = geometry.build_family(b.particles.coords, h, g)
    u0 = S.seed_displacements(b.particles.coords) * 300.0
    outs = []
    for be in (oracle, reference, engine.backend()):
        st = make_state(fam, True)
        st.u = u0.copy()
        be.simulate(b, st, SimulateOptions(15, 0, 0, IntegratorKind.velocity_verlet,
                                           KernelVariant.bond_parallel))
        outs.append(st)
    for other in outs[1:]:
        _assert_same_state(outs[0], other)
    assert int(fam.n_neigh.sum() - outs[2].connectivity.n_neigh.sum()) > 0
    assert np.count_nonzero(outs[2].bond_history) > 0
    st = make_state(fam, True)
    st.u = u0.copy()
    with pytest.raises(abi.InvalidArgument, match="at most 8"):
        engine.simulate(b, st, SimulateOptions(2, 0, 0, IntegratorKind.velocity_verlet,
                                               KernelVariant.fast))
