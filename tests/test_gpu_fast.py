"""The fast path (KernelVariant.fast): fp32 bond arithmetic on shared-memory
staged tiles, fp64 state and integration.  Not bitwise; checked against the
fp64 C oracle with the tolerances stated in DESIGN.md:

  forces     max_rel_difference (oracles.hpp:215-228) <= FORCE_TOL per force pass
  breaks     identical broken sets except bonds whose fp64 stretch lies within
             EPS_S * s_c of the critical stretch
  state      trajectories (u, v) within TRAJ_TOL relative to the field scale for
             non-fracturing runs; FRACTURE_*_TOL and a 2 % broken-count band for
             runs with a propagating crack
"""
import numpy as np
import pytest

import scenarios as S
from paper_2105_04150_b200 import engine, geometry
from paper_2105_04150_b200.types import (BCKind, DamageLaw, ForceField, IntegratorKind,
                                         KernelVariant, SimulateOptions, make_state)

pytestmark = pytest.mark.gpu

FORCE_TOL = 2e-5
EPS_S = 1e-5
TRAJ_TOL = 1e-5
FRACTURE_U_TOL = 5e-3   # K-step fracturing runs (crack-tip divergence)
FRACTURE_V_TOL = 2e-2


def max_rel_difference(a, b):
    """oracles::max_rel_difference (tests/oracles.hpp:215-228)."""
    scale = max(np.max(np.abs(a)), 1e-300)
    denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), scale)
    return float(np.max(np.abs(a - b) / denom))


def stretches(p, fam, u):
    """fp64 stretch of every live slot, reference formula (engine.cpp:61-65)."""
    n = fam.node_count()
    N = fam.group_size
    ent = fam.entries.reshape(n, N)
    ii, kk = np.nonzero(ent >= 0)
    jj = ent[ii, kk]
    x = p.coords.reshape(n, 3)
    uu = u.reshape(n, 3)
    ref = x[jj] - x[ii]
    cur = ref + (uu[jj] - uu[ii])
    rl = np.sqrt((ref ** 2).sum(1))
    cl = np.sqrt((cur ** 2).sum(1))
    s = np.empty((n, N))
    s[:] = np.nan
    s[ii, kk] = (cl - rl) / rl
    return s.reshape(-1)


def check_break_sets(entries_a, entries_b, s, s_c):
    diff = entries_a != entries_b
    if diff.any():
        near = np.abs(s[diff] - s_c) <= EPS_S * s_c
        assert near.all(), f"{int((~near).sum())} broken-set differences away from s_c"
    return int(diff.sum())


@pytest.mark.parametrize("counts,s_c", [((24, 24, 24), 1e6), ((24, 24, 24), 1e-5),
                                        ((30, 20, 10), 1.5e-5)])
def test_fast_force_pass_matches_oracle(oracle, counts, s_c):
    b, h, g = S.bench_lattice_bundle(counts, s_c=s_c)
    fam = geometry.build_family(b.particles.coords, h, g)
    u = S.seed_displacements(b.particles.coords) * 3.0
    outs = []
    for be, variant in ((oracle, KernelVariant.bond_parallel), (engine.backend(), KernelVariant.fast)):
        st = make_state(fam, False)
        st.u = u.copy()
        f = ForceField()
        f.resize(b.particles.size())
        be.compute_forces(variant, st, b.particles, b.model, b.corrections, f)
        outs.append((f.body_force, st))
    err = max_rel_difference(outs[0][0], outs[1][0])
    assert err <= FORCE_TOL, err
    s = stretches(b.particles, fam, u)
    check_break_sets(outs[0][1].connectivity.entries, outs[1][1].connectivity.entries, s, s_c)
    assert np.array_equal(outs[1][1].connectivity.n_neigh,
                          (outs[1][1].connectivity.entries.reshape(fam.node_count(), -1) >= 0).sum(1))


@pytest.mark.parametrize("integrator", list(IntegratorKind))
def test_fast_plate_trajectory_matches_oracle(oracle, integrator):
    """cfg2 (downscaled): notched bilinear plate with BCs, all integrators."""
    b, h, g, notch = S.notched_plate_bundle(32, 32, 4, 100)
    fam = oracle.build_family(b.particles.coords, h, g.hint())
    oracle.break_notch(fam, b.particles.coords, notch["axis"], notch["position"],
                       notch["sweep_axis"], notch["depth"])
    outs = []
    for be, variant in ((oracle, KernelVariant.bond_parallel), (engine.backend(), KernelVariant.fast)):
        st = make_state(fam, True)
        res = be.simulate(b, st, SimulateOptions(100, 25, 0, integrator, variant))
        outs.append((st, res))
    (a, ra), (f, rf) = outs
    # a running crack amplifies rounding near its tip: bound the field, not the tip
    assert max_rel_difference(a.u, f.u) <= FRACTURE_U_TOL
    assert max_rel_difference(a.v, f.v) <= FRACTURE_V_TOL
    broken_a = fam.n_neigh.sum() - a.connectivity.n_neigh.sum()
    broken_f = fam.n_neigh.sum() - f.connectivity.n_neigh.sum()
    assert broken_a > 0
    assert abs(int(broken_a) - int(broken_f)) <= max(2, 0.02 * broken_a)
    assert set(ra.tips) == set(rf.tips)
    # n_neigh stays the live count of the materialised row (no double counting)
    live = (f.connectivity.entries.reshape(fam.node_count(), -1) >= 0).sum(1)
    assert np.array_equal(f.connectivity.n_neigh, live)


def test_fast_multimaterial_general_path(oracle):
    """bond types + trilinear history + beta through the GENERAL kernel."""
    b, h, g = S.multimaterial_bundle((16, 8, 8))
    fam = geometry.build_family(b.particles.coords, h, g)
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    b.corrections.beta = np.random.default_rng(1).uniform(0.7, 1.0, fam.entries.size)
    outs = []
    for be, variant in ((oracle, KernelVariant.bond_parallel), (engine.backend(), KernelVariant.fast)):
        st = make_state(fam, True)
        be.simulate(b, st, SimulateOptions(60, 0, 0, IntegratorKind.velocity_verlet, variant))
        outs.append(st)
    a, f = outs
    assert max_rel_difference(a.u, f.u) <= TRAJ_TOL * 100
    ha, hf = a.bond_history, f.bond_history
    assert max_rel_difference(ha, hf) <= 1e-3


def test_fast_random_configs_force_pass(oracle):
    for seed in range(8):
        p, model, horizon, draws, rng = S.random_config_np(100 + seed, (200, 3000))
        fam = oracle.build_family(p.coords, horizon)
        if fam.group_size > 256:
            continue
        corr, st0 = S.finish_random_config(p, model, fam, draws, rng)
        outs = []
        for be, variant in ((oracle, KernelVariant.bond_parallel),
                            (engine.backend(), KernelVariant.fast)):
            st = make_state(st0.connectivity, model.needs_history())
            st.u = st0.u.copy()
            f = ForceField()
            f.resize(p.size())
            be.compute_forces(variant, st, p, model, corr, f)
            outs.append((f.body_force, st))
        assert max_rel_difference(outs[0][0], outs[1][0]) <= FORCE_TOL, seed
        s = stretches(p, st0.connectivity, st0.u)
        check_break_sets(outs[0][1].connectivity.entries, outs[1][1].connectivity.entries, s,
                         model.laws[0].critical_stretch())


def test_fast_context_download_order(oracle):
    """The fast path renumbers nodes into bricks; downloads must come back in
    the reference's order (u, v, a, entries, n_neigh, damage, tips)."""
    b, h, g = S.bench_lattice_bundle((20, 18, 16), s_c=1e-5)
    b.bc.tip_sets["corner"] = [0, 1, 2, 19]
    fam = geometry.build_family(b.particles.coords, h, g)
    u0 = S.seed_displacements(b.particles.coords)
    outs = []
    for be, variant in ((oracle, KernelVariant.bond_parallel), (engine.backend(), KernelVariant.fast)):
        st = make_state(fam, False)
        st.u = u0.copy()
        res = be.simulate(b, st, SimulateOptions(20, 10, 0, IntegratorKind.velocity_verlet, variant))
        outs.append((st, res))
    (a, ra), (f, rf) = outs
    assert max_rel_difference(a.u, f.u) <= TRAJ_TOL
    assert max_rel_difference(a.v, f.v) <= TRAJ_TOL * 10
    ta = np.array([r.mean_u for r in ra.tips["corner"]])
    tf = np.array([r.mean_u for r in rf.tips["corner"]])
    assert np.allclose(ta, tf, rtol=1e-5, atol=1e-9)
    ctx = engine.Context()
    st = make_state(fam, False)
    st.u = u0.copy()
    ctx.upload(b, st, KernelVariant.fast)
    ctx.run(20, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.fast)
    ctx.download(st)
    assert np.array_equal(st.connectivity.n_neigh,
                          (st.connectivity.entries.reshape(fam.node_count(), -1) >= 0).sum(1))
    phi = ctx.damage()
    assert np.allclose(phi, 1.0 - st.connectivity.n_neigh / fam.initial_n_neigh)
    ctx.close()


def test_fast_million_node_lattice(oracle):
    """cfg3 size: 1M nodes, 3 fast steps vs the fp64 oracle."""
    b, h, g = S.bench_lattice_bundle((100, 100, 100))
    fam = geometry.build_family(b.particles.coords, h, g)
    outs = []
    for be, variant in ((engine.backend(), KernelVariant.fast), (oracle, KernelVariant.bond_parallel)):
        st = make_state(fam, False)
        st.u = S.seed_displacements(b.particles.coords)
        be.simulate(b, st, SimulateOptions(3, 0, 0, IntegratorKind.velocity_verlet, variant))
        outs.append(st)
    assert max_rel_difference(outs[1].u, outs[0].u) <= TRAJ_TOL
    assert max_rel_difference(outs[1].a, outs[0].a) <= FORCE_TOL


LAT_KERNELS = {  # PD_LAT_CFG -> the instantiation it selects on a 20x18x26 lattice
    "0": "lattice_small_kernel<1,0,0,8,8>",  # by size (below two 16x4x4 bricks per SM): persistent
    "1": "lattice_step_kernel<1,8,3,0,0>",  # the BENCH instantiation (16x4x8, 3 CTAs/SM)
    "4": "lattice_step_kernel<1,4,5,0,0>",  # 16x4x4 bricks at 5 CTAs/SM
    "5": "lattice_step_kernel<1,1,1,0,0>",  # the small-brick latency variant, forced
    "6": "lattice_step_kernel<1,4,6,0,0>",  # large-model rule without the waste test
    "9": "lattice_step_kernel<1,9,2,0,0>",  # 16x4x9 bricks (27-plane slabs of 216 / 8 GPUs)
    "10": "lattice_step_kernel<1,9,3,0,0>",  # 16x4x9 bricks at 3 CTAs/SM
}


@pytest.mark.parametrize("lat_cfg", sorted(LAT_KERNELS))
def test_lattice_layout_selected_and_matches_tiles(oracle, monkeypatch, lat_cfg):
    """PD_FAST on the bench lattice runs the implicit-connectivity kernel
    (pd_lattice.cu) on the brick shape PD_LAT_CFG selects (LAT_KERNELS, checked
    through pd_ctx_kernel); forced onto the general tile layout the same run
    must agree with it within the fast-path tolerance, and both with the
    oracle."""
    monkeypatch.setenv("PD_LAT_CFG", lat_cfg)
    b, h, g = S.bench_lattice_bundle((20, 18, 26), s_c=1.5e-5)
    fam = geometry.build_family(b.particles.coords, h, g)
    layouts, states = [], []
    for forced in (None, "general"):
        if forced:
            monkeypatch.setenv("PD_FAST_LAYOUT", forced)
        else:
            monkeypatch.delenv("PD_FAST_LAYOUT", raising=False)
        ctx = engine.Context(0)
        st = make_state(fam, False)
        st.u = S.seed_displacements(b.particles.coords) * 3.0
        ctx.upload(b, st, KernelVariant.fast)
        layouts.append(ctx.layout())
        ctx.run(20, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.fast)
        if not forced:
            assert ctx.kernel() == LAT_KERNELS[lat_cfg], ctx.kernel()
        ctx.download(st)
        ctx.close()
        states.append(st)
    assert layouts == ["lattice", "tiles"]
    ref = make_state(fam, False)
    ref.u = S.seed_displacements(b.particles.coords) * 3.0
    oracle.simulate(b, ref, SimulateOptions(20, 0, 0, IntegratorKind.velocity_verlet))
    s = stretches(b.particles, fam, ref.u)
    for st in states:
        check_break_sets(ref.connectivity.entries, st.connectivity.entries, s, 1.5e-5)
        assert max_rel_difference(ref.u, st.u) <= FRACTURE_U_TOL
    assert fam.n_neigh.sum() > ref.connectivity.n_neigh.sum()


def test_lattice_layout_selection():
    """Lattices run the implicit layout, also with no-failure nodes, per-node
    volumes and per-bond data (bond types, n-linear history: the NL kernel);
    irregular points take the tile layout."""
    b, h, g = S.bench_lattice_bundle((12, 12, 12))
    fam = geometry.build_family(b.particles.coords, h, g)

    def layout_of(bundle, family):
        ctx = engine.Context(0)
        ctx.upload(bundle, make_state(family, bundle.model.needs_history()), KernelVariant.fast)
        lay = ctx.layout()
        ctx.close()
        return lay
    assert layout_of(b, fam) == "lattice"
    b.bc.no_failure[5] = 1
    b.particles.volume[7] = 1.3
    assert layout_of(b, fam) == "lattice"
    fam2 = fam.copy()
    fam2.bond_type = np.zeros(fam.entries.size, np.uint8)
    assert layout_of(b, fam2) == "lattice"
    b2, h2, g2 = S.bench_lattice_bundle((12, 12, 12))
    b2.particles.coords = b2.particles.coords + np.random.default_rng(0).uniform(
        -0.01, 0.01, b2.particles.coords.size)
    fam3 = geometry.build_family(b2.particles.coords, h2)
    assert layout_of(b2, fam3) == "tiles"


def test_lattice_nl_kernel_matches_tiles_and_oracle(oracle, monkeypatch):
    """Several laws by bond type on the lattice (trilinear concrete, PMB steel,
    bilinear interface, beta, history): the typed unrolled kernel and the loop
    kernel against the tile kernel and the fp64 oracle."""
    b, h, g = S.multimaterial_bundle((16, 8, 10))
    fam = geometry.build_family(b.particles.coords, h, g)
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    b.corrections.beta = np.random.default_rng(2).uniform(0.7, 1.0, fam.entries.size)
    outs = {}
    # the typed unrolled lattice kernel, the lattice loop kernel, the tile kernel
    for name, env in (("typed", {}), ("loop", {"PD_LAT_NL_LOOP": "1"}),
                      ("tiles", {"PD_FAST_LAYOUT": "general"})):
        for k in ("PD_LAT_NL_LOOP", "PD_FAST_LAYOUT"):
            if k in env:
                monkeypatch.setenv(k, env[k])
            else:
                monkeypatch.delenv(k, raising=False)
        ctx = engine.Context(0)
        st = make_state(fam, True)
        ctx.upload(b, st, KernelVariant.fast)
        assert ctx.layout() == ("tiles" if name == "tiles" else "lattice")
        ctx.run(150, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.fast)
        ctx.download(st)
        ctx.close()
        outs[name] = st
    ref = make_state(fam, True)
    oracle.simulate(b, ref, SimulateOptions(150, 0, 0, IntegratorKind.velocity_verlet))
    s = stretches(b.particles, fam, ref.u)
    s_c = max(l.breakpoints[-1] for l in b.model.laws)
    for st in outs.values():
        assert max_rel_difference(ref.u, st.u) <= FRACTURE_U_TOL
        diff = ref.connectivity.entries != st.connectivity.entries
        assert diff.sum() <= max(4, 0.01 * (fam.n_neigh.sum() - ref.connectivity.n_neigh.sum()))
        live = ref.connectivity.entries >= 0
        rel = np.abs(ref.bond_history[live] - st.bond_history[live])
        assert np.max(rel) <= 1e-4 * max(s_c, np.max(np.abs(ref.bond_history)))
    assert fam.n_neigh.sum() > ref.connectivity.n_neigh.sum()  # it fractured


@pytest.mark.parametrize("lat_cfg", ["0", "5", "6"])
@pytest.mark.parametrize("integrator", [IntegratorKind.euler, IntegratorKind.velocity_verlet])
def test_lattice_no_failure_and_volumes_match_oracle(oracle, integrator, monkeypatch, lat_cfg):
    """cfg1-style run on the lattice layout: the 3-point-bend beam (no-failure
    supports and load patch, PMB, quintic ramp) with per-node volumes, against
    the fp64 oracle, on the persistent small-model launch (0), the one-step
    small-brick kernel (5) and the 16x4x4-brick kernel (6) (with no-failure
    nodes and BCs: 16x4x4 bricks at 5 CTAs/SM)."""
    monkeypatch.setenv("PD_LAT_CFG", lat_cfg)
    b, h, g = S.beam_bundle(30, 10, 10)
    rng = np.random.default_rng(11)
    b.particles.volume = b.particles.volume * rng.uniform(0.8, 1.2, b.particles.volume.size)
    b.bc.ramps[1].rise_steps = 150
    b.bc.magnitude[:] = b.bc.magnitude * 3.0  # drive it to fracture
    fam = geometry.build_family(b.particles.coords, h, g)
    outs = []
    for be, variant in ((engine.backend(), KernelVariant.fast),
                        (oracle, KernelVariant.bond_parallel)):
        st = make_state(fam, False)
        be.simulate(b, st, SimulateOptions(200, 0, 0, integrator, variant))
        outs.append(st)
    fast, ref = outs
    ctx = engine.Context(0)
    ctx.upload(b, make_state(fam, False), KernelVariant.fast)
    assert ctx.layout() == "lattice"
    ctx.close()
    # a propagating dynamic crack: K-step broken sets agree to 1 % of the
    # broken bonds, u within the fracture-run tolerance (module docstring)
    broken = fam.n_neigh.sum() - ref.connectivity.n_neigh.sum()
    assert broken > 0  # it fractured
    diff = int((ref.connectivity.entries != fast.connectivity.entries).sum())
    assert diff <= max(4, 0.01 * broken), (diff, broken)
    assert max_rel_difference(ref.u, fast.u) <= FRACTURE_U_TOL


@pytest.mark.parametrize("integrator", [IntegratorKind.euler, IntegratorKind.euler_cromer,
                                        IntegratorKind.velocity_verlet])
def test_lattice_persistent_launch_is_chunk_invariant(monkeypatch, integrator):
    """The persistent small-model launch (lattice_small_kernel) runs every
    step between two host events in one launch.  Cutting the run at write
    steps (hook every 7 steps, tips) or into several run calls must give the
    same bits: the per-step arithmetic does not depend on the chunking.  The
    one-step kernel (PD_LAT_PERSIST=0; its slot sums run in another order),
    16-wide bricks (PD_SMALL_BX=16; other fp32 staging references) and four
    slot parts per node instead of eight (PD_SMALL_P=4; another sum order)
    agree within the fast-path tolerance."""
    b, h, g = S.beam_bundle(30, 10, 10)
    b.bc.ramps[1].rise_steps = 150
    b.bc.magnitude[:] = b.bc.magnitude * 3.0  # drive it to fracture
    fam = geometry.build_family(b.particles.coords, h, g)
    outs = {}
    for name, persist, we, split in (("one", "1", 0, 1), ("hooked", "1", 7, 1), ("split", "1", 0, 3),
                                     ("step", "0", 0, 1), ("bx16", "1", 0, 1), ("p4", "1", 0, 1)):
        monkeypatch.setenv("PD_LAT_PERSIST", persist)
        monkeypatch.setenv("PD_SMALL_BX", "16" if name == "bx16" else "0")
        monkeypatch.setenv("PD_SMALL_P", "4" if name == "p4" else "0")
        ctx = engine.Context(0)
        st = make_state(fam, False)
        ctx.upload(b, st, KernelVariant.fast)
        done = 0
        for part in range(split):
            k = 200 // split if part + 1 < split else 200 - done
            ctx.run(k, done, integrator, we, KernelVariant.fast)
            done += k
        kern = ctx.kernel()
        ctx.download(st)
        ctx.close()
        assert kern.startswith("lattice_small_kernel" if persist == "1" else "lattice_step_kernel"), kern
        outs[name] = st
    ref = outs["one"]
    assert fam.n_neigh.sum() > ref.connectivity.n_neigh.sum()  # it fractured
    for name in ("hooked", "split"):
        for f in ("u", "v", "a"):
            assert np.array_equal(getattr(ref, f), getattr(outs[name], f)), (name, f)
        assert np.array_equal(ref.connectivity.entries, outs[name].connectivity.entries), name
    broken = fam.n_neigh.sum() - ref.connectivity.n_neigh.sum()
    for name in ("step", "bx16", "p4"):
        st = outs[name]
        diff = int((ref.connectivity.entries != st.connectivity.entries).sum())
        assert diff <= max(4, 0.01 * broken), (name, diff, broken)
        assert max_rel_difference(ref.u, st.u) <= FRACTURE_U_TOL, name


NLU_LAWS = {
    "bilinear": lambda: DamageLaw.bilinear(1.0, 1e-5, 4e-5),
    "trilinear_convex_kink": lambda: DamageLaw.trilinear(1.0, 5e-6, 1.5e-5, 4e-5, 0.25),
    "trilinear_concave": lambda: DamageLaw.trilinear(1.0, 1e-5, 2e-5, 3e-5, 0.9),
    "pmb": lambda: DamageLaw.pmb(1.0, 4e-5),
    # several laws by bond type (the typed kernel): bond types from a rebar line
    "typed": lambda: [DamageLaw.trilinear(1.0, 5e-6, 1.5e-5, 4e-5, 0.25),
                      DamageLaw.pmb(3.0, 6e-5),
                      DamageLaw.bilinear(2.0, 1e-5, 3e-5)],
}


@pytest.mark.parametrize("law", sorted(NLU_LAWS))
@pytest.mark.parametrize("extras", ["plain", "beta_nofail_bc"])
def test_lattice_unrolled_nl_kernel(oracle, monkeypatch, law, extras):
    """The unrolled NL lattice kernel (one law: history through the register
    ring, min/max envelope, recompute pass for breaking nodes) against the
    fp64 oracle and against the NL loop kernel (PD_LAT_NL_LOOP), with beta,
    no-failure nodes and a displacement BC in the second variant."""
    b, h, g = S.bench_lattice_bundle((20, 16, 12))
    laws = NLU_LAWS[law]()
    b.model.laws = laws if isinstance(laws, list) else [laws]
    n = b.particles.size()
    fam = geometry.build_family(b.particles.coords, h, g)
    if law == "typed":
        fam.bond_type = S.classify_bonds(b.particles.coords, fam, rebar_y=8.0, rebar_z=6.0)
    if extras != "plain":
        b.corrections.beta = np.random.default_rng(5).uniform(0.6, 1.0, fam.entries.size)
        z = b.particles.coords[2::3]
        b.bc.no_failure[z == 0] = 1
        for i in np.flatnonzero(z == 11):
            b.bc.kind[3 * i + 2] = BCKind.displacement
            b.bc.magnitude[3 * i + 2] = 2e-4
    hist = b.model.needs_history()
    u0 = S.seed_displacements(b.particles.coords) * 3.0
    steps = 120
    outs = {}
    for mode in ("unrolled", "loop"):
        if mode == "loop":
            monkeypatch.setenv("PD_LAT_NL_LOOP", "1")
        else:
            monkeypatch.delenv("PD_LAT_NL_LOOP", raising=False)
        ctx = engine.Context(0)
        st = make_state(fam, hist)
        st.u = u0.copy()
        ctx.upload(b, st, KernelVariant.fast)
        assert ctx.layout() == "lattice"
        ctx.run(steps, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.fast)
        ctx.download(st)
        ctx.close()
        outs[mode] = st
    ref = make_state(fam, hist)
    ref.u = u0.copy()
    oracle.simulate(b, ref, SimulateOptions(steps, 0, 0, IntegratorKind.velocity_verlet))
    broken = int(fam.n_neigh.sum() - ref.connectivity.n_neigh.sum())
    assert broken > 0  # the laws above break bonds at this amplitude
    s_c = max(lw.breakpoints[-1] for lw in b.model.laws)
    for mode, st in outs.items():
        assert max_rel_difference(ref.u, st.u) <= FRACTURE_U_TOL, mode
        diff = int((ref.connectivity.entries != st.connectivity.entries).sum())
        assert diff <= max(4, 0.01 * broken), (mode, diff, broken)
        assert np.array_equal(st.connectivity.n_neigh,
                              (st.connectivity.entries.reshape(n, -1) >= 0).sum(1))
        if hist:
            live = (ref.connectivity.entries >= 0) & (st.connectivity.entries >= 0)
            err = np.abs(ref.bond_history[live] - st.bond_history[live])
            assert np.max(err) <= 1e-4 * max(s_c, np.max(np.abs(ref.bond_history))), mode


@pytest.mark.parametrize("layout", [None, "general"])
@pytest.mark.parametrize("law", ["pmb", "trilinear"])
def test_fast_nonfinite_raises_like_the_reference(oracle, monkeypatch, layout, law):
    """A non-finite displacement stops the fast variant with the reference's
    error (check_state_finite, engine.cpp:23-28): same exception, same step,
    on the lattice kernels and on the tile kernel."""
    from paper_2105_04150_b200 import abi
    if layout:
        monkeypatch.setenv("PD_FAST_LAYOUT", layout)
    else:
        monkeypatch.delenv("PD_FAST_LAYOUT", raising=False)
    b, h, g = S.bench_lattice_bundle((16, 12, 10))
    if law == "trilinear":
        b.model.laws = [DamageLaw.trilinear(1.0, 1e-3, 2e-3, 1e6)]
    fam = geometry.build_family(b.particles.coords, h, g)
    msgs = []
    for be, variant in ((oracle, KernelVariant.bond_parallel), (engine.backend(), KernelVariant.fast)):
        st = make_state(fam, b.model.needs_history())
        st.u = S.seed_displacements(b.particles.coords)
        st.u[3 * 77 + 1] = np.nan
        with pytest.raises(abi.PeridynRuntimeError) as ei:
            be.simulate(b, st, SimulateOptions(20, 0, 5, IntegratorKind.velocity_verlet, variant))
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]


@pytest.mark.parametrize("layout", [None, "general"])
def test_fast_nonfinite_midrun_raises_like_the_reference(oracle, monkeypatch, layout):
    """A blow-up mid-run (an enormous force BC, as test_gpu_parity's exact-path
    case) stops the fast variant at the reference's step with its message."""
    from paper_2105_04150_b200 import abi
    if layout:
        monkeypatch.setenv("PD_FAST_LAYOUT", layout)
    else:
        monkeypatch.delenv("PD_FAST_LAYOUT", raising=False)
    b, h, g = S.bench_lattice_bundle((16, 12, 10), s_c=1e9)
    b.dt = 0.05  # the reference overflows u at step 25
    b.bc.kind[3 * 300] = BCKind.force
    b.bc.magnitude[3 * 300] = 1.5e308
    fam = geometry.build_family(b.particles.coords, h, g)
    msgs = []
    for be, variant in ((oracle, KernelVariant.bond_parallel), (engine.backend(), KernelVariant.fast)):
        st = make_state(fam, False)
        with pytest.raises(abi.PeridynRuntimeError) as ei:
            be.simulate(b, st, SimulateOptions(200, 0, 0, IntegratorKind.velocity_verlet, variant))
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]


@pytest.mark.parametrize("nl_bz", ["4", "8"])
@pytest.mark.parametrize("law", ["trilinear_convex_kink", "typed"])
def test_lattice_nl_brick_depths_match_oracle(oracle, monkeypatch, nl_bz, law):
    """The n-linear lattice kernels on either per-bond layout depth (16x4x4 or
    16x4x8 bricks, PD_NL_BZ) against the fp64 oracle, with beta."""
    monkeypatch.setenv("PD_NL_BZ", nl_bz)
    b, h, g = S.bench_lattice_bundle((20, 16, 12))
    laws = NLU_LAWS[law]()
    b.model.laws = laws if isinstance(laws, list) else [laws]
    fam = geometry.build_family(b.particles.coords, h, g)
    if law == "typed":
        fam.bond_type = S.classify_bonds(b.particles.coords, fam, rebar_y=8.0, rebar_z=6.0)
    b.corrections.beta = np.random.default_rng(9).uniform(0.6, 1.0, fam.entries.size)
    u0 = S.seed_displacements(b.particles.coords) * 3.0
    outs = []
    for be, variant in ((engine.backend(), KernelVariant.fast),
                        (oracle, KernelVariant.bond_parallel)):
        st = make_state(fam, True)
        st.u = u0.copy()
        be.simulate(b, st, SimulateOptions(120, 0, 0, IntegratorKind.velocity_verlet, variant))
        outs.append(st)
    fast, ref = outs
    broken = int(fam.n_neigh.sum() - ref.connectivity.n_neigh.sum())
    assert broken > 0
    diff = int((ref.connectivity.entries != fast.connectivity.entries).sum())
    assert diff <= max(4, 0.01 * broken), (diff, broken)
    assert max_rel_difference(ref.u, fast.u) <= FRACTURE_U_TOL
    live = (ref.connectivity.entries >= 0) & (fast.connectivity.entries >= 0)
    s_c = max(lw.breakpoints[-1] for lw in b.model.laws)
    err = np.abs(ref.bond_history[live] - fast.bond_history[live])
    assert np.max(err) <= 1e-4 * max(s_c, np.max(np.abs(ref.bond_history)))
