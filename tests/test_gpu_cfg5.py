"""cfg5, the reinforced-concrete beam, downscaled so the CPU
oracle finishes: a rule-table classifier gives concrete / steel / interface
bond types on the device, surface-correction factors come from the device
(both bitwise against the reference in test_gpu_family_ops.py), and the run
uses three laws (trilinear concrete, linear steel, bilinear interface) with
fp64 history, no-failure supports and quintic displacement loading.

  * the exact variant is bitwise equal to the C oracle over a K-step run;
  * the fast variant (typed lattice kernel) matches the exact path for one
    pass from identical strained states: forces within FORCE_TOL, broken sets
    identical except bonds within EPS_S of their law's critical stretch.
The full ~31M-node beam is timed by scripts/bench_cfg5.py."""
import numpy as np
import pytest

import scenarios as S
from paper_2105_04150_b200 import engine, geometry
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, SimulateOptions, make_state
from test_gpu_bench_parity import EPS_S, FORCE_TOL, max_rel_difference, slot_stretch, step_once

pytestmark = pytest.mark.gpu


def beam(dx_mm):
    b, g, delta, cls = S.rc_beam_setup(dx_mm)
    fam = geometry.build_family(b.particles.coords, delta, g, classify=cls)
    vol = b.particles.volume
    b.corrections.lambda_ = geometry.surface_correction_factors(
        vol, fam, geometry.max_neighborhood_volume(vol, fam))
    return b, fam


def test_cfg5_downscale_exact_matches_oracle(oracle):
    b, fam = beam(12.0)  # 176 x 27 x 16 = 76k nodes
    types = np.unique(fam.bond_type[fam.entries >= 0])
    assert set(types.tolist()) == {0, 1, 2}
    lam = b.corrections.lambda_[fam.entries >= 0]
    # V0 = the largest neighbourhood volume: 1 in the bulk, > 1 near surfaces
    assert lam.min() == 1.0 and lam.max() > 1.5
    # strained start: the seeded field scaled so bonds sit on every segment
    u0 = S.seed_displacements(b.particles.coords / 12e-3) * 12e-3 * 300.0
    outs = []
    for be in (oracle, engine.backend()):
        st = make_state(fam, True)
        st.u = u0.copy()
        be.simulate(b, st, SimulateOptions(25, 0, 0, IntegratorKind.velocity_verlet,
                                           KernelVariant.bond_parallel))
        outs.append(st)
    a, g = outs
    for f in ("u", "v", "a", "bond_history"):
        assert np.array_equal(getattr(a, f).view(np.uint64), getattr(g, f).view(np.uint64)), f
    assert np.array_equal(a.connectivity.entries, g.connectivity.entries)
    assert np.array_equal(a.connectivity.n_neigh, g.connectivity.n_neigh)
    assert int(fam.n_neigh.sum() - g.connectivity.n_neigh.sum()) > 0  # bonds broke


def test_cfg5_downscale_fast_one_pass_matches_exact():
    b, fam = beam(8.0)  # 263 x 40 x 24 = 252k nodes
    N = int(fam.group_size)
    st0 = make_state(fam, True)
    st0.u = S.seed_displacements(b.particles.coords / 8e-3) * 8e-3 * 300.0
    vv = IntegratorKind.velocity_verlet
    # a few exact steps first: history and breaks are populated
    ctx = engine.Context(0)
    ctx.upload(b, st0, KernelVariant.bond_parallel)
    ctx.run(5, 0, vv, 0, KernelVariant.bond_parallel)
    ctx.download(st0)
    ctx.close()
    st0.step = 5
    fast, kernel = step_once(b, st0, KernelVariant.fast, vv)
    assert kernel.startswith("lattice_nl"), kernel
    ref, _ = step_once(b, st0, KernelVariant.bond_parallel, vv)
    e_r, e_f = ref.connectivity.entries, fast.connectivity.entries
    diff = np.flatnonzero(e_r != e_f)
    if diff.size:
        orig = np.where(e_r[diff] >= 0, e_r[diff], e_f[diff])
        ent = np.zeros_like(e_r)
        ent[diff] = orig
        # velocity-Verlet: the force pass of the step sees the drifted u (= ref.u)
        s = slot_stretch(b.particles.coords, ref.u, N, diff, ent)
        s = np.maximum(s, st0.bond_history[diff])
        s_c = np.array([law.breakpoints[-1] for law in b.model.laws])[fam.bond_type[diff]]
        far = np.abs(s - s_c) > EPS_S * s_c
        assert not far.any(), int(far.sum())
    n = fam.node_count()
    ok = np.ones(n, bool)
    ok[np.unique(diff // N)] = False
    err = max_rel_difference(ref.a.reshape(n, 3)[ok], fast.a.reshape(n, 3)[ok])
    assert err <= FORCE_TOL, err
    broke = int(st0.connectivity.n_neigh.sum() - ref.connectivity.n_neigh.sum())
    assert broke > 0
