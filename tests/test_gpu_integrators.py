"""The reference's stand-alone integrators and boundary passes on the device
(pd_verlet_drift / pd_verlet_kick / pd_step_euler / pd_step_euler_cromer /
pd_step_velocity_verlet / pd_apply_boundary ..., engine.hpp:38-78): the
hand-composed flows of test_engine.cpp:196-357, bitwise against the C
oracle at every step, plus the reference's own expectations and errors."""
import ctypes as C
import math

import numpy as np
import pytest

import scenarios as S
from paper_2105_04150_b200 import abi, engine, geometry
from paper_2105_04150_b200.types import (BCKind, BoundaryConditions, Corrections, DamageLaw,
                                         DamageModel, ForceField, KernelVariant, ParticleSet,
                                         RampKind, RampProfile, make_state)

pytestmark = pytest.mark.gpu


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))


def two_node(c=2.0, v1=1.0, v2=1.0, stretch=0.0):
    """TwoNode::make (test_engine.cpp:46-63)."""
    p = ParticleSet(np.array([0, 0, 0, 1, 0, 0], np.float64), np.array([v1, v2]),
                    np.ones(2), np.zeros(2, np.uint16))
    model = DamageModel([DamageLaw.pmb(c, 0.5)])
    fam = geometry.build_family(p.coords, 1.5)
    st = make_state(fam, False)
    st.u[3] = stretch
    return p, model, st


def copy_state(st):
    from paper_2105_04150_b200.types import SimulationState
    return SimulationState(st.u.copy(), st.v.copy(), st.a.copy(), st.step,
                           st.connectivity.copy(), None)


def forces(n):
    f = ForceField()
    f.resize(n)
    return f


def test_force_free_drift_matches_oracle(oracle):
    """test_engine.cpp:196-209"""
    gpu = engine.backend()
    p, model, st = two_node()
    st.v[:] = [0.5, 0, 0, 0.5, 0, 0]
    ref = copy_state(st)
    f = forces(2)
    for _ in range(10):
        for be, s in ((gpu, st), (oracle, ref)):
            be.verlet_drift(s, 0.1)
            be.verlet_kick(s, f, 0.1, 0.0, p.density)
        assert same(st.u, ref.u) and same(st.v, ref.v) and same(st.a, ref.a)
    assert st.u[0] == pytest.approx(0.5, rel=1e-12)
    assert st.v[0] == pytest.approx(0.5, rel=1e-12)


def test_velocity_verlet_oscillator_matches_oracle(oracle):
    """test_engine.cpp:211-240: step_velocity_verlet with a ForceEval, both
    backends composing the same calls; the device's forces come from
    pd_compute_forces."""
    p, model, length, omega = S.oscillator(3.0, 0.8, 1.3, 1.0)
    fam = geometry.build_family(p.coords, length)
    st = make_state(fam, False)
    st.u[0], st.u[3] = -5e-4, 5e-4
    gpu = engine.backend()
    f = forces(2)
    gpu.compute_forces(KernelVariant.bond_parallel, st, p, model, Corrections(), f)
    st.a[:] = f.body_force / np.repeat(p.density, 3)
    ref = copy_state(st)
    dt = 2 * math.pi / omega / 100
    fr = forces(2)
    for k in range(300):
        gpu.step_velocity_verlet(
            st, lambda s, out: gpu.compute_forces(KernelVariant.bond_parallel, s, p, model,
                                                  Corrections(), out), f, dt, 0.0, p.density)
        oracle.step_velocity_verlet(
            ref, lambda s, out: oracle.compute_forces(KernelVariant.bond_parallel, s, p, model,
                                                      Corrections(), out), fr, dt, 0.0,
            p.density)
        assert same(st.u, ref.u) and same(st.v, ref.v) and same(st.a, ref.a), k
    assert st.step == 300


def test_step_velocity_verlet_c_entry_point(oracle):
    """pd_step_velocity_verlet with a C callback (ForceEval) equals the
    composed steps."""
    p, model, length, omega = S.oscillator(3.0, 0.8, 1.3, 1.0)
    fam = geometry.build_family(p.coords, length)
    st = make_state(fam, False)
    st.u[0], st.u[3] = -5e-4, 5e-4
    ref = copy_state(st)
    gpu = engine.backend()
    lib = engine.library()
    EVAL = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(abi.pd_state), C.POINTER(abi.pd_force_field))
    m = abi.Marshal()
    pp, md, cr = m.particles(p), m.model(model), m.corrections(Corrections())

    def cb(user, s, ff):
        return lib.pd_compute_forces(0, s, C.byref(pp), C.byref(md), C.byref(cr), ff)
    lib.pd_compute_forces.argtypes = [C.c_int32, C.POINTER(abi.pd_state),
                                      C.POINTER(abi.pd_particles), C.POINTER(abi.pd_damage_model),
                                      C.POINTER(abi.pd_corrections),
                                      C.POINTER(abi.pd_force_field)]
    lib.pd_step_velocity_verlet.argtypes = [C.POINTER(abi.pd_state), EVAL, C.c_void_p,
                                            C.POINTER(abi.pd_force_field), C.c_double, C.c_double,
                                            C.POINTER(C.c_double), C.c_int64]
    f = forces(2)
    ms = abi.Marshal()
    sd, ff = ms.state(st), ms.forces(f)
    rho = abi.as_f64(p.density)
    fn = EVAL(cb)
    dt = 2 * math.pi / omega / 50
    fr = forces(2)
    for _ in range(20):
        abi.check(lib.pd_step_velocity_verlet(C.byref(sd), fn, None, C.byref(ff), dt, 0.0,
                                              abi.ptr(rho, C.c_double), 2), lib.pd_last_error)
        oracle.step_velocity_verlet(
            ref, lambda s, out: oracle.compute_forces(KernelVariant.bond_parallel, s, p, model,
                                                      Corrections(), out), fr, dt, 0.0,
            p.density)
    assert same(st.u, ref.u) and same(st.v, ref.v) and sd.step == 20 == ref.step


@pytest.mark.parametrize("cromer", [False, True])
def test_euler_energy_matches_oracle(oracle, cromer):
    """test_engine.cpp:242-276: forward Euler grows the energy, Euler-Cromer
    stays bounded; every step bitwise equal to the oracle."""
    p, model, length, omega = S.oscillator(3.0, 0.8, 1.3, 1.0)
    fam = geometry.build_family(p.coords, length)
    gpu = engine.backend()
    states = []
    for be in (gpu, oracle):
        st = make_state(fam, False)
        st.u[0], st.u[3] = -5e-4, 5e-4
        states.append((be, st, forces(2)))
    dt = 2 * math.pi / omega / 100

    def energy(st):
        r = st.u[3] - st.u[0]
        vol = p.volume[0]
        return p.density[0] * vol * (st.v[0] ** 2 + st.v[3] ** 2) / 2 + \
            model.laws[0].stiffness * vol * vol * r * r / (2 * length)
    energies = [energy(states[0][1])]
    for k in range(400):
        for be, st, f in states:
            be.compute_forces(KernelVariant.bond_parallel, st, p, model, Corrections(), f)
            (be.step_euler_cromer if cromer else be.step_euler)(st, f, dt, p.density)
        a, b = states[0][1], states[1][1]
        assert same(a.u, b.u) and same(a.v, b.v) and same(a.a, b.a), k
        if (k + 1) % 100 == 0:
            energies.append(energy(a))
    if cromer:
        assert all(e < 2 * energies[0] for e in energies)
    else:
        assert all(b > a for a, b in zip(energies, energies[1:]))


def test_one_euler_step_with_constant_force():
    """test_engine.cpp:278-288"""
    p, model, st = two_node()
    f = forces(2)
    f.external_force[0] = 3.0
    engine.backend().step_euler(st, f, 0.25, p.density)
    assert st.v[0] == 0.75
    assert st.u[0] == 0.0


def test_damped_terminal_velocity_matches_oracle(oracle):
    """test_engine.cpp:290-317 (the first 400 of its 2000 steps)."""
    p = ParticleSet(np.array([0, 0, 0, 10, 0, 0], np.float64), np.ones(2), np.full(2, 2.0),
                    np.zeros(2, np.uint16))
    fam = geometry.build_family(p.coords, 1.0)
    pair = []
    for be in (engine.backend(), oracle):
        st = make_state(fam, False)
        f = forces(2)
        f.external_force[0] = 8.0
        pair.append((be, st, f))
    prev = 0.0
    for _ in range(400):
        for be, st, f in pair:
            be.verlet_drift(st, 0.01)
            be.verlet_kick(st, f, 0.01, 4.0, p.density)
        a, b = pair[0][1], pair[1][1]
        assert same(a.u, b.u) and same(a.v, b.v)
        assert a.v[0] >= prev - 1e-12
        prev = a.v[0]
    assert 1.9 < a.v[0] < 2.0


def test_apply_boundary_matches_oracle(oracle):
    """test_engine.cpp:338-355 plus a quintic ramp and several steps."""
    outs = []
    for be in (engine.backend(), oracle):
        p, model, st = two_node()
        bc = BoundaryConditions.none(2)
        bc.ramps.append(RampProfile(RampKind.linear, 10, 1.0))
        bc.ramps.append(RampProfile(RampKind.quintic_smooth, 40, 2.0))
        bc.kind[0] = BCKind.displacement
        bc.magnitude[0] = 0.5
        bc.ramp_id[0] = 1
        bc.kind[4] = BCKind.force
        bc.magnitude[4] = 3.0
        bc.kind[5] = BCKind.displacement
        bc.magnitude[5] = -0.3
        bc.ramp_id[5] = 2
        f = forces(2)
        rec = []
        for step in (5, 17, 33, 60):
            be.apply_boundary(st, bc, step, 0.1, f)
            rec.append(np.concatenate([st.u, st.v, st.a, f.external_force]))
        outs.append(rec)
    for a, b in zip(*outs):
        assert same(a, b)
    u, v, ext = outs[0][0][:6], outs[0][0][6:12], outs[0][0][18:]
    assert u[0] == pytest.approx(0.25) and v[0] == pytest.approx(0.5) and ext[4] == 3.0


def test_integrator_errors_match_oracle(oracle):
    msgs = []
    for be in (engine.backend(), oracle):
        p, model, st = two_node()
        f = forces(2)
        got = []
        for call in (lambda: be.verlet_drift(st, 0.0),
                     lambda: be.step_euler(st, f, -1.0, p.density),
                     lambda: be.verlet_kick(st, f, 0.1, 0.0, np.ones(3)),
                     lambda: be.step_euler_cromer(st, f, 0.1, np.array([1.0, 0.0]))):
            with pytest.raises((abi.DomainError, abi.InvalidArgument)) as e:
                call()
            got.append((type(e.value).__name__, str(e.value)))
        bc = BoundaryConditions.none(3)  # wrong node count
        with pytest.raises(abi.InvalidArgument) as e:
            be.apply_boundary(st, bc, 0, 0.1, f)
        got.append(str(e.value))
        msgs.append(got)
    assert msgs[0] == msgs[1]
