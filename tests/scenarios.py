"""Scenario builders shared by the golden generator and the tests.

Each builder restates a fixture of the reference's own test suite or a
BASELINE.json config with the reference's API (types.py mirrors it), so the
same bundle drives the compiled reference, the C oracle and the GPU.
Families are passed in by the caller (built by the oracle or the reference).
"""
from __future__ import annotations

import math

import numpy as np

from paper_2105_04150_b200.geometry import GridDesc, grid_coordinates
from paper_2105_04150_b200.types import (BCKind, BoundaryConditions, Corrections, DamageLaw,
                                         DamageModel, ModelBundle, ParticleSet, RampKind,
                                         RampProfile)


def lattice_particles(counts, spacing=1.0, volume=None, density=1.0):
    g = GridDesc((0.0, 0.0, 0.0), spacing, counts)
    coords = grid_coordinates(g)
    n = g.node_count()
    vol = spacing ** 3 if volume is None else volume
    return g, ParticleSet(coords, np.full(n, vol), np.full(n, float(density)), np.zeros(n, np.uint16))


def small_fracture_bundle():
    """tests/test_engine.cpp:377-403 (horizon 1.8, no grid hint)."""
    g, p = lattice_particles((5, 4, 3))
    n = p.size()
    bc = BoundaryConditions.none(n)
    bc.ramps.append(RampProfile(RampKind.linear, 200, 1.0))
    x = p.coords[0::3]
    for i in range(n):
        if x[i] == 0 or x[i] == 4:
            bc.kind[3 * i] = BCKind.displacement
            bc.magnitude[3 * i] = -0.15 if x[i] == 0 else 0.15
            bc.ramp_id[3 * i] = 1
    bc.tip_sets["pull"] = [0, 1, 2]
    return ModelBundle(p, DamageModel([DamageLaw.pmb(0.05, 0.04)]), Corrections(), bc, 0.05), 1.8, None


def trilinear_bar_bundle():
    """tests/acceptance/main.cpp:368-392 (criterion 8)."""
    g, p = lattice_particles((8, 4, 4))
    n = p.size()
    bc = BoundaryConditions.none(n)
    bc.ramps.append(RampProfile(RampKind.quintic_smooth, 120, 1.0))
    x = p.coords[0::3]
    for i in range(n):
        if x[i] == 7:
            bc.kind[3 * i] = BCKind.displacement
            bc.magnitude[3 * i] = 0.4
            bc.ramp_id[3 * i] = 1
        elif x[i] == 0:
            bc.kind[3 * i] = BCKind.displacement
    model = DamageModel([DamageLaw.trilinear(0.05, 0.02, 0.05, 0.2)])
    return ModelBundle(p, model, Corrections(), bc, 0.05), 1.8, None


def notched_plate_bundle(nx=40, ny=40, nz=4, integrator_steps=200, pull=None):
    """cfg2 (downscaled): pre-cracked plate, Mode I, bilinear law, Euler-Cromer.
    Edge notch at y = ny/2 - 0.5 from x = 0 to x = nx/4; opposite y faces pulled
    apart on a linear ramp; a force patch and a no-failure strip exercise the
    remaining BC kinds.  Notch applied by the caller (break_initial_bonds).
    The pull scales with the plate (0.015 ny per face: a 3 % far-field strain
    at the end of the ramp, above s0 = 2.3 %), so the notch propagates at any
    size (0.6 at ny = 40)."""
    if pull is None:
        pull = 0.015 * ny
    g, p = lattice_particles((nx, ny, nz))
    n = p.size()
    delta = math.pi
    E, G0 = 1.0, 2e-3
    c = 18.0 * (E / 1.5) / (math.pi * delta ** 4)
    s0 = math.sqrt(5.0 * G0 / (6.0 * E * delta))
    model = DamageModel([DamageLaw.bilinear(c, s0, 5.0 * s0)])
    bc = BoundaryConditions.none(n)
    bc.ramps.append(RampProfile(RampKind.linear, integrator_steps, 1.0))
    y = p.coords[1::3]
    x = p.coords[0::3]
    for i in range(n):
        if y[i] == 0:
            bc.kind[3 * i + 1] = BCKind.displacement
            bc.magnitude[3 * i + 1] = -pull
            bc.ramp_id[3 * i + 1] = 1
        elif y[i] == ny - 1:
            bc.kind[3 * i + 1] = BCKind.displacement
            bc.magnitude[3 * i + 1] = pull
            bc.ramp_id[3 * i + 1] = 1
        if x[i] == nx - 1 and y[i] < 3:
            bc.kind[3 * i] = BCKind.force
            bc.magnitude[3 * i] = 1e-4
        if y[i] == 0 or y[i] == ny - 1:
            bc.no_failure[i] = 1
    bc.tip_sets["top"] = [int(i) for i in np.flatnonzero(y == ny - 1)[:16]]
    bc.tip_sets["mouth"] = [int(i) for i in np.flatnonzero((x == 0) & (np.abs(y - (ny / 2 - 0.5)) < 1))]
    notch = dict(axis=1, position=ny / 2 - 0.5, sweep_axis=0, depth=nx / 4)
    return ModelBundle(p, model, Corrections(), bc, 0.3), delta, g, notch


def beam_bundle(nx=50, ny=14, nz=14):
    """cfg1: 3-point-bend plain concrete beam, PMB, Euler.
    175 x 50 x 50 mm at dx = 3.5 mm; supports are zero-displacement no-failure
    patches, the load a central displacement patch on a quintic ramp."""
    dx = 3.5e-3
    g, p = lattice_particles((nx, ny, nz), spacing=dx, density=2346.0)
    n = p.size()
    delta = math.pi * dx
    E, GF = 37.0e9, 143.2
    c = 18.0 * (E / 1.5) / (math.pi * delta ** 4)
    s_c = math.sqrt(5.0 * GF / (6.0 * E * delta))
    model = DamageModel([DamageLaw.pmb(c, s_c)])
    bc = BoundaryConditions.none(n)
    bc.ramps.append(RampProfile(RampKind.quintic_smooth, 1000, 1.0))
    x = p.coords[0::3] / dx
    y = p.coords[1::3] / dx
    for i in range(n):
        if y[i] == 0 and (abs(x[i] - 7) <= 1 or abs(x[i] - (nx - 8)) <= 1):
            for ax in range(3):
                bc.kind[3 * i + ax] = BCKind.displacement
            bc.no_failure[i] = 1
        if y[i] == ny - 1 and abs(x[i] - (nx - 1) / 2) <= 1:
            bc.kind[3 * i + 1] = BCKind.displacement
            bc.magnitude[3 * i + 1] = -1e-4
            bc.ramp_id[3 * i + 1] = 1
            bc.no_failure[i] = 1
    bc.tip_sets["load"] = [int(i) for i in np.flatnonzero((y == ny - 1) & (np.abs(x - (nx - 1) / 2) <= 1))]
    dt = 1.0e-7
    return ModelBundle(p, model, Corrections(), bc, dt), delta, g


def multimaterial_bundle(counts=(12, 8, 8)):
    """cfg5 (downscaled): multi-bond-type trilinear with a stiff linear class
    (rebar) and an interface class, plus surface-correction factors."""
    g, p = lattice_particles(counts)
    n = p.size()
    laws = [DamageLaw.trilinear(1.0, 0.01, 0.02, 0.05),       # concrete-concrete
            DamageLaw.pmb(7.0, 0.5),                           # steel-steel
            DamageLaw.bilinear(3.0, 0.01, 0.03)]               # interface
    model = DamageModel(laws, damping=0.05)
    bc = BoundaryConditions.none(n)
    bc.ramps.append(RampProfile(RampKind.quintic_smooth, 150, 1.0))
    x = p.coords[0::3]
    for i in range(n):
        if x[i] == 0:
            for ax in range(3):
                bc.kind[3 * i + ax] = BCKind.displacement
        elif x[i] == counts[0] - 1:
            bc.kind[3 * i] = BCKind.displacement
            bc.magnitude[3 * i] = 0.6
            bc.ramp_id[3 * i] = 1
    bc.tip_sets["end"] = [int(i) for i in np.flatnonzero(x == counts[0] - 1)]
    return ModelBundle(p, model, Corrections(), bc, 0.05), 2.2, g


def classify_bonds(coords, family, rebar_y=2.0, rebar_z=2.0):
    """bond_type per slot: 1 if both ends lie on the rebar line, 2 if one does."""
    n = family.node_count()
    N = int(family.group_size)
    xyz = np.asarray(coords).reshape(n, 3)
    on = (np.abs(xyz[:, 1] - rebar_y) < 0.5) & (np.abs(xyz[:, 2] - rebar_z) < 0.5)
    ent = family.entries.reshape(n, N)
    bt = np.zeros((n, N), np.uint8)
    live = ent >= 0
    jj = np.where(live, ent, 0)
    both = on[:, None] & on[jj]
    one = on[:, None] ^ on[jj]
    bt[live & both] = 1
    bt[live & one] = 2
    return bt.reshape(-1)


def bench_lattice_bundle(counts, s_c=1e6, horizon=3.0):
    """bench::benchmark_bundle (bench.cpp:76-93) + seed_displacements (:95-104)."""
    g, p = lattice_particles(counts)
    n = p.size()
    bundle = ModelBundle(p, DamageModel([DamageLaw.pmb(1.0, s_c)]), Corrections(),
                         BoundaryConditions.none(n), 1e-3)
    return bundle, horizon, g


def seed_displacements(coords):
    x = coords[0::3]
    y = coords[1::3]
    z = coords[2::3]
    u = np.empty_like(coords)
    u[0::3] = 1e-4 * np.sin(0.1 * x + 0.2 * y)
    u[1::3] = 1e-4 * np.cos(0.15 * y + 0.1 * z)
    u[2::3] = 1e-4 * np.sin(0.12 * z + 0.17 * x)
    return u


def oscillator(c=3.0, volume=0.8, density=1.3, length=1.0):
    """tests/oracles.hpp:233-264"""
    p = ParticleSet(np.array([0, 0, 0, length, 0, 0], dtype=np.float64), np.full(2, volume),
                    np.full(2, density), np.zeros(2, np.uint16))
    model = DamageModel([DamageLaw.pmb(c, 1e9)])
    omega = math.sqrt(2 * c * volume / (density * length))
    return p, model, length * 1.5, omega


def random_config_np(seed, n_range=(10, 500)):
    """A numpy analogue of oracles::make_random_config (oracles.hpp:140-210):
    same distributions (clustered points, horizon 0.3..3.5 box-side units, PMB
    or trilinear, optional lambda/beta, up to 50 % symmetric pre-breaks,
    u in +-0.01), different random stream.  Family built by the caller."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(n_range[0], n_range[1] + 1))
    side = n ** (1.0 / 3.0)
    coords = rng.uniform(0, side, 3 * n)
    volume = 0.5 + rng.uniform(0, 1, n)
    density = 0.5 + rng.uniform(0, 1, n)
    horizon = 0.3 + rng.uniform() * 3.2
    trilinear = rng.uniform() < 0.5
    s_c = 0.05 + 0.1 * rng.uniform()
    if trilinear:
        law = DamageLaw.trilinear(1.0, s_c / 4, s_c / 2, s_c, 0.25 + rng.uniform() / 2)
    else:
        law = DamageLaw.pmb(1.0, s_c)
    draws = dict(lam=rng.uniform() < 0.5, beta=rng.uniform() < 0.3,
                 broken_share=rng.uniform() * 0.5)
    p = ParticleSet(coords, volume, density, np.zeros(n, np.uint16))
    return p, DamageModel([law]), horizon, draws, rng


def finish_random_config(p, model, family, draws, rng):
    """Corrections, symmetric pre-breaks and displacements for random_config_np."""
    from paper_2105_04150_b200.types import make_state
    n = p.size()
    N = int(family.group_size)
    corr = Corrections()
    if draws["lam"]:
        corr.lambda_ = 0.5 + rng.uniform(0, 1, n * N)
    if draws["beta"]:
        corr.beta = 0.5 + rng.uniform(0, 1, n * N) / 2
    state = make_state(family, model.needs_history())
    ent = state.connectivity.entries.reshape(n, N)
    share = draws["broken_share"]
    for i in range(n):
        for k in range(N):
            j = ent[i, k]
            if j < 0 or j < i:
                continue
            if rng.uniform() < share:
                ent[i, k] = -1
                state.connectivity.n_neigh[i] -= 1
                back = np.flatnonzero(ent[j] == i)
                if back.size:
                    ent[j, back[0]] = -1
                    state.connectivity.n_neigh[j] -= 1
    state.u = (rng.uniform(0, 1, 3 * n) - 0.5) * 0.02
    return corr, state


def rc_beam_setup(dx_mm=1.6, length_mm=2100.0, height_mm=320.0, width_mm=190.0):
    """cfg5: the reinforced-concrete beam of PAPER.md:580-597 (Stuttgart shear
    test beam 5): 320 x 190 mm section, 1950 mm span between supports (75 mm
    overhang each end), two 26 mm bars at 270 mm effective depth, four-point
    loading with a shear span of 810 mm.  dx = 1.6 mm gives 1313 x 200 x 119
    = 31.2M nodes (the paper's dx = 5 mm mesh scaled by (5/1.6)^3).
    Materials: concrete E_c = 30.5 GPa, rho 2346,
    trilinear s0/s1/s_c = 1.05e-4 / 6.9e-4 / 5.56e-3 (the Yang 2018 column);
    steel E_s = 208 GPa, rho 7850, linear (never breaks); a bilinear
    steel-concrete interface.  delta = pi dx; c = 18 K / (pi delta^4) with
    K = E / 1.5 (nu = 1/4).  Supports: clamped (left) and roller (right)
    no-failure patches under the bottom face; loads: quintic-ramped downward
    displacement patches on the top face.  Returns (bundle, grid, horizon,
    classifier); the caller builds the family, classifies the bonds and
    computes the surface correction (geometry.build_family / classify /
    surface_correction_factors)."""
    from paper_2105_04150_b200.geometry import Region, RuleClassifier
    dx = dx_mm * 1e-3
    counts = (int(round(length_mm / dx_mm)) + 1, int(round(height_mm / dx_mm)),
              int(round(width_mm / dx_mm)))
    g = GridDesc((0.0, 0.0, 0.0), dx, counts)
    coords = grid_coordinates(g)
    n = g.node_count()
    x, y, z = coords[0::3], coords[1::3], coords[2::3]
    delta = math.pi * dx
    E_c, E_s = 30.5e9, 208.0e9
    c_c = 18.0 * (E_c / 1.5) / (math.pi * delta ** 4)
    c_s = 18.0 * (E_s / 1.5) / (math.pi * delta ** 4)
    c_i = 0.5 * (c_c + c_s)
    laws = [DamageLaw.trilinear(c_c, 1.05e-4, 6.9e-4, 5.56e-3),   # concrete-concrete
            DamageLaw.pmb(c_s, 1.0),                              # steel-steel (linear)
            DamageLaw.bilinear(c_i, 2.0e-4, 1.75e-3)]             # steel-concrete interface
    model = DamageModel(laws, damping=0.0)
    # two bars, 26 mm diameter, centres 50 mm above the bottom face (effective
    # depth 270 mm) and 45 mm in from each side
    yb = (height_mm - 270.0) * 1e-3
    bars = [Region(cls=1, kind="cylinder", axis=0, center=(yb, zc), radius=13e-3)
            for zc in (45e-3, (width_mm - 45.0) * 1e-3)]
    classifier = RuleClassifier(np.array([[0, 2], [2, 1]], dtype=np.uint8), bars)
    on_bar = classifier.node_classes(coords) == 1
    density = np.where(on_bar, 7850.0, 2346.0)
    particles = ParticleSet(coords, np.full(n, dx ** 3), density, np.zeros(n, np.uint16))
    bc = BoundaryConditions.none(n)
    bc.ramps.append(RampProfile(RampKind.quintic_smooth, 200000, 1.0))
    top, bottom = y >= y.max() - 0.5 * dx, y <= 0.5 * dx
    span0, span1 = 75e-3, 75e-3 + 1950e-3
    near = lambda x0: np.abs(x - x0) <= 10e-3  # noqa: E731  (20 mm wide patches)
    left, right = bottom & near(span0), bottom & near(span1)
    load = top & (near(span0 + 810e-3) | near(span1 - 810e-3))
    for ax in range(3):
        bc.kind[3 * np.flatnonzero(left) + ax] = BCKind.displacement      # clamped
    for ax in (1, 2):
        bc.kind[3 * np.flatnonzero(right) + ax] = BCKind.displacement     # roller
    li = 3 * np.flatnonzero(load) + 1
    bc.kind[li] = BCKind.displacement
    bc.magnitude[li] = -2e-3
    bc.ramp_id[li] = 1
    bc.no_failure[left | right | load] = 1
    mid = top & (np.abs(x - 0.5 * (span0 + span1)) <= 0.6 * dx)
    bc.tip_sets["midspan"] = [int(i) for i in np.flatnonzero(mid)]
    bc.tip_sets["load"] = [int(i) for i in np.flatnonzero(load)]
    dt = 2.0e-8
    return ModelBundle(particles, model, Corrections(), bc, dt), g, delta, classifier
