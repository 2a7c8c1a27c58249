"""Setup passes over a family on the device (csrc/pd_family_ops.cu), bitwise
against the UNMODIFIED reference (oracle/_ref):

  * build_family with a BondClassifier (geometry.hpp:45-54, pack_rows
    geometry.cpp:131-161) -- here a rule table (regions -> node class ->
    type table), the reference given a lambda applying the same rules;
  * neighborhood_volumes / max_neighborhood_volume / surface_correction_factors
    (geometry.cpp:238-283), with the reference's domain errors;
  * break_initial_bonds with plane_crossing_predicate / notch_predicate
    (geometry.cpp:285-319).
The rule-table validation (symmetry, ranges) runs before any device work and
is covered on CPU."""
import numpy as np
import pytest

import scenarios as S
from paper_2105_04150_b200 import abi, geometry
from paper_2105_04150_b200.geometry import Region, RuleClassifier


def rc_beam_rules(nx, ny, nz, h=1.0):
    """cfg5-style classes: concrete 0, steel 1 (two rebar cylinders along x
    near the bottom, radius 1.2 h), a stiff support plate 2 (a box at one end);
    types: concrete-concrete 0, steel-steel 1, steel-concrete 2, plate-* 3."""
    y1, y2, z = 0.25 * (ny - 1) * h, 0.75 * (ny - 1) * h, 0.2 * (nz - 1) * h
    regions = [Region(cls=1, kind="cylinder", axis=0, center=(y, z), radius=1.2 * h,
                      lo=(-1e9, -1e9, -1e9), hi=(1e9, 1e9, 1e9)) for y in (y1, y2)]
    regions.append(Region(cls=2, kind="box", lo=(-1.0, -1.0, -1.0), hi=(1.5 * h, 1e9, 1e9)))
    table = np.array([[0, 2, 3], [2, 1, 3], [3, 3, 3]], dtype=np.uint8)
    return RuleClassifier(table, regions)


@pytest.mark.gpu
@pytest.mark.parametrize("jitter", [0.0, 0.2])
def test_classified_family_matches_reference(reference, jitter):
    counts = (30, 12, 10)
    g, p = S.lattice_particles(counts)
    coords = p.coords.copy()
    if jitter:
        coords = coords + np.random.default_rng(3).uniform(-jitter, jitter, coords.shape)
    hint = g.hint() if not jitter else None
    cls = rc_beam_rules(*counts)
    ent, types, N = reference.build_family_classified(coords, 3.0, hint, cls)
    fam = geometry.build_family(coords, 3.0, g if not jitter else None, classify=cls)
    assert fam.group_size == N
    assert np.array_equal(fam.entries, ent)
    assert np.array_equal(fam.bond_type, types)
    # every class pair occurs
    assert set(np.unique(types[ent >= 0])) == {0, 1, 2, 3}


@pytest.mark.gpu
def test_surface_correction_matches_reference(reference):
    counts = (14, 11, 9)
    g, p = S.lattice_particles(counts)
    fam = geometry.build_family(p.coords, np.pi, g)
    rng = np.random.default_rng(5)
    vol = rng.uniform(0.5, 1.5, fam.node_count())
    # with some pre-broken bonds: the reference sums over the current rows
    geometry.break_plane(fam, p.coords, 0, 6.5)
    nb = geometry.neighborhood_volumes(vol, fam)
    assert nb.view(np.uint64).tolist() == reference.neighborhood_volumes(vol, fam).view(np.uint64).tolist()
    for v0 in (geometry.max_neighborhood_volume(vol, fam),
               geometry.analytic_neighborhood_volume(np.pi, 0.9), 17.25):
        lam = geometry.surface_correction_factors(vol, fam, v0)
        ref = reference.surface_correction_factors(vol, fam, v0)
        assert np.array_equal(lam.view(np.uint64), ref.view(np.uint64)), v0
    assert geometry.max_neighborhood_volume(vol, fam) == float(nb.max())


@pytest.mark.gpu
def test_surface_correction_errors_match_reference(reference):
    g, p = S.lattice_particles((5, 4, 3))
    fam = geometry.build_family(p.coords, 1.5, g)
    vol = np.ones(fam.node_count())
    msgs = []
    for be in (geometry, reference):
        with pytest.raises(abi.DomainError) as e1:
            be.surface_correction_factors(vol, fam, 0.0)
        with pytest.raises(abi.DomainError) as e2:
            be.surface_correction_factors(np.zeros_like(vol), fam, 1.0)
        msgs.append((str(e1.value), str(e2.value)))
    assert msgs[0] == msgs[1]
    assert "zero neighborhood volume for bond 0-" in msgs[0][1]


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["plane", "notch"])
def test_initial_breaks_match_reference(reference, kind):
    b, h, g, notch = S.notched_plate_bundle(40, 36, 4)
    coords = b.particles.coords
    rng = np.random.default_rng(9)
    coords = coords + rng.uniform(-0.1, 0.1, coords.shape)  # irregular crossings
    fams = [geometry.build_family(coords, h) for _ in range(2)]
    if kind == "plane":
        geometry.break_plane(fams[0], coords, 1, 17.5)
        reference.break_bonds(fams[1], coords, 0, 1, 17.5)
    else:
        geometry.break_notch(fams[0], coords, notch["axis"], notch["position"],
                             notch["sweep_axis"], notch["depth"])
        reference.break_bonds(fams[1], coords, 1, notch["axis"], notch["position"],
                              notch["sweep_axis"], notch["depth"])
    assert np.array_equal(fams[0].entries, fams[1].entries)
    assert np.array_equal(fams[0].n_neigh, fams[1].n_neigh)
    assert np.array_equal(fams[0].initial_n_neigh, fams[1].initial_n_neigh)
    assert int(fams[0].initial_n_neigh.sum() - fams[0].n_neigh.sum()) > 0


def test_rule_table_validation_on_cpu():
    """Argument checks precede any device work (no GPU needed)."""
    g, p = S.lattice_particles((3, 3, 3))
    from paper_2105_04150_b200.types import NeighborList
    n = p.size()
    fam = NeighborList(np.full(n * 2, -1, np.int32), np.zeros(n, np.int32),
                       np.zeros(n, np.int32), 2, 1.0, None)
    bad = RuleClassifier(np.array([[0, 1], [2, 0]], dtype=np.uint8))
    with pytest.raises(abi.InvalidArgument, match="symmetric"):
        geometry.classify_bonds(p.coords, fam, bad)
    bad = RuleClassifier(np.zeros((2, 2), np.uint8), [Region(cls=5)])
    with pytest.raises(abi.InvalidArgument, match="region"):
        geometry.classify_bonds(p.coords, fam, bad)
    with pytest.raises(abi.DomainError, match="V0 must be positive"):
        geometry.surface_correction_factors(np.ones(n), fam, -1.0)


@pytest.mark.gpu
def test_bad_entries_are_rejected():
    """A row naming a node outside the list is an error, not a device fault."""
    g, p = S.lattice_particles((4, 3, 3))
    fam = geometry.build_family(p.coords, 1.5, g)
    fam.entries[5] = fam.node_count() + 3
    vol = np.ones(fam.node_count())
    with pytest.raises(abi.InvalidArgument, match="out of range in row 0"):
        geometry.neighborhood_volumes(vol, fam)
    with pytest.raises(abi.InvalidArgument, match="out of range"):
        geometry.classify_bonds(p.coords, fam, rc_beam_rules(4, 3, 3))
    with pytest.raises(abi.InvalidArgument, match="out of range"):
        geometry.break_plane(fam, p.coords, 0, 1.5)
