"""Binary containers (io.cpp:297-564): PDST restart state and PDNL family
cache.  The fixtures in tests/golden/*.pdst|*.pdnl were written by the
UNMODIFIED reference (tests/golden/make_golden_io.py).  The product's readers
and writers must round-trip them byte for byte and reject corrupt files with
the reference's messages; on the GPU, a resident run saved straight from
device memory must produce the reference's file byte for byte."""
import os
import shutil

import numpy as np
import pytest

import scenarios as S
from golden_io import same_bits
from paper_2105_04150_b200 import abi, engine
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, SimulateOptions, make_state

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", ["state_trilinear.pdst", "state_pmb.pdst"])
def test_state_round_trip_is_byte_identical(tmp_path, name):
    st = engine.load_state(os.path.join(GOLD, name))
    out = tmp_path / name
    engine.save_state(st, str(out))
    assert _bytes(out) == _bytes(os.path.join(GOLD, name))


def test_cache_round_trip_is_byte_identical(tmp_path):
    fam, corr = engine.load_cache(os.path.join(GOLD, "family.pdnl"))
    assert fam.bond_type is not None and corr.lambda_ is not None and corr.beta is not None
    out = tmp_path / "family.pdnl"
    engine.save_cache(fam, corr, str(out))
    assert _bytes(out) == _bytes(os.path.join(GOLD, "family.pdnl"))


def test_loaded_state_matches_the_oracle_run(oracle):
    """The reference's saved trajectory equals the C oracle's run of the same case."""
    st = engine.load_state(os.path.join(GOLD, "state_trilinear.pdst"))
    b, h, g = S.multimaterial_bundle((7, 5, 6))
    fam = oracle.build_family(b.particles.coords, 2.0, g.hint())
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    ref = make_state(fam, True)
    oracle.simulate(b, ref, SimulateOptions(40, 0, 0, IntegratorKind.velocity_verlet))
    assert st.step == ref.step == 40
    for name in ("u", "v", "a", "bond_history"):
        assert same_bits(getattr(st, name), getattr(ref, name)), name
    assert np.array_equal(st.connectivity.entries, ref.connectivity.entries)
    assert np.array_equal(st.connectivity.n_neigh, ref.connectivity.n_neigh)
    assert np.array_equal(st.connectivity.bond_type, fam.bond_type)


def _corrupt(tmp_path, name, fn):
    src = os.path.join(GOLD, name)
    data = bytearray(_bytes(src))
    data = fn(data)
    p = tmp_path / ("bad_" + name)
    with open(p, "wb") as f:
        f.write(bytes(data))
    return str(p)


@pytest.mark.parametrize("mutate,message", [
    (lambda d: b"XXXX" + d[4:], "bad magic, not a PDST file"),
    (lambda d: d[:4] + (2).to_bytes(4, "little") + d[8:], "unsupported version 2"),
    (lambda d: d[:len(d) - 100], "truncated file"),
    (lambda d: d[:40] + (7).to_bytes(4, "little") + (123).to_bytes(8, "little") + d[52:],
     "section length 123 does not match expected"),
    (lambda d: d + (99).to_bytes(4, "little") + (0).to_bytes(8, "little"),
     "unknown section id 99"),
    (lambda d: d[:8] + (0).to_bytes(8, "little") + d[16:], "corrupt header"),
])
def test_corrupt_state_files_are_rejected(tmp_path, mutate, message):
    """io.cpp:371-393, 507-562 (the reference's test_io.cpp:145-178 cases)."""
    p = _corrupt(tmp_path, "state_pmb.pdst", mutate)
    with pytest.raises(abi.PeridynRuntimeError) as e:
        engine.load_state(p)
    assert str(e.value).startswith(p + ": ") and message in str(e.value)


def test_missing_section_is_rejected(tmp_path):
    # drop the trailing initial_n_neigh section of the PMB state
    def drop_last(d):
        n = int.from_bytes(d[8:16], "little")
        return d[:len(d) - (12 + 4 * n)]
    p = _corrupt(tmp_path, "state_pmb.pdst", drop_last)
    with pytest.raises(abi.PeridynRuntimeError, match="missing required sections"):
        engine.load_state(p)


@pytest.mark.gpu
def test_device_save_state_is_the_reference_file(tmp_path):
    """A resident exact run of the fixture's case, saved straight from HBM,
    is byte-identical to the reference's save_state of its own run."""
    from paper_2105_04150_b200 import geometry
    b, h, g = S.multimaterial_bundle((7, 5, 6))
    fam = geometry.build_family(b.particles.coords, 2.0, g)
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    st = make_state(fam, True)
    ctx = engine.Context(0)
    ctx.upload(b, st, KernelVariant.bond_parallel)
    ctx.run(40, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.bond_parallel)
    out = tmp_path / "dev.pdst"
    ctx.save_state(str(out))
    ctx.close()
    assert _bytes(out) == _bytes(os.path.join(GOLD, "state_trilinear.pdst"))


@pytest.mark.gpu
def test_device_save_state_fast_layouts_round_trip(tmp_path, monkeypatch):
    """Fast layouts (lattice and tiles) save the same state a download sees."""
    b, h, g = S.bench_lattice_bundle((12, 10, 9), s_c=2e-5)
    from paper_2105_04150_b200 import geometry
    fam = geometry.build_family(b.particles.coords, h, g)
    for layout in ("lattice", "tiles"):
        if layout == "tiles":
            monkeypatch.setenv("PD_FAST_LAYOUT", "general")
        st = make_state(fam, False)
        st.u = S.seed_displacements(b.particles.coords) * 4
        ctx = engine.Context(0)
        ctx.upload(b, st, KernelVariant.fast)
        assert ctx.layout() == layout
        ctx.run(15, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.fast)
        p = tmp_path / f"{layout}.pdst"
        ctx.save_state(str(p))
        ctx.download(st)
        ctx.close()
        q = tmp_path / f"{layout}_host.pdst"
        engine.save_state(st, str(q))
        assert _bytes(p) == _bytes(q)
        back = engine.load_state(str(p))
        assert same_bits(back.u, st.u)
        assert np.array_equal(back.connectivity.entries, st.connectivity.entries)


def test_host_snapshot_is_the_reference_file(tmp_path):
    """write_snapshot(make_snapshot(...)) (io.cpp:235-269): 17-digit ASCII, same bytes."""
    st = engine.load_state(os.path.join(GOLD, "state_trilinear.pdst"))
    b, h, g = S.multimaterial_bundle((7, 5, 6))
    out = tmp_path / "snap.pdsnap"
    engine.write_snapshot(st, b.particles, str(out))
    assert _bytes(out) == _bytes(os.path.join(GOLD, "snap_trilinear.pdsnap"))


@pytest.mark.gpu
def test_device_snapshots_sync_and_async(tmp_path, oracle):
    """The resident state's snapshot equals the reference file; snapshots
    queued during run() (written by a host thread while the GPU steps) equal
    the host writer's files of the oracle's states at the same steps."""
    from paper_2105_04150_b200 import geometry
    b, h, g = S.multimaterial_bundle((7, 5, 6))
    fam = geometry.build_family(b.particles.coords, 2.0, g)
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    st = make_state(fam, True)
    ctx = engine.Context(0)
    ctx.upload(b, st, KernelVariant.bond_parallel)
    ctx.snapshot_every(10, str(tmp_path / "async_%06lld.pdsnap"))
    ctx.run(40, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.bond_parallel)
    ctx.write_snapshot(str(tmp_path / "sync.pdsnap"))
    ctx.close()
    assert _bytes(tmp_path / "sync.pdsnap") == _bytes(os.path.join(GOLD, "snap_trilinear.pdsnap"))
    ref = make_state(fam, True)
    written = []

    def hook(s, f):
        p = tmp_path / f"ref_{s.step:06d}.pdsnap"
        engine.write_snapshot(s, b.particles, str(p))
        written.append(s.step)
    oracle.simulate(b, ref, SimulateOptions(40, 10, 0, IntegratorKind.velocity_verlet), hook)
    assert written == [10, 20, 30, 40]
    for step in written:
        assert _bytes(tmp_path / f"async_{step:06d}.pdsnap") == \
            _bytes(tmp_path / f"ref_{step:06d}.pdsnap"), step


@pytest.mark.gpu
def test_device_save_state_keeps_history_under_pmb(tmp_path, oracle):
    """A PMB model run from a state that carries bond_history: the reference
    leaves the history untouched and save_state still writes its section
    (io.cpp section 10); the resident run saves the same bytes."""
    from paper_2105_04150_b200 import geometry
    b, h, g = S.bench_lattice_bundle((9, 8, 7), s_c=1e6)
    fam = geometry.build_family(b.particles.coords, h, g)
    rng = np.random.default_rng(7)
    hist = np.where(fam.entries >= 0, rng.uniform(0, 1e-3, fam.entries.size), 0.0)
    files = []
    for be in ("oracle", "device"):
        st = make_state(fam, False)
        st.u = S.seed_displacements(b.particles.coords)
        st.bond_history = hist.copy()
        p = tmp_path / f"{be}.pdst"
        if be == "oracle":
            oracle.simulate(b, st, SimulateOptions(6, 0, 0, IntegratorKind.velocity_verlet))
            engine.save_state(st, str(p))
        else:
            ctx = engine.Context(0)
            ctx.upload(b, st, KernelVariant.bond_parallel)
            ctx.run(6, 0, IntegratorKind.velocity_verlet, 0, KernelVariant.bond_parallel)
            ctx.save_state(str(p))
            ctx.close()
        files.append(_bytes(p))
    assert files[0] == files[1]
    assert engine.load_state(str(tmp_path / "device.pdst")).bond_history is not None


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [KernelVariant.bond_parallel, KernelVariant.fast])
def test_async_snapshots_stop_at_the_failed_step(tmp_path, oracle, variant):
    """A run that turns non-finite at step e: the reference throws inside step
    e's force pass, so no snapshot after e is written; the queued asynchronous
    snapshots past e are dropped."""
    b, h, _ = S.small_fracture_bundle()
    fam = oracle.build_family(b.particles.coords, h)
    b.model.laws[0] = type(b.model.laws[0]).pmb(0.05, 1e9)
    b.bc.kind[:] = 0
    b.bc.kind[3 * 7] = 2  # force axis with an enormous load
    b.bc.magnitude[3 * 7] = 1.5e308
    ref = make_state(fam, False)
    with pytest.raises(abi.PeridynRuntimeError) as ei:
        oracle.simulate(b, ref, SimulateOptions(120, 0, 0, IntegratorKind.euler))
    failed = int(str(ei.value).rsplit("step", 1)[1].split()[0])
    st = make_state(fam, False)
    ctx = engine.Context(0)
    ctx.upload(b, st, variant)
    ctx.snapshot_every(1, str(tmp_path / "s_%06lld.pdsnap"))
    with pytest.raises(abi.PeridynRuntimeError):
        ctx.run(120, 0, IntegratorKind.euler, 0, variant)
    ctx.close()
    steps = sorted(int(f[2:8]) for f in os.listdir(tmp_path) if f.endswith(".pdsnap"))
    assert steps and max(steps) <= failed, (failed, steps[-3:])
    assert steps == list(range(1, max(steps) + 1))
