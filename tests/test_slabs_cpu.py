"""Multi-GPU z-slab host logic on the CPU (no GPU): partition, local problems,
ghost/send maps and the gather, driven with the C oracle as each rank's
device (tests/slab_emulation.py), as threads and as a world-size-2 gloo
process group.  The owned rows must be BITWISE equal to the global run."""
import os

import numpy as np
import pytest

import scenarios as S
import slab_emulation
from golden_io import same_bits
from paper_2105_04150_b200 import slabs
from paper_2105_04150_b200.types import IntegratorKind, SimulateOptions, make_state


def _plate(oracle, nx=24, ny=16, nz=14, steps=15):
    b, h, g, notch = S.notched_plate_bundle(nx, ny, nz, steps)
    fam = oracle.build_family(b.particles.coords, h, g.hint())
    oracle.break_notch(fam, b.particles.coords, notch["axis"], notch["position"],
                       notch["sweep_axis"], notch["depth"])
    return b, fam


def _same(a, b):
    for name in ("u", "v", "a"):
        assert same_bits(getattr(a, name), getattr(b, name)), name
    assert np.array_equal(a.connectivity.entries, b.connectivity.entries)
    assert np.array_equal(a.connectivity.n_neigh, b.connectivity.n_neigh)
    if a.bond_history is not None and np.asarray(a.bond_history).size:
        assert same_bits(a.bond_history, b.bond_history)


def test_partition_cuts_whole_planes():
    g, p = S.lattice_particles((6, 5, 9))
    ranges = slabs.partition(p.coords, 3)
    assert [r[0] % 30 for r in ranges] == [0, 0, 0]
    assert ranges[0][0] == 0 and ranges[-1][1] == 270
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_plan_rejects_slabs_thinner_than_horizon(oracle):
    b, fam = _plate(oracle, 10, 8, 6)
    with pytest.raises(ValueError, match="thinner than the horizon"):
        slabs.plan(b.particles.coords, fam.entries, fam.group_size, 4)


def test_plan_ghosts_are_one_horizon(oracle):
    b, fam = _plate(oracle)
    parts = slabs.plan(b.particles.coords, fam.entries, fam.group_size, 3)
    plane = 24 * 16
    for p in parts:
        assert p.own_end - p.own_begin == p.g_end - p.g_begin
        assert np.all(np.diff(p.local_ids) > 0)
        # delta = pi over unit spacing: three ghost planes per interior face
        if p.lo >= 0:
            assert p.own_begin == 3 * plane
        if p.hi >= 0:
            assert p.n_local - p.own_end == 3 * plane


def _threads(fn, world):
    import threading
    comms = slabs.ThreadComm.group(world)
    errs = [None] * world
    outs = [None] * world

    def body(r):
        try:
            outs[r] = fn(comms[r])
        except BaseException as e:  # noqa: BLE001
            errs[r] = e
    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return outs


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("integrator", [IntegratorKind.velocity_verlet,
                                        IntegratorKind.euler_cromer])
def test_emulated_slabs_bitwise(oracle, world, integrator):
    b, fam = _plate(oracle)
    b.model.damping = 0.02
    ref = make_state(fam, b.model.needs_history())
    oracle.simulate(b, ref, SimulateOptions(40, 0, 0, integrator))
    assert fam.n_neigh.sum() > ref.connectivity.n_neigh.sum()  # it fractured

    def rank(comm):
        st = make_state(fam, b.model.needs_history())
        slab_emulation.emulate(oracle, b, st, SimulateOptions(40, 0, 0, integrator), comm)
        return st
    for st in _threads(rank, world):
        _same(ref, st)


def test_emulated_slabs_trilinear_multimaterial(oracle):
    b, h, g = S.multimaterial_bundle((8, 8, 18))
    fam = oracle.build_family(b.particles.coords, h, g.hint())
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    ref = make_state(fam, True)
    oracle.simulate(b, ref, SimulateOptions(60, 0, 0, IntegratorKind.velocity_verlet))

    def rank(comm):
        st = make_state(fam, True)
        slab_emulation.emulate(oracle, b, st, SimulateOptions(60, 0, 0,
                                                              IntegratorKind.velocity_verlet), comm)
        return st
    for st in _threads(rank, 2):
        _same(ref, st)


def _gloo_rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import COracle
        oracle = COracle(threads=1)
        b, fam = _plate(oracle)
        st = make_state(fam, b.model.needs_history())
        slab_emulation.emulate(oracle, b, st, SimulateOptions(30, 0, 0,
                                                              IntegratorKind.velocity_verlet),
                               slabs.TorchComm())
        ref = make_state(fam, b.model.needs_history())
        oracle.simulate(b, ref, SimulateOptions(30, 0, 0, IntegratorKind.velocity_verlet))
        _same(ref, st)
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_emulated_slabs_gloo_world2():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
