"""Multi-GPU z-slabs on the device (csrc: peer-store ghost push in the step
epilogue + slab_sync_kernel).  This pool gives one GPU per call, so the ranks
share cuda:0: as threads of one process (ThreadComm, peer pointers are
same-device pointers) and as two processes (gloo + CUDA IPC handles).  The
exact variants must be BITWISE equal to the global oracle run -- u, v, a,
broken sets, n_neigh, history, tip records and write-hook views; the fast
variant within its documented tolerance of the one-GPU fast run."""
import os

import numpy as np
import pytest

import scenarios as S
from golden_io import same_bits, tips_table
from paper_2105_04150_b200 import abi, engine, slabs
from paper_2105_04150_b200.types import (IntegratorKind, KernelVariant, SimulateOptions,
                                         make_state)

pytestmark = pytest.mark.gpu


def _plate(oracle, nx=24, ny=16, nz=14, steps=15):
    b, h, g, notch = S.notched_plate_bundle(nx, ny, nz, steps)
    fam = oracle.build_family(b.particles.coords, h, g.hint())
    oracle.break_notch(fam, b.particles.coords, notch["axis"], notch["position"],
                       notch["sweep_axis"], notch["depth"])
    return b, fam


def _same(a, b):
    assert a.step == b.step
    for name in ("u", "v", "a"):
        assert same_bits(getattr(a, name), getattr(b, name)), name
    assert np.array_equal(a.connectivity.entries, b.connectivity.entries)
    assert np.array_equal(a.connectivity.n_neigh, b.connectivity.n_neigh)
    if a.bond_history is not None and np.asarray(a.bond_history).size:
        assert same_bits(a.bond_history, b.bond_history)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("integrator", list(IntegratorKind))
def test_slabs_exact_bitwise_with_tips_and_hooks(oracle, world, integrator):
    b, fam = _plate(oracle)
    b.model.damping = 0.02
    opts = SimulateOptions(60, 20, 3, integrator, KernelVariant.bond_parallel)
    ref = make_state(fam, b.model.needs_history())
    ref_hooks = []
    ref_res = oracle.simulate(b, ref, opts, lambda s, f: ref_hooks.append(
        (s.step, s.u.copy(), f.body_force.copy(), f.external_force.copy())))
    assert fam.n_neigh.sum() > ref.connectivity.n_neigh.sum()  # it fractured
    st = make_state(fam, b.model.needs_history())
    hooks = []
    res = slabs.simulate_slabs_local(b, st, opts, world, on_write=lambda s, f: hooks.append(
        (s.step, s.u.copy(), f.body_force.copy(), f.external_force.copy())))
    _same(ref, st)
    assert same_bits(tips_table(ref_res), tips_table(res))
    assert len(hooks) == len(ref_hooks) == 3
    for x, y in zip(ref_hooks, hooks):
        assert x[0] == y[0]
        for p, q in zip(x[1:], y[1:]):
            assert same_bits(p, q)


def test_slabs_trilinear_multimaterial_node_variant(oracle):
    b, h, g = S.multimaterial_bundle((8, 8, 24))
    fam = oracle.build_family(b.particles.coords, h, g.hint())
    fam.bond_type = S.classify_bonds(b.particles.coords, fam)
    b.corrections.beta = np.random.default_rng(3).uniform(0.7, 1.0, fam.entries.size)
    opts = SimulateOptions(80, 0, 0, IntegratorKind.velocity_verlet, KernelVariant.node_parallel)
    ref = make_state(fam, True)
    oracle.simulate(b, ref, opts)
    st = make_state(fam, True)
    slabs.simulate_slabs_local(b, st, opts, 3)
    _same(ref, st)


def test_slabs_lattice_fracture_four_ranks(oracle):
    """The bench's fracturing variant (s_c = 1e-5), 4 slabs of a 20 x 20 x 40 lattice."""
    from paper_2105_04150_b200 import geometry
    b, h, g = S.bench_lattice_bundle((20, 20, 40), s_c=1e-5)
    fam = geometry.build_family(b.particles.coords, h, g)
    opts = SimulateOptions(25, 0, 0, IntegratorKind.velocity_verlet)
    ref = make_state(fam, False)
    ref.u = S.seed_displacements(b.particles.coords)
    st = make_state(fam, False)
    st.u = ref.u.copy()
    oracle.simulate(b, ref, opts)
    slabs.simulate_slabs_local(b, st, opts, 4)
    _same(ref, st)
    assert fam.n_neigh.sum() - st.connectivity.n_neigh.sum() > 0


@pytest.mark.parametrize("integrator", [IntegratorKind.velocity_verlet, IntegratorKind.euler])
def test_slabs_nonfinite_stops_every_rank_at_the_same_step(oracle, integrator):
    b, fam = _plate(oracle)
    node = b.particles.size() - 200   # in the last slab: the flag must reach rank 0
    b.bc.kind[3 * node] = 2            # a force axis with an enormous load
    b.bc.magnitude[3 * node] = 1.5e308
    b.bc.ramp_id[3 * node] = 0
    opts = SimulateOptions(120, 0, 2, integrator)
    ref = make_state(fam, False)
    with pytest.raises(abi.PeridynRuntimeError) as e1:
        oracle.simulate(b, ref, opts)
    st = make_state(fam, False)
    with pytest.raises(abi.PeridynRuntimeError) as e2:
        slabs.simulate_slabs_local(b, st, opts, 2)
    assert str(e1.value) == str(e2.value)
    _same(ref, st)


def test_slabs_fast_variant_within_tolerance(oracle):
    from paper_2105_04150_b200 import geometry
    b, h, g = S.bench_lattice_bundle((24, 24, 30), s_c=1e6)
    fam = geometry.build_family(b.particles.coords, h, g)
    opts = SimulateOptions(30, 0, 0, IntegratorKind.velocity_verlet, KernelVariant.fast)
    one = make_state(fam, False)
    one.u = S.seed_displacements(b.particles.coords)
    st = make_state(fam, False)
    st.u = one.u.copy()
    engine.simulate(b, one, opts)
    slabs.simulate_slabs_local(b, st, opts, 3)
    scale = np.max(np.abs(one.u))
    assert np.max(np.abs(one.u - st.u)) <= 1e-6 * scale
    assert np.array_equal(one.connectivity.entries, st.connectivity.entries)


def _proc_rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.pyoracle import COracle
        oracle = COracle(threads=4)
        b, fam = _plate(oracle)
        opts = SimulateOptions(50, 25, 0, IntegratorKind.velocity_verlet)
        st = make_state(fam, b.model.needs_history())
        res = slabs.simulate_slabs(b, st, opts, comm=slabs.TorchComm(), device=0)
        ref = make_state(fam, b.model.needs_history())
        ref_res = oracle.simulate(b, ref, opts)
        _same(ref, st)
        assert same_bits(tips_table(ref_res), tips_table(res))
        q.put((rank, "ok"))
    except BaseException as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


def test_slabs_two_processes_cuda_ipc():
    """Two rank processes (gloo for the handle exchange, CUDA IPC for the
    peer buffers), both on cuda:0 here; on an 8-GPU box the same code maps
    buffers of other GPUs."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
