"""Host mirror of the reference engine API (include/peridyn/engine.hpp) over a
pd-style C ABI.

`Backend(lib, prefix)` binds any library exporting the pd_b200.h entry points
under `prefix`.  The product binds libpd_b200.so ("pd_"); the test checkers
under oracle/ bind the same calls on their own libraries, so a parity test
drives the GPU and its checker through identical Python code.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import abi
from .abi import HOOK, Marshal, check
from .types import (ForceField, IntegratorKind, KernelVariant, ModelBundle, SimulateOptions,
                    SimulateResult, SimulationState, TipRecord, WriteHook)

_PKG = os.path.dirname(os.path.abspath(__file__))
# PD_B200_LIB: an alternative build of the same library (kernel experiments)
LIB_PATH = os.environ.get("PD_B200_LIB") or os.path.join(_PKG, "libpd_b200.so")


class Backend:
    def __init__(self, lib: C.CDLL, prefix: str):
        self.lib = lib
        self.prefix = prefix
        self._last = getattr(lib, prefix + "last_error")
        self._last.restype = C.c_char_p
        self._cf = getattr(lib, prefix + "compute_forces")
        self._cf.argtypes = [C.c_int32, C.POINTER(abi.pd_state), C.POINTER(abi.pd_particles),
                             C.POINTER(abi.pd_damage_model), C.POINTER(abi.pd_corrections),
                             C.POINTER(abi.pd_force_field)]
        self._sim = getattr(lib, prefix + "simulate")
        self._sim.argtypes = [C.POINTER(abi.pd_bundle), C.POINTER(abi.pd_state),
                              C.POINTER(abi.pd_options), HOOK, C.c_void_p,
                              C.POINTER(abi.pd_tip_record), C.c_int64, C.POINTER(C.c_int64)]

    def last_error(self) -> str:
        return self._last().decode()

    def _check(self, rc: int) -> None:
        check(rc, self._last)

    # ---- stand-alone integrators (engine.hpp:38-62, engine.cpp:187-260) ----
    def _integrate(self, name, state, forces, dt, damping, density):
        fn = getattr(self.lib, self.prefix + name)
        m = Marshal()
        st = m.state(state)
        if name == "verlet_drift":
            fn.argtypes = [C.POINTER(abi.pd_state), C.c_double]
            rc = fn(C.byref(st), float(dt))
        else:
            rho = m._k(abi.as_f64(density))
            ff = m.forces(forces)
            args = [C.byref(st), C.byref(ff), float(dt)]
            types = [C.POINTER(abi.pd_state), C.POINTER(abi.pd_force_field), C.c_double]
            if name == "verlet_kick":
                args.append(float(damping))
                types.append(C.c_double)
            fn.argtypes = types + [C.POINTER(C.c_double), C.c_int64]
            rc = fn(*args, abi.ptr(rho, C.c_double), rho.size)
        self._check(rc)

    def verlet_drift(self, state, dt) -> None:
        self._integrate("verlet_drift", state, None, dt, 0.0, None)

    def verlet_kick(self, state, forces, dt, damping, density) -> None:
        self._integrate("verlet_kick", state, forces, dt, damping, density)

    def step_euler(self, state, forces, dt, density) -> None:
        self._integrate("step_euler", state, forces, dt, 0.0, density)

    def step_euler_cromer(self, state, forces, dt, density) -> None:
        self._integrate("step_euler_cromer", state, forces, dt, 0.0, density)

    def step_velocity_verlet(self, state, force_eval, scratch, dt, damping, density) -> None:
        """step_velocity_verlet (engine.cpp:254-260): drift, force_eval(state,
        scratch), kick, ++step."""
        self.verlet_drift(state, dt)
        force_eval(state, scratch)
        self.verlet_kick(state, scratch, dt, damping, density)
        state.step += 1

    # ---- boundary conditions (engine.hpp:64-78, engine.cpp:262-305) ----------
    def apply_displacement_positions(self, state, bc, step) -> None:
        m = Marshal()
        st, b = m.state(state), m.boundary(bc)
        fn = getattr(self.lib, self.prefix + "apply_displacement_positions")
        fn.argtypes = [C.POINTER(abi.pd_state), C.POINTER(abi.pd_boundary), C.c_int64]
        rc = fn(C.byref(st), C.byref(b), int(step))
        if self.prefix == "pd_":
            self._check(rc)

    def apply_displacement_kinematics(self, state, bc, step, dt) -> None:
        m = Marshal()
        st, b = m.state(state), m.boundary(bc)
        fn = getattr(self.lib, self.prefix + "apply_displacement_kinematics")
        fn.argtypes = [C.POINTER(abi.pd_state), C.POINTER(abi.pd_boundary), C.c_int64,
                       C.c_double]
        rc = fn(C.byref(st), C.byref(b), int(step), float(dt))
        if self.prefix == "pd_":
            self._check(rc)

    def accumulate_external_force(self, bc, step, out) -> None:
        m = Marshal()
        b = m.boundary(bc)
        ff = m.forces(out)
        n = out.external_force.size // 3
        fn = getattr(self.lib, self.prefix + "accumulate_external_force")
        if self.prefix == "pd_":
            fn.argtypes = [C.POINTER(abi.pd_boundary), C.c_int64, C.POINTER(abi.pd_force_field),
                           C.c_int64]
            self._check(fn(C.byref(b), int(step), C.byref(ff), n))
        else:
            fn.argtypes = [C.POINTER(abi.pd_boundary), C.c_int64, C.POINTER(C.c_double), C.c_int64]
            fn(C.byref(b), int(step), ff.external_force, n)

    def apply_boundary(self, state, bc, step, dt, out) -> None:
        """apply_boundary (engine.cpp:299-305)."""
        if self.prefix == "pd_":
            m = Marshal()
            st, b, ff = m.state(state), m.boundary(bc), m.forces(out)
            fn = self.lib.pd_apply_boundary
            fn.argtypes = [C.POINTER(abi.pd_state), C.POINTER(abi.pd_boundary), C.c_int64,
                           C.c_double, C.POINTER(abi.pd_force_field)]
            self._check(fn(C.byref(st), C.byref(b), int(step), float(dt), C.byref(ff)))
            return
        m = Marshal()
        b = m.boundary(bc)
        fn = getattr(self.lib, self.prefix + "bc_validate")
        fn.argtypes = [C.POINTER(abi.pd_boundary), C.c_int64]
        self._check(fn(C.byref(b), state.size()))
        self.apply_displacement_positions(state, bc, step)
        self.apply_displacement_kinematics(state, bc, step, dt)
        self.accumulate_external_force(bc, step, out)

    # compute_forces (engine.hpp:35-36, engine.cpp:163-169)
    def compute_forces(self, variant, state: SimulationState, particles, model, corrections,
                       out: ForceField) -> None:
        n = state.size()
        if np.asarray(out.body_force).size != 3 * n:
            out.body_force = np.zeros(3 * n)
        if np.asarray(out.external_force).size != 3 * n:
            out.external_force = np.zeros(3 * n)
        m = Marshal()
        st = m.state(state)
        p = m.particles(particles)
        md = m.model(model)
        cr = m.corrections(corrections)
        ff = m.forces(out)
        rc = self._cf(int(variant), C.byref(st), C.byref(p), C.byref(md), C.byref(cr),
                      C.byref(ff))
        state.step = st.step
        self._check(rc)

    # simulate (engine.hpp:128-129, engine.cpp:374-425)
    def simulate(self, bundle: ModelBundle, state: SimulationState, options: SimulateOptions,
                 on_write: Optional[WriteHook] = None) -> SimulateResult:
        n = bundle.particles.size()
        slots = state.size() * int(state.connectivity.group_size)
        if bundle.model.needs_history() and np.asarray(
                state.bond_history if state.bond_history is not None else []).size != slots:
            state.bond_history = np.zeros(slots)  # engine.cpp:382-384
        names = sorted(bundle.bc.tip_sets)
        writes = 0
        if options.write_every > 0 and options.steps > 0:
            writes = sum(1 for s in range(options.first_step, options.first_step + options.steps)
                         if (s + 1) % options.write_every == 0)
        cap = max(1, writes * len(names))
        recs = (abi.pd_tip_record * cap)()
        n_recs = C.c_int64(0)
        m = Marshal()
        b = m.bundle(bundle)
        st = m.state(state)
        o = Marshal.options(options)
        errors = []

        def bridge(_user, view, ff):
            try:
                v = view.contents
                state.step = v.step
                seen = _state_view(v, state) if v.u else state
                forces = ForceField(
                    np.ctypeslib.as_array(ff.contents.body_force, (3 * n,)).copy(),
                    np.ctypeslib.as_array(ff.contents.external_force, (3 * n,)).copy())
                on_write(seen, forces)
                return 0
            except BaseException as exc:  # propagate after the C call unwinds
                errors.append(exc)
                return 1

        hook = HOOK(bridge) if on_write is not None else HOOK()
        rc = self._sim(C.byref(b), C.byref(st), C.byref(o), hook, None, recs, cap,
                       C.byref(n_recs))
        state.step = st.step
        if errors:
            raise errors[0]
        self._check(rc)
        result = SimulateResult({name: [] for name in names} if names else {})
        for k in range(n_recs.value):
            r = recs[k]
            rec = TipRecord(int(r.step), np.array(r.mean_u[:]), np.array(r.mean_v[:]),
                            np.array(r.mean_a[:]), np.array(r.body_force_sum[:]),
                            np.array(r.external_force_sum[:]))
            result.tips[names[k % len(names)]].append(rec)
        return result


def _state_view(v, like: SimulationState) -> SimulationState:
    """Copy of the state a write hook sees, read through the pd_state view."""
    n = like.size()
    N = int(like.connectivity.group_size)
    arr = np.ctypeslib.as_array
    fam = like.connectivity.copy()
    fam.entries = arr(v.connectivity.entries, (n * N,)).copy()
    fam.n_neigh = arr(v.connectivity.n_neigh, (n,)).copy()
    hist = arr(v.bond_history, (v.bond_history_size,)).copy() if v.bond_history_size else np.zeros(0)
    return SimulationState(arr(v.u, (3 * n,)).copy(), arr(v.v, (3 * n,)).copy(),
                           arr(v.a, (3 * n,)).copy(), int(v.step), fam, hist)


# ---- the product library --------------------------------------------------------

_LIB: Optional[C.CDLL] = None
_BACKEND: Optional[Backend] = None


def library() -> C.CDLL:
    """libpd_b200.so; raises if it was not built (there is no CPU fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise abi.CudaError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        lib = C.CDLL(LIB_PATH)
        lib.pd_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
        lib.pd_ctx_destroy.argtypes = [C.c_void_p]
        lib.pd_ctx_upload.argtypes = [C.c_void_p, C.POINTER(abi.pd_bundle),
                                      C.POINTER(abi.pd_state), C.c_int32]
        lib.pd_ctx_run.argtypes = [C.c_void_p, C.POINTER(abi.pd_options), HOOK, C.c_void_p,
                                   C.c_int32, C.POINTER(abi.pd_tip_record), C.c_int64,
                                   C.POINTER(C.c_int64)]
        lib.pd_ctx_compute_forces.argtypes = [C.c_void_p]
        lib.pd_ctx_download.argtypes = [C.c_void_p, C.POINTER(abi.pd_state),
                                        C.POINTER(abi.pd_force_field), C.c_int32]
        lib.pd_ctx_damage.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        lib.pd_ctx_stream.argtypes = [C.c_void_p]
        lib.pd_ctx_stream.restype = C.c_void_p
        lib.pd_ctx_launch_count.argtypes = [C.c_void_p]
        lib.pd_ctx_launch_count.restype = C.c_int64
        lib.pd_ctx_layout.argtypes = [C.c_void_p]
        lib.pd_ctx_kernel.argtypes = [C.c_void_p]
        lib.pd_ctx_kernel.restype = C.c_char_p
        lib.pd_ctx_live_bonds.argtypes = [C.c_void_p]
        lib.pd_ctx_live_bonds.restype = C.c_int64
        lib.pd_damage.argtypes = [C.POINTER(abi.pd_neighbor_list), C.POINTER(C.c_double)]
        lib.pd_ctx_upload_part.argtypes = [C.c_void_p, C.POINTER(abi.pd_bundle),
                                           C.POINTER(abi.pd_state), C.c_int32, C.c_int64,
                                           C.c_int64]
        lib.pd_ctx_internal_index.argtypes = [C.c_void_p, abi.i64p, C.c_int64, abi.i64p]
        lib.pd_ctx_export.argtypes = [C.c_void_p, C.POINTER(abi.pd_peer_handle)]
        lib.pd_ctx_connect.argtypes = [C.c_void_p, C.c_int32, C.c_int32,
                                       C.POINTER(abi.pd_peer_handle), C.c_int32, C.c_int32,
                                       abi.i64p, abi.i64p]
        lib.pd_ctx_node_values.argtypes = [C.c_void_p, abi.i64p, C.c_int64, abi.f64p]
        lib.pd_last_error.restype = C.c_char_p
        _LIB = lib
    return _LIB


# ---- binary containers (io.cpp:297-564), byte-compatible with the reference --------

def _io_lib():
    lib = library()
    lib.pd_save_state.argtypes = [C.POINTER(abi.pd_state), C.c_char_p]
    lib.pd_state_file_header.argtypes = [C.c_char_p, C.POINTER(abi.pd_file_header)]
    lib.pd_load_state.argtypes = [C.c_char_p, C.POINTER(abi.pd_state)]
    lib.pd_save_cache.argtypes = [C.POINTER(abi.pd_neighbor_list), C.POINTER(abi.pd_corrections),
                                  C.c_char_p]
    lib.pd_cache_file_header.argtypes = [C.c_char_p, C.POINTER(abi.pd_file_header)]
    lib.pd_load_cache.argtypes = [C.c_char_p, C.POINTER(abi.pd_neighbor_list),
                                  C.POINTER(abi.pd_corrections)]
    lib.pd_ctx_save_state.argtypes = [C.c_void_p, C.c_char_p]
    lib.pd_write_snapshot.argtypes = [C.POINTER(abi.pd_state), C.POINTER(abi.pd_particles),
                                      C.c_char_p]
    lib.pd_ctx_write_snapshot.argtypes = [C.c_void_p, C.c_char_p]
    lib.pd_ctx_snapshot_every.argtypes = [C.c_void_p, C.c_int64, C.c_char_p]
    return lib


def write_snapshot(state: SimulationState, particles, path: str) -> None:
    """io::write_snapshot(io::make_snapshot(state, particles)) (io.cpp:235-269)."""
    lib = _io_lib()
    m = Marshal()
    st = m.state(state)
    p = m.particles(particles)
    check(lib.pd_write_snapshot(C.byref(st), C.byref(p), os.fsencode(path)), lib.pd_last_error)


def save_state(state: SimulationState, path: str) -> None:
    """io::save_state (io.cpp:485-505): a PDST restart file."""
    lib = _io_lib()
    st = Marshal().state(state)
    check(lib.pd_save_state(C.byref(st), os.fsencode(path)), lib.pd_last_error)


def load_state(path: str) -> SimulationState:
    """io::load_state (io.cpp:507-562)."""
    from .types import NeighborList
    lib = _io_lib()
    h = abi.pd_file_header()
    check(lib.pd_state_file_header(os.fsencode(path), C.byref(h)), lib.pd_last_error)
    n, N = int(h.n), int(h.group_size)
    fam = NeighborList(np.zeros(n * N, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int32), N,
                       float(h.horizon), np.zeros(n * N if h.has_bond_type else 0, np.uint8))
    st = SimulationState(np.zeros(3 * n), np.zeros(3 * n), np.zeros(3 * n), 0, fam,
                         np.zeros(n * N if h.has_history else 0))
    m = Marshal()
    ps = m.state(st)
    check(lib.pd_load_state(os.fsencode(path), C.byref(ps)), lib.pd_last_error)
    st.step = int(ps.step)
    fam.horizon = float(ps.connectivity.horizon)
    if not h.has_bond_type:
        fam.bond_type = None
    return st


def save_cache(family, corrections, path: str) -> None:
    """io::save_cache (io.cpp:416-434): a PDNL family cache."""
    lib = _io_lib()
    m = Marshal()
    f = m.family(family)
    c = m.corrections(corrections)
    check(lib.pd_save_cache(C.byref(f), C.byref(c), os.fsencode(path)), lib.pd_last_error)


def load_cache(path: str):
    """io::load_cache (io.cpp:436-483) -> (NeighborList, Corrections)."""
    from .types import Corrections, NeighborList
    lib = _io_lib()
    h = abi.pd_file_header()
    check(lib.pd_cache_file_header(os.fsencode(path), C.byref(h)), lib.pd_last_error)
    n, N = int(h.n), int(h.group_size)
    fam = NeighborList(np.zeros(n * N, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int32), N,
                       float(h.horizon), np.zeros(n * N if h.has_bond_type else 0, np.uint8))
    corr = Corrections(np.zeros(n * N) if h.has_lambda else None,
                       np.zeros(n * N) if h.has_beta else None, None)
    m = Marshal()
    f = m.family(fam)
    c = m.corrections(corr)
    check(lib.pd_load_cache(os.fsencode(path), C.byref(f), C.byref(c)), lib.pd_last_error)
    fam.horizon = float(f.horizon)
    if not h.has_bond_type:
        fam.bond_type = None
    return fam, corr


def backend() -> Backend:
    global _BACKEND
    if _BACKEND is None:
        _BACKEND = Backend(library(), "pd_")
    return _BACKEND


def device_count() -> int:
    return int(library().pd_device_count())


def compute_forces(variant, state, particles, model, corrections, out) -> None:
    """compute_forces(KernelVariant, ...) on the B200 (engine.cpp:163-169)."""
    backend().compute_forces(variant, state, particles, model, corrections, out)


def simulate(bundle, state, options, on_write=None) -> SimulateResult:
    """simulate(bundle, state, options, on_write) on the B200 (engine.cpp:374-425)."""
    return backend().simulate(bundle, state, options, on_write)


def simulate_batch(bundles, states, options, threads: int = 0):
    """Independent simulate() calls run concurrently on one GPU
    (pd_simulate_batch): the calibration / UQ outer loop.  Returns one
    SimulateResult per model; raises the first model's error."""
    lib = library()
    k = len(bundles)
    if not (len(states) == len(options) == k):
        raise abi.InvalidArgument("simulate_batch: bundles, states and options differ in length")
    lib.pd_simulate_batch.argtypes = [C.c_int32, C.POINTER(abi.pd_bundle), C.POINTER(abi.pd_state),
                                      C.POINTER(abi.pd_options), C.POINTER(abi.pd_tip_record),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int32), C.c_int32]
    m = Marshal()
    B = (abi.pd_bundle * max(k, 1))()
    S = (abi.pd_state * max(k, 1))()
    O = (abi.pd_options * max(k, 1))()
    offsets = (C.c_int64 * (k + 1))()
    names_per = []
    total = 0
    for q, (b, st, o) in enumerate(zip(bundles, states, options)):
        n = b.particles.size()
        slots = st.size() * int(st.connectivity.group_size)
        if b.model.needs_history() and np.asarray(
                st.bond_history if st.bond_history is not None else []).size != slots:
            st.bond_history = np.zeros(slots)  # engine.cpp:382-384
        B[q] = m.bundle(b)
        S[q] = m.state(st)
        O[q] = Marshal.options(o)
        names = sorted(b.bc.tip_sets)
        writes = 0
        if o.write_every > 0:
            writes = sum(1 for s_ in range(o.first_step, o.first_step + o.steps)
                         if (s_ + 1) % o.write_every == 0)
        offsets[q] = total
        total += writes * len(names)
        names_per.append(names)
        del n
    offsets[k] = total
    recs = (abi.pd_tip_record * max(total, 1))()
    got = (C.c_int64 * max(k, 1))()
    status = (C.c_int32 * max(k, 1))()
    rc = lib.pd_simulate_batch(k, B, S, O, recs, offsets, got, status, int(threads))
    for q, st in enumerate(states):
        st.step = S[q].step
    check(rc, lib.pd_last_error)
    results = []
    for q in range(k):
        names = names_per[q]
        res = SimulateResult({name: [] for name in names} if names else {})
        for r_ in range(got[q]):
            r = recs[offsets[q] + r_]
            res.tips[names[r_ % len(names)]].append(
                TipRecord(int(r.step), np.array(r.mean_u[:]), np.array(r.mean_v[:]),
                          np.array(r.mean_a[:]), np.array(r.body_force_sum[:]),
                          np.array(r.external_force_sum[:])))
        results.append(res)
    return results


def local_damage(family) -> np.ndarray:
    """phi_i = 1 - n_neigh_i / initial_i per node (formulas.hpp:49-55), on the GPU."""
    lib = library()
    m = Marshal()
    f = m.family(family)
    phi = np.zeros(family.node_count())
    check(lib.pd_damage(C.byref(f), phi.ctypes.data_as(C.POINTER(C.c_double))),
          lib.pd_last_error)
    return phi


class Context:
    """A device-resident model + state (pd_ctx): upload once, advance many
    steps with no host traffic except at write steps, download on demand."""

    def __init__(self, device: int = 0):
        self.lib = library()
        h = C.c_void_p()
        check(self.lib.pd_ctx_create(device, C.byref(h)), self.lib.pd_last_error)
        self.h = h
        self.n = 0
        self.N = 0
        self.history = False

    def close(self) -> None:
        if self.h:
            self.lib.pd_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        check(rc, self.lib.pd_last_error)

    def upload(self, bundle: ModelBundle, state: SimulationState,
               variant: KernelVariant = KernelVariant.bond_parallel) -> None:
        m = Marshal()
        b = m.bundle(bundle)
        st = m.state(state)
        self._check(self.lib.pd_ctx_upload(self.h, C.byref(b), C.byref(st), int(variant)))
        self.n = state.size()
        self.N = int(state.connectivity.group_size)
        self.history = bundle.model.needs_history()
        self.tip_names = sorted(bundle.bc.tip_sets)

    # ---- multi-GPU slab parts (pd_b200.h "multi-GPU z-slabs") -------------

    def upload_part(self, bundle: ModelBundle, state: SimulationState, variant,
                    own_begin: int, own_end: int) -> None:
        m = Marshal()
        b = m.bundle(bundle)
        st = m.state(state)
        self._check(self.lib.pd_ctx_upload_part(self.h, C.byref(b), C.byref(st), int(variant),
                                                int(own_begin), int(own_end)))
        self.n = state.size()
        self.N = int(state.connectivity.group_size)
        self.history = bundle.model.needs_history()
        self.tip_names = sorted(bundle.bc.tip_sets)

    def internal_index(self, local: np.ndarray) -> np.ndarray:
        local = np.ascontiguousarray(local, dtype=np.int64)
        out = np.empty_like(local)
        self._check(self.lib.pd_ctx_internal_index(self.h, abi.ptr(local, C.c_int64), local.size,
                                                   abi.ptr(out, C.c_int64)))
        return out

    def export(self) -> bytes:
        h = abi.pd_peer_handle()
        self._check(self.lib.pd_ctx_export(self.h, C.byref(h)))
        return bytes(h)

    def connect(self, rank: int, world: int, handles, lo: int, hi: int,
                send_lo: Optional[np.ndarray], send_hi: Optional[np.ndarray]) -> None:
        arr = (abi.pd_peer_handle * world)()
        for k, hb in enumerate(handles):
            C.memmove(C.byref(arr[k]), hb, C.sizeof(abi.pd_peer_handle))
        keep = []

        def p64(a):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=np.int64)
            keep.append(a)
            return abi.ptr(a, C.c_int64)
        self._check(self.lib.pd_ctx_connect(self.h, int(rank), int(world), arr, int(lo), int(hi),
                                            p64(send_lo), p64(send_hi)))

    def node_values(self, local: np.ndarray) -> np.ndarray:
        """u, v, a, body_force*V, external_force*V of local nodes (k x 15)."""
        local = np.ascontiguousarray(local, dtype=np.int64)
        out = np.empty((local.size, 15))
        if local.size:
            self._check(self.lib.pd_ctx_node_values(self.h, abi.ptr(local, C.c_int64),
                                                     local.size, abi.ptr(out, C.c_double)))
        return out

    def run(self, steps: int, first_step: int, integrator=IntegratorKind.velocity_verlet,
            write_every: int = 0, variant=KernelVariant.bond_parallel) -> SimulateResult:
        opts = abi.pd_options(int(steps), int(write_every), int(first_step), int(integrator),
                              int(variant))
        names = self.tip_names
        writes = 0
        if write_every > 0:
            writes = sum(1 for s in range(first_step, first_step + steps)
                         if (s + 1) % write_every == 0)
        cap = max(1, writes * len(names))
        recs = (abi.pd_tip_record * cap)()
        n_recs = C.c_int64(0)
        self._check(self.lib.pd_ctx_run(self.h, C.byref(opts), HOOK(), None, 0, recs, cap,
                                        C.byref(n_recs)))
        result = SimulateResult({name: [] for name in names})
        for k in range(n_recs.value):
            r = recs[k]
            result.tips[names[k % len(names)]].append(
                TipRecord(int(r.step), np.array(r.mean_u[:]), np.array(r.mean_v[:]),
                          np.array(r.mean_a[:]), np.array(r.body_force_sum[:]),
                          np.array(r.external_force_sum[:])))
        return result

    def compute_forces(self) -> None:
        self._check(self.lib.pd_ctx_compute_forces(self.h))

    def download(self, state: SimulationState, forces: Optional[ForceField] = None,
                 fields: int = abi.PD_FIELD_ALL) -> None:
        m = Marshal()
        if self.history and np.asarray(state.bond_history).size != self.n * self.N:
            state.bond_history = np.zeros(self.n * self.N)
        st = m.state(state)
        if forces is not None:
            forces.resize(self.n)
            ff = m.forces(forces)
            fp = C.byref(ff)
        else:
            fp = None
            fields &= ~abi.PD_FIELD_FORCES
        self._check(self.lib.pd_ctx_download(self.h, C.byref(st), fp, int(fields)))
        state.step = st.step

    def damage(self) -> np.ndarray:
        phi = np.zeros(self.n)
        self._check(self.lib.pd_ctx_damage(self.h, phi.ctypes.data_as(C.POINTER(C.c_double))))
        return phi

    def stream(self) -> int:
        return int(self.lib.pd_ctx_stream(self.h) or 0)

    def save_state(self, path: str) -> None:
        """io::save_state of the resident state, streamed from device memory."""
        lib = _io_lib()
        self._check(lib.pd_ctx_save_state(self.h, os.fsencode(path)))

    def write_snapshot(self, path: str) -> None:
        """The pdsnap file of the resident state."""
        self._check(_io_lib().pd_ctx_write_snapshot(self.h, os.fsencode(path)))

    def snapshot_every(self, every: int, pattern: str) -> None:
        """Asynchronous pdsnap files during run(): pattern % step every `every` steps."""
        self._check(_io_lib().pd_ctx_snapshot_every(self.h, int(every), pattern.encode()))

    def layout(self) -> str:
        """"exact", "tiles" or "lattice" (pd_ctx_layout)."""
        return ("exact", "tiles", "lattice")[self.lib.pd_ctx_layout(self.h)]

    def kernel(self) -> str:
        """The step kernel instantiation the last step launched (pd_ctx_kernel),
        e.g. "lattice_step_kernel<1,8,3,0,0>"."""
        return self.lib.pd_ctx_kernel(self.h).decode()

    def launch_count(self) -> int:
        return int(self.lib.pd_ctx_launch_count(self.h))

    def live_bonds(self) -> int:
        return int(self.lib.pd_ctx_live_bonds(self.h))
