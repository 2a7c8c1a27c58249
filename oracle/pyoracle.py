"""TEST INFRASTRUCTURE ONLY: Python handles on the checkers.

  COracle   -- oracle/_build/libpd_oracle.so, the plain-C restatement
  Reference -- oracle/_ref/libperidyn_ref.so, the unmodified reference
               compiled from /root/reference/proj/src (may be absent on the
               GPU box if it was not built here)

Both take the same pd_* descriptors as the product (paper_2105_04150_b200.abi),
so tests drive product and checker through identical code.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2105_04150_b200 import abi
from paper_2105_04150_b200.engine import Backend
from paper_2105_04150_b200.types import (DamageLaw, DamageModel, Corrections, NeighborList,
                                         ParticleSet, SimulationState)

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libpd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libperidyn_ref.so")


def ensure_built() -> None:
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(
            os.path.join(HERE, "pd_oracle.c")):
        subprocess.run(["make", "-s", "-C", HERE, os.path.join(HERE, "_build", "libpd_oracle.so")],
                       check=True)


def _family_from(lib, prefix, coords, horizon, hint):
    fn = getattr(lib, prefix + "build_family")
    fn.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_double, C.POINTER(C.c_double),
                   C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.POINTER(C.c_int32)),
                   C.POINTER(C.POINTER(C.c_int32)), C.POINTER(C.c_int64)]
    free = getattr(lib, prefix + "free")
    free.argtypes = [C.c_void_p]
    coords = abi.as_f64(coords)
    n = coords.size // 3
    e, nn, ini = C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)()
    g = C.c_int64()
    hint_arr = None if hint is None else np.asarray(hint, dtype=np.float64)
    rc = fn(abi.ptr(coords, C.c_double), n, float(horizon),
            abi.ptr(hint_arr, C.c_double) if hint_arr is not None else None,
            C.byref(e), C.byref(nn), C.byref(ini), C.byref(g))
    last = getattr(lib, prefix + "last_error")
    last.restype = C.c_char_p
    abi.check(rc, last)
    N = g.value
    out = NeighborList(np.ctypeslib.as_array(e, (n * N,)).copy(),
                       np.ctypeslib.as_array(nn, (n,)).copy(),
                       np.ctypeslib.as_array(ini, (n,)).copy(), N, float(horizon), None)
    for p in (e, nn, ini):
        free(C.cast(p, C.c_void_p))
    return out


class COracle(Backend):
    def __init__(self, threads: int = 1):
        ensure_built()
        lib = C.CDLL(ORACLE_SO)
        super().__init__(lib, "orc_")
        lib.orc_set_threads(int(threads))
        lib.orc_ramp_scale.restype = C.c_double
        lib.orc_ramp_rate.restype = C.c_double
        lib.orc_ramp_accel.restype = C.c_double
        for f in ("orc_ramp_scale", "orc_ramp_rate", "orc_ramp_accel"):
            getattr(lib, f).argtypes = [C.POINTER(abi.pd_ramp), C.c_int64]

    def set_threads(self, t: int) -> None:
        self.lib.orc_set_threads(int(t))

    def build_family(self, coords, horizon, hint=None) -> NeighborList:
        return _family_from(self.lib, "orc_", coords, horizon, hint)

    def reduce_group(self, values: np.ndarray):
        v = abi.as_f64(values).copy()
        out = (C.c_double * 3)()
        self.lib.orc_reduce_group.argtypes = [C.POINTER(C.c_double), C.c_int64,
                                              C.POINTER(C.c_double)]
        self._check(self.lib.orc_reduce_group(abi.ptr(v, C.c_double), v.size // 3, out))
        return np.array(out[:])

    def damage(self, family: NeighborList) -> np.ndarray:
        m = abi.Marshal()
        f = m.family(family)
        phi = np.zeros(family.node_count())
        self._check(self.lib.orc_damage(C.byref(f), abi.ptr(phi, C.c_double)))
        return phi

    def ramp(self, which: str, kind: int, rise: int, target: float, step: int) -> float:
        r = abi.pd_ramp(int(kind), int(rise), float(target))
        return getattr(self.lib, "orc_ramp_" + which)(C.byref(r), int(step))

    def break_plane(self, family, coords, axis, position):
        m = abi.Marshal()
        f = m.family(family)
        c = abi.as_f64(coords)
        self.lib.orc_break_plane.argtypes = [C.POINTER(abi.pd_neighbor_list),
                                             C.POINTER(C.c_double), C.c_int, C.c_double]
        self.lib.orc_break_plane(C.byref(f), abi.ptr(c, C.c_double), int(axis), float(position))

    def break_notch(self, family, coords, axis, position, sweep_axis, depth):
        m = abi.Marshal()
        f = m.family(family)
        c = abi.as_f64(coords)
        self.lib.orc_break_notch.argtypes = [C.POINTER(abi.pd_neighbor_list),
                                             C.POINTER(C.c_double), C.c_int, C.c_double,
                                             C.c_int, C.c_double]
        self.lib.orc_break_notch(C.byref(f), abi.ptr(c, C.c_double), int(axis), float(position),
                                 int(sweep_axis), float(depth))


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference(Backend):
    """The compiled reference (oracle/_ref).  Raises OSError if not built."""

    def __init__(self, threads: int = 0):
        if not reference_available():
            raise OSError(f"reference library not built: {REF_SO}")
        lib = C.CDLL(REF_SO)
        super().__init__(lib, "ref_")
        lib.ref_set_threads(int(threads))
        lib.ref_random_config.restype = C.c_void_p
        lib.ref_random_config.argtypes = [C.c_uint]
        lib.ref_random_free.argtypes = [C.c_void_p]
        lib.ref_random_field.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_int64)]
        lib.ref_random_group_size.argtypes = [C.c_void_p]
        lib.ref_random_group_size.restype = C.c_int64
        lib.ref_random_horizon.argtypes = [C.c_void_p]
        lib.ref_random_horizon.restype = C.c_double
        lib.ref_random_law.argtypes = [C.c_void_p, C.POINTER(abi.pd_law)]
        lib.ref_ramp.restype = C.c_double
        lib.ref_ramp.argtypes = [C.c_int32, C.POINTER(abi.pd_ramp), C.c_int64]
        lib.ref_bench_lattice.argtypes = [C.POINTER(C.c_int64), C.c_double, C.c_double, C.c_int64,
                                          C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_double)]
        lib.ref_worker_count.restype = C.c_uint

    def set_threads(self, t: int) -> None:
        self.lib.ref_set_threads(int(t))

    def build_family(self, coords, horizon, hint=None) -> NeighborList:
        return _family_from(self.lib, "ref_", coords, horizon, hint)

    def build_family_classified(self, coords, horizon, hint, classifier):
        """build_family(coords, horizon, hint, classify) of the reference with a
        BondClassifier lambda applying `classifier`'s region rules
        (geometry.py RuleClassifier): (entries, bond_type, group_size)."""
        fn = self.lib.ref_build_family_classified
        fn.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_double, C.POINTER(C.c_double),
                       C.POINTER(abi.pd_classifier), C.POINTER(C.POINTER(C.c_int32)),
                       C.POINTER(C.POINTER(C.c_uint8)), C.POINTER(C.c_int64)]
        self.lib.ref_free.argtypes = [C.c_void_p]
        coords = abi.as_f64(coords)
        n = coords.size // 3
        keep: list = []
        cls = classifier.descriptor(keep)
        e, t = C.POINTER(C.c_int32)(), C.POINTER(C.c_uint8)()
        g = C.c_int64()
        hint_arr = None if hint is None else np.asarray(hint, dtype=np.float64)
        self._check(fn(abi.ptr(coords, C.c_double), n, float(horizon),
                       abi.ptr(hint_arr, C.c_double) if hint_arr is not None else None,
                       C.byref(cls), C.byref(e), C.byref(t), C.byref(g)))
        try:
            N = int(g.value)
            entries = np.ctypeslib.as_array(e, shape=(n * N,)).copy()
            types = np.ctypeslib.as_array(t, shape=(n * N,)).copy()
        finally:
            self.lib.ref_free(e)
            self.lib.ref_free(t)
        return entries, types, N

    def neighborhood_volumes(self, volumes, family) -> np.ndarray:
        self.lib.ref_neighborhood_volumes.argtypes = [C.POINTER(C.c_double),
                                                      C.POINTER(abi.pd_neighbor_list),
                                                      C.POINTER(C.c_double)]
        m = abi.Marshal()
        f = m.family(family)
        v = abi.as_f64(volumes)
        out = np.empty(family.node_count())
        self._check(self.lib.ref_neighborhood_volumes(abi.ptr(v, C.c_double), C.byref(f),
                                                      abi.ptr(out, C.c_double)))
        return out

    def surface_correction_factors(self, volumes, family, v0) -> np.ndarray:
        self.lib.ref_surface_correction_factors.argtypes = [
            C.POINTER(C.c_double), C.POINTER(abi.pd_neighbor_list), C.c_double,
            C.POINTER(C.c_double)]
        m = abi.Marshal()
        f = m.family(family)
        v = abi.as_f64(volumes)
        out = np.empty(family.entries.size)
        self._check(self.lib.ref_surface_correction_factors(abi.ptr(v, C.c_double), C.byref(f),
                                                            float(v0), abi.ptr(out, C.c_double)))
        return out

    def break_bonds(self, family, coords, kind, axis, position, sweep_axis=0, depth=0.0):
        """break_initial_bonds with plane_crossing_predicate (kind 0) or
        notch_predicate (kind 1) of the reference, in place."""
        self.lib.ref_break_bonds.argtypes = [C.POINTER(abi.pd_neighbor_list),
                                             C.POINTER(C.c_double), C.c_int, C.c_int,
                                             C.c_double, C.c_int, C.c_double]
        m = abi.Marshal()
        f = m.family(family)
        c = abi.as_f64(coords)
        self.lib.ref_break_bonds(C.byref(f), abi.ptr(c, C.c_double), int(kind), int(axis),
                                 float(position), int(sweep_axis), float(depth))

    def save_state(self, state, path: str) -> None:
        """io::save_state of the reference."""
        self.lib.ref_save_state.argtypes = [C.POINTER(abi.pd_state), C.c_char_p]
        st = abi.Marshal().state(state)
        self._check(self.lib.ref_save_state(C.byref(st), os.fsencode(path)))

    def write_snapshot(self, state, particles, path: str) -> None:
        """io::write_snapshot(io::make_snapshot(state, particles)) of the reference."""
        self.lib.ref_write_snapshot.argtypes = [C.POINTER(abi.pd_state),
                                                C.POINTER(abi.pd_particles), C.c_char_p]
        m = abi.Marshal()
        st = m.state(state)
        p = m.particles(particles)
        self._check(self.lib.ref_write_snapshot(C.byref(st), C.byref(p), os.fsencode(path)))

    def save_cache(self, family, corrections, path: str) -> None:
        """io::save_cache of the reference."""
        self.lib.ref_save_cache.argtypes = [C.POINTER(abi.pd_neighbor_list),
                                            C.POINTER(abi.pd_corrections), C.c_char_p]
        m = abi.Marshal()
        f = m.family(family)
        c = m.corrections(corrections)
        self._check(self.lib.ref_save_cache(C.byref(f), C.byref(c), os.fsencode(path)))

    def ramp(self, which: str, kind: int, rise: int, target: float, step: int) -> float:
        r = abi.pd_ramp(int(kind), int(rise), float(target))
        return self.lib.ref_ramp({"scale": 0, "rate": 1, "accel": 2}[which], C.byref(r), int(step))

    def random_config(self, seed: int):
        """oracles::make_random_config(seed) (tests/oracles.hpp:140-210)."""
        h = self.lib.ref_random_config(int(seed))
        try:
            def field(name, dtype):
                p = C.c_void_p()
                cnt = C.c_int64()
                assert self.lib.ref_random_field(h, name.encode(), C.byref(p), C.byref(cnt)) == 0
                if cnt.value == 0:
                    return np.zeros(0, dtype=dtype)
                buf = (C.c_char * (cnt.value * np.dtype(dtype).itemsize)).from_address(p.value)
                return np.frombuffer(buf, dtype=dtype).copy()
            law = abi.pd_law()
            self.lib.ref_random_law(h, C.byref(law))
            nbp = law.n_breakpoints
            dl = DamageLaw(law.stiffness, list(law.breakpoints[:nbp]), list(law.forces[:nbp]))
            N = int(self.lib.ref_random_group_size(h))
            horizon = float(self.lib.ref_random_horizon(h))
            n_neigh = field("n_neigh", np.int32)
            fam = NeighborList(field("entries", np.int32), n_neigh, field("initial_n_neigh", np.int32),
                               N, horizon, None)
            n = n_neigh.size
            particles = ParticleSet(field("coords", np.float64), field("volume", np.float64),
                                    field("density", np.float64), np.zeros(n, np.uint16))
            state = SimulationState(field("u", np.float64), np.zeros(3 * n), np.zeros(3 * n), 0,
                                    fam, field("bond_history", np.float64))
            corr = Corrections(field("lambda", np.float64), field("beta", np.float64), None)
            return particles, DamageModel([dl]), corr, state
        finally:
            self.lib.ref_random_free(h)

    def bench_lattice_runs(self, dims, horizon: float, s_c: float, run_steps, threads,
                           law: int = 0):
        """ref_bench_lattice_runs: the bench fixture built once, then one
        simulate() call per entry of run_steps on threads[r] workers (0 = all),
        continuing the same state.  Returns (seconds per run, live bonds at
        the start, family build seconds)."""
        k = len(run_steps)
        d = (C.c_int64 * 3)(*[int(x) for x in dims])
        rs = (C.c_int64 * k)(*[int(x) for x in run_steps])
        th = (C.c_int * k)(*[int(x) for x in threads])
        secs = (C.c_double * k)()
        live = C.c_int64()
        build = C.c_double()
        self.lib.ref_bench_lattice_runs.argtypes = [
            C.POINTER(C.c_int64), C.c_double, C.c_double, C.c_int, C.POINTER(C.c_int64),
            C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64),
            C.POINTER(C.c_double)]
        self._check(self.lib.ref_bench_lattice_runs(d, float(horizon), float(s_c), int(law), rs,
                                                    th, k,
                                                    secs, C.byref(live), C.byref(build)))
        return list(secs), live.value, build.value

    def bench_lattice(self, dims, horizon: float, s_c: float, steps: int, threads: int):
        d = (C.c_int64 * 3)(*[int(x) for x in dims])
        secs = C.c_double()
        live = C.c_int64()
        build = C.c_double()
        self._check(self.lib.ref_bench_lattice(d, float(horizon), float(s_c), int(steps),
                                               int(threads), C.byref(secs), C.byref(live),
                                               C.byref(build)))
        return secs.value, live.value, build.value
