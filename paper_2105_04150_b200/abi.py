"""ctypes mirror of include/pd_b200.h plus marshalling from the Python types.

The descriptor structs are shared by the product library (libpd_b200.so) and
by the test checkers under oracle/ (which take the same descriptors), so one
marshalling layer feeds the GPU, the C restatement and the compiled reference.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PD_MAX_BREAKPOINTS = 32
PD_MAX_LAWS = 256

PD_OK = 0
PD_E_INVALID_ARGUMENT = 1
PD_E_DOMAIN = 2
PD_E_RUNTIME = 3
PD_E_CUDA = 4
PD_E_NO_DEVICE = 5

PD_FIELD_U, PD_FIELD_V, PD_FIELD_A = 1, 2, 4
PD_FIELD_CONNECTIVITY, PD_FIELD_HISTORY, PD_FIELD_FORCES = 8, 16, 32
PD_FIELD_ALL = 63

i64 = C.c_int64
i32 = C.c_int32
f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)
i64p = C.POINTER(C.c_int64)


class pd_particles(C.Structure):
    _fields_ = [("n", i64), ("coords", f64p), ("coords_size", i64), ("volume", f64p),
                ("density", f64p), ("density_size", i64)]


class pd_neighbor_list(C.Structure):
    _fields_ = [("n", i64), ("group_size", i64), ("entries", i32p), ("n_neigh", i32p),
                ("initial_n_neigh", i32p), ("bond_type", u8p), ("bond_type_size", i64),
                ("horizon", C.c_double)]


class pd_law(C.Structure):
    _fields_ = [("stiffness", C.c_double), ("n_breakpoints", i32),
                ("breakpoints", C.c_double * PD_MAX_BREAKPOINTS),
                ("forces", C.c_double * PD_MAX_BREAKPOINTS)]


class pd_damage_model(C.Structure):
    _fields_ = [("laws", C.POINTER(pd_law)), ("n_laws", i32), ("damping", C.c_double)]


class pd_corrections(C.Structure):
    _fields_ = [("lambda_", f64p), ("lambda_size", i64), ("beta", f64p), ("beta_size", i64),
                ("no_failure", u8p), ("no_failure_size", i64)]


class pd_state(C.Structure):
    _fields_ = [("u", f64p), ("v", f64p), ("a", f64p), ("step", i64),
                ("connectivity", pd_neighbor_list), ("bond_history", f64p),
                ("bond_history_size", i64)]


class pd_force_field(C.Structure):
    _fields_ = [("body_force", f64p), ("external_force", f64p)]


class pd_ramp(C.Structure):
    _fields_ = [("kind", i32), ("rise_steps", i64), ("target_scale", C.c_double)]


class pd_boundary(C.Structure):
    _fields_ = [("kind", u8p), ("kind_size", i64), ("magnitude", f64p), ("magnitude_size", i64),
                ("ramp_id", u8p), ("ramp_id_size", i64), ("ramps", C.POINTER(pd_ramp)),
                ("n_ramps", i32), ("no_failure", u8p), ("no_failure_size", i64),
                ("n_tip_sets", i32), ("tip_offsets", i64p), ("tip_nodes", i64p)]


class pd_bundle(C.Structure):
    _fields_ = [("particles", pd_particles), ("model", pd_damage_model),
                ("corrections", pd_corrections), ("bc", pd_boundary), ("dt", C.c_double)]


class pd_options(C.Structure):
    _fields_ = [("steps", i64), ("write_every", i64), ("first_step", i64), ("integrator", i32),
                ("variant", i32)]


class pd_tip_record(C.Structure):
    _fields_ = [("step", i64), ("mean_u", C.c_double * 3), ("mean_v", C.c_double * 3),
                ("mean_a", C.c_double * 3), ("body_force_sum", C.c_double * 3),
                ("external_force_sum", C.c_double * 3)]


HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(pd_state), C.POINTER(pd_force_field))


# ---- errors (the reference's exception types) ---------------------------------

class pd_file_header(C.Structure):
    _fields_ = [("n", i64), ("group_size", i64), ("step", i64), ("horizon", C.c_double),
                ("has_bond_type", i32), ("has_history", i32), ("has_lambda", i32),
                ("has_beta", i32)]


PD_MAX_RANKS = 16


class pd_peer_handle(C.Structure):
    _fields_ = [("device", i32), ("pid", i32), ("ipc_u0", C.c_uint8 * 64),
                ("ipc_u1", C.c_uint8 * 64), ("ipc_sync", C.c_uint8 * 64),
                ("u0", C.c_uint64), ("u1", C.c_uint64), ("sync", C.c_uint64)]


PD_REGION_BOX, PD_REGION_CYLINDER = 0, 1
PD_PREDICATE_PLANE, PD_PREDICATE_NOTCH = 0, 1


class pd_region(C.Structure):
    _fields_ = [("kind", i32), ("axis", i32), ("cls", i32), ("pad", i32),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("c", C.c_double * 2),
                ("radius", C.c_double)]


class pd_classifier(C.Structure):
    _fields_ = [("n_classes", i32), ("default_class", i32), ("n_regions", i32), ("pad", i32),
                ("regions", C.POINTER(pd_region)), ("type_table", u8p)]


class pd_bond_predicate(C.Structure):
    _fields_ = [("kind", i32), ("axis", i32), ("sweep_axis", i32), ("pad", i32),
                ("position", C.c_double), ("depth", C.c_double)]


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ValueError):
    """std::domain_error"""


class PeridynRuntimeError(RuntimeError):
    """std::runtime_error"""


class CudaError(RuntimeError):
    """CUDA failure or no B200 visible (no reference counterpart)."""


_ERRORS = {PD_E_INVALID_ARGUMENT: InvalidArgument, PD_E_DOMAIN: DomainError,
           PD_E_RUNTIME: PeridynRuntimeError, PD_E_CUDA: CudaError, PD_E_NO_DEVICE: CudaError}


def check(rc: int, last_error) -> None:
    if rc != PD_OK:
        msg = last_error()
        if isinstance(msg, bytes):
            msg = msg.decode()
        raise _ERRORS.get(rc, RuntimeError)(msg)


# ---- array helpers -------------------------------------------------------------

def ptr(arr, ctype):
    if arr is None or arr.size == 0:
        return C.cast(None, C.POINTER(ctype))
    return arr.ctypes.data_as(C.POINTER(ctype))


def as_f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(-1))


def as_i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32).reshape(-1))


def as_u8(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint8).reshape(-1))


class Marshal:
    """Builds pd_* descriptors from the Python types and keeps every array the
    descriptors point into alive.  Mutable state arrays are normalised IN PLACE
    on the owning objects so that the library writes straight into them."""

    def __init__(self):
        self.keep = []

    def _k(self, a):
        self.keep.append(a)
        return a

    def particles(self, p) -> pd_particles:
        p.coords = as_f64(p.coords)
        p.volume = as_f64(p.volume)
        p.density = as_f64(p.density)
        return pd_particles(p.volume.size, ptr(p.coords, C.c_double), p.coords.size,
                            ptr(p.volume, C.c_double), ptr(p.density, C.c_double), p.density.size)

    def family(self, f) -> pd_neighbor_list:
        f.entries = as_i32(f.entries)
        f.n_neigh = as_i32(f.n_neigh)
        f.initial_n_neigh = as_i32(f.initial_n_neigh)
        f.bond_type = as_u8(f.bond_type if f.bond_type is not None else [])
        return pd_neighbor_list(f.n_neigh.size, int(f.group_size), ptr(f.entries, C.c_int32),
                                ptr(f.n_neigh, C.c_int32), ptr(f.initial_n_neigh, C.c_int32),
                                ptr(f.bond_type, C.c_uint8), f.bond_type.size, float(f.horizon))

    def model(self, m) -> pd_damage_model:
        if len(m.laws) > PD_MAX_LAWS:
            raise InvalidArgument(f"DamageModel: more than {PD_MAX_LAWS} laws")
        arr = (pd_law * max(1, len(m.laws)))()
        for k, law in enumerate(m.laws):
            if len(law.breakpoints) > PD_MAX_BREAKPOINTS:
                raise InvalidArgument(
                    f"DamageLaw: more than {PD_MAX_BREAKPOINTS} breakpoints is not supported")
            if len(law.breakpoints) != len(law.forces):
                raise InvalidArgument(
                    "DamageLaw: breakpoints and forces must match and be non-empty")
            arr[k].stiffness = float(law.stiffness)
            arr[k].n_breakpoints = len(law.breakpoints)
            for b, (s, f) in enumerate(zip(law.breakpoints, law.forces)):
                arr[k].breakpoints[b] = float(s)
                arr[k].forces[b] = float(f)
        self._k(arr)
        return pd_damage_model(C.cast(arr, C.POINTER(pd_law)), len(m.laws), float(m.damping))

    def corrections(self, c) -> pd_corrections:
        lam = self._k(as_f64(c.lambda_ if c.lambda_ is not None else []))
        beta = self._k(as_f64(c.beta if c.beta is not None else []))
        nf = self._k(as_u8(c.no_failure if c.no_failure is not None else []))
        return pd_corrections(ptr(lam, C.c_double), lam.size, ptr(beta, C.c_double), beta.size,
                              ptr(nf, C.c_uint8), nf.size)

    def state(self, s) -> pd_state:
        s.u = as_f64(s.u)
        s.v = as_f64(s.v)
        s.a = as_f64(s.a)
        s.bond_history = as_f64(s.bond_history if s.bond_history is not None else [])
        fam = self.family(s.connectivity)
        return pd_state(ptr(s.u, C.c_double), ptr(s.v, C.c_double), ptr(s.a, C.c_double),
                        int(s.step), fam, ptr(s.bond_history, C.c_double), s.bond_history.size)

    def forces(self, f) -> pd_force_field:
        f.body_force = as_f64(f.body_force)
        f.external_force = as_f64(f.external_force)
        return pd_force_field(ptr(f.body_force, C.c_double), ptr(f.external_force, C.c_double))

    def boundary(self, bc) -> pd_boundary:
        kind = self._k(as_u8(bc.kind))
        mag = self._k(as_f64(bc.magnitude))
        rid = self._k(as_u8(bc.ramp_id))
        nf = self._k(as_u8(bc.no_failure))
        ramps = (pd_ramp * max(1, len(bc.ramps)))()
        for k, r in enumerate(bc.ramps):
            ramps[k].kind = int(r.kind)
            ramps[k].rise_steps = int(r.rise_steps)
            ramps[k].target_scale = float(r.target_scale)
        self._k(ramps)
        names = sorted(bc.tip_sets)  # std::map order
        offs = [0]
        nodes = []
        for name in names:
            nodes.extend(int(i) for i in bc.tip_sets[name])
            offs.append(len(nodes))
        offs = self._k(np.asarray(offs, dtype=np.int64))
        nodes = self._k(np.asarray(nodes if nodes else [0], dtype=np.int64))
        return pd_boundary(ptr(kind, C.c_uint8), kind.size, ptr(mag, C.c_double), mag.size,
                           ptr(rid, C.c_uint8), rid.size, C.cast(ramps, C.POINTER(pd_ramp)),
                           len(bc.ramps), ptr(nf, C.c_uint8), nf.size, len(names),
                           offs.ctypes.data_as(i64p), nodes.ctypes.data_as(i64p))

    def bundle(self, b) -> pd_bundle:
        return pd_bundle(self.particles(b.particles), self.model(b.model),
                         self.corrections(b.corrections), self.boundary(b.bc), float(b.dt))

    @staticmethod
    def options(o) -> pd_options:
        return pd_options(int(o.steps), int(o.write_every), int(o.first_step),
                          int(o.integrator), int(o.variant))


def load(path: str, prefix: str):
    """Load a library exposing the pd-style entry points under `prefix`."""
    if not os.path.exists(path):
        raise OSError(f"library not built: {path}")
    return C.CDLL(path)
