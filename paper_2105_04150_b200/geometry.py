"""Setup-time geometry mirroring include/peridyn/geometry.hpp.

build_family runs on the B200 (csrc/pd_family.cu) and reproduces the
reference's cell-list rows exactly; so do the setup passes over a family
(csrc/pd_family_ops.cu): the bond classifier (as a rule table), neighbourhood
volumes, surface-correction factors and pre-crack predicates.
grid_coordinates is an O(n) host array expression with the reference's
operation order (not on the time-step path).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import abi
from .engine import library
from .types import NeighborList


@dataclass
class GridDesc:
    """geometry.hpp:14-21"""
    origin: Sequence[float] = (0.0, 0.0, 0.0)
    spacing: float = 0.0
    counts: Sequence[int] = (0, 0, 0)

    def node_count(self) -> int:
        return int(self.counts[0]) * int(self.counts[1]) * int(self.counts[2])

    def hint(self) -> np.ndarray:
        return np.array([*map(float, self.origin), float(self.spacing),
                         *map(float, self.counts)], dtype=np.float64)


def grid_coordinates(grid: GridDesc) -> np.ndarray:
    """geometry.cpp:25-38: x fastest, flat n x 3, origin + k * spacing."""
    if not grid.spacing > 0 or min(int(c) for c in grid.counts) < 1:
        raise abi.InvalidArgument("grid: spacing and counts must be positive")
    nx, ny, nz = (int(c) for c in grid.counts)
    kz, ky, kx = np.meshgrid(np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
                             np.arange(nx, dtype=np.float64), indexing="ij")
    out = np.empty((nz, ny, nx, 3))
    out[..., 0] = grid.origin[0] + kx * grid.spacing
    out[..., 1] = grid.origin[1] + ky * grid.spacing
    out[..., 2] = grid.origin[2] + kz * grid.spacing
    return out.reshape(-1)


@dataclass
class Region:
    """One classifier rule: an axis-aligned box (inclusive bounds), or a
    cylinder along `axis` with centre `center` in the two other axes (in
    ascending axis order), `radius`, and extent [lo[axis], hi[axis]]."""
    cls: int
    kind: str = "box"
    lo: Sequence[float] = (-math.inf, -math.inf, -math.inf)
    hi: Sequence[float] = (math.inf, math.inf, math.inf)
    axis: int = 0
    center: Sequence[float] = (0.0, 0.0)
    radius: float = 0.0

    def contains(self, x: np.ndarray) -> np.ndarray:
        """Host evaluation (same expression order as the device)."""
        x = np.asarray(x, dtype=np.float64).reshape(-1, 3)
        if self.kind == "box":
            return np.all((x >= np.asarray(self.lo)) & (x <= np.asarray(self.hi)), axis=1)
        a = self.axis
        b0, b1 = (1, 2) if a == 0 else ((0, 2) if a == 1 else (0, 1))
        inside = (x[:, a] >= self.lo[a]) & (x[:, a] <= self.hi[a])
        d0 = x[:, b0] - self.center[0]
        d1 = x[:, b1] - self.center[1]
        return inside & (d0 * d0 + d1 * d1 <= self.radius * self.radius)


@dataclass
class RuleClassifier:
    """A BondClassifier (geometry.hpp:45-54) as a rule table: a node's class is
    that of the last region containing it (else `default_class`); the bond
    type of (i, j) is table[class_i][class_j] (must be symmetric, as the
    reference requires of a classifier)."""
    table: np.ndarray
    regions: List[Region] = field(default_factory=list)
    default_class: int = 0

    def descriptor(self, keep: list) -> abi.pd_classifier:
        table = np.ascontiguousarray(np.asarray(self.table, dtype=np.uint8))
        nc = table.shape[0]
        regs = (abi.pd_region * max(1, len(self.regions)))()
        for k, r in enumerate(self.regions):
            regs[k] = abi.pd_region(abi.PD_REGION_BOX if r.kind == "box" else abi.PD_REGION_CYLINDER,
                                    int(r.axis), int(r.cls), 0, (C.c_double * 3)(*r.lo),
                                    (C.c_double * 3)(*r.hi), (C.c_double * 2)(*r.center),
                                    float(r.radius))
        keep += [table, regs]
        return abi.pd_classifier(nc, int(self.default_class), len(self.regions), 0, regs,
                                 abi.ptr(table.reshape(-1), C.c_uint8))

    def node_classes(self, coords: np.ndarray) -> np.ndarray:
        x = np.asarray(coords, dtype=np.float64).reshape(-1, 3)
        out = np.full(x.shape[0], self.default_class, dtype=np.int64)
        for r in self.regions:
            out[r.contains(x)] = r.cls
        return out


def build_family(coords: np.ndarray, horizon: float,
                 grid_hint: Optional[GridDesc] = None,
                 classify: Optional[RuleClassifier] = None) -> NeighborList:
    """build_family (geometry.cpp:97-211) on the device; with `classify`, the
    bond types pack_rows assigns (geometry.cpp:147-158), also on the device."""
    fam = _build_family(coords, horizon, grid_hint)
    if classify is not None:
        fam.bond_type = classify_bonds(coords, fam, classify)
    return fam


def classify_bonds(coords: np.ndarray, family: NeighborList,
                   classify: RuleClassifier) -> np.ndarray:
    """bond_type (n x N, 0 on padding) of `family` under a rule-table classifier."""
    lib = library()
    lib.pd_classify_bonds.argtypes = [C.POINTER(C.c_double), C.POINTER(abi.pd_neighbor_list),
                                      C.POINTER(abi.pd_classifier), C.POINTER(C.c_uint8)]
    m = abi.Marshal()
    keep: list = []
    f = m.family(family)
    c = abi.as_f64(coords)
    cls = classify.descriptor(keep)
    out = np.zeros(family.entries.size, dtype=np.uint8)
    abi.check(lib.pd_classify_bonds(abi.ptr(c, C.c_double), C.byref(f), C.byref(cls),
                                    abi.ptr(out, C.c_uint8)), lib.pd_last_error)
    return out


def neighborhood_volumes(volumes: np.ndarray, family: NeighborList) -> np.ndarray:
    """neighborhood_volumes (geometry.cpp:238-252) on the device."""
    lib = library()
    lib.pd_neighborhood_volumes.argtypes = [C.POINTER(C.c_double),
                                            C.POINTER(abi.pd_neighbor_list),
                                            C.POINTER(C.c_double)]
    m = abi.Marshal()
    f = m.family(family)
    v = abi.as_f64(volumes)
    out = np.empty(family.node_count(), dtype=np.float64)
    abi.check(lib.pd_neighborhood_volumes(abi.ptr(v, C.c_double), C.byref(f),
                                          abi.ptr(out, C.c_double)), lib.pd_last_error)
    return out


def max_neighborhood_volume(volumes: np.ndarray, family: NeighborList) -> float:
    """max_neighborhood_volume (geometry.cpp:254-261)."""
    nb = neighborhood_volumes(volumes, family)
    return float(max(0.0, nb.max())) if nb.size else 0.0


def analytic_neighborhood_volume(horizon: float, packing: float = 1.0) -> float:
    """analytic_neighborhood_volume (geometry.cpp:231-236), same operation order."""
    if not (horizon > 0) or not (packing > 0):
        raise abi.DomainError("analytic_neighborhood_volume: inputs must be positive")
    return packing * 4.0 / 3.0 * math.pi * horizon * horizon * horizon


def surface_correction_factors(volumes: np.ndarray, family: NeighborList, v0: float) -> np.ndarray:
    """surface_correction_factors (geometry.cpp:263-283) on the device:
    lambda_ij = 2 V0 / (V_i + V_j) per live slot, 1 on padding."""
    lib = library()
    lib.pd_surface_correction_factors.argtypes = [C.POINTER(C.c_double),
                                                  C.POINTER(abi.pd_neighbor_list), C.c_double,
                                                  C.POINTER(C.c_double)]
    m = abi.Marshal()
    f = m.family(family)
    v = abi.as_f64(volumes)
    out = np.empty(family.entries.size, dtype=np.float64)
    abi.check(lib.pd_surface_correction_factors(abi.ptr(v, C.c_double), C.byref(f), float(v0),
                                                abi.ptr(out, C.c_double)), lib.pd_last_error)
    return out


def _build_family(coords: np.ndarray, horizon: float,
                  grid_hint: Optional[GridDesc] = None) -> NeighborList:
    """build_family (geometry.cpp:97-211) on the device."""
    lib = library()
    lib.pd_build_family.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_double,
                                    C.POINTER(C.c_double), C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_int64)]
    lib.pd_family_download.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32)]
    lib.pd_family_free.argtypes = [C.c_void_p]
    coords = abi.as_f64(coords)
    n = coords.size // 3
    hint = grid_hint.hint() if grid_hint is not None else None
    h = C.c_void_p()
    group = C.c_int64(0)
    abi.check(lib.pd_build_family(abi.ptr(coords, C.c_double), n, float(horizon),
                                  abi.ptr(hint, C.c_double) if hint is not None else None,
                                  C.byref(h), C.byref(group)), lib.pd_last_error)
    try:
        entries = np.empty(n * group.value, dtype=np.int32)
        n_neigh = np.empty(n, dtype=np.int32)
        initial = np.empty(n, dtype=np.int32)
        abi.check(lib.pd_family_download(h, abi.ptr(entries, C.c_int32), abi.ptr(n_neigh, C.c_int32),
                                         abi.ptr(initial, C.c_int32)), lib.pd_last_error)
    finally:
        lib.pd_family_free(h)
    return NeighborList(entries, n_neigh, initial, int(group.value), float(horizon), None)


def _break(family: NeighborList, coords: np.ndarray, pred: abi.pd_bond_predicate) -> None:
    lib = library()
    lib.pd_break_initial_bonds.argtypes = [C.POINTER(abi.pd_neighbor_list),
                                           C.POINTER(C.c_double),
                                           C.POINTER(abi.pd_bond_predicate)]
    m = abi.Marshal()
    f = m.family(family)
    c = abi.as_f64(coords)
    abi.check(lib.pd_break_initial_bonds(C.byref(f), abi.ptr(c, C.c_double), C.byref(pred)),
              lib.pd_last_error)


def break_plane(family: NeighborList, coords: np.ndarray, axis: int, position: float) -> None:
    """break_initial_bonds(plane_crossing_predicate(axis, position)) (geometry.cpp:285-306),
    on the device."""
    _break(family, coords, abi.pd_bond_predicate(abi.PD_PREDICATE_PLANE, int(axis), 0, 0,
                                                 float(position), 0.0))


def break_notch(family: NeighborList, coords: np.ndarray, axis: int, position: float,
                sweep_axis: int, depth: float) -> None:
    """break_initial_bonds(notch_predicate(...)) (geometry.cpp:308-319), on the device."""
    _break(family, coords, abi.pd_bond_predicate(abi.PD_PREDICATE_NOTCH, int(axis),
                                                 int(sweep_axis), 0, float(position),
                                                 float(depth)))
