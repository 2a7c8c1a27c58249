"""Setup-time geometry mirroring include/peridyn/geometry.hpp.

build_family runs on the B200 (csrc/pd_family.cu) and reproduces the
reference's cell-list rows exactly.  grid_coordinates and the pre-crack
predicates are O(n) host array expressions with the reference's operation
order (not on the time-step path).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

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


def build_family(coords: np.ndarray, horizon: float,
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


def _break(family: NeighborList, coords: np.ndarray, hit_fn) -> None:
    N = int(family.group_size)
    n = family.node_count()
    ent = family.entries.reshape(n, N)
    live = ent != -1
    xyz = np.asarray(coords, dtype=np.float64).reshape(n, 3)
    ii = np.broadcast_to(np.arange(n)[:, None], ent.shape)[live]
    jj = ent[live]
    hit = hit_fn(xyz[ii], xyz[jj])
    rows = ii[hit]
    pos = np.flatnonzero(live.reshape(-1))[hit]
    family.entries.reshape(-1)[pos] = -1
    np.subtract.at(family.n_neigh, rows, 1)


def break_plane(family: NeighborList, coords: np.ndarray, axis: int, position: float) -> None:
    """break_initial_bonds(plane_crossing_predicate(axis, position)) (geometry.cpp:285-306)."""
    _break(family, coords, lambda a, b: (a[:, axis] - position) * (b[:, axis] - position) < 0)


def break_notch(family: NeighborList, coords: np.ndarray, axis: int, position: float,
                sweep_axis: int, depth: float) -> None:
    """break_initial_bonds(notch_predicate(...)) (geometry.cpp:308-319)."""
    def hit(a, b):
        da = a[:, axis] - position
        db = b[:, axis] - position
        cross_ok = da * db < 0
        with np.errstate(divide="ignore", invalid="ignore"):
            t = da / (da - db)
            cross = a[:, sweep_axis] + t * (b[:, sweep_axis] - a[:, sweep_axis])
        return cross_ok & (cross <= depth)
    _break(family, coords, hit)
