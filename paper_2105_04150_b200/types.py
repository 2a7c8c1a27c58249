"""Value types mirroring the reference's C++ API (include/peridyn/types.hpp and
engine.hpp), numpy-backed with the reference's flat layouts: vectors are flat
n x 3 float64, per-slot arrays flat n x N.  Names, fields and factory
behaviour follow the reference so user code ports line for line.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Dict, List, Optional

import numpy as np

from .abi import InvalidArgument


class KernelVariant(IntEnum):
    """engine.hpp:15, plus the B200 fast path."""
    bond_parallel = 0  # fp64, bitwise equal to compute_forces_bond_parallel
    node_parallel = 1  # fp64, bitwise equal to compute_forces_node_parallel
    fast = 2           # fp64 state, fp32 bond arithmetic (DESIGN.md tolerance)


class IntegratorKind(IntEnum):
    """engine.hpp:87"""
    velocity_verlet = 0
    euler = 1
    euler_cromer = 2


class BCKind(IntEnum):
    """types.hpp:127"""
    free = 0
    displacement = 1
    force = 2


@dataclass
class ParticleSet:
    """types.hpp:52-60"""
    coords: np.ndarray
    volume: np.ndarray
    density: np.ndarray
    material_tag: Optional[np.ndarray] = None

    def size(self) -> int:
        return int(np.asarray(self.volume).size)


@dataclass
class NeighborList:
    """types.hpp:66-76: padded rows, -1 = broken or padding."""
    entries: np.ndarray
    n_neigh: np.ndarray
    initial_n_neigh: np.ndarray
    group_size: int
    horizon: float = 0.0
    bond_type: Optional[np.ndarray] = None

    def node_count(self) -> int:
        return int(np.asarray(self.n_neigh).size)

    def copy(self) -> "NeighborList":
        return NeighborList(np.array(self.entries, dtype=np.int32, copy=True),
                            np.array(self.n_neigh, dtype=np.int32, copy=True),
                            np.array(self.initial_n_neigh, dtype=np.int32, copy=True),
                            int(self.group_size), float(self.horizon),
                            None if self.bond_type is None else np.array(self.bond_type, copy=True))


def _law_validate(stiffness, bps, forces):
    # DamageLaw::validate (types.cpp:50-65)
    if not stiffness > 0:
        raise InvalidArgument("DamageLaw: stiffness must be positive")
    if len(bps) == 0 or len(bps) != len(forces):
        raise InvalidArgument("DamageLaw: breakpoints and forces must match and be non-empty")
    prev = 0.0
    for b in bps:
        if not b > prev:
            raise InvalidArgument("DamageLaw: breakpoints must be strictly increasing and positive")
        prev = b
    f0 = stiffness * bps[0]
    if abs(forces[0] - f0) > 1e-9 * max(abs(f0), 1.0):
        raise InvalidArgument("DamageLaw: envelope must leave the origin with slope c")


@dataclass
class DamageLaw:
    """types.hpp:83-96; factories as types.cpp:67-83."""
    stiffness: float
    breakpoints: List[float]
    forces: List[float]

    def critical_stretch(self) -> float:
        return self.breakpoints[-1]

    def validate(self) -> None:
        _law_validate(self.stiffness, self.breakpoints, self.forces)

    @staticmethod
    def pmb(c: float, s_c: float) -> "DamageLaw":
        law = DamageLaw(float(c), [float(s_c)], [float(c) * float(s_c)])
        law.validate()
        return law

    @staticmethod
    def bilinear(c: float, s0: float, s_c: float) -> "DamageLaw":
        law = DamageLaw(float(c), [float(s0), float(s_c)], [float(c) * float(s0), 0.0])
        law.validate()
        return law

    @staticmethod
    def trilinear(c: float, s0: float, s1: float, s_c: float,
                  kink_beta: float = 0.25) -> "DamageLaw":
        c, s0 = float(c), float(s0)
        law = DamageLaw(c, [s0, float(s1), float(s_c)], [c * s0, float(kink_beta) * c * s0, 0.0])
        law.validate()
        return law


@dataclass
class DamageModel:
    """types.hpp:99-110"""
    laws: List[DamageLaw] = field(default_factory=list)
    damping: float = 0.0
    use_surface_correction: bool = False
    use_partial_volume: bool = False

    def needs_history(self) -> bool:
        return any(len(l.breakpoints) > 1 for l in self.laws)


@dataclass
class SimulationState:
    """types.hpp:115-122"""
    u: np.ndarray
    v: np.ndarray
    a: np.ndarray
    step: int
    connectivity: NeighborList
    bond_history: Optional[np.ndarray] = None

    def size(self) -> int:
        return self.connectivity.node_count()


def make_state(family: NeighborList, with_history: bool) -> SimulationState:
    """types.cpp:107-117: zero fields and a copy of the connectivity."""
    n = family.node_count()
    hist = np.zeros(n * int(family.group_size)) if with_history else np.zeros(0)
    return SimulationState(np.zeros(3 * n), np.zeros(3 * n), np.zeros(3 * n), 0, family.copy(),
                           hist)


class RampKind(IntEnum):
    """types.hpp:132"""
    constant = 0
    linear = 1
    quintic_smooth = 2


@dataclass
class RampProfile:
    """types.hpp:131-142 (scale/rate/accel evaluated on the device)."""
    kind: RampKind = RampKind.constant
    rise_steps: int = 0
    target_scale: float = 1.0


@dataclass
class BoundaryConditions:
    """types.hpp:145-155"""
    kind: np.ndarray
    magnitude: np.ndarray
    ramp_id: np.ndarray
    ramps: List[RampProfile]
    no_failure: np.ndarray
    tip_sets: Dict[str, List[int]] = field(default_factory=dict)

    @staticmethod
    def none(n: int) -> "BoundaryConditions":
        return BoundaryConditions(np.zeros(3 * n, np.uint8), np.zeros(3 * n), np.zeros(3 * n, np.uint8),
                                  [RampProfile()], np.zeros(n, np.uint8), {})


@dataclass
class Corrections:
    """types.hpp:161-165 (empty arrays = identity)."""
    lambda_: Optional[np.ndarray] = None
    beta: Optional[np.ndarray] = None
    no_failure: Optional[np.ndarray] = None


@dataclass
class ForceField:
    """types.hpp:170-178"""
    body_force: np.ndarray = field(default_factory=lambda: np.zeros(0))
    external_force: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def resize(self, n: int) -> None:
        self.body_force = np.zeros(3 * n)
        self.external_force = np.zeros(3 * n)


@dataclass
class ModelBundle:
    """engine.hpp:90-98"""
    particles: ParticleSet
    model: DamageModel
    corrections: Corrections
    bc: BoundaryConditions
    dt: float = 0.0


@dataclass
class SimulateOptions:
    """engine.hpp:100-106"""
    steps: int = 0
    write_every: int = 0
    first_step: int = 0
    integrator: IntegratorKind = IntegratorKind.velocity_verlet
    variant: KernelVariant = KernelVariant.bond_parallel


@dataclass
class TipRecord:
    """engine.hpp:110-114"""
    step: int
    mean_u: np.ndarray
    mean_v: np.ndarray
    mean_a: np.ndarray
    body_force_sum: np.ndarray
    external_force_sum: np.ndarray


@dataclass
class SimulateResult:
    """engine.hpp:120-122"""
    tips: Dict[str, List[TipRecord]] = field(default_factory=dict)


WriteHook = Callable[[SimulationState, ForceField], None]
