"""B200-native explicit bond-based peridynamics time step (arXiv 2105.04150).

A drop-in for the reference engine's force pass and simulate loop
(/root/reference/proj/include/peridyn/engine.hpp) backed by hand-written
sm_100a kernels in libpd_b200.so.  There is no CPU fallback: every entry
point raises CudaError when the library or a B200 is missing.
"""
from .abi import CudaError, DomainError, InvalidArgument, PeridynRuntimeError
from .engine import (Context, compute_forces, device_count, load_cache, load_state, local_damage,
                     save_cache, save_state, simulate, write_snapshot)
from .geometry import GridDesc, break_notch, break_plane, build_family, grid_coordinates
from .types import (BCKind, BoundaryConditions, Corrections, DamageLaw, DamageModel, ForceField,
                    IntegratorKind, KernelVariant, ModelBundle, NeighborList, ParticleSet,
                    RampKind, RampProfile, SimulateOptions, SimulateResult, SimulationState,
                    TipRecord, make_state)

__all__ = [
    "BCKind", "BoundaryConditions", "Context", "Corrections", "CudaError", "DamageLaw",
    "DamageModel", "DomainError", "ForceField", "GridDesc", "IntegratorKind", "InvalidArgument",
    "KernelVariant", "ModelBundle", "NeighborList", "ParticleSet", "PeridynRuntimeError",
    "RampKind", "RampProfile", "SimulateOptions", "SimulateResult", "SimulationState",
    "TipRecord", "break_notch", "break_plane", "build_family", "compute_forces",
    "device_count", "grid_coordinates", "load_cache", "load_state", "local_damage", "make_state",
    "save_cache", "save_state", "simulate", "write_snapshot",
]
