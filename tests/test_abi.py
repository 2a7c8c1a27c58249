"""The C-ABI library: it loads, exports every symbol include/pd_b200.h
declares, its struct layouts match the ctypes mirror, and without a GPU it
fails loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2105_04150_b200 import abi, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pd_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(pd_[a-z_0-9]+)\s*\(", text))
    return sorted(n for n in names if n != "pd_write_hook")


def test_library_exports_every_declared_symbol():
    lib = engine.library()
    names = declared_functions()
    assert len(names) >= 19
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", engine.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (pd_\w+)", out))
    assert set(names) <= exported


def test_library_is_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", engine.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version():
    assert engine.library().pd_abi_version() == 1


PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "pd_b200.h"
#define S(t) printf(#t " %zu\n", sizeof(t));
#define O(t, f) printf(#t "." #f " %zu\n", offsetof(t, f));
int main(void) {
  S(pd_particles) S(pd_neighbor_list) S(pd_law) S(pd_damage_model) S(pd_corrections)
  S(pd_state) S(pd_force_field) S(pd_ramp) S(pd_boundary) S(pd_bundle) S(pd_options)
  S(pd_tip_record)
  O(pd_state, connectivity) O(pd_state, bond_history_size) O(pd_bundle, bc) O(pd_bundle, dt)
  O(pd_boundary, tip_nodes) O(pd_law, forces) O(pd_options, variant)
  return 0;
}
"""


def test_struct_layouts_match_ctypes(tmp_path):
    src = tmp_path / "probe.c"
    src.write_text(PROBE)
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run(
        [str(exe)], capture_output=True, text=True, check=True).stdout.splitlines())
    for name, value in got.items():
        if "." in name:
            t, f = name.split(".")
            assert getattr(getattr(abi, t), f).offset == int(value), name
        else:
            assert C.sizeof(getattr(abi, name)) == int(value), name


def _has_gpu():
    try:
        return engine.device_count() > 0
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    """The product fails loudly when no B200 is visible."""
    import scenarios as S
    from paper_2105_04150_b200 import ForceField, KernelVariant, make_state
    lib = engine.library()
    assert lib.pd_device_count() == 0
    h = C.c_void_p()
    assert lib.pd_ctx_create(0, C.byref(h)) == abi.PD_E_NO_DEVICE
    bundle, hz, _ = S.small_fracture_bundle()
    from oracle.pyoracle import COracle
    fam = COracle().build_family(bundle.particles.coords, hz)
    st = make_state(fam, False)
    f = ForceField()
    with pytest.raises(abi.CudaError):
        engine.compute_forces(KernelVariant.bond_parallel, st, bundle.particles, bundle.model,
                              bundle.corrections, f)
    with pytest.raises(abi.CudaError):
        engine.Context()
    from paper_2105_04150_b200.geometry import build_family
    with pytest.raises(abi.CudaError):
        build_family(bundle.particles.coords, hz)


def test_validation_errors_precede_device_use():
    """check_force_inputs order (engine.cpp:30-49): size and finiteness errors
    are raised with the reference's types before any device work."""
    import scenarios as S
    from oracle.pyoracle import COracle
    from paper_2105_04150_b200 import (DamageLaw, DamageModel, ForceField, KernelVariant,
                                       SimulateOptions, make_state)
    bundle, hz, _ = S.small_fracture_bundle()
    fam = COracle().build_family(bundle.particles.coords, hz)
    st = make_state(fam, False)
    st.u[4] = np.nan
    st.step = 31
    with pytest.raises(abi.PeridynRuntimeError, match="non-finite displacement at step 31"):
        engine.compute_forces(KernelVariant.bond_parallel, st, bundle.particles, bundle.model,
                              bundle.corrections, ForceField())
    st = make_state(fam, True)
    bad = DamageModel([DamageLaw(1.0, [0.2, 0.1], [0.2, 0.0])])
    with pytest.raises(abi.InvalidArgument, match="strictly increasing"):
        engine.compute_forces(KernelVariant.bond_parallel, st, bundle.particles, bad,
                              bundle.corrections, ForceField())
    with pytest.raises(abi.InvalidArgument, match="steps must be >= 1"):
        engine.simulate(bundle, make_state(fam, False), SimulateOptions(0))
