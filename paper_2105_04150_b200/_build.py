"""In-tree build of the CUDA library (sm_100a) -- no JIT cache, so the .so
travels with the repo snapshot to the GPU box.

Each translation unit has its own floating-point contract:
  pd_exact.cu, pd_aux.cu, pd_host.cu  -fmad=false  (bitwise parity with the reference)
  pd_fast.cu                          FMA allowed   (the tolerance-bound fast path)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libpd_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2",
          "-Xptxas", "-warn-spills", "-I" + os.path.join(ROOT, "include")]
UNITS = {
    "pd_exact.cu": ["-fmad=false"],
    "pd_aux.cu": ["-fmad=false"],
    "pd_host.cu": ["-fmad=false"],
    "pd_fast.cu": ["-fmad=true", "-diag-suppress=186"],
    "pd_family.cu": ["-fmad=false"],
    "pd_family_ops.cu": ["-fmad=false"],
    "pd_layout.cu": ["-fmad=false"],
    "pd_lattice.cu": ["-fmad=true", "-diag-suppress=177"],
    "pd_lattice_nlu0.cu": ["-fmad=true", "-diag-suppress=177"],
    "pd_lattice_nlu1.cu": ["-fmad=true", "-diag-suppress=177"],
    "pd_lattice_nlu2.cu": ["-fmad=true", "-diag-suppress=177"],
    "pd_lattice_nlu3.cu": ["-fmad=true", "-diag-suppress=177"],
    "pd_xfer.cpp": ["-x", "cu"],
    "pd_io.cpp": ["-x", "cu"],
}
HEADERS = ["pd_device.cuh", "pd_internal.h", "pd_fast.cuh", "pd_lattice.cuh", "pd_lattice_nlu.cuh"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _mtime(p: str) -> float:
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(verbose: bool = False, force: bool = False) -> str:
    nvcc = _nvcc()
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] +
                [_mtime(os.path.join(ROOT, "include", "pd_b200.h"))])
    objs, cmds = [], []
    for unit, flags in UNITS.items():
        src = os.path.join(CSRC, unit)
        if not os.path.exists(src):
            continue
        obj = os.path.join(OBJ, os.path.splitext(unit)[0] + ".o")
        objs.append(obj)
        if force or _mtime(obj) < max(_mtime(src), hdr_t, _mtime(__file__)):
            cmds.append([nvcc, *ARCH, *COMMON, *flags, "-c", src, "-o", obj])
    # translation units compile in parallel (the lattice unit dominates)
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for cmd in cmds:
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
        for f in [ex.submit(subprocess.run, cmd, check=True) for cmd in cmds]:
            f.result()
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """Build the checkers (oracle/): the C restatement always, the reference
    library only where /root/reference is mounted.  Test infrastructure."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
    build_oracle(verbose=True)
