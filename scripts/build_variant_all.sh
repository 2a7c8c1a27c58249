# build a variant library with extra nvcc flags for every translation unit (vbuild/<name>)
name=$1; shift
mkdir -p vbuild/$name
python - "$name" "$@" <<'PY'
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.getcwd())
from paper_2105_04150_b200 import _build as B
name, extra = sys.argv[1], sys.argv[2:]
out = os.path.join("vbuild", name)
cmds, objs = [], []
for unit, flags in B.UNITS.items():
    o = os.path.join(out, os.path.splitext(unit)[0] + ".o")
    objs.append(o)
    cmds.append([B._nvcc(), *B.ARCH, *B.COMMON, *flags, *extra, "-c", os.path.join(B.CSRC, unit), "-o", o])
with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
    for f in [ex.submit(subprocess.run, c, check=True, capture_output=True) for c in cmds]:
        f.result()
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", os.path.join(out, "libpd_b200.so"), *objs], check=True)
for o in objs:
    os.remove(o)
PY
