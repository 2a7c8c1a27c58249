mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg1.csv python scripts/cfg1_one.py 50 > /dev/null 2>&1
python3 - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/launches_cfg1.csv')) if len(r)>10]
h={k:i for i,k in enumerate(rows[0])}
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[r[h['Kernel Name']].split('(')[0][-60:]].append(float(r[h['Metric Value']].replace(',','')))
for k,v in sorted(agg.items(), key=lambda kv:-sum(kv[1]))[:4]: print(len(v), round(sum(v)/len(v)/1e3,2), 'us', k)
PY
python - <<'PY'
import sys, time, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import scenarios as S
from paper_2105_04150_b200 import engine, geometry
from paper_2105_04150_b200.types import IntegratorKind, KernelVariant, make_state
import torch
b, h, g = S.beam_bundle()
fam = geometry.build_family(b.particles.coords, h, g)
ctx = engine.Context(0)
st = make_state(fam, False)
ctx.upload(b, st, KernelVariant.fast)
ctx.run(10, 0, IntegratorKind.euler, 0, KernelVariant.fast)
torch.cuda.synchronize()
for n in (1000, 1000):
    t0 = time.perf_counter(); ctx.run(n, 10, IntegratorKind.euler, 0, KernelVariant.fast); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"run({n}): host enqueue {1e3*(t1-t0):.2f} ms, until idle {1e3*(t2-t0):.2f} ms")
PY
