# tile-configuration experiment: parity tests, then the 10M / 1M bench per PD_FAST_CFG
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 0 1 2 3; do
  PD_FAST_CFG=$c timeout 600 python bench.py --steps 30 --no-cpu --e2e-steps 5 > gpurun_out/exp_cfg$c.log 2>&1
  PD_FAST_CFG=$c timeout 600 python bench.py --size 100 --steps 50 --no-cpu --e2e-steps 5 > gpurun_out/exp100_cfg$c.log 2>&1
done
tail -3 gpurun_out/pytest_gpu.log
for c in 0 1 2 3; do python - "$c" <<'PY'
import json,sys
c=sys.argv[1]
for f in (f"gpurun_out/exp_cfg{c}.log", f"gpurun_out/exp100_cfg{c}.log"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(c, f, round(d["ms_per_step"],4), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])
    except Exception as e: print(c, f, "ERR", e)
PY
done
