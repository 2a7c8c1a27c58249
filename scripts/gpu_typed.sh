# typed multi-law lattice kernel: fast-path tests, cfg5-style multi-law bench (typed vs loop), trilinear
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/pytest_fast.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fast.log
timeout 600 python bench.py --law multi --steps 50 --no-cpu --e2e-steps 5 > gpurun_out/multi216.log 2>&1
PD_LAT_NL_LOOP=1 timeout 600 python bench.py --law multi --steps 20 --no-cpu --e2e-steps 2 > gpurun_out/multi216_loop.log 2>&1
timeout 600 python bench.py --law trilinear --steps 50 --no-cpu --e2e-steps 5 > gpurun_out/tri216.log 2>&1
tail -4 gpurun_out/pytest_fast.log
for f in multi216 multi216_loop tri216; do tail -1 gpurun_out/$f.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['config']['layout'], '%.3e' % d['value'])" || tail -5 gpurun_out/$f.log; done
