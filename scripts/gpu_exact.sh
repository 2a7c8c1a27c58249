# exact (fp64 parity) variant: parity + slab tests, 10M and 1M step time
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_batch.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
grep -E 'passed|failed' gpurun_out/pytest_parity.log | tail -2
timeout 900 python bench.py --variant exact --steps 10 --no-cpu --e2e-steps 2 > gpurun_out/exact216.log 2>&1
timeout 900 python bench.py --variant exact --size 100 --steps 20 --no-cpu --e2e-steps 2 > gpurun_out/exact100.log 2>&1
for f in exact216 exact100; do tail -1 gpurun_out/$f.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],4), '%.3e' % d['value'])"; done
