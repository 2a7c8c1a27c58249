mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_slabs.py -q > gpurun_out/pytest_fast.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fast.log
grep -E 'passed|failed' gpurun_out/pytest_fast.log | tail -3
timeout 300 python scripts/cfg1_one.py 1000
PD_LAT_CFG=6 timeout 300 python scripts/cfg1_one.py 1000
timeout 600 python bench.py --size 100 --steps 100 --no-cpu --e2e-steps 2 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('1M', d['ms_per_step'])"
timeout 600 python bench.py --size 40 --steps 100 --no-cpu --e2e-steps 2 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('40^3', d['ms_per_step'])"
PD_LAT_CFG=6 timeout 600 python bench.py --size 40 --steps 100 --no-cpu --e2e-steps 2 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('40^3 cfg6', d['ms_per_step'])"
timeout 600 env K=16 python scripts/bench_batch.py 2>&1 | tail -1 | cut -c1-600
