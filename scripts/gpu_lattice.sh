mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_slabs.py -q -x > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
timeout 600 python bench.py --steps 40 --no-cpu --e2e-steps 200 > gpurun_out/lat216.log 2>&1
timeout 600 python bench.py --size 100 --steps 50 --no-cpu --e2e-steps 20 > gpurun_out/lat100.log 2>&1
PD_FAST_LAYOUT=general timeout 600 python bench.py --steps 40 --no-cpu --e2e-steps 20 > gpurun_out/gen216.log 2>&1
tail -3 gpurun_out/pytest_fast.log
for f in lat216 lat100 gen216; do tail -1 gpurun_out/$f.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), round(d['e2e']['value']/1e9,1))"; done
