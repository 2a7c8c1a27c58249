mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_slabs.py -q -x > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
for c in 0 4; do
  PD_LAT_CFG=$c timeout 600 python bench.py --steps 40 --no-cpu --e2e-steps 5 > gpurun_out/latcfg$c.log 2>&1
done
tail -2 gpurun_out/pytest_fast.log
for c in 0 4; do tail -1 gpurun_out/latcfg$c.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c', round(d['ms_per_step'],4), round(d['roofline']['frac'],4))"; done
