mkdir -p gpurun_out
PD_TIMING=1 timeout 900 python bench.py --no-cpu --steps 50 > gpurun_out/bench216_e2e.log 2>&1
grep "pd timing" gpurun_out/bench216_e2e.log | tail -8
tail -1 gpurun_out/bench216_e2e.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['seconds'])"
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
