mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
PD_TIMING=1 timeout 900 python bench.py --no-cpu > gpurun_out/bench216_e2e.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; grep "pd timing" gpurun_out/bench216_e2e.log | tail -9
tail -1 gpurun_out/bench216_e2e.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['e2e'], d['clocks'])"
