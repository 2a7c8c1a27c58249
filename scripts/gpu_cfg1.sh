mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_slabs.py tests/test_gpu_batch.py -q > gpurun_out/pytest_fast.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fast.log
grep -E 'passed|failed|Error' gpurun_out/pytest_fast.log | tail -5
timeout 300 python scripts/cfg1_one.py 1000
PD_LAT_CFG=9 timeout 300 python scripts/cfg1_one.py 1000
timeout 600 env K=16 python scripts/bench_batch.py 2>&1 | tail -1 > gpurun_out/batch_cfg1.json; cut -c1-700 gpurun_out/batch_cfg1.json
