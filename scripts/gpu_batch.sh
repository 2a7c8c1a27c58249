mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -q -x > gpurun_out/pytest_batch.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_batch.log
timeout 900 python scripts/bench_batch.py > gpurun_out/batch.json 2> gpurun_out/batch.err
tail -3 gpurun_out/pytest_batch.log; tail -1 gpurun_out/batch.json; tail -3 gpurun_out/batch.err
