mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py -q -x > gpurun_out/pytest_slabs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_slabs.log
tail -30 gpurun_out/pytest_slabs.log
