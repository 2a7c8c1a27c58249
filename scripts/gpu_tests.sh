# GPU test suite + smoke on the box (logs under gpurun_out/)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rA ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
grep -E "passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -3; tail -4 gpurun_out/smoke.log
