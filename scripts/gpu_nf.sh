mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_slabs.py -q > gpurun_out/pytest_nf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nf.log
for law in pmb trilinear multi; do timeout 600 python bench.py --law $law --steps 100 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$law', d['ms_per_step'])"; done
grep -E 'passed|failed|Error' gpurun_out/pytest_nf.log | tail -8
