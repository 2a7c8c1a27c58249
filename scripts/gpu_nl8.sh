mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_slabs.py tests/test_gpu_parity.py -q > gpurun_out/pytest_nl8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nl8.log
grep -E 'passed|failed|Error' gpurun_out/pytest_nl8.log | tail -4
for law in trilinear multi; do timeout 600 python bench.py --law $law --steps 100 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$law', d['ms_per_step'])"; done
PD_LAT_NL_LOOP=1 timeout 600 python bench.py --law multi --steps 20 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('multi loop', d['ms_per_step'])"
