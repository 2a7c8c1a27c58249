mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
grep -E 'passed|failed|Error' gpurun_out/pytest_gpu.log | tail -4
for law in trilinear multi; do timeout 600 python bench.py --law $law --steps 100 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$law', d['ms_per_step'])"; done
timeout 1200 python scripts/bench_configs.py --save > gpurun_out/configs.log 2>&1; grep '^cfg2' gpurun_out/configs.log | cut -c1-300
