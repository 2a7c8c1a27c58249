# exact (bitwise) variant: parity tests + timing per lanes-per-node choice; logs under gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_cfg5.py tests/test_gpu_integrators.py -q -x -m gpu > gpurun_out/pytest_exact.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_exact.log
for g in ${GS:-32 16 8}; do
PD_EXACT_G=$g timeout 900 python bench.py --variant exact --steps 20 --warmup 3 --no-cpu --no-probe --sustain-steps 0 --e2e-steps 3 --size ${SIZE:-216} > gpurun_out/bench_exact_$g.log 2>&1; echo "G=$g rc=$?"
tail -1 gpurun_out/bench_exact_$g.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['ms_per_step'],d['config']['kernel'],d['value'])"
done
