mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py -q -x -m gpu > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_fast.log
for cfg in ${CFGS:-0}; do
PD_FAST_CFG=$cfg PD_FAST_LAYOUT=general timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu --e2e-steps 20 ${BENCH_ARGS:-} > gpurun_out/bench_tiles_$cfg.log 2>&1; echo "bench cfg $cfg rc=$?"
tail -1 gpurun_out/bench_tiles_$cfg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print(d['ms_per_step'],d['config']['kernel'],d['config']['sustained']['ms_per_step'],r.get('issue_frac'),r.get('occupancy'),r.get('thread_instructions_per_bond'),r.get('traffic'))"
done
