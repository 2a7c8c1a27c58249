mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "fast" > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --e2e-steps 30 > gpurun_out/bench_fast216.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_step -s 4 -c 1 -o gpurun_out/prof_fast2 python bench.py --size 100 --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_fast.log 2>&1
tail -5 gpurun_out/pytest_fast.log; tail -1 gpurun_out/bench_fast216.log | cut -c1-1000
