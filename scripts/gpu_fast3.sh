mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "fast" > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu --e2e-steps 30 > gpurun_out/bench_fast216.log 2>&1
timeout 600 python bench.py --size 100 --steps 30 --warmup 5 --no-cpu --e2e-steps 30 > gpurun_out/bench_fast100.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_step -s 3 -c 1 -o gpurun_out/prof_fast3 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_fast.log 2>&1
tail -3 gpurun_out/pytest_fast.log; tail -1 gpurun_out/bench_fast216.log | cut -c1-700; tail -1 gpurun_out/bench_fast100.log | cut -c1-400
