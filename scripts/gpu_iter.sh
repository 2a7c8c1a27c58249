# one build -> measure iteration: gpu tests, 10M and 1M bench, ncu of the lattice step at 10M
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu --e2e-steps 1000 > gpurun_out/bench_iter216.log 2>&1
timeout 900 python bench.py --size 100 --steps 200 --warmup 5 --no-cpu --e2e-steps 200 > gpurun_out/bench_iter100.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_step -s 3 -c 1 -o gpurun_out/prof_iter python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_iter.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench_iter216.log | cut -c1-400; tail -1 gpurun_out/bench_iter100.log | cut -c1-400
