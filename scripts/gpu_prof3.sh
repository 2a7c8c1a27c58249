mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fast.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_step -s 3 -c 1 -o gpurun_out/prof_lat216d python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_lat.log 2>&1
tail -3 gpurun_out/pytest_fast.log
