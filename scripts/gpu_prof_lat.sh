mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_step -s 3 -c 1 -o gpurun_out/prof_lat216 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_lat.log 2>&1
tail -3 gpurun_out/ncu_lat.log
