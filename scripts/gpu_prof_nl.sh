mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_nl -s 3 -c 1 -o gpurun_out/prof_nl python bench.py --law trilinear --size 128 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_nl.log 2>&1
tail -2 gpurun_out/ncu_nl.log
