# ncu captures of the current PMB lattice step and the n-linear (trilinear) lattice step at 10M
mkdir -p gpurun_out
timeout 900 python bench.py --law trilinear --steps 50 --no-cpu --e2e-steps 5 > gpurun_out/tri216.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lat216.csv python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_step -s 3 -c 1 -o gpurun_out/prof_lat216c python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_lat.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_nl -s 3 -c 1 -o gpurun_out/prof_nl216 python bench.py --law trilinear --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_nl.log 2>&1
tail -1 gpurun_out/tri216.log | cut -c1-600
