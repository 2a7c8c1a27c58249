mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_step -s 3 -c 1 -o gpurun_out/prof_fast216 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_fast.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fast216.csv python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
