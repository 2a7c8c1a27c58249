# checkpoint: all gpu tests, smoke, default bench (10M PMB + CPU baseline), 1M, trilinear, multi, exact; launch list + ncu of PMB and NL steps
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench216.log 2>&1
timeout 600 python bench.py --size 100 --no-cpu --e2e-steps 200 > gpurun_out/bench100.log 2>&1
timeout 600 python bench.py --law trilinear --no-cpu --e2e-steps 20 > gpurun_out/tri216.log 2>&1
timeout 600 python bench.py --law multi --no-cpu --e2e-steps 20 > gpurun_out/multi216.log 2>&1
timeout 900 python bench.py --variant exact --steps 10 --no-cpu --e2e-steps 2 > gpurun_out/exact216.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lat216.csv python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tri216.csv python bench.py --law trilinear --steps 5 --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/ncu_launch_tri.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_step -s 3 -c 1 -o gpurun_out/prof_lat216 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_lat.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_nlu -s 3 -c 1 -o gpurun_out/prof_nlu216 python bench.py --law trilinear --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_nlu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for f in bench216 bench100 tri216 multi216 exact216; do tail -1 gpurun_out/$f.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), '%.3e' % d['value'], 'e2e %.3e' % d['e2e']['value'])"; done
timeout 600 env K=16 python scripts/bench_batch.py 2>&1 | tail -1 > gpurun_out/batch_cfg1.json
timeout 300 python scripts/cfg1_one.py 1000 > gpurun_out/cfg1_one.log 2>&1
cut -c1-300 gpurun_out/batch_cfg1.json; tail -1 gpurun_out/cfg1_one.log
