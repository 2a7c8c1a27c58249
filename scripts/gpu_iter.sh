# build -> measure: gpu tests (fast + lattice), 10M PMB and trilinear/multi bench, ncu of the PMB step
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu --e2e-steps 1000 > gpurun_out/bench_iter216.log 2>&1
timeout 600 python bench.py --law trilinear --steps 50 --no-cpu --e2e-steps 5 > gpurun_out/tri216.log 2>&1
timeout 600 python bench.py --law multi --steps 50 --no-cpu --e2e-steps 5 > gpurun_out/multi216.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_step -s 3 -c 1 -o gpurun_out/prof_iter python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_iter.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for f in bench_iter216 tri216 multi216; do tail -1 gpurun_out/$f.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), '%.3e' % d['value'], 'e2e %.3e' % d['e2e']['value'])"; done
