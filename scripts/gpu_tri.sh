mkdir -p gpurun_out
timeout 900 python bench.py --law trilinear --steps 30 --no-cpu --e2e-steps 5 > gpurun_out/tri216.log 2>&1
timeout 900 python bench.py --law trilinear --variant exact --size 100 --steps 10 --no-cpu --e2e-steps 2 > gpurun_out/tri100_exact.log 2>&1
timeout 900 python bench.py --variant exact --steps 10 --no-cpu --e2e-steps 2 > gpurun_out/exact216.log 2>&1
for f in tri216 tri100_exact exact216; do tail -1 gpurun_out/$f.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['config']['layout'], d['value'])"; done
