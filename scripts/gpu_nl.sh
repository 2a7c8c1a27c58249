mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_all.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_all.log
timeout 900 python bench.py --law trilinear --steps 30 --no-cpu --e2e-steps 5 > gpurun_out/tri216.log 2>&1
tail -1 gpurun_out/tri216.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('tri216', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['config']['layout'], d['value'])"
PD_FAST_LAYOUT=general timeout 900 python bench.py --law trilinear --steps 30 --no-cpu --e2e-steps 5 > gpurun_out/tri216_tiles.log 2>&1
tail -1 gpurun_out/tri216_tiles.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('tri216 tiles', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['config']['layout'], d['value'])"
bash scripts/gpu_prof_nl.sh
