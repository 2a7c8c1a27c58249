# e2e phase breakdown of the 10M-node 1000-step simulate() call
mkdir -p gpurun_out
PD_TIMING=1 timeout 600 python bench.py --steps 20 --no-cpu --e2e-steps 1000 > gpurun_out/e2e_t.log 2>&1
grep -v '^{' gpurun_out/e2e_t.log | tail -30; tail -1 gpurun_out/e2e_t.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
