# gpu tests + e2e phase breakdown of the 10M-node 1000-step simulate() call
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for t in 1 2; do
PD_TIMING=1 timeout 600 python bench.py --steps 20 --no-cpu --e2e-steps 1000 > gpurun_out/e2e_t$t.log 2>&1
echo "run $t"; grep -v '^{' gpurun_out/e2e_t$t.log | grep 'upload\|simulate' | tail -9; tail -1 gpurun_out/e2e_t$t.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['value'], d['e2e']['seconds'])"
done
