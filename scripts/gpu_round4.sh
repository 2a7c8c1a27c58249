# checkpoint: gpu tests, smoke, default bench (10M + CPU baseline), reference arm, slab bench path at 2 and 4 ranks sharing cuda:0
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench216.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
for w in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $w --master-addr 127.0.0.1 --master-port 2951$w bench.py --gpus $w --steps 20 --warmup 3 --e2e-steps 50 > gpurun_out/bench_slab$w.log 2>&1; echo "rc=$?" >> gpurun_out/bench_slab$w.log
done
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for f in bench216 bench_ref bench_slab2 bench_slab4; do grep '^{' gpurun_out/$f.log | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d.get('n_gpus'), d.get('ms_per_step'), '%.3e' % d['value'], 'e2e %.3e' % d['e2e']['value'])" || tail -3 gpurun_out/$f.log; done
