# slab bench path on one GPU (2 ranks share cuda:0; gloo plumbing) + default single bench with timing
mkdir -p gpurun_out
PD_TIMING=1 timeout 900 python bench.py --no-cpu --steps 20 --e2e-steps 200 > gpurun_out/bench216_t.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --size 64 --steps 10 --warmup 3 --e2e-steps 20 > gpurun_out/bench_slab2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_slab2.log
grep "pd timing" gpurun_out/bench216_t.log; tail -1 gpurun_out/bench216_t.log | cut -c1-400
tail -5 gpurun_out/bench_slab2.log | cut -c1-1500
