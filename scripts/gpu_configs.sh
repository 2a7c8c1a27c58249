mkdir -p gpurun_out
timeout 1200 python scripts/bench_configs.py --save > gpurun_out/configs.log 2>&1; echo "rc=$?"
tail -5 gpurun_out/configs.log | cut -c1-900
timeout 600 env K=16 python scripts/bench_batch.py 2>&1 | tail -1 > gpurun_out/batch_cfg1.json; cut -c1-400 gpurun_out/batch_cfg1.json
