bash scripts/gpu_tests.sh
timeout 900 python scripts/bench_slab_local.py > gpurun_out/slab_local.json 2> gpurun_out/slab_local.err; echo "slab rc=$?"; tail -3 gpurun_out/slab_local.err
timeout 1200 python scripts/bench_configs.py --save > gpurun_out/configs.log 2>&1; echo "configs rc=$?"; tail -2 gpurun_out/configs.log | cut -c1-1500
