mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lattice_nl -s 2 -c 1 -o gpurun_out/cfg5_nlu python scripts/bench_cfg5.py --steps 2 --warmup 2 --exact-steps 0 > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_cfg5.log
