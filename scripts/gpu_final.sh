mkdir -p gpurun_out
bash scripts/gpu_tests.sh
LAWS="pmb fracture" REF=1 STEPS=20 bash scripts/gpu_bench.sh
bash scripts/gpu_configs.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lattice_small -c 1 -o gpurun_out/small_cfg1 python scripts/cfg1_run.py 200 > gpurun_out/ncu_small.log 2>&1; echo "ncu small rc=$?"
python scripts/cfg1_run.py 1000 > gpurun_out/cfg1_final.log 2>&1; cat gpurun_out/cfg1_final.log
