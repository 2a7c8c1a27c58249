mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lattice_split -s 500 -c 1 -o gpurun_out/prof_split python scripts/cfg1_one.py 1000 > gpurun_out/ncu_split.log 2>&1
tail -3 gpurun_out/ncu_split.log
