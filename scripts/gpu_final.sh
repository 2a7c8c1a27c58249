# the round-end refresh (logs under gpurun_out/): the -m gpu suite + smoke, the
# driver's bench lines with the reference arm (BENCH=1), cfg1-cfg3 and the
# batched cfg1 sweep, the persistent small-model kernel (timing, ncu capture,
# and the clock64 breakdown when vbuild/prof holds a -DPD_SMALL_PROF build)
mkdir -p gpurun_out
bash scripts/gpu_tests.sh
if [ -n "${BENCH:-}" ]; then LAWS="pmb fracture" REF=1 STEPS=20 bash scripts/gpu_bench.sh; fi
bash scripts/gpu_configs.sh
python scripts/cfg1_run.py 1000 > gpurun_out/cfg1_final.log 2>&1; cat gpurun_out/cfg1_final.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lattice_small -c 1 -o gpurun_out/small_cfg1 python scripts/cfg1_run.py 200 > gpurun_out/ncu_small.log 2>&1; echo "ncu small rc=$?"
if [ -f vbuild/prof/libpd_b200.so ]; then
  PD_B200_LIB=vbuild/prof/libpd_b200.so python scripts/cfg1_run.py 1000 2>&1 | grep "small prof" | sort | uniq > gpurun_out/small_prof.log
  awk "NR%4==1" gpurun_out/small_prof.log
fi
