# A/B of variant libraries (vbuild/<name>/libpd_b200.so, scripts/build_variant.sh) on one bench line
mkdir -p gpurun_out
for v in base ${VARIANTS:-}; do
  lib=paper_2105_04150_b200/libpd_b200.so; [ "$v" != base ] && lib=vbuild/$v/libpd_b200.so
  PD_B200_LIB=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-probe --sustain-steps 0 --e2e-steps 3 ${BENCH_ARGS:-} > gpurun_out/var_$v.log 2>&1
  echo "$v rc=$? $(tail -1 gpurun_out/var_$v.log | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(round(d["ms_per_step"],4),d["config"]["kernel"])' 2>&1 | tail -1)"
done
