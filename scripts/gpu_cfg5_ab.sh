# cfg5 fast step time per library variant (vbuild/<name>); base = the in-tree library
mkdir -p gpurun_out
for v in base ${VARIANTS:-}; do
  lib=paper_2105_04150_b200/libpd_b200.so; [ "$v" != base ] && lib=vbuild/$v/libpd_b200.so
  PD_B200_LIB=$PWD/$lib timeout 900 python scripts/bench_cfg5.py --dx ${DX:-1.6} --steps 20 --exact-steps 0 > gpurun_out/cfg5_$v.json 2>/dev/null
  echo "$v rc=$? $(python -c "import json;d=json.load(open('gpurun_out/cfg5_$v.json'));print(round(d['fast']['ms_per_step'],3), d['fast']['kernel'])" 2>&1 | tail -1)"
done
