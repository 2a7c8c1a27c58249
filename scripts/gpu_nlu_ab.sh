# A/B of the unrolled NL kernel: per-slot L2 prefetch distance (main = 24, build/var pfd*), bulk L2 prefetch on/off
mkdir -p gpurun_out
for rep in 1 2; do
for v in main build/var/*.so; do
for pf in 0 1; do
  if [ "$v" = main ]; then unset PD_B200_LIB; else export PD_B200_LIB=$PWD/$v; fi
  echo "$v pf$pf $(PD_NLU_PF=$pf timeout 600 python bench.py --law trilinear --steps 50 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')" >> gpurun_out/nlu_ab3.log
done; done; done
unset PD_B200_LIB
cat gpurun_out/nlu_ab3.log
