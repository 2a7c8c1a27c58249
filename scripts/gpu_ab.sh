# A/B: in-tree library (main) against build/var/*.so on the 10M trilinear and multi-law steps
mkdir -p gpurun_out
rm -f gpurun_out/ab.log
for rep in 1 2; do
for v in main build/var/*.so; do
  if [ "$v" = main ]; then unset PD_B200_LIB; else export PD_B200_LIB=$PWD/$v; fi
  for law in trilinear multi; do
  echo "$v $law $(timeout 600 python bench.py --law $law --steps 100 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')" >> gpurun_out/ab.log
  done
done; done
unset PD_B200_LIB
cat gpurun_out/ab.log
