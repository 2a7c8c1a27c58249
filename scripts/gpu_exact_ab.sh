# exact kernel occupancy A/B (main vs build/var 4 CTAs/SM)
mkdir -p gpurun_out
for v in main build/var/libpd_b200_ex4.so main build/var/libpd_b200_ex4.so; do
  if [ "$v" = main ]; then unset PD_B200_LIB; else export PD_B200_LIB=$PWD/$v; fi
  echo "$v $(timeout 600 python bench.py --variant exact --steps 10 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
done
