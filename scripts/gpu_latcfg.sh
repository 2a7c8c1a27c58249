for rep in 1 2; do
for v in main build/var/libpd_b200_pl3.so; do
  if [ "$v" = main ]; then unset PD_B200_LIB; else export PD_B200_LIB=$PWD/$v; fi
  for c in 0 10; do
    echo "$v cfg$c $(PD_LAT_CFG=$c timeout 600 python bench.py --steps 100 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
  done
done; done
