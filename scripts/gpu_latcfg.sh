# PMB lattice kernel brick/occupancy configs at 10M, plane-wise (main) vs flat (build/var) staging
for v in main build/var/libpd_b200_flat.so; do
  if [ "$v" = main ]; then unset PD_B200_LIB; else export PD_B200_LIB=$PWD/$v; fi
  for c in 0 1 3 7 8; do
    echo "$v cfg$c $(PD_LAT_CFG=$c timeout 600 python bench.py --steps 100 --no-cpu --e2e-steps 2 2>&1 | tail -1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"
  done
done
