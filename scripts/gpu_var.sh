# A/B of kernel variants built into build/var (PD_B200_LIB) against the in-tree library
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/pytest_fast.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fast.log
for rep in 1 2; do
for v in main build/var/*.so; do
  if [ "$v" = main ]; then unset PD_B200_LIB; else export PD_B200_LIB=$PWD/$v; fi
  echo "$v $(timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --e2e-steps 10 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])')" >> gpurun_out/var.log
done; done
unset PD_B200_LIB
tail -2 gpurun_out/pytest_fast.log; cat gpurun_out/var.log
