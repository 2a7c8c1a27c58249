# unrolled NL kernel: fast-path tests, trilinear 10M bench with / without the bulk L2 prefetch, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fast.py -q -x > gpurun_out/pytest_fast.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fast.log
for pf in 1 0 1 0; do
PD_NLU_PF=$pf timeout 600 python bench.py --law trilinear --steps 50 --no-cpu --e2e-steps 5 > gpurun_out/tri216_pf$pf.log 2>&1
tail -1 gpurun_out/tri216_pf$pf.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf$pf', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['config']['layout'], d['value'])" >> gpurun_out/nlu_ab.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lattice_nlu -s 3 -c 1 -o gpurun_out/prof_nlu216pf python bench.py --law trilinear --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/ncu_nlu.log 2>&1
tail -4 gpurun_out/pytest_fast.log; cat gpurun_out/nlu_ab.log
