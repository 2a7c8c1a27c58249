# final: smoke, the driver's default bench line and the reference arm
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench216.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
tail -3 gpurun_out/smoke.log; tail -1 gpurun_out/bench216.log | cut -c1-600; tail -1 gpurun_out/bench_ref.log | cut -c1-300
