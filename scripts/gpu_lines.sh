# extra bench lines for profiles/ (one JSON per line under gpurun_out/line_*.log) + the slab barrier
mkdir -p gpurun_out
timeout 900 python scripts/bench_slab_local.py --barrier-only > gpurun_out/barrier.json 2> gpurun_out/barrier.err; echo "barrier rc=$?"; cat gpurun_out/barrier.json
run() { name=$1; shift; timeout 900 python bench.py --steps 20 --warmup 5 "$@" > gpurun_out/line_$name.log 2>&1; echo "$name rc=$? $(tail -1 gpurun_out/line_$name.log | cut -c1-160)"; }
run trilinear216 --law trilinear --no-cpu
run multi216 --law multi --no-cpu
run exact216 --variant exact --no-cpu --e2e-steps 50
run pmb100 --size 100
run fracture100 --size 100 --law fracture --no-cpu
