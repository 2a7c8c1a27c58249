# the driver's bench lines (ours + the reference arm) plus extra law lines; logs under gpurun_out/
# usage: LAWS="pmb fracture" bash scripts/gpu_bench.sh
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
for law in ${LAWS:-pmb}; do
  timeout 900 python bench.py --gpus 1 --steps ${STEPS:-20} --warmup 5 --law $law ${BENCH_ARGS:-} \
    > gpurun_out/bench_$law.log 2>&1; echo "bench $law rc=$?"
  tail -1 gpurun_out/bench_$law.log | cut -c1-400
done
if [ -n "${REF:-}" ]; then
  timeout 900 python bench.py --impl reference --gpus 1 --steps ${STEPS:-20} --warmup 5 \
    > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-400
fi
