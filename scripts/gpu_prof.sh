# ncu capture of one step kernel + the launch list of the same bench command (logs under gpurun_out/)
# usage: KERNEL=lattice_step NAME=lattice216 BENCH_ARGS="--law pmb" bash scripts/gpu_prof.sh
mkdir -p gpurun_out
K=${KERNEL:-lattice_step}; N=${NAME:-prof}
ARGS="--steps 2 --warmup 3 --no-cpu --no-probe --sustain-steps 0 --e2e-steps 2 ${BENCH_ARGS:-}"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
  -o gpurun_out/$N python bench.py $ARGS > gpurun_out/ncu_$N.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$N.csv python bench.py $ARGS > gpurun_out/ncu_launch_$N.log 2>&1
echo "launch list rc=$?"
