# cfg5 parity (downscale) + the full-size RC beam timing; logs under gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_family_ops.py tests/test_gpu_cfg5.py -q -x -m gpu -rA > gpurun_out/pytest_cfg5.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error" gpurun_out/pytest_cfg5.log | tail -5
timeout 1500 python scripts/bench_cfg5.py --dx ${DX:-1.6} > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err; echo "cfg5 rc=$?"; tail -4 gpurun_out/cfg5.err | cut -c1-600; cut -c1-1500 gpurun_out/cfg5.json
