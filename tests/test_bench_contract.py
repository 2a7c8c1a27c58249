"""bench.py's JSON contract and byte accounting, on CPU (no GPU work):
the SURVEY 8(d) algorithmic-bytes formula at cfg3 / cfg4, the keys of the
line the driver reads, and the run split of the CPU baseline."""
import argparse
import json

import bench


def test_algorithmic_bytes_match_survey():
    # cfg3 687.4 MB, cfg4 7016.7 MB per step (fp64 state)
    assert bench.algorithmic_bytes(100 ** 3, 128, 117_844_248) == 687_376_992
    assert bench.algorithmic_bytes(216 ** 3, 128, 1_209_979_144) == 7_016_698_912


def test_summary_line_has_the_driver_keys():
    args = argparse.Namespace(size=216, law="pmb", mesh="lattice", steps=20, warmup=5,
                              variant="fast")
    e2e = {"value": 8.9e11, "unit": bench.UNIT, "h2d_bytes_per_step": 1, "d2h_bytes_per_step": 1}
    probe = {"dram_bytes": 1.8e9, "issue_active_pct": 74.0, "warps_active_pct": 72.0,
             "warp_instructions": 9.5e8}
    n, N, live = 216 ** 3, 128, 1_209_979_144
    b = bench.algorithmic_bytes(n, N, live)
    out = bench._summary(args, 1.08e12, 1.12, 1, n, N, live, b, b / 1.12e-3 / 1e9, e2e, 21,
                         {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []}, None, "fast",
                         probe, {"kernel": "lattice_step_kernel<1,8,3,0,0>"})
    line = json.loads(json.dumps(out))
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert key in line, key
    r = line["roofline"]
    assert r["bound"] == "issue" and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert abs(r["traffic"] - 1.8) < 1e-12 and 0 < r["dram_frac"] < 1
    assert line["config"]["workload"].startswith("cfg4 lattice 216^3")


def test_cpu_baseline_runs_are_at_least_three_by_three():
    for k in (9, 20, 100):
        runs = bench.split_runs(k)
        assert len(runs) >= 3 and min(runs) >= 3 and sum(runs) == k
    assert bench.split_runs(3) == [3]
