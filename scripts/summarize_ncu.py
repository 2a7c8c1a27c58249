#!/usr/bin/env python
"""Condense ncu output into the committed profiles/ summaries.

  python scripts/summarize_ncu.py --rep gpurun_out/prof.ncu-rep \
      --launches gpurun_out/launches.csv --bytes 7016698912 --out profiles/r01_fast216.md

--rep       an `ncu --set full` capture of the step kernel (one launch)
--launches  the `--metrics gpu__time_duration.sum` launch list of the same command
--bytes     the algorithmic bytes of one launch
"""
import argparse
import collections
import csv
import io
import subprocess

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], check=True, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out[out.index('"'):])))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--bytes", type=float, required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    lines = [f"# {a.title or a.rep}", ""]
    raw = ncu_csv(["-i", a.rep, "--page", "raw", "--csv"])
    hdr, units, vals = raw[0], raw[1], raw[2]
    lines.append(f"kernel: `{vals[hdr.index('Kernel Name')]}`")
    lines.append("")
    lines.append("| metric | value |")
    lines.append("|---|---|")
    got = {}
    for key, name in RAW:
        if key in hdr:
            i = hdr.index(key)
            got[key] = (vals[i], units[i])
            lines.append(f"| {name} (`{key}`) | {vals[i]} {units[i]} |")
    if "dram__bytes_read.sum" in got and "gpu__time_duration.sum" in got:
        rd = to_bytes(*got["dram__bytes_read.sum"])
        wr = to_bytes(*got["dram__bytes_write.sum"])
        dur_v, dur_u = got["gpu__time_duration.sum"]
        dur = float(dur_v.replace(",", "")) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(dur_u, 1)
        lines += ["", f"- traffic (read + write) per launch: {(rd + wr) / 1e9:.3f} GB",
                  f"- algorithmic bytes per launch (SURVEY.md 8(d) formula): {a.bytes / 1e9:.3f} GB",
                  f"- traffic / algorithmic: {(rd + wr) / a.bytes:.3f}",
                  f"- algorithmic GB/s under ncu (cold, serialised): {a.bytes / dur / 1e9:.1f}"]
    if a.launches:
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        h = {k: i for i, k in enumerate(rows[0])}
        agg = collections.defaultdict(lambda: [0, 0.0])
        for r in rows[1:]:
            if r[h["Metric Name"]] != "gpu__time_duration.sum":
                continue
            k = r[h["Kernel Name"]].split("(")[0]
            agg[k][0] += 1
            agg[k][1] += float(r[h["Metric Value"]].replace(",", "")) * (
                {"ns": 1e-3, "us": 1.0, "ms": 1e3}[r[h["Metric Unit"]]])
        total = sum(v[1] for v in agg.values())
        lines += ["", "## launch list (whole command, cold-cache serialised)", "",
                  "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {c} | {t:.1f} | {t / c:.1f} | {t / total:.1%} |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
