#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list (csv from
`ncu --metrics gpu__time_duration.sum --csv`) and/or a `--set full` report.

    python scripts/ncu_summary.py --launches gpurun_out/launches.csv [--skip-setup]
    python scripts/ncu_summary.py --report gpurun_out/prof_k_raytrace.ncu-rep
"""

import argparse
import collections
import csv
import io
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__grid_size",
    "launch__block_size",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_wait_per_warp_active.pct",
    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def to_us(v, unit):
    return {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3,
            "second": v * 1e6, "s": v * 1e6}.get(unit.strip(), v)


def launches(path, skip_prefix=("k_compress", "k_widen", "k_octant_union", "k_group4")):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        if any(p in name for p in skip_prefix):
            continue
        agg[name][0] += 1
        agg[name][1] += to_us(float(r[vi].replace(",", "")), r[ui])
    tot = sum(a[1] for a in agg.values())
    out = [{"kernel": k, "launches": n, "total_us": round(t, 1), "share": round(t / tot, 4)}
           for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
    return {"total_us_excluding_volume_setup": round(tot, 1), "kernels": out}


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, units, vals = r[0], r[1], r[2]
    res = {}
    for m in FULL_METRICS:
        if m in h:
            i = h.index(m)
            res[m] = f"{vals[i]} {units[i]}".strip()
    kn = h.index("Kernel Name") if "Kernel Name" in h else None
    if kn is not None:
        res["kernel"] = vals[kn]
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    a = ap.parse_args()
    out = {}
    if a.launches:
        out["launch_list"] = launches(a.launches)
    if a.report:
        out["full_capture"] = report(a.report)
    json.dump(out, sys.stdout, indent=1)
    print()
