#!/usr/bin/env python
"""Per-stage device time and DRAM traffic per frame from an ncu launch list
taken with
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
over `bench.py --steps 1 --warmup 1 --no-cpu-baseline` (4 frames: warm-up,
timed, e2e warm-up, e2e).  Volume setup kernels are excluded.  ncu replays
each launch cold and serialised, so compare shares, not absolute times.

  python scripts/ncu_frame_traffic.py gpurun_out/launches.csv --frames 4 > profiles/rNN_frame_traffic.json
"""

import argparse
import collections
import csv
import json

STAGE_OF = [
    ("k_traverse", "traverse"),
    ("k_rt_prep", "rt_inputs"), ("k_rt_", "raytrace"), ("k_raytrace", "raytrace"), ("k_contrib", "raytrace"),
    ("k_decode_insert", "cache_decode"), ("k_evict", "cache_decode"), ("k_stamp_hist", "cache_decode"),
    ("k_mark_victims", "cache_decode"), ("SinkList", "cache_decode"), ("SinkBitsIdx", "cache_decode"),
    ("LookupStamp", "mark"),
    ("k_cache_plan", "cache_decode"),
    ("k_iso_bitmap", "reset"), ("k_iso_cell_mask", "reset"), ("k_init_rays", "reset"), ("k_cache_unmap", "reset"),
    ("PredActive", "reset"), ("k_frame_start", "reset"),
    ("k_composite", "composite"), ("SinkCompact<wc::LoadU32>", "composite"),
    ("k_radix", "group"), ("k_run_offsets", "group"),
]
SETUP = ("k_compress", "k_widen", "k_octant_union", "k_group4", "k_range_extent", "k_range_quantize")


def unit_scale(u):
    u = u.strip()
    return {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
            "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--frames", type=int, default=5)  # bench --steps 1 --warmup 1: warm-up, timed, staged, e2e x2
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, vi, ui, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), \
        h.index("Metric Unit"), h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        d = launches.setdefault(r[ii], {"kernel": name})
        d[r[mi]] = float(r[vi].replace(",", "")) * unit_scale(r[ui])
    stage = collections.defaultdict(lambda: {"us": 0.0, "dram_bytes": 0.0, "launches": 0})
    kern = collections.defaultdict(lambda: {"us": 0.0, "dram_bytes": 0.0, "launches": 0})
    for d in launches.values():
        name = d["kernel"]
        if any(s in name for s in SETUP):
            continue
        st = next((s for p, s in STAGE_OF if p in name), "mark")
        if "at::" in name or "elementwise" in name:
            st = "torch (L2 flush, not part of the frame)"
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        for tgt in (stage[st], kern[name]):
            tgt["us"] += d.get("gpu__time_duration.sum", 0.0)
            tgt["dram_bytes"] += b
            tgt["launches"] += 1
    f = a.frames
    out = {
        "source": a.csv,
        "frames": f,
        "per_frame_by_stage": {k: {"us": round(v["us"] / f, 1), "dram_bytes": int(v["dram_bytes"] / f),
                                   "launches": v["launches"] / f} for k, v in stage.items()},
        "per_frame_by_kernel": {k: {"us": round(v["us"] / f, 1), "dram_bytes": int(v["dram_bytes"] / f),
                                    "launches": v["launches"] / f}
                                for k, v in sorted(kern.items(), key=lambda x: -x[1]["us"])},
    }
    json.dump(out, __import__("sys").stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
