#!/usr/bin/env python
"""Copy the outputs of scripts/gpu_evidence_r2b.sh (gpurun_out/ev_*) into the
tracked profiles/r02_* files: bench lines, the C2 speculation sweep, the GPU
test log, the per-frame ncu traffic and the --set full summaries of the top
kernels.

    python scripts/collect_evidence_r2.py [--src gpurun_out] [--dst profiles]
"""

import argparse
import json
import os
import shutil
import subprocess
import sys

BENCH = ["c2", "c3", "c4", "c5", "c3_spec1", "shard1", "share2", "share4", "share8", "reference"]
FULL = {
    "traverse": "k_traverse<2>, its 5th launch in bench.py --steps 1 --warmup 1 = pass 0 of the second frame "
                "(956,484 rays, n_spec 2; thread per ray)",
    "rt_find": "k_rt_find, 5th launch (pass 0 of the second frame)",
    "decode_insert": "k_decode_insert (bulk-copy pipeline), 5th launch",
    "mark_extract": "k_mark_extract<2> (visible + active extraction in one launch), 5th launch",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--src", default="gpurun_out")
    ap.add_argument("--dst", default="profiles")
    args = ap.parse_args()
    here = os.path.dirname(os.path.abspath(__file__))
    for name in BENCH:
        line = open(os.path.join(args.src, f"ev_{name}.json")).read().strip().splitlines()[-1]
        json.loads(line)  # one JSON line
        with open(os.path.join(args.dst, f"r02_bench_{name}.json"), "w") as f:
            f.write(line + "\n")
    sweep = {"what": "C2 (512^3 Gaussians, 1920x1080) at max_spec 1..64: bench.py --config c2 --max-spec M "
                     "--steps 10 --warmup 3", "lines": {}}
    for m in (1, 2, 4, 8, 16, 32, 64):
        d = json.loads(open(os.path.join(args.src, f"ev_c2_ms{m}.json")).read().strip().splitlines()[-1])
        sweep["lines"][str(m)] = {k: d.get(k) for k in ("ms_per_step", "passes", "pass_ms", "stage_ms_per_frame",
                                                         "clocks")}
        sweep["lines"][str(m)]["ms_per_frame"] = sweep["lines"][str(m)].pop("ms_per_step")
    json.dump(sweep, open(os.path.join(args.dst, "r02_c2_spec_sweep.json"), "w"), indent=1)
    shutil.copy(os.path.join(args.src, "ev_gpu_tests.log"), os.path.join(args.dst, "r02_gpu_tests.log"))
    shutil.copy(os.path.join(args.src, "ev_launches.csv"), os.path.join(args.dst, "r02_launches.csv"))
    traffic = subprocess.run([sys.executable, os.path.join(here, "ncu_frame_traffic.py"),
                              os.path.join(args.src, "ev_launches.csv"), "--frames", "4"],
                             check=True, capture_output=True, text=True).stdout
    open(os.path.join(args.dst, "r02_frame_traffic.json"), "w").write(traffic)
    for k, what in FULL.items():
        out = subprocess.run([sys.executable, os.path.join(here, "ncu_summary.py"), "--report",
                              os.path.join(args.src, f"ev_full_k_{k}.ncu-rep")],
                             capture_output=True, text=True).stdout
        d = json.loads(out)
        d = {"what": f"ncu --set full --clock-control none of {what}, cold caches, serialised", **d}
        json.dump(d, open(os.path.join(args.dst, f"r02_ncu_full_k_{k}.json"), "w"), indent=1)
    # the traversal summary bench.py cites in its roofline (r02_k_traverse_ncu.json)
    p = os.path.join(args.dst, "r02_k_traverse_ncu.json")
    d = json.load(open(p))
    f = json.load(open(os.path.join(args.dst, "r02_ncu_full_k_traverse.json")))["full_capture"]
    num = lambda k: float(f[k].split()[0])
    d["duration_us"] = num("gpu__time_duration.sum")
    d["dram_bytes_per_launch"] = int(round((num("dram__bytes_read.sum") + num("dram__bytes_write.sum")) * 1e6))
    d["dram_gbs"] = round(d["dram_bytes_per_launch"] / d["duration_us"] / 1e3, 1)
    d["warp_exec_threads_per_instr"] = num("smsp__thread_inst_executed_per_inst_executed.ratio")
    d["warp_exec_efficiency"] = round(d["warp_exec_threads_per_instr"] / 32, 4)
    d["l2_hit_rate"] = num("lts__t_sector_hit_rate.pct") / 100
    d["l1_hit_rate"] = num("l1tex__t_sector_hit_rate.pct") / 100
    d["warps_active"] = num("sm__warps_active.avg.pct_of_peak_sustained_active") / 100
    d["issue_active"] = num("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100
    d["fp64_pipe"] = num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100
    d["registers"] = f["launch__registers_per_thread"]
    json.dump(d, open(p, "w"), indent=1)
    print("collected into", args.dst)


if __name__ == "__main__":
    main()
