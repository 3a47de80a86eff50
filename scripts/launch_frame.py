"""Print the kernels of the last frame of an ncu launch list with their
device time (us) and DRAM bytes, one line per launch, pass by pass.

  python scripts/launch_frame.py gpurun_out/launches.csv [--frame -1]
"""
import argparse
import collections
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--frame", type=int, default=-1, help="which frame (by k_init_rays launches)")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = L.setdefault(r[ii], {"k": r[ki]})
    v = float(r[vi].replace(",", ""))
    u = r[ui].strip()
    v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
    d[r[mi]] = v
ks = list(L.values())
starts = [i for i, d in enumerate(ks) if "k_init_rays" in d["k"]]
s0 = starts[a.frame]
s1 = starts[a.frame + 1] if a.frame + 1 < len(starts) and a.frame != -1 else len(ks)
tot = 0.0
p = -1
for d in ks[s0:s1]:
    name = d["k"].split("(")[0].replace("void ", "").replace("wc::", "")
    if "k_traverse" in name:
        p += 1
        print(f"--- pass {p}")
    t = d.get("gpu__time_duration.sum", 0.0)
    b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot += t
    print(f"{t:9.1f} us {b / 1e6:9.1f} MB  {name[:90]}")
print(f"total {tot:.1f} us")
