"""Top SASS lines by warp-stall samples of an ncu --set full report.

  python scripts/ncu_hot.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"
body = [r for r in rows[hi + 1:] if len(r) > ix[S] and r[ix[S]] not in ("", "0")]
tot = sum(float(r[ix[S]]) for r in body)
body.sort(key=lambda r: -float(r[ix[S]]))
print(f"total samples {tot:.0f}")
for r in body[:n]:
    print(f"{float(r[ix[S]]) / tot * 100:5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:100]}")
