"""Golden report of the reference's bench protocol (cli.py:122-195) on a
small volume, for tests/test_gpu_parity.py::test_bench_report_matches_reference.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_bench_golden.py

Writes bench_small.wcz (the reference's compress_volume of a 40^3
value-noise field) and bench_small_report.json (cmd_bench's report,
produced by the reference's own cmd_bench through its CLI entry point).
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import wavecast as wc  # noqa: E402
from wavecast import cli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
ARGS = ["--isovalues", "3", "--orbit-steps", "4", "--seed", "5", "--width", "48", "--height", "32"]


def main():
    vol = wc.synthesize("value_noise", (40, 40, 40), seed=2)
    cv = wc.compress_volume(vol, 16)
    wcz = os.path.join(HERE, "bench_small.wcz")
    wc.write_wcz(cv, wcz)
    out = os.path.join(HERE, "bench_small_report.json")
    rc = cli.main(["bench", "--volume", wcz, *ARGS, "--report", out])
    assert rc == 0
    with open(out) as f:
        rep = json.load(f)
    rep["config"]["volume"] = "bench_small.wcz"  # path-independent
    with open(out, "w") as f:
        json.dump({"args": ARGS, "report": rep}, f, indent=2, sort_keys=True)
    print("wrote", wcz, out)


if __name__ == "__main__":
    main()
