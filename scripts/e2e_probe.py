"""Where render()'s end-to-end time goes at C3 (diagnostic): device frame time
vs wall time per call, the pass the framebuffer copy starts after, and the
host patch.  WAVECAST_TRACE=1 prints render_to_host's own split."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2309_10212_b200 as wc  # noqa: E402
from paper_2309_10212_b200.benchmark import orbit_camera  # noqa: E402

wc._lib.ensure_device(0)
wl = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c3")
field = wc.volume.separable_field(wl["kind"], wl["dims"], wl["seed"])
cv = wc.compress_separable(field, wl["qbits"])
grids = wc.build_grids(cv)
lo, hi = float(cv.raw_block_ranges[:, 0].min()), float(cv.raw_block_ranges[:, 1].max())
iso = lo + wl["iso_frac"] * (hi - lo)
cam = orbit_camera(wl["dims"], 0, 1)
opts = wc.RenderOptions(width=wl["w"], height=wl["h"])
for i in range(12):
    t = time.perf_counter()
    fb, st = wc.render(cv, grids, cam, iso, opts)
    wall = (time.perf_counter() - t) * 1e3
    s = wc.engine.session_pool.get(cv, grids, opts, cam)
    print(f"render {i}: wall {wall:.3f} ms  device frame {s.frame_ms():.3f} ms  passes {len(st)}", flush=True)

if os.environ.get("PROBE_PROFILE"):
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    for i in range(50):
        wc.render(cv, grids, cam, iso, opts)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
