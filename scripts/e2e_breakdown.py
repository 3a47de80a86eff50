"""Where the e2e time of render() goes at C3: wall time of the public call,
the C call alone, the device frame time, and (WAVECAST_TRACE=1) the
read-back timings printed by the library."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2309_10212_b200 as wc
from paper_2309_10212_b200.benchmark import orbit_camera

wc._lib.ensure_device(0)
f = wc.volume.separable_field("turbulence", (2048, 2048, 1920), 1)
cv = wc.compress_separable(f, 16)
g = wc.build_grids(cv)
r = cv.raw_block_ranges
lo, hi = float(r[:, 0].min()), float(r[:, 1].max())
iso = lo + 0.5 * (hi - lo)
cam = orbit_camera(cv.dims, 0, 1)
opts = wc.RenderOptions(width=1920, height=1080)
for i in range(8):
    wc.render(cv, g, cam, iso, opts)
s = wc.engine.session_pool.items[-1][1]
walls, calls = [], []
for i in range(10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fb, st = wc.render(cv, g, cam, iso, opts)
    t1 = time.perf_counter()
    walls.append((t1 - t0) * 1e3)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s.render_frame_host(cam, iso)
    t3 = time.perf_counter()
    calls.append((t3 - t2) * 1e3)
    print(f"render() {walls[-1]:.3f} ms  render_frame_host {calls[-1]:.3f} ms  device frame {s.frame_ms():.3f} ms")
walls.sort(); calls.sort()
print(f"median render() {walls[5]:.3f}  median C call {calls[5]:.3f}")
