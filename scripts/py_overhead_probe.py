import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import bench
import paper_2309_10212_b200 as wc
from paper_2309_10212_b200 import _lib, engine
from paper_2309_10212_b200.benchmark import orbit_camera
wc._lib.ensure_device(0)
wl = bench.workload("c3")
field = wc.volume.separable_field(wl["kind"], wl["dims"], wl["seed"])
cv = wc.compress_separable(field, wl["qbits"])
grids = wc.build_grids(cv)
lo, hi = float(cv.raw_block_ranges[:, 0].min()), float(cv.raw_block_ranges[:, 1].max())
iso = lo + wl["iso_frac"] * (hi - lo)
cam = orbit_camera(wl["dims"], 0, 1)
opts = wc.RenderOptions(width=wl["w"], height=wl["h"])
orig_call = _lib.call
tc = []
def timed_call(name, *args):
    t = time.perf_counter()
    r = orig_call(name, *args)
    if name == "wc_session_render_host":
        tc.append(time.perf_counter() - t)
    return r
_lib.call = timed_call
engine._lib.call = timed_call
for i in range(30):
    t = time.perf_counter()
    fb, st = wc.render(cv, grids, cam, iso, opts)
    wall = time.perf_counter() - t
    s = engine.session_pool.get(cv, grids, opts, cam)
    if i >= 10:
        print(f"wall {wall*1e3:.3f}  C call {tc[-1]*1e3:.3f}  python {1e3*(wall - tc[-1]):.3f}  device {s.frame_ms():.3f}")
