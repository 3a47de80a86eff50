"""Is the per-frame reset host-bound?  Times, on a C3 session, the host
enqueue of wc_session_reset, a reset + sync, and 20 back-to-back resets."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import bench
import paper_2309_10212_b200 as wc
from paper_2309_10212_b200 import engine
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
s = engine.RenderSession(cv, grids, cam, iso, opts)
s.run()
s.sync()
for rep in range(3):
    t0 = time.perf_counter(); s.reset(cam, iso); t1 = time.perf_counter(); s.sync(); t2 = time.perf_counter()
    print(f"reset enqueue {1e3*(t1-t0):.3f} ms, enqueue+sync {1e3*(t2-t0):.3f} ms")
    t0 = time.perf_counter()
    for _ in range(20):
        s.reset(cam, iso)
    t1 = time.perf_counter(); s.sync(); t2 = time.perf_counter()
    print(f"20 resets: enqueue {1e3*(t1-t0)/20:.3f} ms each, total/20 {1e3*(t2-t0)/20:.3f} ms")
    t0 = time.perf_counter(); s.render_frame(cam, iso); t1 = time.perf_counter(); s.sync(); t2 = time.perf_counter()
    print(f"frame: enqueue {1e3*(t1-t0):.3f} ms, total {1e3*(t2-t0):.3f} ms, device frame_ms {s.frame_ms():.3f}")
