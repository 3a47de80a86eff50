"""A small render workload for compute-sanitizer: one scene
through render(), render_passes() (streamed snapshots), the eviction path
and the stage-level API, each checked against the oracle so a sanitizer run
is also a parity run.

  compute-sanitizer --tool memcheck python scripts/sanitize_scene.py c1
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2309_10212_b200 as wc  # noqa: E402
from helpers import host_volume, iso_at, oracle_volume, orbit, wc_camera  # noqa: E402
from oracle import oracle as orc  # noqa: E402

SCENES = {
    # name: (kind, dims, qbits, w, h, iso fraction, speculation, cache)
    "c1": ("marschner_lobb", 64, 16, 256, 256, 0.5, False, None),
    "c1spec": ("marschner_lobb", 64, 16, 256, 256, 0.5, True, None),
    "evict": ("value_noise", 48, 12, 120, 90, 0.35, True, 40),
    "c2s": ("gaussians", 512, 16, 320, 180, 0.3, True, None),  # C2's 512^3 volume at a reduced image
}


def main(name):
    kind, n, qbits, w, h, isof, spec, cache = SCENES[name]
    wc._lib.ensure_device(0)
    if n == 512:
        field = wc.volume.separable_field(kind, (n, n, n), 0)
        cv = wc.compress_separable(field, qbits)
        lo, hi = float(cv.raw_block_ranges[:, 0].min()), float(cv.raw_block_ranges[:, 1].max())
        iso = lo + isof * (hi - lo)
        pay, rng = orc.compress_separable(field.amp, field.fx, field.fy, field.fz, (n, n, n), qbits, 16)
        ov = orc.volume_from_payload((n, n, n), qbits, pay, rng)
    else:
        vol = host_volume(kind, n)
        cv = wc.compress_volume(vol, qbits)
        iso = iso_at(vol, isof)
        ov = oracle_volume(cv)
    grids = wc.build_grids(cv)
    cam_t = orbit(cv.dims, 0.2)
    cam = wc_camera(wc, cam_t)
    opts = wc.RenderOptions(width=w, height=h, speculation=spec, cache_capacity=cache)
    o, d = orc.camera_rays(cam_t, w, h)
    rgba, depth, st = orc.render(ov, o, d, w, h, iso, speculation=spec, cache_capacity=cache or 0)
    for _ in range(2):  # second frame replays the captured pass graphs
        fb, stats = wc.render(cv, grids, cam, iso, opts)
        assert np.array_equal(fb.rgba.reshape(-1, 4), rgba) and np.array_equal(fb.depth.reshape(-1), depth)
        assert len(stats) == len(st)
    frames = [f for f, _ in wc.render_passes(cv, grids, cam, iso, opts)]
    assert np.array_equal(frames[-1].rgba.reshape(-1, 4), rgba)
    if n <= 64:  # stage-level API
        rays = wc.RaySoA.from_camera(cam, w, h, cv.dims)
        offs, _ = wc.prims.exclusive_scan(rays.active_mask.astype(np.uint32))
        wc.traverse_to_next_blocks(rays, grids, iso, 1, offs)
        vis, act = wc.mark_blocks(rays.block_slots, cv.block_dims)
        pb = wc.build_rt_inputs(rays.block_slots, rays.ray_slots, vis)
        cache_ = wc.BlockCache(64)
        cache_.ensure_resident(act, cv)
        assert pb.n_entries == int((rays.block_slots != 0xFFFFFFFF).sum())
    print(f"sanitize scene {name}: {len(stats)} passes, parity ok")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c1")
