"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Every array here is produced by the unmodified reference package
(/root/reference/pkg/src/wavecast) through its own public functions; the
fixtures pin the CPU oracle (oracle/) and, through it, the GPU path.  The
reference cannot travel to the GPU box, the fixtures do.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
import wavecast as wc  # noqa: E402
from wavecast import engine, prims  # noqa: E402
from wavecast.cache import BlockCache  # noqa: E402
from wavecast.traversal import UINT_MAX, RaySoA, traverse_to_next_blocks  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def orbit(dims, frac):
    c = tuple((d - 1) / 2 for d in dims)
    dist = 1.8 * max(dims)
    a = 2 * np.pi * frac
    return wc.Camera.look_at((c[0] + dist * np.sin(a), c[1], c[2] + dist * np.cos(a)), c)


def cam_arrays(cam):
    return np.array([*cam.eye, *cam.look_dir, *cam.up, cam.fov_y], dtype=np.float64)


def frame_fixture(name, cv, cam, iso, w, h, spec, max_spec=64, passes_detail=1):
    """Full render_passes run: final frame, per-pass stats and the first
    passes' stage buffers (slots, block sets, grouped entries, rgbz)."""
    out = {}
    rays = wc.init_rays(cam, w, h, cv.dims)
    sub = slice(0, None, 61)  # every 61st ray keeps the fixture small
    out["ray_dir"] = rays.direction[sub].copy()
    out["ray_t_enter"] = rays.t_enter[sub].copy()
    out["ray_t_exit"] = rays.t_exit[sub].copy()
    out["ray_status"] = rays.status[sub].copy()
    out["ray_fine_cell"] = rays.fine_cell[sub].copy()
    out["ray_coarse_cell"] = rays.coarse_cell[sub].copy()
    out["ray_fine_tmax"] = rays.fine_tmax[sub].copy()
    out["ray_coarse_tmax"] = rays.coarse_tmax[sub].copy()
    stats = []
    # replay of engine.render_passes keeping stage buffers of early passes
    grids = wc.build_grids(cv)
    n = rays.n
    fb = engine.Framebuffer.blank(w, h)
    cache = BlockCache(engine.initial_capacity(w, h))
    rgbz_rgb = np.zeros((n, 3), np.float32)
    rgbz_z = np.full(n, np.inf, np.float32)
    p = 0
    while rays.n_active:
        n_act = rays.n_active
        offs, _ = prims.exclusive_scan(rays.active_mask.astype(np.uint32))
        n_spec = engine.compute_n_spec(n_act, w, h, max_spec) if spec else 1
        traverse_to_next_blocks(rays, grids, iso, n_spec, offs)
        vis, act = engine.mark_blocks(rays.block_slots, cv.block_dims)
        cst = cache.ensure_resident(act, cv)
        pb = engine.build_rt_inputs(rays.block_slots, rays.ray_slots, vis)
        rgbz_z.fill(np.inf)
        rgbz_rgb.fill(0.0)
        if len(pb.visible_ids):
            contrib, coords, cells = engine._contributor_table(cv, cache, pb.visible_ids)
            engine._raytrace_visible_kernel(pb.visible_ids, pb.rays_per_block, pb.block_ray_offsets,
                                            pb.sorted_ray_ids, pb.sorted_hit_slots, contrib, cache.slot_values,
                                            coords, cells, rays.origin, rays.direction, rays.t_enter, float(iso),
                                            0.85, 0.85, 0.85, rgbz_rgb, rgbz_z)
        engine.composite(rgbz_rgb, rgbz_z, rays, n_spec, offs, pb.valid_prefix, fb)
        stats.append([p, n_act, n_spec, int(vis.sum()), int(act.sum()), cst.new_decompressed, cst.evicted,
                      cst.grown_to, pb.n_entries, rays.n_active])
        if p < passes_detail:
            out[f"p{p}_block_slots"] = rays.block_slots.copy()
            out[f"p{p}_ray_slots"] = rays.ray_slots.copy()
            out[f"p{p}_visible_ids"] = np.nonzero(vis)[0].astype(np.uint32)
            out[f"p{p}_active_ids"] = np.nonzero(act)[0].astype(np.uint32)
            out[f"p{p}_sorted_ray_ids"] = pb.sorted_ray_ids
            out[f"p{p}_sorted_hit_slots"] = pb.sorted_hit_slots
            out[f"p{p}_rays_per_block"] = pb.rays_per_block
            out[f"p{p}_rgbz_z"] = rgbz_z[: pb.n_entries].copy()
            out[f"p{p}_rgbz_rgb"] = rgbz_rgb[: pb.n_entries].copy()
        p += 1
    # cross-check the replay against the public generator
    ref_fb, ref_stats = wc.render(cv, grids, cam, iso, wc.RenderOptions(width=w, height=h, speculation=spec,
                                                                        max_spec=max_spec))
    assert np.array_equal(ref_fb.rgba, fb.rgba) and np.array_equal(ref_fb.depth, fb.depth)
    assert [s.n_active_before for s in ref_stats] == [s[1] for s in stats]
    out["rgba"] = fb.rgba
    out["depth"] = fb.depth
    out["stats"] = np.array(stats, dtype=np.int64)
    out["utilization"] = np.array([s.utilization for s in ref_stats])
    out["completeness"] = np.array([s.completeness for s in ref_stats])
    out["camera"] = cam_arrays(cam)
    out["meta"] = np.array([w, h, int(spec), max_spec], dtype=np.int64)
    out["iso"] = np.array([iso])
    return out


def volume_fixture(cv):
    return {
        "dims": np.array(cv.dims, np.int64),
        "qbits": np.array([cv.qbits], np.int64),
        "payload": cv.payload,
        "ranges": cv.raw_block_ranges,
        "bounds": cv.block_error_bounds,
    }


def main():
    fixtures = {}

    # ---- C1: 64^3 Marschner-Lobb, 256x256, iso 0.5 (BASELINE.json configs[0])
    vol = wc.synthesize("marschner_lobb", (64, 64, 64))
    cv = wc.compress_volume(vol, 16)
    g = wc.build_grids(cv)
    c1 = volume_fixture(cv)
    import hashlib

    c1["values_sha256"] = np.frombuffer(hashlib.sha256(vol.values.tobytes()).digest(), np.uint8)
    c1.update({f"grid_{k}": getattr(g, k) for k in ("fine_min", "fine_max", "coarse_min", "coarse_max")})
    cam = orbit(cv.dims, 0.0)
    for spec in (False, True):
        f = frame_fixture("c1", cv, cam, 0.5, 256, 256, spec, passes_detail=1)
        c1.update({f"spec{int(spec)}_{k}": v for k, v in f.items()})
    dec = wc.decode_full(cv)
    ref = wc.reference_render(dec, cam, 0.5, 256, 256)
    c1["bruteforce_rgba"] = ref.rgba
    c1["bruteforce_depth"] = ref.depth
    np.savez_compressed(os.path.join(HERE, "c1_marschner_lobb.npz"), **c1)

    # ---- value-noise scene with eviction pressure (cache budget 40 slots)
    vol = wc.synthesize("value_noise", (48, 48, 48), seed=3)
    cv = wc.compress_volume(vol, 12)
    vn = volume_fixture(cv)
    lo, hi = vol.value_range
    iso = lo + 0.35 * (hi - lo)
    cam = orbit(cv.dims, 0.7)
    orig = engine.initial_capacity
    engine.initial_capacity = lambda w_, h_: 40
    try:
        f = frame_fixture("vn", cv, cam, iso, 120, 90, True, passes_detail=1)
    finally:
        engine.initial_capacity = orig
    vn.update(f)
    np.savez_compressed(os.path.join(HERE, "value_noise48_evict.npz"), **vn)

    # ---- codec KATs: qbits 4..26 on 8x8x8 uniform(-100, 100) volumes
    codec = {}
    rng = np.random.default_rng(3)
    for q in range(4, 27):
        v = rng.uniform(-100.0, 100.0, (8, 8, 8)).astype(np.float32)
        if q == 10:
            v[:4, :4, :4] = 0.0  # zero-sentinel block
        volq = wc.volume.Volume((8, 8, 8), v.reshape(-1), (float(v.min()), float(v.max())))
        cq = wc.compress_volume(volq, q)
        codec[f"q{q}_values"] = v.reshape(-1)
        codec[f"q{q}_payload"] = cq.payload
        codec[f"q{q}_ranges"] = cq.raw_block_ranges
        codec[f"q{q}_decoded"] = np.stack([wc.decompress_block(cq, b) for b in range(cq.block_count)])
    # extreme exponents (float64 decode fallback)
    v = np.zeros((8, 8, 8), np.float32)
    v[:4, :4, :4] = (np.float32(3e-38) * np.linspace(-1, 1, 64).astype(np.float32)).reshape(4, 4, 4)
    v[4:, 4:, 4:] = (np.float32(3e38) * np.linspace(-1, 1, 64).astype(np.float32)).reshape(4, 4, 4)
    for q in (8, 16, 25, 26):
        volq = wc.volume.Volume((8, 8, 8), v.reshape(-1), (float(v.min()), float(v.max())))
        cq = wc.compress_volume(volq, q)
        codec[f"x{q}_values"] = v.reshape(-1)
        codec[f"x{q}_payload"] = cq.payload
        codec[f"x{q}_decoded"] = np.stack([wc.decompress_block(cq, b) for b in range(cq.block_count)])
    np.savez_compressed(os.path.join(HERE, "codec_kats.npz"), **codec)

    # ---- LRU traces (cache.py) : 200 random passes, capacity 16
    vol = wc.synthesize("value_noise", (16, 16, 16), seed=5)
    cvl = wc.compress_volume(vol, 12)
    rng = np.random.default_rng(47)
    cache = BlockCache(16)
    trace = {"payload": cvl.payload, "dims": np.array(cvl.dims), "qbits": np.array([12])}
    act_lists, stats, resid = [], [], []
    for _ in range(200):
        k = int(rng.integers(1, 25))
        ids = np.sort(rng.choice(cvl.block_count, size=k, replace=False))
        m = np.zeros(cvl.block_count, bool)
        m[ids] = True
        s = cache.ensure_resident(m, cvl)
        act_lists.append(ids)
        stats.append([s.new_decompressed, s.evicted, s.grown_to])
        resid.append(np.concatenate([cache.block_of_slot, [-2], cache.last_used_pass]))
    trace["active_flat"] = np.concatenate(act_lists)
    trace["active_len"] = np.array([len(a) for a in act_lists])
    trace["stats"] = np.array(stats)
    trace["state_flat"] = np.concatenate(resid)
    trace["state_len"] = np.array([len(r) for r in resid])
    trace["final_slot_values"] = cache.slot_values
    np.savez_compressed(os.path.join(HERE, "lru_trace.npz"), **trace)

    # ---- traversal / intersection / grouping KATs from the reference tests
    kats = {}
    v = np.zeros((8, 8, 8), np.float32)
    v[0, 0, 0] = 10.0
    v[0, 0, 4] = 10.0
    vk = wc.volume.Volume((8, 8, 8), v.reshape(-1), (0.0, 10.0))
    cvk = wc.compress_volume(vk, 16)
    gk = wc.build_grids(cvk)
    o = np.repeat([[-5.0, 1.0, 1.0]], 3, axis=0)
    d = np.repeat([[1.0, 0.0, 0.0]], 3, axis=0)
    rays = RaySoA.from_rays(o, d, cvk.dims)
    rays.status[1:] = 2
    offs, _ = prims.exclusive_scan(rays.active_mask.astype(np.uint32))
    traverse_to_next_blocks(rays, gk, 5.0, 3, offs)
    kats["partial_payload"] = cvk.payload
    kats["partial_ranges"] = cvk.raw_block_ranges
    kats["partial_block_slots"] = rays.block_slots.copy()
    kats["partial_exited"] = rays.exited.copy()
    # intersection: linear field midpoint + frozen double-dip cases (test_blocktrace.py:85-119)
    inv = 1.0 / math.sqrt(3.0)
    cases = np.array([
        [0.12882564961910248, -0.031002115458250046, 0.7976475358009338, -0.8279751539230347,
         0.39230889081954956, -0.34403541684150696, -0.6491804718971252, 0.349597305059433],
        [0.3825429677963257, 0.8259482383728027, 0.6456142663955688, -0.6418746113777161,
         0.4964485466480255, -0.826637327671051, -0.14828751981258392, -0.2064962238073349],
        [0.14086264371871948, 0.30610644817352295, -0.6372244358062744, -0.06068112701177597,
         0.9843357801437378, -0.9682947397232056, -0.2580127716064453, -0.3313750624656677],
    ], dtype=np.float32)
    from wavecast.blocktrace import _cell_overlap
    oo = (-0.1 * inv, -0.1 * inv, -0.1 * inv)
    dd = (inv, inv, inv)
    t0, t1 = _cell_overlap(*oo, *dd, 0.0, 0.0, 0.0)
    kats["dd_corners"] = cases
    kats["dd_o"] = np.array(oo)
    kats["dd_d"] = np.array(dd)
    kats["dd_t01"] = np.array([t0, t1])
    kats["dd_t"] = np.array([wc.intersect_cell(c, oo, dd, (0, 0, 0), t0, t1, 0.0) for c in cases])
    rng = np.random.default_rng(99)
    rc = rng.uniform(-1, 1, (400, 8)).astype(np.float32)
    ro = rng.uniform(-0.5, 1.5, (400, 3))
    rd = rng.normal(size=(400, 3))
    rd /= np.linalg.norm(rd, axis=1, keepdims=True)
    rt = []
    for i in range(400):
        a, b = _cell_overlap(*ro[i], *rd[i], 0.0, 0.0, 0.0)
        t = wc.intersect_cell(rc[i], ro[i], rd[i], (0, 0, 0), a, b, 0.1) if a <= b else None
        rt.append([a, b, np.inf if t is None else t])
    kats["rand_corners"] = rc
    kats["rand_o"] = ro
    kats["rand_d"] = rd
    kats["rand_t"] = np.array(rt)
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **kats)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
