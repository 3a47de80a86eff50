"""The CPU oracle vs the LIVE reference package (runs in the build container
where /root/reference exists; skipped on the GPU box).  Broader than the
committed fixtures: 8 scenes x (payload, ranges, grids, rays, every pass's
stats, final frame), random-ray traversal sequences and LRU traces."""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.reference

SCENES = [
    ("marschner_lobb", 64, 16, 256, 256, 0.5, 0.0, False, 64, None),
    ("marschner_lobb", 64, 16, 256, 256, 0.5, 0.0, True, 64, None),
    ("sphere", 64, 16, 96, 96, 0.3, 0.13, True, 64, None),
    ("value_noise", 64, 16, 64, 64, 0.5, 0.4, True, 64, None),
    ("value_noise", 64, 8, 128, 100, 0.5, 0.4, False, 64, None),
    ("value_noise", 48, 12, 120, 90, 0.35, 0.7, True, 64, 40),
    ("marschner_lobb", 41, 26, 90, 70, 0.6, 0.25, True, 64, None),
    ("value_noise", 64, 4, 100, 100, 0.5, 0.1, True, 8, None),
]


@pytest.mark.parametrize("scene", SCENES, ids=[f"{s[0]}-{s[1]}-q{s[2]}-spec{int(s[7])}" for s in SCENES])
def test_scene_bit_exact(ref_wavecast, scene):
    wc = ref_wavecast
    import wavecast.engine as E

    kind, n, q, w, h, isof, camf, spec, max_spec, cap = scene
    vol = wc.synthesize(kind, (n, n, n), seed=3)
    cv = wc.compress_volume(vol, q)
    grids = wc.build_grids(cv)
    pay, rng, _ = orc.compress(vol.values, vol.dims, q)
    assert np.array_equal(pay, cv.payload) and np.array_equal(rng, cv.raw_block_ranges)
    ov = orc.volume_from_payload(cv.dims, q, cv.payload, cv.raw_block_ranges)
    assert np.array_equal(ov.bounds, cv.block_error_bounds)
    for k in ("fine_min", "fine_max", "coarse_min", "coarse_max"):
        assert np.array_equal(getattr(ov, k), getattr(grids, k)), k
    lo, hi = vol.value_range
    iso = lo + isof * (hi - lo)
    c = tuple((d - 1) / 2 for d in cv.dims)
    dist = 1.8 * max(cv.dims)
    ang = 2 * np.pi * camf
    cam = wc.Camera.look_at((c[0] + dist * np.sin(ang), c[1], c[2] + dist * np.cos(ang)), c)
    rays = wc.init_rays(cam, w, h, cv.dims)
    o, d = orc.camera_rays((cam.eye, cam.look_dir, cam.up, cam.fov_y), w, h)
    assert np.array_equal(o, rays.origin) and np.array_equal(d, rays.direction)
    orig = E.initial_capacity
    if cap is not None:
        E.initial_capacity = lambda w_, h_: cap
    try:
        fb, stats = wc.render(cv, grids, cam, iso, wc.RenderOptions(width=w, height=h, speculation=spec,
                                                                    max_spec=max_spec))
    finally:
        E.initial_capacity = orig
    rgba, depth, ost = orc.render(ov, o, d, w, h, iso, speculation=spec, max_spec=max_spec, cache_capacity=cap or 0)
    assert len(stats) == len(ost)
    for a, b in zip(stats, ost):
        for k in ("n_active_before", "n_spec", "visible_blocks", "active_blocks", "new_decompressed", "cache_slots",
                  "utilization", "completeness"):
            assert getattr(a, k) == b[k], k
    assert np.array_equal(fb.rgba.reshape(-1, 4), rgba)
    assert np.array_equal(fb.depth.reshape(-1), depth)


def test_random_ray_traversal_and_frames(ref_wavecast):
    """Arbitrary rays (RaySoA.from_rays) through a value-noise volume: the
    oracle's per-pass slot buffers equal traverse_to_next_blocks'."""
    wc = ref_wavecast
    from wavecast import engine, prims
    from wavecast.traversal import RaySoA, traverse_to_next_blocks

    vol = wc.synthesize("value_noise", (32, 32, 32), seed=31)
    cv = wc.compress_volume(vol, 8)
    grids = wc.build_grids(cv)
    rng = np.random.default_rng(37)
    hi = np.asarray(cv.dims, float) - 1.0
    phi = rng.uniform(0, 2 * np.pi, 400)
    ct = rng.uniform(-1, 1, 400)
    st = np.sqrt(1 - ct**2)
    origins = hi / 2 + (np.linalg.norm(hi) + 10) * np.stack([st * np.cos(phi), st * np.sin(phi), ct], 1)
    dirs = rng.uniform(0.2, 0.8, (400, 3)) * hi - origins
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    iso = float(np.median(vol.values))
    ov = orc.volume_from_payload(cv.dims, 8, cv.payload, cv.raw_block_ranges)
    s = orc.Session(ov, origins, dirs, 400, 1, iso, max_spec=4)
    rays = RaySoA.from_rays(origins, dirs, cv.dims)
    r = s.rays()
    for k in ("t_enter", "t_exit", "status", "fine_cell", "coarse_cell", "fine_tmax", "coarse_tmax"):
        assert np.array_equal(r[k], getattr(rays, k)), k
    while rays.n_active:
        n_act = rays.n_active
        offs, _ = prims.exclusive_scan(rays.active_mask.astype(np.uint32))
        n_spec = engine.compute_n_spec(n_act, 400, 1, 4)
        traverse_to_next_blocks(rays, grids, iso, n_spec, offs)
        st = s.step()
        pb = s.pass_buffers()
        assert st["n_spec"] == n_spec
        assert np.array_equal(pb["block_slots"], rays.block_slots)
        assert np.array_equal(pb["ray_slots"], rays.ray_slots)
        rr = s.rays()
        assert np.array_equal(rr["exited"], rays.exited)
        # mirror the oracle's composite decisions into the reference rays
        rays.status[:] = rr["status"]


def test_lru_matches_reference_simulator(ref_wavecast):
    import sys

    sys.path.insert(0, "/root/reference/pkg/tests")
    from reference_impl import LRUSimulator

    wc = ref_wavecast
    cv = wc.compress_volume(wc.synthesize("value_noise", (16, 16, 16), seed=5), 12)
    ov = orc.volume_from_payload(cv.dims, 12, cv.payload, cv.raw_block_ranges)
    rng = np.random.default_rng(11)
    for cap0 in (1, 3, 16):
        c = orc.Cache(cap0, ov)
        sim = LRUSimulator(cap0)
        for _ in range(150):
            ids = rng.choice(cv.block_count, size=int(rng.integers(1, 30)), replace=False)
            st = c.ensure_resident(ids)
            ref = sim.update(ids)
            assert st["new_decompressed"] == ref["new"] and st["evicted"] == len(ref["victims"])
            assert st["grown_to"] == ref["capacity"]
            bos, _, _ = c.state()
            assert sorted(bos[bos >= 0].tolist()) == sorted(sim.resident)
