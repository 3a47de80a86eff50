"""GPU parity: the sm_100a render path vs the CPU oracle, bit for bit.

Every test calls through the C ABI (libwavecast_b200.so via the package's
public API) and compares with oracle/ (the CPU restatement pinned against
the reference's own golden vectors in tests/golden/).  Bar: bit-exact for
voxels, ray state, slot buffers, block sets, cache residency, grouped
entries, RGBZ, RGBA and depth.
"""

import numpy as np
import pytest

from helpers import host_volume, iso_at, lockstep, oracle_volume, orbit
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wc():
    import paper_2309_10212_b200 as wc

    wc._lib.ensure_device(0)
    return wc


# ----------------------------------------------------------------- codec
@pytest.mark.parametrize("qbits", [4, 7, 11, 16, 20, 25, 26])
def test_compress_and_decode_bit_exact(wc, qbits):
    rng = np.random.default_rng(qbits)
    vals = rng.uniform(-100.0, 100.0, (13, 10, 9)).astype(np.float32)
    vals[:4, :4, :4] = 0.0  # an all-zero block -> sentinel
    vol = wc.volume.make_volume((9, 10, 13), vals)
    cv = wc.compress_volume(vol, qbits)
    pay, rng_, _ = orc.compress(vol.values, vol.dims, qbits)
    assert np.array_equal(cv.payload, pay), "GPU compressor payload"
    assert np.array_equal(cv.raw_block_ranges.view(np.uint32), rng_.view(np.uint32)), "GPU ranges"
    ov = oracle_volume(cv)
    ids = np.arange(cv.block_count)
    got = np.empty((cv.block_count, 64), np.float32)
    wc.decompress_blocks_into(cv, ids, got)
    assert np.array_equal(got.view(np.uint32), orc.decode_blocks(ov, ids).view(np.uint32))


def test_decode_extreme_exponents(wc):
    # tiny and huge magnitudes exercise the float64 fallback (subnormal / e>127)
    vals = np.zeros((8, 8, 8), np.float32)
    vals[:4, :4, :4] = np.float32(3e-38) * np.linspace(-1, 1, 64).reshape(4, 4, 4).astype(np.float32)
    vals[4:, 4:, 4:] = np.float32(3e38) * np.linspace(-1, 1, 64).reshape(4, 4, 4).astype(np.float32)
    vals[:4, 4:, :4] = np.float32(1e-30)
    vol = wc.volume.make_volume((8, 8, 8), vals)
    for qbits in (8, 16, 25, 26):
        cv = wc.compress_volume(vol, qbits)
        pay, _, _ = orc.compress(vol.values, vol.dims, qbits)
        assert np.array_equal(cv.payload, pay)
        ids = np.arange(cv.block_count)
        got = np.empty((cv.block_count, 64), np.float32)
        wc.decompress_blocks_into(cv, ids, got)
        assert np.array_equal(got.view(np.uint32), orc.decode_blocks(oracle_volume(cv), ids).view(np.uint32))


def test_grids_bit_exact(wc):
    vol = host_volume("value_noise", (37, 29, 45))
    cv = wc.compress_volume(vol, 12)
    g = wc.build_grids(cv)
    ov = oracle_volume(cv)
    for k in ("fine_min", "fine_max", "coarse_min", "coarse_max"):
        assert np.array_equal(getattr(g, k), getattr(ov, k)), k


def test_separable_synthesis_matches_host(wc):
    f = wc.turbulence_field((40, 36, 44), seed=1)
    cv = wc.compress_separable(f, 16)
    pay, rng_, _ = orc.compress(f.evaluate().reshape(-1), f.dims, 16)
    assert np.array_equal(cv.payload, pay)
    assert np.array_equal(cv.raw_block_ranges, rng_)


# ------------------------------------------------------------- full frames
SCENES = [
    # kind, n, qbits, w, h, iso frac, camera frac, speculation, max_spec, cache
    ("marschner_lobb", 64, 16, 256, 256, 0.5, 0.0, False, 64, None),   # C1
    ("marschner_lobb", 64, 16, 256, 256, 0.5, 0.0, True, 64, None),
    ("sphere", 64, 16, 96, 96, 0.3, 0.13, True, 64, None),
    ("value_noise", 64, 16, 64, 64, 0.5, 0.4, True, 64, None),
    ("value_noise", 64, 8, 128, 100, 0.5, 0.4, False, 64, None),
    ("value_noise", 48, 12, 120, 90, 0.35, 0.7, True, 64, 40),          # heavy eviction
    ("value_noise", 48, 12, 96, 72, 0.5, 0.3, False, 64, 48),           # eviction across many pass stamps
    ("marschner_lobb", 41, 26, 90, 70, 0.6, 0.25, True, 64, None),     # qbits 26 fallback
    ("value_noise", 64, 4, 100, 100, 0.5, 0.1, True, 8, None),
    ("gaussians", 96, 16, 160, 90, 0.3, 0.0, True, 64, None),
    ("turbulence", (72, 64, 60), 16, 128, 72, 0.5, 0.3, True, 64, 1024),
    ("value_noise", 128, 12, 12, 12, 0.5, 0.2, True, 64, None),        # few rays per block: sparse extraction
    ("value_noise", 112, 10, 14, 11, 0.45, 0.6, False, 64, 40),         # ... with eviction
    # rows of whole bitmap words (bdx % 32 == 0): word-level active marking,
    # +x carries across words and the row / plane edges
    ("turbulence", (256, 40, 36), 16, 120, 90, 0.5, 0.2, True, 64, None),
    ("gaussians", (128, 72, 56), 16, 96, 80, 0.3, 0.35, True, 64, None),
    ("value_noise", (256, 36, 28), 12, 96, 72, 0.5, 0.3, True, 64, 60),  # ... with eviction
]


@pytest.mark.parametrize("scene", SCENES, ids=[f"{s[0]}-{s[1] if isinstance(s[1], int) else 'x'.join(map(str, s[1]))}-q{s[2]}-{s[3]}x{s[4]}-spec{int(s[7])}" for s in SCENES])
def test_render_lockstep_vs_oracle(wc, scene):
    kind, n, qbits, w, h, isof, camf, spec, max_spec, cache = scene
    vol = host_volume(kind, n, seed=1 if kind == "turbulence" else (0 if kind == "gaussians" else 3))
    cv = wc.compress_volume(vol, qbits)
    ov = oracle_volume(cv)
    lockstep(wc, cv, ov, orbit(cv.dims, camf), w, h, iso_at(vol, isof), speculation=spec, max_spec=max_spec,
             cache_capacity=cache)


def test_long_ray_handoff_lockstep(wc):
    """Passes of <= 150K short rays (n_spec < 16) hand rays still walking
    after 12 iterations to the warp-per-ray k_traverse_long: an isovalue near
    the top of the range leaves long empty walks, so the hand-off runs, and
    every pass still equals the oracle's bit for bit."""
    from paper_2309_10212_b200 import debug

    vol = host_volume("value_noise", 256, seed=3)
    cv = wc.compress_volume(vol, 12)
    ov = oracle_volume(cv)
    handed = []
    lockstep(wc, cv, ov, orbit(cv.dims, 0.15), 256, 256, iso_at(vol, 0.93), max_spec=8,
             probe=lambda sess, p: handed.append(debug.sizes(sess)["n_handed_off"]))
    assert sum(handed) > 0, f"no ray was handed off ({handed})"


@pytest.mark.parametrize("bound", ["fine_min", "fine_max"])
def test_iso_on_a_grid_bound(wc, bound):
    # iso exactly equal to a float64 grid bound: the 16-bit screening bitmap
    # (Volume::fine_q) must fall through to the exact test for that block
    vol = host_volume("value_noise", 40, seed=5)
    cv = wc.compress_volume(vol, 12)
    g = wc.build_grids(cv)
    vals = np.sort(getattr(g, bound)[np.isfinite(getattr(g, bound))])
    iso = float(vals[len(vals) // 2])
    ov = oracle_volume(cv)
    lockstep(wc, cv, ov, orbit(cv.dims, 0.2), 64, 48, iso, speculation=True, max_spec=64, cache_capacity=None)


def test_render_api_matches_generator(wc):
    vol = host_volume("value_noise", 64)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    cam = wc.Camera.look_at((31.5, 31.5, 31.5 + 115.2), (31.5, 31.5, 31.5))
    opts = wc.RenderOptions(width=80, height=60)
    fb, stats = wc.render(cv, grids, cam, iso_at(vol, 0.5), opts)
    last = None
    prev_written = None
    for snap, ps in wc.render_passes(cv, grids, cam, iso_at(vol, 0.5), opts):
        written = np.isfinite(snap.depth)
        if prev_written is not None:  # pixels, once written, never change
            assert np.array_equal(snap.rgba[prev_written], last.rgba[prev_written])
        last, prev_written = snap, written
    assert np.array_equal(last.rgba, fb.rgba) and np.array_equal(last.depth, fb.depth)
    assert last.completeness == 1.0 == fb.completeness


def test_speculation_invariance(wc):
    vol = host_volume("value_noise", 64)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    cam = wc.Camera.look_at((31.5 + 115.2 * np.sin(0.8 * np.pi), 31.5, 31.5 + 115.2 * np.cos(0.8 * np.pi)),
                            (31.5, 31.5, 31.5))
    iso = iso_at(vol, 0.5)
    on, s_on = wc.render(cv, grids, cam, iso, wc.RenderOptions(width=64, height=64, speculation=True))
    off, s_off = wc.render(cv, grids, cam, iso, wc.RenderOptions(width=64, height=64, speculation=False))
    assert np.array_equal(on.rgba, off.rgba) and np.array_equal(on.depth, off.depth)
    assert len(s_on) <= len(s_off) and all(s.n_spec == 1 for s in s_off)


def test_camera_misses_volume(wc):
    cv = wc.compress_volume(host_volume("sphere", 64), 16)
    cam = wc.Camera((31.5, 31.5, 200.0), (0.0, 0.0, 1.0), (0.0, 1.0, 0.0), 45.0)
    fb, stats = wc.render(cv, wc.build_grids(cv), cam, 20.0, wc.RenderOptions(width=16, height=16))
    assert stats == [] and fb.completeness == 1.0 and not np.isfinite(fb.depth).any()


def test_iso_outside_range_single_pass(wc):
    cv = wc.compress_volume(host_volume("sphere", 64), 16)
    cam = wc.Camera.look_at((31.5, 31.5, 31.5 + 115.2), (31.5, 31.5, 31.5))
    fb, stats = wc.render(cv, wc.build_grids(cv), cam, 1000.0, wc.RenderOptions(width=32, height=32))
    assert len(stats) == 1 and fb.completeness == 1.0 and not np.isfinite(fb.depth).any()


def test_arbitrary_rays_lockstep(wc):
    vol = host_volume("value_noise", 32)
    cv = wc.compress_volume(vol, 8)
    rng = np.random.default_rng(37)
    hi = np.asarray(cv.dims, float) - 1.0
    phi = rng.uniform(0, 2 * np.pi, 500)
    ct = rng.uniform(-1, 1, 500)
    st = np.sqrt(1 - ct**2)
    origins = hi / 2 + (np.linalg.norm(hi) + 10) * np.stack([st * np.cos(phi), st * np.sin(phi), ct], 1)
    d = rng.uniform(0.2, 0.8, (500, 3)) * hi - origins
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    lockstep(wc, cv, oracle_volume(cv), None, 500, 1, float(np.median(vol.values)), origins=origins, dirs=d,
             max_spec=4)


def test_more_passes_than_histogram_bins(wc):
    """Speculation off on rays that graze a long slab of candidate blocks: one
    pass per block (> 64 passes, past the device-kept stamp histogram, so the
    later passes take the host-recount path), with a small cache that evicts
    every pass.  Every pass's buffers and cache state are compared."""
    nx, ny, nz = 448, 16, 12
    y = np.arange(ny, dtype=np.float64)
    f = np.sin(2 * np.pi * y / 8.0).astype(np.float32)  # varies in y only
    vol = wc.volume.make_volume((nx, ny, nz), np.broadcast_to(f[None, :, None], (nz, ny, nx)))
    cv = wc.compress_volume(vol, 12)
    rng = np.random.default_rng(11)
    n = 48
    origins = np.stack([np.full(n, -5.0), rng.uniform(2.1, 2.9, n), rng.uniform(0.5, nz - 1.5, n)], 1)
    origins[: n // 3, 1] = rng.uniform(0.2, 15.0, n // 3)  # these rays cross the surface early
    d = np.stack([np.ones(n), rng.uniform(-2e-4, 2e-4, n), rng.uniform(-1e-3, 1e-3, n)], 1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    stats, _, _ = lockstep(wc, cv, oracle_volume(cv), None, n, 1, 0.5, origins=origins, dirs=d,
                           speculation=False, cache_capacity=40)
    assert len(stats) > 70, len(stats)


def test_corrupt_cache_hook_breaks_parity(wc):
    vol = host_volume("sphere", 64)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    cam = wc.Camera.look_at((31.5, 31.5, 31.5 + 115.2), (31.5, 31.5, 31.5))
    good, _ = wc.render(cv, grids, cam, 20.0, wc.RenderOptions(width=48, height=48))
    bad, _ = wc.render(cv, grids, cam, 20.0, wc.RenderOptions(width=48, height=48, corrupt_cache=True))
    assert wc.compare_images(good, bad)["hit_mask_mismatches"] > 0


def test_tile_sharding_stitches_bit_exact(wc):
    """N interleaved tile sessions on one GPU, stitched == one full frame
    (the multi-GPU decomposition)."""
    from paper_2309_10212_b200 import dist

    vol = host_volume("gaussians", 96, seed=0)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    cam = wc.Camera.look_at((47.5, 47.5, 47.5 + 1.8 * 96), (47.5, 47.5, 47.5))
    w, h = 150, 110
    iso = iso_at(vol, 0.3)
    full, _ = wc.render(cv, grids, cam, iso, wc.RenderOptions(width=w, height=h))
    for world in (2, 3, 4, 8):
        rgba = np.zeros((h * w, 4), np.uint8)
        depth = np.zeros(h * w, np.float32)
        for rank in range(world):
            pix = dist.tile_pixels(w, h, rank, world, tile=16)
            with wc.RenderSession(cv, grids, cam, iso, wc.RenderOptions(width=w, height=h), pixel_ids=pix) as s:
                s.run()
                r, d = s.read()
            rgba[pix] = r
            depth[pix] = d
        assert np.array_equal(rgba.reshape(h, w, 4), full.rgba), world
        assert np.array_equal(depth.reshape(h, w), full.depth), world


# ------------------------------------------------------------- brute force
def test_brute_force_reference_render(wc):
    vol = host_volume("sphere", 64)
    cv = wc.compress_volume(vol, 16)
    cam_t = orbit(cv.dims, 0.13)
    cam = wc.Camera(*cam_t)
    dec = wc.decode_full(cv)
    w = h = 96
    ref = wc.reference_render(dec, cam, 20.0, w, h)
    o, d = orc.camera_rays(cam_t, w, h)
    rgba, depth = orc.reference_render(dec.as_3d(), o, d, 20.0)
    assert np.array_equal(ref.rgba.reshape(-1, 4), rgba)
    assert np.array_equal(ref.depth.reshape(-1), depth)
    fb, _ = wc.render(cv, wc.build_grids(cv), cam, 20.0, wc.RenderOptions(width=w, height=h))
    diff = wc.compare_images(fb, ref)  # test_engine.py:155-163
    assert diff["hit_mask_mismatches"] == 0 and diff["max_rgb_delta"] == 0 and diff["max_depth_delta"] <= 1e-3


# --------------------------------------------------------------- prims
def test_prims_scan_sort(wc):
    rng = np.random.default_rng(5)
    for n in (0, 1, 7, 2048, 2049, 100000, 1 << 20, 3_000_017):  # > 1184 tiles: several tiles per CTA
        v = rng.integers(0, 1000, n).astype(np.uint32)
        out, tot = wc.prims.exclusive_scan(v)
        ref = np.concatenate([[0], np.cumsum(v.astype(np.uint64))[:-1]]).astype(np.uint32) if n else v
        assert np.array_equal(out, ref) and tot == int(v.astype(np.uint64).sum())
        keys = rng.integers(0, 50, n).astype(np.uint32)
        vals = np.arange(n, dtype=np.uint32)
        k2, v2 = wc.prims.sort_by_key(keys, vals)
        order = np.argsort(keys, kind="stable")
        assert np.array_equal(k2, keys[order]) and np.array_equal(v2, vals[order])


def test_session_reset_reuses_allocations(wc):
    """render() pools sessions: a reset with a new camera / iso must equal a
    fresh oracle render (cache, rays and framebuffer all reset)."""
    vol = host_volume("value_noise", 48)
    cv = wc.compress_volume(vol, 12)
    ov = oracle_volume(cv)
    grids = wc.build_grids(cv)
    opts = wc.RenderOptions(width=72, height=56, cache_capacity=64)
    for i, (frac, isof) in enumerate([(0.1, 0.4), (0.6, 0.55), (0.1, 0.4), (0.35, 0.3)]):
        cam_t = orbit(cv.dims, frac)
        fb, stats = wc.render(cv, grids, wc.Camera(*cam_t), iso_at(vol, isof), opts)
        o, d = orc.camera_rays(cam_t, 72, 56)
        rgba, depth, ost = orc.render(ov, o, d, 72, 56, iso_at(vol, isof), cache_capacity=64)
        assert np.array_equal(fb.rgba.reshape(-1, 4), rgba), i
        assert np.array_equal(fb.depth.reshape(-1), depth), i
        assert [s.new_decompressed for s in stats] == [s["new_decompressed"] for s in ost], i
        assert [s.cache_slots for s in stats] == [s["cache_slots"] for s in ost], i


# ------------------------------------------------- volume I/O (§8(f) row 2)
def test_load_wcz_streams_to_device(wc, tmp_path):
    vol = host_volume("value_noise", (150, 131, 170), seed=2)
    cv = wc.compress_volume(vol, 16)
    p = tmp_path / "v.wcz"
    wc.write_wcz(cv, p)
    # 1 MiB chunks: the 10 MB payload crosses both pinned buffers many times
    dv = wc.codec.load_wcz(p, chunk_bytes=1 << 20)
    assert dv.dims == cv.dims and dv.qbits == 16
    assert np.array_equal(dv.payload, cv.payload)
    assert np.array_equal(dv.raw_block_ranges.view(np.uint32), cv.raw_block_ranges.view(np.uint32))
    g0, g1 = wc.build_grids(cv), wc.build_grids(dv)
    for k in ("fine_min", "fine_max", "coarse_min", "coarse_max"):
        assert np.array_equal(getattr(g0, k), getattr(g1, k)), k
    with pytest.raises(wc.DataError):
        (tmp_path / "t.wcz").write_bytes(p.read_bytes()[:-3])
        wc.codec.load_wcz(tmp_path / "t.wcz")


def test_volume_alloc_fill_finalize_matches_upload(wc):
    # the receiving side of dist.broadcast_volume on one GPU: allocate, write
    # payload + ranges into the device buffers through __cuda_array_interface__
    # views, finalize -> same grids as a volume uploaded from the host
    import ctypes as C

    import torch

    from paper_2309_10212_b200 import _lib, dist

    vol = host_volume("sphere", 48)
    cv = wc.compress_volume(vol, 12)
    h = C.c_void_p()
    _lib.call("wc_volume_alloc", *cv.dims, cv.qbits, C.byref(h))
    rv = wc.CompressedVolume(cv.dims, cv.qbits, handle=h)
    pp, pb, rp, rb = C.c_void_p(), C.c_uint64(), C.c_void_p(), C.c_uint64()
    _lib.call("wc_volume_device_buffers", h, C.byref(pp), C.byref(pb), C.byref(rp), C.byref(rb))
    assert pb.value == cv.payload.nbytes and rb.value == cv.raw_block_ranges.nbytes
    torch.as_tensor(dist._DeviceBytes(pp.value, pb.value), device="cuda").copy_(torch.from_numpy(cv.payload))
    torch.as_tensor(dist._DeviceBytes(rp.value, rb.value), device="cuda").copy_(
        torch.from_numpy(cv.raw_block_ranges.reshape(-1).view(np.uint8)))
    torch.cuda.synchronize()
    _lib.call("wc_volume_finalize", h)
    assert np.array_equal(rv.payload, cv.payload)
    g0, g1 = wc.build_grids(cv), wc.build_grids(rv)
    for k in ("fine_min", "fine_max", "coarse_min", "coarse_max"):
        assert np.array_equal(getattr(g0, k), getattr(g1, k)), k


def test_decoded_value_range_matches_oracle(wc):
    for kind, n, q in (("value_noise", (37, 29, 45), 16), ("gaussians", 40, 9)):
        vol = host_volume(kind, n, seed=0)
        cv = wc.compress_volume(vol, q)
        dense = orc.decode_full(oracle_volume(cv))
        lo, hi = wc.codec.decoded_value_range(cv)
        assert (lo, hi) == (float(dense.min()), float(dense.max()))


# --------------------------------------------- bench protocol (§8(f) row 4)
def test_bench_report_matches_reference(wc):
    # cmd_bench's report (cli.py:136-195) from the device path equals the one
    # the reference wrote for the same .wcz and arguments
    # (tests/golden/make_bench_golden.py)
    import json
    import os

    from paper_2309_10212_b200.benchmark import bench_report

    here = os.path.join(os.path.dirname(__file__), "golden")
    gold = json.load(open(os.path.join(here, "bench_small_report.json")))
    a = gold["args"]
    kw = {a[i].lstrip("-").replace("-", "_"): int(a[i + 1]) for i in range(0, len(a), 2)}
    cv = wc.read_wcz(os.path.join(here, "bench_small.wcz"))
    rep, tim = bench_report(cv, wc.build_grids(cv), volume="bench_small.wcz", **kw)
    assert rep == gold["report"]
    assert len(tim["frame_ms"]) == rep["n_renders"] and all(t > 0 for t in tim["frame_ms"])


def test_repeated_renders_with_overlapped_readback(wc):
    # render() reuses a pooled session: from its second frame the framebuffer
    # copy starts after the pass that (last frame) left <= 1/8 of the rays
    # active and the still-active pixels are patched afterwards.  Every frame
    # must equal the step-by-step generator's final frame.
    vol = host_volume("value_noise", 64, seed=4)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    opts = wc.RenderOptions(width=96, height=80)
    for k, frac in enumerate((0.0, 0.0, 0.3, 0.55, 0.55)):
        eye, look, up, fov = orbit(cv.dims, frac)
        cam = wc.Camera(tuple(eye), tuple(look), tuple(up), fov)
        iso = iso_at(vol, 0.45 + 0.05 * (k % 2))
        fb, stats = wc.render(cv, grids, cam, iso, opts)
        last = None
        for snap, _ in wc.render_passes(cv, grids, cam, iso, opts):
            last = snap
        assert np.array_equal(fb.rgba, last.rgba) and np.array_equal(fb.depth, last.depth), k
        assert len(stats) >= 2


def test_split_range_tests_assemble_to_the_whole(wc):
    # dist.render_frame_split on one GPU: the per-iso range tests computed in
    # 3 coarse-cell slices (wc_session_reset_part), assembled as the NCCL
    # all-gather would, give the same frame as the whole reset
    import torch

    from paper_2309_10212_b200 import dist

    vol = host_volume("value_noise", (96, 80, 72), seed=6)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    eye, look, up, fov = orbit(cv.dims, 0.15)
    cam = wc.Camera(tuple(eye), tuple(look), tuple(up), fov)
    iso = iso_at(vol, 0.5)
    opts = wc.RenderOptions(width=72, height=64)
    s = wc.RenderSession(cv, grids, cam, iso, opts)
    ref = s.render_frame(cam, iso)
    rgba0, depth0 = (x.copy() for x in s.read())
    parts = 3
    cb, cm, chunk = s.mask_buffers(parts)
    bits = torch.as_tensor(dist._DeviceBytes(cb, 4 * chunk * parts), device="cuda")
    masks = torch.as_tensor(dist._DeviceBytes(cm, 8 * 32 * chunk * parts), device="cuda")
    acc_b, acc_m = torch.zeros_like(bits), torch.zeros_like(masks)
    for part in range(parts):
        s.reset_part(cam, iso, part, parts)
        s.sync()
        pb, pm = 4 * chunk, 8 * 32 * chunk
        acc_b[part * pb:(part + 1) * pb] = bits[part * pb:(part + 1) * pb]
        acc_m[part * pm:(part + 1) * pm] = masks[part * pm:(part + 1) * pm]
    bits.copy_(acc_b)
    masks.copy_(acc_m)
    torch.cuda.synchronize()
    stats = s.run()
    rgba1, depth1 = s.read()
    assert [x.n_active_before for x in stats] == [x.n_active_before for x in ref]
    assert np.array_equal(rgba0, rgba1) and np.array_equal(depth0, depth1)
    s.close()


# The product path per pass: ray-ordered entries (no grouping) with every pass
# replayed as a captured CUDA graph, over two frames on one session (the
# second frame replays the graphs the first captured).
GRAPH_SCENES = [
    ("marschner_lobb", 64, 16, 256, 256, 0.5, 0.0, False, 64, None),
    ("value_noise", 64, 16, 64, 64, 0.5, 0.4, True, 64, None),
    ("value_noise", 48, 12, 120, 90, 0.35, 0.7, True, 64, 40),
    ("turbulence", (256, 40, 36), 16, 120, 90, 0.5, 0.2, True, 64, None),
    ("value_noise", 128, 12, 12, 12, 0.5, 0.2, True, 64, None),
]


@pytest.mark.parametrize("scene", GRAPH_SCENES, ids=[f"{s[0]}-{s[3]}x{s[4]}-spec{int(s[7])}" for s in GRAPH_SCENES])
def test_graph_replay_ungrouped_lockstep(wc, scene):
    kind, n, qbits, w, h, isof, camf, spec, max_spec, cache = scene
    vol = host_volume(kind, n, seed=1 if kind == "turbulence" else (0 if kind == "gaussians" else 3))
    cv = wc.compress_volume(vol, qbits)
    ov = oracle_volume(cv)
    lockstep(wc, cv, ov, orbit(cv.dims, camf), w, h, iso_at(vol, isof), speculation=spec, max_spec=max_spec,
             cache_capacity=cache, group=False,
             frames=[(orbit(cv.dims, camf + 0.31), iso_at(vol, isof * 0.9 + 0.05)),
                     (orbit(cv.dims, camf), iso_at(vol, isof))])
