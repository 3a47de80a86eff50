"""The CPU oracle vs the reference's own outputs (tests/golden/, made by
tests/golden/make_golden.py from the unmodified reference).  These pin the
oracle; the GPU tests then compare the CUDA path against the oracle."""

import os

import numpy as np
import pytest

from oracle import oracle as orc

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def cam_tuple(arr):
    return tuple(arr[0:3]), tuple(arr[3:6]), tuple(arr[6:9]), float(arr[9])


def test_codec_kats_all_qbits():
    z = load("codec_kats.npz")
    for q in range(4, 27):
        v = z[f"q{q}_values"]
        pay, rng, _ = orc.compress(v, (8, 8, 8), q)
        assert np.array_equal(pay, z[f"q{q}_payload"]), q
        assert np.array_equal(rng, z[f"q{q}_ranges"]), q
        ov = orc.volume_from_payload((8, 8, 8), q, pay, rng)
        dec = orc.decode_blocks(ov, np.arange(8))
        assert np.array_equal(dec.view(np.uint32), z[f"q{q}_decoded"].view(np.uint32)), q
    for q in (8, 16, 25, 26):
        pay, _, _ = orc.compress(z[f"x{q}_values"], (8, 8, 8), q)
        assert np.array_equal(pay, z[f"x{q}_payload"])
        ov = orc.volume_from_payload((8, 8, 8), q, pay, np.zeros((8, 2), np.float32))
        assert np.array_equal(orc.decode_blocks(ov, np.arange(8)).view(np.uint32), z[f"x{q}_decoded"].view(np.uint32))


def test_zero_block_sentinel_bytes():
    # test_codec.py:23-30: an all-zero block is 00 80 followed by zeros
    pay, _, _ = orc.compress(np.zeros(512, np.float32), (8, 8, 8), 16)
    stride = orc.stride_of(16)
    for b in range(8):
        assert pay[b * stride] == 0x00 and pay[b * stride + 1] == 0x80
        assert not pay[b * stride + 2:(b + 1) * stride].any()


def test_constant_one_block_identity():
    # test_codec.py:33-40: constant 1.0 -> e = 0 and exact 1.0
    pay, rng, e = orc.compress(np.ones(64, np.float32), (4, 4, 4), 16)
    assert e[0] == 0
    ov = orc.volume_from_payload((4, 4, 4), 16, pay, rng)
    assert (orc.decode_blocks(ov, [0]) == 1.0).all()


def _check_frame(z, prefix, ov):
    cam = cam_tuple(z[f"{prefix}camera"])
    w, h, spec, max_spec = (int(x) for x in z[f"{prefix}meta"])
    iso = float(z[f"{prefix}iso"][0])
    o, d = orc.camera_rays(cam, w, h)
    sub = slice(0, None, 61)
    assert np.array_equal(d[sub], z[f"{prefix}ray_dir"]), "camera ray directions"
    sess = orc.Session(ov, o, d, w, h, iso, speculation=bool(spec), max_spec=max_spec,
                       cache_capacity=int(z[f"{prefix}stats"][0][7]) if prefix.startswith("vn") else 0)
    r = sess.rays()
    for k in ("t_enter", "t_exit", "status", "fine_cell", "coarse_cell", "fine_tmax", "coarse_tmax"):
        assert np.array_equal(r[k][sub], z[f"{prefix}ray_{k}"]), k
    stats = []
    p = 0
    while True:
        st = sess.step()
        if st is None:
            break
        if f"{prefix}p{p}_block_slots" in z:
            pb = sess.pass_buffers()
            for k in ("block_slots", "ray_slots", "visible_ids", "active_ids", "sorted_ray_ids", "sorted_hit_slots",
                      "rays_per_block"):
                assert np.array_equal(pb[k], z[f"{prefix}p{p}_{k}"]), (p, k)
            ne = pb["n_entries"]
            assert np.array_equal(pb["rgbz_z"][:ne].view(np.uint32), z[f"{prefix}p{p}_rgbz_z"].view(np.uint32))
            assert np.array_equal(pb["rgbz_rgb"][:ne].view(np.uint32), z[f"{prefix}p{p}_rgbz_rgb"].view(np.uint32))
        stats.append([st["pass_index"], st["n_active_before"], st["n_spec"], st["visible_blocks"],
                      st["active_blocks"], st["new_decompressed"], st["evicted"], st["cache_slots"],
                      st["n_entries"], st["n_active_after"]])
        p += 1
    assert np.array_equal(np.array(stats), z[f"{prefix}stats"])
    rgba, depth = sess.framebuffer()
    assert np.array_equal(rgba, z[f"{prefix}rgba"].reshape(-1, 4))
    assert np.array_equal(depth.view(np.uint32), z[f"{prefix}depth"].reshape(-1).view(np.uint32))
    sess.close()


def test_c1_volume_grids_and_frames():
    """BASELINE.json configs[0]: 64^3 Marschner-Lobb, 256x256, iso 0.5 --
    compressed volume, grids, rays, per-pass stage buffers, stats and final
    RGBA/depth, speculation off and on, identical to the reference."""
    z = load("c1_marschner_lobb.npz")
    dims = tuple(int(x) for x in z["dims"])
    ov = orc.volume_from_payload(dims, int(z["qbits"][0]), z["payload"], z["ranges"])
    assert np.array_equal(ov.bounds, z["bounds"])
    for k in ("fine_min", "fine_max", "coarse_min", "coarse_max"):
        assert np.array_equal(getattr(ov, k), z[f"grid_{k}"]), k
    _check_frame(z, "spec0_", ov)
    _check_frame(z, "spec1_", ov)
    # brute-force oracle.reference_render (oracle.py:93-122)
    cam = cam_tuple(z["spec0_camera"])
    o, d = orc.camera_rays(cam, 256, 256)
    rgba, depth = orc.reference_render(orc.decode_full(ov), o, d, 0.5)
    assert np.array_equal(rgba, z["bruteforce_rgba"].reshape(-1, 4))
    assert np.array_equal(depth, z["bruteforce_depth"].reshape(-1))


def test_c1_volume_synthesis_matches_reference():
    import hashlib

    import paper_2309_10212_b200.volume as V

    z = load("c1_marschner_lobb.npz")
    vol = V.synthesize("marschner_lobb", (64, 64, 64))
    assert hashlib.sha256(vol.values.tobytes()).digest() == bytes(z["values_sha256"])
    pay, rng, _ = orc.compress(vol.values, vol.dims, 16)
    assert np.array_equal(pay, z["payload"]) and np.array_equal(rng, z["ranges"])


def test_eviction_scene_frames():
    z = load("value_noise48_evict.npz")
    dims = tuple(int(x) for x in z["dims"])
    ov = orc.volume_from_payload(dims, int(z["qbits"][0]), z["payload"], z["ranges"])
    cam = cam_tuple(z["camera"])
    w, h, spec, max_spec = (int(x) for x in z["meta"])
    iso = float(z["iso"][0])
    o, d = orc.camera_rays(cam, w, h)
    rgba, depth, st = orc.render(ov, o, d, w, h, iso, max_spec=max_spec, cache_capacity=40)
    got = np.array([[s["pass_index"], s["n_active_before"], s["n_spec"], s["visible_blocks"], s["active_blocks"],
                     s["new_decompressed"], s["evicted"], s["cache_slots"], s["n_entries"], s["n_active_after"]]
                    for s in st])
    assert np.array_equal(got, z["stats"])
    assert got[:, 6].sum() > 0, "scene must exercise eviction"
    assert np.array_equal(rgba, z["rgba"].reshape(-1, 4)) and np.array_equal(depth, z["depth"].reshape(-1))


def test_lru_trace_matches_reference_cache():
    """cache.py:66-111 over 200 random passes (test_cache.py:70-85)."""
    z = load("lru_trace.npz")
    dims = tuple(int(x) for x in z["dims"])
    ov = orc.volume_from_payload(dims, 12, z["payload"], np.zeros((64, 2), np.float32))
    c = orc.Cache(16, ov)
    off = np.concatenate([[0], np.cumsum(z["active_len"])])
    soff = np.concatenate([[0], np.cumsum(z["state_len"])])
    for i in range(len(z["active_len"])):
        ids = z["active_flat"][off[i]:off[i + 1]]
        s = c.ensure_resident(ids)
        assert [s["new_decompressed"], s["evicted"], s["grown_to"]] == list(z["stats"][i]), i
        bos, lu, sv = c.state()
        state = z["state_flat"][soff[i]:soff[i + 1]]
        cap = (len(state) - 1) // 2
        assert np.array_equal(bos, state[:cap]) and np.array_equal(lu, state[cap + 1:]), i
    assert np.array_equal(sv, z["final_slot_values"])


def test_traversal_partial_fill_kat():
    # test_traversal.py:176-191: candidates [b(0,0,0), b(1,0,0), UINT_MAX], exited
    z = load("kats.npz")
    ov = orc.volume_from_payload((8, 8, 8), 16, z["partial_payload"], z["partial_ranges"])
    o = np.repeat([[-5.0, 1.0, 1.0]], 3, axis=0)
    d = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])  # rays 1, 2 miss -> free slots
    s = orc.Session(ov, o, d, 3, 1, 5.0, speculation=True, max_spec=3)
    st = s.step()
    assert st["n_spec"] == 3
    pb = s.pass_buffers()
    assert np.array_equal(pb["block_slots"], z["partial_block_slots"])
    assert list(z["partial_block_slots"]) == [0, 1, orc.UINT_MAX]
    assert s.rays()["exited"][0] == z["partial_exited"][0] == 1
    s.close()


def test_intersection_kats():
    z = load("kats.npz")
    for c, t in zip(z["dd_corners"], z["dd_t"]):
        got = orc.intersect_cell(c, z["dd_o"], z["dd_d"], (0, 0, 0), z["dd_t01"][0], z["dd_t01"][1], 0.0)
        assert got == t
    for c, o, d, (t0, t1, t) in zip(z["rand_corners"], z["rand_o"], z["rand_d"], z["rand_t"]):
        if t0 <= t1:
            got = orc.intersect_cell(c, o, d, (0, 0, 0), t0, t1, 0.1)
            assert (got is None and t == np.inf) or got == t
    # test_blocktrace.py:85-90: linear field -> exactly 0.5
    corners = np.array([-1, 1, -1, 1, -1, 1, -1, 1], np.float32)
    assert orc.intersect_cell(corners, (0.0, 0.5, 0.5), (1.0, 0.0, 0.0), (0, 0, 0), 0.0, 1.0, 0.0) == 0.5


def _ragged(z, name):
    flat, lens = z[f"{name}_flat"], z[f"{name}_len"]
    offs = np.concatenate([[0], np.cumsum(lens)])
    return [flat[offs[i]:offs[i + 1]] for i in range(len(lens))]


@pytest.mark.parametrize("cap", [4, 16])
def test_stage_cache_traces_pin_the_oracle_cache(cap):
    """tests/golden/stage_kats.npz (make_stage_golden.py, the reference
    BlockCache with growth from capacity 4 / 16): the oracle's cache."""
    z = load("stage_kats.npz")
    import paper_2309_10212_b200.volume as V

    vol = V.synthesize("value_noise", (16, 16, 16), seed=5)
    ov = orc.volume_from_values(vol.values, vol.dims, 12)
    c = orc.Cache(cap, ov)
    act, bos, lu = _ragged(z, f"cache{cap}_active"), _ragged(z, f"cache{cap}_block_of_slot"), \
        _ragged(z, f"cache{cap}_last_used")
    for i, ids in enumerate(act):
        s = c.ensure_resident(ids.astype(np.int64))
        assert [s["new_decompressed"], s["evicted"], s["grown_to"]] == list(z[f"cache{cap}_stats"][i]), i
        b, l_, sv = c.state()
        assert np.array_equal(b, bos[i]) and np.array_equal(l_, lu[i]), i
    assert np.array_equal(sv.view(np.uint32), z[f"cache{cap}_final_values"].view(np.uint32))


def test_stage_intersections_pin_the_oracle():
    z = load("stage_kats.npz")
    t01 = z["isec_t01"]
    for i in range(len(t01)):
        if t01[i, 0] > t01[i, 1]:
            continue
        got = orc.intersect_cell(z["isec_corners"][i], z["isec_o"][i], z["isec_d"][i], (0, 0, 0), t01[i, 0],
                                 t01[i, 1], z["isec_iso"][i])
        assert (got is None and z["isec_t"][i] == np.inf) or got == z["isec_t"][i], i


def test_bitmap_helpers_round_trip():
    from paper_2309_10212_b200.bitmaps import mask_to_words, n_words, words_to_mask

    rng = np.random.default_rng(3)
    for n in (0, 1, 31, 32, 33, 64, 1000):
        m = rng.random(n) < 0.3
        w = mask_to_words(m)
        assert w.dtype == np.uint32 and len(w) == n_words(n)
        assert np.array_equal(words_to_mask(w, n), m)
        for b in np.nonzero(m)[0]:
            assert (int(w[b >> 5]) >> int(b & 31)) & 1
