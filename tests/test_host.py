"""Host-side logic of the package (no GPU): camera validation, container I/O,
speculation count, tile sharding, synthetic generators."""

import math

import numpy as np
import pytest

import paper_2309_10212_b200 as wc
from paper_2309_10212_b200 import dist, volume
from paper_2309_10212_b200.codec import CompressedVolume, block_stride_bytes, error_bound, quant_scale


def test_compute_n_spec_kats():  # test_engine.py:28-33
    assert wc.compute_n_spec(1280 * 720, 1280, 720) == 1
    assert wc.compute_n_spec(2, 3, 2) == 3
    assert wc.compute_n_spec(100, 1280, 720) == 64
    assert wc.compute_n_spec(100, 1280, 720, max_spec=128) == 128
    assert wc.compute_n_spec(5, 2, 2) == 1


def test_camera_validation():  # test_traversal.py:40-49
    with pytest.raises(wc.UsageError):
        wc.Camera((0, 0, 0), (0, 0, 2.0), (0, 1, 0), 45.0)
    with pytest.raises(wc.UsageError):
        wc.Camera((0, 0, 0), (0, 0, 1.0), (0, 0, -1.0), 45.0)
    with pytest.raises(wc.UsageError):
        wc.Camera.look_at((1, 2, 3), (1, 2, 3))
    assert wc.Camera.look_at((0, 0, 10), (0, 0, 0)).look_dir == (0.0, 0.0, -1.0)


def test_camera_c_struct_matches_reference_basis():
    cam = wc.Camera.look_at((10.0, 3.0, 200.0), (31.5, 31.5, 31.5), fov_y=35.0)
    c = cam.to_c(640, 480)
    look = np.asarray(cam.look_dir)
    right = np.cross(look, np.asarray(cam.up))
    right /= np.linalg.norm(right)
    assert list(c.right) == list(right)
    assert list(c.up) == list(np.cross(right, look))
    assert c.tan_half == math.tan(math.radians(35.0) * 0.5)


def test_stride_and_scale():  # test_codec.py:138-144
    for q in range(4, 27):
        s = block_stride_bytes(q)
        assert s % 4 == 0 and s * 8 >= 16 + 64 * q
    assert block_stride_bytes(16) == 132 and quant_scale(8) == 127
    assert error_bound(0, 16) == 1.0 / (2 * 32767)


def test_qbits_checked():
    with pytest.raises(wc.UsageError):
        CompressedVolume((4, 4, 4), 3, payload=np.zeros(100, np.uint8))
    with pytest.raises(wc.UsageError):
        CompressedVolume((4, 4, 4), 27, payload=np.zeros(100, np.uint8))


def _host_cv(dims, q, seed=7):
    from oracle import oracle as orc

    rng = np.random.default_rng(seed)
    v = rng.uniform(-3, 7, int(np.prod(dims))).astype(np.float32)
    pay, ranges, _ = orc.compress(v, dims, q)
    return CompressedVolume(dims, q, payload=pay, raw_block_ranges=ranges)


def test_wcz_round_trip(tmp_path):  # test_codec.py:147-162
    cv = _host_cv((9, 10, 11), 14)
    p = tmp_path / "v.wcz"
    wc.write_wcz(cv, p)
    assert p.stat().st_size == 28 + 8 * cv.block_count + cv.block_count * cv.block_stride_bytes
    back = wc.read_wcz(p)
    assert back.dims == cv.dims and back.qbits == 14 and back.block_dims == cv.block_dims
    assert np.array_equal(back.payload, cv.payload)
    assert np.array_equal(back.raw_block_ranges, cv.raw_block_ranges)
    assert np.array_equal(back.block_error_bounds, cv.block_error_bounds)


def test_wcz_errors(tmp_path):
    p = tmp_path / "bad.wcz"
    p.write_bytes(b"NOPE" + bytes(40))
    with pytest.raises(wc.DataError):
        wc.read_wcz(p)
    cv = _host_cv((8, 8, 8), 10)
    good = tmp_path / "g.wcz"
    wc.write_wcz(cv, good)
    blob = good.read_bytes()
    (tmp_path / "t.wcz").write_bytes(blob[:-1])
    with pytest.raises(wc.DataError):
        wc.read_wcz(tmp_path / "t.wcz")
    bad_stride = bytearray(blob)
    bad_stride[24:28] = (999).to_bytes(4, "little")
    (tmp_path / "s.wcz").write_bytes(bytes(bad_stride))
    with pytest.raises(wc.DataError):
        wc.read_wcz(tmp_path / "s.wcz")


def test_native_wcz_probe_matches_read_wcz(tmp_path):
    # the device loader's header checks (wc_wcz_probe, host only) raise what
    # read_wcz raises, with the reference's messages (codec.py:246-262)
    cv = _host_cv((9, 10, 11), 14)
    good = tmp_path / "g.wcz"
    wc.write_wcz(cv, good)
    assert wc.codec.probe_wcz(good) == ((9, 10, 11), 14, cv.block_stride_bytes, cv.block_count)
    blob = good.read_bytes()
    nb = cv.block_count
    cases = {
        "magic.wcz": (b"NOPE" + blob[4:], wc.DataError, "not a WCZ1 container"),
        "short.wcz": (blob[:20], wc.DataError, "not a WCZ1 container"),
        "version.wcz": (blob[:4] + (2).to_bytes(4, "little") + blob[8:], wc.DataError,
                        "unsupported container version 2"),
        "qbits.wcz": (blob[:20] + (30).to_bytes(4, "little") + blob[24:], wc.UsageError,
                      "qbits must be in [4, 26], got 30"),
        "stride.wcz": (blob[:24] + (999).to_bytes(4, "little") + blob[28:], wc.DataError,
                       "stride 999 inconsistent with qbits 14"),
        "size.wcz": (blob[:-1], wc.DataError,
                     f"expected {28 + 8 * nb + nb * cv.block_stride_bytes} bytes, found {len(blob) - 1}"),
    }
    for name, (data, exc, msg) in cases.items():
        p = tmp_path / name
        p.write_bytes(data)
        for fn in (wc.read_wcz, wc.codec.probe_wcz):
            with pytest.raises(exc) as ei:
                fn(p)
            assert msg in str(ei.value), (name, fn.__name__, str(ei.value))
            if exc is wc.DataError:
                assert str(ei.value).startswith(str(p)), str(ei.value)


def test_block_id_round_trip():  # test_codec.py:71-83
    cv = _host_cv((16, 16, 16), 8)
    assert cv.block_dims == (4, 4, 4) and cv.block_id(1, 2, 3) == 57
    for b in range(cv.block_count):
        assert cv.block_id(*cv.block_coords(b)) == b
    with pytest.raises(IndexError):
        cv.block_id(4, 0, 0)


def test_raw_volume_io(tmp_path):
    vol = wc.synthesize("sphere", (9, 10, 11))
    p = tmp_path / "v.raw"
    wc.save_raw(vol, p)
    back = wc.load_raw(p, (9, 10, 11), "f32")
    assert np.array_equal(back.values, vol.values)
    with pytest.raises(wc.DataError):
        wc.load_raw(p, (9, 10, 12), "f32")
    with pytest.raises(wc.UsageError):
        wc.load_raw(p, (9, 10, 11), "f64")


def test_tile_pixels_partition():
    w, h = 150, 97
    for world in (1, 2, 3, 4, 8):
        parts = [dist.tile_pixels(w, h, r, world, 16) for r in range(world)]
        allp = np.concatenate(parts)
        assert len(allp) == w * h and len(np.unique(allp)) == w * h
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 16 * 16 * 4  # round-robin tiles balance (edge tiles are partial)


def test_oracle_tile_deal_matches_product():
    from oracle import oracle as orc

    for world in (1, 3, 8):
        for r in range(world):
            assert np.array_equal(dist.tile_pixels(1920, 1080, r, world, 32).astype(np.int64),
                                  orc.tile_pixels(1920, 1080, r, world, 32))


def test_separable_fields_evaluate_in_float32_order():
    f = volume.turbulence_field((10, 9, 8), seed=1)
    dense = f.evaluate()
    x, y, z = 7, 3, 5
    v = np.float32(0.0)
    for k in range(len(f.amp)):
        v = np.float32(v + np.float32(np.float32(np.float32(f.amp[k] * f.fz[k][z]) * f.fy[k][y]) * f.fx[k][x]))
    assert dense[z, y, x] == v
    g = volume.gaussians_field((12, 12, 12))
    assert len(g.amp) == 24 and g.evaluate().dtype == np.float32


def test_generators_deterministic():
    for kind in ("sphere", "marschner_lobb", "value_noise", "gaussians", "turbulence"):
        a = wc.synthesize(kind, (12, 10, 9), seed=2)
        b = wc.synthesize(kind, (12, 10, 9), seed=2)
        assert np.array_equal(a.values, b.values)
    with pytest.raises(wc.UsageError):
        wc.synthesize("sphere", (4, 8, 8))
    with pytest.raises(wc.UsageError):
        wc.synthesize("nope", (8, 8, 8))
