"""Streamed per-pass snapshots of render_passes (engine.py:308-382, the
snapshot per pass of engine.py:62-63 and service.py:192-216): every yielded
frame equals the oracle's framebuffer after the same pass, whether the
consumer reads it at once, later, out of order, or never."""

import numpy as np
import pytest

from helpers import host_volume, iso_at, oracle_volume, orbit, wc_camera
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wc():
    import paper_2309_10212_b200 as wc

    wc._lib.ensure_device(0)
    return wc


def oracle_frames(ov, cam_tuple, w, h, iso, spec):
    o, d = orc.camera_rays(cam_tuple, w, h)
    s = orc.Session(ov, o, d, w, h, iso, speculation=spec)
    frames = []
    while s.step() is not None:
        rgba, depth = s.framebuffer()
        frames.append((rgba.copy(), depth.copy()))
    s.close()
    return frames


@pytest.mark.parametrize("mode", ["immediate", "late_reverse", "skip_odd"])
@pytest.mark.parametrize("spec", [False, True])
def test_streamed_snapshots_equal_oracle_per_pass(wc, mode, spec):
    vol = host_volume("value_noise", 64)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    cam_t = orbit(cv.dims, 0.4)
    w, h = 96, 80
    iso = iso_at(vol, 0.5)
    ref = oracle_frames(oracle_volume(cv), cam_t, w, h, iso, spec)
    cam = wc_camera(wc, cam_t)
    opts = wc.RenderOptions(width=w, height=h, speculation=spec)
    got = []
    for k, (fb, ps) in enumerate(wc.render_passes(cv, grids, cam, iso, opts)):
        assert ps.pass_index == k
        if mode == "immediate":
            got.append((fb.rgba.reshape(-1, 4).copy(), fb.depth.reshape(-1).copy()))
        else:
            got.append(fb)
    assert len(got) == len(ref) and len(ref) >= (6 if not spec else 2)
    order = range(len(got) - 1, -1, -1) if mode == "late_reverse" else range(len(got))
    for k in order:
        if mode == "skip_odd" and k % 2:
            continue
        g = got[k] if mode == "immediate" else (got[k].rgba.reshape(-1, 4), got[k].depth.reshape(-1))
        assert np.array_equal(g[0], ref[k][0]), f"pass {k} rgba"
        assert np.array_equal(g[1].view(np.uint32), ref[k][1].view(np.uint32)), f"pass {k} depth"


def test_streamed_snapshots_many_passes_held(wc):
    """A speculation-off run holding every frame (more frames than the
    pinned pool recycles once rays get long), all exact."""
    vol = host_volume("value_noise", 64)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    cam_t = orbit(cv.dims, 0.0)
    w, h = 128, 128
    iso = iso_at(vol, 0.5)
    ref = oracle_frames(oracle_volume(cv), cam_t, w, h, iso, False)
    cam = wc_camera(wc, cam_t)
    frames = [fb for fb, _ in wc.render_passes(cv, grids, cam, iso, wc.RenderOptions(width=w, height=h,
                                                                                    speculation=False))]
    assert len(frames) == len(ref) >= 6
    for k, fb in enumerate(frames):
        assert np.array_equal(fb.rgba.reshape(-1, 4), ref[k][0]), k
        assert np.array_equal(fb.depth.reshape(-1).view(np.uint32), ref[k][1].view(np.uint32)), k
        snap = fb.snapshot()
        assert np.array_equal(snap.rgba, fb.rgba) and snap.completeness == fb.completeness


@pytest.mark.parametrize("host_patch", [False, True])
def test_render_host_readback_equals_oracle(wc, monkeypatch, host_patch):
    """render()'s read-back: the bulk copy starts before the last passes and
    the pixels still active then are patched -- by the GPU straight into the
    pinned host framebuffer, or (WAVECAST_HOST_PATCH=1, and for pageable
    buffers) on the host.  Frames after the first (which choose the copy's
    pass from the previous frame's pass times) equal the oracle's."""
    if host_patch:
        monkeypatch.setenv("WAVECAST_HOST_PATCH", "1")
    else:
        monkeypatch.delenv("WAVECAST_HOST_PATCH", raising=False)
    vol = host_volume("value_noise", 96, seed=4)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    ov = oracle_volume(cv)
    w, h = 320, 240
    opts = wc.RenderOptions(width=w, height=h)
    for k, frac in enumerate((0.1, 0.1, 0.35, 0.6)):
        cam_t = orbit(cv.dims, frac)
        cam = wc_camera(wc, cam_t)
        iso = iso_at(vol, 0.45 + 0.05 * k)
        if k == 0:
            sess = wc.RenderSession(cv, grids, cam, iso, opts)  # a session of its own (the env is read at creation)
        stats, rgba, depth = sess.render_frame_host(cam, iso)
        o, d = orc.camera_rays(cam_t, w, h)
        orgba, odepth, _ = orc.render(ov, o, d, w, h, iso)
        assert np.array_equal(rgba.reshape(-1, 4), orgba), (host_patch, k)
        assert np.array_equal(depth.reshape(-1).view(np.uint32), odepth.view(np.uint32)), (host_patch, k)
    sess.close()
