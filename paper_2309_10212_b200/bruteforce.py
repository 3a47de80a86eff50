"""Ground-truth renderer and image comparison (mirrors wavecast/oracle.py).

``reference_render`` is the brute-force single-pass raycaster of
oracle.py:42-122 run on the GPU (csrc/wc_engine.cu k_reference_render):
every ray marches every dual cell of the fully decoded volume with the same
intersection code, so it scales to volumes the CPU brute force cannot.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .codec import CompressedVolume, decompress_blocks_into
from .engine import BASE_COLOR, Framebuffer
from .errors import UsageError
from .traversal import Camera, RaySoA
from .volume import Volume


def decode_full(cv: CompressedVolume) -> Volume:
    """Decode every block into a dense volume, padding dropped (oracle.py:22-39)."""
    nx, ny, nz = cv.dims
    bdx, bdy, bdz = cv.block_dims
    flat = np.empty((cv.block_count, 64), dtype=np.float32)
    decompress_blocks_into(cv, np.arange(cv.block_count, dtype=np.int64), flat)
    grid = flat.reshape(bdz, bdy, bdx, 4, 4, 4).transpose(0, 3, 1, 4, 2, 5).reshape(bdz * 4, bdy * 4, bdx * 4)
    vals = np.ascontiguousarray(grid[:nz, :ny, :nx]).reshape(-1)
    return Volume((nx, ny, nz), vals, (float(vals.min()), float(vals.max())))


def reference_render_compressed(cv: CompressedVolume, cam: Camera, iso: float, w: int, h: int,
                                base_color=BASE_COLOR) -> Framebuffer:
    """Brute force straight from a device-resident compressed volume."""
    rays = RaySoA.from_camera(cam, w, h, cv.dims)
    rgba = np.empty((w * h, 4), dtype=np.uint8)
    depth = np.empty(w * h, dtype=np.float32)
    _lib.call("wc_reference_render", cv.device_handle(), _lib.ptr(np.ascontiguousarray(rays.origin)),
              _lib.ptr(rays.direction), w * h, float(iso), *[float(c) for c in base_color], _lib.ptr(rgba),
              _lib.ptr(depth))
    fb = Framebuffer(w, h, rgba.reshape(h, w, 4), depth.reshape(h, w), 1.0)
    return fb


def reference_render(vol: Volume, cam: Camera, iso: float, w: int, h: int, base_color=BASE_COLOR) -> Framebuffer:
    """oracle.py:93-122 on a dense (decoded) volume, on the GPU."""
    rays = RaySoA.from_camera(cam, w, h, vol.dims)
    rgba = np.empty((w * h, 4), dtype=np.uint8)
    depth = np.empty(w * h, dtype=np.float32)
    vals = np.ascontiguousarray(vol.values, dtype=np.float32)
    _lib.call("wc_reference_render_dense", _lib.ptr(vals), *vol.dims, _lib.ptr(np.ascontiguousarray(rays.origin)),
              _lib.ptr(rays.direction), w * h, float(iso), *[float(c) for c in base_color], _lib.ptr(rgba),
              _lib.ptr(depth))
    return Framebuffer(w, h, rgba.reshape(h, w, 4), depth.reshape(h, w), 1.0)


def compare_images(a: Framebuffer, b: Framebuffer) -> dict:
    """Exhaustive per-pixel diff (oracle.py:125-141)."""
    if (a.w, a.h) != (b.w, b.h):
        raise UsageError(f"framebuffer dims differ: {(a.w, a.h)} vs {(b.w, b.h)}")
    hit_a = np.isfinite(a.depth)
    hit_b = np.isfinite(b.depth)
    both = hit_a & hit_b
    return {
        "hit_mask_mismatches": int(np.count_nonzero(hit_a != hit_b)),
        "max_depth_delta": float(np.abs(a.depth[both] - b.depth[both]).max()) if both.any() else 0.0,
        "max_rgb_delta": int(np.abs(a.rgba[..., :3].astype(np.int16) - b.rgba[..., :3].astype(np.int16)).max()),
    }
