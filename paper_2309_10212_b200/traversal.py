"""Camera, ray state and traversal entry points (mirrors wavecast/traversal.py).

Geometry (traversal.py:3-11): voxel values at integer coordinates, the
volume spans [0, dims-1]^3, fine cells are 4 voxels (one block), coarse
cells 16.  The camera basis and tan(fov/2) are computed here on the host
with the reference's own numpy expressions (traversal.py:65-70, :111); the
per-pixel rays, slab clipping and iterator seeding run on the GPU
(csrc/wc_engine.cu k_init_rays) in the same float64 operation order.
"""

from __future__ import annotations

import ctypes as C
import functools
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import UsageError

UINT_MAX = 0xFFFFFFFF
STATUS_ACTIVE = 0
STATUS_HIT = 1
STATUS_MISS = 2
ENTRY_EPS = 4e-4
FINE_CELL = 4.0
COARSE_CELL = 16.0


@dataclass(frozen=True)
class Camera:
    """Pinhole camera; look_dir and up must be unit length (traversal.py:38-70)."""

    eye: tuple[float, float, float]
    look_dir: tuple[float, float, float]
    up: tuple[float, float, float]
    fov_y: float

    def __post_init__(self):
        ld = np.asarray(self.look_dir, dtype=np.float64)
        if abs(np.linalg.norm(ld) - 1.0) > 1e-6:
            raise UsageError("camera look_dir must be unit length")
        if np.linalg.norm(np.cross(ld, np.asarray(self.up, dtype=np.float64))) < 1e-9:
            raise UsageError("camera up is parallel to look_dir")

    @classmethod
    def look_at(cls, eye, target, up=(0.0, 1.0, 0.0), fov_y=45.0) -> "Camera":
        eye = np.asarray(eye, dtype=np.float64)
        ld = np.asarray(target, dtype=np.float64) - eye
        norm = np.linalg.norm(ld)
        if norm < 1e-12:
            raise UsageError("camera eye coincides with look-at target")
        ld = ld / norm
        return cls(tuple(eye), tuple(ld), tuple(np.asarray(up, dtype=np.float64)), float(fov_y))

    def basis(self):
        look = np.asarray(self.look_dir, dtype=np.float64)
        right = np.cross(look, np.asarray(self.up, dtype=np.float64))
        right /= np.linalg.norm(right)
        return look, right, np.cross(right, look)

    def to_c(self, w: int, h: int) -> "_lib.CameraC":
        """wc_camera for the C ABI: basis + tan_half exactly as the reference.
        (The camera is frozen: its record is built once per image size.)"""
        return _camera_c(self, int(w), int(h))

    def _to_c(self, w: int, h: int) -> "_lib.CameraC":
        look, right, up_v = self.basis()
        c = _lib.CameraC()
        c.eye[:] = [float(v) for v in self.eye]
        c.look[:] = [float(v) for v in look]
        c.right[:] = [float(v) for v in right]
        c.up[:] = [float(v) for v in up_v]
        c.tan_half = math.tan(math.radians(self.fov_y) * 0.5)
        c.img_w = int(w)
        c.img_h = int(h)
        return c


@functools.lru_cache(maxsize=256)
def _camera_c(cam: Camera, w: int, h: int) -> "_lib.CameraC":
    return cam._to_c(w, h)


def fine_dims(dims):
    return tuple(-(int(d) // -4) for d in dims)


def coarse_dims(dims):
    return tuple(-(f // -4) for f in fine_dims(dims))


class RaySoA:
    """Host view of per-ray state (traversal.py:73-103)."""

    def __init__(self, n: int, w: int, h: int):
        self.w, self.h = w, h
        self.origin = np.zeros((n, 3))
        self.direction = np.zeros((n, 3))
        self.t_enter = np.zeros(n)
        self.t_exit = np.zeros(n)
        self.status = np.zeros(n, dtype=np.uint8)
        self.exited = np.zeros(n, dtype=np.uint8)
        self.coarse_cell = np.full(n, UINT_MAX, dtype=np.uint32)
        self.coarse_tmax = np.zeros((n, 3))
        self.fine_cell = np.full(n, UINT_MAX, dtype=np.uint32)
        self.fine_tmax = np.zeros((n, 3))
        self.block_slots = np.full(n, UINT_MAX, dtype=np.uint32)
        self.ray_slots = np.full(n, UINT_MAX, dtype=np.uint32)

    @property
    def n(self) -> int:
        return self.origin.shape[0]

    @property
    def active_mask(self) -> np.ndarray:
        return self.status == STATUS_ACTIVE

    @property
    def n_active(self) -> int:
        return int(np.count_nonzero(self.status == STATUS_ACTIVE))

    def _fill_from_device(self, cam_c, pixel_ids, origins, dirs, dims):
        n = self.n
        pid = None if pixel_ids is None else np.ascontiguousarray(pixel_ids, dtype=np.uint32)
        o = None if origins is None else np.ascontiguousarray(origins, dtype=np.float64)
        d = None if dirs is None else np.ascontiguousarray(dirs, dtype=np.float64)
        _lib.call("wc_init_rays", None if cam_c is None else C.byref(cam_c), _lib.ptr(pid), n, _lib.ptr(o),
                  _lib.ptr(d), *[int(v) for v in dims], _lib.ptr(self.direction), _lib.ptr(self.t_enter),
                  _lib.ptr(self.t_exit), _lib.ptr(self.status), _lib.ptr(self.exited), _lib.ptr(self.coarse_cell),
                  _lib.ptr(self.fine_cell), _lib.ptr(self.coarse_tmax), _lib.ptr(self.fine_tmax))

    @classmethod
    def from_camera(cls, cam: Camera, w: int, h: int, dims) -> "RaySoA":
        """Pinhole rays through pixel centres, ray = y*w + x (traversal.py:105-120)."""
        if w < 1 or h < 1:
            raise UsageError(f"image size must be at least 1x1, got {w}x{h}")
        rays = cls(w * h, w, h)
        rays._fill_from_device(cam.to_c(w, h), None, None, None, dims)
        rays.origin[:] = np.asarray(cam.eye, dtype=np.float64)
        return rays

    @classmethod
    def from_rays(cls, origins, dirs, dims, w: int | None = None, h: int | None = None) -> "RaySoA":
        """Clip arbitrary rays against the box and seed iterators (traversal.py:122-170)."""
        origins = np.ascontiguousarray(origins, dtype=np.float64)
        n = origins.shape[0]
        rays = cls(n, w if w is not None else n, h if h is not None else 1)
        rays.origin[:] = origins
        rays._fill_from_device(None, None, origins, dirs, dims)
        return rays


def init_rays(cam: Camera, w: int, h: int, dims) -> RaySoA:
    """traversal.py:190-192."""
    return RaySoA.from_camera(cam, w, h, dims)


def traverse_to_next_blocks(rays: RaySoA, grids, iso: float, n_spec: int, active_offsets: np.ndarray,
                            variant: int = 0) -> None:
    """Advance every active ray to its next up-to-n_spec candidate blocks
    (traversal.py:406-452) with the session's traversal kernels
    (k_traverse / k_traverse_warp; ``variant`` 1 or 2 forces one).

    Candidate block ids land in rays.block_slots (owning ray in
    rays.ray_slots) at offset active_offsets[ray] * n_spec; unfilled slots
    stay UINT_MAX.  Iterator state is saved past the last emitted block;
    rays that run out of volume get their exited flag set."""
    assert n_spec >= 1
    n = rays.n
    fd = np.asarray(grids.fine_dims, dtype=np.int32)
    cd = np.asarray(grids.coarse_dims, dtype=np.int32)
    vol = grids.bound_volume
    if vol is not None:
        arrs = (None, None, None, None)
        vh = vol.device_handle()
    else:
        arrs = tuple(np.ascontiguousarray(a, dtype=np.float64) for a in
                     (grids.fine_min, grids.fine_max, grids.coarse_min, grids.coarse_max))
        vh = None
    fields = {}
    for name, dt in (("origin", np.float64), ("direction", np.float64), ("t_exit", np.float64),
                     ("status", np.uint8), ("exited", np.uint8), ("coarse_cell", np.uint32),
                     ("coarse_tmax", np.float64), ("fine_cell", np.uint32), ("fine_tmax", np.float64),
                     ("block_slots", np.uint32), ("ray_slots", np.uint32)):
        a = getattr(rays, name)
        if a.dtype != dt or not a.flags["C_CONTIGUOUS"]:
            a = np.ascontiguousarray(a, dtype=dt)
            setattr(rays, name, a)
        fields[name] = a
    offs = np.ascontiguousarray(active_offsets, dtype=np.int64)
    _lib.call("wc_traverse", vh, *[_lib.ptr(a) for a in arrs], _lib.ptr(fd), _lib.ptr(cd), n,
              *[_lib.ptr(fields[k]) for k in ("origin", "direction", "t_exit", "status", "exited", "coarse_cell",
                                              "coarse_tmax", "fine_cell", "fine_tmax", "block_slots", "ray_slots")],
              _lib.ptr(offs), float(iso), int(n_spec), int(variant))


def dda_step(cell, tmax, direction, grid_dims, cell_size):
    """One Amanatides-Woo step (traversal.py:195-214); ties step x, then y, then z."""
    cell = [int(c) for c in cell]
    tmax = [float(t) for t in tmax]
    d = [float(v) for v in direction]
    axis = 0 if (tmax[0] <= tmax[1] and tmax[0] <= tmax[2]) else (1 if tmax[1] <= tmax[2] else 2)
    t_cross = tmax[axis]
    cell[axis] += 1 if d[axis] > 0 else -1
    tmax[axis] += cell_size / abs(d[axis]) if d[axis] != 0.0 else math.inf
    done = not all(0 <= cell[a] < grid_dims[a] for a in range(3))
    return tuple(cell), tuple(tmax), t_cross, done
