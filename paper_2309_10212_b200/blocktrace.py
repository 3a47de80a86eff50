"""Per-block isosurface intersection (mirrors wavecast/blocktrace.py).

The stage-level blocktrace API of the reference (blocktrace.py:35-530) on
the device: every call runs the device functions the render path uses
(csrc/wc_trace.cuh: ``cell_overlap``, ``intersect_cubic`` with the Illinois
refinement, ``shade_grad``, ``trace_region``) through the C ABI, batched.
The dual grid of a block is gathered from a device ``BlockCache``
(csrc/wc_stage.cu ``k_dual_grid``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .cache import BlockCache
from .codec import CompressedVolume

AMBIENT = 0.2                    # blocktrace.py:26
BASE_COLOR = (0.85, 0.85, 0.85)  # blocktrace.py:27


@dataclass(frozen=True)
class DualGrid:
    """A block's local 4^3 values plus one vertex layer from +x/y/z neighbours (blocktrace.py:35-41)."""

    values: np.ndarray            # float32 (5,5,5) indexed [z,y,x]
    cells_per_axis: tuple[int, int, int]
    block_origin: tuple[int, int, int]


def dual_cells_per_axis(dims, block_coords) -> tuple[int, int, int]:
    """blocktrace.py:44-47: clip(dims - 1 - 4*coords, 0, 4) per axis."""
    return tuple(int(np.clip(int(dims[a]) - 1 - 4 * int(block_coords[a]), 0, 4)) for a in range(3))


def contributor_slots(cache: BlockCache, cv: CompressedVolume, block_id: int) -> np.ndarray:
    """Cache slots of a block and its 7 positive-octant neighbours, -1 where
    the neighbour lies outside the volume (blocktrace.py:97-110)."""
    bdx, bdy, bdz = cv.block_dims
    bx, by, bz = cv.block_coords(block_id)
    slots = np.full(8, -1, dtype=np.int64)
    for oz in (0, 1):
        for oy in (0, 1):
            for ox in (0, 1):
                nx, ny, nz = bx + ox, by + oy, bz + oz
                if nx < bdx and ny < bdy and nz < bdz:
                    slot = cache.lookup(nx + bdx * (ny + bdy * nz))
                    assert slot is not None, "required neighbor block not resident"
                    slots[ox + 2 * oy + 4 * oz] = slot
    return slots


def assemble_dual_grid(cache: BlockCache, cv: CompressedVolume, block_id: int) -> DualGrid:
    """Gather a resident block's dual grid from the device cache (blocktrace.py:113-123)."""
    coords = cv.block_coords(int(block_id))
    out = np.empty(125, dtype=np.float32)
    _lib.call("wc_cache_dual_grid", cache._h, int(block_id), _lib.ptr(out))
    return DualGrid(values=out.reshape(5, 5, 5), cells_per_axis=dual_cells_per_axis(cv.dims, coords),
                    block_origin=tuple(4 * c for c in coords))


def _vec3(v, n=None):
    a = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1, 3))
    return a if n is None else np.ascontiguousarray(np.broadcast_to(a, (n, 3)))


def cell_overlaps(origins, dirs, cells):
    """Batched _cell_overlap (blocktrace.py:126-158): (t0, t1) of each ray
    against its unit cell (t0 > t1 when they miss)."""
    o, d, c = _vec3(origins), _vec3(dirs), _vec3(cells)
    n = max(len(o), len(d), len(c))
    o, d, c = _vec3(o, n), _vec3(d, n), _vec3(c, n)
    t0, t1 = np.empty(n), np.empty(n)
    _lib.call("wc_cell_overlaps", n, _lib.ptr(o), _lib.ptr(d), _lib.ptr(c), _lib.ptr(t0), _lib.ptr(t1))
    return t0, t1


def _cell_overlap(ox, oy, oz, dx, dy, dz, cx, cy, cz):
    """blocktrace.py:126-158 (scalar signature of the reference)."""
    t0, t1 = cell_overlaps([ox, oy, oz], [dx, dy, dz], [cx, cy, cz])
    return float(t0[0]), float(t1[0])


def intersect_cells(corners, origins, dirs, cells, t0, t1, iso) -> np.ndarray:
    """Batched intersect_cell: smallest root per cell in [t0, t1], +inf if none."""
    c = np.ascontiguousarray(np.asarray(corners, dtype=np.float32).reshape(-1, 8))
    n = len(c)
    o, d, cl = _vec3(origins, n), _vec3(dirs, n), _vec3(cells, n)
    a0 = np.ascontiguousarray(np.broadcast_to(np.asarray(t0, dtype=np.float64), (n,)))
    a1 = np.ascontiguousarray(np.broadcast_to(np.asarray(t1, dtype=np.float64), (n,)))
    out = np.empty(n)
    _lib.call("wc_intersect_cells", n, _lib.ptr(c), _lib.ptr(o), _lib.ptr(d), _lib.ptr(cl), _lib.ptr(a0),
              _lib.ptr(a1), float(iso), _lib.ptr(out))
    return out


def intersect_cell(corners, origin, direction, cell, t0, t1, iso):
    """Smallest ray parameter where the trilinear field in the unit cell at
    integer corner `cell` equals iso within [t0, t1], or None (blocktrace.py:452-472)."""
    c = np.ascontiguousarray(corners, dtype=np.float32)
    assert c.shape == (8,)
    t = intersect_cells(c, origin, direction, cell, t0, t1, iso)[0]
    return None if t == np.inf else float(t)


def shade(grad, direction, base_color=BASE_COLOR):
    """Two-sided headlight Lambertian with an ambient floor (blocktrace.py:475-488)."""
    g = _vec3(grad)
    d = _vec3(direction)
    base = np.ascontiguousarray(np.asarray(base_color, dtype=np.float64).reshape(3))
    out = np.empty(3)
    _lib.call("wc_shade", 1, _lib.ptr(g), _lib.ptr(d), _lib.ptr(base), _lib.ptr(out))
    return float(out[0]), float(out[1]), float(out[2])


def raytrace_block(dg: DualGrid, ray_ids: np.ndarray, rays, iso: float, rgbz_rgb: np.ndarray, rgbz_z: np.ndarray,
                   hit_slots: np.ndarray, base_color=BASE_COLOR) -> None:
    """Intersect the given rays against one block's dual cells (blocktrace.py:491-530):
    the hit colour and depth of ray_ids[j] go to rgbz slot hit_slots[j];
    misses leave the slot untouched."""
    ids = np.asarray(ray_ids, dtype=np.int64).reshape(-1)
    n = len(ids)
    if n == 0:
        return
    o = np.ascontiguousarray(rays.origin[ids], dtype=np.float64)
    d = np.ascontiguousarray(rays.direction[ids], dtype=np.float64)
    te = np.ascontiguousarray(rays.t_enter[ids], dtype=np.float64)
    vals = np.ascontiguousarray(dg.values, dtype=np.float32).reshape(-1)
    org = np.asarray(dg.block_origin, dtype=np.int32)
    cells = np.asarray(dg.cells_per_axis, dtype=np.int32)
    base = np.ascontiguousarray(np.asarray(base_color, dtype=np.float64).reshape(3))
    rgb = np.zeros((n, 3), dtype=np.float32)
    z = np.full(n, np.inf, dtype=np.float32)
    hit = np.zeros(n, dtype=np.uint8)
    _lib.call("wc_raytrace_block", _lib.ptr(vals), _lib.ptr(org), _lib.ptr(cells), n, _lib.ptr(o), _lib.ptr(d),
              _lib.ptr(te), float(iso), _lib.ptr(base), _lib.ptr(rgb), _lib.ptr(z), _lib.ptr(hit))
    h = hit.astype(bool)
    slots = np.asarray(hit_slots, dtype=np.int64).reshape(-1)[h]
    rgbz_z[slots] = z[h]
    rgbz_rgb[slots] = rgb[h]
