"""ctypes front-end of the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  The product package
``paper_2309_10212_b200`` never does: the oracle is the checker, not the
thing measured or shipped.

The C restatement lives in wc_oracle.c; this file restates the host-side
numpy pieces of the reference that feed it (camera basis, traversal.py:65-70
and :111; orbit camera, cli.py:48-58) so the oracle shares no code with the
product.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
UINT_MAX = 0xFFFFFFFF

_i64 = C.c_int64
_dbl = C.c_double
_vp = C.c_void_p


class PassStatsC(C.Structure):
    _fields_ = [
        ("pass_index", _i64),
        ("n_active_before", _i64),
        ("n_spec", _i64),
        ("visible_blocks", _i64),
        ("active_blocks", _i64),
        ("new_decompressed", _i64),
        ("evicted", _i64),
        ("cache_slots", _i64),
        ("n_entries", _i64),
        ("n_active_after", _i64),
        ("utilization", _dbl),
        ("completeness", _dbl),
        ("duration", _dbl),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class CameraC(C.Structure):
    _fields_ = [
        ("eye", _dbl * 3),
        ("look", _dbl * 3),
        ("right", _dbl * 3),
        ("up", _dbl * 3),
        ("tan_half", _dbl),
        ("img_w", C.c_int32),
        ("img_h", C.c_int32),
    ]


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
        os.path.join(_HERE, "wc_oracle.c")
    ):
        build()
    L = C.CDLL(_LIB_PATH)
    L.orc_session_create.restype = _vp
    L.orc_session_create.argtypes = [_vp] * 6 + [C.c_int] * 5 + [_vp, _vp, _i64, _i64, _i64, _dbl, C.c_int, C.c_int, _i64, C.c_int]
    L.orc_session_destroy.argtypes = [_vp]
    L.orc_session_pass.argtypes = [_vp, _vp]
    L.orc_session_pass.restype = C.c_int
    L.orc_session_set_base_color.argtypes = [_vp, _dbl, _dbl, _dbl]
    L.orc_get_rays.argtypes = [_vp] * 9
    L.orc_get_framebuffer.argtypes = [_vp] * 3
    L.orc_get_pass_sizes.argtypes = [_vp] * 2
    L.orc_get_slots.argtypes = [_vp] * 4
    L.orc_get_visible_active.argtypes = [_vp] * 3
    L.orc_get_rt_inputs.argtypes = [_vp] * 6
    L.orc_get_rgbz.argtypes = [_vp] * 3
    L.orc_cache_capacity.argtypes = [_vp]
    L.orc_cache_capacity.restype = _i64
    L.orc_get_cache.argtypes = [_vp] * 4
    L.orc_decode_blocks.argtypes = [_vp, C.c_int, C.c_int, _vp, _i64, _vp]
    L.orc_compress.argtypes = [_vp, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp]
    L.orc_compress_separable.argtypes = [C.c_int, _vp, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, _vp, _vp]
    L.orc_error_bounds.argtypes = [_vp, _i64, C.c_int, C.c_int, _vp]
    L.orc_build_grids.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp]
    L.orc_camera_rays.argtypes = [_vp, _vp, _i64, _vp, _vp]
    L.orc_cache_create.restype = _vp
    L.orc_cache_create.argtypes = [_i64, _i64]
    L.orc_cache_destroy.argtypes = [_vp]
    L.orc_cache_update.argtypes = [_vp, _vp, C.c_int, C.c_int, _vp, _i64, _vp]
    L.orc_cache_lookup.argtypes = [_vp, _i64]
    L.orc_cache_lookup.restype = _i64
    L.orc_cache_capacity_of.argtypes = [_vp]
    L.orc_cache_capacity_of.restype = _i64
    L.orc_cache_state.argtypes = [_vp] * 4
    L.orc_reference_render.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _i64, _dbl, _dbl, _dbl, _dbl, _vp, _vp]
    L.orc_intersect_cell.argtypes = [_vp, _vp, _vp, _vp, _dbl, _dbl, _dbl]
    L.orc_intersect_cell.restype = _dbl
    _lib = L
    return L


def _p(a: np.ndarray):
    return a.ctypes.data_as(_vp) if a is not None else None


# ------------------------------------------------------------------ camera
def camera_basis(eye, look_dir, up, fov_y):
    """traversal.py:65-70 basis() + traversal.py:111 tan_half (host numpy)."""
    look = np.asarray(look_dir, dtype=np.float64)
    right = np.cross(look, np.asarray(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    up_v = np.cross(right, look)
    tan_half = math.tan(math.radians(fov_y) * 0.5)
    return np.asarray(eye, dtype=np.float64), look, right, up_v, tan_half


def look_at(eye, target, up=(0.0, 1.0, 0.0), fov_y=45.0):
    """traversal.py:55-63 Camera.look_at -> (eye, look_dir, up, fov)."""
    eye = np.asarray(eye, dtype=np.float64)
    ld = np.asarray(target, dtype=np.float64) - eye
    ld = ld / np.linalg.norm(ld)
    return tuple(eye), tuple(ld), tuple(np.asarray(up, dtype=np.float64)), float(fov_y)


def orbit_camera(dims, step: int, steps: int, fov_y: float = 45.0):
    """cli.py:48-58 orbit_camera."""
    center = tuple((d - 1) / 2.0 for d in dims)
    dist = 1.8 * max(dims)
    angle = 2.0 * np.pi * step / steps
    eye = (center[0] + dist * np.sin(angle), center[1], center[2] + dist * np.cos(angle))
    return look_at(eye, center, fov_y=fov_y)


def camera_rays(cam, w: int, h: int, pixel_ids=None):
    """RaySoA.from_camera rays (traversal.py:105-120) for all or some pixels."""
    eye, look, right, up_v, tan_half = camera_basis(*cam)
    cc = CameraC()
    cc.eye[:] = list(eye)
    cc.look[:] = list(look)
    cc.right[:] = list(right)
    cc.up[:] = list(up_v)
    cc.tan_half = tan_half
    cc.img_w = w
    cc.img_h = h
    if pixel_ids is None:
        n = w * h
        pid = None
    else:
        pid = np.ascontiguousarray(pixel_ids, dtype=np.int64)
        n = len(pid)
    o = np.empty((n, 3), dtype=np.float64)
    d = np.empty((n, 3), dtype=np.float64)
    lib().orc_camera_rays(C.byref(cc), _p(pid), n, _p(o), _p(d))
    return o, d


# ------------------------------------------------------------------ volume
@dataclass
class OracleVolume:
    dims: tuple
    qbits: int
    stride: int
    payload: np.ndarray
    ranges: np.ndarray
    bounds: np.ndarray
    fine_min: np.ndarray
    fine_max: np.ndarray
    coarse_min: np.ndarray
    coarse_max: np.ndarray

    @property
    def block_dims(self):
        return tuple(-(d // -4) for d in self.dims)

    @property
    def block_count(self):
        bx, by, bz = self.block_dims
        return bx * by * bz


def stride_of(qbits: int) -> int:
    return -((16 + 64 * qbits) // -32) * 4


def compress(values_xfast: np.ndarray, dims, qbits: int):
    nx, ny, nz = dims
    bd = [-(d // -4) for d in dims]
    nb = bd[0] * bd[1] * bd[2]
    stride = stride_of(qbits)
    payload = np.zeros(nb * stride, dtype=np.uint8)
    ranges = np.empty((nb, 2), dtype=np.float32)
    expo = np.empty(nb, dtype=np.int32)
    v = np.ascontiguousarray(values_xfast, dtype=np.float32).reshape(-1)
    lib().orc_compress(_p(v), nx, ny, nz, qbits, _p(payload), _p(ranges), _p(expo))
    return payload, ranges, expo


def compress_separable(amp, fx, fy, fz, dims, qbits: int, threads: int = 1):
    """Synthesise + compress a separable field on host threads (ctypes drops
    the GIL, so block layers run in parallel).  Bit-identical to compress()
    of the evaluated field."""
    from concurrent.futures import ThreadPoolExecutor

    nx, ny, nz = dims
    bd = [-(d // -4) for d in dims]
    nb = bd[0] * bd[1] * bd[2]
    stride = stride_of(qbits)
    payload = np.zeros(nb * stride, dtype=np.uint8)
    ranges = np.empty((nb, 2), dtype=np.float32)
    arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (amp, fx, fy, fz)]
    K = len(arrs[0])
    bz = bd[2]
    chunks = max(1, min(bz, threads * 4))
    edges = [bz * i // chunks for i in range(chunks + 1)]

    def work(i):
        lib().orc_compress_separable(K, *[_p(a) for a in arrs], nx, ny, nz, qbits, edges[i], edges[i + 1],
                                     _p(payload), _p(ranges))

    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        list(ex.map(work, range(chunks)))
    return payload, ranges


def tile_pixels(w: int, h: int, rank: int, world: int, tile: int = 32) -> np.ndarray:
    """Same interleaved tile deal as the product's dist.tile_pixels (restated
    here so the oracle shares no code with the product)."""
    tx = -(w // -tile)
    ty = -(h // -tile)
    out = []
    for t in range(rank, tx * ty, world):
        x0, y0 = (t % tx) * tile, (t // tx) * tile
        xs = np.arange(x0, min(x0 + tile, w))
        for y in range(y0, min(y0 + tile, h)):
            out.append(y * w + xs)
    return np.concatenate(out).astype(np.int64) if out else np.zeros(0, np.int64)


def render_parallel(vol, cam, w, h, iso, threads: int, tile: int = 32, **kw):
    """Tile-parallel oracle render on `threads` host threads (one oracle
    session per thread over interleaved tiles; speculation invariance makes
    the stitched frame identical to a single-thread render).  Returns
    (rgba (w*h,4), depth (w*h,), per-thread stats lists)."""
    from concurrent.futures import ThreadPoolExecutor

    rgba = np.zeros((w * h, 4), np.uint8)
    depth = np.zeros(w * h, np.float32)

    def work(t):
        pix = tile_pixels(w, h, t, threads, tile)
        if len(pix) == 0:
            return []
        o, d = camera_rays(cam, w, h, pix)
        r, z, st = render(vol, o, d, len(pix), 1, iso, **kw)  # slot budget = rays of the tile set
        rgba[pix] = r
        depth[pix] = z
        return st

    with ThreadPoolExecutor(max_workers=threads) as ex:
        stats = list(ex.map(work, range(threads)))
    return rgba, depth, stats


def volume_from_payload(dims, qbits, payload, ranges) -> OracleVolume:
    stride = stride_of(qbits)
    bd = [-(d // -4) for d in dims]
    nb = bd[0] * bd[1] * bd[2]
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    ranges = np.ascontiguousarray(ranges, dtype=np.float32).reshape(nb, 2)
    bounds = np.empty(nb, dtype=np.float64)
    lib().orc_error_bounds(_p(payload), nb, qbits, stride, _p(bounds))
    cd = [-(b // -4) for b in bd]
    nc = cd[0] * cd[1] * cd[2]
    fmin = np.empty(nb)
    fmax = np.empty(nb)
    cmin = np.empty(nc)
    cmax = np.empty(nc)
    lib().orc_build_grids(_p(ranges), _p(bounds), bd[0], bd[1], bd[2], _p(fmin), _p(fmax), _p(cmin), _p(cmax))
    return OracleVolume(tuple(dims), qbits, stride, payload, ranges, bounds, fmin, fmax, cmin, cmax)


def volume_from_values(values_xfast, dims, qbits) -> OracleVolume:
    payload, ranges, _ = compress(values_xfast, dims, qbits)
    return volume_from_payload(dims, qbits, payload, ranges)


def decode_blocks(vol: OracleVolume, ids) -> np.ndarray:
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty((len(ids), 64), dtype=np.float32)
    lib().orc_decode_blocks(_p(vol.payload), vol.qbits, vol.stride, _p(ids), len(ids), _p(out))
    return out


def decode_full(vol: OracleVolume) -> np.ndarray:
    """oracle.py:22-39 decode_full -> dense (nz, ny, nx) float32."""
    bdx, bdy, bdz = vol.block_dims
    nx, ny, nz = vol.dims
    flat = decode_blocks(vol, np.arange(vol.block_count))
    g = flat.reshape(bdz, bdy, bdx, 4, 4, 4).transpose(0, 3, 1, 4, 2, 5).reshape(bdz * 4, bdy * 4, bdx * 4)
    return np.ascontiguousarray(g[:nz, :ny, :nx])


# ----------------------------------------------------------------- session
class Session:
    """engine.render_passes restated (one pass per .step())."""

    def __init__(self, vol: OracleVolume, origin, direction, w, h, iso, speculation=True,
                 max_spec=64, cache_capacity=0, corrupt_cache=False, base_color=None):
        self.vol = vol
        self.origin = np.ascontiguousarray(origin, dtype=np.float64)
        self.direction = np.ascontiguousarray(direction, dtype=np.float64)
        self.n = self.origin.shape[0]
        nx, ny, nz = vol.dims
        self._h = lib().orc_session_create(
            _p(vol.payload), _p(vol.ranges), _p(vol.fine_min), _p(vol.fine_max),
            _p(vol.coarse_min), _p(vol.coarse_max), nx, ny, nz, vol.qbits, vol.stride,
            _p(self.origin), _p(self.direction), self.n, w, h, float(iso),
            int(bool(speculation)), int(max_spec), int(cache_capacity), int(bool(corrupt_cache)))
        if base_color is not None:
            lib().orc_session_set_base_color(self._h, *[float(c) for c in base_color])

    def close(self):
        if self._h:
            lib().orc_session_destroy(self._h)
            self._h = None

    __del__ = close

    def step(self):
        st = PassStatsC()
        ran = lib().orc_session_pass(self._h, C.byref(st))
        return st.as_dict() if ran else None

    def framebuffer(self):
        rgba = np.empty((self.n, 4), dtype=np.uint8)
        depth = np.empty(self.n, dtype=np.float32)
        lib().orc_get_framebuffer(self._h, _p(rgba), _p(depth))
        return rgba, depth

    def rays(self):
        n = self.n
        out = dict(
            t_enter=np.empty(n), t_exit=np.empty(n), status=np.empty(n, np.uint8),
            exited=np.empty(n, np.uint8), coarse_cell=np.empty(n, np.uint32),
            fine_cell=np.empty(n, np.uint32), coarse_tmax=np.empty((n, 3)), fine_tmax=np.empty((n, 3)))
        lib().orc_get_rays(self._h, *[_p(out[k]) for k in (
            "t_enter", "t_exit", "status", "exited", "coarse_cell", "fine_cell", "coarse_tmax", "fine_tmax")])
        return out

    def pass_buffers(self):
        sizes = np.empty(4, dtype=np.int64)
        lib().orc_get_pass_sizes(self._h, _p(sizes))
        used, nv, na, ne = (int(x) for x in sizes)
        n = self.n
        bs = np.empty(n, np.uint32)
        rs = np.empty(n, np.uint32)
        ao = np.empty(n, np.uint32)
        lib().orc_get_slots(self._h, _p(bs), _p(rs), _p(ao))
        vis = np.empty(nv, np.uint32)
        act = np.empty(na, np.uint32)
        lib().orc_get_visible_active(self._h, _p(vis), _p(act))
        rpb = np.empty(nv, np.uint32)
        off = np.empty(nv, np.uint32)
        sr = np.empty(ne, np.uint32)
        sh = np.empty(ne, np.uint32)
        vp = np.empty(n, np.uint32)
        lib().orc_get_rt_inputs(self._h, _p(rpb), _p(off), _p(sr), _p(sh), _p(vp))
        rgb = np.empty((n, 3), np.float32)
        z = np.empty(n, np.float32)
        lib().orc_get_rgbz(self._h, _p(rgb), _p(z))
        return dict(slots_used=used, block_slots=bs, ray_slots=rs, active_offsets=ao,
                    visible_ids=vis, active_ids=act, rays_per_block=rpb, block_ray_offsets=off,
                    sorted_ray_ids=sr, sorted_hit_slots=sh, valid_prefix=vp, n_entries=ne,
                    rgbz_rgb=rgb, rgbz_z=z)

    def cache_state(self, with_values=False):
        cap = lib().orc_cache_capacity(self._h)
        bos = np.empty(cap, np.int64)
        lu = np.empty(cap, np.int64)
        sv = np.empty((cap, 64), np.float32) if with_values else None
        lib().orc_get_cache(self._h, _p(bos), _p(lu), _p(sv))
        return bos, lu, sv


def render(vol: OracleVolume, origin, direction, w, h, iso, **kw):
    """engine.render restated: returns (rgba (n,4), depth (n,), stats list)."""
    s = Session(vol, origin, direction, w, h, iso, **kw)
    stats = []
    while True:
        st = s.step()
        if st is None:
            break
        stats.append(st)
    rgba, depth = s.framebuffer()
    s.close()
    return rgba, depth, stats


def reference_render(dense_zyx: np.ndarray, origin, direction, iso, base_color=(0.85, 0.85, 0.85)):
    nz, ny, nx = dense_zyx.shape
    v = np.ascontiguousarray(dense_zyx, dtype=np.float32)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    d = np.ascontiguousarray(direction, dtype=np.float64)
    n = o.shape[0]
    rgba = np.empty((n, 4), np.uint8)
    depth = np.empty(n, np.float32)
    lib().orc_reference_render(_p(v), nx, ny, nz, _p(o), _p(d), n, float(iso), *[float(c) for c in base_color],
                               _p(rgba), _p(depth))
    return rgba, depth


class Cache:
    """cache.BlockCache restated (cache.py:27-111)."""

    def __init__(self, capacity: int, vol: OracleVolume):
        self.vol = vol
        self._h = lib().orc_cache_create(int(capacity), vol.block_count)

    def close(self):
        if self._h:
            lib().orc_cache_destroy(self._h)
            self._h = None

    __del__ = close

    def ensure_resident(self, active_ids):
        ids = np.ascontiguousarray(np.sort(np.asarray(active_ids, dtype=np.int64)))
        st = np.empty(3, np.int64)
        lib().orc_cache_update(self._h, _p(self.vol.payload), self.vol.qbits, self.vol.stride, _p(ids), len(ids), _p(st))
        return {"new_decompressed": int(st[0]), "evicted": int(st[1]), "grown_to": int(st[2])}

    def lookup(self, b: int):
        s = lib().orc_cache_lookup(self._h, int(b))
        return None if s < 0 else int(s)

    def state(self):
        cap = lib().orc_cache_capacity_of(self._h)
        bos = np.empty(cap, np.int64)
        lu = np.empty(cap, np.int64)
        sv = np.empty((cap, 64), np.float32)
        lib().orc_cache_state(self._h, _p(bos), _p(lu), _p(sv))
        return bos, lu, sv


def intersect_cell(corners, o, d, cell, t0, t1, iso):
    c = np.ascontiguousarray(corners, dtype=np.float32)
    oo = np.ascontiguousarray(o, dtype=np.float64)
    dd = np.ascontiguousarray(d, dtype=np.float64)
    cc = np.ascontiguousarray(cell, dtype=np.float64)
    t = lib().orc_intersect_cell(_p(c), _p(oo), _p(dd), _p(cc), float(t0), float(t1), float(iso))
    return None if t == math.inf else t
