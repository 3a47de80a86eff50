"""Per-pass wavefront renderer -- the drop-in boundary (mirrors wavecast/engine.py).

``render_passes(cv, grids, cam, iso, opts)`` keeps the reference generator
protocol (engine.py:308-382): one ``(Framebuffer, PassStats)`` per pass.
Everything between ray setup and composite runs on the B200 inside one
``wc_session`` (csrc/wc_engine.cu); the host only reads a few counters per
pass and, when asked, the framebuffer.  Speculation never changes final
pixels (engine.py:1-9), which is what makes image-tile sharding exact.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterator

import numpy as np

from . import _lib
from .bitmaps import mask_to_words, n_words, words_to_mask
from .codec import CompressedVolume
from .errors import UsageError
from .grids import MacrocellGrids
from .traversal import Camera

BACKGROUND_RGBA = (0, 0, 0, 255)
STAGES = ("traverse", "mark", "cache_decode", "rt_inputs", "raytrace", "composite")
MAX_SPEC_DEFAULT = 64
AMBIENT = 0.2
BASE_COLOR = (0.85, 0.85, 0.85)


@dataclass
class RenderOptions:
    """engine.py:37-44 (+ cache_capacity: the LRU budget, cache.py:122-125 when None)."""

    width: int = 1280
    height: int = 720
    speculation: bool = True
    max_spec: int = MAX_SPEC_DEFAULT
    base_color: tuple[float, float, float] = BASE_COLOR
    corrupt_cache: bool = False  # test hook: zero the slot pool every pass
    cache_capacity: int | None = None
    # build_rt_inputs grouping (engine.py:121-149).  Off by default on B200:
    # the thread-per-entry raytrace is as fast on ray-ordered entries; turn
    # on to get the reference's PassBuffers layout (debug.pass_buffers).
    group_entries: bool = False


@dataclass
class Framebuffer:
    w: int
    h: int
    rgba: np.ndarray   # uint8 (h, w, 4)
    depth: np.ndarray  # float32 (h, w), +inf = background
    completeness: float

    @classmethod
    def blank(cls, w: int, h: int) -> "Framebuffer":
        rgba = np.empty((h, w, 4), dtype=np.uint8)
        rgba[...] = BACKGROUND_RGBA
        return cls(w, h, rgba, np.full((h, w), np.inf, dtype=np.float32), 0.0)

    def snapshot(self) -> "Framebuffer":
        return Framebuffer(self.w, self.h, self.rgba.copy(), self.depth.copy(), self.completeness)


class StreamedFramebuffer:
    """A per-pass framebuffer snapshot (engine.py:62-63) whose pixels are
    still in flight: the session copied its framebuffer on the device and is
    moving the copy to page-locked host memory on a copy stream while the
    next passes run (wc_session_snapshot).  ``rgba`` / ``depth`` wait for that
    copy on first access, so a consumer that looks at every frame sees the
    copy overlapped with rendering, and one that skips frames never waits."""

    def __init__(self, session: "RenderSession", ticket: int, base: np.ndarray, completeness: float):
        self.w, self.h = session.w, session.h
        self.completeness = completeness
        n = session.n
        self._rgba = base[:4 * n].reshape(self.h, self.w, 4)
        self._depth = base[4 * n:8 * n].view(np.float32).reshape(self.h, self.w)
        self._session = session
        self._ticket = ticket

    def _land(self):
        s = self._session
        if s is not None:
            self._session = None
            if s._h is not None:
                _lib.call("wc_session_snapshot_wait", s._h, self._ticket)

    @property
    def rgba(self) -> np.ndarray:
        self._land()
        return self._rgba

    @property
    def depth(self) -> np.ndarray:
        self._land()
        return self._depth

    def snapshot(self) -> Framebuffer:
        return Framebuffer(self.w, self.h, self.rgba.copy(), self.depth.copy(), self.completeness)


@dataclass(frozen=True)
class PassStats:
    pass_index: int
    n_active_before: int
    n_spec: int
    visible_blocks: int
    active_blocks: int
    new_decompressed: int
    cache_slots: int
    utilization: float
    completeness: float
    duration: float


@dataclass(frozen=True)
class PassBuffers:
    visible_ids: np.ndarray
    rays_per_block: np.ndarray
    block_ray_offsets: np.ndarray
    sorted_ray_ids: np.ndarray
    sorted_hit_slots: np.ndarray
    valid_prefix: np.ndarray
    n_entries: int


def compute_n_spec(n_act: int, w: int, h: int, max_spec: int = MAX_SPEC_DEFAULT) -> int:
    """Free slots shared evenly, clamped to [1, max_spec] (engine.py:91-94)."""
    assert n_act >= 1
    return min(max_spec, max(1, (w * h) // n_act))


UINT_MAX = 0xFFFFFFFF


def mark_blocks(block_slots: np.ndarray, block_dims) -> tuple[np.ndarray, np.ndarray]:
    """engine.py:97-118 on the device: visible = referenced by a slot; active
    adds each visible block's existing +octant neighbours.  The session's
    marking kernels (bitmap extraction + word/bit dilation, csrc/wc_stage.cu)."""
    bdx, bdy, bdz = (int(v) for v in block_dims)
    n_blocks = bdx * bdy * bdz
    slots = np.ascontiguousarray(np.asarray(block_slots).reshape(-1), dtype=np.uint32)
    vis = np.zeros(n_words(n_blocks), dtype=np.uint32)
    act = np.zeros_like(vis)
    _lib.call("wc_mark_blocks", _lib.ptr(slots), len(slots), bdx, bdy, bdz, _lib.ptr(vis), _lib.ptr(act))
    return words_to_mask(vis, n_blocks), words_to_mask(act, n_blocks)


def build_rt_inputs(block_slots: np.ndarray, ray_slots: np.ndarray, visible_mask: np.ndarray) -> PassBuffers:
    """engine.py:121-149 on the device: scan of slot validity, compaction,
    stable radix sort of the entries by block, per-block counts by visible
    rank (csrc/wc_stage.cu)."""
    bs = np.ascontiguousarray(np.asarray(block_slots).reshape(-1), dtype=np.uint32)
    rs = np.ascontiguousarray(np.asarray(ray_slots).reshape(-1), dtype=np.uint32)
    assert bs.shape == rs.shape, "slot buffers differ in length"
    vm = np.asarray(visible_mask, dtype=bool).reshape(-1)
    n, nb = len(bs), len(vm)
    words = mask_to_words(vm)
    vis = np.empty(nb + 1, dtype=np.uint32)
    counts = np.empty(nb + 1, dtype=np.uint32)
    offs = np.empty(nb + 1, dtype=np.uint32)
    sr = np.empty(n, dtype=np.uint32)
    sh = np.empty(n, dtype=np.uint32)
    vp = np.empty(n, dtype=np.uint32)
    sizes = np.zeros(3, dtype=np.int64)
    _lib.call("wc_build_rt_inputs", _lib.ptr(bs), _lib.ptr(rs), n, _lib.ptr(words), nb, _lib.ptr(vis),
              _lib.ptr(counts), _lib.ptr(offs), _lib.ptr(sr), _lib.ptr(sh), _lib.ptr(vp), _lib.ptr(sizes))
    ne, nv, nc = (int(x) for x in sizes)
    return PassBuffers(visible_ids=vis[:nv].copy(), rays_per_block=counts[:nc].copy(),
                       block_ray_offsets=offs[:nc].copy(), sorted_ray_ids=sr[:ne].copy(),
                       sorted_hit_slots=sh[:ne].copy(), valid_prefix=vp, n_entries=ne)


def composite(rgbz_rgb: np.ndarray, rgbz_z: np.ndarray, rays, n_spec: int, active_offsets: np.ndarray,
              valid_prefix: np.ndarray, fb: Framebuffer) -> None:
    """engine.py:261-283 on the device: each active ray's closest speculated
    hit (strict <, earliest slot wins); finished rays terminate."""
    rgb = np.ascontiguousarray(rgbz_rgb, dtype=np.float32).reshape(-1, 3)
    z = np.ascontiguousarray(rgbz_z, dtype=np.float32).reshape(-1)
    assert len(rgb) == len(z), "rgbz buffers differ in length"
    status = np.ascontiguousarray(rays.status, dtype=np.uint8)
    exited = np.ascontiguousarray(rays.exited, dtype=np.uint8)
    offs = np.ascontiguousarray(active_offsets, dtype=np.int64)
    bs = np.ascontiguousarray(rays.block_slots, dtype=np.uint32)
    vp = np.ascontiguousarray(valid_prefix, dtype=np.uint32)
    rgba = np.ascontiguousarray(fb.rgba.reshape(-1, 4))
    depth = np.ascontiguousarray(fb.depth.reshape(-1))
    n = len(status)
    _lib.call("wc_composite", _lib.ptr(rgb), _lib.ptr(z), len(z), n, _lib.ptr(status), _lib.ptr(exited),
              _lib.ptr(offs), int(n_spec), _lib.ptr(bs), len(bs), _lib.ptr(vp), _lib.ptr(rgba), _lib.ptr(depth))
    rays.status[:] = status
    fb.rgba.reshape(-1, 4)[:] = rgba
    fb.depth.reshape(-1)[:] = depth
    fb.completeness = float(rays.n - rays.n_active) / rays.n


def _stats_from_c(s: _lib.PassStatsC) -> PassStats:
    return PassStats(int(s.pass_index), int(s.n_active_before), int(s.n_spec), int(s.visible_blocks),
                     int(s.active_blocks), int(s.new_decompressed), int(s.cache_slots), float(s.utilization),
                     float(s.completeness), float(s.duration))


class RenderSession:
    """One render on the device: rays, cache, scratch and framebuffer in HBM.

    ``pixel_ids`` (optional) restricts the session to a subset of the
    image's pixels -- the unit of image-tile sharding.  Arbitrary rays
    (RaySoA.from_rays semantics) go through ``origins``/``dirs``.
    """

    def __init__(self, cv: CompressedVolume, grids: MacrocellGrids | None, cam: Camera | None, iso: float,
                 opts: RenderOptions, pixel_ids=None, origins=None, dirs=None):
        if grids is not None:
            grids.bind(cv)
        self.cv = cv
        self.opts = opts
        self.w, self.h = int(opts.width), int(opts.height)
        self._pix = None if pixel_ids is None else np.ascontiguousarray(pixel_ids, dtype=np.uint32)
        o = None if origins is None else np.ascontiguousarray(origins, dtype=np.float64)
        d = None if dirs is None else np.ascontiguousarray(dirs, dtype=np.float64)
        if d is not None:
            n = d.shape[0]
        elif self._pix is not None:
            n = len(self._pix)
        else:
            n = self.w * self.h
        self.n = n
        cam_c = cam.to_c(self.w, self.h) if cam is not None else None
        cap = 0 if opts.cache_capacity is None else int(opts.cache_capacity)
        self._h = C.c_void_p()
        _lib.call("wc_session_create", cv.device_handle(), None if cam_c is None else C.byref(cam_c),
                  _lib.ptr(self._pix), n, _lib.ptr(o), _lib.ptr(d), float(iso), int(bool(opts.speculation)),
                  int(opts.max_spec), cap, int(bool(opts.corrupt_cache)), C.byref(self._h))
        if tuple(opts.base_color) != BASE_COLOR:
            _lib.call("wc_session_set_base_color", self._h, *[float(c) for c in opts.base_color])
        _lib.call("wc_session_set_grouping", self._h, int(bool(opts.group_entries)))
        self.last_c_stats = None

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().wc_session_sync(self._h)  # streamed snapshots have landed
            for ref in getattr(self, "_streamed", ()):
                fb = ref()
                if fb is not None:
                    fb._session = None
            _lib.lib().wc_session_destroy(self._h)
            self._h = None

    def snapshot(self, completeness: float) -> StreamedFramebuffer:
        """This pass's framebuffer, copied to host memory in the background
        (see StreamedFramebuffer); whole-image sessions only."""
        import weakref

        if self._pix is not None or self.n != self.w * self.h:
            raise UsageError("streamed snapshots need a whole-image camera session")
        base = _lib.pinned_pool.get(8 * self.n)
        t = C.c_int64()
        rgba = base[:4 * self.n]
        depth = base[4 * self.n:8 * self.n]
        _lib.call("wc_session_snapshot", self._h, _lib.ptr(rgba), _lib.ptr(depth), C.byref(t))
        fb = StreamedFramebuffer(self, int(t.value), base, completeness)
        # A pinned buffer must not be handed out again while a copy into it
        # is in flight, even if the consumer dropped its frame: the copy of
        # snapshot k has landed once the session stream has passed snapshot
        # k + 3's ring-slot wait (three ring slots, one sync per step).
        if not hasattr(self, "_streamed"):
            import collections

            self._streamed = []
            self._inflight = collections.deque(maxlen=4)
        self._inflight.append(base)
        self._streamed = [r for r in self._streamed if r() is not None and r()._session is not None]
        self._streamed.append(weakref.ref(fb))
        return fb

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def n_active(self) -> int:
        v = C.c_int64()
        _lib.call("wc_session_n_active", self._h, C.byref(v))
        return int(v.value)

    def step(self) -> PassStats | None:
        st = _lib.PassStatsC()
        ran = C.c_int()
        _lib.call("wc_session_pass", self._h, C.byref(st), C.byref(ran))
        if not ran.value:
            return None
        self.last_c_stats = st
        return _stats_from_c(st)

    _MAX_STATS = 4096

    def _stats_buf(self):
        """The session's PassStatsC records buffer (allocated once: a fresh
        4096-record array per frame costs ~0.1 ms of host time)."""
        buf = getattr(self, "_sbuf", None)
        if buf is None:
            buf = (_lib.PassStatsC * self._MAX_STATS)()
            self._sbuf = buf
        return buf

    def run(self) -> list[PassStats]:
        """All remaining passes (render, engine.py:385-401)."""
        buf = self._stats_buf()
        k = C.c_int64()
        _lib.call("wc_session_run", self._h, buf, self._MAX_STATS, C.byref(k))
        return self._frame_stats(buf, k.value)

    def _frame_stats(self, buf, k: int) -> list[PassStats]:
        """PassStats of a frame; the C records (with evicted / n_entries) stay in last_frame_c."""
        k = min(int(k), self._MAX_STATS)
        recs = (_lib.PassStatsC * k)()  # a copy: the records buffer is reused by the next frame
        C.memmove(recs, buf, C.sizeof(_lib.PassStatsC) * k)
        self._last_recs = recs
        return [_stats_from_c(r) for r in recs]

    @property
    def last_frame_c(self) -> list[dict]:
        """The last frame's C records as dicts (PassStats fields + evicted / n_entries)."""
        recs = getattr(self, "_last_recs", None) or []
        return [{f: getattr(r, f) for f, _ in _lib.PassStatsC._fields_} for r in recs]

    def render_frame(self, cam: Camera | None, iso: float) -> list[PassStats]:
        """reset(cam, iso) + run() in a single C call (no Python inside the frame)."""
        cam_c = cam.to_c(self.w, self.h) if cam is not None else None
        buf = self._stats_buf()
        k = C.c_int64()
        _lib.call("wc_session_render", self._h, None if cam_c is None else C.byref(cam_c), float(iso), buf,
                  self._MAX_STATS, C.byref(k))
        return self._frame_stats(buf, k.value)

    def reset_part(self, cam: Camera | None, iso: float, part: int, parts: int) -> None:
        """reset with the per-iso range tests computed for coarse-cell slice
        `part` of `parts` only (dist.render_frame_split gathers the rest)."""
        cam_c = cam.to_c(self.w, self.h) if cam is not None else None
        _lib.call("wc_session_reset_part", self._h, None if cam_c is None else C.byref(cam_c), float(iso), int(part),
                  int(parts))

    def mask_buffers(self, parts: int):
        """(coarse bitmap ptr, fine mask ptr, words per part) of the range-test buffers."""
        cb, cm, ch = C.c_void_p(), C.c_void_p(), C.c_int64()
        _lib.call("wc_session_mask_buffers", self._h, int(parts), C.byref(cb), C.byref(cm), C.byref(ch))
        return cb.value, cm.value, ch.value

    def sync(self) -> None:
        _lib.call("wc_session_sync", self._h)

    def set_graphs(self, on: bool) -> None:
        """Replay passes as captured CUDA graphs (default) or launch them one
        kernel at a time with per-stage timing (stage_ms)."""
        _lib.call("wc_session_set_graphs", self._h, int(bool(on)))

    def render_frame_host(self, cam: Camera | None, iso: float):
        """render_frame + the framebuffer in (pinned) host memory, most of the
        copy overlapped with the frame's last passes.  -> (stats, rgba, depth)."""
        cam_c = cam.to_c(self.w, self.h) if cam is not None else None
        buf = self._stats_buf()
        k = C.c_int64()
        base = _lib.pinned_pool.get(8 * self.n)
        rgba = base[:4 * self.n].reshape(self.n, 4)
        depth = base[4 * self.n:8 * self.n].view(np.float32)
        _lib.call("wc_session_render_host", self._h, None if cam_c is None else C.byref(cam_c), float(iso), buf,
                  self._MAX_STATS, C.byref(k), _lib.ptr(rgba), _lib.ptr(depth))
        return self._frame_stats(buf, k.value), rgba, depth

    def reset(self, cam: Camera | None, iso: float) -> None:
        """New frame on the same allocations (fresh rays, framebuffer, cache)."""
        cam_c = cam.to_c(self.w, self.h) if cam is not None else None
        _lib.call("wc_session_reset", self._h, None if cam_c is None else C.byref(cam_c), float(iso))

    def frame_ms(self) -> float:
        """Device ms from the last create/reset to the end of the last pass."""
        v = C.c_double()
        _lib.call("wc_session_frame_ms", self._h, C.byref(v))
        return float(v.value)

    def stage_ms(self) -> dict:
        """Accumulated device ms per stage since the last reset."""
        a = (C.c_double * 7)()
        _lib.call("wc_session_stage_ms", self._h, a)
        return dict(zip(STAGES + ("reset",), [float(x) for x in a]))

    def pass_stage_ms(self, pass_index: int) -> dict:
        """Device ms per stage of one pass of the current frame."""
        a = (C.c_double * 6)()
        _lib.call("wc_session_pass_stage_ms", self._h, int(pass_index), a)
        return dict(zip(STAGES, [float(x) for x in a]))

    def set_frame_target(self, target) -> None:
        """Also write every final pixel into ``target`` (dist.FrameTarget: a
        full-frame buffer on this or a peer GPU) as its ray terminates; None
        stops.  Pixel positions come from the session's pixel ids."""
        self._target = target  # (keeps it alive while the session writes into it)
        _lib.call("wc_session_set_frame_target", self._h, None if target is None else target.handle)

    def set_kernel_profile(self, on: bool) -> None:
        """Collect per-kernel device times of passes launched kernel by
        kernel (set_graphs(False)); clears the previous collection."""
        _lib.call("wc_session_set_kernel_profile", self._h, int(bool(on)))

    def kernel_profile(self) -> list[dict]:
        """[{pass, kernel, launches, ms}] accumulated since set_kernel_profile(True)."""
        n = C.c_int64()
        _lib.call("wc_session_kernel_profile", self._h, None, 0, C.byref(n))
        buf = C.create_string_buffer(int(n.value) + 1)
        _lib.call("wc_session_kernel_profile", self._h, buf, int(n.value) + 1, C.byref(n))
        rows = []
        for line in buf.value.decode().splitlines():
            p, k, c, ms = line.split("\t")
            rows.append({"pass": int(p), "kernel": k, "launches": int(c), "ms": float(ms)})
        return rows

    def last_pass_ms(self) -> float:
        v = C.c_double()
        _lib.call("wc_session_last_pass_ms", self._h, C.byref(v))
        return float(v.value)

    def read(self, rgba=None, depth=None):
        """Framebuffer of this session's rays: (rgba (n,4) u8, depth (n,) f32)."""
        if rgba is None and depth is None:  # one recycled pinned buffer for both (full-speed D2H)
            base = _lib.pinned_pool.get(8 * self.n)
            rgba = base[:4 * self.n].reshape(self.n, 4)
            depth = base[4 * self.n:8 * self.n].view(np.float32)
        if rgba is None:
            rgba = np.empty((self.n, 4), dtype=np.uint8)
        if depth is None:
            depth = np.empty(self.n, dtype=np.float32)
        _lib.call("wc_session_framebuffer", self._h, _lib.ptr(rgba), _lib.ptr(depth))
        return rgba, depth

    def framebuffer(self, completeness: float) -> Framebuffer:
        rgba, depth = self.read()
        return Framebuffer(self.w, self.h, rgba.reshape(self.h, self.w, 4), depth.reshape(self.h, self.w),
                           completeness)


def render_passes(cv: CompressedVolume, grids: MacrocellGrids, cam: Camera, iso: float,
                  opts: RenderOptions) -> Iterator[tuple[Framebuffer, PassStats]]:
    """engine.py:308-382: yield a framebuffer snapshot + stats per pass.

    Each snapshot is streamed (StreamedFramebuffer): copied on the device
    after its pass and moved to host memory on a copy stream while the next
    passes run; its pixels are waited for only when the consumer reads them
    (the reference copies the whole framebuffer every pass, engine.py:62-63)."""
    with RenderSession(cv, grids, cam, iso, opts) as s:
        while True:
            ps = s.step()
            if ps is None:
                break
            yield s.snapshot(ps.completeness), ps


class _SessionPool:
    """Keeps the last render session per (volume, image, options) so that
    repeated ``render`` calls -- a viewer orbiting its camera -- reuse the
    device allocations (wc_session_reset) instead of re-allocating HBM."""

    def __init__(self, size: int = 2):
        self.size = size
        self.items: list[tuple[tuple, RenderSession]] = []

    def get(self, cv, grids, opts, cam):
        """A pooled session for (cv, opts), created (with `cam`) if needed."""
        key = (id(cv), int(opts.width), int(opts.height), bool(opts.speculation), int(opts.max_spec),
               bool(opts.group_entries),
               tuple(opts.base_color), bool(opts.corrupt_cache), opts.cache_capacity)
        for i, (k, s) in enumerate(self.items):
            if k == key and s.cv is cv:
                if grids is not None:
                    grids.bind(cv)
                self.items.append(self.items.pop(i))
                return s
        s = RenderSession(cv, grids, cam, 0.0, opts)
        self.items.append((key, s))
        while len(self.items) > self.size:
            self.items.pop(0)[1].close()
        return s

    def clear(self):
        while self.items:
            self.items.pop()[1].close()


session_pool = _SessionPool()


def render(cv: CompressedVolume, grids: MacrocellGrids, cam: Camera, iso: float,
           opts: RenderOptions) -> tuple[Framebuffer, list[PassStats]]:
    """engine.py:385-401: render to completion; only the final frame is read back."""
    s = session_pool.get(cv, grids, opts, cam)
    stats, rgba, depth = s.render_frame_host(cam, iso)
    if not stats:  # camera missed the volume on every pixel
        fb = Framebuffer.blank(opts.width, opts.height)
        fb.completeness = 1.0
        return fb, stats
    return Framebuffer(s.w, s.h, rgba.reshape(s.h, s.w, 4), depth.reshape(s.h, s.w), stats[-1].completeness), stats
