"""ctypes binding of libwavecast_b200.so (include/wavecast_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is usable, every call raises.  ``build()`` compiles it in-tree
with nvcc for sm_100a.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

from .errors import DataError, UsageError

_PKG = os.path.dirname(os.path.abspath(__file__))
# WAVECAST_LIB selects an alternative in-tree build (tuning variants).
LIB_PATH = os.environ.get("WAVECAST_LIB") or os.path.join(_PKG, "libwavecast_b200.so")
_CSRC = os.path.join(_PKG, "csrc")

WC_OK, WC_E_USAGE, WC_E_DATA, WC_E_INVARIANT, WC_E_CUDA = 0, 2, 3, 4, 5

_i64 = C.c_int64
_i32 = C.c_int
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


def build(verbose: bool = False) -> str:
    """nvcc-compile the CUDA sources into paper_2309_10212_b200/libwavecast_b200.so."""
    r = subprocess.run(["make", "-C", _CSRC, "-j8"], capture_output=True, text=True)
    if verbose or r.returncode != 0:
        print(r.stdout[-4000:], r.stderr[-4000:])
    if r.returncode != 0:
        raise RuntimeError("building libwavecast_b200.so failed")
    return LIB_PATH


_SIGS = {
    "wc_last_error": (C.c_char_p, []),
    "wc_init": (_i32, [_i32]),
    "wc_launch_count": (C.c_longlong, []),
    "wc_host_alloc": (_i32, [C.c_uint64, _vp]),
    "wc_host_free": (_i32, [_vp]),
    "wc_build_info": (C.c_char_p, []),
    "wc_volume_create": (_i32, [_vp, C.c_uint64, _vp, _i32, _i32, _i32, _i32, _i32, _vp]),
    "wc_volume_compress": (_i32, [_vp, _i32, _i32, _i32, _i32, _vp]),
    "wc_volume_synthesize": (_i32, [_i32, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]),
    "wc_volume_destroy": (_i32, [_vp]),
    "wc_volume_info": (_i32, [_vp, _vp, _vp, _vp]),
    "wc_volume_download": (_i32, [_vp] * 7),
    "wc_volume_set_grids": (_i32, [_vp] * 5),
    "wc_volume_value_range": (_i32, [_vp, _vp, _vp]),
    "wc_wcz_probe": (_i32, [C.c_char_p, _vp, _vp, _vp, _vp, _vp, _vp]),
    "wc_volume_load_wcz": (_i32, [C.c_char_p, _i64, _vp]),
    "wc_volume_alloc": (_i32, [_i32, _i32, _i32, _i32, _vp]),
    "wc_volume_device_buffers": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "wc_volume_finalize": (_i32, [_vp]),
    "wc_decode_blocks": (_i32, [_vp, _vp, _i64, _vp]),
    "wc_decode_bench": (_i32, [_vp, _vp, _i64, _i32, _vp]),
    "wc_session_create": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp, _dbl, _i32, _i32, _i64, _i32, _vp]),
    "wc_session_set_base_color": (_i32, [_vp, _dbl, _dbl, _dbl]),
    "wc_session_set_grouping": (_i32, [_vp, _i32]),
    "wc_session_reset_part": (_i32, [_vp, _vp, _dbl, _i64, _i64]),
    "wc_session_mask_buffers": (_i32, [_vp, _i64, _vp, _vp, _vp]),
    "wc_session_sync": (_i32, [_vp]),
    "wc_session_set_graphs": (_i32, [_vp, _i32]),
    "wc_session_pass": (_i32, [_vp, _vp, _vp]),
    "wc_session_run": (_i32, [_vp, _vp, _i64, _vp]),
    "wc_session_render_host": (_i32, [_vp, _vp, _dbl, _vp, _i64, _vp, _vp, _vp]),
    "wc_session_n_active": (_i32, [_vp, _vp]),
    "wc_session_render": (_i32, [_vp, _vp, _dbl, _vp, _i64, _vp]),
    "wc_session_framebuffer": (_i32, [_vp, _vp, _vp]),
    "wc_session_framebuffer_device": (_i32, [_vp, _vp, _vp]),
    "wc_session_snapshot": (_i32, [_vp, _vp, _vp, _vp]),
    "wc_session_set_kernel_profile": (_i32, [_vp, _i32]),
    "wc_session_stream": (_i32, [_vp, _vp]),
    "wc_session_framebuffer_packed": (_i32, [_vp, _vp, _i64]),
    "wc_scatter_pixels": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "wc_frame_target_create": (_i32, [_i64, _vp]),
    "wc_frame_target_ipc_handles": (_i32, [_vp, _vp]),
    "wc_frame_target_open": (_i32, [_vp, _i64, _vp]),
    "wc_frame_target_download": (_i32, [_vp, _vp, _vp]),
    "wc_frame_target_destroy": (_i32, [_vp]),
    "wc_session_set_frame_target": (_i32, [_vp, _vp]),
    "wc_session_kernel_profile": (_i32, [_vp, _vp, _i64, _vp]),
    "wc_session_snapshot_wait": (_i32, [_vp, _i64]),
    "wc_session_last_pass_ms": (_i32, [_vp, _vp]),
    "wc_session_destroy": (_i32, [_vp]),
    "wc_session_sizes": (_i32, [_vp, _vp]),
    "wc_session_reset": (_i32, [_vp, _vp, _dbl]),
    "wc_session_frame_ms": (_i32, [_vp, _vp]),
    "wc_session_stage_ms": (_i32, [_vp, _vp]),
    "wc_session_pass_stage_ms": (_i32, [_vp, _i64, _vp]),
    "wc_session_rays": (_i32, [_vp] * 10),
    "wc_session_slots": (_i32, [_vp] * 4),
    "wc_session_blocks": (_i32, [_vp] * 3),
    "wc_session_rt_inputs": (_i32, [_vp] * 4),
    "wc_session_rgbz": (_i32, [_vp, _vp]),
    "wc_session_cache": (_i32, [_vp] * 4),
    "wc_init_rays": (_i32, [_vp, _vp, _i64, _vp, _vp, _i32, _i32, _i32] + [_vp] * 9),
    "wc_reference_render": (_i32, [_vp, _vp, _vp, _i64, _dbl, _dbl, _dbl, _dbl, _vp, _vp]),
    "wc_reference_render_dense": (_i32, [_vp, _i32, _i32, _i32, _vp, _vp, _i64, _dbl, _dbl, _dbl, _dbl, _vp, _vp]),
    "wc_traverse": (_i32, [_vp] * 7 + [_i64] + [_vp] * 12 + [_dbl, _i32, _i32]),
    "wc_mark_blocks": (_i32, [_vp, _i64, _i32, _i32, _i32, _vp, _vp]),
    "wc_build_rt_inputs": (_i32, [_vp, _vp, _i64, _vp, _i64] + [_vp] * 7),
    "wc_composite": (_i32, [_vp, _vp, _i64, _i64, _vp, _vp, _vp, _i32, _vp, _i64, _vp, _vp, _vp]),
    "wc_cache_create": (_i32, [_i64, _vp]),
    "wc_cache_destroy": (_i32, [_vp]),
    "wc_cache_ensure_resident": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "wc_cache_info": (_i32, [_vp] * 5),
    "wc_cache_lookup": (_i32, [_vp, _i64, _vp]),
    "wc_cache_state": (_i32, [_vp] * 5),
    "wc_cache_dual_grid": (_i32, [_vp, _i64, _vp]),
    "wc_intersect_cells": (_i32, [_i64] + [_vp] * 6 + [_dbl, _vp]),
    "wc_cell_overlaps": (_i32, [_i64] + [_vp] * 5),
    "wc_check_fastdiv": (_i32, [_i64, C.c_uint64, _vp, _vp]),
    "wc_shade": (_i32, [_i64] + [_vp] * 4),
    "wc_raytrace_block": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _dbl, _vp, _vp, _vp, _vp]),
    "wc_exclusive_scan": (_i32, [_vp, _i64, _vp, _vp]),
    "wc_sort_by_key": (_i32, [_vp, _vp, _i64]),
    "wc_compact_indices": (_i32, [_vp, _i64, _vp, _vp]),
}

_lib = None
_lock = threading.Lock()
_initialised = False


def lib():
    """Load the CUDA library (fails loudly: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the render path)"
            )
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ensure_device(device: int | None = None) -> None:
    """Bind the calling thread to the CUDA device (LOCAL_RANK or 0)."""
    global _initialised
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    check(lib().wc_init(device))
    _initialised = True


def check(status: int) -> None:
    if status == WC_OK:
        return
    msg = lib().wc_last_error().decode(errors="replace")
    if status == WC_E_USAGE:
        raise UsageError(msg)
    if status == WC_E_DATA:
        raise DataError(msg)
    if status == WC_E_INVARIANT:
        raise AssertionError(msg)
    raise RuntimeError(f"CUDA failure in libwavecast_b200: {msg}")


def call(name: str, *args) -> None:
    if not _initialised:
        ensure_device()
    check(getattr(lib(), name)(*args))


def call_host(name: str, *args) -> None:
    """A library call that touches no device (header parsing and the like)."""
    check(getattr(lib(), name)(*args))


def ptr(a):
    """Data pointer of a contiguous numpy array (None passes through)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C ABI must be contiguous"
    return a.ctypes.data_as(_vp)


def out(shape, dtype):
    return np.empty(shape, dtype=dtype)


class PinnedPool:
    """Recycled page-locked host buffers for framebuffer read-back.

    ``get(nbytes)`` returns a uint8 numpy array over pinned memory.  A buffer
    is handed out again only once every array viewing it has been garbage
    collected (tracked with a weakref on the base array), so callers can
    keep returned frames as long as they like; past ``limit`` live buffers
    the pool falls back to ordinary (pageable) arrays."""

    def __init__(self, limit: int = 8):
        import weakref

        self._weakref = weakref
        self.limit = limit
        self.slots: list[list] = []  # [ptr, nbytes, weakref to base or None]

    def get(self, nbytes: int) -> np.ndarray:
        for slot in self.slots:
            ptr, cap, ref = slot
            if cap >= nbytes and (ref is None or ref() is None):
                return self._hand_out(slot, nbytes)
        if len(self.slots) >= self.limit:
            return np.empty(nbytes, dtype=np.uint8)
        p = C.c_void_p()
        call("wc_host_alloc", C.c_uint64(nbytes), C.byref(p))
        slot = [p.value, nbytes, None]
        self.slots.append(slot)
        return self._hand_out(slot, nbytes)

    def _hand_out(self, slot, nbytes):
        base = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(slot[0]))
        slot[2] = self._weakref.ref(base)
        return base


pinned_pool = PinnedPool()
