"""Slot-addressed LRU cache of decompressed blocks (mirrors wavecast/cache.py).

``BlockCache`` is the reference's stage-level cache (cache.py:21-111) backed
by the device: each ``ensure_resident`` runs the render session's cache
update (csrc/wc_engine.cu ``CacheStore``: stamp the hits, list the misses in
ascending id order, grow to ceil(1.5 * needed), pick victims in
(last_used, block_id) order from per-stamp bitmaps, decode the misses
straight into their slots) on a ``wc_cache`` handle.  The host views
(``slot_values``, ``block_of_slot``, ``last_used_pass``) are copies read back
on access, shaped as the reference's arrays.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .bitmaps import mask_to_words
from .codec import CompressedVolume


@dataclass(frozen=True)
class CacheUpdateStats:
    """cache.py:20-24."""

    new_decompressed: int
    evicted: int
    grown_to: int


class BlockCache:
    """cache.py:27-111 on the device."""

    def __init__(self, capacity_slots: int):
        self._h = C.c_void_p()
        _lib.call("wc_cache_create", int(capacity_slots), C.byref(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib._lib is not None:
            _lib.lib().wc_cache_destroy(self._h)
            self._h = None

    __del__ = close

    def _info(self):
        cap, phys, cur, nb = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _lib.call("wc_cache_info", self._h, C.byref(cap), C.byref(phys), C.byref(cur), C.byref(nb))
        return cap.value, phys.value, cur.value, nb.value

    @property
    def capacity_slots(self) -> int:
        return self._info()[0]

    @property
    def current_pass(self) -> int:
        return self._info()[2]

    def _state(self):
        cap, phys, _, nb = self._info()
        sv = np.zeros((cap, 64), dtype=np.float32)
        bos = np.full(cap, -1, dtype=np.int32)
        lu = np.zeros(cap, dtype=np.int32)
        sob = np.full(nb, -1, dtype=np.int32)
        if phys:
            dv = np.empty((phys, 64), dtype=np.float32)
            db = np.empty(phys, dtype=np.int32)
            dl = np.empty(phys, dtype=np.int32)
            _lib.call("wc_cache_state", self._h, _lib.ptr(dv), _lib.ptr(db), _lib.ptr(dl), _lib.ptr(sob))
            occ = db >= 0  # a free slot holds no block; the reference keeps it zeroed (cache.py:31)
            sv[:phys][occ] = dv[occ]
            bos[:phys] = db
            lu[:phys] = dl
        return sv, bos.astype(np.int64), lu.astype(np.int64), sob.astype(np.int64)

    @property
    def slot_values(self) -> np.ndarray:
        return self._state()[0]

    @property
    def block_of_slot(self) -> np.ndarray:
        return self._state()[1]

    @property
    def last_used_pass(self) -> np.ndarray:
        return self._state()[2]

    @property
    def _slot_of_block(self):
        if self._info()[3] == 0:
            return None
        return self._state()[3]

    def lookup(self, block_id: int):
        """Slot index of a resident block, or None. Never touches recency (cache.py:55-60)."""
        if self._info()[3] == 0:
            return None
        s = C.c_int64()
        _lib.call("wc_cache_lookup", self._h, int(block_id), C.byref(s))
        return int(s.value) if s.value >= 0 else None

    @property
    def resident_blocks(self) -> np.ndarray:
        bos = self.block_of_slot
        return np.sort(bos[bos >= 0])

    def ensure_resident(self, active_mask: np.ndarray, cv: CompressedVolume) -> CacheUpdateStats:
        """Make every block flagged in active_mask resident (cache.py:66-111)."""
        mask = np.asarray(active_mask, dtype=bool).reshape(-1)
        words = mask_to_words(mask)
        nd, ev, gt = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.call("wc_cache_ensure_resident", self._h, cv.device_handle(), _lib.ptr(words), len(mask),
                  int(np.count_nonzero(mask)), C.byref(nd), C.byref(ev), C.byref(gt))
        return CacheUpdateStats(new_decompressed=int(nd.value), evicted=int(ev.value), grown_to=int(gt.value))


def ensure_resident(cache: BlockCache, active_mask: np.ndarray, cv: CompressedVolume) -> CacheUpdateStats:
    return cache.ensure_resident(active_mask, cv)


def lookup(cache: BlockCache, block_id: int):
    return cache.lookup(block_id)


def initial_capacity(w: int, h: int) -> int:
    """Default cache sizing (cache.py:122-125): twice the expected visible
    blocks (w*h/64), floored at 1024 slots."""
    return max(1024, 2 * (w * h) // 64)
