"""Deterministic data-parallel primitives on the GPU (mirrors wavecast/prims.py).

The contracts are sequential (prims.py:1-7): outputs equal a plain loop,
and ``sort_by_key`` is stable.  The device implementations are the ones
the render path uses internally (csrc/wc_prims.cu): a 3-phase exclusive
scan and an LSD radix sort whose per-warp ``__match_any_sync`` ranking
keeps equal keys in input order.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def exclusive_scan(values) -> tuple[np.ndarray, int]:
    """out[i] = sum(values[:i]) as uint32, plus the total (prims.py:13-23)."""
    v = np.ascontiguousarray(np.asarray(values), dtype=np.uint32)
    out = np.empty(len(v), dtype=np.uint32)
    tot = C.c_uint64()
    _lib.call("wc_exclusive_scan", _lib.ptr(v), len(v), _lib.ptr(out), C.byref(tot))
    return out, int(tot.value)


def compact(values, mask) -> np.ndarray:
    """Keep values[i] where mask[i] != 0, order preserved (prims.py:26-31):
    the kept indices come from the device's single-pass scan + compaction."""
    values = np.asarray(values)
    mask = np.asarray(mask)
    assert values.shape[0] == mask.shape[0], "compact: length mismatch"
    m = np.ascontiguousarray(mask.astype(bool).astype(np.uint8))
    idx = np.empty(len(m), dtype=np.uint32)
    tot = C.c_uint64()
    _lib.call("wc_compact_indices", _lib.ptr(m), len(m), _lib.ptr(idx), C.byref(tot))
    return values[idx[:tot.value]]


def sort_by_key(keys, values) -> tuple[np.ndarray, np.ndarray]:
    """Stable ascending sort of (keys, values) pairs (prims.py:34-40).

    uint32-representable keys are sorted on the device by value index; the
    permutation is then applied to both arrays."""
    keys = np.asarray(keys)
    values = np.asarray(values)
    assert keys.shape[0] == values.shape[0], "sort_by_key: length mismatch"
    n = len(keys)
    if n == 0:
        return keys.copy(), values.copy()
    k = np.ascontiguousarray(keys.astype(np.uint32))
    if not np.array_equal(k.astype(keys.dtype), keys):
        raise ValueError("sort_by_key keys must be representable as uint32")
    order = np.arange(n, dtype=np.uint32)
    _lib.call("wc_sort_by_key", _lib.ptr(k), _lib.ptr(order), n)
    return keys[order], values[order]
