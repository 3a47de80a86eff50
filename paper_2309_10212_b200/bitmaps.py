"""Boolean block masks <-> the 32-bit bitmaps the device kernels use
(bit b of word b // 32), for the stage-level entry points."""

from __future__ import annotations

import numpy as np


def mask_to_words(mask) -> np.ndarray:
    """bool[n] -> uint32[ceil(n / 32)] (little-endian bit order)."""
    m = np.ascontiguousarray(np.asarray(mask, dtype=bool).reshape(-1))
    b = np.packbits(m, bitorder="little")
    pad = (-len(b)) % 4
    if pad or len(b) == 0:
        b = np.concatenate([b, np.zeros(pad if len(b) else 4, dtype=np.uint8)])
    return np.ascontiguousarray(b).view(np.uint32)


def words_to_mask(words: np.ndarray, n: int) -> np.ndarray:
    """uint32 bitmap -> bool[n]."""
    return np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")[:n].astype(bool)


def n_words(n: int) -> int:
    return max(1, -(-int(n) // 32))
