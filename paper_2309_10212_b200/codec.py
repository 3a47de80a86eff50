"""Fixed-rate WCZ1 block codec, device resident (mirrors wavecast/codec.py).

Format (codec.py:1-12): per 4^3 block, a signed 16-bit exponent e (0x8000
= all-zero block) followed by 64 signed qbits-bit integers packed LSB-first,
q = rint(v * 2^-e * S), S = 2^(qbits-1) - 1, padded to 32-bit words.

A ``CompressedVolume`` lives in HBM (payload + raw ranges + float64 grids,
see csrc/wc_volume.cuh).  Host views (``payload``, ``raw_block_ranges``,
``block_error_bounds``) are materialised lazily, so an 8.05B-voxel volume
synthesised on the device never round-trips through host memory.
Compression and decoding run on the GPU (csrc/wc_volume.cu); only the
.wcz container I/O is host code.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import struct

import numpy as np

from . import _lib
from .errors import DataError, UsageError
from .volume import SeparableField, Volume

QBITS_MIN = 4
QBITS_MAX = 26
ZERO_EXPONENT_SENTINEL = 0x8000
WCZ_MAGIC = b"WCZ1"
WCZ_VERSION = 1


def block_stride_bytes(qbits: int) -> int:
    """Bytes per block record, rounded up to whole 32-bit words (codec.py:68-69)."""
    return ((16 + 64 * qbits + 31) // 32) * 4


def quant_scale(qbits: int) -> int:
    return (1 << (qbits - 1)) - 1


def check_qbits(qbits: int) -> None:
    if not (QBITS_MIN <= qbits <= QBITS_MAX):
        raise UsageError(f"qbits must be in [{QBITS_MIN}, {QBITS_MAX}], got {qbits}")


def error_bound(e: int, qbits: int) -> float:
    """2^e / (2S): worst-case reconstruction error of a block (codec.py:108-110)."""
    return math.ldexp(1.0, int(e)) / (2.0 * quant_scale(qbits))


def _block_dims(dims):
    return tuple(-(int(d) // -4) for d in dims)


def payload_exponents(payload: np.ndarray, block_count: int, stride: int) -> np.ndarray:
    rec = payload.reshape(block_count, stride)
    e16 = rec[:, 0].astype(np.uint16) | (rec[:, 1].astype(np.uint16) << 8)
    return e16.view(np.int16).astype(np.int32)


def bounds_from_exponents(exponents: np.ndarray, qbits: int) -> np.ndarray:
    zero = exponents == -(2**15)
    e = np.where(zero, 0, exponents).astype(np.float64)
    return np.where(zero, 0.0, 2.0**e / (2.0 * float(quant_scale(qbits))))


class CompressedVolume:
    """Independently decodable fixed-rate 4^3 blocks (codec.py:34-65)."""

    def __init__(self, dims, qbits: int, payload=None, raw_block_ranges=None, handle=None):
        check_qbits(qbits)
        self.dims = tuple(int(d) for d in dims)
        self.block_dims = _block_dims(self.dims)
        self.qbits = int(qbits)
        self.block_stride_bytes = block_stride_bytes(qbits)
        self._payload = None if payload is None else np.ascontiguousarray(payload, dtype=np.uint8)
        self._ranges = None if raw_block_ranges is None else np.ascontiguousarray(
            raw_block_ranges, dtype=np.float32).reshape(self.block_count, 2)
        self._bounds = None
        self._handle = handle
        if handle is None and self._payload is None:
            raise UsageError("a CompressedVolume needs a payload or a device handle")
        if self._payload is not None and len(self._payload) != self.block_count * self.block_stride_bytes:
            raise DataError("payload size does not match dims/qbits")

    # -- identity
    @property
    def block_count(self) -> int:
        bx, by, bz = self.block_dims
        return bx * by * bz

    def block_id(self, bx: int, by: int, bz: int) -> int:
        bdx, bdy, bdz = self.block_dims
        if not (0 <= bx < bdx and 0 <= by < bdy and 0 <= bz < bdz):
            raise IndexError(f"block coords {(bx, by, bz)} out of range {self.block_dims}")
        return bx + bdx * (by + bdy * bz)

    def block_coords(self, block_id: int) -> tuple[int, int, int]:
        bdx, bdy, _ = self.block_dims
        if not (0 <= block_id < self.block_count):
            raise IndexError(f"block id {block_id} out of range {self.block_count}")
        return block_id % bdx, (block_id // bdx) % bdy, block_id // (bdx * bdy)

    # -- device residency
    def device_handle(self):
        """wc_volume* in HBM (payload, ranges, float64 grids); created on first use."""
        if self._handle is None:
            import ctypes as C

            h = C.c_void_p()
            _lib.call("wc_volume_create", _lib.ptr(self._payload), self._payload.nbytes, _lib.ptr(self._ranges),
                      *self.dims, self.qbits, self.block_stride_bytes, C.byref(h))
            self._handle = h
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            _lib.lib().wc_volume_destroy(h)
            self._handle = None

    def _download(self):
        pay = np.empty(self.block_count * self.block_stride_bytes, dtype=np.uint8)
        rng = np.empty((self.block_count, 2), dtype=np.float32)
        _lib.call("wc_volume_download", self._handle, _lib.ptr(pay), _lib.ptr(rng), None, None, None, None)
        self._payload, self._ranges = pay, rng

    # -- host views (lazy for device-born volumes)
    @property
    def payload(self) -> np.ndarray:
        if self._payload is None:
            self._download()
        return self._payload

    @property
    def raw_block_ranges(self) -> np.ndarray:
        if self._ranges is None:
            self._download()
        return self._ranges

    @property
    def block_error_bounds(self) -> np.ndarray:
        if self._bounds is None:
            e = payload_exponents(self.payload, self.block_count, self.block_stride_bytes)
            self._bounds = bounds_from_exponents(e, self.qbits)
        return self._bounds

    def __repr__(self):
        return f"CompressedVolume(dims={self.dims}, qbits={self.qbits}, blocks={self.block_count})"


def compress_volume(vol: Volume, qbits: int) -> CompressedVolume:
    """compress_volume (codec.py:177-198) on the GPU, bit-exact."""
    import ctypes as C

    check_qbits(qbits)
    h = C.c_void_p()
    vals = np.ascontiguousarray(vol.values, dtype=np.float32)
    _lib.call("wc_volume_compress", _lib.ptr(vals), *vol.dims, int(qbits), C.byref(h))
    return CompressedVolume(vol.dims, qbits, handle=h)


def compress_separable(field: SeparableField, qbits: int) -> CompressedVolume:
    """Synthesise + compress a separable field block by block on the GPU
    (no dense field in host or device memory)."""
    import ctypes as C

    check_qbits(qbits)
    K = len(field.amp)
    arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (field.amp, field.fx, field.fy, field.fz)]
    h = C.c_void_p()
    _lib.call("wc_volume_synthesize", K, *[_lib.ptr(a) for a in arrs], *field.dims, int(qbits), C.byref(h))
    return CompressedVolume(field.dims, qbits, handle=h)


def decompress_block(cv: CompressedVolume, block_id: int) -> np.ndarray:
    """Decode one block to float32[64], x fastest (codec.py:201-206)."""
    assert 0 <= block_id < cv.block_count, f"block id {block_id} out of range"
    out = np.empty((1, 64), dtype=np.float32)
    decompress_blocks_into(cv, np.array([block_id], dtype=np.int64), out)
    return out[0]


def decompress_blocks_into(cv: CompressedVolume, block_ids, out: np.ndarray) -> None:
    """Decode many blocks at once (codec.py:209-217); out is (n, 64) float32."""
    ids = np.ascontiguousarray(block_ids, dtype=np.int64)
    assert out.shape == (len(ids), 64) and out.dtype == np.float32 and out.flags["C_CONTIGUOUS"]
    if len(ids) == 0:
        return
    _lib.call("wc_decode_blocks", cv.device_handle(), _lib.ptr(ids), len(ids), _lib.ptr(out))


def write_wcz(cv: CompressedVolume, path) -> None:
    """.wcz container (codec.py:226-240): header, float32 ranges, payload."""
    header = WCZ_MAGIC + struct.pack("<IIIIII", WCZ_VERSION, *cv.dims, cv.qbits, cv.block_stride_bytes)
    with open(path, "wb") as f:
        f.write(header)
        f.write(cv.raw_block_ranges.astype("<f4").tobytes())
        f.write(cv.payload.tobytes())


def probe_wcz(path):
    """Header of a .wcz container with read_wcz's validation (codec.py:246-262):
    returns (dims, qbits, stride, n_blocks); errors are DataError/UsageError
    with the reference's messages.  Host only."""
    v = [C.c_int() for _ in range(5)]
    nb = C.c_int64()
    _lib.call_host("wc_wcz_probe", os.fsencode(os.fspath(path)), *[C.byref(x) for x in v], C.byref(nb))
    return (v[0].value, v[1].value, v[2].value), v[3].value, v[4].value, nb.value


def load_wcz(path, chunk_bytes: int = 0) -> CompressedVolume:
    """read_wcz (codec.py:243-273) straight into HBM: the native loader streams
    the ranges and payload through two pinned chunks (file reads overlap the
    host-to-device copies) and builds the grids on the device.  The host
    views (payload, raw_block_ranges) are downloaded only if asked for."""
    dims, qbits, _, _ = probe_wcz(path)
    h = C.c_void_p()
    _lib.call("wc_volume_load_wcz", os.fsencode(os.fspath(path)), int(chunk_bytes), C.byref(h))
    return CompressedVolume(dims, qbits, handle=h)


def decoded_value_range(cv: CompressedVolume) -> tuple[float, float]:
    """oracle.decode_full(cv).value_range (oracle.py:22-39) computed on the
    device without materialising the dense volume: (min, max) of the decoded
    voxels inside dims, as float32 values widened to float."""
    lo, hi = C.c_double(), C.c_double()
    _lib.call("wc_volume_value_range", cv.device_handle(), C.byref(lo), C.byref(hi))
    return float(lo.value), float(hi.value)


def read_wcz(path) -> CompressedVolume:
    """Parse a .wcz container (codec.py:243-273); validation errors are DataError."""
    with open(path, "rb") as f:
        blob = f.read()
    if len(blob) < 28 or blob[:4] != WCZ_MAGIC:
        raise DataError(f"{path}: not a WCZ1 container")
    version, nx, ny, nz, qbits, stride = struct.unpack_from("<IIIIII", blob, 4)
    if version != WCZ_VERSION:
        raise DataError(f"{path}: unsupported container version {version}")
    check_qbits(qbits)
    if stride != block_stride_bytes(qbits):
        raise DataError(f"{path}: stride {stride} inconsistent with qbits {qbits}")
    bdx, bdy, bdz = _block_dims((nx, ny, nz))
    nb = bdx * bdy * bdz
    expected = 28 + 8 * nb + nb * stride
    if len(blob) != expected:
        raise DataError(f"{path}: expected {expected} bytes, found {len(blob)}")
    ranges = np.frombuffer(blob, dtype="<f4", count=2 * nb, offset=28).reshape(nb, 2).copy()
    payload = np.frombuffer(blob, dtype=np.uint8, offset=28 + 8 * nb).copy()
    return CompressedVolume((nx, ny, nz), int(qbits), payload=payload, raw_block_ranges=ranges)
