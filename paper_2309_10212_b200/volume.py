"""Dense scalar volumes and deterministic synthetic fields (host side).

Mirrors wavecast/volume.py (Volume :28-44, load_raw/save_raw :56-81,
synthesize :84-102).  Volume synthesis is input preparation, not the render
path, so it stays numpy.  Two generators are new:
``gaussians`` and ``turbulence``.  Both are *separable sums*

    v(x, y, z) = sum_k ((a_k * fz_k[z]) * fy_k[y]) * fx_k[x]     (float32)

with float32 1-D factor tables computed in float64 on the host.  The same
tables drive the device generator (wc_volume_synthesize), which evaluates
the identical float32 expression block by block, so a 8.05B-voxel field is
never materialised and the GPU and numpy fields are bit-identical.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .errors import DataError, UsageError

_RAW_TYPES = {"u8": np.dtype("<u1"), "u16": np.dtype("<u2"), "f32": np.dtype("<f4")}

ML_FREQ = 6.0    # Marschner-Lobb f_M (volume.py:23-25)
ML_ALPHA = 0.25


@dataclass(frozen=True)
class Volume:
    """Dense float32 field, x fastest: flat index x + nx*(y + ny*z)."""

    dims: tuple[int, int, int]
    values: np.ndarray
    value_range: tuple[float, float]

    def __post_init__(self):
        nx, ny, nz = self.dims
        assert self.values.dtype == np.float32
        assert self.values.shape == (nx * ny * nz,)

    def as_3d(self) -> np.ndarray:
        nx, ny, nz = self.dims
        return self.values.reshape(nz, ny, nx)


def make_volume(dims, values) -> Volume:
    flat = np.ascontiguousarray(np.asarray(values).reshape(-1), dtype=np.float32)
    return Volume(tuple(int(d) for d in dims), flat, (float(flat.min()), float(flat.max())))


def load_raw(path, dims, dtype: str) -> Volume:
    """Headerless little-endian raw volume; integers cast to float32 as-is."""
    if dtype not in _RAW_TYPES:
        raise UsageError(f"unknown dtype {dtype!r}; expected one of {sorted(_RAW_TYPES)}")
    nx, ny, nz = (int(d) for d in dims)
    if min(nx, ny, nz) < 1:
        raise UsageError(f"dims must be positive, got {(nx, ny, nz)}")
    want = nx * ny * nz * _RAW_TYPES[dtype].itemsize
    have = os.path.getsize(path)
    if have != want:
        raise DataError(f"{path}: expected {want} bytes for dims {(nx, ny, nz)} dtype {dtype}, file has {have} bytes")
    return make_volume((nx, ny, nz), np.fromfile(path, dtype=_RAW_TYPES[dtype]).astype(np.float32))


def save_raw(volume: Volume, path) -> None:
    volume.values.astype("<f4").tofile(path)


# ------------------------------------------------------------ reference kinds
def _axes(nx, ny, nz):
    z, y, x = np.meshgrid(np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
                          np.arange(nx, dtype=np.float64), indexing="ij")
    return x, y, z


def _sphere(nx, ny, nz):
    x, y, z = _axes(nx, ny, nz)
    c = ((nx - 1) / 2.0, (ny - 1) / 2.0, (nz - 1) / 2.0)
    return np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2).astype(np.float32)


def _marschner_lobb(nx, ny, nz):
    x, y, z = _axes(nx, ny, nz)
    u = 2.0 * x / (nx - 1) - 1.0
    v = 2.0 * y / (ny - 1) - 1.0
    w = 2.0 * z / (nz - 1) - 1.0
    r = np.sqrt(u * u + v * v)
    rho = np.cos(2.0 * np.pi * ML_FREQ * np.cos(np.pi * r / 2.0))
    f = (1.0 - np.sin(np.pi * w / 2.0) + ML_ALPHA * (1.0 + rho)) / (2.0 * (1.0 + ML_ALPHA))
    return f.astype(np.float32)


_M64 = (1 << 64) - 1


def _splitmix_finalize(h):
    with np.errstate(over="ignore"):
        h = (h ^ (h >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        h = (h ^ (h >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return h ^ (h >> np.uint64(31))


def _splitmix_int(h: int) -> int:
    h &= _M64
    h = ((h ^ (h >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    h = ((h ^ (h >> 27)) * 0x94D049BB133111EB) & _M64
    return h ^ (h >> 31)


def _hash01(ix, iy, iz, salt):
    h = (ix.astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
         ^ iy.astype(np.uint64) * np.uint64(0xC2B2AE3D27D4EB4F)
         ^ iz.astype(np.uint64) * np.uint64(0x165667B19E3779F9)
         ^ salt)
    return (_splitmix_finalize(h) >> np.uint64(11)).astype(np.float64) * (1.0 / 2**53)


def _value_noise(nx, ny, nz, seed: int):
    x, y, z = _axes(nx, ny, nz)
    acc_all = np.zeros((nz, ny, nx), dtype=np.float64)
    amp, norm = 1.0, 0.0
    for octave in range(4):
        cell = 16.0 / (1 << octave)
        salt = np.uint64(_splitmix_int(int(seed) + octave + 1))
        fx, fy, fz = x / cell, y / cell, z / cell
        ix, iy, iz = np.floor(fx), np.floor(fy), np.floor(fz)
        tx, ty, tz = fx - ix, fy - iy, fz - iz
        tx = tx * tx * (3.0 - 2.0 * tx)  # smoothstep: C1 across lattice cells
        ty = ty * ty * (3.0 - 2.0 * ty)
        tz = tz * tz * (3.0 - 2.0 * tz)
        octave_sum = np.zeros_like(acc_all)
        for oz in (0.0, 1.0):
            wz = tz if oz else 1.0 - tz
            for oy in (0.0, 1.0):
                wy = ty if oy else 1.0 - ty
                for ox in (0.0, 1.0):
                    wx = tx if ox else 1.0 - tx
                    octave_sum += _hash01(ix + ox, iy + oy, iz + oz, salt) * (wx * wy * wz)
        acc_all += amp * octave_sum
        norm += amp
        amp *= 0.5
    return (acc_all / norm).astype(np.float32)


# ------------------------------------------------------ separable generators
@dataclass(frozen=True)
class SeparableField:
    """v = sum_k ((amp[k] * fz[k, z]) * fy[k, y]) * fx[k, x], all float32."""

    dims: tuple[int, int, int]
    amp: np.ndarray  # float32 (K,)
    fx: np.ndarray   # float32 (K, nx)
    fy: np.ndarray   # float32 (K, ny)
    fz: np.ndarray   # float32 (K, nz)

    def evaluate(self) -> np.ndarray:
        """Dense (nz, ny, nx) float32 field in the device's operation order."""
        nx, ny, nz = self.dims
        out = np.zeros((nz, ny, nx), dtype=np.float32)
        for k in range(len(self.amp)):
            term = self.amp[k] * self.fz[k][:, None, None]
            term = term * self.fy[k][None, :, None]
            term = term * self.fx[k][None, None, :]
            out += term
        return out


def gaussians_field(dims, n_terms: int = 24, seed: int = 0) -> SeparableField:
    """C2: sum of isotropic Gaussians."""
    n = np.asarray(dims, dtype=np.float64)
    rng = np.random.default_rng(seed)
    scale = float(n.max())
    centres = rng.uniform(0.15, 0.85, (n_terms, 3)) * n
    sigma = rng.uniform(0.04 * scale, 0.12 * scale, n_terms)
    amp = rng.uniform(0.5, 1.0, n_terms).astype(np.float32)

    def axis(a):
        t = np.arange(int(n[a]), dtype=np.float64)[None, :]
        return np.exp(-((t - centres[:, a, None]) ** 2) / (2.0 * sigma[:, None] ** 2)).astype(np.float32)

    return SeparableField(tuple(int(d) for d in dims), amp, axis(0), axis(1), axis(2))


def turbulence_field(dims, n_modes: int = 12, seed: int = 1) -> SeparableField:
    """C3: separable Fourier modes with a k^(-5/3)-like energy spectrum
    (SURVEY.md §8(d) C3, Appendix B)."""
    rng = np.random.default_rng(seed)
    freq = rng.uniform(0.5, 12.0, (n_modes, 3)) * (2.0 * np.pi)
    amp = ((np.linalg.norm(freq, axis=1) / (2.0 * np.pi)) ** (-5.0 / 6.0)).astype(np.float32)
    phase = rng.uniform(0.0, 2.0 * np.pi, (n_modes, 3))

    def axis(a):
        m = int(dims[a])
        t = np.arange(m, dtype=np.float64)[None, :]
        return np.sin(freq[:, a, None] * t / m + phase[:, a, None]).astype(np.float32)

    return SeparableField(tuple(int(d) for d in dims), amp, axis(0), axis(1), axis(2))


def separable_field(kind: str, dims, seed: int | None = None) -> SeparableField:
    if kind == "gaussians":
        return gaussians_field(dims, seed=0 if seed is None else seed)
    if kind == "turbulence":
        return turbulence_field(dims, seed=1 if seed is None else seed)
    raise UsageError(f"{kind!r} is not a separable volume kind")


SEPARABLE_KINDS = ("gaussians", "turbulence")


def synthesize(kind: str, dims, seed: int = 0) -> Volume:
    """Deterministic test volume (volume.py:84-102 kinds + C2/C3 kinds)."""
    nx, ny, nz = (int(d) for d in dims)
    if min(nx, ny, nz) < 8:
        raise UsageError(f"synthesized dims must be at least (8,8,8), got {(nx, ny, nz)}")
    if kind == "sphere":
        vals = _sphere(nx, ny, nz)
    elif kind == "marschner_lobb":
        vals = _marschner_lobb(nx, ny, nz)
    elif kind == "value_noise":
        vals = _value_noise(nx, ny, nz, seed)
    elif kind in SEPARABLE_KINDS:
        vals = separable_field(kind, (nx, ny, nz), seed).evaluate()
    else:
        raise UsageError(f"unknown volume kind {kind!r}")
    return make_volume((nx, ny, nz), vals)
