"""Two-level value-range grids (mirrors wavecast/grids.py).

Built on the device (csrc/wc_volume.cu k_widen / k_octant_union / k_group4,
grids.py:71-94) when a volume becomes resident, stored as float64
(min, max) pairs.  ``MacrocellGrids`` is a handle to those arrays with lazy
host views, or -- when constructed from caller arrays -- a host object that
``render_passes`` uploads into the volume.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .codec import CompressedVolume


@dataclass(frozen=True)
class ValueRange:
    min: float
    max: float

    def contains(self, iso: float) -> bool:
        return self.min <= iso <= self.max


class MacrocellGrids:
    """fine (one cell per block) and coarse (4^3 blocks) float64 ranges."""

    def __init__(self, fine_dims, fine_min=None, fine_max=None, coarse_dims=None, coarse_min=None,
                 coarse_max=None, volume: CompressedVolume | None = None):
        self.fine_dims = tuple(int(d) for d in fine_dims)
        self.coarse_dims = tuple(int(d) for d in coarse_dims) if coarse_dims is not None else tuple(
            -(d // -4) for d in self.fine_dims)
        self._host = None
        if fine_min is not None:
            self._host = tuple(np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
                               for a in (fine_min, fine_max, coarse_min, coarse_max))
        self._volume = volume

    @property
    def bound_volume(self):
        return self._volume

    def _arrays(self):
        if self._host is None:
            v = self._volume
            nb = int(np.prod(self.fine_dims))
            nc = int(np.prod(self.coarse_dims))
            arrs = (np.empty(nb), np.empty(nb), np.empty(nc), np.empty(nc))
            _lib.call("wc_volume_download", v.device_handle(), None, None, *[_lib.ptr(a) for a in arrs])
            self._host = arrs
        return self._host

    @property
    def fine_min(self):
        return self._arrays()[0]

    @property
    def fine_max(self):
        return self._arrays()[1]

    @property
    def coarse_min(self):
        return self._arrays()[2]

    @property
    def coarse_max(self):
        return self._arrays()[3]

    def fine_range(self, block_id: int) -> ValueRange:
        return ValueRange(float(self.fine_min[block_id]), float(self.fine_max[block_id]))

    def coarse_range(self, cell_id: int) -> ValueRange:
        return ValueRange(float(self.coarse_min[cell_id]), float(self.coarse_max[cell_id]))

    def bind(self, cv: CompressedVolume) -> None:
        """Make these ranges the ones the device traversal of `cv` reads."""
        if self._volume is cv:
            return
        fmin, fmax, cmin, cmax = self._arrays()
        _lib.call("wc_volume_set_grids", cv.device_handle(), *[_lib.ptr(a) for a in (fmin, fmax, cmin, cmax)])
        self._volume = cv


def build_grids(cv: CompressedVolume) -> MacrocellGrids:
    """grids.py:71-94 -- the device builds them with the volume; this binds a view."""
    cv.device_handle()
    bd = cv.block_dims
    return MacrocellGrids(bd, coarse_dims=tuple(-(d // -4) for d in bd), volume=cv)
