"""The reference's benchmark protocol on the device path.

``bench_report`` is ``wavecast bench`` (cli.py:122-195): random isovalues
drawn from the decoded value range (5 % margins, seeded), each rendered from
an equal-angle orbit of cameras, summarised into the same report dict (same
keys, same statistics of the per-pass ``PassStats``).  The PassStats are
bit-exact with the reference, so the report is too.  It also returns the
device timings of the renders, which the reference does not measure.
"""

from __future__ import annotations

import time

import numpy as np

from .codec import decoded_value_range
from .engine import RenderOptions, session_pool
from .traversal import Camera

REPORT_VERSION = 1  # cli.py:22


def volume_center(dims) -> tuple[float, float, float]:
    """cli.py:44-45"""
    return tuple((d - 1) / 2.0 for d in dims)


def orbit_camera(dims, step: int, steps: int, fov_y: float = 45.0) -> Camera:
    """Equal-angle azimuth orbit in the y = centre plane (cli.py:48-58)."""
    center = volume_center(dims)
    dist = 1.8 * max(dims)
    angle = 2.0 * np.pi * step / steps
    eye = (center[0] + dist * np.sin(angle), center[1], center[2] + dist * np.cos(angle))
    return Camera.look_at(eye, center, fov_y=fov_y)


def bench_scenes(dims, value_range, isovalues: int, orbit_steps: int, seed: int, iso_range=None):
    """(iso, camera) pairs in the reference's order (cli.py:122-133)."""
    lo, hi = value_range
    if iso_range is not None:
        iso_lo, iso_hi = iso_range
    else:
        span = hi - lo
        iso_lo, iso_hi = lo + 0.05 * span, hi - 0.05 * span
    rng = np.random.default_rng(seed)
    for iso in rng.uniform(iso_lo, iso_hi, isovalues):
        for k in range(orbit_steps):
            yield float(iso), orbit_camera(dims, k, orbit_steps)


def bench_report(cv, grids, *, isovalues: int = 100, orbit_steps: int = 10, seed: int = 0, width: int = 1280,
                 height: int = 720, speculation: str = "on", iso_range=None, volume: str = "",
                 value_range=None, max_spec: int = 64, cache_capacity=None):
    """cmd_bench (cli.py:136-195) -> (report, timings).

    ``value_range`` defaults to the decoded range computed on the device
    (oracle.decode_full(cv).value_range in the reference).  Renders go
    through the same pooled device session as ``render`` (its HBM allocations
    are reused; each render starts from fresh rays and an empty cache, as the
    reference's do).
    ``timings`` holds the device ms of every render and their summary."""
    if value_range is None:
        value_range = decoded_value_range(cv)
    opts = RenderOptions(width=width, height=height, speculation=speculation == "on", max_spec=max_spec,
                         cache_capacity=cache_capacity)
    pass_counts, visible_fracs, spec_counts, utilizations = [], [], [], []
    completeness_curves, new_per_pass = [], []
    max_slots = 0
    frame_ms, wall_ms, views, all_stats = [], [], [], []
    for iso, cam in bench_scenes(cv.dims, value_range, isovalues, orbit_steps, seed, iso_range):
        t0 = time.perf_counter()
        sess = session_pool.get(cv, grids, opts, cam)
        stats = sess.render_frame(cam, iso)
        wall_ms.append((time.perf_counter() - t0) * 1e3)
        frame_ms.append(sess.frame_ms())
        views.append((iso, cam))
        all_stats.append(stats)
        pass_counts.append(len(stats))
        if stats:
            visible_fracs.append(float(np.mean([s.visible_blocks for s in stats])) / cv.block_count)
            spec_counts.extend(s.n_spec for s in stats)
            utilizations.extend(s.utilization for s in stats)
            new_per_pass.extend(s.new_decompressed for s in stats)
            max_slots = max(max_slots, max(s.cache_slots for s in stats))
            completeness_curves.append([s.completeness for s in stats])
    max_passes = max((len(c) for c in completeness_curves), default=0)
    mean_completeness = [float(np.mean([c[i] if i < len(c) else 1.0 for c in completeness_curves]))
                         for i in range(max_passes)]
    report = {
        "report_version": REPORT_VERSION,
        "config": {
            "volume": str(volume),
            "qbits": cv.qbits,
            "isovalues": isovalues,
            "orbit_steps": orbit_steps,
            "seed": seed,
            "width": width,
            "height": height,
            "speculation": speculation,
            "iso_range": list(iso_range) if iso_range else None,
        },
        "n_renders": len(pass_counts),
        "median_passes": float(np.median(pass_counts)) if pass_counts else 0.0,
        "avg_visible_fraction": float(np.mean(visible_fracs)) if visible_fracs else 0.0,
        "median_spec_count": float(np.median(spec_counts)) if spec_counts else 0.0,
        "avg_utilization": float(np.mean(utilizations)) if utilizations else 0.0,
        "mean_completeness_by_pass": mean_completeness,
        "cache": {
            "mean_new_decompressed_per_pass": float(np.mean(new_per_pass)) if new_per_pass else 0.0,
            "max_cache_slots": int(max_slots),
        },
    }
    timings = {
        "frame_ms": frame_ms,
        "wall_ms": wall_ms,
        "mean_frame_ms": float(np.mean(frame_ms)) if frame_ms else 0.0,
        "median_frame_ms": float(np.median(frame_ms)) if frame_ms else 0.0,
        "max_frame_ms": float(np.max(frame_ms)) if frame_ms else 0.0,
        "passes": pass_counts,
        "value_range": list(value_range),
        "views": views,          # (iso, Camera) of every render, in order
        "stats": all_stats,      # its PassStats
    }
    return report, timings
