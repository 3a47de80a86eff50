"""Per-stage views of a device session, in the reference's buffer formats.

After ``RenderSession.step()`` these return what the reference engine would
hold after the same pass (engine.py:326-366): RaySoA fields, the slot
buffers of traverse_to_next_blocks, the visible / active block sets of
mark_blocks, BlockCache state and the PassBuffers of build_rt_inputs.  Used
by the parity tests; not on the render path.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .engine import PassBuffers, RenderSession

UINT_MAX = 0xFFFFFFFF


def sizes(sess: RenderSession) -> dict:
    s = np.empty(9, dtype=np.int64)
    _lib.call("wc_session_sizes", sess.handle, _lib.ptr(s))
    keys = ("slots_used", "n_visible", "n_active_blocks", "n_entries", "n_spec", "n_active_before", "cache_capacity",
            "cache_physical", "n_handed_off")
    return {k: int(v) for k, v in zip(keys, s)}


def session_rays(sess: RenderSession) -> dict:
    n = sess.n
    out = dict(dir=np.empty((n, 3)), t_enter=np.empty(n), t_exit=np.empty(n), status=np.empty(n, np.uint8),
               exited=np.empty(n, np.uint8), coarse_cell=np.empty(n, np.uint32), fine_cell=np.empty(n, np.uint32),
               coarse_tmax=np.empty((n, 3)), fine_tmax=np.empty((n, 3)))
    _lib.call("wc_session_rays", sess.handle, *[_lib.ptr(out[k]) for k in (
        "dir", "t_enter", "t_exit", "status", "exited", "coarse_cell", "fine_cell", "coarse_tmax", "fine_tmax")])
    return out


def pass_buffers(sess: RenderSession) -> dict:
    """Last pass's buffers in reference layout (engine.py / traversal.py)."""
    z = sizes(sess)
    n = sess.n
    used, nv, na, ne, n_prev = z["slots_used"], z["n_visible"], z["n_active_blocks"], z["n_entries"], z[
        "n_active_before"]
    bs = np.empty(max(used, 1), np.uint32)
    rs = np.empty(max(used, 1), np.uint32)
    alist = np.empty(max(n_prev, 1), np.uint32)
    _lib.call("wc_session_slots", sess.handle, _lib.ptr(bs), _lib.ptr(rs), _lib.ptr(alist))
    block_slots = np.full(n, UINT_MAX, np.uint32)
    ray_slots = np.full(n, UINT_MAX, np.uint32)
    block_slots[:used] = bs[:used]
    ray_slots[:used] = rs[:used]
    alist = alist[:n_prev]
    active_offsets = np.searchsorted(alist, np.arange(n, dtype=np.uint32)).astype(np.uint32)
    vis = np.empty(max(nv, 1), np.uint32)
    act = np.empty(max(na, 1), np.uint32)
    _lib.call("wc_session_blocks", sess.handle, _lib.ptr(vis), _lib.ptr(act))
    off = np.empty(nv + 1, np.uint32)
    sorted_k = np.empty(max(ne, 1), np.uint32)
    ent_ray = np.empty(max(ne, 1), np.uint32)
    _lib.call("wc_session_rt_inputs", sess.handle, _lib.ptr(off), _lib.ptr(sorted_k), _lib.ptr(ent_ray))
    sorted_k = sorted_k[:ne]
    ent_ray = ent_ray[:ne]
    rgbz4 = np.empty((max(ne, 1), 4), np.float32)
    _lib.call("wc_session_rgbz", sess.handle, _lib.ptr(rgbz4))
    rgbz_rgb = np.zeros((n, 3), np.float32)
    rgbz_z = np.full(n, np.inf, np.float32)
    rgbz_rgb[:ne] = rgbz4[:ne, :3]
    rgbz_z[:ne] = rgbz4[:ne, 3]
    valid = (block_slots != UINT_MAX).astype(np.uint64)
    valid_prefix = (np.cumsum(valid) - valid).astype(np.uint32)
    pb = PassBuffers(
        visible_ids=vis[:nv],
        rays_per_block=np.diff(off).astype(np.uint32) if ne else np.zeros(0, np.uint32),
        block_ray_offsets=off[:nv] if ne else np.zeros(0, np.uint32),
        sorted_ray_ids=ent_ray[sorted_k] if ne else np.zeros(0, np.uint32),
        sorted_hit_slots=sorted_k,
        valid_prefix=valid_prefix,
        n_entries=ne,
    )
    return dict(slots_used=used, n_spec=z["n_spec"], block_slots=block_slots, ray_slots=ray_slots,
                active_offsets=active_offsets, active_list=alist, visible_ids=vis[:nv], active_ids=act[:na],
                rt=pb, rgbz_rgb=rgbz_rgb, rgbz_z=rgbz_z)


def cache_state(sess: RenderSession, with_values: bool = False) -> dict:
    z = sizes(sess)
    phys = z["cache_physical"]
    bos = np.empty(phys, np.int32)
    lu = np.empty(phys, np.int32)
    sv = np.empty((phys, 64), np.float32) if with_values else None
    _lib.call("wc_session_cache", sess.handle, _lib.ptr(bos), _lib.ptr(lu), _lib.ptr(sv))
    return dict(capacity=z["cache_capacity"], physical=phys, block_of_slot=bos, last_used=lu, slot_values=sv)
