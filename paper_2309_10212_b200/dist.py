"""Image-tile sharding across GPUs.

Each rank holds the full compressed volume and its own LRU cache and renders
an interleaved subset of square tiles as one device session (its own pass
loop, n_act and n_spec).  Because speculation never changes final pixels
(engine.py:1-9), the stitched frame equals the single-GPU frame bit for bit.
The only exchange step is the final tile gather: every rank's RGBA8+depth
(8 B/pixel) goes to rank 0 with one NCCL collective over NVLink
(``torch.distributed``; gloo on CPU for tests).
"""

from __future__ import annotations

import numpy as np


def tile_pixels(w: int, h: int, rank: int, world: int, tile: int = 32) -> np.ndarray:
    """Pixel ids of the tiles owned by `rank`, tile-major, row-major inside a
    tile (a warp traces one 32-pixel tile row).  Tiles are dealt round-robin
    over a row-major tile order, which interleaves ranks across the image so
    the surface-heavy centre is shared evenly."""
    tx = -(w // -tile)
    ty = -(h // -tile)
    out = []
    for t in range(rank, tx * ty, world):
        x0 = (t % tx) * tile
        y0 = (t // tx) * tile
        xs = np.arange(x0, min(x0 + tile, w))
        for y in range(y0, min(y0 + tile, h)):
            out.append(y * w + xs)
    if not out:
        return np.zeros(0, dtype=np.uint32)
    return np.concatenate(out).astype(np.uint32)


_GATHER_CACHE: dict = {}


def _gather_plan(w, h, world, tile, dev):
    """Per (image, world, tile): every rank's pixel list is a pure function of
    (w, h, rank, world, tile), so no pixel ids travel -- rank 0 scatters each
    rank's block of words with a precomputed index (padding -> dummy slot w*h)."""
    import torch

    key = (w, h, world, tile, str(dev))
    plan = _GATHER_CACHE.get(key)
    if plan is None:
        pix = [tile_pixels(w, h, r, world, tile) for r in range(world)]
        n_max = max(1, max(len(p) for p in pix))
        index = np.full((world, n_max), w * h, dtype=np.int64)
        for r, p in enumerate(pix):
            index[r, :len(p)] = p
        plan = {
            "n_max": n_max,
            "index": torch.from_numpy(index.reshape(-1)).to(dev),
            "send": torch.zeros((2, n_max), dtype=torch.int32, device=dev),
            "recv": torch.empty((world, 2, n_max), dtype=torch.int32, device=dev),
            "frame": torch.zeros((2, w * h + 1), dtype=torch.int32, device=dev),
        }
        _GATHER_CACHE.clear()
        _GATHER_CACHE[key] = plan
    return plan


def gather_tiles(rgba_local, depth_local, w: int, h: int, tile: int = 32, group=None):
    """The finished tiles -> rank 0 (the pass loop's only exchange step):
    one all_gather_into_tensor of every rank's [RGBA words | depth bits]
    (8 B per pixel, over NCCL/NVLink; gloo on CPU), then one scatter into the
    frame on rank 0.  Inputs are the rank's (n,4) uint8 and (n,) float32
    torch tensors in tile_pixels order.  Returns (rgba (h,w,4) uint8,
    depth (h,w) float32) numpy on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = rgba_local.device
    plan = _gather_plan(w, h, world, tile, dev)
    k = rgba_local.shape[0]
    send = plan["send"]
    if k:
        send[0, :k] = rgba_local.reshape(-1).view(torch.int32)
        send[1, :k] = depth_local.view(torch.int32)
    dist.all_gather_into_tensor(plan["recv"].view(-1), send.view(-1), group=group)
    if rank != 0:
        return None
    frame = plan["frame"]
    idx = plan["index"]
    frame[0].index_copy_(0, idx, plan["recv"][:, 0, :].reshape(-1))
    frame[1].index_copy_(0, idx, plan["recv"][:, 1, :].reshape(-1))
    frame = frame[:, : w * h]  # [rgba words | depth bits], dummy slot dropped
    if dev.type == "cuda":  # read back into a recycled page-locked buffer (full-speed D2H)
        from . import _lib

        base = _lib.pinned_pool.get(8 * w * h)
        torch.from_numpy(base.view(np.int32)).view(2, w * h).copy_(frame)
    else:
        base = frame.contiguous().numpy().view(np.uint8).reshape(-1)
    rgba_np = base[:4 * w * h].reshape(h, w, 4)
    depth_np = base[4 * w * h:].view(np.float32).reshape(h, w)
    return rgba_np, depth_np


def render_frame_split(sess, cam, iso, group=None):
    """One frame of a rank's tile session with the per-iso range tests split
    across the ranks (the exchange step of a multi-GPU frame besides the tile
    gather): each rank computes its slice of coarse cells (coarse bitmap
    words and 64-bit fine masks) during reset, one all-gather per buffer over
    NCCL assembles them in place, then the passes run.  Returns the stats."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return sess.render_frame(cam, iso)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    sess.reset_part(cam, iso, rank, world)
    cb, cm, chunk = sess.mask_buffers(world)
    bits = torch.as_tensor(_DeviceBytes(cb, 4 * chunk * world), device=dev)
    masks = torch.as_tensor(_DeviceBytes(cm, 8 * 32 * chunk * world), device=dev)
    sess.sync()  # the slice is written (session stream) before NCCL reads it
    for buf, per in ((bits, 4 * chunk), (masks, 8 * 32 * chunk)):
        dist.all_gather_into_tensor(buf, buf[rank * per:(rank + 1) * per], group=group)
    torch.cuda.current_stream(dev).synchronize()  # gathered before the passes read them
    return sess.run()


_SHARD_SESSIONS: dict = {}


def render_sharded(cv, grids, cam, iso, opts, tile: int = 32, group=None):
    """Render this rank's tiles on its GPU, gather the frame to rank 0.
    Returns (framebuffer or None, local PassStats list, session device ms)."""
    import torch
    import torch.distributed as dist

    from .engine import Framebuffer, RenderSession

    from . import _lib

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    # one pooled session (and tile set) per (volume, image, options, world):
    # later frames reuse its HBM allocations through wc_session_render
    key = (id(cv), opts.width, opts.height, opts.speculation, opts.max_spec, opts.cache_capacity,
           opts.group_entries, tuple(opts.base_color), world, rank, tile)
    ent = _SHARD_SESSIONS.get(key)
    if ent is None or ent[0].cv is not cv:
        pix = tile_pixels(opts.width, opts.height, rank, world, tile)
        s = RenderSession(cv, grids, cam, iso, opts, pixel_ids=pix) if len(pix) else None
        ent = (s, pix)
        _SHARD_SESSIONS.clear()
        _SHARD_SESSIONS[key] = ent
    s, pix = ent
    n = len(pix)
    rgba_t = torch.empty((n, 4), dtype=torch.uint8, device=dev)
    depth_t = torch.empty(n, dtype=torch.float32, device=dev)
    stats = []
    if n:
        stats = render_frame_split(s, cam, iso, group)
        _lib.call("wc_session_framebuffer_device", s.handle, rgba_t.data_ptr(), depth_t.data_ptr())
    out = gather_tiles(rgba_t, depth_t, opts.width, opts.height, tile, group)
    if out is None:
        return None, stats
    rgba, depth = out
    return Framebuffer(opts.width, opts.height, rgba, depth, 1.0), stats


class _DeviceBytes:
    """``__cuda_array_interface__`` view of raw device memory, so torch (and
    NCCL through torch.distributed) can write straight into library buffers."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3}


def broadcast_volume(cv, src: int = 0, group=None):
    """Give every rank the same compressed volume.

    Rank ``src`` passes its CompressedVolume (e.g. from ``codec.load_wcz``);
    the other ranks pass None.  Over NCCL the payload and raw ranges are
    broadcast from the source's HBM straight into a volume the receivers
    allocated on their GPU (``wc_volume_alloc`` / ``wc_volume_device_buffers``),
    and each receiver builds its grids locally (``wc_volume_finalize``; the
    grids are a pure function of payload and ranges, grids.py:71-94), so no
    rank stages 16.6 GB through host memory.  Over gloo (CPU tests) the host
    arrays are broadcast instead and host-backed volumes are returned."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from . import _lib
    from .codec import CompressedVolume

    rank = dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
    meta = torch.zeros(4, dtype=torch.int64, device=dev)
    if rank == src:
        meta[:] = torch.tensor([*cv.dims, cv.qbits], dtype=torch.int64)
    dist.broadcast(meta, src, group)
    dims, qbits = tuple(int(x) for x in meta[:3].tolist()), int(meta[3])
    if not nccl:
        if rank == src:
            pay = torch.from_numpy(cv.payload.copy())
            rng = torch.from_numpy(cv.raw_block_ranges.reshape(-1).copy())
        else:
            from .codec import _block_dims, block_stride_bytes

            bd = _block_dims(dims)
            nb = bd[0] * bd[1] * bd[2]
            pay = torch.empty(nb * block_stride_bytes(qbits), dtype=torch.uint8)
            rng = torch.empty(2 * nb, dtype=torch.float32)
        dist.broadcast(pay, src, group)
        dist.broadcast(rng, src, group)
        if rank == src:
            return cv
        return CompressedVolume(dims, qbits, payload=pay.numpy(), raw_block_ranges=rng.numpy().reshape(-1, 2))
    if rank != src:
        h = C.c_void_p()
        _lib.call("wc_volume_alloc", *dims, qbits, C.byref(h))
        cv = CompressedVolume(dims, qbits, handle=h)
    pp, pb, rp, rb = C.c_void_p(), C.c_uint64(), C.c_void_p(), C.c_uint64()
    _lib.call("wc_volume_device_buffers", cv.device_handle(), C.byref(pp), C.byref(pb), C.byref(rp), C.byref(rb))
    torch.cuda.synchronize()  # the source's volume stream has finished writing
    for p_, n_ in ((pp, pb), (rp, rb)):
        t = torch.as_tensor(_DeviceBytes(p_.value, n_.value), device=dev)
        dist.broadcast(t, src, group)
    torch.cuda.synchronize()
    if rank != src:
        _lib.call("wc_volume_finalize", cv.device_handle())
    return cv
