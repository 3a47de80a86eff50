"""Image-tile sharding across GPUs.

Each rank holds the full compressed volume and its own LRU cache and renders
an interleaved subset of square tiles as one device session (its own pass
loop, n_act and n_spec).  Because speculation never changes final pixels
(engine.py:1-9), the stitched frame equals the single-GPU frame bit for bit.
The exchange steps are the per-iso range tests (each rank computes a slice,
two in-place all-gathers assemble them) and the frame assembly: by default
every rank's sessions write each final pixel straight into rank 0's frame
over NVLink peer memory (FrameTarget, CUDA IPC) the moment its ray
terminates -- the collective fused into the composite, overlapped with the
remaining passes; alternatively every rank's RGBA8+depth (8 B/pixel) goes to
rank 0 alone with one NCCL gather, scattered into the frame on rank 0's GPU
(wc_scatter_pixels).
All of it is ordered on the session's CUDA stream, so a frame has no host
synchronisation besides the pass loop's own (``torch.distributed``; gloo on
CPU for tests).
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
    (w, h, rank, world, tile), so no pixel ids travel.  Each rank sends one
    block of [RGBA words | depth bits] padded to n_max pixels; the pixel id of
    every received word is precomputed (-1 = padding)."""
    import torch

    key = (w, h, world, tile, str(dev))
    plan = _GATHER_CACHE.get(key)
    if plan is None:
        pix = [tile_pixels(w, h, r, world, tile) for r in range(world)]
        n_max = max(1, max(len(p) for p in pix))
        index = np.full((world, n_max), -1, dtype=np.int64)
        for r, p in enumerate(pix):
            index[r, :len(p)] = p
        plan = {
            "n_max": n_max,
            "index_np": index,
            "index": torch.from_numpy(index.reshape(-1)).to(dev),
            "send": torch.zeros(2 * n_max, dtype=torch.int32, device=dev),
            "recv": torch.zeros((world, 2 * n_max), dtype=torch.int32, device=dev),
            "frame": torch.zeros((2, w * h), dtype=torch.int32, device=dev),
        }
        _GATHER_CACHE.clear()
        _GATHER_CACHE[key] = plan
    return plan


def check_tiles(w: int, h: int, world: int, tile: int) -> None:
    """Every rank must own at least one tile: the frame's collectives (range
    tests, tile gather) need all ranks (UsageError otherwise)."""
    from .errors import UsageError

    n_tiles = (-(w // -tile)) * (-(h // -tile))
    if n_tiles < world:
        raise UsageError(f"{w}x{h} in {tile}x{tile} tiles gives {n_tiles} tiles for {world} ranks: "
                         "use smaller tiles or fewer ranks")


def _to_frame(plan, w, h, dev, stream=None):
    """Rank 0: the scattered frame -> (rgba (h,w,4) u8, depth (h,w) f32) in host memory."""
    import torch

    frame = plan["frame"]
    if dev.type == "cuda":  # read back into a recycled page-locked buffer (full-speed D2H)
        from . import _lib

        base = _lib.pinned_pool.get(8 * w * h)
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            torch.from_numpy(base.view(np.int32)).view(2, w * h).copy_(frame, non_blocking=True)
        (stream or torch.cuda.current_stream(dev)).synchronize()
    else:
        base = frame.contiguous().numpy().view(np.uint8).reshape(-1)
    return base[:4 * w * h].reshape(h, w, 4), base[4 * w * h:].view(np.float32).reshape(h, w)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def gather_tiles(rgba_local, depth_local, w: int, h: int, tile: int = 32, group=None):
    """The finished tiles -> rank 0 (the pass loop's only exchange step):
    one gather of every rank's [RGBA words | depth bits] (8 B per pixel, over
    NCCL/NVLink; gloo on CPU) to rank 0 alone, then the scatter into the frame
    (wc_scatter_pixels on the device).  Inputs are the rank's (n,4) uint8 and
    (n,) float32 torch tensors in tile_pixels order.  Returns (rgba (h,w,4)
    uint8, depth (h,w) float32) numpy on rank 0, None elsewhere."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = rgba_local.device
    check_tiles(w, h, world, tile)
    plan = _gather_plan(w, h, world, tile, dev)
    k = rgba_local.shape[0]
    n_max = plan["n_max"]
    send = plan["send"]
    send[:k] = rgba_local.reshape(-1).view(dtype=__import__("torch").int32)
    send[n_max:n_max + k] = depth_local.view(dtype=__import__("torch").int32)
    return _gather_and_scatter(plan, rank, world, w, h, dev, group, None)


def _gather_and_scatter(plan, rank, world, w, h, dev, group, stream):
    import torch.distributed as dist

    recv = plan["recv"]
    dist.gather(plan["send"], list(recv.unbind(0)) if rank == 0 else None, dst=0, group=group)
    if rank != 0:
        return None
    frame = plan["frame"]
    n_max = plan["n_max"]
    if dev.type == "cuda":
        from . import _lib

        _lib.call("wc_scatter_pixels", recv.data_ptr(), n_max, plan["index"].data_ptr(), world * n_max,
                  frame[0].data_ptr(), frame[1].data_ptr(), stream.cuda_stream if stream is not None else
                  __import__("torch").cuda.current_stream(dev).cuda_stream)
    else:  # gloo (CPU tests): the same scatter on the host
        idx = plan["index_np"]
        r = recv.numpy().reshape(world, 2, n_max)
        f = frame.numpy()
        ok = idx >= 0
        f[0][idx[ok]] = r[:, 0, :][ok]
        f[1][idx[ok]] = r[:, 1, :][ok]
    return _to_frame(plan, w, h, dev, stream)


def session_stream(sess):
    """The session's CUDA stream as a torch stream (collectives on the session's
    buffers are ordered on it: no host synchronisation around them)."""
    import ctypes as C

    import torch

    from . import _lib

    p = C.c_void_p()
    _lib.call("wc_session_stream", sess.handle, C.byref(p))
    return torch.cuda.ExternalStream(p.value, device=torch.device("cuda", torch.cuda.current_device()))


def render_frame_split(sess, cam, iso, group=None, split=None):
    """One frame of a rank's tile session with the per-iso range tests split
    across the ranks (the exchange step of a multi-GPU frame besides the tile
    gather): each rank computes its slice of coarse cells (coarse bitmap
    words and 64-bit fine masks) during reset, two all-gathers over NCCL
    assemble them in place -- enqueued on the session's stream, after the
    reset and before the passes, with no host synchronisation -- then the
    passes run.  Returns the stats."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if not (world > 1 if split is None else split):  # one rank: nothing to exchange
        return sess.render_frame(cam, iso)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    sess.reset_part(cam, iso, rank, world)
    cb, cm, chunk = sess.mask_buffers(world)
    bits = torch.as_tensor(_DeviceBytes(cb, 4 * chunk * world), device=dev)
    masks = torch.as_tensor(_DeviceBytes(cm, 8 * 32 * chunk * world), device=dev)
    with torch.cuda.stream(session_stream(sess)):
        for buf, per in ((bits, 4 * chunk), (masks, 8 * 32 * chunk)):
            dist.all_gather_into_tensor(buf, buf[rank * per:(rank + 1) * per], group=group)
    return sess.run()


class FrameTarget:
    """The assembled frame on one GPU (the fused option):
    RGBA8 + depth for npix pixels that every rank's session writes its final
    pixels into -- over NVLink peer memory for the other ranks (CUDA IPC) --
    as its rays terminate, so the frame is complete when the last rank's last
    pass is, with no gather.  Created by the owner (``handles`` None), opened
    by the others from the owner's 128-byte IPC handles."""

    def __init__(self, npix: int, handles: bytes | None = None):
        import ctypes as C

        from . import _lib

        self.npix = int(npix)
        h = C.c_void_p()
        if handles is None:
            _lib.call("wc_frame_target_create", self.npix, C.byref(h))
        else:
            buf = C.create_string_buffer(bytes(handles), 128)
            _lib.call("wc_frame_target_open", buf, self.npix, C.byref(h))
        self.handle = h.value
        self.owner = handles is None

    def ipc_handles(self) -> bytes:
        import ctypes as C

        from . import _lib

        buf = C.create_string_buffer(128)
        _lib.call("wc_frame_target_ipc_handles", self.handle, buf)
        return buf.raw

    def download(self, w: int, h: int):
        """-> (rgba (h,w,4) uint8, depth (h,w) float32) in page-locked host memory."""
        from . import _lib

        base = _lib.pinned_pool.get(8 * self.npix)
        rgba = base[:4 * self.npix]
        depth = base[4 * self.npix:].view(np.float32)
        _lib.call("wc_frame_target_download", self.handle, _lib.ptr(rgba), _lib.ptr(depth))
        return rgba.reshape(h, w, 4), depth.reshape(h, w)

    def close(self):
        from . import _lib

        if self.handle:
            _lib.call("wc_frame_target_destroy", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_TARGETS: dict = {}


def _frame_target(w: int, h: int, world: int, rank: int, group):
    """Rank 0's full-frame target, opened by every rank (one per image size
    and group): the owner's IPC handles travel once, by an object broadcast."""
    import torch.distributed as dist

    key = (w, h, world, id(group))
    t = _TARGETS.get(key)
    if t is None:
        owner = FrameTarget(w * h) if rank == 0 else None
        if world > 1:
            obj = [owner.ipc_handles() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            t = owner if rank == 0 else FrameTarget(w * h, obj[0])
        else:
            t = owner
        _TARGETS.clear()
        _TARGETS[key] = t
    return t


_SHARD_SESSIONS: dict = {}


def render_sharded(cv, grids, cam, iso, opts, tile: int = 32, group=None, split=None, assembly: str = "peer"):
    """Render this rank's tiles on its GPU and assemble the frame on rank 0.
    Returns (framebuffer or None, local PassStats list).

    assembly="peer" (default): every rank's session writes its final pixels
    straight into rank 0's frame target over NVLink peer memory as its rays
    terminate (FrameTarget); a barrier, then rank 0 reads the frame back.
    assembly="nccl": the framebuffer pack, one NCCL gather to rank 0 and the
    scatter, ordered on the session's stream."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .engine import Framebuffer, RenderSession

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    check_tiles(opts.width, opts.height, world, tile)
    # one pooled session (and tile set) per (volume, image, options, world):
    # later frames reuse its HBM allocations through wc_session_render
    key = (id(cv), opts.width, opts.height, opts.speculation, opts.max_spec, opts.cache_capacity,
           opts.group_entries, tuple(opts.base_color), world, rank, tile)
    ent = _SHARD_SESSIONS.get(key)
    if ent is None or ent[0].cv is not cv:
        pix = tile_pixels(opts.width, opts.height, rank, world, tile)
        s = RenderSession(cv, grids, cam, iso, opts, pixel_ids=pix)
        ent = (s, pix)
        _SHARD_SESSIONS.clear()
        _SHARD_SESSIONS[key] = ent
    s, pix = ent
    if assembly == "peer":
        target = _frame_target(opts.width, opts.height, world, rank, group)
        if getattr(s, "_target", None) is not target:
            s.set_frame_target(target)
        stats = render_frame_split(s, cam, iso, group, split)
        session_stream(s).synchronize()  # this rank's pixels have landed in the target
        if world > 1:
            dist.barrier(group=group)
        if rank != 0:
            return None, stats
        rgba, depth = target.download(opts.width, opts.height)
        return Framebuffer(opts.width, opts.height, rgba, depth, 1.0), stats
    if getattr(s, "_target", None) is not None:
        s.set_frame_target(None)
    stats = render_frame_split(s, cam, iso, group, split)
    plan = _gather_plan(opts.width, opts.height, world, tile, dev)
    stream = session_stream(s)
    _lib.call("wc_session_framebuffer_packed", s.handle, plan["send"].data_ptr(), plan["n_max"])
    with torch.cuda.stream(stream):
        out = _gather_and_scatter(plan, rank, world, opts.width, opts.height, dev, group, stream)
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
