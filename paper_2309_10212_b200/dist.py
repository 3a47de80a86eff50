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


def gather_tiles(rgba_local, depth_local, pix_local, w: int, h: int, group=None):
    """Gather every rank's (rgba u8 (n,4) as int32 words, depth f32) to rank 0
    and stitch.  Inputs are torch tensors on the rank's device (CUDA for
    NCCL, CPU for gloo).  Returns (rgba (h,w,4) uint8, depth (h,w)) numpy on
    rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = rgba_local.device
    n_local = torch.tensor([rgba_local.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(counts, n_local, group=group)
    n_max = int(max(int(c.item()) for c in counts))
    # one packed buffer per rank: [pixel id, rgba word, depth bits] x n_max
    packed = torch.full((n_max, 3), -1, dtype=torch.int32, device=dev)
    k = rgba_local.shape[0]
    if k:
        packed[:k, 0] = pix_local.to(torch.int32)
        packed[:k, 1] = rgba_local.view(torch.int32).reshape(-1)
        packed[:k, 2] = depth_local.view(torch.int32)
    bufs = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(bufs, packed, group=group)
    if rank != 0:
        return None
    allp = torch.cat(bufs, 0)
    allp = allp[allp[:, 0] >= 0]
    rgba = torch.zeros(w * h, dtype=torch.int32, device=dev)
    depth = torch.zeros(w * h, dtype=torch.int32, device=dev)
    idx = allp[:, 0].long()
    rgba[idx] = allp[:, 1]
    depth[idx] = allp[:, 2]
    rgba_np = rgba.cpu().numpy().view(np.uint8).reshape(h, w, 4)
    depth_np = depth.cpu().numpy().view(np.float32).reshape(h, w)
    return rgba_np, depth_np


def render_sharded(cv, grids, cam, iso, opts, tile: int = 32, group=None):
    """Render this rank's tiles on its GPU, gather the frame to rank 0.
    Returns (framebuffer or None, local PassStats list, session device ms)."""
    import torch
    import torch.distributed as dist

    from .engine import Framebuffer, RenderSession

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    pix = tile_pixels(opts.width, opts.height, rank, world, tile)
    dev = torch.device("cuda", torch.cuda.current_device())
    n = len(pix)
    rgba_t = torch.empty((n, 4), dtype=torch.uint8, device=dev)
    depth_t = torch.empty(n, dtype=torch.float32, device=dev)
    stats = []
    if n:
        with RenderSession(cv, grids, cam, iso, opts, pixel_ids=pix) as s:
            stats = s.run()
            torch.cuda.synchronize()
            from . import _lib

            _lib.call("wc_session_framebuffer_device", s.handle, rgba_t.data_ptr(), depth_t.data_ptr())
    pix_t = torch.from_numpy(pix.astype(np.int64)).to(dev)
    out = gather_tiles(rgba_t, depth_t, pix_t, opts.width, opts.height, group)
    if out is None:
        return None, stats
    rgba, depth = out
    return Framebuffer(opts.width, opts.height, rgba, depth, 1.0), stats
