"""Multi-GPU host logic on CPU: 2 gloo ranks each render their interleaved
tiles (oracle standing in for the per-rank GPU session) and
dist.gather_tiles stitches the frame on rank 0; it must equal the one-rank
frame bit for bit (speculation invariance, engine.py:1-9)."""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_2309_10212_b200 import dist as wdist
    import paper_2309_10212_b200.volume as V

    vol = V.synthesize("gaussians", (40, 40, 40), seed=0)
    ov = orc.volume_from_values(vol.values, vol.dims, 16)
    w, h = 70, 50
    lo, hi = vol.value_range
    iso = lo + 0.3 * (hi - lo)
    cam = orc.orbit_camera(vol.dims, 0, 1)
    pix = wdist.tile_pixels(w, h, rank, world, 16)
    o, d = orc.camera_rays(cam, w, h, pix)
    rgba, depth, _ = orc.render(ov, o, d, len(pix), 1, iso)
    out = wdist.gather_tiles(torch.from_numpy(rgba), torch.from_numpy(depth), w, h, tile=16)
    if rank == 0:
        o, d = orc.camera_rays(cam, w, h)
        full_rgba, full_depth, _ = orc.render(ov, o, d, w, h, iso)
        ok = np.array_equal(out[0].reshape(-1, 4), full_rgba) and np.array_equal(out[1].reshape(-1), full_depth)
        q.put((ok, int(np.isfinite(full_depth).sum())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_tile_gather_stitches_bit_exact(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, hits = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok and hits > 0


def _bcast_worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_2309_10212_b200 import dist as wdist
    from paper_2309_10212_b200.codec import CompressedVolume

    dims = (13, 9, 11)
    v = np.random.default_rng(7).uniform(-2, 5, int(np.prod(dims))).astype(np.float32)
    pay, ranges, _ = orc.compress(v, dims, 12)
    cv = CompressedVolume(dims, 12, payload=pay, raw_block_ranges=ranges) if rank == 0 else None
    got = wdist.broadcast_volume(cv, src=0)
    ok = (got.dims == dims and got.qbits == 12 and np.array_equal(got.payload, pay)
          and np.array_equal(got.raw_block_ranges, ranges))
    q.put((rank, bool(ok)))
    dist.destroy_process_group()


def test_gloo_volume_broadcast():
    # host orchestration of dist.broadcast_volume (metadata, sizes, payload and
    # ranges); on NCCL the same calls write straight into the receivers' HBM
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bcast_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res == {0: True, 1: True}


def test_sharding_rejects_fewer_tiles_than_ranks():
    # every rank takes part in the frame's collectives, so each must own a tile
    from paper_2309_10212_b200 import dist as wdist
    from paper_2309_10212_b200.errors import UsageError

    with pytest.raises(UsageError, match="tiles"):
        wdist.check_tiles(64, 64, 8, 32)
    wdist.check_tiles(64, 64, 4, 32)
    assert sum(len(wdist.tile_pixels(64, 64, r, 4, 32)) for r in range(4)) == 64 * 64
