"""The multi-GPU data plane (dist.py) on one GPU: under a
one-rank NCCL group (the tile session, the range-test all-gathers, and the
frame assembly -- peer-memory frame target or NCCL gather + device scatter),
with several tile sessions writing one frame target, and with two processes
writing one frame target through CUDA IPC: every assembled frame equals
render()'s, bit for bit."""

import os
import socket

import numpy as np
import pytest

from helpers import host_volume, iso_at, orbit, wc_camera

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl():
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def wc():
    import paper_2309_10212_b200 as wc

    wc._lib.ensure_device(0)
    return wc


@pytest.mark.parametrize("assembly", ["peer", "nccl"])
@pytest.mark.parametrize("tile,split", [(32, True), (16, True), (32, False)])
def test_render_sharded_one_rank_equals_render(wc, nccl, tile, split, assembly):
    from paper_2309_10212_b200 import dist as wdist

    vol = host_volume("value_noise", 64)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    opts = wc.RenderOptions(width=150, height=97)
    for k, frac in enumerate((0.1, 0.45, 0.1)):  # a pooled session over several frames
        cam = wc_camera(wc, orbit(cv.dims, frac))
        iso = iso_at(vol, 0.4 + 0.1 * k)
        ref, ref_stats = wc.render(cv, grids, cam, iso, opts)
        ref_rgba, ref_depth = ref.rgba.copy(), ref.depth.copy()
        fb, stats = wdist.render_sharded(cv, grids, cam, iso, opts, tile=tile, split=split, assembly=assembly)
        assert np.array_equal(fb.rgba, ref_rgba), (tile, k)
        assert np.array_equal(fb.depth.view(np.uint32), ref_depth.view(np.uint32)), (tile, k)
        assert [s.n_active_before for s in stats] == [s.n_active_before for s in ref_stats]


def test_tile_sessions_write_one_frame_target(wc):
    """Three tile sessions (the tile sets of a 3-way split) write their final
    pixels into one frame target as their rays terminate: the target holds
    render()'s frame, over several frames of the same sessions."""
    from paper_2309_10212_b200 import dist as wdist

    vol = host_volume("value_noise", 64, seed=2)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    w, h, world = 131, 90, 3
    opts = wc.RenderOptions(width=w, height=h)
    target = wdist.FrameTarget(w * h)
    cam0 = wc_camera(wc, orbit(cv.dims, 0.2))
    sessions = []
    for r in range(world):
        s = wc.RenderSession(cv, grids, cam0, iso_at(vol, 0.5), opts, pixel_ids=wdist.tile_pixels(w, h, r, world, 16))
        s.set_frame_target(target)
        sessions.append(s)
    for k, frac in enumerate((0.2, 0.6, 0.2)):
        cam = wc_camera(wc, orbit(cv.dims, frac))
        iso = iso_at(vol, 0.45 + 0.05 * k)
        ref, _ = wc.render(cv, grids, cam, iso, opts)
        ref_rgba, ref_depth = ref.rgba.copy(), ref.depth.copy()
        for s in sessions:
            s.render_frame(cam, iso)
        for s in sessions:
            wdist.session_stream(s).synchronize()
        rgba, depth = target.download(w, h)
        assert np.array_equal(rgba, ref_rgba), k
        assert np.array_equal(depth.view(np.uint32), ref_depth.view(np.uint32)), k
    for s in sessions:
        s.close()
    target.close()


def _ipc_rank(rank, world, port, out_path):
    """One process of a 2-rank gloo group on the same GPU: rank 0 owns the
    frame target, rank 1 writes into it through CUDA IPC."""
    import torch
    import torch.distributed as dist

    import paper_2309_10212_b200 as wc
    from paper_2309_10212_b200 import dist as wdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    wc._lib.ensure_device(0)
    vol = host_volume("value_noise", 64, seed=6)
    cv = wc.compress_volume(vol, 16)
    grids = wc.build_grids(cv)
    opts = wc.RenderOptions(width=140, height=100)
    ok = True
    for k, frac in enumerate((0.3, 0.7)):
        cam = wc_camera(wc, orbit(cv.dims, frac))
        iso = iso_at(vol, 0.5)
        fb, _ = wdist.render_sharded(cv, grids, cam, iso, opts, tile=32, split=False, assembly="peer")
        if rank == 0:
            ref, _ = wc.render(cv, grids, cam, iso, opts)
            ok &= bool(np.array_equal(fb.rgba, ref.rgba)) and bool(
                np.array_equal(fb.depth.view(np.uint32), ref.depth.view(np.uint32)))
        dist.barrier()
    if rank == 0:
        with open(out_path, "w") as f:
            f.write("ok" if ok else "mismatch")
    dist.destroy_process_group()


def test_two_processes_assemble_through_ipc(tmp_path):
    """Rank 1's tiles reach rank 0's frame through CUDA IPC peer memory (two
    processes on one GPU; nothing waits on another rank inside a kernel)."""
    import torch.multiprocessing as mp

    out = tmp_path / "ipc.txt"
    mp.start_processes(_ipc_rank, args=(2, _free_port(), str(out)), nprocs=2, join=True, start_method="spawn")
    assert out.read_text() == "ok"
