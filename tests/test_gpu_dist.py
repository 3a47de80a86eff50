"""The multi-GPU data plane (dist.py) under a one-rank NCCL
group on one GPU: the tile session, the range-test all-gathers and the tile
gather + device scatter, all ordered on the session stream, give the frame
render() gives, bit for bit."""

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


@pytest.mark.parametrize("tile,split", [(32, True), (16, True), (32, False)])
def test_render_sharded_one_rank_equals_render(wc, nccl, tile, split):
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
        fb, stats = wdist.render_sharded(cv, grids, cam, iso, opts, tile=tile, split=split)
        assert np.array_equal(fb.rgba, ref_rgba), (tile, k)
        assert np.array_equal(fb.depth.view(np.uint32), ref_depth.view(np.uint32)), (tile, k)
        assert [s.n_active_before for s in stats] == [s.n_active_before for s in ref_stats]
