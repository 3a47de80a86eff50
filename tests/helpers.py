"""Shared test helpers: scenes, cameras, lock-step GPU-vs-oracle comparison."""

from __future__ import annotations

import functools

import numpy as np

from oracle import oracle as orc

UINT_MAX = 0xFFFFFFFF
STAT_KEYS = ("pass_index", "n_active_before", "n_spec", "visible_blocks", "active_blocks", "new_decompressed",
             "cache_slots", "utilization", "completeness")


def orbit(dims, frac=0.0, fov=45.0):
    """cli.py:48-58 orbit camera as (eye, look_dir, up, fov) for the oracle."""
    return orc.orbit_camera(dims, frac, 1.0, fov) if frac else orc.orbit_camera(dims, 0, 1, fov)


def wc_camera(wc, cam_tuple):
    eye, look, up, fov = cam_tuple
    return wc.Camera(tuple(eye), tuple(look), tuple(up), fov)


@functools.lru_cache(maxsize=None)
def host_volume(kind: str, n, seed: int = 3):
    import paper_2309_10212_b200.volume as V

    dims = (n, n, n) if isinstance(n, int) else tuple(n)
    return V.synthesize(kind, dims, seed=seed)


def oracle_volume(cv):
    return orc.volume_from_payload(cv.dims, cv.qbits, cv.payload, cv.raw_block_ranges)


def iso_at(vol, frac):
    lo, hi = vol.value_range
    return lo + frac * (hi - lo)


def lockstep(wc, cv, ov, cam_tuple, w, h, iso, *, speculation=True, max_spec=64, cache_capacity=None,
             pixel_ids=None, origins=None, dirs=None, internals=True, corrupt=False, group=None, frames=None,
             probe=None):
    """Run the GPU session and the oracle session pass by pass; assert every
    per-pass stat, per-stage buffer and the final framebuffer are identical.

    group: sort entries by block (build_rt_inputs' PassBuffers compared too);
    default = internals.  group=False is the product path: ray-ordered
    entries, every pass replayed as a captured CUDA graph; all buffers but the
    grouped ones are compared (rgbz per entry id is order-independent).
    frames: extra [(cam_tuple, iso)] rendered after the first on the same
    session (wc_session_reset: the pass graphs captured by the first frame are
    replayed), each against a fresh oracle session.
    probe: called as probe(session, pass_index) after each compared pass."""
    if group is None:
        group = internals
    cam = wc_camera(wc, cam_tuple) if cam_tuple is not None else None
    opts = wc.RenderOptions(width=w, height=h, speculation=speculation, max_spec=max_spec,
                            cache_capacity=cache_capacity, corrupt_cache=corrupt, group_entries=group)
    sess = wc.RenderSession(cv, wc.build_grids(cv), cam, iso, opts, pixel_ids=pixel_ids, origins=origins, dirs=dirs)
    from paper_2309_10212_b200 import debug

    out = None
    for fi, (ct, fiso) in enumerate([(cam_tuple, iso)] + list(frames or [])):
        if fi > 0:
            sess.reset(wc_camera(wc, ct) if ct is not None else None, fiso)
        if dirs is None:
            o, d = orc.camera_rays(ct, w, h, pixel_ids)
        else:
            o, d = np.asarray(origins, dtype=np.float64), np.asarray(dirs, dtype=np.float64)
        os_ = orc.Session(ov, o, d, w, h, fiso, speculation=speculation, max_spec=max_spec,
                          cache_capacity=cache_capacity or 0, corrupt_cache=corrupt)
        # ray setup parity (traversal.py:105-187)
        if internals:
            g = debug.session_rays(sess)
            r = os_.rays()
            assert np.array_equal(g["dir"], d), "ray directions"
            for k in ("t_enter", "t_exit", "status", "coarse_cell", "fine_cell", "coarse_tmax", "fine_tmax"):
                assert np.array_equal(g[k], r[k]), f"frame {fi} init {k}"
        n_pass = 0
        stats = []
        while True:
            gs = sess.step()
            rs = os_.step()
            assert (gs is None) == (rs is None), f"frame {fi}: pass count differs at pass {n_pass}"
            if gs is None:
                break
            for k in STAT_KEYS:
                assert getattr(gs, k) == rs[k], f"frame {fi} pass {n_pass} stat {k}: gpu {getattr(gs, k)} " \
                                                f"oracle {rs[k]}"
            assert sess.last_c_stats.evicted == rs["evicted"], f"frame {fi} pass {n_pass} evicted"
            if internals:
                compare_pass(sess, os_, n_pass, grouped=group)
            if probe is not None:
                probe(sess, n_pass)
            stats.append(gs)
            n_pass += 1
        rgba, depth = sess.read()
        orgba, odepth = os_.framebuffer()
        assert np.array_equal(rgba, orgba), f"frame {fi} final RGBA"
        assert np.array_equal(depth.view(np.uint32), odepth.view(np.uint32)), f"frame {fi} final depth (bitwise)"
        os_.close()
        if out is None:
            out = (stats, rgba.copy(), depth.copy())
    sess.close()
    return out


def compare_pass(sess, os_, n_pass, with_values=True, grouped=True):
    """Every stage buffer of the last pass, GPU vs oracle, bit for bit."""
    from paper_2309_10212_b200 import debug

    g = debug.pass_buffers(sess)
    o = os_.pass_buffers()
    tag = f"pass {n_pass}"
    assert g["slots_used"] == o["slots_used"], f"{tag} slots used"
    for k in ("block_slots", "ray_slots"):
        assert np.array_equal(g[k], o[k]), f"{tag} {k} (traverse_to_next_blocks)"
    used_rays = o["active_offsets"]
    assert np.array_equal(g["active_offsets"], used_rays), f"{tag} active offsets (O_Act)"
    assert np.array_equal(g["visible_ids"], o["visible_ids"]), f"{tag} visible ids (mark_blocks)"
    assert np.array_equal(g["active_ids"], o["active_ids"]), f"{tag} active ids (mark_blocks)"
    rt = g["rt"]
    assert rt.n_entries == o["n_entries"], f"{tag} n_entries"
    if grouped:
        assert np.array_equal(rt.rays_per_block, o["rays_per_block"]), f"{tag} rays_per_block"
        assert np.array_equal(rt.block_ray_offsets, o["block_ray_offsets"]), f"{tag} block_ray_offsets"
        assert np.array_equal(rt.sorted_ray_ids, o["sorted_ray_ids"]), f"{tag} sorted_ray_ids"
        assert np.array_equal(rt.sorted_hit_slots, o["sorted_hit_slots"]), f"{tag} sorted_hit_slots"
    else:  # ray-ordered entries: entry k is the k-th valid slot (engine.py:124-128)
        valid = o["block_slots"] != UINT_MAX
        assert np.array_equal(rt.sorted_hit_slots, np.arange(rt.n_entries, dtype=np.uint32)), f"{tag} entry order"
        assert np.array_equal(rt.sorted_ray_ids, o["ray_slots"][valid]), f"{tag} entry rays"
    assert np.array_equal(rt.valid_prefix, o["valid_prefix"]), f"{tag} valid_prefix"
    assert np.array_equal(g["rgbz_z"].view(np.uint32), o["rgbz_z"].view(np.uint32)), f"{tag} rgbz z"
    assert np.array_equal(g["rgbz_rgb"].view(np.uint32), o["rgbz_rgb"].view(np.uint32)), f"{tag} rgbz rgb"
    gc = debug.cache_state(sess, with_values=with_values)
    bos, lu, sv = os_.cache_state(with_values=with_values)
    phys = gc["physical"]
    assert gc["capacity"] == len(bos), f"{tag} cache capacity"
    assert np.array_equal(gc["block_of_slot"].astype(np.int64), bos[:phys]), f"{tag} block_of_slot"
    assert (bos[phys:] == -1).all(), f"{tag} slots beyond the physical pool must be free"
    assert np.array_equal(gc["last_used"].astype(np.int64), lu[:phys]), f"{tag} last_used"
    if with_values:  # occupied slots only: a free slot's contents are never read
        occ = gc["block_of_slot"] >= 0
        assert np.array_equal(gc["slot_values"][occ].view(np.uint32), sv[:phys][occ].view(np.uint32)), \
            f"{tag} slot values"
    r = debug.session_rays(sess)
    orr = os_.rays()
    for k in ("status", "exited", "coarse_cell", "fine_cell", "coarse_tmax", "fine_tmax"):
        assert np.array_equal(r[k], orr[k]), f"{tag} ray {k}"
