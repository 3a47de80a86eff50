"""Golden fixtures for the stage-level API, made by running the REFERENCE.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_stage_golden.py

Every expected array comes from the unmodified reference package's own
stage functions (traverse_to_next_blocks, mark_blocks, build_rt_inputs,
composite, BlockCache, assemble_dual_grid, intersect_cell, shade,
raytrace_block).  tests/test_gpu_stages.py replays the same inputs through
paper_2309_10212_b200's device-backed stage functions and compares bit for
bit.  Output: tests/golden/stage_kats.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import wavecast as wc  # noqa: E402
from wavecast import engine, prims  # noqa: E402
from wavecast.blocktrace import _cell_overlap  # noqa: E402
from wavecast.cache import BlockCache  # noqa: E402
from wavecast.traversal import STATUS_ACTIVE, STATUS_MISS, UINT_MAX, RaySoA, traverse_to_next_blocks  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def ragged(name, arrays, out):
    out[f"{name}_flat"] = np.concatenate([np.asarray(a).reshape(-1) for a in arrays]) if arrays else np.zeros(0)
    out[f"{name}_len"] = np.array([np.asarray(a).size for a in arrays], dtype=np.int64)


def traversal_fixture(out):
    """Successive traverse_to_next_blocks calls over 400 random rays of a
    value-noise volume, n_spec varying, exited rays retired between calls."""
    vol = wc.synthesize("value_noise", (40, 36, 44), seed=7)
    cv = wc.compress_volume(vol, 12)
    grids = wc.build_grids(cv)
    rng = np.random.default_rng(11)
    n = 400
    c = np.array([(d - 1) / 2 for d in cv.dims])
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    o = c + 80.0 * u
    o[:40] = c + rng.uniform(-15, 15, (40, 3))  # some rays start inside the volume
    tgt = c + rng.uniform(-18, 18, (n, 3))
    d = tgt - o
    d[5] = [1.0, 0.0, 0.0]  # axis-aligned rays (zero direction components)
    d[6] = [0.0, -1.0, 0.0]
    d[7] = [0.0, 0.7, -0.7]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rays = RaySoA.from_rays(o, d, cv.dims)
    lo, hi = float(cv.raw_block_ranges[:, 0].min()), float(cv.raw_block_ranges[:, 1].max())
    iso = lo + 0.47 * (hi - lo)
    out["trav_dims"] = np.array(cv.dims)
    out["trav_origin"] = o
    out["trav_dir"] = d
    out["trav_iso"] = np.array([iso])
    for k in ("fine_min", "fine_max", "coarse_min", "coarse_max"):
        out[f"trav_{k}"] = getattr(grids, k)
    out["trav_init_status"] = rays.status.copy()
    retired = (np.arange(n) % 3 != 0) & (rays.status == STATUS_ACTIVE)  # free slots for speculation
    rays.status[retired] = STATUS_MISS
    out["trav_init_exited"] = rays.exited.copy()
    out["trav_init_coarse_cell"] = rays.coarse_cell.copy()
    out["trav_init_fine_cell"] = rays.fine_cell.copy()
    out["trav_init_coarse_tmax"] = rays.coarse_tmax.copy()
    out["trav_init_fine_tmax"] = rays.fine_tmax.copy()
    out["trav_init_t_exit"] = rays.t_exit.copy()
    specs, status, fields = [], [], {k: [] for k in ("block_slots", "ray_slots", "exited", "coarse_cell",
                                                   "fine_cell", "coarse_tmax", "fine_tmax")}
    want = [1, 3, 8, 2, 5, 1, 16, 4, 64, 2, 7, 3, 1, 9, 2, 6]
    for step in range(40):
        n_act = rays.n_active
        if n_act == 0:
            break
        spec = max(1, min(want[step % len(want)], n // n_act))
        offs, _ = prims.exclusive_scan(rays.active_mask.astype(np.uint32))
        status.append(rays.status.copy())
        traverse_to_next_blocks(rays, grids, iso, spec, offs)
        specs.append(spec)
        for k in fields:
            fields[k].append(getattr(rays, k).copy())
        # retire rays that ran out of volume, and a few random ones (as hits)
        rays.status[(rays.exited == 1) & (rays.status == STATUS_ACTIVE)] = STATUS_MISS
        kill = rng.random(n) < 0.12
        rays.status[kill & (rays.status == STATUS_ACTIVE)] = 1
    out["trav_specs"] = np.array(specs)
    out["trav_status"] = np.stack(status)
    for k, v in fields.items():
        out[f"trav_{k}"] = np.stack(v)


def mark_fixture(out):
    rng = np.random.default_rng(5)
    cases = [(4, 4, 4), (5, 3, 7), (32, 3, 2), (64, 2, 3), (1, 1, 1), (7, 1, 9)]
    slots, dims, vis, act = [], [], [], []
    for bd in cases:
        nb = bd[0] * bd[1] * bd[2]
        for k in (0, 1, 6, 40):
            s = rng.integers(0, nb, k + 3).astype(np.uint32)
            s[rng.random(len(s)) < 0.3] = UINT_MAX
            v, a = engine.mark_blocks(s, bd)
            slots.append(s)
            dims.append(bd)
            vis.append(v)
            act.append(a)
    ragged("mark_slots", slots, out)
    out["mark_dims"] = np.array(dims)
    ragged("mark_vis", vis, out)
    ragged("mark_act", act, out)


def grouping_fixture(out):
    rng = np.random.default_rng(67)
    res = {k: [] for k in ("slots", "rays", "vis_mask", "visible_ids", "rays_per_block", "block_ray_offsets",
                           "sorted_ray_ids", "sorted_hit_slots", "valid_prefix")}
    n_ent = []
    cases = []
    for _ in range(25):
        n_blocks = int(rng.choice([8, 64, 300, 4096]))
        n = int(rng.integers(1, 400))
        s = rng.integers(0, n_blocks, n).astype(np.uint32)
        s[rng.random(n) < 0.4] = UINT_MAX
        r = rng.integers(0, 100000, n).astype(np.uint32)
        vis = np.zeros(n_blocks, bool)
        vis[s[s != UINT_MAX]] = True
        cases.append((s, r, vis))
    s = np.array([5, 2, 5, UINT_MAX], dtype=np.uint32)  # engine worked example (test_engine.py:54-65)
    cases.append((s, np.array([0, 1, 2, 0], np.uint32), engine.mark_blocks(s, (2, 2, 2))[0]))
    s = np.full(6, UINT_MAX, dtype=np.uint32)  # empty
    cases.append((s, np.zeros(6, np.uint32), np.zeros(8, bool)))
    for s, r, vis in cases:
        pb = engine.build_rt_inputs(s, r, vis)
        res["slots"].append(s)
        res["rays"].append(r)
        res["vis_mask"].append(vis)
        for k in ("visible_ids", "rays_per_block", "block_ray_offsets", "sorted_ray_ids", "sorted_hit_slots",
                  "valid_prefix"):
            res[k].append(getattr(pb, k))
        n_ent.append(pb.n_entries)
    for k, v in res.items():
        ragged(f"grp_{k}", v, out)
    out["grp_n_entries"] = np.array(n_ent)


def composite_fixture(out):
    rng = np.random.default_rng(31)
    recs = {k: [] for k in ("status_in", "exited", "slots", "z", "rgb", "status_out", "rgba", "depth")}
    specs = []
    for case in range(12):
        n = int(rng.integers(4, 120))
        rays = RaySoA(n, n, 1)
        rays.status[:] = rng.choice([0, 0, 0, 1, 2], n).astype(np.uint8)
        rays.exited[:] = (rng.random(n) < 0.3).astype(np.uint8)
        n_act = rays.n_active
        spec = int(max(1, min(rng.integers(1, 6), n // max(1, n_act))))
        rays.block_slots[:] = UINT_MAX
        offs, _ = prims.exclusive_scan(rays.active_mask.astype(np.uint32))
        used = n_act * spec
        valid = rng.random(used) < 0.6
        rays.block_slots[:used][valid] = rng.integers(0, 50, int(valid.sum())).astype(np.uint32)
        vp, n_valid = prims.exclusive_scan((rays.block_slots != UINT_MAX).astype(np.uint32))
        z = np.full(n, np.inf, np.float32)
        zz = rng.uniform(1, 9, n_valid).astype(np.float32)
        zz[rng.random(n_valid) < 0.3] = np.inf
        if n_valid > 2:
            zz[1] = zz[0]  # ties: the earliest slot wins
        z[:n_valid] = zz
        rgb = rng.uniform(-0.2, 1.2, (n, 3)).astype(np.float32)
        fb = engine.Framebuffer.blank(n, 1)
        recs["status_in"].append(rays.status.copy())
        recs["exited"].append(rays.exited.copy())
        recs["slots"].append(rays.block_slots.copy())
        recs["z"].append(z)
        recs["rgb"].append(rgb)
        engine.composite(rgb, z, rays, spec, offs, vp, fb)
        recs["status_out"].append(rays.status.copy())
        recs["rgba"].append(fb.rgba.reshape(-1))
        recs["depth"].append(fb.depth.reshape(-1))
        specs.append(spec)
    for k, v in recs.items():
        ragged(f"comp_{k}", v, out)
    out["comp_specs"] = np.array(specs)


def cache_fixture(out):
    """BlockCache traces with growth: capacity 4 and 16 over 120 passes each,
    with every slot's block / stamp and the slot values after each pass."""
    vol = wc.synthesize("value_noise", (16, 16, 16), seed=5)
    cv = wc.compress_volume(vol, 12)
    out["cache_payload_dims"] = np.array(cv.dims)
    for cap in (4, 16):
        rng = np.random.default_rng(100 + cap)
        cache = BlockCache(cap)
        act, stats, bos, lu = [], [], [], []
        for step in range(120):
            k = int(rng.integers(0, 30)) if step % 17 else 40
            ids = np.sort(rng.choice(cv.block_count, size=min(k, cv.block_count), replace=False))
            m = np.zeros(cv.block_count, bool)
            m[ids] = True
            s = cache.ensure_resident(m, cv)
            act.append(ids)
            stats.append([s.new_decompressed, s.evicted, s.grown_to])
            bos.append(cache.block_of_slot.copy())
            lu.append(cache.last_used_pass.copy())
        ragged(f"cache{cap}_active", act, out)
        out[f"cache{cap}_stats"] = np.array(stats)
        ragged(f"cache{cap}_block_of_slot", bos, out)
        ragged(f"cache{cap}_last_used", lu, out)
        out[f"cache{cap}_final_values"] = cache.slot_values
        out[f"cache{cap}_lookup"] = np.array([-1 if cache.lookup(b) is None else cache.lookup(b)
                                              for b in range(cv.block_count)])


def blocktrace_fixture(out):
    # dual grids of every block of a ragged volume (boundary clamps)
    vol = wc.synthesize("value_noise", (12, 9, 10), seed=19)
    cv = wc.compress_volume(vol, 10)
    cache = BlockCache(cv.block_count)
    cache.ensure_resident(np.ones(cv.block_count, bool), cv)
    out["dual_vals"] = np.stack([wc.assemble_dual_grid(cache, cv, b).values for b in range(cv.block_count)])
    out["dual_cells"] = np.array([wc.assemble_dual_grid(cache, cv, b).cells_per_axis for b in range(cv.block_count)])
    # intersect_cell over random cells / rays, various isovalues
    rng = np.random.default_rng(123)
    n = 600
    c = rng.uniform(-1, 1, (n, 8)).astype(np.float32)
    o = rng.uniform(-0.5, 1.5, (n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d[:20, 0] = 0.0  # rays parallel to a face
    d[:20] /= np.linalg.norm(d[:20], axis=1, keepdims=True)
    iso = rng.uniform(-0.4, 0.4, n)
    t01 = np.array([_cell_overlap(*o[i], *d[i], 0.0, 0.0, 0.0) for i in range(n)])
    t = np.array([np.inf if (t01[i, 0] > t01[i, 1]) else
                  (lambda r: np.inf if r is None else r)(wc.intersect_cell(c[i], o[i], d[i], (0, 0, 0), t01[i, 0],
                                                                           t01[i, 1], iso[i]))
                  for i in range(n)])
    out.update(isec_corners=c, isec_o=o, isec_d=d, isec_iso=iso, isec_t01=t01, isec_t=t)
    # shade
    g = rng.normal(size=(200, 3))
    g[:5] = 0.0
    dd = rng.normal(size=(200, 3))
    dd /= np.linalg.norm(dd, axis=1, keepdims=True)
    base = (0.7, 0.5, 0.25)
    out.update(shade_grad=g, shade_dir=dd, shade_base=np.array(base),
               shade_rgb=np.array([wc.shade(g[i], dd[i], base) for i in range(200)]))
    # raytrace_block: sphere, rays through a front block at random offsets
    vol = wc.synthesize("sphere", (64, 64, 64))
    cvs = wc.compress_volume(vol, 16)
    bx, by, bz = 7, 7, 12
    b = cvs.block_id(bx, by, bz)
    needed = [cvs.block_id(bx + ox, by + oy, bz + oz) for ox in (0, 1) for oy in (0, 1) for oz in (0, 1)]
    cs = BlockCache(64)
    m = np.zeros(cvs.block_count, bool)
    m[needed] = True
    cs.ensure_resident(m, cvs)
    dg = wc.assemble_dual_grid(cs, cvs, b)
    nr = 256
    oo = np.column_stack([rng.uniform(28, 33, nr), rng.uniform(28, 33, nr), np.full(nr, 120.0)])
    tg = np.column_stack([rng.uniform(28, 33, nr), rng.uniform(28, 33, nr), np.full(nr, 48.0)])
    dv = tg - oo
    dv /= np.linalg.norm(dv, axis=1, keepdims=True)
    rays = RaySoA.from_rays(oo, dv, cvs.dims)
    ids = np.arange(nr)[::-1].copy()
    slots = rng.permutation(nr)
    rgb = np.zeros((nr, 3), np.float32)
    z = np.full(nr, np.inf, np.float32)
    wc.raytrace_block(dg, ids, rays, 20.0, rgb, z, slots, (0.85, 0.6, 0.4))
    out.update(rtb_o=oo, rtb_d=dv, rtb_ids=ids, rtb_slots=slots, rtb_rgb=rgb, rtb_z=z, rtb_block=np.array([b]),
               rtb_values=dg.values)


def main():
    out = {}
    traversal_fixture(out)
    mark_fixture(out)
    grouping_fixture(out)
    composite_fixture(out)
    cache_fixture(out)
    blocktrace_fixture(out)
    path = os.path.join(HERE, "stage_kats.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
