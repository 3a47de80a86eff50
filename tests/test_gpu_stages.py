"""The reference's stage-level API (wavecast/__init__.py:3-56) on the device.

Each stage function of paper_2309_10212_b200 runs the render path's device
code through the C ABI; these tests drive them the way the reference's own
unit tests drive wavecast (tests/test_traversal.py, test_cache.py,
test_engine.py, test_blocktrace.py) and compare, bit for bit, with fixtures
made by running the reference (tests/golden/make_stage_golden.py).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

UINT_MAX = 0xFFFFFFFF


@pytest.fixture(scope="module")
def wc():
    import paper_2309_10212_b200 as wc

    wc._lib.ensure_device(0)
    return wc


@pytest.fixture(scope="module")
def G():
    import os

    return np.load(os.path.join(os.path.dirname(__file__), "golden", "stage_kats.npz"))


def ragged(G, name):
    flat, lens = G[f"{name}_flat"], G[f"{name}_len"]
    offs = np.concatenate([[0], np.cumsum(lens)])
    return [flat[offs[i]:offs[i + 1]] for i in range(len(lens))]


def vol_from(wc, values_zyx):
    v = np.asarray(values_zyx, dtype=np.float32)
    nz, ny, nx = v.shape
    return wc.Volume((nx, ny, nz), v.reshape(-1), (float(v.min()), float(v.max())))


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64 if a.dtype == np.float64 else np.uint32)


# ------------------------------------------------------------ traversal
@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("grid_src", ["volume", "arrays"])
def test_traverse_matches_reference_sequence(wc, G, variant, grid_src):
    """traversal.py:406-452: successive calls with varying n_spec over random
    rays (inside / outside / axis-aligned); slots, exit flags and the saved
    iterators equal the reference's after every call."""
    dims = tuple(int(x) for x in G["trav_dims"])
    cv = wc.compress_volume(wc.synthesize("value_noise", dims, seed=7), 12)
    if grid_src == "volume":
        grids = wc.build_grids(cv)
    else:  # caller-supplied MacrocellGrids arrays (the reference's grids)
        fd = cv.block_dims
        grids = wc.MacrocellGrids(fd, G["trav_fine_min"], G["trav_fine_max"], None, G["trav_coarse_min"],
                                  G["trav_coarse_max"])
    for k in ("fine_min", "fine_max", "coarse_min", "coarse_max"):
        assert np.array_equal(bits(getattr(grids, k)), bits(G[f"trav_{k}"])), k
    rays = wc.RaySoA.from_rays(G["trav_origin"], G["trav_dir"], cv.dims)
    for k in ("status", "exited", "coarse_cell", "fine_cell", "coarse_tmax", "fine_tmax", "t_exit"):
        assert np.array_equal(bits(getattr(rays, k)) if getattr(rays, k).dtype.kind == "f" else getattr(rays, k),
                              bits(G[f"trav_init_{k}"]) if G[f"trav_init_{k}"].dtype.kind == "f"
                              else G[f"trav_init_{k}"]), f"from_rays {k}"
    iso = float(G["trav_iso"][0])
    specs = G["trav_specs"]
    assert len(specs) >= 6
    for step, spec in enumerate(specs):
        rays.status[:] = G["trav_status"][step]
        offs, _ = wc.prims.exclusive_scan(rays.active_mask.astype(np.uint32))
        wc.traverse_to_next_blocks(rays, grids, iso, int(spec), offs, variant=variant)
        for k in ("block_slots", "ray_slots", "exited", "coarse_cell", "fine_cell"):
            assert np.array_equal(getattr(rays, k), G[f"trav_{k}"][step]), f"call {step} {k}"
        for k in ("coarse_tmax", "fine_tmax"):
            assert np.array_equal(bits(getattr(rays, k)), bits(G[f"trav_{k}"][step])), f"call {step} {k}"


def _bump(wc, xs):
    v = np.zeros((8, 8, 8), np.float32)
    for x in xs:
        v[0, 0, x] = 10.0
    return wc.compress_volume(vol_from(wc, v), 16)


@pytest.mark.parametrize("variant", [1, 2])
def test_traverse_single_candidate_then_exit(wc, variant):
    cv = _bump(wc, [0])
    grids = wc.build_grids(cv)
    rays = wc.RaySoA.from_rays(np.array([[-5.0, 1.0, 1.0]]), np.array([[1.0, 0.0, 0.0]]), cv.dims)
    offs, _ = wc.prims.exclusive_scan(rays.active_mask.astype(np.uint32))
    wc.traverse_to_next_blocks(rays, grids, 5.0, 1, offs, variant=variant)
    assert rays.block_slots[0] == 0 and rays.ray_slots[0] == 0 and rays.exited[0] == 0
    wc.traverse_to_next_blocks(rays, grids, 5.0, 1, offs, variant=variant)
    assert rays.block_slots[0] == UINT_MAX and rays.exited[0] == 1


def test_traverse_iso_outside_range_and_partial_fill(wc):
    cv = _bump(wc, [0])
    grids = wc.build_grids(cv)
    cam = wc.Camera.look_at((3.5, 3.5, 30.0), (3.5, 3.5, 3.5))
    rays = wc.init_rays(cam, 8, 8, cv.dims)
    offs, _ = wc.prims.exclusive_scan(rays.active_mask.astype(np.uint32))
    wc.traverse_to_next_blocks(rays, grids, 99.0, 2, offs)
    assert (rays.block_slots == UINT_MAX).all()
    assert (rays.exited[rays.status == 0] == 1).all()

    cv = _bump(wc, [0, 4])
    grids = wc.build_grids(cv)
    o = np.repeat([[-5.0, 1.0, 1.0]], 3, axis=0)
    d = np.repeat([[1.0, 0.0, 0.0]], 3, axis=0)
    rays = wc.RaySoA.from_rays(o, d, cv.dims)
    rays.status[1:] = 2  # only ray 0 active; the others' slots are free
    offs, _ = wc.prims.exclusive_scan(rays.active_mask.astype(np.uint32))
    wc.traverse_to_next_blocks(rays, grids, 5.0, 3, offs)
    assert [int(b) for b in rays.block_slots] == [cv.block_id(0, 0, 0), cv.block_id(1, 0, 0), UINT_MAX]
    assert rays.exited[0] == 1


def test_terminated_rays_never_write_and_budget(wc):
    cv = _bump(wc, [0])
    grids = wc.build_grids(cv)
    o = np.array([[-5.0, 1.0, 1.0], [-5.0, 1.0, 1.0]])
    d = np.array([[1.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    rays = wc.RaySoA.from_rays(o, d, cv.dims)
    rays.status[0] = 2
    offs, _ = wc.prims.exclusive_scan(rays.active_mask.astype(np.uint32))
    before = (rays.coarse_cell[0], rays.fine_cell[0], rays.exited[0])
    wc.traverse_to_next_blocks(rays, grids, 5.0, 2, offs)
    assert (rays.coarse_cell[0], rays.fine_cell[0], rays.exited[0]) == before
    assert list(rays.ray_slots) == [1, UINT_MAX]
    rays.status[:] = 0
    offs, _ = wc.prims.exclusive_scan(rays.active_mask.astype(np.uint32))
    with pytest.raises(AssertionError, match="slot budget"):
        wc.traverse_to_next_blocks(rays, grids, 5.0, 2, offs)


# ------------------------------------------------------------ marking / grouping / composite
def test_mark_blocks_matches_reference(wc, G):
    slots, vis, act = ragged(G, "mark_slots"), ragged(G, "mark_vis"), ragged(G, "mark_act")
    for i, bd in enumerate(G["mark_dims"]):
        v, a = wc.mark_blocks(slots[i].astype(np.uint32), tuple(int(x) for x in bd))
        assert np.array_equal(v, vis[i].astype(bool)), f"case {i} visible"
        assert np.array_equal(a, act[i].astype(bool)), f"case {i} active"


def test_mark_blocks_interior_and_corner(wc):
    bd = (4, 4, 4)
    s = np.full(16, UINT_MAX, np.uint32)
    s[3] = 1 + 4 * (1 + 4 * 1)
    v, a = wc.mark_blocks(s, bd)
    assert v.sum() == 1 and a.sum() == 8 and a[2 + 4 * (2 + 4 * 2)]
    s = np.full(16, UINT_MAX, np.uint32)
    s[0] = 3 + 4 * (3 + 4 * 3)
    v, a = wc.mark_blocks(s, bd)
    assert v.sum() == 1 and a.sum() == 1
    v, a = wc.mark_blocks(np.full(16, UINT_MAX, np.uint32), bd)
    assert v.sum() == 0 and a.sum() == 0


def test_build_rt_inputs_matches_reference(wc, G):
    cols = {k: ragged(G, f"grp_{k}") for k in ("slots", "rays", "vis_mask", "visible_ids", "rays_per_block",
                                                "block_ray_offsets", "sorted_ray_ids", "sorted_hit_slots",
                                                "valid_prefix")}
    for i, ne in enumerate(G["grp_n_entries"]):
        pb = wc.build_rt_inputs(cols["slots"][i].astype(np.uint32), cols["rays"][i].astype(np.uint32),
                                cols["vis_mask"][i].astype(bool))
        assert pb.n_entries == ne, f"case {i}"
        for k in ("visible_ids", "rays_per_block", "block_ray_offsets", "sorted_ray_ids", "sorted_hit_slots",
                  "valid_prefix"):
            got = getattr(pb, k)
            assert got.dtype == np.uint32, k
            assert np.array_equal(got, cols[k][i]), f"case {i} {k}"


def test_build_rt_inputs_worked_example(wc):
    s = np.array([5, 2, 5, UINT_MAX], np.uint32)
    v, _ = wc.mark_blocks(s, (2, 2, 2))
    pb = wc.build_rt_inputs(s, np.array([0, 1, 2, 0], np.uint32), v)
    assert pb.visible_ids.tolist() == [2, 5] and pb.rays_per_block.tolist() == [1, 2]
    assert pb.block_ray_offsets.tolist() == [0, 1]
    assert pb.sorted_ray_ids.tolist() == [1, 0, 2] and pb.sorted_hit_slots.tolist() == [1, 0, 2]
    assert pb.n_entries == 3


def test_composite_matches_reference(wc, G):
    cols = {k: ragged(G, f"comp_{k}") for k in ("status_in", "exited", "slots", "z", "rgb", "status_out", "rgba",
                                                 "depth")}
    for i, spec in enumerate(G["comp_specs"]):
        n = len(cols["status_in"][i])
        rays = wc.RaySoA(n, n, 1)
        rays.status[:] = cols["status_in"][i]
        rays.exited[:] = cols["exited"][i]
        rays.block_slots[:] = cols["slots"][i]
        offs, _ = wc.prims.exclusive_scan(rays.active_mask.astype(np.uint32))
        vp, _ = wc.prims.exclusive_scan((rays.block_slots != UINT_MAX).astype(np.uint32))
        fb = wc.Framebuffer.blank(n, 1)
        wc.composite(cols["rgb"][i].reshape(-1, 3).astype(np.float32), cols["z"][i].astype(np.float32), rays,
                     int(spec), offs, vp, fb)
        assert np.array_equal(rays.status, cols["status_out"][i]), f"case {i} status"
        assert np.array_equal(fb.rgba.reshape(-1), cols["rgba"][i]), f"case {i} rgba"
        assert np.array_equal(bits(fb.depth.reshape(-1)), bits(cols["depth"][i].astype(np.float32))), f"case {i}"
        assert fb.completeness == float(n - rays.n_active) / n


# ------------------------------------------------------------ BlockCache
def _cache_cv(wc):
    return wc.compress_volume(wc.synthesize("value_noise", (16, 16, 16), seed=5), 12)


@pytest.mark.parametrize("cap", [4, 16])
def test_block_cache_trace_matches_reference(wc, G, cap):
    """cache.py:66-111 pass by pass: stats, every slot's block and stamp,
    lookups and the slot values equal the reference BlockCache's."""
    cv = _cache_cv(wc)
    cache = wc.BlockCache(cap)
    act = ragged(G, f"cache{cap}_active")
    bos, lu = ragged(G, f"cache{cap}_block_of_slot"), ragged(G, f"cache{cap}_last_used")
    for step, ids in enumerate(act):
        m = np.zeros(cv.block_count, bool)
        m[ids.astype(np.int64)] = True
        s = cache.ensure_resident(m, cv)
        assert [s.new_decompressed, s.evicted, s.grown_to] == G[f"cache{cap}_stats"][step].tolist(), f"pass {step}"
        assert np.array_equal(cache.block_of_slot, bos[step]), f"pass {step} block_of_slot"
        assert np.array_equal(cache.last_used_pass, lu[step]), f"pass {step} last_used_pass"
        assert cache.current_pass == step + 1
    assert np.array_equal(bits(cache.slot_values), bits(G[f"cache{cap}_final_values"]))
    look = np.array([-1 if cache.lookup(b) is None else cache.lookup(b) for b in range(cv.block_count)])
    assert np.array_equal(look, G[f"cache{cap}_lookup"])


def test_block_cache_200_pass_lru_trace(wc):
    """The 200-pass random trace of test_cache.py:70-85 (tests/golden/lru_trace.npz,
    recorded from the reference): more passes than the device stamp histogram holds."""
    import os

    T = np.load(os.path.join(os.path.dirname(__file__), "golden", "lru_trace.npz"))
    cv = wc.CompressedVolume(tuple(int(x) for x in T["dims"]), int(T["qbits"][0]), payload=T["payload"],
                             raw_block_ranges=np.zeros((int(np.prod([-(-int(d) // 4) for d in T["dims"]])), 2),
                                                       np.float32))
    cache = wc.BlockCache(16)
    offs = np.concatenate([[0], np.cumsum(T["active_len"])])
    soffs = np.concatenate([[0], np.cumsum(T["state_len"])])
    for step in range(200):
        ids = T["active_flat"][offs[step]:offs[step + 1]]
        m = np.zeros(cv.block_count, bool)
        m[ids] = True
        s = cache.ensure_resident(m, cv)
        assert [s.new_decompressed, s.evicted, s.grown_to] == T["stats"][step].tolist(), f"pass {step}"
        st = T["state_flat"][soffs[step]:soffs[step + 1]]
        k = int(np.nonzero(st == -2)[0][0])
        assert np.array_equal(cache.block_of_slot, st[:k]), f"pass {step}"
        assert np.array_equal(cache.last_used_pass, st[k + 1:]), f"pass {step}"
        for b in ids:
            assert cache.lookup(int(b)) is not None
    assert np.array_equal(bits(cache.slot_values), bits(T["final_slot_values"]))


def test_block_cache_lru_kats(wc):
    cv = _cache_cv(wc)

    def mask(ids):
        m = np.zeros(cv.block_count, bool)
        m[list(ids)] = True
        return m

    c = wc.BlockCache(2)
    s1 = c.ensure_resident(mask([0, 1]), cv)
    assert (s1.new_decompressed, s1.evicted) == (2, 0)
    s2 = c.ensure_resident(mask([1, 2]), cv)
    assert (s2.new_decompressed, s2.evicted) == (1, 1)
    assert c.lookup(0) is None and c.lookup(1) is not None and c.lookup(2) is not None
    c = wc.BlockCache(8)
    c.ensure_resident(mask([3, 4, 5]), cv)
    s = c.ensure_resident(mask([3, 4, 5]), cv)
    assert (s.new_decompressed, s.evicted) == (0, 0)
    c = wc.BlockCache(4)
    s = c.ensure_resident(mask(range(5)), cv)
    assert s.grown_to == 8 and s.new_decompressed == 5
    c = wc.BlockCache(4)
    assert c.lookup(7) is None and c.current_pass == 0
    c.ensure_resident(mask([7]), cv)
    assert c.lookup(7) == c.lookup(7) and c.lookup(8) is None and c.current_pass == 1
    c = wc.BlockCache(8)
    c.ensure_resident(mask([2, 9, 33]), cv)
    for b in (2, 9, 33):
        assert np.array_equal(c.slot_values[c.lookup(b)], wc.decompress_block(cv, b))
    assert wc.cache.initial_capacity(64, 64) == 1024
    assert wc.cache.initial_capacity(1280, 720) == 2 * (1280 * 720) // 64


# ------------------------------------------------------------ blocktrace
def test_assemble_dual_grid_matches_reference(wc, G):
    cv = wc.compress_volume(wc.synthesize("value_noise", (12, 9, 10), seed=19), 10)
    cache = wc.BlockCache(cv.block_count)
    cache.ensure_resident(np.ones(cv.block_count, bool), cv)
    for b in range(cv.block_count):
        dg = wc.assemble_dual_grid(cache, cv, b)
        assert np.array_equal(bits(dg.values), bits(G["dual_vals"][b])), f"block {b}"
        assert dg.cells_per_axis == tuple(int(x) for x in G["dual_cells"][b])
        assert dg.block_origin == tuple(4 * c for c in cv.block_coords(b))
    part = wc.BlockCache(8)
    part.ensure_resident(np.eye(1, cv.block_count, 0, dtype=bool)[0], cv)
    with pytest.raises(AssertionError, match="not resident"):
        wc.assemble_dual_grid(part, cv, 0)


def test_intersect_cell_matches_reference(wc, G):
    t01 = G["isec_t01"]
    ok = t01[:, 0] <= t01[:, 1]
    got = np.array([wc.blocktrace.intersect_cells(G["isec_corners"][i], G["isec_o"][i], G["isec_d"][i],
                                                  [0.0, 0.0, 0.0], t01[i, 0], t01[i, 1], G["isec_iso"][i])[0]
                    for i in np.nonzero(ok)[0]])
    assert np.array_equal(bits(got), bits(G["isec_t"][ok]))
    t0, t1 = wc.blocktrace.cell_overlaps(G["isec_o"], G["isec_d"], np.zeros((len(t01), 3)))
    assert np.array_equal(bits(t0), bits(t01[:, 0])) and np.array_equal(bits(t1), bits(t01[:, 1]))


def test_intersect_cell_kats(wc):
    corners = np.array([-1, 1, -1, 1, -1, 1, -1, 1], dtype=np.float32)
    assert wc.intersect_cell(corners, (0.0, 0.5, 0.5), (1.0, 0.0, 0.0), (0, 0, 0), 0.0, 1.0, 0.0) == 0.5
    assert wc.intersect_cell(np.full(8, 5.0, np.float32), (0, 0.5, 0.5), (1, 0, 0), (0, 0, 0), 0.0, 1.0, 3.0) is None
    inv = 1.0 / math.sqrt(3.0)
    t0, t1 = wc.blocktrace._cell_overlap(-0.1 * inv, -0.1 * inv, -0.1 * inv, inv, inv, inv, 0.0, 0.0, 0.0)
    assert t0 < t1


def test_shade_matches_reference(wc, G):
    base = tuple(G["shade_base"])
    for i in range(len(G["shade_grad"])):
        got = wc.shade(G["shade_grad"][i], G["shade_dir"][i], base)
        assert np.array_equal(bits(np.array(got)), bits(G["shade_rgb"][i])), i
    b = (0.85, 0.85, 0.85)
    assert wc.shade((0, 0, 1), (0, 0, -1), b) == pytest.approx(b, abs=1e-12)
    assert wc.shade((0, 0, 1), (0, 0, 1), b) == pytest.approx(b, abs=1e-12)
    assert wc.shade((1, 0, 0), (0, 0, -1), b) == pytest.approx(tuple(0.2 * c for c in b), abs=1e-12)
    assert wc.shade((0, 0, 0), (0, 0, -1), b) == pytest.approx(tuple(0.2 * c for c in b), abs=1e-12)


def test_raytrace_block_matches_reference(wc, G):
    cv = wc.compress_volume(wc.synthesize("sphere", (64, 64, 64)), 16)
    bx, by, bz = 7, 7, 12
    b = cv.block_id(bx, by, bz)
    assert b == int(G["rtb_block"][0])
    cache = wc.BlockCache(64)
    m = np.zeros(cv.block_count, bool)
    for ox in (0, 1):
        for oy in (0, 1):
            for oz in (0, 1):
                m[cv.block_id(bx + ox, by + oy, bz + oz)] = True
    cache.ensure_resident(m, cv)
    dg = wc.assemble_dual_grid(cache, cv, b)
    assert np.array_equal(bits(dg.values), bits(G["rtb_values"]))
    rays = wc.RaySoA.from_rays(G["rtb_o"], G["rtb_d"], cv.dims)
    n = len(G["rtb_ids"])
    rgb = np.zeros((n, 3), np.float32)
    z = np.full(n, np.inf, np.float32)
    wc.raytrace_block(dg, G["rtb_ids"], rays, 20.0, rgb, z, G["rtb_slots"], (0.85, 0.6, 0.4))
    assert np.isfinite(z).sum() > n // 2
    assert np.array_equal(bits(z), bits(G["rtb_z"])) and np.array_equal(bits(rgb), bits(G["rtb_rgb"]))
    # a ray that misses the block leaves its slot untouched
    miss = wc.RaySoA.from_rays(np.array([[0.0, 0.0, 120.0]]), np.array([[0.0, 0.0, -1.0]]), cv.dims)
    r1, z1 = np.zeros((1, 3), np.float32), np.full(1, np.inf, np.float32)
    wc.raytrace_block(dg, np.array([0]), miss, 20.0, r1, z1, np.array([0]))
    assert z1[0] == np.inf and not r1.any()
