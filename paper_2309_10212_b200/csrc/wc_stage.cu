// wc_stage.cu -- the reference's lower-level API on the device.
//
// The render session (wc_engine.cu) fuses the per-pass stages into one
// device-driven pipeline.  The reference also exposes each stage on its own
// (wavecast/__init__.py:3-56) and its unit tests drive them one at a time:
//   traverse_to_next_blocks   traversal.py:406-452
//   mark_blocks               engine.py:97-118
//   build_rt_inputs           engine.py:121-149
//   composite                 engine.py:222-283
//   BlockCache                cache.py:21-111
//   assemble_dual_grid, intersect_cell, shade, raytrace_block
//                             blocktrace.py:35-113, 452-530
// Each entry point here takes the reference's host arrays, runs the same
// device code the session runs (the same kernels where the data layout
// allows, the same device functions otherwise) and returns host arrays.
#include <algorithm>
#include <cstring>

#include "wc_engine.cuh"
#include "wc_stage.cuh"
#include "wc_trace.cuh"

namespace wc {

namespace {

template <typename T>
void to_dev(DevBuf<T> &d, const T *h, int64_t n, cudaStream_t st) {
    d.alloc(std::max<int64_t>(1, n));
    if (n > 0) WC_CUDA(cudaMemcpyAsync(d.p, h, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice, st));
}
template <typename T>
void to_host(T *h, const T *d, int64_t n, cudaStream_t st) {
    if (h && n > 0) WC_CUDA(cudaMemcpyAsync(h, d, sizeof(T) * (size_t)n, cudaMemcpyDeviceToHost, st));
}

struct Stream {  // a private stream per stage call
    cudaStream_t st = nullptr;
    Stream() { WC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); }
    ~Stream() {
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }
    void sync() { WC_CUDA(cudaStreamSynchronize(st)); }
};

}  // namespace

// ------------------------------------------------------------- traversal

// per-iso fine range tests laid out for the traversal (bit 16*(fx&3) +
// (fy&3) + 4*(fz&3) of cell_mask[coarse cell]), evaluated exactly in float64
// from the grid itself (traversal.py:297); the session streams a 16-bit
// screening copy instead (k_iso_cell_mask), which needs a volume.
__global__ void k_iso_cell_mask_exact(const double2 *__restrict__ fine_mm, int fdx, int fdy, int fdz, int cdx, int cdy,
                                      double iso, unsigned long long *cell_mask) {
    pdl_wait();
    const int64_t nf = (int64_t)fdx * fdy * fdz;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf; f += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = fine_mm[f];
        if (!(v.x <= iso && iso <= v.y)) continue;
        const int fx = (int)(f % fdx), fy = (int)((f / fdx) % fdy), fz = (int)(f / ((int64_t)fdx * fdy));
        const int64_t c = (fx >> 2) + (int64_t)cdx * ((fy >> 2) + (int64_t)cdy * (fz >> 2));
        atomicOr(cell_mask + c, 1ull << (16 * (fx & 3) + (fy & 3) + 4 * (fz & 3)));
    }
}

// act_list[active_offsets[r]] = r for every active ray (the traversal's
// O_Act; the offsets are a permutation of [0, n_act))
__global__ void k_act_list(const uint8_t *status, const int64_t *offsets, int64_t n, uint32_t *act_list) {
    pdl_wait();
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        if (status[r] == 0) act_list[offsets[r]] = (uint32_t)r;
}

void stage_traverse(const Volume *vol, const double *fine_min, const double *fine_max, const double *coarse_min,
                    const double *coarse_max, const int fd[3], const int cd[3], int64_t n, const double *origin,
                    const double *dir, const double *t_exit, const uint8_t *status, uint8_t *exited,
                    uint32_t *coarse_cell, double *coarse_tmax, uint32_t *fine_cell, double *fine_tmax,
                    uint32_t *block_slots, uint32_t *ray_slots, const int64_t *active_offsets, double iso, int n_spec,
                    int variant) {
    if (n_spec < 1) throw InvariantError("n_spec must be >= 1");  // traversal.py:419
    int64_t n_act = 0;
    for (int64_t r = 0; r < n; r++) n_act += status[r] == 0;
    if (n_act * n_spec > n) throw InvariantError("slot budget exceeded");  // traversal.py:420-422
    {  // the kernels index the active list by offset: it must be a permutation of [0, n_act)
        std::vector<uint8_t> seen((size_t)std::max<int64_t>(1, n_act), 0);
        for (int64_t r = 0; r < n; r++) {
            if (status[r] != 0) continue;
            const int64_t o = active_offsets[r];
            if (o < 0 || o >= n_act || seen[(size_t)o])
                throw UsageError("active_offsets must number the active rays 0..n_active-1 (exclusive scan)");
            seen[(size_t)o] = 1;
        }
    }
    Stream S;
    cudaStream_t st = S.st;
    const int64_t nf = (int64_t)fd[0] * fd[1] * fd[2], nc = (int64_t)cd[0] * cd[1] * cd[2];
    DevBuf<double2> fmm, cmm;
    const double2 *d_fine = nullptr, *d_coarse = nullptr;
    if (vol) {
        if (vol->bdx != fd[0] || vol->bdy != fd[1] || vol->bdz != fd[2]) throw UsageError("grids do not match the volume");
        d_fine = vol->fine_mm.p;
        d_coarse = vol->coarse_mm.p;
    } else {  // caller grids (MacrocellGrids arrays): interleave (min, max) pairs
        std::vector<double2> hf((size_t)nf), hc((size_t)nc);
        for (int64_t i = 0; i < nf; i++) hf[(size_t)i] = make_double2(fine_min[i], fine_max[i]);
        for (int64_t i = 0; i < nc; i++) hc[(size_t)i] = make_double2(coarse_min[i], coarse_max[i]);
        to_dev(fmm, hf.data(), nf, st);
        to_dev(cmm, hc.data(), nc, st);
        d_fine = fmm.p;
        d_coarse = cmm.p;
    }
    DevBuf<uint32_t> coarse_bm, vis_bm, ctl, act_list, emitted, d_cc, d_fc, d_bs, d_rs;
    DevBuf<unsigned long long> cell_mask;
    coarse_bm.alloc(ceil_div(nc, 32));
    cell_mask.alloc(nc);
    WC_CUDA(cudaMemsetAsync(cell_mask.p, 0, 8 * nc, st));
    launch_iso_bitmap(d_coarse, nc, iso, coarse_bm.p, st);
    launch_pdl(k_iso_cell_mask_exact, grid_for(nf, 256), 256, 0, st, d_fine, fd[0], fd[1], fd[2], cd[0], cd[1], iso,
               cell_mask.p);
    WC_LAUNCH_CHECK();

    DevBuf<double> d_o, d_d, d_te, d_ct, d_ft;
    DevBuf<uint8_t> d_st, d_ex;
    DevBuf<int64_t> d_off;
    to_dev(d_o, origin, 3 * n, st);
    to_dev(d_d, dir, 3 * n, st);
    to_dev(d_te, t_exit, n, st);
    to_dev(d_st, status, n, st);
    to_dev(d_ex, exited, n, st);
    to_dev(d_cc, coarse_cell, n, st);
    to_dev(d_fc, fine_cell, n, st);
    to_dev(d_ct, coarse_tmax, 3 * n, st);
    to_dev(d_ft, fine_tmax, 3 * n, st);
    to_dev(d_off, active_offsets, n, st);
    d_bs.alloc(n);
    d_rs.alloc(n);
    WC_CUDA(cudaMemsetAsync(d_bs.p, 0xFF, 4 * n, st));  // traversal.py:423-424
    WC_CUDA(cudaMemsetAsync(d_rs.p, 0xFF, 4 * n, st));
    act_list.alloc(std::max<int64_t>(1, n_act));
    emitted.alloc(std::max<int64_t>(1, n_act));
    launch_pdl(k_act_list, grid_for(n, 256), 256, 0, st, d_st.p, d_off.p, n, act_list.p);
    WC_LAUNCH_CHECK();
    vis_bm.alloc(ceil_div(nf, 32));
    WC_CUDA(cudaMemsetAsync(vis_bm.p, 0, 4 * vis_bm.n, st));
    ctl.alloc(C_COUNT);
    std::vector<uint32_t> h_ctl(C_COUNT, 0u);
    h_ctl[C_NACT] = (uint32_t)n_act;
    h_ctl[C_NSPEC] = (uint32_t)n_spec;
    WC_CUDA(cudaMemcpyAsync(ctl.p, h_ctl.data(), 4 * C_COUNT, cudaMemcpyHostToDevice, st));
    if (n_act > 0) {
        TraverseArgs ta{};
        ta.rays = RayView{d_o.p, d_d.p, nullptr, nullptr};
        ta.t_exit = d_te.p;
        ta.exited = d_ex.p;
        ta.coarse_cell = d_cc.p;
        ta.fine_cell = d_fc.p;
        ta.coarse_tmax = d_ct.p;
        ta.fine_tmax = d_ft.p;
        ta.act_list = act_list.p;
        ta.coarse_bm = coarse_bm.p;
        ta.cell_mask = cell_mask.p;
        ta.fdx = fd[0];
        ta.fdy = fd[1];
        ta.fdz = fd[2];
        ta.cdx = cd[0];
        ta.cdy = cd[1];
        ta.cdz = cd[2];
        ta.iso = iso;
        ta.block_slots = d_bs.p;
        ta.ray_slots = d_rs.p;
        ta.emitted = emitted.p;
        ta.vis_bm = vis_bm.p;
        ta.work = ctl.p + C_WORK;
        ta.ctl = ctl.p;
        launch_traverse(ta, n_act, variant, st);
    }
    to_host(exited, d_ex.p, n, st);
    to_host(coarse_cell, d_cc.p, n, st);
    to_host(fine_cell, d_fc.p, n, st);
    to_host(coarse_tmax, d_ct.p, 3 * n, st);
    to_host(fine_tmax, d_ft.p, 3 * n, st);
    to_host(block_slots, d_bs.p, n, st);
    to_host(ray_slots, d_rs.p, n, st);
    S.sync();
}

// ------------------------------------------------------------- marking

// engine.py:104-106: every valid slot marks its block visible
__global__ void k_mark_slots(const uint32_t *slots, int64_t n, uint32_t *vis_bm) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = slots[i];
        if (b != WC_UINT_MAX) atomicOr(&vis_bm[b >> 5], 1u << (b & 31));
    }
}

void stage_mark_blocks(const uint32_t *slots, int64_t n, int bdx, int bdy, int bdz, uint32_t *vis_words,
                       uint32_t *act_words) {
    const int64_t n_blocks = (int64_t)bdx * bdy * bdz;
    for (int64_t i = 0; i < n; i++)
        if (slots[i] != WC_UINT_MAX && (int64_t)slots[i] >= n_blocks) throw UsageError("block id out of range");
    Stream S;
    cudaStream_t st = S.st;
    const int64_t nwords = ceil_div(n_blocks, 32);
    DevBuf<uint32_t> d_slots, vis_bm, act_bm, ids, partials, cnt;
    to_dev(d_slots, slots, n, st);
    vis_bm.alloc(nwords);
    act_bm.alloc(nwords);
    ids.alloc(n_blocks);
    cnt.alloc(1);
    partials.alloc(scan_scratch_words(nwords));
    WC_CUDA(cudaMemsetAsync(partials.p, 0, 4 * partials.n, st));
    WC_CUDA(cudaMemsetAsync(vis_bm.p, 0, 4 * nwords, st));
    WC_CUDA(cudaMemsetAsync(act_bm.p, 0, 4 * nwords, st));
    if (n > 0) {
        launch_pdl(k_mark_slots, grid_for(n, 256), 256, 0, st, d_slots.p, n, vis_bm.p);
        WC_LAUNCH_CHECK();
    }
    // the session's marking: visible ids from the bitmap, then the +octant
    // dilation (word-parallel when rows are whole words)
    bitmap_extract_dense(vis_bm.p, nwords, nullptr, ids.p, cnt.p, false, partials.p, st);
    launch_mark_active(ids.p, cnt.p, vis_bm.p, bdx, bdy, bdz, n_blocks, act_bm.p, st);
    to_host(vis_words, vis_bm.p, nwords, st);
    to_host(act_words, act_bm.p, nwords, st);
    S.sync();
}

// ------------------------------------------------------------- grouping

struct LoadValid {  // engine.py:124: valid = block_slots != UINT_MAX
    const uint32_t *s;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return s[i] != WC_UINT_MAX; }
};

// engine.py:125-128: compact blocks, rays and entry ids of the valid slots
__global__ void k_entries_from_slots(const uint32_t *block_slots, const uint32_t *ray_slots,
                                     const uint32_t *valid_prefix, int64_t n, uint32_t *blk, uint32_t *ray,
                                     uint32_t *val) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = block_slots[i];
        if (b == WC_UINT_MAX) continue;
        const uint32_t k = valid_prefix[i];
        blk[k] = b;
        ray[k] = ray_slots[i];
        val[k] = k;
    }
}

// sorted_ray_ids[j] = rays[sorted entry j]; rays_per_block = bincount of the
// visible rank of each entry's block (engine.py:130-137)
__global__ void k_group_gather(const uint32_t *sorted_val, const uint32_t *sorted_blk, const uint32_t *ray,
                               const uint32_t *d_n_ent, const uint32_t *vis_bm, const uint32_t *word_pref,
                               uint32_t *sorted_ray, uint32_t *counts) {
    pdl_wait();
    const int64_t n_ent = *d_n_ent;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_ent; j += (int64_t)gridDim.x * blockDim.x) {
        sorted_ray[j] = ray[sorted_val[j]];
        const uint32_t b = sorted_blk[j], w = b >> 5;
        atomicAdd(&counts[word_pref[w] + __popc(vis_bm[w] & ((1u << (b & 31)) - 1u))], 1u);
    }
}

static int bits_for_ids(uint64_t max_value) {
    int b = 0;
    while (b < 64 && (max_value >> b)) b++;
    return b;
}

void stage_build_rt_inputs(const uint32_t *block_slots, const uint32_t *ray_slots, int64_t n,
                           const uint32_t *vis_words, int64_t n_blocks, uint32_t *visible_ids, uint32_t *rays_per_block,
                           uint32_t *block_ray_offsets, uint32_t *sorted_ray_ids, uint32_t *sorted_hit_slots,
                           uint32_t *valid_prefix, int64_t *sizes) {
    Stream S;
    cudaStream_t st = S.st;
    const int64_t nwords = ceil_div(std::max<int64_t>(1, n_blocks), 32);
    uint32_t max_blk = 0;
    for (int64_t i = 0; i < n; i++)
        if (block_slots[i] != WC_UINT_MAX) {
            if ((int64_t)block_slots[i] >= n_blocks) throw UsageError("block id out of range");
            max_blk = std::max(max_blk, block_slots[i]);
        }
    DevBuf<uint32_t> d_bs, d_rs, d_vp, blk, ray, val, vis_bm, vis_ids, word_pref, counts, offs, sorted_ray, partials, tot;
    to_dev(d_bs, block_slots, n, st);
    to_dev(d_rs, ray_slots, n, st);
    to_dev(vis_bm, vis_words, nwords, st);
    const int64_t big = std::max<int64_t>({n, nwords, n_blocks + 1, 1});
    partials.alloc(scan_scratch_words(big));
    WC_CUDA(cudaMemsetAsync(partials.p, 0, 4 * partials.n, st));
    tot.alloc(4);
    d_vp.alloc(n);
    // valid_prefix / n_entries (engine.py:124-125)
    scan_exclusive(LoadValid{d_bs.p}, n, d_vp.p, tot.p, partials.p, st);
    blk.alloc(n);
    ray.alloc(n);
    val.alloc(n);
    if (n > 0) {
        launch_pdl(k_entries_from_slots, grid_for(n, 256), 256, 0, st, d_bs.p, d_rs.p, d_vp.p, n, blk.p, ray.p, val.p);
        WC_LAUNCH_CHECK();
    }
    // visible ids (compact(arange, visible)) and every word's visible rank prefix
    vis_ids.alloc(std::max<int64_t>(1, n_blocks));
    word_pref.alloc(nwords);
    bitmap_extract_dense(vis_bm.p, nwords, nullptr, vis_ids.p, tot.p + 1, false, partials.p, st);
    scan_exclusive(LoadPopc{vis_bm.p}, nwords, word_pref.p, tot.p + 2, partials.p, st);
    uint32_t h_tot[3] = {0, 0, 0};
    to_host(h_tot, tot.p, 3, st);
    S.sync();
    const int64_t n_ent = h_tot[0], n_vis = h_tot[1];
    // stable sort of the entries by block id (prims.py:34-40: sort_by_key)
    RadixScratch rs;
    if (n_ent > 1) radix_sort_pairs(blk.p, val.p, n_ent, bits_for_ids(max_blk), rs, st);
    counts.alloc(n_vis + 1);
    WC_CUDA(cudaMemsetAsync(counts.p, 0, 4 * (n_vis + 1), st));
    sorted_ray.alloc(std::max<int64_t>(1, n_ent));
    if (n_ent > 0) {
        launch_pdl(k_group_gather, grid_for(n_ent, 256), 256, 0, st, val.p, blk.p, ray.p, tot.p, vis_bm.p, word_pref.p,
                   sorted_ray.p, counts.p);
        WC_LAUNCH_CHECK();
    }
    uint32_t tail = 0;  // np.bincount(minlength=n_vis) grows past n_vis only for blocks above the last visible one
    to_host(&tail, counts.p + n_vis, 1, st);
    S.sync();
    const int64_t n_counts = n_vis + (tail ? 1 : 0);
    offs.alloc(std::max<int64_t>(1, n_counts));
    scan_exclusive(LoadU32{counts.p}, n_counts, offs.p, tot.p + 3, partials.p, st);
    uint32_t total = 0;
    to_host(&total, tot.p + 3, 1, st);
    to_host(visible_ids, vis_ids.p, n_vis, st);
    to_host(rays_per_block, counts.p, n_counts, st);
    to_host(block_ray_offsets, offs.p, n_counts, st);
    to_host(sorted_ray_ids, sorted_ray.p, n_ent, st);
    to_host(sorted_hit_slots, val.p, n_ent, st);
    to_host(valid_prefix, d_vp.p, n, st);
    S.sync();
    if ((int64_t)total != n_ent) throw InvariantError("ray-block grouping is inconsistent");  // engine.py:140
    sizes[0] = n_ent;
    sizes[1] = n_vis;
    sizes[2] = n_counts;
}

// ------------------------------------------------------------- composite

// engine.py:222-258 _composite_kernel on the reference's buffers: closest
// speculated hit per active ray (strict <, earliest slot wins), then
// terminate (hit / exited) or keep.
__global__ void k_composite_slots(int64_t n, uint8_t *status, const uint8_t *exited, const int64_t *offsets, int n_spec,
                                  const uint32_t *block_slots, const uint32_t *valid_prefix, const float *rgb,
                                  const float *z, uint8_t *rgba, float *depth) {
    pdl_wait();
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        if (status[r] != 0) continue;
        const int64_t base = offsets[r] * n_spec;
        float best = CUDART_INF_F;
        int64_t best_slot = -1;
        for (int k = 0; k < n_spec; k++) {
            const int64_t s = base + k;
            if (block_slots[s] != WC_UINT_MAX) {
                const int64_t slot = valid_prefix[s];
                const float zz = z[slot];
                if (zz < best) {
                    best = zz;
                    best_slot = slot;
                }
            }
        }
        if (best_slot >= 0) {
            depth[r] = best;
            rgba[4 * r] = (uint8_t)rgb_u8((double)rgb[3 * best_slot]);
            rgba[4 * r + 1] = (uint8_t)rgb_u8((double)rgb[3 * best_slot + 1]);
            rgba[4 * r + 2] = (uint8_t)rgb_u8((double)rgb[3 * best_slot + 2]);
            rgba[4 * r + 3] = 255;
            status[r] = 1;
        } else if (exited[r] == 1) {
            status[r] = 2;
        }
    }
}

void stage_composite(const float *rgb, const float *z, int64_t n_rgbz, int64_t n, uint8_t *status,
                     const uint8_t *exited, const int64_t *offsets, int n_spec, const uint32_t *block_slots,
                     int64_t n_slots, const uint32_t *valid_prefix, uint8_t *rgba, float *depth) {
    for (int64_t r = 0; r < n; r++)  // the slots an active ray reads must exist
        if (status[r] == 0 && (offsets[r] < 0 || (offsets[r] + 1) * (int64_t)n_spec > n_slots))
            throw UsageError("active_offsets * n_spec beyond the slot buffers");
    Stream S;
    cudaStream_t st = S.st;
    DevBuf<float> d_rgb, d_z, d_depth;
    DevBuf<uint8_t> d_st, d_ex, d_rgba;
    DevBuf<int64_t> d_off;
    DevBuf<uint32_t> d_bs, d_vp;
    to_dev(d_rgb, rgb, 3 * n_rgbz, st);
    to_dev(d_z, z, n_rgbz, st);
    to_dev(d_st, status, n, st);
    to_dev(d_ex, exited, n, st);
    to_dev(d_off, offsets, n, st);
    to_dev(d_bs, block_slots, n_slots, st);
    to_dev(d_vp, valid_prefix, n_slots, st);
    to_dev(d_rgba, rgba, 4 * n, st);
    to_dev(d_depth, depth, n, st);
    if (n > 0) {
        launch_pdl(k_composite_slots, grid_for(n, 256), 256, 0, st, n, d_st.p, d_ex.p, d_off.p, n_spec, d_bs.p, d_vp.p,
                   d_rgb.p, d_z.p, d_rgba.p, d_depth.p);
        WC_LAUNCH_CHECK();
    }
    to_host(status, d_st.p, n, st);
    to_host(rgba, d_rgba.p, 4 * n, st);
    to_host(depth, d_depth.p, n, st);
    S.sync();
}

// ------------------------------------------------------------- BlockCache

StageCache::StageCache(int64_t capacity) {
    cap = std::max<int64_t>(1, capacity);  // cache.py:28
    WC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    ctl.alloc(C_COUNT + kHistBins);
    WC_CUDA(cudaMemsetAsync(ctl.p, 0, 4 * ctl.n, st));
    h_ctl.alloc(C_COUNT);
}

StageCache::~StageCache() {
    if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
}

void StageCache::bind(const Volume *v) {
    if (vol) {
        if (v != vol && v->n_blocks != n_blocks) throw UsageError("BlockCache is bound to a volume of another size");
        vol = v;
        return;
    }
    vol = v;
    n_blocks = v->n_blocks;
    const int64_t nwords = ceil_div(n_blocks, 32);
    slot_of_block.alloc(n_blocks);
    WC_CUDA(cudaMemsetAsync(slot_of_block.p, 0xFF, 4 * n_blocks, st));  // cache.py:36-40
    act_bm.alloc(nwords);
    active_ids.alloc(n_blocks + 1);
    miss_ids.alloc(n_blocks + 1);
    partials.alloc(scan_scratch_words(std::max<int64_t>(nwords, n_blocks)));
    WC_CUDA(cudaMemsetAsync(partials.p, 0, 4 * partials.n, st));
    phys = std::min<int64_t>(cap, n_blocks);
    reserve_slots(phys);
    WC_CUDA(cudaMemsetAsync(block_of_slot.p, 0xFF, 4 * phys, st));
    WC_CUDA(cudaMemsetAsync(last_used.p, 0, 4 * phys, st));
    std::vector<uint32_t> h(C_COUNT, 0u);
    h[C_NACT] = 1;  // a pass with work (the slot-stamp recount reads it)
    h[C_CAP] = (uint32_t)cap;
    h[C_PHYS] = h[C_PHYS_OLD] = (uint32_t)phys;
    WC_CUDA(cudaMemcpyAsync(ctl.p, h.data(), 4 * C_COUNT, cudaMemcpyHostToDevice, st));
    WC_CUDA(cudaStreamSynchronize(st));
}

// Physical slots for `need` (contents kept).  The maps of slots a growth
// brings into use are initialised by the update that does it (k_decode_insert).
void StageCache::reserve_slots(int64_t need) {
    reserve_store(need, std::max<int64_t>(ceil_div(n_blocks, 32), n_blocks), partials, st);
}

void StageCache::ensure_resident(const Volume *v, const uint32_t *mask_words, int64_t needed, int64_t *new_decompressed,
                                 int64_t *evicted, int64_t *grown_to) {
    bind(v);
    const int64_t nwords = ceil_div(n_blocks, 32);
    current_pass++;  // cache.py:67
    const int32_t stamp = (int32_t)current_pass;
    // physical slots for the capacity this update can grow to (cache.py:74-75)
    const int64_t cap_after = needed > cap ? (3 * needed + 1) / 2 : cap;
    reserve_slots(std::min<int64_t>(cap_after, n_blocks));
    prepare_regions(stamp, n_blocks, partials, st);
    WC_CUDA(cudaMemcpyAsync(act_bm.p, mask_words, 4 * nwords, cudaMemcpyHostToDevice, st));
    // active ids ascending (np.nonzero), the session's bitmap extraction
    bitmap_extract_dense(act_bm.p, nwords, nullptr, active_ids.p, ctl.p + C_NACTB, true, partials.p, st);
    const int64_t nmax = std::max<int64_t>(1, needed);
    enqueue_lookup(ctl.p, active_ids.p, nmax, stamp, n_blocks, partials.p, st);
    if (stamp >= kHistBins) enqueue_slow_plan(ctl.p, stamp, true, n_blocks, st);
    enqueue_insert(ctl.p, nmax, stamp, vol, partials.p, st);
    WC_CUDA(cudaMemcpyAsync(h_ctl.p, ctl.p, 4 * C_COUNT, cudaMemcpyDeviceToHost, st));
    WC_CUDA(cudaStreamSynchronize(st));
    const uint32_t *c = h_ctl.p;
    if (c[C_ERR_CAND]) throw InvariantError("cache: fewer eviction candidates than needed");
    if (c[C_ERR_CAP]) throw InvariantError("cache: capacity beyond the reserved slots");
    if ((int64_t)c[C_NACTB] != needed) throw InvariantError("cache: active set size mismatch");
    *new_decompressed = c[C_NMISS];
    *evicted = c[C_NEVICT];
    cap = c[C_CAP];
    phys = c[C_PHYS];
    *grown_to = cap;
    // the occupied prefix after this update (the session's pass_end)
    const uint32_t hw_next = c[C_HW_NEXT];
    WC_CUDA(cudaMemcpyAsync(ctl.p + C_HW, &hw_next, 4, cudaMemcpyHostToDevice, st));
    WC_CUDA(cudaStreamSynchronize(st));
}

int64_t StageCache::lookup(int64_t block) {
    if (!vol) return -1;
    if (block < 0 || block >= n_blocks) throw UsageError("block id out of range");
    int32_t s = -1;
    WC_CUDA(cudaMemcpyAsync(&s, slot_of_block.p + block, 4, cudaMemcpyDeviceToHost, st));
    WC_CUDA(cudaStreamSynchronize(st));
    return s;
}

void StageCache::download(float *slot_values_out, int32_t *block_of_slot_out, int32_t *last_used_out,
                          int32_t *slot_of_block_out) {
    if (!vol) return;
    to_host(slot_values_out, slot_values.p, phys * 64, st);
    to_host(block_of_slot_out, block_of_slot.p, phys, st);
    to_host(last_used_out, last_used.p, phys, st);
    to_host(slot_of_block_out, slot_of_block.p, n_blocks, st);
    WC_CUDA(cudaStreamSynchronize(st));
}

// blocktrace.py:49-94 _assemble_dual from the cache (contributor_slots,
// blocktrace.py:97-110): lattice point (x, y, z) of the 5^3 dual grid lives
// in the slot of octant (x>>2, y>>2, z>>2) at offset (x&3)+4(y&3)+16(z&3);
// absent neighbours (outside the volume) leave zeros.
__global__ void k_dual_grid(const float *slot_values, const int32_t *slot_of_block, int bdx, int bdy, int bdz,
                            int64_t block, float *out, uint32_t *err) {
    pdl_wait();
    const int i = threadIdx.x;
    if (i >= 125) return;
    const int x = i % 5, y = (i / 5) % 5, z = i / 25;
    const int bx = (int)(block % bdx), by = (int)((block / bdx) % bdy), bz = (int)(block / ((int64_t)bdx * bdy));
    const int ox = x >> 2, oy = y >> 2, oz = z >> 2;
    float v = 0.0f;
    if (bx + ox < bdx && by + oy < bdy && bz + oz < bdz) {
        const int32_t s = slot_of_block[(bx + ox) + (int64_t)bdx * ((by + oy) + (int64_t)bdy * (bz + oz))];
        if (s < 0)
            atomicAdd(err, 1u);  // "required neighbor block not resident" (blocktrace.py:107)
        else
            v = slot_values[(int64_t)s * 64 + (x & 3) + 4 * (y & 3) + 16 * (z & 3)];
    }
    out[i] = v;  // [z][y][x]
}

void StageCache::dual_grid(int64_t block, float *values125) {
    if (!vol) throw InvariantError("required neighbor block not resident");
    if (block < 0 || block >= n_blocks) throw UsageError("block id out of range");
    DevBuf<float> out;
    DevBuf<uint32_t> err;
    out.alloc(125);
    err.alloc(1);
    WC_CUDA(cudaMemsetAsync(err.p, 0, 4, st));
    launch_pdl(k_dual_grid, 1, 128, 0, st, slot_values.p, slot_of_block.p, vol->bdx, vol->bdy, vol->bdz, block, out.p,
               err.p);
    WC_LAUNCH_CHECK();
    uint32_t e = 0;
    to_host(values125, out.p, 125, st);
    to_host(&e, err.p, 1, st);
    WC_CUDA(cudaStreamSynchronize(st));
    if (e) throw InvariantError("required neighbor block not resident");
}

// ------------------------------------------------------------- blocktrace

__global__ void k_intersect_cells(int64_t n, const float *corners, const double *o, const double *d,
                                  const double *cell, const double *t0, const double *t1, double iso, double *t_out) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float c[8];
#pragma unroll
        for (int k = 0; k < 8; k++) c[k] = corners[8 * i + k];
        const double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]}, dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
        const double cc[3] = {cell[3 * i], cell[3 * i + 1], cell[3 * i + 2]};
        t_out[i] = intersect_cubic(c, oo, dd, cc, t0[i], t1[i], iso);  // blocktrace.py:236-280
    }
}

__global__ void k_cell_overlaps(int64_t n, const double *o, const double *d, const double *cell, double *t0,
                                double *t1) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]}, dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
        const double cc[3] = {cell[3 * i], cell[3 * i + 1], cell[3 * i + 2]};
        const Recip rd[3] = {recip_of(dd[0]), recip_of(dd[1]), recip_of(dd[2])};
        cell_overlap(oo, dd, rd, cc, t0[i], t1[i]);  // blocktrace.py:126-158
    }
}

__global__ void k_shade(int64_t n, const double *grad, const double *dir, double br, double bg, double bb,
                        double *rgb) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double dd[3] = {dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]};
        shade_grad(grad[3 * i], grad[3 * i + 1], grad[3 * i + 2], dd, br, bg, bb, rgb + 3 * i);  // blocktrace.py:306-314
    }
}

struct DualGridField {  // a block's 5^3 dual grid, [z][y][x] (DualGrid.values)
    const float *v;
    __device__ __forceinline__ float point(int x, int y, int z) const { return v[x + 5 * y + 25 * z]; }
    __device__ __forceinline__ void corners(int lx, int ly, int lz, float c[8]) const {
#pragma unroll
        for (int idx = 0; idx < 8; idx++) c[idx] = point(lx + (idx & 1), ly + ((idx >> 1) & 1), lz + (idx >> 2));
    }
};

// blocktrace.py:491-530 raytrace_block: each ray traces the block's dual
// cells (_trace_region, blocktrace.py:317-449); hit -> (rgb, z) at its slot
__global__ void k_raytrace_block(const float *values125, int ox, int oy, int oz, int ncx, int ncy, int ncz, int64_t n,
                                 const double *o, const double *d, const double *t_enter, double iso, double br,
                                 double bg, double bb, float *rgb, float *z, uint8_t *hit) {
    pdl_wait();
    __shared__ float sv[125];
    for (int i = threadIdx.x; i < 125; i += blockDim.x) sv[i] = values125[i];
    __syncthreads();
    const DualGridField f{sv};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double oo[3] = {o[3 * i], o[3 * i + 1], o[3 * i + 2]}, dd[3] = {d[3 * i], d[3 * i + 1], d[3 * i + 2]};
        float c[3];
        const double t = trace_region(f, ox, oy, oz, ox, oy, oz, ncx, ncy, ncz, oo, dd, t_enter[i], iso, br, bg, bb, c);
        hit[i] = t != CUDART_INF;
        if (t != CUDART_INF) {
            z[i] = (float)t;
            rgb[3 * i] = c[0];
            rgb[3 * i + 1] = c[1];
            rgb[3 * i + 2] = c[2];
        }
    }
}

void stage_intersect_cells(int64_t n, const float *corners, const double *o, const double *d, const double *cell,
                           const double *t0, const double *t1, double iso, double *t_out) {
    if (n <= 0) return;
    Stream S;
    DevBuf<float> dc;
    DevBuf<double> dO, dD, dC, d0, d1, dt;
    to_dev(dc, corners, 8 * n, S.st);
    to_dev(dO, o, 3 * n, S.st);
    to_dev(dD, d, 3 * n, S.st);
    to_dev(dC, cell, 3 * n, S.st);
    to_dev(d0, t0, n, S.st);
    to_dev(d1, t1, n, S.st);
    dt.alloc(n);
    launch_pdl(k_intersect_cells, grid_for(n, 128), 128, 0, S.st, n, dc.p, dO.p, dD.p, dC.p, d0.p, d1.p, iso, dt.p);
    WC_LAUNCH_CHECK();
    to_host(t_out, dt.p, n, S.st);
    S.sync();
}

// Self-check of the factored division (wc_common.cuh div_by): n operand
// pairs from a counter-based hash, a mix of the path's own magnitudes (grid
// coordinates minus ray origins over unit-vector components) and arbitrary
// bit patterns; counts quotients whose bits differ from a / b.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    return x ^ (x >> 33);
}
__global__ void k_fastdiv_check(uint64_t n, uint64_t seed, unsigned long long *bad, double *example) {
    unsigned long long local = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h1 = mix64(seed ^ (2 * i)), h2 = mix64(seed ^ (2 * i + 1));
        double a, b;
        switch (h1 & 3) {
            case 0:  // the path: (grid coordinate - origin) / direction component
                a = (double)(int)((h1 >> 8) % 9000) - 4500.0 + __longlong_as_double((h2 & 0x000FFFFFFFFFFFFFull) |
                                                                                    0x3FF0000000000000ull);
                b = __longlong_as_double(((h2 >> 3) & 0x000FFFFFFFFFFFFFull) |
                                         ((uint64_t)(1022 - ((h2 >> 58) & 31)) << 52)) *
                    ((h1 >> 4) & 1 ? -1.0 : 1.0);
                break;
            case 1:  // constants over components (4 / d, 16 / d, 1 / d)
                a = (double)(1u << (2 * ((h1 >> 8) % 3)));
                b = __longlong_as_double((h2 & 0x000FFFFFFFFFFFFFull) | ((uint64_t)(1023 - ((h2 >> 52) & 63)) << 52)) *
                    ((h1 >> 4) & 1 ? -1.0 : 1.0);
                break;
            default:  // arbitrary bit patterns (incl. subnormals, infinities, NaN)
                a = __longlong_as_double((long long)h1);
                b = __longlong_as_double((long long)h2);
                break;
        }
        const double q = div_by(a, recip_of(b)), ref = a / b;
        const bool same = __double_as_longlong(q) == __double_as_longlong(ref) || (q != q && ref != ref);
        if (!same) {
            local++;
            example[0] = a;
            example[1] = b;
        }
    }
    if (local) atomicAdd(bad, local);
}

int64_t stage_check_fastdiv(int64_t n, uint64_t seed, double *example) {
    DevBuf<unsigned long long> d_bad;
    DevBuf<double> d_ex;
    d_bad.alloc(1);
    d_ex.alloc(2);
    WC_CUDA(cudaMemset(d_bad.p, 0, sizeof(unsigned long long)));
    WC_CUDA(cudaMemset(d_ex.p, 0, 2 * sizeof(double)));
    k_fastdiv_check<<<num_sms() * 8, 256>>>((uint64_t)n, seed, d_bad.p, d_ex.p);
    WC_LAUNCH_CHECK();
    unsigned long long bad = 0;
    WC_CUDA(cudaMemcpy(&bad, d_bad.p, sizeof(bad), cudaMemcpyDeviceToHost));
    if (example) WC_CUDA(cudaMemcpy(example, d_ex.p, 2 * sizeof(double), cudaMemcpyDeviceToHost));
    return (int64_t)bad;
}

void stage_cell_overlaps(int64_t n, const double *o, const double *d, const double *cell, double *t0, double *t1) {
    if (n <= 0) return;
    Stream S;
    DevBuf<double> dO, dD, dC, d0, d1;
    to_dev(dO, o, 3 * n, S.st);
    to_dev(dD, d, 3 * n, S.st);
    to_dev(dC, cell, 3 * n, S.st);
    d0.alloc(n);
    d1.alloc(n);
    launch_pdl(k_cell_overlaps, grid_for(n, 128), 128, 0, S.st, n, dO.p, dD.p, dC.p, d0.p, d1.p);
    WC_LAUNCH_CHECK();
    to_host(t0, d0.p, n, S.st);
    to_host(t1, d1.p, n, S.st);
    S.sync();
}

void stage_shade(int64_t n, const double *grad, const double *dir, const double base[3], double *rgb) {
    if (n <= 0) return;
    Stream S;
    DevBuf<double> dg, dd, dr;
    to_dev(dg, grad, 3 * n, S.st);
    to_dev(dd, dir, 3 * n, S.st);
    dr.alloc(3 * n);
    launch_pdl(k_shade, grid_for(n, 128), 128, 0, S.st, n, dg.p, dd.p, base[0], base[1], base[2], dr.p);
    WC_LAUNCH_CHECK();
    to_host(rgb, dr.p, 3 * n, S.st);
    S.sync();
}

void stage_raytrace_block(const float *values125, const int origin[3], const int cells[3], int64_t n, const double *o,
                          const double *d, const double *t_enter, double iso, const double base[3], float *rgb,
                          float *z, uint8_t *hit) {
    if (n <= 0) return;
    Stream S;
    DevBuf<float> dv, drgb, dz;
    DevBuf<double> dO, dD, dT;
    DevBuf<uint8_t> dh;
    to_dev(dv, values125, 125, S.st);
    to_dev(dO, o, 3 * n, S.st);
    to_dev(dD, d, 3 * n, S.st);
    to_dev(dT, t_enter, n, S.st);
    to_dev(drgb, rgb, 3 * n, S.st);
    to_dev(dz, z, n, S.st);
    dh.alloc(n);
    launch_pdl(k_raytrace_block, grid_for(n, 128), 128, 0, S.st, dv.p, origin[0], origin[1], origin[2], cells[0],
               cells[1], cells[2], n, dO.p, dD.p, dT.p, iso, base[0], base[1], base[2], drgb.p, dz.p, dh.p);
    WC_LAUNCH_CHECK();
    to_host(rgb, drgb.p, 3 * n, S.st);
    to_host(z, dz.p, n, S.st);
    to_host(hit, dh.p, n, S.st);
    S.sync();
}

}  // namespace wc
