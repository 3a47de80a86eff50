// wc_stage.cuh -- stage-level entry points (the reference's lower-level API,
// wavecast/__init__.py:3-56) on the device; see wc_stage.cu.
#pragma once

#include "wc_engine.cuh"

namespace wc {

// traverse_to_next_blocks (traversal.py:406-452).  Grids from `vol` (device)
// or, when vol is null, from the caller's float64 arrays.  variant: 0 picks
// the kernel as the session does, 1 thread-per-ray, 2 warp-per-ray.
void stage_traverse(const Volume *vol, const double *fine_min, const double *fine_max, const double *coarse_min,
                    const double *coarse_max, const int fd[3], const int cd[3], int64_t n, const double *origin,
                    const double *dir, const double *t_exit, const uint8_t *status, uint8_t *exited,
                    uint32_t *coarse_cell, double *coarse_tmax, uint32_t *fine_cell, double *fine_tmax,
                    uint32_t *block_slots, uint32_t *ray_slots, const int64_t *active_offsets, double iso, int n_spec,
                    int variant);
// mark_blocks (engine.py:97-118) -> visible / active bitmaps (32 blocks per word)
void stage_mark_blocks(const uint32_t *slots, int64_t n, int bdx, int bdy, int bdz, uint32_t *vis_words,
                       uint32_t *act_words);
// build_rt_inputs (engine.py:121-149); sizes = n_entries, n_visible, len(rays_per_block)
void stage_build_rt_inputs(const uint32_t *block_slots, const uint32_t *ray_slots, int64_t n,
                           const uint32_t *vis_words, int64_t n_blocks, uint32_t *visible_ids, uint32_t *rays_per_block,
                           uint32_t *block_ray_offsets, uint32_t *sorted_ray_ids, uint32_t *sorted_hit_slots,
                           uint32_t *valid_prefix, int64_t *sizes);
// composite (engine.py:222-283) on the reference's buffers
void stage_composite(const float *rgb, const float *z, int64_t n_rgbz, int64_t n, uint8_t *status,
                     const uint8_t *exited, const int64_t *offsets, int n_spec, const uint32_t *block_slots,
                     int64_t n_slots, const uint32_t *valid_prefix, uint8_t *rgba, float *depth);

// BlockCache (cache.py:21-111) on the device: the session's cache update
// (CacheStore) driven one ensure_resident at a time.
struct StageCache : CacheStore {
    const Volume *vol = nullptr;  // bound at the first update (cache.py:36-40)
    int64_t n_blocks = 0, cap = 0, phys = 0;
    int64_t current_pass = 0;
    cudaStream_t st = nullptr;
    DevBuf<uint32_t> ctl, partials, act_bm, active_ids;
    PinnedBuf<uint32_t> h_ctl;

    explicit StageCache(int64_t capacity);
    ~StageCache();
    void ensure_resident(const Volume *v, const uint32_t *mask_words, int64_t needed, int64_t *new_decompressed,
                         int64_t *evicted, int64_t *grown_to);
    int64_t lookup(int64_t block);  // slot or -1 (cache.py:55-60)
    void download(float *slot_values_out, int32_t *block_of_slot_out, int32_t *last_used_out,
                  int32_t *slot_of_block_out);
    void dual_grid(int64_t block, float *values125);  // blocktrace.py:113-123 assemble_dual_grid

   private:
    void bind(const Volume *v);
    void reserve_slots(int64_t need);
};

// blocktrace.py:126-158, 236-280, 306-314, 491-530 (batched)
void stage_intersect_cells(int64_t n, const float *corners, const double *o, const double *d, const double *cell,
                           const double *t0, const double *t1, double iso, double *t_out);
int64_t stage_check_fastdiv(int64_t n, uint64_t seed, double *example);
void stage_cell_overlaps(int64_t n, const double *o, const double *d, const double *cell, double *t0, double *t1);
void stage_shade(int64_t n, const double *grad, const double *dir, const double base[3], double *rgb);
void stage_raytrace_block(const float *values125, const int origin[3], const int cells[3], int64_t n, const double *o,
                          const double *d, const double *t_enter, double iso, const double base[3], float *rgb,
                          float *z, uint8_t *hit);

}  // namespace wc
