/*
 * wavecast_b200.h -- C ABI of libwavecast_b200.so, the sm_100a render path.
 *
 * The reference (`wavecast`, /root/reference/pkg/src/wavecast) is a pure
 * Python + numba package with no FFI of its own; its drop-in boundary is
 * the Python API re-exported by wavecast/__init__.py:3-56.  Each entry point
 * below is what that API's hot path binds to through ctypes
 * (paper_2309_10212_b200/_lib.py); the reference interface it replaces is
 * cited per function.  No torch types cross this boundary: plain pointers,
 * sizes and opaque handles.  Every function returns 0 on success or a
 * WC_E_* code, with a message in wc_last_error().
 */
#ifndef WAVECAST_B200_H
#define WAVECAST_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WC_OK 0
#define WC_E_USAGE 2     /* maps to wavecast.errors.UsageError (errors.py:4-5) */
#define WC_E_DATA 3      /* maps to wavecast.errors.DataError  (errors.py:8-9) */
#define WC_E_INVARIANT 4 /* maps to AssertionError (engine.py:302,332,341)    */
#define WC_E_CUDA 5      /* CUDA runtime failure (no GPU, OOM, fault)         */

typedef struct wc_volume wc_volume;
typedef struct wc_session wc_session;
typedef struct wc_cache wc_cache;
typedef struct wc_frame_target wc_frame_target;

/* engine.py:66-77 PassStats (+ evicted, n_entries, n_active_after) */
typedef struct {
    int64_t pass_index;
    int64_t n_active_before;
    int64_t n_spec;
    int64_t visible_blocks;
    int64_t active_blocks;
    int64_t new_decompressed;
    int64_t evicted;
    int64_t cache_slots;
    int64_t n_entries;
    int64_t n_active_after;
    double utilization;
    double completeness;
    double duration;
} wc_pass_stats;

/* Camera basis as computed by traversal.py:65-70 (look, right, up) and
 * :111 (tan_half), plus the full image size (traversal.py:113-114). */
typedef struct {
    double eye[3];
    double look[3];
    double right[3];
    double up[3];
    double tan_half;
    int32_t img_w;
    int32_t img_h;
} wc_camera;

const char *wc_last_error(void);
/* Select the CUDA device (fails loudly when no GPU is present). */
int wc_init(int device);
/* Number of kernels this library has launched so far (all threads). */
long long wc_launch_count(void);
/* Page-locked host memory for framebuffer read-back (full-bandwidth D2H). */
int wc_host_alloc(uint64_t bytes, void **out);
int wc_host_free(void *p);
/* Build-time identity string (arch, flags). */
const char *wc_build_info(void);

/* ---- volume: CompressedVolume (codec.py:34-65) + build_grids (grids.py:71-94)
 * Uploads a WCZ1 payload + raw ranges to HBM and builds the float64 fine /
 * coarse value-range grids on the device. */
int wc_volume_create(const uint8_t *payload, uint64_t payload_bytes, const float *ranges, int nx, int ny, int nz,
                     int qbits, int stride, wc_volume **out);
/* compress_volume (codec.py:177-198) of a dense float32 field (x-fastest,
 * host pointer) on the device, then build_grids. */
int wc_volume_compress(const float *values, int nx, int ny, int nz, int qbits, wc_volume **out);
/* Same for a separable synthetic field v = sum_k ((amp[k]*fz[k][z])*fy[k][y])*fx[k][x]
 * generated on the device block by block (no dense field in memory). */
int wc_volume_synthesize(int K, const float *amp, const float *fx, const float *fy, const float *fz, int nx, int ny,
                         int nz, int qbits, wc_volume **out);
int wc_volume_destroy(wc_volume *v);
/* Replace the device grids with caller-supplied MacrocellGrids arrays
 * (grids.py:32-45; float64 fine n_blocks and coarse n_coarse entries). */
int wc_volume_set_grids(wc_volume *v, const double *fine_min, const double *fine_max, const double *coarse_min,
                        const double *coarse_max);
/* n_blocks, n_coarse, payload bytes */
int wc_volume_info(const wc_volume *v, int64_t *n_blocks, int64_t *n_coarse, int64_t *payload_bytes);
/* Copy the device payload / ranges / grids back to host buffers (nullable). */
int wc_volume_download(const wc_volume *v, uint8_t *payload, float *ranges, double *fine_min, double *fine_max,
                       double *coarse_min, double *coarse_max);
/* (min, max) of the decoded voxels inside dims -- the value_range of
 * oracle.decode_full (oracle.py:22-39), computed on the device. */
int wc_volume_value_range(const wc_volume *v, double *lo, double *hi);

/* ---- .wcz container (read_wcz, codec.py:243-273) straight to HBM
 * Header/size validation with read_wcz's DataError / UsageError messages
 * (no device needed). */
int wc_wcz_probe(const char *path, int *nx, int *ny, int *nz, int *qbits, int *stride, int64_t *n_blocks);
/* Stream the ranges and payload from the file into device memory through two
 * pinned chunks (chunk_bytes, 0 = 64 MiB; reads overlap the H2D copies),
 * then build the grids on the device. */
int wc_volume_load_wcz(const char *path, int64_t chunk_bytes, wc_volume **out);
/* A volume whose payload/ranges are filled on the device by the caller
 * (e.g. an NCCL broadcast from the rank that loaded the file): alloc, write
 * through wc_volume_device_buffers, then wc_volume_finalize builds the grids. */
int wc_volume_alloc(int nx, int ny, int nz, int qbits, wc_volume **out);
int wc_volume_device_buffers(wc_volume *v, void **payload, uint64_t *payload_bytes, void **ranges,
                             uint64_t *ranges_bytes);
int wc_volume_finalize(wc_volume *v);

/* decompress_block(s) (codec.py:201-217): host ids in, host float32[n*64] out. */
int wc_decode_blocks(const wc_volume *v, const int64_t *ids, int64_t n, float *out);
/* Device-only timing of decode: decodes `n` blocks (ids on host, uploaded
 * once) `reps` times into a device buffer; returns average ms per launch. */
int wc_decode_bench(const wc_volume *v, const int64_t *ids, int64_t n, int reps, double *ms_per_launch);

/* ---- session: engine.render_passes (engine.py:308-382)
 * Camera rays (origins == dirs == NULL) for all w*h pixels or for the
 * `pixel_ids` subset (tile sharding; n = number of pixels), or arbitrary
 * rays (RaySoA.from_rays, traversal.py:122-170) through origins/dirs (n x 3).
 * cache_capacity <= 0 selects initial_capacity (cache.py:122-125). */
int wc_session_create(wc_volume *v, const wc_camera *cam, const uint32_t *pixel_ids, int64_t n, const double *origins,
                      const double *dirs, double iso, int speculation, int max_spec, int64_t cache_capacity,
                      int corrupt_cache, wc_session **out);
int wc_session_set_base_color(wc_session *s, double r, double g, double b);
/* build_rt_inputs (engine.py:121-149) grouping on (1) or off (0, default):
 * the raytrace is correct either way (same pixels); grouping yields the
 * reference's PassBuffers layout (required by wc_session_rt_inputs). */
int wc_session_set_grouping(wc_session *s, int group_entries);
/* Tile-split frames: reset computing the per-iso range
 * tests (coarse bitmap words, 64-bit fine masks) only for coarse-cell slice
 * `part` of `parts`; the caller all-gathers the slices (each `chunk_words`
 * bitmap words = 32 x chunk_words masks, at offset part x chunk) into the
 * buffers wc_session_mask_buffers returns, then runs the passes
 * (wc_session_run).  wc_session_sync waits for the session's stream. */
int wc_session_reset_part(wc_session *s, const wc_camera *cam, double iso, int64_t part, int64_t parts);
int wc_session_mask_buffers(wc_session *s, int64_t parts, void **coarse_bm, void **cell_mask, int64_t *chunk_words);
int wc_session_sync(wc_session *s);  /* waits for the session's stream and its copies */
/* Replay passes as captured CUDA graphs (default on; WAVECAST_NO_GRAPHS=1 in
 * the environment turns it off).  Off = plain launches with per-stage
 * timing (wc_session_stage_ms); on = the pass timed as a whole. */
int wc_session_set_graphs(wc_session *s, int on);
/* One pass; *ran = 0 once every ray has terminated. */
int wc_session_pass(wc_session *s, wc_pass_stats *stats, int *ran);
/* Run passes until done (render, engine.py:385-401); returns pass count. */
int wc_session_run(wc_session *s, wc_pass_stats *stats_out, int64_t max_stats, int64_t *n_passes);
/* reset(cam, iso) + run in one call: one frame of render (engine.py:385-401)
 * on the session's allocations with no host round trip between the two. */
int wc_session_render(wc_session *s, const wc_camera *cam, double iso, wc_pass_stats *stats_out, int64_t max_stats,
                      int64_t *n_passes);
/* reset + run (as wc_session_render) with the framebuffer delivered into
 * host memory (RGBA8 packed u32[n], depth f32[n]; page-locked buffers from
 * wc_host_alloc for full-speed copies): the bulk of the copy starts on a
 * second stream once most rays are done (the last frame tells when) and
 * overlaps the tail passes; the pixels still active then are patched after. */
int wc_session_render_host(wc_session *s, const wc_camera *cam, double iso, wc_pass_stats *stats_out,
                           int64_t max_stats, int64_t *n_passes, uint32_t *rgba, float *depth);
int wc_session_n_active(const wc_session *s, int64_t *n_active);
/* Framebuffer.snapshot (engine.py:62-63): RGBA8 (n x 4) + float32 depth (n). */
int wc_session_framebuffer(wc_session *s, uint8_t *rgba, float *depth);
/* Streamed snapshot of the current framebuffer (render_passes yields one per
 * pass, engine.py:62-63, :380-382): copied on the device into a ring slot
 * (session stream), then to the caller's host buffers (n RGBA8 words + n
 * float32, page-locked for full speed) on a copy stream, overlapped with the
 * passes that follow.  The buffers must stay valid until
 * wc_session_snapshot_wait(ticket) returns (or wc_session_sync). */
int wc_session_snapshot(wc_session *s, uint32_t *rgba_host, float *depth_host, int64_t *ticket);
int wc_session_snapshot_wait(wc_session *s, int64_t ticket);
/* The session's CUDA stream (cudaStream_t), so a caller can order its own
 * device work -- e.g. NCCL collectives over the session's buffers -- on it
 * without host synchronisation. */
int wc_session_stream(const wc_session *s, void **stream);
/* The framebuffer packed into a caller DEVICE buffer: RGBA8 words at
 * [0, n), depth bits at [stride, stride + n) (stride >= n), ordered on the
 * session stream: a tile gather's send buffer. */
int wc_session_framebuffer_packed(wc_session *s, void *dst_dev, int64_t stride_words);
/* Multi-GPU frame assembly: packed holds n / stride blocks of
 * [stride RGBA8 words | stride depth bits] (one per rank, a gather's receive
 * buffer); pixel_ids (int64, n; < 0 = padding) maps block b's entry i to its
 * pixel.  Writes frame rgba / depth (DEVICE, u32 per pixel) on `stream`. */
int wc_scatter_pixels(const void *packed_dev, int64_t stride_words, const void *pixel_ids_dev, int64_t n,
                      void *rgba_dev, void *depth_dev, void *stream);
/* Multi-GPU frame assembly over peer memory (the fused
 * option): rank 0 creates a full-frame target (RGBA8 + depth, npix pixels) on
 * its GPU and exports two CUDA IPC handles (128 bytes); every other rank opens
 * them.  A session given a target writes each pixel's final value into it the
 * moment the ray terminates (at reset for rays that miss the volume, in the
 * pass's composite for the others), so the frame assembles over NVLink while
 * the remaining passes run and no gather is needed.  Once every rank's frame
 * has completed, rank 0 downloads the target. */
int wc_frame_target_create(int64_t npix, wc_frame_target **out);
int wc_frame_target_ipc_handles(const wc_frame_target *t, void *handles);
int wc_frame_target_open(const void *handles, int64_t npix, wc_frame_target **out);
int wc_frame_target_download(const wc_frame_target *t, uint32_t *rgba_host, float *depth_host);
int wc_frame_target_destroy(wc_frame_target *t);
/* The session's final pixels also go to `t` (NULL: stop); camera sessions. */
int wc_session_set_frame_target(wc_session *s, const wc_frame_target *t);
/* Same into caller-owned DEVICE buffers (for NCCL tile gathers). */
int wc_session_framebuffer_device(wc_session *s, void *rgba_dev, void *depth_dev);
/* Device time of the last pass (CUDA events on the session stream). */
int wc_session_last_pass_ms(const wc_session *s, double *ms);
int wc_session_destroy(wc_session *s);
/* Start a new frame on the same allocations (a viewer moving its camera):
 * fresh rays for `cam` (NULL keeps the camera; arbitrary-ray sessions
 * re-seed their rays), new iso, blank framebuffer, empty cache. */
int wc_session_reset(wc_session *s, const wc_camera *cam, double iso);
/* Device time (CUDA events on the session stream) from the last
 * create/reset to the end of the last pass. */
int wc_session_frame_ms(wc_session *s, double *ms);
/* Accumulated device ms per stage since the last reset, then the reset itself:
 * [traverse, mark+extract, cache+decode, raytrace inputs (+ grouping sort), raytrace, composite, reset]
 * (7 doubles) */
int wc_session_stage_ms(const wc_session *s, double *ms6);
/* The same split for one pass (pass_index < 128) of the current frame. */
int wc_session_pass_stage_ms(const wc_session *s, int64_t pass_index, double *ms6);

/* Per-kernel device time of the passes launched kernel by kernel (graphs
 * off, wc_session_set_graphs(s, 0)) while profiling is on: CUDA events on the
 * session stream around every launch.  The text has one row per (pass,
 * kernel): "pass<TAB>kernel<TAB>launches<TAB>ms".  *len = its length. */
int wc_session_set_kernel_profile(wc_session *s, int on); /* also clears */
int wc_session_kernel_profile(const wc_session *s, char *buf, int64_t cap, int64_t *len);

/* ---- per-stage views of the last pass (parity tests) */
/* sizes[9] = slots_used, n_visible, n_active_blocks, n_entries, n_spec,
 *            n_active_before, cache_capacity, cache_physical,
 *            rays the traversal handed to its warp-per-ray long-ray pass */
int wc_session_sizes(const wc_session *s, int64_t *sizes);
/* RaySoA fields (traversal.py:76-91), each nullable */
int wc_session_rays(const wc_session *s, double *dir, double *t_enter, double *t_exit, uint8_t *status,
                    uint8_t *exited, uint32_t *coarse_cell, uint32_t *fine_cell, double *coarse_tmax,
                    double *fine_tmax);
/* block_slots / ray_slots prefix [0, slots_used) and the last pass's
 * compacted active-ray list [0, n_active_before) */
int wc_session_slots(const wc_session *s, uint32_t *block_slots, uint32_t *ray_slots, uint32_t *active_list);
int wc_session_blocks(const wc_session *s, uint32_t *visible_ids, uint32_t *active_ids);
/* grouped RT inputs (engine.py:121-149): block_ray_offsets[n_visible+1],
 * sorted entry ids (== sorted_hit_slots) and the owning ray per entry id */
int wc_session_rt_inputs(const wc_session *s, uint32_t *block_ray_offsets, uint32_t *sorted_entries,
                         uint32_t *entry_ray);
/* rgbz per entry id: float4 (r, g, b, z) x n_entries */
int wc_session_rgbz(const wc_session *s, float *rgbz);
/* cache state over the physical slots: block_of_slot / last_used (int32),
 * slot_values (float32 x 64) -- each nullable */
int wc_session_cache(const wc_session *s, int32_t *block_of_slot, int32_t *last_used, float *slot_values);

/* ---- standalone pieces */
/* RaySoA.from_camera / from_rays (traversal.py:105-187) on the device */
int wc_init_rays(const wc_camera *cam, const uint32_t *pixel_ids, int64_t n, const double *origins,
                 const double *dirs, int nx, int ny, int nz, double *dir_out, double *t_enter, double *t_exit,
                 uint8_t *status, uint8_t *exited, uint32_t *coarse_cell, uint32_t *fine_cell, double *coarse_tmax,
                 double *fine_tmax);
/* oracle.reference_render (oracle.py:42-122): brute-force over the fully
 * decoded volume on the device (for parity at scales the CPU cannot do). */
int wc_reference_render(const wc_volume *v, const double *origins, const double *dirs, int64_t n, double iso,
                        double base_r, double base_g, double base_b, uint8_t *rgba, float *depth);
/* same over a dense float32 field (x-fastest) given by the caller */
int wc_reference_render_dense(const float *values, int nx, int ny, int nz, const double *origins, const double *dirs,
                              int64_t n, double iso, double base_r, double base_g, double base_b, uint8_t *rgba,
                              float *depth);
/* prims.py:13-40 on the device (host arrays in/out) */
int wc_exclusive_scan(const uint32_t *values, int64_t n, uint32_t *out, uint64_t *total);
int wc_sort_by_key(uint32_t *keys, uint32_t *values, int64_t n);
/* compact (prims.py:26-31): indices i < n with mask[i] != 0, ascending */
int wc_compact_indices(const uint8_t *mask, int64_t n, uint32_t *out, uint64_t *total);

/* ---- stage-level entry points: the reference's lower-level API
 * (wavecast/__init__.py:3-56), each one stage on the device with host
 * arrays in and out, for callers and tests that drive the stages one at a
 * time.  The render session above fuses the same stages into one pipeline. */

/* traverse_to_next_blocks (traversal.py:406-452): advance every active ray
 * (status == 0) to its next <= n_spec candidate blocks.  Grids from `v`
 * (its device copy) or, when v is NULL, from the four float64 arrays
 * (MacrocellGrids, grids.py:32-45).  RaySoA fields in/out as in
 * traversal.py:76-91; block_slots / ray_slots (n) are overwritten.
 * active_offsets (n, int64) must number the active rays 0..n_active-1.
 * variant: 0 as the session picks, 1 thread per ray, 2 warp per ray.
 * Slot budget (n_active * n_spec <= n, traversal.py:420) -> WC_E_INVARIANT. */
int wc_traverse(const wc_volume *v, const double *fine_min, const double *fine_max, const double *coarse_min,
                const double *coarse_max, const int *fine_dims, const int *coarse_dims, int64_t n,
                const double *origin, const double *dir, const double *t_exit, const uint8_t *status, uint8_t *exited,
                uint32_t *coarse_cell, double *coarse_tmax, uint32_t *fine_cell, double *fine_tmax,
                uint32_t *block_slots, uint32_t *ray_slots, const int64_t *active_offsets, double iso, int n_spec,
                int variant);
/* mark_blocks (engine.py:97-118): visible / active block sets as bitmaps
 * (bit b of word b / 32), ceil(bdx*bdy*bdz / 32) words each. */
int wc_mark_blocks(const uint32_t *block_slots, int64_t n, int bdx, int bdy, int bdz, uint32_t *visible_words,
                   uint32_t *active_words);
/* build_rt_inputs (engine.py:121-149).  visible_words: the visible mask as a
 * bitmap.  Output capacities: visible_ids / rays_per_block /
 * block_ray_offsets n_blocks + 1, sorted_* n, valid_prefix n.
 * sizes[3] = n_entries, n_visible, len(rays_per_block). */
int wc_build_rt_inputs(const uint32_t *block_slots, const uint32_t *ray_slots, int64_t n,
                       const uint32_t *visible_words, int64_t n_blocks, uint32_t *visible_ids,
                       uint32_t *rays_per_block, uint32_t *block_ray_offsets, uint32_t *sorted_ray_ids,
                       uint32_t *sorted_hit_slots, uint32_t *valid_prefix, int64_t *sizes);
/* composite (engine.py:222-283): rgbz (n_rgbz x 3 float32 + n_rgbz float32),
 * ray status (in/out) / exited (n), slot buffers (n_slots), framebuffer
 * RGBA8 (n x 4, in/out) and depth (n, in/out). */
int wc_composite(const float *rgbz_rgb, const float *rgbz_z, int64_t n_rgbz, int64_t n, uint8_t *status,
                 const uint8_t *exited, const int64_t *active_offsets, int n_spec, const uint32_t *block_slots,
                 int64_t n_slots, const uint32_t *valid_prefix, uint8_t *rgba, float *depth);

/* BlockCache (cache.py:21-111) on the device: the session's cache update
 * (stamp, miss list, growth to ceil(1.5 needed), (last_used, id) victims,
 * decode straight into the slots) one ensure_resident at a time. */
int wc_cache_create(int64_t capacity_slots, wc_cache **out);
int wc_cache_destroy(wc_cache *c);
/* active_words: the active mask as a bitmap over n_blocks (== the volume's);
 * needed = its popcount.  Returns CacheUpdateStats (cache.py:20-24). */
int wc_cache_ensure_resident(wc_cache *c, const wc_volume *v, const uint32_t *active_words, int64_t n_blocks,
                             int64_t needed, int64_t *new_decompressed, int64_t *evicted, int64_t *grown_to);
/* logical capacity, physical (initialised) slots, pass counter, block count */
int wc_cache_info(const wc_cache *c, int64_t *capacity, int64_t *physical, int64_t *current_pass, int64_t *n_blocks);
/* lookup (cache.py:55-60): slot of a resident block or -1 */
int wc_cache_lookup(wc_cache *c, int64_t block_id, int64_t *slot);
/* slot_values (physical x 64), block_of_slot / last_used (physical),
 * slot_of_block (n_blocks); each nullable */
int wc_cache_state(wc_cache *c, float *slot_values, int32_t *block_of_slot, int32_t *last_used, int32_t *slot_of_block);
/* assemble_dual_grid (blocktrace.py:113-123): the 5^3 dual grid ([z][y][x])
 * of a resident block from its +octant contributors */
int wc_cache_dual_grid(wc_cache *c, int64_t block_id, float *values125);

/* blocktrace.py, batched over n cells / rays:
 * intersect_cell (:452-472): smallest root in [t0, t1] or +inf;
 * _cell_overlap (:126-158); shade (:475-488) of a gradient;
 * raytrace_block (:491-530): trace the block's dual cells per ray. */
int wc_intersect_cells(int64_t n, const float *corners, const double *origin, const double *dir, const double *cell,
                       const double *t0, const double *t1, double iso, double *t_out);
int wc_cell_overlaps(int64_t n, const double *origin, const double *dir, const double *cell, double *t0, double *t1);

/* Self-check (no reference counterpart): the kernels divide by a ray's
 * direction components through a factored float64 division (one reciprocal
 * refinement per divisor, reused); this compares it with the plain division
 * over n hashed operand pairs from `seed` and reports the mismatching count
 * (0 expected) and the last mismatching (a, b) in example[0..1]. */
int wc_check_fastdiv(int64_t n, uint64_t seed, int64_t *mismatches, double *example);
int wc_shade(int64_t n, const double *grad, const double *dir, const double *base_color, double *rgb);
int wc_raytrace_block(const float *values125, const int *block_origin, const int *cells_per_axis, int64_t n,
                      const double *origin, const double *dir, const double *t_enter, double iso,
                      const double *base_color, float *rgb, float *z, uint8_t *hit);

#ifdef __cplusplus
}
#endif
#endif
