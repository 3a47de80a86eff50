/*
 * wc_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C, single-threaded restatement of the reference `wavecast` render
 * path (/root/reference/pkg/src/wavecast, pure Python + numba).  It exists so
 * that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg can
 * CHECK the CUDA product path; nothing in paper_2309_10212_b200/ may link,
 * load or call it.  Parity of this restatement with the reference is pinned
 * by tests/golden/ (fixtures produced by importing the reference itself, see
 * tests/golden/make_golden.py) and by tests/test_oracle_vs_reference.py when
 * /root/reference is present.
 *
 * Every function cites the reference file:line it restates.
 */
#ifndef WC_ORACLE_H
#define WC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_UINT_MAX 0xFFFFFFFFu

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
} orc_pass_stats;

/* Camera basis computed by the host exactly as traversal.py:65-70,111. */
typedef struct {
    double eye[3];
    double look[3];
    double right[3];
    double up[3];
    double tan_half;
    int32_t img_w;
    int32_t img_h;
} orc_camera;

/* codec.py:143-174 */
void orc_decode_blocks(const uint8_t *payload, int qbits, int stride,
                       const int64_t *ids, int64_t n, float *out);
/* codec.py:177-198 (+ _gather_blocks :81-97, _block_exponents :100-105,
 * _pack_blocks :120-140). payload must be zeroed by the caller. */
void orc_compress(const float *values, int nx, int ny, int nz, int qbits,
                  uint8_t *payload, float *ranges, int32_t *exponents);
/* compress of a separable field sum_k ((amp*fz)*fy)*fx, block layers [bz0,bz1) */
void orc_compress_separable(int K, const float *amp, const float *fx, const float *fy, const float *fz, int nx,
                            int ny, int nz, int qbits, int bz0, int bz1, uint8_t *payload, float *ranges);
/* codec.py:113-117 over the exponents stored in the payload (:220-223) */
void orc_error_bounds(const uint8_t *payload, int64_t n_blocks, int qbits,
                      int stride, double *bounds);
/* grids.py:71-94 */
void orc_build_grids(const float *ranges, const double *bounds, int bdx,
                     int bdy, int bdz, double *fine_min, double *fine_max,
                     double *coarse_min, double *coarse_max);

/* Ray generation traversal.py:105-187.  pixel_ids (nullable) selects a
 * subset of the full image's pixels (tile sharding); n = number of rays. */
void orc_camera_rays(const orc_camera *cam, const int64_t *pixel_ids,
                     int64_t n, double *origin, double *direction);

typedef struct orc_session orc_session;

/* engine.py:308-322.  All pointers are borrowed for the session lifetime.
 * origin/direction: n x 3 float64 (from orc_camera_rays or arbitrary rays,
 * RaySoA.from_rays semantics).  cache_capacity <= 0 => initial_capacity(w,h)
 * (cache.py:122-125) with w*h == n_total_pixels. */
orc_session *orc_session_create(const uint8_t *payload, const float *ranges,
                                const double *fine_min, const double *fine_max,
                                const double *coarse_min,
                                const double *coarse_max, int nx, int ny,
                                int nz, int qbits, int stride,
                                const double *origin, const double *direction,
                                int64_t n, int64_t w, int64_t h, double iso,
                                int speculation, int max_spec,
                                int64_t cache_capacity, int corrupt_cache);
void orc_session_destroy(orc_session *s);
/* RenderOptions.base_color (engine.py:42); default (0.85, 0.85, 0.85) */
void orc_session_set_base_color(orc_session *s, double r, double g, double b);
/* One pass of engine.py:326-382. Returns 1 if a pass ran, 0 if done. */
int orc_session_pass(orc_session *s, orc_pass_stats *st);

/* Getters (copy out) for per-stage parity checks. */
void orc_get_rays(const orc_session *s, double *t_enter, double *t_exit,
                  uint8_t *status, uint8_t *exited, uint32_t *coarse_cell,
                  uint32_t *fine_cell, double *coarse_tmax, double *fine_tmax);
void orc_get_framebuffer(const orc_session *s, uint8_t *rgba, float *depth);
/* last pass buffers; returns sizes through the int64 array:
 * [n_slots_used, n_visible, n_active_blocks, n_entries] */
void orc_get_pass_sizes(const orc_session *s, int64_t *sizes);
void orc_get_slots(const orc_session *s, uint32_t *block_slots,
                   uint32_t *ray_slots, uint32_t *active_offsets);
void orc_get_visible_active(const orc_session *s, uint32_t *visible_ids,
                            uint32_t *active_ids);
void orc_get_rt_inputs(const orc_session *s, uint32_t *rays_per_block,
                       uint32_t *block_ray_offsets, uint32_t *sorted_ray_ids,
                       uint32_t *sorted_hit_slots, uint32_t *valid_prefix);
void orc_get_rgbz(const orc_session *s, float *rgb, float *z);
int64_t orc_cache_capacity(const orc_session *s);
/* block_of_slot over the logical capacity (-1 = free) */
void orc_get_cache(const orc_session *s, int64_t *block_of_slot,
                   int64_t *last_used, float *slot_values);

/* Standalone LRU cache, cache.py:27-111 (for BlockCache parity tests). */
typedef struct orc_cache orc_cache;
orc_cache *orc_cache_create(int64_t capacity, int64_t n_blocks);
void orc_cache_destroy(orc_cache *c);
/* active_ids ascending; returns stats[3] = new_decompressed, evicted, grown_to */
void orc_cache_update(orc_cache *c, const uint8_t *payload, int qbits,
                      int stride, const int64_t *active_ids, int64_t n_active,
                      int64_t *stats);
int64_t orc_cache_lookup(const orc_cache *c, int64_t block_id);
int64_t orc_cache_capacity_of(const orc_cache *c);
void orc_cache_state(const orc_cache *c, int64_t *block_of_slot,
                     int64_t *last_used, float *slot_values);

/* Brute-force oracle: oracle.py:42-122 over a dense decoded volume
 * (values x-fastest).  status/t_enter follow RaySoA.from_rays. */
void orc_reference_render(const float *values, int nx, int ny, int nz,
                          const double *origin, const double *direction,
                          int64_t n, double iso, double base_r, double base_g,
                          double base_b, uint8_t *rgba, float *depth);
/* blocktrace.py:236-280 (intersect_cell wrapper :452-472); returns +inf if none */
double orc_intersect_cell(const float *corners, const double *o,
                          const double *d, const double *cell, double t0,
                          double t1, double iso);

#ifdef __cplusplus
}
#endif
#endif
