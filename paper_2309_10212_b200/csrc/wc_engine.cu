// wc_engine.cu -- per-pass wavefront pipeline on sm_100a (engine.py:308-382).
//
// One pass = traverse (+ fused visibility marking) -> scan of emitted
// counts -> visible-id extraction from the bitmap -> +octant active marking
// -> LRU residency with fused decode -> stable radix grouping of entries by
// visible block -> warp-per-block dual-grid raytrace -> min-depth composite
// + compaction of surviving rays.  Three small host reads per pass (entry /
// block counts, miss / free counts, surviving-ray count).
#include <math_constants.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>

#include <cstdlib>
#include <cxxabi.h>

#include "wc_engine.cuh"
#include "wc_trace.cuh"

// Resident CTAs (of 128 threads) per SM requested from ptxas for the two
// float64-heavy kernels; trades registers for latency hiding (tuned on B200
// with scripts/gpu_variants.sh).
#ifndef WC_SENTINEL_LATE
#define WC_SENTINEL_LATE 1
#endif
#ifndef WC_TRAVERSE_MIN_CTAS
#define WC_TRAVERSE_MIN_CTAS 5
#endif
// 1: one kernel with warp phases (k_rt_fused; measured slower at C3: raytrace
// 1.15 vs 0.96 ms/frame, the solves' divergence and 96 registers); 0: the
// work-list version below
#ifndef WC_RT_FUSED
#define WC_RT_FUSED 0
#endif
// 1: two-phase raytrace (k_rt_find / k_rt_solve / k_rt_shade); 0: fused k_raytrace.
#ifndef WC_SPLIT_RAYTRACE
#define WC_SPLIT_RAYTRACE 1
#endif
// 1: the thread-per-ray traversal queues its descents (k_traverse_q)
#ifndef WC_TRAVERSE_Q
#define WC_TRAVERSE_Q 0  // measured neutral at C3 (0.93 vs 0.91 ms/frame traverse): kept for comparison builds
#endif
// Passes with at most this many active rays use the warp-per-ray traversal.
#ifndef WC_WARP_TRAVERSE_MAX
#define WC_WARP_TRAVERSE_MAX 16384
#endif
// ... and passes of long rays (n_spec >= WC_WARP_LONG_SPEC) up to this many
// (a 4-way split's third pass: 22K rays at n_spec 23, 0.20 -> 0.12 ms; the
// whole frame's: 60K rays at n_spec 34 stay thread per ray, 0.30 vs 0.38 ms)
#ifndef WC_WARP_TRAVERSE_MAX_LONG
#define WC_WARP_TRAVERSE_MAX_LONG 32768
#endif
#ifndef WC_WARP_LONG_SPEC
#define WC_WARP_LONG_SPEC 16
#endif
// long-ray hand-off from the thread-per-ray traversal (k_traverse_long):
// in mid-size passes (one rank's share of a tile split) the pass time is the
// few long rays of the last lanes; 8-way share 0.93 -> 0.88 ms
#ifndef WC_TRAV_DEFER
#define WC_TRAV_DEFER 1
#endif
#ifndef WC_PASS_FORK
#define WC_PASS_FORK 1
#endif
// mark_blocks as one launch (mark_extract) when a bitmap word never straddles an x-row
#ifndef WC_MARK_FUSED
#define WC_MARK_FUSED 1
#endif
#ifndef WC_DEFER_ITERS
#define WC_DEFER_ITERS 12
#endif
#ifndef WC_DEFER_ITERS_LONG
#define WC_DEFER_ITERS_LONG 48  // passes of long rays hand off later (C3 third pass, 60K rays at n_spec 34: 0.90 -> 0.85 ms)
#endif
#ifndef WC_DEFER_CAP
#define WC_DEFER_CAP 16384
#endif
#ifndef WC_DEFER_ITERS_BIG
#define WC_DEFER_ITERS_BIG 0x7fffffff  // passes of more short rays: off (24: C3 -0.03 ms, C5 +0.13 ms mean)
#endif
#ifndef WC_DEFER_MAX_ACT
#define WC_DEFER_MAX_ACT 150000  // (a 2-way share's second pass, 205K rays: 0.145 -> 0.157 ms handed off)
#endif
// k_iso_cell_mask: coarse cells per half-warp in flight
#ifndef WC_ISO_KU
#define WC_ISO_KU 4
#endif
// k_decode_insert: warps per CTA, records staged per warp, CTAs per SM
#ifndef WC_DEC_WARPS
#define WC_DEC_WARPS 8
#endif
#ifndef WC_DEC_REC
#define WC_DEC_REC 16
#endif
#ifndef WC_DEC_CTAS
#define WC_DEC_CTAS 3
#endif
#ifndef WC_DEC_PIPE
#define WC_DEC_PIPE 2
#endif
#ifndef WC_DEC_PREC
#define WC_DEC_PREC 8
#endif
// k_traverse: idle lanes that trigger a refill of the warp
#ifndef WC_REFILL_MIN
#define WC_REFILL_MIN 8
#endif
#ifndef WC_RTFIND_MIN_CTAS
#define WC_RTFIND_MIN_CTAS 8
#endif
#ifndef WC_ISO_MIN_CTAS
#define WC_ISO_MIN_CTAS 1
#endif
#ifndef WC_RTFIND_GRID
#define WC_RTFIND_GRID 64
#endif
#ifndef WC_RTSHADE_GRID
#define WC_RTSHADE_GRID 16
#endif
#ifndef WC_RAYTRACE_MIN_CTAS
#define WC_RAYTRACE_MIN_CTAS 6
#endif

namespace wc {

// --------------------------------------------------------------- ray setup

struct RayInitArgs {
    CameraParams cam;
    const uint32_t *pixel_ids;   // nullable: identity
    const double *origin_in;     // nullable: camera rays
    const double *dir_in;        // nullable: camera rays
    int nx, ny, nz;
    const unsigned long long *target;  // nullable: the frame target's {rgba, depth} device addresses (FrameTarget)
};

// A pixel's final value into the frame target (another rank's framebuffer in
// peer memory over NVLink, or a local one): written once, when the ray
// terminates (init or composite), so the full frame is assembled while the
// remaining passes run.  target[0] == 0: no target.
__device__ __forceinline__ void target_write(const unsigned long long *target, const uint32_t *pixel_ids, uint32_t r,
                                             uint32_t rgba, float depth) {
    if (!target) return;
    uint32_t *tr = reinterpret_cast<uint32_t *>(target[0]);
    if (!tr) return;
    float *td = reinterpret_cast<float *>(target[1]);
    const uint32_t px = pixel_ids ? pixel_ids[r] : r;
    tr[px] = rgba;
    td[px] = depth;
}

// traversal.py:105-187 (from_camera + from_rays + _tmax_init) for ray r.
__global__ void k_init_rays(RayInitArgs a, int64_t n, double *origin_out, double *dir, double *t_enter, double *t_exit,
                            uint8_t *status, uint8_t *exited, uint32_t *coarse_cell, uint32_t *fine_cell,
                            double *coarse_tmax, double *fine_tmax, uint32_t *rgba, float *depth) {
    pdl_wait();
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        double o[3], d[3];
        if (a.dir_in) {
#pragma unroll
            for (int k = 0; k < 3; k++) {
                o[k] = a.origin_in[3 * r + k];
                d[k] = a.dir_in[3 * r + k];
            }
        } else {
            const int64_t p = a.pixel_ids ? (int64_t)a.pixel_ids[r] : r;
            const int64_t w = a.cam.img_w, h = a.cam.img_h;
            const int64_t px = p % w, py = p / w;
            const double aspect = (double)w / (double)h;
            const double xs = ((2.0 * ((double)px + 0.5)) / (double)w - 1.0) * a.cam.tan_half * aspect;
            const double ys = (1.0 - (2.0 * ((double)py + 0.5)) / (double)h) * a.cam.tan_half;
#pragma unroll
            for (int k = 0; k < 3; k++) d[k] = (a.cam.look[k] + xs * a.cam.right[k]) + ys * a.cam.up[k];
            const double nrm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
#pragma unroll
            for (int k = 0; k < 3; k++) {
                d[k] = d[k] / nrm;
                o[k] = a.cam.eye[k];
            }
        }
#pragma unroll
        for (int k = 0; k < 3; k++) {
            dir[3 * r + k] = d[k];
            if (origin_out) origin_out[3 * r + k] = o[k];
        }
        const double hi[3] = {(double)a.nx - 1.0, (double)a.ny - 1.0, (double)a.nz - 1.0};
        const int fd[3] = {(a.nx + 3) / 4, (a.ny + 3) / 4, (a.nz + 3) / 4};
        const int cd[3] = {(fd[0] + 3) / 4, (fd[1] + 3) / 4, (fd[2] + 3) / 4};
        double nr[3], fr[3];
#pragma unroll
        for (int k = 0; k < 3; k++) {
            if (d[k] != 0.0) {
                const double t1 = (0.0 - o[k]) / d[k];
                const double t2 = (hi[k] - o[k]) / d[k];
                nr[k] = t1 < t2 ? t1 : t2;  // np.minimum
                fr[k] = t1 > t2 ? t1 : t2;  // np.maximum
            } else if (o[k] < 0.0 || o[k] > hi[k]) {
                nr[k] = CUDART_INF;
                fr[k] = -CUDART_INF;
            } else {
                nr[k] = -CUDART_INF;
                fr[k] = CUDART_INF;
            }
        }
        double t_near = nr[0] > nr[1] ? nr[0] : nr[1];
        t_near = t_near > nr[2] ? t_near : nr[2];
        double t_far = fr[0] < fr[1] ? fr[0] : fr[1];
        t_far = t_far < fr[2] ? t_far : fr[2];
        const bool hit = (t_near <= t_far) && (t_far >= 0.0);
        const double te = t_near > 0.0 ? t_near : 0.0;
        t_enter[r] = te;
        t_exit[r] = t_far;
        status[r] = hit ? 0 : 2;
        exited[r] = 0;
        uint32_t fcell = WC_UINT_MAX, ccell = WC_UINT_MAX;
        double ft[3] = {0.0, 0.0, 0.0}, ct[3] = {0.0, 0.0, 0.0};
        if (hit) {
            int fc[3], cc[3];
#pragma unroll
            for (int k = 0; k < 3; k++) {
                const double p0 = o[k] + d[k] * (te + kEntryEps);
                int c = (int)floor(p0 / 4.0);
                c = c < 0 ? 0 : (c > fd[k] - 1 ? fd[k] - 1 : c);
                fc[k] = c;
                cc[k] = c / 4;
                if (d[k] == 0.0) {
                    ft[k] = CUDART_INF;
                    ct[k] = CUDART_INF;
                } else {
                    const double flo = (double)c * 4.0, clo = (double)cc[k] * 16.0;
                    ft[k] = ((d[k] > 0 ? flo + 4.0 : flo) - o[k]) / d[k];
                    ct[k] = ((d[k] > 0 ? clo + 16.0 : clo) - o[k]) / d[k];
                }
            }
            fcell = (uint32_t)(fc[0] + fd[0] * (fc[1] + fd[1] * fc[2]));
            ccell = (uint32_t)(cc[0] + cd[0] * (cc[1] + cd[1] * cc[2]));
        }
        fine_cell[r] = fcell;
        coarse_cell[r] = ccell;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            fine_tmax[3 * r + k] = ft[k];
            coarse_tmax[3 * r + k] = ct[k];
        }
        if (rgba) {
            rgba[r] = 0xFF000000u;  // BACKGROUND_RGBA (engine.py:29)
            depth[r] = CUDART_INF_F;
            if (!hit) target_write(a.target, a.pixel_ids, (uint32_t)r, 0xFF000000u, CUDART_INF_F);  // final already
        }
    }
}

void init_rays_device(const CameraParams *cam, const uint32_t *d_pixel_ids, int64_t n, const double *d_origin_in,
                      const double *d_dir_in, int nx, int ny, int nz, double *d_origin_out, double *d_dir,
                      double *t_enter, double *t_exit, uint8_t *status, uint8_t *exited, uint32_t *coarse_cell,
                      uint32_t *fine_cell, double *coarse_tmax, double *fine_tmax, cudaStream_t st) {
    RayInitArgs a{};
    if (cam) a.cam = *cam;
    a.pixel_ids = d_pixel_ids;
    a.origin_in = d_origin_in;
    a.dir_in = d_dir_in;
    a.nx = nx;
    a.ny = ny;
    a.nz = nz;
    launch_pdl(k_init_rays, grid_for(n, 256), 256, 0, st, a, n, d_origin_out, d_dir, t_enter, t_exit, status, exited,
                                                  coarse_cell, fine_cell, coarse_tmax, fine_tmax, nullptr, nullptr);
    WC_LAUNCH_CHECK();
}

// ---------------------------------------------------------- compaction glue

struct PredActive {  // status == STATUS_ACTIVE
    const uint8_t *s;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return s[i] == 0; }
};
struct PredMiss {  // active block not resident (cache.py:69-72)
    const uint32_t *ids;
    const int32_t *slot_of_block;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return slot_of_block[ids[i]] < 0; }
};

// cache.py:69-78 in one pass over the active ids: a resident block's slot is
// stamped with this pass (its last_used moves from bin `old` to bin pass_no
// of the stamp histogram kept after the counters, via per-CTA bins), a
// non-resident block is a miss (the scan's value 1, compacted in ascending
// id order).  The scan runs this loader only in the tile's owner, at most
// twice per element and by the same thread, so a plain read-modify-write
// moves each hit's histogram count once.
__device__ __forceinline__ int32_t *stamp_bins() {
    __shared__ int32_t bins[kHistBins + 1];  // [kHistBins]: hits moved into this pass's bin
    return bins;
}
struct LookupStamp {
    const uint32_t *ids;
    const int32_t *slot_of_block;
    int32_t *last_used;
    int32_t pass_no;
    uint32_t *hist;  // nullptr: no histogram upkeep (passes past kHistBins)
    __device__ __forceinline__ uint32_t operator()(int64_t i) const {
        const int32_t s = slot_of_block[ids[i]];
        if (s < 0) return 1u;
        const int32_t old = last_used[s];
        if (old != pass_no) {  // (a second load of the element by its thread finds it stamped)
            last_used[s] = pass_no;
            if (hist) {
                atomicSub(&stamp_bins()[old], 1);
                atomicAdd(&stamp_bins()[kHistBins], 1);
            }
        }
        return 0u;
    }
    __device__ __forceinline__ void cta_begin() const {
        if (hist)
            for (int b = threadIdx.x; b <= kHistBins; b += blockDim.x) stamp_bins()[b] = 0;
    }
    __device__ __forceinline__ void cta_end() const {
        if (!hist) return;
        __syncthreads();
        for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) {
            const int32_t v = stamp_bins()[b];
            if (v) atomicAdd(&hist[b], (uint32_t)v);  // two's complement: subtracts
        }
        if (threadIdx.x == 0 && stamp_bins()[kHistBins]) atomicAdd(&hist[pass_no], (uint32_t)stamp_bins()[kHistBins]);
        __threadfence();  // performed before the CTA's end arrival (the cache plan reads the histogram)
        __syncthreads();
    }
};

template <class Pred>
__global__ void k_compact_index(Pred pred, int64_t n, const uint32_t *off, uint32_t *out) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (pred(i)) out[off[i]] = (uint32_t)i;
}

// --------------------------------------------------------------- traverse

// Mark block b visible: traversal emission fused with mark_blocks
// (engine.py:97-106), one fire-and-forget RED.OR per emit.  (De-duplicating
// the lanes that emit the same block with a warp match first, WC_MARK_MATCH=1,
// costs more than the L2 atomics it saves: C3 traversal 0.72 -> 0.76 ms.)
#ifndef WC_MARK_MATCH
#define WC_MARK_MATCH 0
#endif
__device__ __forceinline__ void mark_visible(uint32_t *bm, uint32_t b) {
#if !WC_MARK_MATCH
    atomicOr(&bm[b >> 5], 1u << (b & 31));
    return;
#endif
    const uint32_t active = __activemask();
    const uint32_t peers = __match_any_sync(active, b);
    const int lane = threadIdx.x & 31;
    if ((peers & ((1u << lane) - 1u)) == 0) atomicOr(&bm[b >> 5], 1u << (b & 31));
}

// Amanatides-Woo state of one ray on one grid level.
struct Dda {
    int cx, cy, cz;
    double tx, ty, tz;
};

// One step; ties step x, then y, then z (traversal.py:303-314, :333-344).
// Returns the crossing parameter of the face just crossed.
// Branch-free form (predicated selects): lanes walking different rays (or
// the same ray different steps ahead) take different axes, and a branchy
// step would serialise the three paths across the warp.  The adds of the
// axes not taken are computed and discarded, so every value is unchanged.
#ifndef WC_DDA_BRANCHFREE
#define WC_DDA_BRANCHFREE 1
#endif
__device__ __forceinline__ double dda_step(Dda &s, int sx, int sy, int sz, double dlx, double dly, double dlz) {
#if WC_DDA_BRANCHFREE
    const bool mx = s.tx <= s.ty && s.tx <= s.tz;
    const bool my = !mx && s.ty <= s.tz;
    const bool mz = !mx && !my;
    const double t = mx ? s.tx : (my ? s.ty : s.tz);
    const double nx = s.tx + dlx, ny = s.ty + dly, nz = s.tz + dlz;
    s.cx += mx ? sx : 0;
    s.cy += my ? sy : 0;
    s.cz += mz ? sz : 0;
    s.tx = mx ? nx : s.tx;
    s.ty = my ? ny : s.ty;
    s.tz = mz ? nz : s.tz;
    return t;
#else
    double t;
    if (s.tx <= s.ty && s.tx <= s.tz) {
        t = s.tx;
        s.cx += sx;
        s.tx += dlx;
    } else if (s.ty <= s.tz) {
        t = s.ty;
        s.cy += sy;
        s.ty += dly;
    } else {
        t = s.tz;
        s.cz += sz;
        s.tz += dlz;
    }
    return t;
#endif
}

constexpr int kFineRun = 10;  // a monotone ray visits at most 4+4+4-2 fine cells of one coarse cell
#ifndef WC_CA_SPLIT
#define WC_CA_SPLIT 1
#endif
#ifndef WC_COARSE_AHEAD
#define WC_COARSE_AHEAD 2
#endif

// bit of fine cell f in its coarse cell's iso mask (k_iso_cell_mask)
__device__ __forceinline__ int fine_local(const Dda &f) { return 16 * (f.cx & 3) + (f.cy & 3) + 4 * (f.cz & 3); }

#ifndef WC_TRAV_PLAIN
#define WC_TRAV_PLAIN 0  // measured neutral at C3 (0.828 vs 0.824 ms), slower at C4 (2.01 vs 1.95 ms)
#endif
#ifndef WC_TRAV_KEEP
#define WC_TRAV_KEEP 1
#endif
#ifndef WC_TRAV_AXIS
#define WC_TRAV_AXIS 0  // per-axis exit tests (measured slower at C3: 0.88 vs 0.80 ms)
#endif
// dda_step that also reports the axis it stepped (0, 1, 2) and that axis'
// new cell coordinate: only that coordinate changed, so the grid-exit and
// leave-the-coarse-cell tests of the reference (traversal.py:315-355) reduce
// to tests on it (the other two were inside before the step and still are).
__device__ __forceinline__ double dda_step_ax(Dda &s, int sx, int sy, int sz, double dlx, double dly, double dlz,
                                              int &ax, int &v) {
    const bool mx = s.tx <= s.ty && s.tx <= s.tz;
    const bool my = !mx && s.ty <= s.tz;
    const double t = dda_step(s, sx, sy, sz, dlx, dly, dlz);
    ax = mx ? 0 : (my ? 1 : 2);
    v = mx ? s.cx : (my ? s.cy : s.cz);
    return t;
}
__device__ __forceinline__ int pick3(int ax, int a, int b, int c) { return ax == 0 ? a : (ax == 1 ? b : c); }

// traversal.py:217-403 _traverse_kernel, restructured for latency on B200:
//  * persistent: a lane that finishes its ray fetches the next active ray
//    from a warp-aggregated work counter, so divergent per-ray step counts do
//    not idle the warp;
//  * one L2 round trip per coarse cell: a coarse step loads the coarse range
//    bit and the 64-bit fine mask of the cell together; the fine run inside
//    the cell (<= 10 cells) then walks from registers.  Every iteration is
//    "coarse step (if not inside a run), then the rest of the run", so lanes
//    stay converged;
//  * CA > 1: CA coarse steps are simulated arithmetically first (the DDA
//    never depends on grid values) and their range bits fetched with
//    independent loads, then consumed in the reference's order.
// Every emitted slot, saved iterator and exit flag is the reference's, bit
// for bit.
template <int CA>
__device__ __forceinline__ void traverse_rays_thread(TraverseArgs a) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int fdx = a.fdx, fdy = a.fdy, fdz = a.fdz, cdx = a.cdx, cdy = a.cdy, cdz = a.cdz;
    bool have = false, exhausted = false;
    uint32_t i = 0, r = 0;
    double ox = 0, oy = 0, oz = 0, dx = 0, dy = 0, dz = 0, te = 0;
    double fdel_x = 0, fdel_y = 0, fdel_z = 0;  // coarse deltas: 4 * fdel (16/|d| == 4 * RN(4/|d|) exactly)
    int sx = 0, sy = 0, sz = 0, emitted = 0;
    Dda f{0, 0, 0, 0, 0, 0}, c{0, 0, 0, 0, 0, 0};
    bool in_fine_run = false;
    unsigned long long fm = 0;  // iso mask of the fine cells of coarse cell c
    int64_t base = 0;
    // A run is plain when no step of it can end the ray: coarse cell c and
    // its neighbours lie inside the grid (a step out of c lands in the grid)
    // and c's exit crossing (min of c's tmax: every fine crossing inside c is
    // earlier, up to a few ulps of accumulated rounding) is below t_exit by a
    // relative 1e-9.  Then the reference's exit test (traversal.py:315-320)
    // is false at every step and only the leave-c test remains.
#if WC_TRAV_DEFER
    int iters = 0;
    // (passes of short rays only: with n_spec >= WC_WARP_LONG_SPEC most rays
    // would be handed off -- a whole frame's third pass: 0.29 -> 0.36 ms)
    const bool long_rays = a.n_spec >= WC_WARP_LONG_SPEC;
    const int defer_k = !a.long_q ? 0x7fffffff
                        : a.n_act > (int64_t)WC_DEFER_MAX_ACT
                            ? (long_rays ? 0x7fffffff : WC_DEFER_ITERS_BIG)
                            : (long_rays ? WC_DEFER_ITERS_LONG : WC_DEFER_ITERS);
#endif
    bool plain = false;
    auto plain_cell = [&]() {
#if WC_TRAV_PLAIN
        const double tcx = fmin(c.tx, fmin(c.ty, c.tz));
        return c.cx >= 1 && c.cy >= 1 && c.cz >= 1 && 4 * c.cx + 5 <= fdx && 4 * c.cy + 5 <= fdy &&
               4 * c.cz + 5 <= fdz && tcx > 0.0 && tcx < te * (1.0 - 1e-9);
#else
        return false;
#endif
    };
    for (;;) {
        if (!exhausted) {  // refill idle lanes (warp-uniform branch)
            const uint32_t need = __ballot_sync(0xffffffffu, !have);
            // batched: the refill path (ray loads, FP64 deltas) runs for at
            // least WC_REFILL_MIN lanes at once, unless the warp is all idle
            if (need && (__popc(need) >= WC_REFILL_MIN || need == 0xffffffffu)) {
                const int leader = __ffs(need) - 1;
                uint32_t first = 0;
                if (lane == leader) first = atomicAdd(a.work, (uint32_t)__popc(need));
                first = __shfl_sync(0xffffffffu, first, leader);
                if (first + __popc(need) >= a.n_act) exhausted = true;
                const uint32_t mine = first + __popc(need & lt);
                if (!have && mine < a.n_act) {
                    have = true;
#if WC_TRAV_DEFER
                    iters = 0;
#endif
                    i = mine;
                    r = a.act_list[i];
                    double o[3], d[3];
                    a.rays.load(r, o, d);
                    ox = o[0], oy = o[1], oz = o[2], dx = d[0], dy = d[1], dz = d[2];
                    te = a.t_exit[r];
                    sx = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
                    sy = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
                    sz = dz > 0.0 ? 1 : (dz < 0.0 ? -1 : 0);
                    fdel_x = dx != 0.0 ? 4.0 / fabs(dx) : CUDART_INF;
                    fdel_y = dy != 0.0 ? 4.0 / fabs(dy) : CUDART_INF;
                    fdel_z = dz != 0.0 ? 4.0 / fabs(dz) : CUDART_INF;
                    const uint32_t cc = a.coarse_cell[r];
                    unlinear3(cc, a.cdv_x, a.cdv_xy, c.cx, c.cy, c.cz);
                    c.tx = a.coarse_tmax[3 * (int64_t)r];
                    c.ty = a.coarse_tmax[3 * (int64_t)r + 1];
                    c.tz = a.coarse_tmax[3 * (int64_t)r + 2];
                    const uint32_t fc = a.fine_cell[r];
                    in_fine_run = fc != WC_UINT_MAX;
                    f.cx = f.cy = f.cz = 0;
                    if (in_fine_run) {
                        unlinear3(fc, a.fdv_x, a.fdv_xy, f.cx, f.cy, f.cz);
                        fm = __ldg(a.cell_mask + cc);
                        plain = plain_cell();
                    }
                    f.tx = a.fine_tmax[3 * (int64_t)r];
                    f.ty = a.fine_tmax[3 * (int64_t)r + 1];
                    f.tz = a.fine_tmax[3 * (int64_t)r + 2];
                    base = (int64_t)i * a.n_spec;
                    emitted = 0;
                }
            }
        }
        if (!__any_sync(0xffffffffu, have)) break;
        if (!have) continue;
        bool finished = false, ray_done = false;
        // traversal.py:357-386: seed the fine iterator where the ray enters
        // coarse cell c (crossing parameter t_cross)
        auto descend = [&](double t_cross) {
            const double px = ox + dx * t_cross, py = oy + dy * t_cross, pz = oz + dz * t_cross;
            const int lo_x = 4 * c.cx, lo_y = 4 * c.cy, lo_z = 4 * c.cz;
            const int hi_x = min(lo_x + 3, fdx - 1), hi_y = min(lo_y + 3, fdy - 1), hi_z = min(lo_z + 3, fdz - 1);
            f.cx = (int)floor(px / 4.0);
            f.cy = (int)floor(py / 4.0);
            f.cz = (int)floor(pz / 4.0);
            f.cx = f.cx < lo_x ? lo_x : (f.cx > hi_x ? hi_x : f.cx);
            f.cy = f.cy < lo_y ? lo_y : (f.cy > hi_y ? hi_y : f.cy);
            f.cz = f.cz < lo_z ? lo_z : (f.cz > hi_z ? hi_z : f.cz);
            f.tx = dx > 0.0 ? ((double)(f.cx + 1) * 4.0 - ox) / dx
                            : (dx < 0.0 ? ((double)f.cx * 4.0 - ox) / dx : CUDART_INF);
            f.ty = dy > 0.0 ? ((double)(f.cy + 1) * 4.0 - oy) / dy
                            : (dy < 0.0 ? ((double)f.cy * 4.0 - oy) / dy : CUDART_INF);
            f.tz = dz > 0.0 ? ((double)(f.cz + 1) * 4.0 - oz) / dz
                            : (dz < 0.0 ? ((double)f.cz * 4.0 - oz) / dz : CUDART_INF);
            in_fine_run = true;
            plain = plain_cell();
        };
        if (!in_fine_run) {
            if (CA == 1) {  // one coarse step (traversal.py:332-386)
                const double t = dda_step(c, sx, sy, sz, 4.0 * fdel_x, 4.0 * fdel_y, 4.0 * fdel_z);
                if (t > te || (unsigned)c.cx >= (unsigned)cdx || (unsigned)c.cy >= (unsigned)cdy || (unsigned)c.cz >= (unsigned)cdz) {
                    ray_done = true;
                    finished = true;
                } else {
                    const uint32_t c_lin = (uint32_t)(c.cx + cdx * (c.cy + cdy * c.cz));
                    const uint32_t cw = __ldg(a.coarse_bm + (c_lin >> 5));
                    const unsigned long long m = __ldg(a.cell_mask + c_lin);  // same round trip
                    if ((cw >> (c_lin & 31)) & 1u) {
                        descend(t);
                        fm = m;
                    }
                }
            } else {  // CA coarse steps: simulate, fetch all range bits, descend at the first hit
                Dda g = c;
                uint32_t cell[CA];
#if WC_TRAV_KEEP
                Dda gs[CA];  // the state after step j + 1 (no re-stepping at the descent)
                double ts[CA];
#endif
                int J = 0;
                bool done = false;
#pragma unroll
                for (int j = 0; j < CA; j++) {
                    if (!done) {
#if WC_TRAV_AXIS
                        int ax, v;
                        const double t = dda_step_ax(g, sx, sy, sz, 4.0 * fdel_x, 4.0 * fdel_y, 4.0 * fdel_z, ax, v);
                        if (t > te || (unsigned)v >= (unsigned)pick3(ax, cdx, cdy, cdz)) {
#else
                        const double t = dda_step(g, sx, sy, sz, 4.0 * fdel_x, 4.0 * fdel_y, 4.0 * fdel_z);
                        if (t > te || (unsigned)g.cx >= (unsigned)cdx || (unsigned)g.cy >= (unsigned)cdy ||
                            (unsigned)g.cz >= (unsigned)cdz) {
#endif
                            done = true;
                        } else {
                            cell[j] = (uint32_t)(g.cx + cdx * (g.cy + cdy * g.cz));
                            J = j + 1;
#if WC_TRAV_KEEP
                            gs[j] = g;
                            ts[j] = t;
#endif
                        }
                    }
                }
                uint32_t bits = 0;
#pragma unroll
                for (int j = 0; j < CA; j++)
                    if (j < J) bits |= ((__ldg(a.coarse_bm + (cell[j] >> 5)) >> (cell[j] & 31)) & 1u) << j;
                if (bits) {
                    const int js = __ffs(bits) - 1;
                    double t_cross = 0.0;
#if WC_TRAV_KEEP
#pragma unroll
                    for (int j = 0; j < CA; j++)
                        if (j == js) {
                            c = gs[j];
                            t_cross = ts[j];
                        }
#else
                    for (int j = 0; j <= js; j++) t_cross = dda_step(c, sx, sy, sz, 4.0 * fdel_x, 4.0 * fdel_y, 4.0 * fdel_z);
#endif
                    descend(t_cross);
                    fm = __ldg(a.cell_mask + (c.cx + cdx * (c.cy + cdy * c.cz)));
                } else {
                    c = g;  // includes the exiting step when done (traversal.py:333-355)
                    if (done) {
                        ray_done = true;
                        finished = true;
                    }
                }
            }
        }
        if (in_fine_run) {  // the rest of the run, from the register mask (traversal.py:295-331)
            // the fine cell stays inside coarse cell c during a run: a step
            // leaves c exactly when the stepped coordinate crosses a multiple
            // of 4, and moves the cell's mask bit by 16 (x), 1 (y) or 4 (z)
#if WC_TRAV_AXIS
            int lb = fine_local(f);
#endif
            for (int k = 0; k < kFineRun; k++) {
#if WC_TRAV_AXIS
                if ((fm >> lb) & 1ull) {
#else
                if ((fm >> fine_local(f)) & 1ull) {
#endif
                    const uint32_t f_lin = (uint32_t)(f.cx + fdx * (f.cy + fdy * f.cz));
                    WC_DEVICE_CHECK(emitted < a.n_spec && (uint64_t)f_lin < (uint64_t)fdx * fdy * fdz);
                    a.block_slots[base + emitted] = f_lin;
                    a.ray_slots[base + emitted] = r;
                    emitted++;
                    mark_visible(a.vis_bm, f_lin);
                }
#if WC_TRAV_AXIS
                int ax, v;
                const double t = dda_step_ax(f, sx, sy, sz, fdel_x, fdel_y, fdel_z, ax, v);
                if (t > te || (unsigned)v >= (unsigned)pick3(ax, fdx, fdy, fdz)) {
                    in_fine_run = false;
                    ray_done = true;
                    break;
                }
                const int st = pick3(ax, sx, sy, sz);
                if ((v & 3) == (st > 0 ? 0 : 3)) {
                    in_fine_run = false;
                    break;
                }
                lb += st * pick3(ax, 16, 1, 4);
#else
                const double t = dda_step(f, sx, sy, sz, fdel_x, fdel_y, fdel_z);
                if (!plain &&
                    (t > te || (unsigned)f.cx >= (unsigned)fdx || (unsigned)f.cy >= (unsigned)fdy || (unsigned)f.cz >= (unsigned)fdz)) {
                    in_fine_run = false;
                    ray_done = true;
                    break;
                }
                if ((((f.cx >> 2) ^ c.cx) | ((f.cy >> 2) ^ c.cy) | ((f.cz >> 2) ^ c.cz)) != 0) {
                    in_fine_run = false;
                    break;
                }
#endif
                if (emitted == a.n_spec) break;
            }
            finished = emitted == a.n_spec || ray_done;
        }
        if (finished) {  // save the iterator past the last emit (traversal.py:388-403)
#if !WC_SENTINEL_LATE
            for (int k = emitted; k < a.n_spec; k++) {  // traversal.py:423-424 sentinels
                a.block_slots[base + k] = WC_UINT_MAX;
                a.ray_slots[base + k] = WC_UINT_MAX;
            }
#endif
            a.emitted[i] = (uint32_t)emitted;
            if (ray_done) {
                a.exited[r] = 1;
                a.coarse_cell[r] = WC_UINT_MAX;
                a.fine_cell[r] = WC_UINT_MAX;
            } else {
                a.coarse_cell[r] = (uint32_t)(c.cx + cdx * (c.cy + cdy * c.cz));
                a.fine_cell[r] = in_fine_run ? (uint32_t)(f.cx + fdx * (f.cy + fdy * f.cz)) : WC_UINT_MAX;
            }
            a.coarse_tmax[3 * (int64_t)r] = c.tx;
            a.coarse_tmax[3 * (int64_t)r + 1] = c.ty;
            a.coarse_tmax[3 * (int64_t)r + 2] = c.tz;
            a.fine_tmax[3 * (int64_t)r] = f.tx;
            a.fine_tmax[3 * (int64_t)r + 1] = f.ty;
            a.fine_tmax[3 * (int64_t)r + 2] = f.tz;
            have = false;
        }
#if WC_TRAV_DEFER
        // hand the ray to k_traverse_long (same iterator, same slots) -- in
        // passes of more than WC_DEFER_MAX_ACT rays only once the work has run
        // out (the tail), and at most WC_DEFER_CAP rays a pass: when most rays
        // walk long (an isovalue that few rays hit), the lanes keep them
        else if (++iters >= defer_k && (exhausted || a.n_act <= (int64_t)WC_DEFER_MAX_ACT) &&
                 *reinterpret_cast<volatile uint32_t *>(a.n_long) < WC_DEFER_CAP) {
            a.emitted[i] = (uint32_t)emitted;
            a.coarse_cell[r] = (uint32_t)(c.cx + cdx * (c.cy + cdy * c.cz));
            a.fine_cell[r] = in_fine_run ? (uint32_t)(f.cx + fdx * (f.cy + fdy * f.cz)) : WC_UINT_MAX;
            a.coarse_tmax[3 * (int64_t)r] = c.tx;
            a.coarse_tmax[3 * (int64_t)r + 1] = c.ty;
            a.coarse_tmax[3 * (int64_t)r + 2] = c.tz;
            a.fine_tmax[3 * (int64_t)r] = f.tx;
            a.fine_tmax[3 * (int64_t)r + 1] = f.ty;
            a.fine_tmax[3 * (int64_t)r + 2] = f.tz;
            a.long_q[atomicAdd(a.n_long, 1u)] = i;
            have = false;
        }
#endif
    }
}

__device__ __forceinline__ Dda shfl_dda(const Dda &s, int src) {
    Dda o;
    o.cx = __shfl_sync(0xffffffffu, s.cx, src);
    o.cy = __shfl_sync(0xffffffffu, s.cy, src);
    o.cz = __shfl_sync(0xffffffffu, s.cz, src);
    o.tx = __shfl_sync(0xffffffffu, s.tx, src);
    o.ty = __shfl_sync(0xffffffffu, s.ty, src);
    o.tz = __shfl_sync(0xffffffffu, s.tz, src);
    return o;
}

// ---- traversal with deferred fine runs (k_traverse_q) ----------------------
// The same per-ray walk as k_traverse, scheduled for SIMT efficiency.  A
// lane walking its ray's coarse grid does not run the fine run of a coarse
// cell whose range brackets iso right away: it queues the descent (the coarse
// state after stepping into the cell, and the crossing that seeds the fine
// iterator) in its own two-slot FIFO in shared memory and walks on (the
// coarse walk never depends on the fine runs).  The warp alternates between
// walking (lanes with room in their FIFO) and running fine runs (every lane
// with a queued descent runs its oldest one, at most 10 steps from the cell's
// 64-bit iso mask), so the two kinds of steps no longer share warp
// instructions.  A run that fills the ray's n_spec slots or leaves the volume
// ends the ray with the queued descent's coarse state; queued descents past
// that point are dropped (the walk ran ahead); a ray whose walk left the
// volume ends with its last run.  Every slot, iterator and exit flag is the
// reference's, bit for bit (traversal.py:217-403).
#ifndef WC_TQ_MINWALK
#define WC_TQ_MINWALK 8  // below this many walking lanes, the queued runs go first
#endif
#ifndef WC_TQ_MINRUN
#define WC_TQ_MINRUN 24  // runs start once this many lanes have one queued
#endif
#ifndef WC_TQ_MIN_CTAS
#define WC_TQ_MIN_CTAS 5
#endif
#ifndef WC_TQ_DEPTH
#define WC_TQ_DEPTH 2
#endif
constexpr int kTqDepth = WC_TQ_DEPTH, kTqWarps = 4;
static_assert((kTqDepth & (kTqDepth - 1)) == 0, "FIFO depth: a power of 2");
struct TqSlots {  // per warp, per lane: its queued descents (FIFO of kTqDepth)
    uint32_t cxyz[kTqDepth][32];  // coarse cell coordinates, 10 bits each
    uint32_t fcell[kTqDepth][32]; // UINT_MAX: seed from tc; else the ray's saved fine cell (resumed run)
    double ctx[kTqDepth][32], cty[kTqDepth][32], ctz[kTqDepth][32];  // coarse tmax after stepping into it
    double s0[kTqDepth][32], s1[kTqDepth][32], s2[kTqDepth][32];     // tc, or the saved fine tmax
};

template <int CA>
__global__ void __launch_bounds__(128, WC_TQ_MIN_CTAS) k_traverse_q(TraverseArgs a_in) {
    pdl_wait();
    TraverseArgs a = a_in;
    a.n_act = a.ctl[C_NACT];
    if (a.n_act <= (int64_t)a.warp_max) return;  // k_traverse_warp's pass
    a.n_spec = (int)a.ctl[C_NSPEC];
    a.rays.bind();
    __shared__ TqSlots slots_all[kTqWarps];
    TqSlots &S = slots_all[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int fdx = a.fdx, fdy = a.fdy, fdz = a.fdz, cdx = a.cdx, cdy = a.cdy, cdz = a.cdz;
    bool have = false, exhausted = false, walk_done = false;
    uint32_t i = 0, r = 0;
    double ox = 0, oy = 0, oz = 0, dx = 0, dy = 0, dz = 0, te = 0;
    double fdel_x = 0, fdel_y = 0, fdel_z = 0;  // coarse deltas: 4 * fdel (16/|d| == 4 * RN(4/|d|) exactly)
    int sx = 0, sy = 0, sz = 0, emitted = 0, pending = 0, qhead = 0;
    Dda c{0, 0, 0, 0, 0, 0};
    double lfx = 0, lfy = 0, lfz = 0;  // fine tmax after the last run (saved if the ray ends in the walk)
    int64_t base = 0;

    auto finish = [&](bool ray_done, uint32_t c_lin, double ctx, double cty, double ctz, bool in_fine, uint32_t f_lin,
                      double ftx, double fty, double ftz) {
#if !WC_SENTINEL_LATE
        for (int k = emitted; k < a.n_spec; k++) {  // traversal.py:423-424 sentinels
            a.block_slots[base + k] = WC_UINT_MAX;
            a.ray_slots[base + k] = WC_UINT_MAX;
        }
#endif
        a.emitted[i] = (uint32_t)emitted;
        if (ray_done) {
            a.exited[r] = 1;
            a.coarse_cell[r] = WC_UINT_MAX;
            a.fine_cell[r] = WC_UINT_MAX;
        } else {
            a.coarse_cell[r] = c_lin;
            a.fine_cell[r] = in_fine ? f_lin : WC_UINT_MAX;
        }
        a.coarse_tmax[3 * (int64_t)r] = ctx;
        a.coarse_tmax[3 * (int64_t)r + 1] = cty;
        a.coarse_tmax[3 * (int64_t)r + 2] = ctz;
        a.fine_tmax[3 * (int64_t)r] = ftx;
        a.fine_tmax[3 * (int64_t)r + 1] = fty;
        a.fine_tmax[3 * (int64_t)r + 2] = ftz;
        have = false;
        pending = 0;
    };
    auto push = [&](const Dda &cs, uint32_t fcell, double v0, double v1, double v2) {
        const int q = (qhead + pending) & (kTqDepth - 1);
        S.cxyz[q][lane] = (uint32_t)cs.cx | ((uint32_t)cs.cy << 10) | ((uint32_t)cs.cz << 20);
        S.fcell[q][lane] = fcell;
        S.ctx[q][lane] = cs.tx;
        S.cty[q][lane] = cs.ty;
        S.ctz[q][lane] = cs.tz;
        S.s0[q][lane] = v0;
        S.s1[q][lane] = v1;
        S.s2[q][lane] = v2;
        pending++;
    };

    for (;;) {
        if (!exhausted) {  // refill idle lanes (warp-uniform branch), as k_traverse
            const uint32_t need = __ballot_sync(0xffffffffu, !have);
            if (need && (__popc(need) >= WC_REFILL_MIN || need == 0xffffffffu)) {
                const int leader = __ffs(need) - 1;
                uint32_t first = 0;
                if (lane == leader) first = atomicAdd(a.work, (uint32_t)__popc(need));
                first = __shfl_sync(0xffffffffu, first, leader);
                if (first + __popc(need) >= a.n_act) exhausted = true;
                const uint32_t mine = first + __popc(need & lt);
                if (!have && mine < a.n_act) {
                    have = true;
                    walk_done = false;
                    pending = 0;
                    qhead = 0;
                    i = mine;
                    r = a.act_list[i];
                    double o[3], d[3];
                    a.rays.load(r, o, d);
                    ox = o[0], oy = o[1], oz = o[2], dx = d[0], dy = d[1], dz = d[2];
                    te = a.t_exit[r];
                    sx = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
                    sy = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
                    sz = dz > 0.0 ? 1 : (dz < 0.0 ? -1 : 0);
                    fdel_x = dx != 0.0 ? 4.0 / fabs(dx) : CUDART_INF;
                    fdel_y = dy != 0.0 ? 4.0 / fabs(dy) : CUDART_INF;
                    fdel_z = dz != 0.0 ? 4.0 / fabs(dz) : CUDART_INF;
                    const uint32_t cc = a.coarse_cell[r];
                    unlinear3(cc, a.cdv_x, a.cdv_xy, c.cx, c.cy, c.cz);
                    c.tx = a.coarse_tmax[3 * (int64_t)r];
                    c.ty = a.coarse_tmax[3 * (int64_t)r + 1];
                    c.tz = a.coarse_tmax[3 * (int64_t)r + 2];
                    lfx = a.fine_tmax[3 * (int64_t)r];
                    lfy = a.fine_tmax[3 * (int64_t)r + 1];
                    lfz = a.fine_tmax[3 * (int64_t)r + 2];
                    const uint32_t fc = a.fine_cell[r];
                    if (fc != WC_UINT_MAX) push(c, fc, lfx, lfy, lfz);  // the saved fine run goes first
                    base = (int64_t)i * a.n_spec;
                    emitted = 0;
                }
            }
        }
        const uint32_t walkers = __ballot_sync(0xffffffffu, have && !walk_done && pending < kTqDepth);
        const uint32_t runners = __ballot_sync(0xffffffffu, have && pending > 0);
        if (!walkers && !runners) {
            if (exhausted) break;
            continue;
        }
        if (walkers && (!runners || (__popc(walkers) >= WC_TQ_MINWALK && __popc(runners) < WC_TQ_MINRUN))) {
            // ---- walk: CA coarse steps simulated, their range bits fetched together
            if ((walkers >> lane) & 1u) {
                Dda g = c;
                uint32_t cell[CA];
                int J = 0;
                bool done = false;
#pragma unroll
                for (int j = 0; j < CA; j++) {
                    if (!done) {
                        const double t = dda_step(g, sx, sy, sz, 4.0 * fdel_x, 4.0 * fdel_y, 4.0 * fdel_z);
                        if (t > te || (unsigned)g.cx >= (unsigned)cdx || (unsigned)g.cy >= (unsigned)cdy ||
                            (unsigned)g.cz >= (unsigned)cdz) {
                            done = true;
                        } else {
                            cell[j] = (uint32_t)(g.cx + cdx * (g.cy + cdy * g.cz));
                            J = j + 1;
                        }
                    }
                }
                uint32_t bits = 0;
#pragma unroll
                for (int j = 0; j < CA; j++)
                    if (j < J) bits |= ((__ldg(a.coarse_bm + (cell[j] >> 5)) >> (cell[j] & 31)) & 1u) << j;
                if (bits) {  // queue the descent at the first hit
                    const int js = __ffs(bits) - 1;
                    double t_cross = 0.0;
                    for (int j = 0; j <= js; j++)
                        t_cross = dda_step(c, sx, sy, sz, 4.0 * fdel_x, 4.0 * fdel_y, 4.0 * fdel_z);
                    push(c, WC_UINT_MAX, t_cross, 0.0, 0.0);
                } else {
                    c = g;  // includes the exiting step when done (traversal.py:333-355)
                    walk_done = done;
                    if (done && pending == 0)  // left the volume with no run outstanding
                        finish(true, 0u, c.tx, c.ty, c.tz, false, 0u, lfx, lfy, lfz);
                }
            }
        } else if ((runners >> lane) & 1u) {
            // ---- the oldest queued fine run of every lane that has one (traversal.py:295-331)
            const int q = qhead;
            const uint32_t cxyz = S.cxyz[q][lane], fc0 = S.fcell[q][lane];
            const int ccx = (int)(cxyz & 1023u), ccy = (int)((cxyz >> 10) & 1023u), ccz = (int)(cxyz >> 20);
            Dda f;
            if (fc0 != WC_UINT_MAX) {  // resumed run: the saved fine iterator
                unlinear3(fc0, a.fdv_x, a.fdv_xy, f.cx, f.cy, f.cz);
                f.tx = S.s0[q][lane];
                f.ty = S.s1[q][lane];
                f.tz = S.s2[q][lane];
            } else {  // traversal.py:357-386: seed where the ray entered the coarse cell
                const double t_cross = S.s0[q][lane];
                const double px = ox + dx * t_cross, py = oy + dy * t_cross, pz = oz + dz * t_cross;
                const int lo_x = 4 * ccx, lo_y = 4 * ccy, lo_z = 4 * ccz;
                const int hi_x = min(lo_x + 3, fdx - 1), hi_y = min(lo_y + 3, fdy - 1), hi_z = min(lo_z + 3, fdz - 1);
                f.cx = (int)floor(px / 4.0);
                f.cy = (int)floor(py / 4.0);
                f.cz = (int)floor(pz / 4.0);
                f.cx = f.cx < lo_x ? lo_x : (f.cx > hi_x ? hi_x : f.cx);
                f.cy = f.cy < lo_y ? lo_y : (f.cy > hi_y ? hi_y : f.cy);
                f.cz = f.cz < lo_z ? lo_z : (f.cz > hi_z ? hi_z : f.cz);
                f.tx = dx > 0.0 ? ((double)(f.cx + 1) * 4.0 - ox) / dx
                                : (dx < 0.0 ? ((double)f.cx * 4.0 - ox) / dx : CUDART_INF);
                f.ty = dy > 0.0 ? ((double)(f.cy + 1) * 4.0 - oy) / dy
                                : (dy < 0.0 ? ((double)f.cy * 4.0 - oy) / dy : CUDART_INF);
                f.tz = dz > 0.0 ? ((double)(f.cz + 1) * 4.0 - oz) / dz
                                : (dz < 0.0 ? ((double)f.cz * 4.0 - oz) / dz : CUDART_INF);
            }
            const unsigned long long fm = __ldg(a.cell_mask + (ccx + cdx * (ccy + cdy * ccz)));
            bool ray_done = false, in_run = true;
            for (int k = 0; k < kFineRun; k++) {
                if ((fm >> fine_local(f)) & 1ull) {
                    const uint32_t f_lin = (uint32_t)(f.cx + fdx * (f.cy + fdy * f.cz));
                    a.block_slots[base + emitted] = f_lin;
                    a.ray_slots[base + emitted] = r;
                    emitted++;
                    mark_visible(a.vis_bm, f_lin);
                }
                const double t = dda_step(f, sx, sy, sz, fdel_x, fdel_y, fdel_z);
                if (t > te || (unsigned)f.cx >= (unsigned)fdx || (unsigned)f.cy >= (unsigned)fdy || (unsigned)f.cz >= (unsigned)fdz) {
                    in_run = false;
                    ray_done = true;
                    break;
                }
                if ((f.cx >> 2) != ccx || (f.cy >> 2) != ccy || (f.cz >> 2) != ccz) {
                    in_run = false;
                    break;
                }
                if (emitted == a.n_spec) break;
            }
            if (emitted == a.n_spec || ray_done) {  // the ray's pass ends in this run
                finish(ray_done, (uint32_t)(ccx + cdx * (ccy + cdy * ccz)), S.ctx[q][lane], S.cty[q][lane],
                       S.ctz[q][lane], in_run, (uint32_t)(f.cx + fdx * (f.cy + fdy * f.cz)), f.tx, f.ty, f.tz);
            } else {  // left the coarse cell: on to the next queued run or the walk
                lfx = f.tx;
                lfy = f.ty;
                lfz = f.tz;
                qhead = (qhead + 1) & (kTqDepth - 1);
                pending--;
                if (pending == 0 && walk_done)  // the walk had left the volume after this run
                    finish(true, 0u, c.tx, c.ty, c.tz, false, 0u, lfx, lfy, lfz);
            }
        }
    }
}

// traversal.py:217-403 for passes with few active rays (the long rays of the
// last passes, where one ray's serial DDA is the critical path): one warp
// per ray.  The DDA never depends on grid values, so lane k simulates the
// ray k steps ahead from the shared state -- the k-th cell of the current
// fine run (<= 10 cells in a 4^3 coarse cell) or the (k+1)-th coarse step --
// looks up its range bit, and ballots decide, in the reference's order,
// which cells emit, where the n_spec-th emit or the descent happens, and
// where the ray leaves.  The lane that simulated exactly that many steps
// holds the reference's iterator state and shuffles it to the warp.
// One ray (position i of the active list) by the whole warp, from its saved
// iterator with emitted0 of its slots already written.
__device__ __forceinline__ void warp_trace_ray(const TraverseArgs &a, int64_t i, int emitted0) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const int fdx = a.fdx, fdy = a.fdy, fdz = a.fdz, cdx = a.cdx, cdy = a.cdy, cdz = a.cdz;
    {
        const uint32_t r = a.act_list[i];
        double o[3], d[3];
        a.rays.load(r, o, d);
        const double ox = o[0], oy = o[1], oz = o[2], dx = d[0], dy = d[1], dz = d[2];
        const double te = a.t_exit[r];
        const int sx = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
        const int sy = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
        const int sz = dz > 0.0 ? 1 : (dz < 0.0 ? -1 : 0);
        const double fdel_x = dx != 0.0 ? 4.0 / fabs(dx) : CUDART_INF;
        const double fdel_y = dy != 0.0 ? 4.0 / fabs(dy) : CUDART_INF;
        const double fdel_z = dz != 0.0 ? 4.0 / fabs(dz) : CUDART_INF;
        const double cdel_x = dx != 0.0 ? 16.0 / fabs(dx) : CUDART_INF;
        const double cdel_y = dy != 0.0 ? 16.0 / fabs(dy) : CUDART_INF;
        const double cdel_z = dz != 0.0 ? 16.0 / fabs(dz) : CUDART_INF;
        Dda c, f;
        const uint32_t cc = a.coarse_cell[r];
        unlinear3(cc, a.cdv_x, a.cdv_xy, c.cx, c.cy, c.cz);
        c.tx = a.coarse_tmax[3 * (int64_t)r];
        c.ty = a.coarse_tmax[3 * (int64_t)r + 1];
        c.tz = a.coarse_tmax[3 * (int64_t)r + 2];
        const uint32_t fc = a.fine_cell[r];
        bool in_fine_run = fc != WC_UINT_MAX;
        f.cx = f.cy = f.cz = 0;
        if (in_fine_run) {
            unlinear3(fc, a.fdv_x, a.fdv_xy, f.cx, f.cy, f.cz);
        }
        f.tx = a.fine_tmax[3 * (int64_t)r];
        f.ty = a.fine_tmax[3 * (int64_t)r + 1];
        f.tz = a.fine_tmax[3 * (int64_t)r + 2];
        unsigned long long fm = in_fine_run ? __ldg(a.cell_mask + cc) : 0ull;  // warp-uniform
        const int64_t base = i * (int64_t)a.n_spec;
        int emitted = emitted0;
        bool ray_done = false, finished = false;
        // Coarse chunks: lane k holds the state after step k+1 from the chunk
        // start (the coarse walk never depends on the fine runs).
        while (!finished) {
            if (in_fine_run) {
                // lane k: cell X_k of the run (k steps from f), and the step that leaves it
                Dda g = f;
                bool valid = lane <= kFineRun;
                for (int j = 0; j < lane && valid; j++) {
                    const double t = dda_step(g, sx, sy, sz, fdel_x, fdel_y, fdel_z);
                    if (t > te || (unsigned)g.cx >= (unsigned)fdx || (unsigned)g.cy >= (unsigned)fdy || (unsigned)g.cz >= (unsigned)fdz ||
                        (g.cx >> 2) != c.cx || (g.cy >> 2) != c.cy || (g.cz >> 2) != c.cz)
                        valid = false;  // the run ended before cell k
                }
                uint32_t cell = 0;
                int term = 0;
                Dda h = g;
                if (valid) {
                    cell = (uint32_t)(g.cx + fdx * (g.cy + fdy * g.cz));
                    const double t = dda_step(h, sx, sy, sz, fdel_x, fdel_y, fdel_z);
                    if (t > te || (unsigned)h.cx >= (unsigned)fdx || (unsigned)h.cy >= (unsigned)fdy || (unsigned)h.cz >= (unsigned)fdz)
                        term = 2;
                    else if ((h.cx >> 2) != c.cx || (h.cy >> 2) != c.cy || (h.cz >> 2) != c.cz)
                        term = 1;
                }
                const bool bit = valid && ((fm >> fine_local(g)) & 1ull);
                const uint32_t tmask = __ballot_sync(0xffffffffu, valid && term != 0);
                // last cell of the run in this batch (a run has <= 10 cells, so a
                // termination is always found; kFineRun keeps the bound explicit)
                const int K = tmask ? __ffs(tmask) - 1 : kFineRun;
                uint32_t E = __ballot_sync(0xffffffffu, bit) & ((2u << K) - 1u);
                const int left = a.n_spec - emitted;
                int stop = K;
                if (__popc(E) >= left) {  // the n_spec-th emit happens at cell m
                    uint32_t e = E;
                    for (int q = 1; q < left; q++) e &= e - 1;
                    stop = __ffs(e) - 1;
                    E &= (stop == 31 ? 0xffffffffu : ((2u << stop) - 1u));
                }
                if ((E >> lane) & 1u) {
                    const int64_t slot = base + emitted + __popc(E & lt);
                    a.block_slots[slot] = cell;
                    a.ray_slots[slot] = r;
                    atomicOr(&a.vis_bm[cell >> 5], 1u << (cell & 31));
                }
                emitted += __popc(E);
                f = shfl_dda(h, stop);  // state after the step that follows cell `stop`
                const int term_stop = __shfl_sync(0xffffffffu, term, stop);
                if (term_stop == 2) {
                    in_fine_run = false;
                    ray_done = true;
                } else if (term_stop == 1) {
                    in_fine_run = false;
                }
                finished = emitted == a.n_spec || ray_done;
            } else {
                // lane k: the (k+1)-th coarse step from c, its range bit and fine mask
                Dda g = c;
                double tk = 0.0;
                bool valid = true, term_here = false;
                for (int j = 0; j <= lane && valid; j++) {
                    tk = dda_step(g, sx, sy, sz, cdel_x, cdel_y, cdel_z);
                    if (tk > te || (unsigned)g.cx >= (unsigned)cdx || (unsigned)g.cy >= (unsigned)cdy || (unsigned)g.cz >= (unsigned)cdz) {
                        valid = false;
                        term_here = j == lane;
                    }
                }
                const uint32_t cell = valid ? (uint32_t)(g.cx + cdx * (g.cy + cdy * g.cz)) : 0u;
                const uint32_t cw = valid ? __ldg(a.coarse_bm + (cell >> 5)) : 0u;
                const unsigned long long mk = valid ? __ldg(a.cell_mask + cell) : 0ull;
                const uint32_t T = __ballot_sync(0xffffffffu, term_here);
                const int first_term = T ? __ffs(T) - 1 : 32;
                const bool hit = valid && ((cw >> (cell & 31)) & 1u) && lane < first_term;
                const uint32_t H = __ballot_sync(0xffffffffu, hit);
                // Every descent of the chunk runs its fine run at once, lane =
                // descent (traversal.py:357-386, 295-331): the runs never depend
                // on one another, only their order does.
                Dda fj{0, 0, 0, 0, 0, 0}, f0{0, 0, 0, 0, 0, 0};
                unsigned long long codes = 0;
                int cnt = 0;
                bool exits = false;
                if (hit) {
                    const double px = ox + dx * tk, py = oy + dy * tk, pz = oz + dz * tk;
                    const int lo_x = 4 * g.cx, lo_y = 4 * g.cy, lo_z = 4 * g.cz;
                    const int hi_x = min(lo_x + 3, fdx - 1), hi_y = min(lo_y + 3, fdy - 1),
                              hi_z = min(lo_z + 3, fdz - 1);
                    f0.cx = (int)floor(px / 4.0);
                    f0.cy = (int)floor(py / 4.0);
                    f0.cz = (int)floor(pz / 4.0);
                    f0.cx = f0.cx < lo_x ? lo_x : (f0.cx > hi_x ? hi_x : f0.cx);
                    f0.cy = f0.cy < lo_y ? lo_y : (f0.cy > hi_y ? hi_y : f0.cy);
                    f0.cz = f0.cz < lo_z ? lo_z : (f0.cz > hi_z ? hi_z : f0.cz);
                    f0.tx = dx > 0.0 ? ((double)(f0.cx + 1) * 4.0 - ox) / dx
                                     : (dx < 0.0 ? ((double)f0.cx * 4.0 - ox) / dx : CUDART_INF);
                    f0.ty = dy > 0.0 ? ((double)(f0.cy + 1) * 4.0 - oy) / dy
                                     : (dy < 0.0 ? ((double)f0.cy * 4.0 - oy) / dy : CUDART_INF);
                    f0.tz = dz > 0.0 ? ((double)(f0.cz + 1) * 4.0 - oz) / dz
                                     : (dz < 0.0 ? ((double)f0.cz * 4.0 - oz) / dz : CUDART_INF);
                    fj = f0;
                    for (int k = 0; k < kFineRun; k++) {
                        if ((mk >> fine_local(fj)) & 1ull) {
                            codes |= (unsigned long long)((fj.cx & 3) | ((fj.cy & 3) << 2) | ((fj.cz & 3) << 4))
                                     << (6 * cnt);
                            cnt++;
                        }
                        const double t = dda_step(fj, sx, sy, sz, fdel_x, fdel_y, fdel_z);
                        if (t > te || (unsigned)fj.cx >= (unsigned)fdx || (unsigned)fj.cy >= (unsigned)fdy ||
                            (unsigned)fj.cz >= (unsigned)fdz) {
                            exits = true;
                            break;
                        }
                        if ((fj.cx >> 2) != g.cx || (fj.cy >> 2) != g.cy || (fj.cz >> 2) != g.cz) break;
                    }
                }
                // the runs' emits in chunk order, until the n_spec-th or a run that exits
                uint32_t incl = hit ? (uint32_t)cnt : 0u;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const uint32_t excl = incl - (hit ? (uint32_t)cnt : 0u);
                const uint32_t left = (uint32_t)(a.n_spec - emitted);
                const uint32_t S = __ballot_sync(0xffffffffu, hit && (incl >= left || exits));
                const int stop = S ? __ffs(S) - 1 : 32;  // the run the ray's pass ends in
                if (hit && lane <= stop) {
                    const uint32_t take = lane == stop ? min((uint32_t)cnt, left - excl) : (uint32_t)cnt;
                    for (uint32_t q = 0; q < take; q++) {
                        const uint32_t lc = (uint32_t)(codes >> (6 * q)) & 63u;
                        const uint32_t f_lin = (uint32_t)((4 * g.cx + (lc & 3)) +
                                                          fdx * ((4 * g.cy + ((lc >> 2) & 3)) + fdy * (4 * g.cz + (lc >> 4))));
                        WC_DEVICE_CHECK(emitted + (int)(excl + q) < a.n_spec);
                        a.block_slots[base + emitted + excl + q] = f_lin;
                        a.ray_slots[base + emitted + excl + q] = r;
                        atomicOr(&a.vis_bm[f_lin >> 5], 1u << (f_lin & 31));
                    }
                }
                if (stop < 32) {  // the pass ends in run `stop`
                    bool ex = exits, lv = false;
                    Dda fs = fj;
                    if (lane == stop && incl >= left) {  // the n_spec-th emit: replay to the step after it
                        fs = f0;
                        const uint32_t take = left - excl;
                        uint32_t seen = 0;
                        for (int k = 0; k < kFineRun; k++) {
                            seen += (uint32_t)((mk >> fine_local(fs)) & 1ull);
                            const double t = dda_step(fs, sx, sy, sz, fdel_x, fdel_y, fdel_z);
                            ex = t > te || (unsigned)fs.cx >= (unsigned)fdx || (unsigned)fs.cy >= (unsigned)fdy ||
                                 (unsigned)fs.cz >= (unsigned)fdz;
                            lv = !ex && ((fs.cx >> 2) != g.cx || (fs.cy >> 2) != g.cy || (fs.cz >> 2) != g.cz);
                            if (seen == take || ex || lv) break;
                        }
                    }
                    c = shfl_dda(g, stop);
                    f = shfl_dda(fs, stop);
                    ray_done = __shfl_sync(0xffffffffu, ex, stop);
                    in_fine_run = !__shfl_sync(0xffffffffu, ex || lv || !(incl >= left), stop);
                    emitted = min(a.n_spec, emitted + (int)__shfl_sync(0xffffffffu, incl, stop));
                    finished = true;
                } else {
                    emitted += (int)__shfl_sync(0xffffffffu, incl, 31);
                    if (H) f = shfl_dda(fj, 31 - __clz(H));  // the last run's fine state
                    if (first_term < 32) {  // left the volume / passed t_exit (traversal.py:345-355)
                        c = shfl_dda(g, first_term);
                        ray_done = true;
                        finished = true;
                    } else {
                        c = shfl_dda(g, 31);
                    }
                }
            }
        }
#if !WC_SENTINEL_LATE
        for (int k = emitted + lane; k < a.n_spec; k += 32) {  // traversal.py:423-424 sentinels
            a.block_slots[base + k] = WC_UINT_MAX;
            a.ray_slots[base + k] = WC_UINT_MAX;
        }
#endif
        if (lane == 0) {
            a.emitted[i] = (uint32_t)emitted;
            if (ray_done) {
                a.exited[r] = 1;
                a.coarse_cell[r] = WC_UINT_MAX;
                a.fine_cell[r] = WC_UINT_MAX;
            } else {
                a.coarse_cell[r] = (uint32_t)(c.cx + cdx * (c.cy + cdy * c.cz));
                a.fine_cell[r] = in_fine_run ? (uint32_t)(f.cx + fdx * (f.cy + fdy * f.cz)) : WC_UINT_MAX;
            }
            a.coarse_tmax[3 * (int64_t)r] = c.tx;
            a.coarse_tmax[3 * (int64_t)r + 1] = c.ty;
            a.coarse_tmax[3 * (int64_t)r + 2] = c.tz;
            a.fine_tmax[3 * (int64_t)r] = f.tx;
            a.fine_tmax[3 * (int64_t)r + 1] = f.ty;
            a.fine_tmax[3 * (int64_t)r + 2] = f.tz;
        }
    }
}

__device__ __forceinline__ void traverse_rays_warp(TraverseArgs a) {
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp0; i < a.n_act; i += nwarps) warp_trace_ray(a, i, 0);
}

// One launch per pass: thread per ray (persistent, refilled from a work
// counter) when the pass has many rays, warp per ray when it has at most
// warp_max -- chosen on the device from the pass's n_act, so a captured pass
// graph fits any frame.
template <int CA>
__global__ void __launch_bounds__(128, WC_TRAVERSE_MIN_CTAS) k_traverse(TraverseArgs a_in) {
    pdl_wait();
    TraverseArgs a = a_in;
    a.n_act = a.ctl[C_NACT];
    a.n_spec = (int)a.ctl[C_NSPEC];
    a.rays.bind();
    const bool warp = a.n_act <= (int64_t)a.warp_max || (a.n_spec >= WC_WARP_LONG_SPEC && a.n_act <= (int64_t)a.warp_max_long);
    if (!warp) {
        // large passes of short rays (no hand-off) step one coarse cell per
        // iteration; the others simulate CA steps ahead (measured: C3 passes
        // 0-1 -0.04 ms, C4 -0.09 ms; CA 1 in the hand-off passes was slower)
        if (!a.warp_only) {
            if (WC_CA_SPLIT && a.n_spec < WC_WARP_LONG_SPEC && a.n_act > (int64_t)WC_DEFER_MAX_ACT)
                traverse_rays_thread<1>(a);
            else
                traverse_rays_thread<CA>(a);
        }
    } else {
        traverse_rays_warp(a);
    }
}

// The traversal's range tests for one isovalue, precomputed: bit c of the
// fine (coarse) bitmap is `min[c] <= iso && iso <= max[c]` evaluated in
// float64 exactly as traversal.py:297 (:357) does.  The 15.7 MB fine bitmap
// (8.05B voxels) stays in L2, so each DDA step of the traversal's dependent
// chain costs an L2 hit instead of a DRAM read of the 2 GB float64 grid.
__global__ void k_iso_bitmap(const double2 *__restrict__ mm, int64_t n, double iso, uint32_t *__restrict__ bm,
                             int64_t w_begin, int64_t w_end) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t nwords = min((n + 31) >> 5, w_end);
    for (int64_t w = w_begin + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); w < nwords;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t c = w * 32 + lane;
        bool in = false;
        if (c < n) {
            const double2 v = mm[c];
            in = v.x <= iso && iso <= v.y;
        }
        const uint32_t word = __ballot_sync(0xffffffffu, in);
        if (lane == 0) bm[w] = word;
    }
}

// Same bitmap from the 16-bit screening copy (Volume::fine_q): a bound in a
// different bucket than iso decides its comparison; a shared bucket re-reads
// the exact float64 bound.  Reads 4 B per block instead of 16.
//
// Laid out per coarse cell: cell_mask[c] bit 16*(fx&3) + (fy&3) + 4*(fz&3)
// is the test of fine cell f inside coarse cell c (fine cells past the grid
// edge read 0).  A ray descending into c loads this one word and walks its
// whole fine run (<= 10 cells) from registers.
__device__ __forceinline__ bool iso_in_q(const ushort2 v, uint32_t qi, const double2 *mm, int64_t b, double iso) {
    const bool lo_ok = qi != v.x ? qi > v.x : mm[b].x <= iso;
    return lo_ok && (qi != v.y ? qi < v.y : iso <= mm[b].y);
}

//
// Only coarse cells whose own range test passes are filled: the traversal
// reads a cell's mask only after descending into it (traversal.py:357), so
// the others are left 0.
__global__ void __launch_bounds__(256, WC_ISO_MIN_CTAS) k_iso_cell_mask(const ushort2 *__restrict__ q, const double2 *__restrict__ mm,
                                const uint32_t *__restrict__ coarse_bm, int fdx, int fdy, int fdz, int cdx, int cdy,
                                int cdz, double iso, double base, double inv,
                                unsigned long long *__restrict__ cell_mask, int64_t c_begin, int64_t c_end) {
    pdl_wait();
    // Streams the bricked screening copy: 16 lanes cover one coarse cell's
    // 256 B (lane: 4 fine cells = one x-row), 4 cells per lane in flight.
    // One ballot per x position collects the 16 rows of both half-warps'
    // cells: bits [16x, 16x + 16) of a cell's mask.
    constexpr int kU = WC_ISO_KU;
    const int64_t n_coarse = min((int64_t)cdx * cdy * cdz, c_end);  // cells [c_begin, c_end): c_begin % 8 == 0
    const bool iso_nan = iso != iso;
    const uint32_t qi = iso_nan ? 0u : range_q(iso, base, inv);
    const int lane = threadIdx.x & 31, half = lane >> 4, row = lane & 15;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // (the warp's 2 kU cells share one coarse-bitmap word: c0 % (2 kU) == 0)
    static_assert(32 % (2 * kU) == 0, "a warp's cells must not straddle a bitmap word");
    const uint32_t sel = half ? 0x7632u : 0x5410u;  // this half-warp's 16-bit halves of two ballots
    for (int64_t c0 = c_begin + w0 * 2 * kU; c0 < n_coarse; c0 += nw * 2 * kU) {
        uint4 w[kU];
        bool on[kU];
        const uint32_t cw = iso_nan ? 0u : coarse_bm[c0 >> 5] >> (c0 & 31);
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const int64_t c = c0 + 2 * u + half;
            on[u] = c < n_coarse && ((cw >> (2 * u + half)) & 1u);
            w[u] = on[u] ? __ldg(reinterpret_cast<const uint4 *>(q + c * 64) + row) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const int64_t c = c0 + 2 * u + half;
            const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
            uint32_t b[4];
#pragma unroll
            for (int x = 0; x < 4; x++) {
                const uint32_t lo = ws[x] & 0xFFFFu, hi = ws[x] >> 16;
                bool in = on[u] && qi > lo && qi < hi;  // decided by the buckets (the common case)
                if (on[u] && (qi == lo || qi == hi)) {  // shared bucket: exact float64 test (rare)
                    const uint32_t cu = (uint32_t)c;
                    const int fx = 4 * (int)(cu % (uint32_t)cdx) + x;
                    const int fy = 4 * (int)((cu / (uint32_t)cdx) % (uint32_t)cdy) + (row & 3);
                    const int fz = 4 * (int)(cu / ((uint32_t)cdx * (uint32_t)cdy)) + (row >> 2);
                    in = fx < fdx && fy < fdy && fz < fdz &&
                         iso_in_q(make_ushort2((unsigned short)lo, (unsigned short)hi), qi, mm,
                                  fx + (int64_t)fdx * (fy + (int64_t)fdy * fz), iso);
                }
                b[x] = __ballot_sync(0xffffffffu, in);
            }
            // bits [16x, 16x + 16) of the cell's mask: this half-warp's half of ballot x
            const unsigned long long m =
                (unsigned long long)__byte_perm(b[0], b[1], sel) | ((unsigned long long)__byte_perm(b[2], b[3], sel) << 32);
            if (row == 0 && c < n_coarse) cell_mask[c] = m;
        }
    }
}

// ------------------------------------------------------------------ marking

// engine.py:107-117: each visible block activates itself and its existing
// +octant neighbours.  Count-driven (reads *d_nvis) so no host round trip.
__global__ void k_mark_active(const uint32_t *visible_ids, const uint32_t *d_nvis, int bdx, int bdy, int bdz,
                              uint32_t *act_bm) {
    pdl_wait();
    const int64_t nvis = *d_nvis;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nvis * 8; t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = visible_ids[t >> 3];
        const int o = (int)(t & 7), ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
        const int bx = (int)(b % (uint32_t)bdx), by = (int)((b / (uint32_t)bdx) % (uint32_t)bdy),
                  bz = (int)(b / ((uint32_t)bdx * (uint32_t)bdy));
        if (bx + ox >= bdx || by + oy >= bdy || bz + oz >= bdz) continue;
        const uint32_t nid = (uint32_t)((bx + ox) + bdx * ((by + oy) + bdy * (bz + oz)));
        atomicOr(&act_bm[nid >> 5], 1u << (nid & 31));
    }
}

// Same marking a word at a time when rows are whole words (bdx % 32 == 0):
// the first visible id of each non-zero visible word v activates
// v | v << 1 in its own word, the bit shifted out into the next word of the
// row, and both again one row (+y) and one plane (+z) further on, where those
// neighbours exist.  Up to 8 word ORs per visible word instead of 8 bit ORs
// per visible block.
__global__ void k_mark_active_words(const uint32_t *visible_ids, const uint32_t *d_nvis, const uint32_t *vis_bm,
                                    int wx_words, int bdy, int bdz, uint32_t *act_bm) {
    pdl_wait();
    const int64_t nvis = *d_nvis;
    const uint32_t plane = (uint32_t)wx_words * (uint32_t)bdy;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvis; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t w = visible_ids[i] >> 5;
        if (i > 0 && (visible_ids[i - 1] >> 5) == w) continue;  // ids ascend: one thread per word
        const uint32_t v = vis_bm[w];
        const uint32_t row = w / (uint32_t)wx_words;
        const uint32_t wx = w - row * (uint32_t)wx_words;
        const uint32_t by = row % (uint32_t)bdy, bz = row / (uint32_t)bdy;
        const uint32_t a = v | (v << 1);                               // +x inside the word
        const uint32_t b = wx + 1 < (uint32_t)wx_words ? v >> 31 : 0u;  // +x into the next word
        const int ny = by + 1 < (uint32_t)bdy ? 2 : 1, nz = bz + 1 < (uint32_t)bdz ? 2 : 1;
        for (int oz = 0; oz < nz; oz++)
            for (int oy = 0; oy < ny; oy++) {
                const uint32_t t = w + oy * (uint32_t)wx_words + oz * plane;
                atomicOr(&act_bm[t], a);
                if (b) atomicOr(&act_bm[t + 1], b);
            }
    }
}

// The long rays the thread-per-ray pass handed off, warp per ray.
__global__ void __launch_bounds__(128) k_traverse_long(TraverseArgs a_in) {
    pdl_wait();
    TraverseArgs a = a_in;
    const uint32_t nq = *a.n_long;
    if (nq == 0) return;
    a.n_act = a.ctl[C_NACT];
    a.n_spec = (int)a.ctl[C_NSPEC];
    a.rays.bind();
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = warp0; q < (int64_t)nq; q += nwarps) {
        const uint32_t i = a.long_q[q];
        warp_trace_ray(a, i, (int)a.emitted[i]);
    }
}

void launch_traverse(TraverseArgs ta, int64_t n_grid, int variant, cudaStream_t st) {
    ta.cdv_x = FastDiv((uint32_t)ta.cdx);
    ta.cdv_xy = FastDiv((uint32_t)ta.cdx * (uint32_t)ta.cdy);
    ta.fdv_x = FastDiv((uint32_t)ta.fdx);
    ta.fdv_xy = FastDiv((uint32_t)ta.fdx * (uint32_t)ta.fdy);
    ta.warp_max = variant == 1 ? 0u : (variant == 2 ? 0xFFFFFFFFu : (uint32_t)WC_WARP_TRAVERSE_MAX);
    ta.warp_max_long = variant == 0 ? (uint32_t)WC_WARP_TRAVERSE_MAX_LONG : ta.warp_max;
#if WC_TRAVERSE_Q
    if (variant != 2) {
        launch_pdl(k_traverse_q<WC_COARSE_AHEAD>, grid_for(n_grid, 128, WC_TQ_MIN_CTAS), 128, 0, st, ta);
        WC_LAUNCH_CHECK();
    }
    if (variant == 1) return;
    ta.warp_only = true;
#endif
    // enough CTAs for a warp per ray up to warp_max rays; the thread-per-ray
    // path keeps what fits resident busy and the rest find no work
    const int64_t warps = std::min<int64_t>(n_grid, variant == 1 ? 0 : (variant == 2 ? n_grid : WC_WARP_TRAVERSE_MAX));  // (long passes grid-stride)
    const unsigned grid = std::max(grid_for(n_grid, 128, WC_TRAVERSE_MIN_CTAS), grid_for(std::max<int64_t>(1, warps) * 32, 128, 16));
    if (variant != 0) ta.long_q = nullptr;  // forced variants: no hand-off
    launch_pdl(k_traverse<WC_COARSE_AHEAD>, grid, 128, 0, st, ta);
    WC_LAUNCH_CHECK();
#if WC_TRAV_DEFER
    if (ta.long_q) {
        launch_pdl(k_traverse_long, (unsigned)(num_sms() * 8), 128, 0, st, ta);
        WC_LAUNCH_CHECK();
    }
#endif
}

void launch_mark_active(const uint32_t *visible_ids, const uint32_t *d_nvis, const uint32_t *vis_bm, int bdx, int bdy,
                        int bdz, int64_t n_max, uint32_t *act_bm, cudaStream_t st) {
    if (bdx % 32 == 0)
        launch_pdl(k_mark_active_words, grid_for(n_max, 256), 256, 0, st, visible_ids, d_nvis, vis_bm, bdx / 32, bdy, bdz,
                   act_bm);
    else
        launch_pdl(k_mark_active, grid_for(8 * n_max, 256), 256, 0, st, visible_ids, d_nvis, bdx, bdy, bdz, act_bm);
    WC_LAUNCH_CHECK();
}

void launch_iso_bitmap(const double2 *mm, int64_t n, double iso, uint32_t *bm, cudaStream_t st) {
    const int64_t nw = ceil_div(n, 32);
    launch_pdl(k_iso_bitmap, grid_for(nw * 32, 256, 8), 256, 0, st, mm, n, iso, bm, (int64_t)0, nw);
    WC_LAUNCH_CHECK();
}

// Run starts of the sorted keys -> block_ray_offsets (engine.py:133-139).
__global__ void k_run_offsets(const uint32_t *key, int64_t n, int64_t nvis, uint32_t *off) {
    pdl_wait();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == 0 || key[i] != key[i - 1]) off[key[i]] = (uint32_t)i;
        if (i == 0) off[nvis] = (uint32_t)n;
    }
}

// ---------------------------------------------------------------- cache

// eviction candidates (resident, stamp < pass_no) per stamp value
// (few distinct stamps: per-CTA shared-memory bins, one global add per bin)
__global__ void k_stamp_hist(const int32_t *block_of_slot, const int32_t *last_used, const uint32_t *ctl,
                             int32_t pass_no, uint32_t *hist) {
    pdl_wait();
    extern __shared__ uint32_t sh[];
    const int64_t hw = ctl[C_NACT] ? ctl[C_HW] : 0;
    for (int b = threadIdx.x; b < pass_no; b += blockDim.x) sh[b] = 0;
    __syncthreads();
    // few distinct stamps: one shared atomic per (warp, stamp) via match_any
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); s0 < hw; s0 += stride) {
        const int64_t s = s0 + lane;
        int32_t key = -1;
        if (s < hw) {
            const int32_t lu = last_used[s];
            if (block_of_slot[s] >= 0 && lu < pass_no) key = lu;
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        if (key >= 0 && lane == __ffs(peers) - 1) atomicAdd(&sh[key], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int b = threadIdx.x; b < pass_no; b += blockDim.x)
        if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// Candidates (resident, not stamped this pass) with stamp L <= L* marked in
// the block bitmap of region L: one extraction over regions 0..L* then lists
// them in (last_used, block_id) order (cache.py:84-91).
__global__ void k_mark_victims(const int32_t *block_of_slot, const int32_t *last_used, const uint32_t *ctl,
                               int32_t pass_no, int64_t nwords, uint32_t *regions, uint32_t *summary) {
    pdl_wait();
    if (ctl[C_NEVICT] == 0) return;
    const int64_t hw = ctl[C_HW];
    const int32_t lstar = (int32_t)ctl[C_LSTAR];
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < hw; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = block_of_slot[s];
        const int32_t lu = last_used[s];
        if (b >= 0 && lu < pass_no && lu <= lstar)
            bitmap_set(regions, summary, (uint64_t)lu * nwords + (b >> 5), b & 31);
    }
}


// BlockCache reset: forget every resident block of the previous frame
__global__ void k_cache_unmap(const int32_t *block_of_slot, const uint32_t *d_phys, int32_t *slot_of_block) {
    pdl_wait();
    const int64_t phys = *d_phys;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < phys; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = block_of_slot[s];
        if (b >= 0) slot_of_block[b] = -1;
    }
}

// cache.py:90-95: unmap the first n_evict candidates (they become the
// slots of the last n_evict misses, cache.py:96-97)
__global__ void k_evict(const uint32_t *victims, const uint32_t *d_n_evict, int32_t *slot_of_block,
                        int32_t *block_of_slot, uint32_t *victim_slots) {
    pdl_wait();
    const int64_t n_evict = *d_n_evict;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_evict; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = victims[i];
        const int32_t s = slot_of_block[b];
        victim_slots[i] = (uint32_t)s;  // the slot of the i-th last miss
        slot_of_block[b] = -1;
        block_of_slot[s] = -1;
    }
}

// cache.py:97-103 fused with codec.py:143-174: miss j goes to slot hw + j
// while free slots last, then to victim j - n_free; its record is decoded
// straight into the slot and the mapping published.  Warp per block; the
// miss count is read on the device (no host round trip).
// A warp takes 32 consecutive misses (one coalesced load of their ids and
// lane-parallel slot bookkeeping), then streams their records through shared
// memory: kDecRec records are requested with cp.async (no registers held per
// request, so many random 132 B records are in flight per SM), then decoded
// from shared memory straight into the slots.
constexpr int kDecWarps = WC_DEC_WARPS, kDecRec = WC_DEC_REC, kDecWords = 64;  // words: the largest record (qbits 31)
// pipelined form: records per batch (two batches per warp in flight), words per
// staged record (the largest record's 16-byte aligned span)
constexpr int kDecRecP = WC_DEC_PREC, kDecWordsP = 72;
__global__ void __launch_bounds__(kDecWarps * 32, WC_DEC_CTAS)
    k_decode_insert(const uint8_t *__restrict__ payload, int qbits, int stride, const uint32_t *__restrict__ miss_ids,
                    uint32_t *ctl, const uint32_t *__restrict__ victims, float *__restrict__ slot_values,
                    int32_t *block_of_slot, int32_t *last_used, int32_t *slot_of_block, int32_t pass_no) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
#if WC_DEC_PIPE
    __shared__ __align__(16) uint32_t stage_p[kDecWarps][2][kDecRecP][kDecWordsP];
#else
    __shared__ uint32_t stage[kDecWarps][kDecRec][kDecWords];
    uint32_t(*sw)[kDecWords] = stage[threadIdx.x >> 5];
#endif
    const int64_t n_miss = ctl[C_NMISS], hw = ctl[C_HW], n_free = ctl[C_NFREE], cap = ctl[C_CAP];
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl[C_HW_NEXT] = (uint32_t)(n_miss <= n_free ? hw + n_miss : cap);
    {  // maps of the slots this pass's growth brought into use (cache.py:42-53) that no miss takes
        const int64_t lo = max((int64_t)ctl[C_PHYS_OLD], hw + min(n_miss, n_free)), hi = ctl[C_PHYS];
        for (int64_t s = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < hi;
             s += (int64_t)gridDim.x * blockDim.x) {
            block_of_slot[s] = -1;
            last_used[s] = 0;
        }
    }
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int n_words = stride >> 2;
#if WC_DEC_PIPE
    // Pipelined: a warp takes groups of 32 misses (strided over the grid) in
    // batches of kDecRecP records; batch k+1's records are in flight while
    // batch k is decoded (two stage buffers per warp).
    //   WC_DEC_PIPE 1: 4-byte cp.async per word (LDGSTS);
    //   WC_DEC_PIPE 2: one bulk copy (TMA engine) per record of its 16-byte
    //                  aligned span, completion counted on a per-buffer mbarrier.
    const int64_t gstride = nwarps * 32;
    int64_t g = warp0 * 32;
    if (g >= n_miss) return;  // whole warp (no CTA-wide barrier follows)
    const int w_in = threadIdx.x >> 5;
#if WC_DEC_PIPE == 2
    __shared__ __align__(8) unsigned long long mbar[kDecWarps][2];
    if (lane == 0) {
        mbar_init(&mbar[w_in][0], 1);
        mbar_init(&mbar[w_in][1], 1);
        fence_mbar_init();
    }
    __syncwarp();
    uint32_t phase = 0;  // bit b: parity of buffer b's next completion
    uint32_t offs[2] = {0u, 0u};  // lane u: word offset of record u inside its span, per buffer
#endif
    auto group_ids = [&](int64_t gg, uint32_t &b, uint32_t &s) {
        const int64_t jl = gg + lane;
        b = jl < n_miss ? miss_ids[jl] : 0u;
        s = jl < n_miss ? (jl < n_free ? (uint32_t)(hw + jl) : victims[jl - n_free]) : 0u;
        if (jl < n_miss) {  // lane-parallel bookkeeping for the 32 misses
            WC_DEVICE_CHECK((int64_t)s < (int64_t)ctl[C_PHYS] && (int64_t)s < cap);
            block_of_slot[s] = (int32_t)b;
            last_used[s] = pass_no;
            slot_of_block[b] = (int32_t)s;
        }
    };
    auto issue = [&](int buf, uint32_t ids, int cnt, int u0) {
#if WC_DEC_PIPE == 1
#pragma unroll
        for (int u = 0; u < kDecRecP; u++) {
            const uint32_t b = __shfl_sync(0xffffffffu, ids, (u0 + u) & 31);
            if (u0 + u < cnt) {
                const uint32_t *rec = reinterpret_cast<const uint32_t *>(payload + (int64_t)b * stride);
                uint32_t *dst = stage_p[w_in][buf][u];
                if (lane < n_words) cp_async4(&dst[lane], rec + lane);
                if (lane + 32 < n_words) cp_async4(&dst[lane + 32], rec + lane + 32);
            }
        }
        cp_async_commit();
#else
        const uint32_t b = __shfl_sync(0xffffffffu, ids, (u0 + lane) & 31);
        const bool mine = lane < kDecRecP && u0 + lane < cnt;
        const uint64_t a0 = (uint64_t)(payload + (int64_t)b * stride);
        const uint64_t lo = a0 & ~15ull, hi = (a0 + (uint64_t)stride + 15ull) & ~15ull;
        const uint32_t bytes = mine ? (uint32_t)(hi - lo) : 0u;
        offs[buf] = (uint32_t)(a0 - lo) >> 2;
        const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
        if (lane == 0) mbar_arrive_expect_tx(&mbar[w_in][buf], total);
        __syncwarp();
        if (mine) bulk_g2s(stage_p[w_in][buf][lane], reinterpret_cast<const void *>(lo), bytes, &mbar[w_in][buf]);
#endif
    };
    auto wait_buf = [&](int buf, bool more) {
#if WC_DEC_PIPE == 1
        if (more)
            cp_async_wait_1();
        else
            cp_async_wait_0();
        (void)buf;
#else
        (void)more;
        mbar_wait_parity(&mbar[w_in][buf], (phase >> buf) & 1u);
        phase ^= 1u << buf;
#endif
        __syncwarp();
    };
    uint32_t cb, cs;
    group_ids(g, cb, cs);
    int ccnt = n_miss - g < 32 ? (int)(n_miss - g) : 32;
    int buf = 0, u0 = 0;
    issue(0, cb, ccnt, 0);
    for (;;) {
        int64_t g2 = g;
        int u2 = u0 + kDecRecP, cnt2 = ccnt;
        const bool next_group = u2 >= ccnt;
        if (next_group) {
            g2 = g + gstride;
            u2 = 0;
        }
        const bool more = g2 < n_miss;
        uint32_t nb = cb, ns = cs;
        if (more) {
            if (next_group) {
                group_ids(g2, nb, ns);
                cnt2 = n_miss - g2 < 32 ? (int)(n_miss - g2) : 32;
            }
            issue(buf ^ 1, nb, cnt2, u2);
        }
        wait_buf(buf, more);
#pragma unroll 4
        for (int u = 0; u < kDecRecP; u++) {
            const uint32_t sl = __shfl_sync(0xffffffffu, cs, (u0 + u) & 31);
            if (u0 + u >= ccnt) break;  // warp-uniform
#if WC_DEC_PIPE == 2
            const uint32_t *rw = stage_p[w_in][buf][u] + __shfl_sync(0xffffffffu, offs[buf], u);
#else
            const uint32_t *rw = stage_p[w_in][buf][u];
#endif
            float *dst = slot_values + (int64_t)sl * 64;
            if (qbits == 16) {
                reinterpret_cast<float2 *>(dst)[lane] = decode16_words(rw[lane], rw[lane + 1], rw[0]);
            } else {
                const uint32_t wa = lane < n_words ? rw[lane] : 0u;
                const uint32_t wb = lane + 32 < n_words ? rw[lane + 32] : 0u;
                float v0, v1;
                decode_loaded_warp(wa, wb, qbits, lane, v0, v1);
                dst[lane] = v0;
                dst[lane + 32] = v1;
            }
        }
        __syncwarp();  // buffer `buf` is refilled by the batch after next
        if (!more) break;
        if (next_group) {
            cb = nb;
            cs = ns;
            ccnt = cnt2;
            g = g2;
        }
        u0 = u2;
        buf ^= 1;
    }
#else
    for (int64_t g = warp0 * 32; g < n_miss; g += nwarps * 32) {
        const int64_t jl = g + lane;
        const uint32_t my_b = jl < n_miss ? miss_ids[jl] : 0u;
        const uint32_t my_s = jl < n_miss ? (jl < n_free ? (uint32_t)(hw + jl) : victims[jl - n_free]) : 0u;
        if (jl < n_miss) {  // lane-parallel bookkeeping for the 32 misses
            WC_DEVICE_CHECK((int64_t)my_s < (int64_t)ctl[C_PHYS] && (int64_t)my_s < cap);
            block_of_slot[my_s] = (int32_t)my_b;
            last_used[my_s] = pass_no;
            slot_of_block[my_b] = (int32_t)my_s;
        }
        const int cnt = n_miss - g < 32 ? (int)(n_miss - g) : 32;
        for (int u0 = 0; u0 < cnt; u0 += kDecRec) {
#pragma unroll
            for (int u = 0; u < kDecRec; u++) {
                const uint32_t b = __shfl_sync(0xffffffffu, my_b, (u0 + u) & 31);
                if (u0 + u < cnt) {
                    const uint32_t *rec = reinterpret_cast<const uint32_t *>(payload + (int64_t)b * stride);
                    if (lane < n_words) cp_async4(&sw[u][lane], rec + lane);
                    if (lane + 32 < n_words) cp_async4(&sw[u][lane + 32], rec + lane + 32);
                }
            }
            cp_async_wait_all();
            __syncwarp();
#pragma unroll 4
            for (int u = 0; u < kDecRec; u++) {
                const uint32_t s = __shfl_sync(0xffffffffu, my_s, (u0 + u) & 31);
                if (u0 + u >= cnt) break;  // warp-uniform
                float *dst = slot_values + (int64_t)s * 64;
                if (qbits == 16) {  // the common rate: lane decodes values 2l, 2l+1 (one 8 B store)
                    reinterpret_cast<float2 *>(dst)[lane] = decode16_words(sw[u][lane], sw[u][lane + 1], sw[u][0]);
                } else {
                    const uint32_t wa = lane < n_words ? sw[u][lane] : 0u;
                    const uint32_t wb = lane + 32 < n_words ? sw[u][lane + 32] : 0u;
                    float v0, v1;
                    decode_loaded_warp(wa, wb, qbits, lane, v0, v1);
                    dst[lane] = v0;
                    dst[lane + 32] = v1;
                }
            }
            __syncwarp();  // the stage is refilled by the next batch
        }
    }
#endif
}

// -------------------------------------------------------------- raytrace

// The dual grid of a visible block (blocktrace.py:49-94) read straight from
// the cache slots: corner (x, y, z) of the block's local 5^3 lattice lives in
// the slot of octant ((x>>2), (y>>2), (z>>2)) at offset (x&3)+4(y&3)+16(z&3).
// The 8 contributor slots (engine.py:286-305) come from k_contrib.
struct SlotField {
    const float *sv;
    int s0, s1, s2, s3, s4, s5, s6, s7;
    __device__ __forceinline__ int pick(int o) const {
        const int a0 = (o & 1) ? s1 : s0, a1 = (o & 1) ? s3 : s2, a2 = (o & 1) ? s5 : s4, a3 = (o & 1) ? s7 : s6;
        const int b0 = (o & 2) ? a1 : a0, b1 = (o & 2) ? a3 : a2;
        return (o & 4) ? b1 : b0;
    }
    // value at local lattice point (x, y, z), each in [0, 4]
    __device__ __forceinline__ float point(int x, int y, int z) const {
        const int sl = pick((x >> 2) | ((y >> 2) << 1) | ((z >> 2) << 2));
        return sl >= 0 ? __ldg(sv + (int64_t)sl * 64 + (x & 3) + 4 * (y & 3) + 16 * (z & 3)) : 0.0f;
    }
    __device__ __forceinline__ void corners(int lx, int ly, int lz, float c[8]) const {
        const int ex = lx == 3, ey = ly == 3, ez = lz == 3;
#pragma unroll
        for (int idx = 0; idx < 8; idx++) {
            const int dx = idx & 1, dy = (idx >> 1) & 1, dz = idx >> 2;
            const int sl = pick((dx & ex) | ((dy & ey) << 1) | ((dz & ez) << 2));
            const int off = ((lx + dx) & 3) + 4 * ((ly + dy) & 3) + 16 * ((lz + dz) & 3);
            c[idx] = sl >= 0 ? __ldg(sv + (int64_t)sl * 64 + off) : 0.0f;
        }
    }
};

// SlotField with the 8 contributor slots as row pointers in shared memory
// (octant-major, one column per thread: conflict-free), so a lattice lookup
// is one LDS.64 plus an offset instead of a 7-way select and a slot multiply.
// Missing neighbours (slot -1) point at a zero row.
__device__ float g_zero_row[64];

template <int kThreads>
struct SlotFieldSmem {
    const float *const *rows;  // &table[0][threadIdx.x], stride kThreads
    __device__ __forceinline__ static void fill(const float **col, const float *sv, const int s[8]) {
#pragma unroll
        for (int o = 0; o < 8; o++) col[o * kThreads] = s[o] >= 0 ? sv + (int64_t)s[o] * 64 : g_zero_row;
    }
    __device__ __forceinline__ float point(int x, int y, int z) const {
        const int o = (x >> 2) | ((y >> 2) << 1) | ((z >> 2) << 2);
        return __ldg(rows[o * kThreads] + ((x & 3) + 4 * (y & 3) + 16 * (z & 3)));
    }
    __device__ __forceinline__ void corners(int lx, int ly, int lz, float c[8]) const {
#pragma unroll
        for (int idx = 0; idx < 8; idx++) c[idx] = point(lx + (idx & 1), ly + ((idx >> 1) & 1), lz + (idx >> 2));
    }
};

struct DenseFieldView {  // fully decoded volume, x-fastest
    const float *p;
    int64_t sy, sz;
    __device__ __forceinline__ void corners(int lx, int ly, int lz, float c[8]) const {
        const float *q = p + lx + sy * ly + sz * lz;
        c[0] = q[0];
        c[1] = q[1];
        c[2] = q[sy];
        c[3] = q[sy + 1];
        c[4] = q[sz];
        c[5] = q[sz + 1];
        c[6] = q[sz + sy];
        c[7] = q[sz + sy + 1];
    }
};

// engine.py:286-305 _contributor_table: cache slots of each visible block
// and its 7 +octant neighbours (-1 outside the volume), 32 B per block.
// Also clears the visibility bitmap for the next pass (its ranks were last
// read by k_build_entries): every visible id zeroes its word.
__device__ __forceinline__ void contrib_row(int64_t v, const uint32_t *visible_ids, const int32_t *slot_of_block,
                                            int bdx, int bdy, int bdz, const FastDiv &dv_x, const FastDiv &dv_xy,
                                            int4 *contrib, uint32_t *err) {
    {
        const uint32_t b = visible_ids[v];
        int bx, by, bz;
        unlinear3(b, dv_x, dv_xy, bx, by, bz);
        int s[8];
#pragma unroll
        for (int o = 0; o < 8; o++) {
            const int ox = o & 1, oy = (o >> 1) & 1, oz = o >> 2;
            s[o] = (bx + ox < bdx && by + oy < bdy && bz + oz < bdz)
                       ? slot_of_block[(bx + ox) + bdx * ((by + oy) + bdy * (bz + oz))]
                       : -1;
        }
        if (s[0] < 0) atomicAdd(err, 1u);  // "visible block not resident" (engine.py:302)
        contrib[2 * v] = make_int4(s[0], s[1], s[2], s[3]);
        contrib[2 * v + 1] = make_int4(s[4], s[5], s[6], s[7]);
    }
}

// The raytrace's inputs in one launch, after the cache update: the entries
// (k_build_entries' work, a thread per ray slot) and the contributor rows (a
// thread per visible block).  The visibility bitmap the entries rank against
// is cleared later, by k_rt_find.
struct BuildEntriesArgs {
    const uint32_t *ctl, *act_list, *emitted, *entry_off, *block_slots, *vis_bm, *vis_word_off;
    uint32_t *ent_key, *ent_val, *ent_ray, *ent_blk;
    uint32_t *sent_block, *sent_ray;  // the slot lists again: their sentinels are written here (WC_SENTINEL_LATE)
};
// traversal.py:423-424: a ray's slots past its last emit hold sentinels.
// With WC_SENTINEL_LATE the traversal skips them (a thread-per-ray lane wrote
// them one by one, scattered, up to 2 x 63 per ray) and the entry builder,
// which visits every slot (thread per slot), writes them coalesced; nothing
// reads the slot lists in between.
__device__ __forceinline__ void write_sentinel(const BuildEntriesArgs &be, int64_t t) {
#if WC_SENTINEL_LATE
    be.sent_block[t] = WC_UINT_MAX;
    be.sent_ray[t] = WC_UINT_MAX;
#endif
}
// The two halves of k_rt_prep as separate kernels, for the forked pass (the
// entries need only the traversal and mark_blocks, so they are built on a
// side branch while the cache is updated; the contributor rows need the
// slots the decode just mapped).
__global__ void k_rt_entries(BuildEntriesArgs be) {
    pdl_wait();
    const int64_t n_act = be.ctl[C_NACT], n_spec = be.ctl[C_NSPEC];
    const int64_t n_slots = n_act * n_spec;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_slots; t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)t / (uint32_t)n_spec;  // slots <= rays < 2^32
        const uint32_t j = (uint32_t)t - i * (uint32_t)n_spec;
        if (j >= be.emitted[i]) {
            write_sentinel(be, t);
            continue;
        }
        const uint32_t eo = be.entry_off[i] + j;
        const uint32_t b = be.block_slots[t];
        WC_DEVICE_CHECK(eo < be.ctl[C_NENT] && b != WC_UINT_MAX);
        const uint32_t w = b >> 5;
        be.ent_key[eo] = be.vis_word_off[w] + __popc(be.vis_bm[w] & ((1u << (b & 31)) - 1u));
        if (be.ent_val) be.ent_val[eo] = eo;
        be.ent_ray[eo] = be.act_list[i];
        be.ent_blk[eo] = b;
    }
}
__global__ void k_rt_contrib(const uint32_t *visible_ids, const uint32_t *d_nvis, const int32_t *slot_of_block, int bdx,
                             int bdy, int bdz, FastDiv dv_x, FastDiv dv_xy, int4 *contrib, uint32_t *err) {
    pdl_wait();
    const int64_t nvis = *d_nvis;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvis; v += (int64_t)gridDim.x * blockDim.x)
        contrib_row(v, visible_ids, slot_of_block, bdx, bdy, bdz, dv_x, dv_xy, contrib, err);
}

__global__ void k_rt_prep(BuildEntriesArgs be, const uint32_t *visible_ids, const uint32_t *d_nvis,
                          const int32_t *slot_of_block, int bdx, int bdy, int bdz, FastDiv dv_x, FastDiv dv_xy,
                          int4 *contrib, uint32_t *err) {
    pdl_wait();
    const int64_t n_act = be.ctl[C_NACT], n_spec = be.ctl[C_NSPEC];
    const int64_t n_slots = n_act * n_spec, nvis = *d_nvis;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n_slots + nvis;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (t >= n_slots) {
            contrib_row(t - n_slots, visible_ids, slot_of_block, bdx, bdy, bdz, dv_x, dv_xy, contrib, err);
            continue;
        }
        const uint32_t i = (uint32_t)t / (uint32_t)n_spec;  // slots <= rays < 2^32
        const uint32_t j = (uint32_t)t - i * (uint32_t)n_spec;
        if (j >= be.emitted[i]) {
            write_sentinel(be, t);
            continue;
        }
        const uint32_t eo = be.entry_off[i] + j;
        const uint32_t b = be.block_slots[t];
        WC_DEVICE_CHECK(eo < be.ctl[C_NENT] && b != WC_UINT_MAX);
        const uint32_t w = b >> 5;
        be.ent_key[eo] = be.vis_word_off[w] + __popc(be.vis_bm[w] & ((1u << (b & 31)) - 1u));
        if (be.ent_val) be.ent_val[eo] = eo;
        be.ent_ray[eo] = be.act_list[i];
        be.ent_blk[eo] = b;
    }
}

// every visible id zeroes its word of the visibility bitmap (its ranks were
// read by k_rt_prep), ready for the next pass's traversal
__device__ __forceinline__ void clear_visible_words(const uint32_t *visible_ids, const uint32_t *d_nvis,
                                                    uint32_t *vis_bm) {
    const int64_t nvis = *d_nvis;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvis; v += (int64_t)gridDim.x * blockDim.x)
        vis_bm[visible_ids[v] >> 5] = 0u;
}

struct RaytraceArgs {
    const uint32_t *visible_ids, *ent_key, *ent_val, *ent_ray, *ent_blk;
    uint32_t *vis_bm;         // cleared by k_rt_find (clear_visible_words)
    const uint32_t *d_nvis;
    bool identity;  // entries in their build order (not grouped): entry k at position k
    int64_t n_ent;
    const int4 *contrib;
    const float *slot_values;
    int bdx, bdy, bdz, nx, ny, nz;
    FastDiv bdv_x, bdv_xy;  // bdx, bdx bdy
    RayView rays;
    const double *fp;  // FrameParams (device): [3] iso, [4..6] base colour
    float4 *rgbz;
    const uint32_t *d_n_ent;  // entry count on the device (Counter C_NENT)
};

#if !WC_SPLIT_RAYTRACE  // the fused single-kernel raytrace (measured slower; kept for comparison builds)
// engine.py:161-219 _raytrace_visible_kernel, one thread per ray-block entry
// of the grouped (sorted-by-block) list, so neighbouring lanes trace the
// same block and share its slot lines in L1.  Each entry runs the region
// tracer (blocktrace.py:317-449) over the block's <= 4^3 dual cells and
// writes (rgb, z) -- or (0, 0, 0, +inf) on a miss -- at its entry id.
__global__ void __launch_bounds__(128, WC_RAYTRACE_MIN_CTAS) k_raytrace(RaytraceArgs a) {
    pdl_wait();
    clear_visible_words(a.visible_ids, a.d_nvis, a.vis_bm);
    a.rays.bind();
    const int64_t n_ent = *a.d_n_ent;
    const double iso = a.fp[3], br = a.fp[4], bg = a.fp[5], bb = a.fp[6];
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_ent; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = a.ent_key[j], k = a.ent_val[j];
        const int64_t r = a.ent_ray[k];
        const uint32_t b = a.visible_ids[v];
        const int bx = (int)(b % (uint32_t)a.bdx), by = (int)((b / (uint32_t)a.bdx) % (uint32_t)a.bdy),
                  bz = (int)(b / ((uint32_t)a.bdx * (uint32_t)a.bdy));
        const int4 c0 = a.contrib[2 * v], c1 = a.contrib[2 * v + 1];
        const SlotField field{a.slot_values, c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        const int cx = max(0, min(4, a.nx - 1 - 4 * bx));
        const int cy = max(0, min(4, a.ny - 1 - 4 * by));
        const int cz = max(0, min(4, a.nz - 1 - 4 * bz));
        double o[3], d[3];
        a.rays.load(r, o, d);
        float rgb[3];
        const double t = trace_region(field, 4 * bx, 4 * by, 4 * bz, 4 * bx, 4 * by, 4 * bz, cx, cy, cz, o, d,
                                      a.rays.t_enter[r], iso, br, bg, bb, rgb);
        a.rgbz[k] = t != CUDART_INF ? make_float4(rgb[0], rgb[1], rgb[2], (float)t)
                                    : make_float4(0.0f, 0.0f, 0.0f, CUDART_INF_F);
    }
}

#endif

// ---- two-phase raytrace: the same per-entry result as k_raytrace, with the
// float64 cubic solves run as a dense work list so that the divergent DDA
// and the uniform root finding no longer share warps.
// A candidate cell carries everything the solve and the shade need, so they
// start from one coalesced read instead of the entry -> ray -> block -> slot
// chain: info = (entry k, ray r, block b, lx | ly << 3 | lz << 6 | seq << 9)
// and the cell's 8 float corners (corner order idx = dx + 2 dy + 4 dz).
constexpr unsigned long long kNoRoot = ~0ull;
struct SplitArgs {
    RaytraceArgs a;
    uint4 *item_info;
    float4 *item_corners;  // 2 per item
    uint32_t *n_items;
    unsigned long long *best;  // per entry: (seq << 32 | item) of its earliest root
    double *item_t;
    int64_t item_cap;
};

struct EntryCtx {  // everything an entry's trace needs, rebuilt from its position j
    uint32_t k;
    int64_t r;
    int bx, by, bz, cx, cy, cz;
    SlotField field;
    double o[3], d[3], te;
};

__device__ __forceinline__ EntryCtx entry_ctx(const RaytraceArgs &a, const RayView &rv, int64_t j) {
    EntryCtx e;
    // ungrouped entries sit at their own index: ray and block load in the
    // same round trip as the visible rank
    const uint32_t v = a.ent_key[j];
    e.k = a.identity ? (uint32_t)j : a.ent_val[j];
    e.r = a.ent_ray[e.k];
    const uint32_t b = a.ent_blk[e.k];
    unlinear3(b, a.bdv_x, a.bdv_xy, e.bx, e.by, e.bz);
    const int4 c0 = a.contrib[2 * v], c1 = a.contrib[2 * v + 1];
    e.field = SlotField{a.slot_values, c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    e.cx = max(0, min(4, a.nx - 1 - 4 * e.bx));
    e.cy = max(0, min(4, a.ny - 1 - 4 * e.by));
    e.cz = max(0, min(4, a.nz - 1 - 4 * e.bz));
    rv.load(e.r, e.o, e.d);
    e.te = rv.t_enter[e.r];
    return e;
}

#ifndef WC_WALK_PREFETCH
#define WC_WALK_PREFETCH 0  // the two-phase walk measured slower (raytrace 0.96 vs 0.90 ms/frame)
#endif
#if WC_WALK_PREFETCH
#define WC_WALK walk_bracketing_cells_prefetch
#else
#define WC_WALK walk_bracketing_cells
#endif
// phase 1: walk each entry's dual cells, list the bracketing ones
__global__ void __launch_bounds__(128, WC_RTFIND_MIN_CTAS) k_rt_find(SplitArgs s) {
    pdl_wait();
    const RaytraceArgs &a = s.a;
    clear_visible_words(a.visible_ids, a.d_nvis, a.vis_bm);
    RayView rv = a.rays;
    rv.bind();
    const int lane = threadIdx.x & 31;
    __shared__ const float *rowtab[8][128];
    const SlotFieldSmem<128> sf{&rowtab[0][threadIdx.x]};
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // warp-uniform trip count: the list append below is a full-warp scan
    const int64_t n_ent = *a.d_n_ent;
    const double iso = a.fp[3];
    for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); j0 < n_ent; j0 += stride) {
        const int64_t j = j0 + lane;
        // the <= 10 bracketing cells of the walk, 6-bit local codes in DDA order
        int found = 0;
        unsigned long long codes = 0;
        uint32_t ek = 0, er = 0, eb = 0;  // kept for the item write-out
        SlotField ef{a.slot_values, -1, -1, -1, -1, -1, -1, -1, -1};
        if (j < n_ent) {
            const EntryCtx e = entry_ctx(a, rv, j);
            ek = e.k;
            er = (uint32_t)e.r;
            eb = (uint32_t)(e.bx + a.bdx * (e.by + a.bdy * e.bz));
            ef = e.field;
            s.best[e.k] = kNoRoot;
            const int sl[8] = {ef.s0, ef.s1, ef.s2, ef.s3, ef.s4, ef.s5, ef.s6, ef.s7};
            SlotFieldSmem<128>::fill(&rowtab[0][threadIdx.x], a.slot_values, sl);
            WC_WALK(sf, 4 * e.bx, 4 * e.by, 4 * e.bz, 4 * e.bx, 4 * e.by, 4 * e.bz, e.cx, e.cy,
                                  e.cz, e.o, e.d, e.te, iso, [&](int cx, int cy, int cz, int seq) {
                                      const uint32_t lc = (uint32_t)((cx - 4 * e.bx) | ((cy - 4 * e.by) << 2) |
                                                                     ((cz - 4 * e.bz) << 4));
                                      codes |= (unsigned long long)lc << (6 * seq);
                                      found++;
                                  });
            if (!found) a.rgbz[e.k] = make_float4(0.0f, 0.0f, 0.0f, CUDART_INF_F);
        }
        __syncwarp();  // the owners' row pointers (shared memory) are read across the warp below
        // one list append per warp (a per-cell atomic on the shared counter
        // serialises at L2)
        uint32_t incl = (uint32_t)found;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        uint32_t base_it = 0;
        if (lane == 31 && total) base_it = atomicAdd(s.n_items, total);
        base_it = __shfl_sync(0xffffffffu, base_it, 31);
        // The warp's items are written cooperatively, item t by lane t % 32
        // (the owning entry's lane is found by a search over the prefix
        // sums), instead of each lane looping over its own <= 10 items.  The
        // corners were just walked by the owner: these loads hit L1, through
        // the owner's row pointers in shared memory.
        const unsigned long long codes_lane = codes;
        for (uint32_t t0 = 0; t0 < total; t0 += 32) {
            const uint32_t t = t0 + lane;
            int owner = 0;  // smallest lane whose inclusive prefix exceeds t
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, owner + step - 1);
                if (v <= t) owner += step;
            }
            const uint32_t o_incl = __shfl_sync(0xffffffffu, incl, owner);
            const uint32_t o_found = (uint32_t)__shfl_sync(0xffffffffu, found, owner);
            const unsigned long long o_codes = __shfl_sync(0xffffffffu, codes_lane, owner);
            const uint32_t o_ek = __shfl_sync(0xffffffffu, ek, owner), o_er = __shfl_sync(0xffffffffu, er, owner),
                           o_eb = __shfl_sync(0xffffffffu, eb, owner);
            const uint32_t it = base_it + t;
            WC_DEVICE_CHECK(t >= total || it < s.item_cap);  // 10 dual cells per entry at most
            if (t < total && it < s.item_cap) {
                const uint32_t q = t - (o_incl - o_found);
                const uint32_t lc = (uint32_t)(o_codes >> (6 * q)) & 63u;
                const int lx = lc & 3, ly = (lc >> 2) & 3, lz = lc >> 4;
                const SlotFieldSmem<128> of{&rowtab[0][(threadIdx.x & ~31) + owner]};
                float c[8];
                of.corners(lx, ly, lz, c);
                s.item_info[it] = make_uint4(o_ek, o_er, o_eb, (uint32_t)(lx | (ly << 3) | (lz << 6)) | (q << 9));
                s.item_corners[2 * (int64_t)it] = make_float4(c[0], c[1], c[2], c[3]);
                s.item_corners[2 * (int64_t)it + 1] = make_float4(c[4], c[5], c[6], c[7]);
            }
        }
        __syncwarp();  // the row pointers are refilled by the next entries
    }
}

// phase 2: one thread per candidate cell; the earliest cell (in DDA order)
// with a root wins through an atomicMin on (seq, item)
__global__ void __launch_bounds__(128, WC_RAYTRACE_MIN_CTAS) k_rt_solve(SplitArgs s) {
    pdl_wait();
    const RaytraceArgs &a = s.a;
    RayView rv = a.rays;
    rv.bind();
    const int64_t n_items = min((int64_t)*s.n_items, s.item_cap);
    const double iso = a.fp[3];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_items; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 info = s.item_info[i];
        const float4 c0 = s.item_corners[2 * i], c1 = s.item_corners[2 * i + 1];
        const float c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        const uint32_t k = info.x, r = info.y, b = info.z, code = info.w;
        const int lx = code & 7, ly = (code >> 3) & 7, lz = (code >> 6) & 7, seq = code >> 9;
        int bx, by, bz;
        unlinear3(b, a.bdv_x, a.bdv_xy, bx, by, bz);
        double o[3], d[3];
        rv.load(r, o, d);
        const double th = solve_cell(c, o, d, 4 * bx + lx, 4 * by + ly, 4 * bz + lz, rv.t_enter[r], iso);
        if (th != CUDART_INF) {
            s.item_t[i] = th;
            atomicMin(&s.best[k], ((unsigned long long)seq << 32) | (unsigned long long)i);
        }
    }
}

// phase 3: shade each entry's winning cell (or record the miss)
// phase 3: shade each entry's earliest root.  Entries without one only
// write their miss value; the hits of a warp's successive 32-entry rounds
// are queued in shared memory and shaded 32 at a time, so every lane of a
// shading round has a hit (most entries of a pass have none).
__device__ __forceinline__ void shade_entry(const SplitArgs &s, const RayView &rv, uint32_t k, uint32_t i) {
    const RaytraceArgs &a = s.a;
    const uint4 info = s.item_info[i];
    const float4 c0 = s.item_corners[2 * (int64_t)i], c1 = s.item_corners[2 * (int64_t)i + 1];
    const float c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const uint32_t r = info.y, b = info.z, code = info.w;
    const int lx = code & 7, ly = (code >> 3) & 7, lz = (code >> 6) & 7;
    int bx, by, bz;
    unlinear3(b, a.bdv_x, a.bdv_xy, bx, by, bz);
    double o[3], d[3];
    rv.load(r, o, d);
    float rgb[3];
    const double th = s.item_t[i];
    shade_hit(c, o, d, 4 * bx + lx, 4 * by + ly, 4 * bz + lz, th, a.fp[4], a.fp[5], a.fp[6], rgb);
    a.rgbz[k] = make_float4(rgb[0], rgb[1], rgb[2], (float)th);
}

__global__ void __launch_bounds__(128) k_rt_shade(SplitArgs s) {
    pdl_wait();
    const RaytraceArgs &a = s.a;
    RayView rv = a.rays;
    rv.bind();
    __shared__ uint2 queue[4][64];  // per warp: (entry, winning item) of the hits not yet shaded
    uint2 *q = queue[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    int nq = 0;  // warp-uniform
    const int64_t n_ent = *a.d_n_ent;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); j0 < n_ent; j0 += stride) {
        const int64_t j = j0 + lane;
        uint32_t k = 0;
        unsigned long long bst = kNoRoot;
        if (j < n_ent) {
            k = a.identity ? (uint32_t)j : a.ent_val[j];
            bst = s.best[k];
            if (bst == kNoRoot) a.rgbz[k] = make_float4(0.0f, 0.0f, 0.0f, CUDART_INF_F);
        }
        const uint32_t hits = __ballot_sync(0xffffffffu, bst != kNoRoot);
        if (bst != kNoRoot) q[nq + __popc(hits & ((1u << lane) - 1u))] = make_uint2(k, (uint32_t)bst);
        nq += __popc(hits);
        __syncwarp();
        if (nq >= 32) {  // a full round of hits
            const uint2 e = q[nq - 32 + lane];
            __syncwarp();
            nq -= 32;
            shade_entry(s, rv, e.x, e.y);
        }
    }
    __syncwarp();
    if (lane < nq) {
        const uint2 e = q[lane];
        shade_entry(s, rv, e.x, e.y);
    }
}

#if WC_RT_FUSED
// ---- one-kernel raytrace with warp phases (WC_RT_FUSED): the same
// per-entry result as k_rt_find + k_rt_solve + k_rt_shade without the global
// work list.  A warp walks 32 entries' dual cells (lane = entry), lists the
// bracketing cells in registers (6-bit codes, DDA order), then solves them in
// rounds of 32 with lane = cell (the owner found by a search over the warp's
// prefix sums, corners through the owner's row pointers); the first cell of
// an entry with a root (blocktrace.py:420-433) shades it in place.
#ifndef WC_RTFUSED_MIN_CTAS
#define WC_RTFUSED_MIN_CTAS 5
#endif
__global__ void __launch_bounds__(128, WC_RTFUSED_MIN_CTAS) k_rt_fused(SplitArgs s) {
    pdl_wait();
    const RaytraceArgs &a = s.a;
    clear_visible_words(a.visible_ids, a.d_nvis, a.vis_bm);
    RayView rv = a.rays;
    rv.bind();
    const int lane = threadIdx.x & 31;
    __shared__ const float *rowtab[8][128];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_ent = *a.d_n_ent;
    const double iso = a.fp[3], br = a.fp[4], bg = a.fp[5], bb = a.fp[6];
    for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); j0 < n_ent; j0 += stride) {
        const int64_t j = j0 + lane;
        int found = 0;
        unsigned long long codes = 0;
        uint32_t ek = 0, er = 0;
        int ebx = 0, eby = 0, ebz = 0;
        if (j < n_ent) {
            const EntryCtx e = entry_ctx(a, rv, j);
            ek = e.k;
            er = (uint32_t)e.r;
            ebx = e.bx;
            eby = e.by;
            ebz = e.bz;
            const int sl[8] = {e.field.s0, e.field.s1, e.field.s2, e.field.s3, e.field.s4, e.field.s5, e.field.s6,
                               e.field.s7};
            SlotFieldSmem<128>::fill(&rowtab[0][threadIdx.x], a.slot_values, sl);
            const SlotFieldSmem<128> sf{&rowtab[0][threadIdx.x]};
            walk_bracketing_cells(sf, 4 * e.bx, 4 * e.by, 4 * e.bz, 4 * e.bx, 4 * e.by, 4 * e.bz, e.cx, e.cy, e.cz,
                                  e.o, e.d, e.te, iso, [&](int cx, int cy, int cz, int seq) {
                                      const uint32_t lc = (uint32_t)((cx - 4 * e.bx) | ((cy - 4 * e.by) << 2) |
                                                                     ((cz - 4 * e.bz) << 4));
                                      codes |= (unsigned long long)lc << (6 * seq);
                                      found++;
                                  });
        }
        __syncwarp();  // the owners' row pointers are read across the warp below
        uint32_t incl = (uint32_t)found;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        uint32_t won = 0;  // owner lanes whose entry has its root (warp-uniform)
        for (uint32_t t0 = 0; t0 < total; t0 += 32) {
            const uint32_t t = t0 + lane;
            int owner = 0;  // smallest lane whose inclusive prefix exceeds t
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, owner + step - 1);
                if (v <= t) owner += step;
            }
            const uint32_t o_incl = __shfl_sync(0xffffffffu, incl, owner);
            const uint32_t o_found = (uint32_t)__shfl_sync(0xffffffffu, found, owner);
            const unsigned long long o_codes = __shfl_sync(0xffffffffu, codes, owner);
            const uint32_t o_ek = __shfl_sync(0xffffffffu, ek, owner), o_er = __shfl_sync(0xffffffffu, er, owner);
            const int o_bx = __shfl_sync(0xffffffffu, ebx, owner), o_by = __shfl_sync(0xffffffffu, eby, owner),
                      o_bz = __shfl_sync(0xffffffffu, ebz, owner);
            const bool live = t < total && !((won >> owner) & 1u);
            double th = CUDART_INF;
            float c[8];
            int cx = 0, cy = 0, cz = 0;
            double o[3], d[3];
            if (live) {
                const uint32_t q = t - (o_incl - o_found);
                const uint32_t lc = (uint32_t)(o_codes >> (6 * q)) & 63u;
                const int lx = lc & 3, ly = (lc >> 2) & 3, lz = lc >> 4;
                const SlotFieldSmem<128> of{&rowtab[0][(threadIdx.x & ~31) + owner]};
                of.corners(lx, ly, lz, c);
                cx = 4 * o_bx + lx;
                cy = 4 * o_by + ly;
                cz = 4 * o_bz + lz;
                rv.load(o_er, o, d);
                th = solve_cell(c, o, d, cx, cy, cz, rv.t_enter[o_er], iso);
            }
            // the owner's first cell (in DDA order) with a root wins: the
            // cells of an owner are consecutive lanes in seq order
            const uint32_t roots = __ballot_sync(0xffffffffu, th != CUDART_INF);
            const uint32_t same = __match_any_sync(0xffffffffu, owner);
            const uint32_t first = roots & same;
            const bool winner = th != CUDART_INF && (first & ((1u << lane) - 1u)) == 0u;
            if (winner) {
                float rgb[3];
                shade_hit(c, o, d, cx, cy, cz, th, br, bg, bb, rgb);
                a.rgbz[o_ek] = make_float4(rgb[0], rgb[1], rgb[2], (float)th);
            }
            won |= __reduce_or_sync(0xffffffffu, winner ? (1u << owner) : 0u);
        }
        if (j < n_ent && !((won >> lane) & 1u)) a.rgbz[ek] = make_float4(0.0f, 0.0f, 0.0f, CUDART_INF_F);
        __syncwarp();  // the row pointers are refilled by the next entries
    }
}
#endif

// ------------------------------------------------------------- composite

// engine.py:222-258 _composite_kernel: closest speculated hit per active
// ray (strict <, earliest entry wins ties), then terminate or keep.
constexpr uint32_t kWarpCompositeSpec = 8;  // n_spec from which a warp composites one ray

// engine.py:222-258 for active ray i: the closest speculated hit (strict <,
// earliest entry wins ties), then terminate (hit / exited) or keep.
__device__ __forceinline__ void composite_ray(int64_t i, uint32_t r, float best, int64_t bk, const float4 *rgbz,
                                              const uint8_t *exited, uint8_t *status, uint32_t *rgba, float *depth,
                                              uint32_t *keep, const unsigned long long *target,
                                              const uint32_t *pixel_ids) {
    uint32_t kp = 0;
    if (bk >= 0) {
        const float4 c = rgbz[bk];
        const uint32_t v = rgb_u8((double)c.x) | (rgb_u8((double)c.y) << 8) | (rgb_u8((double)c.z) << 16) | 0xFF000000u;
        depth[r] = best;
        rgba[r] = v;
        status[r] = 1;
        target_write(target, pixel_ids, r, v, best);
    } else if (exited[r] == 1) {
        status[r] = 2;
        target_write(target, pixel_ids, r, rgba[r], depth[r]);  // the background it kept
    } else {
        kp = 1;
    }
    keep[i] = kp;
}

// Thread per ray, or (n_spec >= kWarpCompositeSpec, read on the device) a
// warp per ray: the lexicographic (depth, entry) minimum over the lanes is
// the first strict minimum in order.
__global__ void k_composite(const uint32_t *ctl, const uint32_t *act_list, const uint32_t *emitted,
                            const uint32_t *entry_off, const float4 *rgbz, const uint8_t *exited, uint8_t *status,
                            uint32_t *rgba, float *depth, uint32_t *keep, const unsigned long long *target,
                            const uint32_t *pixel_ids) {
    pdl_wait();
    const int64_t n_act = ctl[C_NACT];
    if (ctl[C_NSPEC] < kWarpCompositeSpec) {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_act;
             i += (int64_t)gridDim.x * blockDim.x) {
            const uint32_t r = act_list[i], ne = emitted[i], eo = entry_off[i];
            WC_DEVICE_CHECK(eo + ne <= ctl[C_NENT] && ne <= ctl[C_NSPEC]);
            float best = CUDART_INF_F;
            int64_t bk = -1;
            for (uint32_t j = 0; j < ne; j++) {
                const float z = rgbz[eo + j].w;
                if (z < best) {
                    best = z;
                    bk = eo + j;
                }
            }
            composite_ray(i, r, best, bk, rgbz, exited, status, rgba, depth, keep, target, pixel_ids);
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w0; i < n_act; i += nw) {
        const uint32_t r = act_list[i], ne = emitted[i], eo = entry_off[i];
        float best = CUDART_INF_F;
        uint32_t bj = 0xFFFFFFFFu;
        for (uint32_t j = lane; j < ne; j += 32) {
            const float z = rgbz[eo + j].w;
            if (z < best) {
                best = z;
                bj = j;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float zb = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t jb = __shfl_xor_sync(0xffffffffu, bj, o);
            if (zb < best || (zb == best && jb < bj)) {
                best = zb;
                bj = jb;
            }
        }
        if (lane == 0) composite_ray(i, r, best, bj != 0xFFFFFFFFu ? (int64_t)eo + bj : -1, rgbz, exited, status, rgba,
                                     depth, keep, target, pixel_ids);
    }
}

// ------------------------------------------------------------ brute force

__global__ void __launch_bounds__(128) k_reference_render(const float *values, int nx, int ny, int nz,
                                                          const double *origin, const double *dir, int64_t n,
                                                          double iso, double br, double bg, double bb, uint32_t *rgba,
                                                          float *depth) {
    pdl_wait();
    const DenseFieldView field{values, nx, (int64_t)nx * ny};
    const double hi[3] = {(double)nx - 1.0, (double)ny - 1.0, (double)nz - 1.0};
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        double o[3], d[3];
        for (int k = 0; k < 3; k++) {
            o[k] = origin[3 * r + k];
            d[k] = dir[3 * r + k];
        }
        // RaySoA.from_rays status / t_enter (traversal.py:132-154)
        double nr[3], fr[3];
        for (int k = 0; k < 3; k++) {
            if (d[k] != 0.0) {
                const double t1 = (0.0 - o[k]) / d[k], t2 = (hi[k] - o[k]) / d[k];
                nr[k] = t1 < t2 ? t1 : t2;
                fr[k] = t1 > t2 ? t1 : t2;
            } else if (o[k] < 0.0 || o[k] > hi[k]) {
                nr[k] = CUDART_INF;
                fr[k] = -CUDART_INF;
            } else {
                nr[k] = -CUDART_INF;
                fr[k] = CUDART_INF;
            }
        }
        double t_near = nr[0] > nr[1] ? nr[0] : nr[1];
        t_near = t_near > nr[2] ? t_near : nr[2];
        double t_far = fr[0] < fr[1] ? fr[0] : fr[1];
        t_far = t_far < fr[2] ? t_far : fr[2];
        rgba[r] = 0xFF000000u;
        depth[r] = CUDART_INF_F;
        if (!((t_near <= t_far) && (t_far >= 0.0))) continue;
        const double te = t_near > 0.0 ? t_near : 0.0;
        double rgb[3];
        const double t = trace_region(field, 0, 0, 0, 0, 0, 0, nx - 1, ny - 1, nz - 1, o, d, te, iso, br, bg, bb, rgb);
        if (t != CUDART_INF) {
            depth[r] = (float)t;
            rgba[r] = rgb_u8(rgb[0]) | (rgb_u8(rgb[1]) << 8) | (rgb_u8(rgb[2]) << 16) | 0xFF000000u;
        }
    }
}

void reference_render_device(const float *d_values, int nx, int ny, int nz, const double *d_origin,
                             const double *d_dir, int64_t n, double iso, double br, double bg, double bb,
                             uint32_t *d_rgba, float *d_depth, cudaStream_t st) {
    if (n <= 0) return;
    launch_pdl(k_reference_render, grid_for(n, 128, 16), 128, 0, st, d_values, nx, ny, nz, d_origin, d_dir, n, iso, br, bg,
                                                             bb, d_rgba, d_depth);
    WC_LAUNCH_CHECK();
}

// ------------------------------------------------------------- control
// Single-thread kernels that make the pass's host decisions on the device,
// so passes are enqueued back to back without host round trips.

// engine.py:91-94 compute_n_spec (1 when speculation is off, engine.py:333)
__device__ __forceinline__ int64_t n_spec_of(int64_t n, int64_t n_act, int speculation, int max_spec) {
    if (!speculation || n_act <= 0) return 1;
    const int64_t q = n / n_act;
    return min((int64_t)max_spec, q > 1 ? q : (int64_t)1);
}

// after the initial active scan (C_NACT): the first pass's n_spec and an
// empty cache of the initial capacity (cache.py:27-40)
__global__ void k_frame_start(uint32_t *ctl, int64_t n, int speculation, int max_spec, int64_t cap, int64_t phys,
                              int64_t nwords, uint32_t frame, double *fp, double ex, double ey, double ez, double iso,
                              double br, double bg, double bb) {
    pdl_wait();
    // FrameParams: what changes between frames lives in device memory, so the
    // captured pass graphs are frame-invariant
    fp[0] = ex;
    fp[1] = ey;
    fp[2] = ez;
    fp[3] = iso;
    fp[4] = br;
    fp[5] = bg;
    fp[6] = bb;
    ctl[C_FRAME] = frame;
    const int64_t n_act = ctl[C_NACT];
    ctl[C_NSPEC] = (uint32_t)n_spec_of(n, n_act, speculation, max_spec);
    ctl[C_CAP] = (uint32_t)cap;
    ctl[C_PHYS] = ctl[C_PHYS_OLD] = (uint32_t)phys;
    ctl[C_HW] = ctl[C_HW_NEXT] = 0;
    for (int b = 0; b < kHistBins; b++) ctl[C_COUNT + b] = 0;  // the cache is empty: no stamps
}

// cache.py:66-96 decisions of ensure_resident once the hits are stamped and
// the misses listed: growth to ceil(1.5 * needed), free suffix, number of
// victims and the last stamp bucket they reach (from the stamp histogram)
__device__ __forceinline__ void cache_plan(uint32_t *ctl, uint32_t *hist, int32_t pass_no, int64_t n_blocks,
                                           int64_t slot_alloc, bool maintain) {
    const int64_t nactb = ctl[C_NACTB], n_miss = ctl[C_NMISS], hw = ctl[C_HW];
    int64_t cap = ctl[C_CAP], phys = ctl[C_PHYS];
    ctl[C_PHYS_OLD] = (uint32_t)phys;
    if (nactb > cap) {  // cache.py:74-75
        cap = (3 * nactb + 1) / 2;
        phys = max(phys, min(cap, n_blocks));
    }
    if (phys > slot_alloc) {  // cannot happen: slots are reserved for the largest possible capacity
        ctl[C_ERR_CAP] = 1;
        phys = slot_alloc;
    }
    ctl[C_CAP] = (uint32_t)cap;
    ctl[C_PHYS] = (uint32_t)phys;
    const int64_t n_free = cap - hw;
    ctl[C_NFREE] = (uint32_t)n_free;
    int64_t n_evict = 0;
    uint32_t lstar = 0xFFFFFFFFu;
    if (n_miss > n_free) {  // cache.py:80-96
        n_evict = n_miss - n_free;
        if (hw - (nactb - n_miss) < n_evict) ctl[C_ERR_CAND] = 1;
        int64_t acc = 0;
        for (int L = 0; L < pass_no && acc < n_evict; L++) {
            acc += hist[L];
            lstar = (uint32_t)L;
        }
        if (acc < n_evict) ctl[C_ERR_CAND] = 1;
    }
    ctl[C_NEVICT] = (uint32_t)n_evict;
    ctl[C_LSTAR] = lstar;
    // the victims' regions are stamps 0..L*: their summary words are the
    // only ones k_mark_victims can set
    ctl[C_VSUM] = n_evict ? (uint32_t)(((int64_t)lstar + 1) * ceil_div(n_blocks, 32) / 32 + 1) : 0u;
    if (maintain) {  // the victims leave their bins (in (last_used, id) order), the misses enter bin pass_no
        int64_t left = n_evict;
        for (int L = 0; L < pass_no && left > 0; L++) {
            const int64_t take = min(left, (int64_t)hist[L]);
            hist[L] -= (uint32_t)take;
            left -= take;
        }
        hist[pass_no] += (uint32_t)n_miss;
    }
}
__global__ void k_cache_plan(uint32_t *ctl, uint32_t *hist, int32_t pass_no, int64_t n_blocks, int64_t slot_alloc,
                             bool maintain) {
    pdl_wait();
    cache_plan(ctl, hist, pass_no, n_blocks, slot_alloc, maintain);
}

// the same decisions as the epilogue of the miss compaction (its count is
// the n_miss they need), saving a launch per pass
struct CachePlanEpilogue {
    uint32_t *ctl, *hist;
    int32_t pass_no;
    int64_t n_blocks, slot_alloc;
    __device__ __forceinline__ void operator()(uint32_t n_miss) const {
        ctl[C_NMISS] = n_miss;
        cache_plan(ctl, hist, pass_no, n_blocks, slot_alloc, true);
    }
};

// maps of the slots the growth just brought into use (cache.py:42-53)

// end of pass: the PassStats record, then the next pass's n_act / n_spec
// (engine.py:331-333, slot budget engine.py:341)
__device__ __forceinline__ void pass_end(uint32_t *ctl, uint32_t *row, int64_t n, int speculation, int max_spec) {
    const int64_t n_act = ctl[C_NACT], n_after = ctl[C_NACT_NEXT];
    row[L_NACT] = (uint32_t)n_act;
    row[L_NSPEC] = ctl[C_NSPEC];
    row[L_NVIS] = ctl[C_NVIS];
    row[L_NACTB] = ctl[C_NACTB];
    row[L_NMISS] = ctl[C_NMISS];
    row[L_NEVICT] = ctl[C_NEVICT];
    row[L_CAP] = ctl[C_CAP];
    row[L_NENT] = ctl[C_NENT];
    row[L_NAFTER] = (uint32_t)n_after;
    row[L_NITEMS] = ctl[C_NITEMS];
    row[L_PHYS] = ctl[C_PHYS];
    row[L_HW] = ctl[C_HW_NEXT];
    row[L_NLONG] = ctl[C_NLONG];
    ctl[C_WORK] = 0;  // the next pass's traversal work counter and raytrace list start empty
    ctl[C_NLONG] = 0;
    ctl[C_NITEMS] = 0;
    if (n_act == 0) return;  // an enqueued pass after the last one: no state change
    ctl[C_HW] = ctl[C_HW_NEXT];
    const int64_t n_spec = n_spec_of(n, n_after, speculation, max_spec);
    if (n_after * n_spec > n) ctl[C_ERR_BUDGET] = 1;
    ctl[C_NACT] = (uint32_t)n_after;
    ctl[C_NSPEC] = (uint32_t)n_spec;
}

// pass_end as the epilogue of the compaction of the surviving rays (its
// count is n_after).  It rewrites the count that compaction reads
// (ctl[C_NACT]); a scan epilogue runs in the CTA that finishes last, after
// every CTA of the scan has read the count (k_scan_onepass).
struct PassEndEpilogue {
    uint32_t *ctl, *row;
    int64_t n;
    int speculation, max_spec;
    __device__ __forceinline__ void operator()(uint32_t n_after) const {
        ctl[C_NACT_NEXT] = n_after;
        pass_end(ctl, row, n, speculation, max_spec);
    }
};

// ---------------------------------------------------- frame target (peer memory)
FrameTarget::~FrameTarget() {
    if (opened) {
        if (p_rgba) cudaIpcCloseMemHandle(p_rgba);
        if (p_depth) cudaIpcCloseMemHandle(p_depth);
    }
}
void FrameTarget::create(int64_t n) {
    npix = n;
    rgba.alloc(n);
    depth.alloc(n);
    p_rgba = rgba.p;
    p_depth = depth.p;
}
void FrameTarget::ipc_handles(void *out) const {
    cudaIpcMemHandle_t h[2];
    WC_CUDA(cudaIpcGetMemHandle(&h[0], p_rgba));
    WC_CUDA(cudaIpcGetMemHandle(&h[1], p_depth));
    std::memcpy(out, h, sizeof(h));
}
void FrameTarget::open(const void *handles, int64_t n) {
    cudaIpcMemHandle_t h[2];
    std::memcpy(h, handles, sizeof(h));
    npix = n;
    void *a = nullptr, *b = nullptr;
    WC_CUDA(cudaIpcOpenMemHandle(&a, h[0], cudaIpcMemLazyEnablePeerAccess));
    WC_CUDA(cudaIpcOpenMemHandle(&b, h[1], cudaIpcMemLazyEnablePeerAccess));
    p_rgba = static_cast<uint32_t *>(a);
    p_depth = static_cast<float *>(b);
    opened = true;
}

// The session's pixels go to `t` as they become final (nullptr: none).  The
// addresses live in device memory, so the captured pass graphs stay valid.
void Session::set_frame_target(const FrameTarget *t) {
    const unsigned long long v[2] = {t ? (unsigned long long)(uintptr_t)t->p_rgba : 0ull,
                                     t ? (unsigned long long)(uintptr_t)t->p_depth : 0ull};
    if (t && !uniform_origin) throw UsageError("a frame target needs camera rays (pixel ids)");
    WC_CUDA(cudaMemcpyAsync(tgt.p, v, sizeof(v), cudaMemcpyHostToDevice, st));
    WC_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------- framebuffer read-back

// rays still active after the snapshot pass (their pixels may still change)
__global__ void k_snapshot_list(uint32_t *ctl, const uint32_t *act, uint32_t *snap) {
    pdl_wait();
    const int64_t n = ctl[C_NACT];
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl[C_NSNAP] = (uint32_t)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        snap[i] = act[i];
}

// their final pixels: (ray, rgba, depth bits)
__global__ void k_gather_patch(const uint32_t *ctl, const uint32_t *snap, const uint32_t *rgba, const float *depth,
                               uint4 *patch) {
    pdl_wait();
    const int64_t n = ctl[C_NSNAP];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = snap[i];
        patch[i] = make_uint4(r, rgba[r], __float_as_uint(depth[r]), 0u);
    }
}

// The same patch written by the GPU straight into the host framebuffer
// (pinned, device-mapped), after the bulk copy has landed.
__global__ void k_patch_host(const uint32_t *ctl, const uint32_t *snap, const uint32_t *rgba, const float *depth,
                             uint32_t *h_rgba, float *h_depth) {
    pdl_wait();
    const int64_t n = ctl[C_NSNAP];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = snap[i];
        h_rgba[r] = rgba[r];
        h_depth[r] = depth[r];
    }
}

// device address of a pinned host buffer (nullptr: pageable / not mapped)
static void *mapped_device_ptr(void *host) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

// ------------------------------------------------------------------ session

static int bits_for(uint64_t max_value) {
    int b = 0;
    while (b < 64 && (max_value >> b)) b++;
    return b;
}

Session::Session(Volume *v, const CameraParams *cam, const uint32_t *pixel_ids, int64_t n_rays,
                 const double *origins, const double *dirs, double iso_, int speculation_, int max_spec_,
                 int64_t cache_capacity, int corrupt_)
    : vol(v), n(n_rays), iso(iso_), speculation(speculation_), max_spec(max_spec_), corrupt(corrupt_) {
    if (n < 1) throw UsageError("a session needs at least one ray");
    WC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    WC_CUDA(cudaStreamCreateWithFlags(&st_side, cudaStreamNonBlocking));
    WC_CUDA(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
    for (auto &e : ev_fork) WC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    uniform_origin = dirs == nullptr;
    dir.alloc(n * 3);
    if (!uniform_origin) origin.alloc(n * 3);
    WC_CUDA(cudaEventCreate(&ev_frame0));
    WC_CUDA(cudaEventCreate(&ev_reset_end));
    t_enter.alloc(n);
    t_exit.alloc(n);
    coarse_tmax.alloc(n * 3);
    fine_tmax.alloc(n * 3);
    status.alloc(n);
    exited.alloc(n);
    coarse_cell.alloc(n);
    fine_cell.alloc(n);
    act_list[0].alloc(n);
    act_list[1].alloc(n);
    keep.alloc(n);
    emitted.alloc(n);
    long_q.alloc(n);
    entry_off.alloc(n);
    block_slots.alloc(n);
    ray_slots.alloc(n);
    ent_key.alloc(n);
    ent_val.alloc(n);
    ent_ray.alloc(n);
    ent_blk.alloc(n);
    rgbz.alloc(n);
    visible_ids.alloc(n);
    block_ray_off.alloc(n + 1);
    rgba.alloc(n);
    depth.alloc(n);
    const int64_t nwords = ceil_div(vol->n_blocks, 32);
    vis_bm.alloc(nwords);
    act_bm.alloc(nwords);
    int64_t chunk0;
    mask_buffers(1, chunk0);
    vis_word_off.alloc(nwords);  // prefix of each non-zero visible word (bitmap rank)
    WC_CUDA(cudaMemsetAsync(vis_bm.p, 0, 4 * nwords, st));
    WC_CUDA(cudaMemsetAsync(act_bm.p, 0, 4 * nwords, st));
    active_ids.alloc(std::min<int64_t>(8 * n, vol->n_blocks) + 1);
    miss_ids.alloc(active_ids.n);
    counters.alloc(C_COUNT + kHistBins);
    WC_CUDA(cudaMemsetAsync(counters.p, 0, 4 * C_COUNT, st));
    h_counters.alloc(C_COUNT + kHistBins);
    partials.alloc(scan_scratch_words(std::max<int64_t>({n, nwords, active_ids.n, 1})));
    WC_CUDA(cudaMemsetAsync(partials.p, 0, 4 * partials.n, st));
    partials_side.alloc(scan_scratch_words(n));  // the forked pass's side-branch scan
    WC_CUDA(cudaMemsetAsync(partials_side.p, 0, 4 * partials_side.n, st));

    slot_of_block.alloc(vol->n_blocks);
    WC_CUDA(cudaMemsetAsync(slot_of_block.p, 0xFF, 4 * vol->n_blocks, st));
    if (pixel_ids) {
        pix.alloc(n);
        WC_CUDA(cudaMemcpyAsync(pix.p, pixel_ids, 4 * n, cudaMemcpyHostToDevice, st));
    }
    if (dirs) {
        dir_in.alloc(3 * n);
        WC_CUDA(cudaMemcpyAsync(origin.p, origins, 24 * n, cudaMemcpyHostToDevice, st));
        WC_CUDA(cudaMemcpyAsync(dir_in.p, dirs, 24 * n, cudaMemcpyHostToDevice, st));
    }
    init_cap = cache_capacity;
    use_graphs = getenv("WAVECAST_NO_GRAPHS") == nullptr;
    contrib.alloc(2 * n);
    // every buffer a pass touches, at its largest size (a pass never allocates):
    // the cache for ceil(1.5 * min(8 N, n_blocks)) slots (cache.py:74-75 on the
    // most active blocks a pass can have), the raytrace work list for 10 N items
    const int64_t cap0 = std::max<int64_t>(1, init_cap <= 0 ? std::max<int64_t>(1024, 2 * n / 64) : init_cap);
    const int64_t max_active = std::min<int64_t>(8 * n, vol->n_blocks);
    reserve_slots(std::min<int64_t>(vol->n_blocks, std::max<int64_t>(cap0, (3 * max_active + 1) / 2)));
    item_info.alloc(10 * n);
    item_corners.alloc(20 * n);
    item_t.alloc(10 * n);
    best.alloc(n);
    plog.alloc((int64_t)kMaxPassLog * L_COUNT);
    fparams.alloc(8);
    tgt.alloc(2);
    WC_CUDA(cudaMemsetAsync(tgt.p, 0, 2 * sizeof(unsigned long long), st));
    h_plog.alloc((int64_t)kMaxPassLog * L_COUNT);
    reset(cam, iso_);
    precapture(kPrecapturePasses);
}

// A new frame on the same allocations: fresh rays for (cam, iso), a blank
// framebuffer and an empty cache of the initial logical capacity (the
// reference builds a new RaySoA / BlockCache per render, engine.py:316-320).
// Coarse-cell words [w0, w1) of part `part` of `parts` (32 cells per word),
// and the per-part chunk the mask buffers are padded to.
static void mask_part(int64_t n_coarse, int64_t part, int64_t parts, int64_t &w0, int64_t &w1, int64_t &chunk) {
    const int64_t nw = ceil_div(n_coarse, 32);
    chunk = ceil_div(nw, std::max<int64_t>(1, parts));
    w0 = std::min<int64_t>(nw, part * chunk);
    w1 = std::min<int64_t>(nw, w0 + chunk);
}

void Session::mask_buffers(int64_t parts, int64_t &chunk_words) {
    int64_t w0, w1;
    mask_part(vol->n_coarse, 0, parts, w0, w1, chunk_words);
    const int64_t words = std::max<int64_t>(parts * chunk_words, ceil_div(vol->n_coarse, 32));
    if (coarse_bm.n < words || cell_mask.n < 32 * words) {
        coarse_bm.alloc(words);
        cell_mask.alloc(32 * words);
        drop_graphs();  // they read the old buffers
    }
}

void Session::reset(const CameraParams *cam, double iso_) { reset_part(cam, iso_, 0, 1); }

// reset for part `part` of `parts`: the per-iso range tests are computed for
// that slice of coarse cells only; the caller assembles the others (an
// all-gather across the ranks of a tile split) before running the passes.
void Session::reset_part(const CameraParams *cam, double iso_, int64_t part, int64_t parts) {
    iso = iso_;
    if (cam) {
        cam_params = *cam;
        eye[0] = cam->eye[0];
        eye[1] = cam->eye[1];
        eye[2] = cam->eye[2];
    }
    WC_CUDA(cudaEventRecord(ev_frame0, st));
    int64_t w0, w1, chunk;
    mask_buffers(parts, chunk);
    mask_part(vol->n_coarse, part, parts, w0, w1, chunk);
    const int64_t c_end = std::min<int64_t>(vol->n_coarse, 32 * w1);
    // The per-iso range tests run on a side stream, overlapped with the ray
    // and cache setup below (they depend on neither); joined before the
    // reset ends.  The fork follows ev_frame0, i.e. the previous frame's
    // passes that read the old tests.
    const bool masks = w1 > w0;
    if (masks) {
        WC_CUDA(cudaStreamWaitEvent(st_side, ev_frame0, 0));
        launch_pdl(k_iso_bitmap, grid_for((w1 - w0) * 32, 256, 8), 256, 0, st_side, vol->coarse_mm.p, vol->n_coarse, iso,
                                                                           coarse_bm.p, w0, w1);
        WC_LAUNCH_CHECK();
        launch_pdl(k_iso_cell_mask, grid_for((c_end - 32 * w0) * 16, 256, 8), 256, 0, st_side, 
            vol->fine_q.p, vol->fine_mm.p, coarse_bm.p, vol->bdx, vol->bdy, vol->bdz, vol->cdx, vol->cdy, vol->cdz,
            iso, vol->q_base, vol->q_inv, cell_mask.p, 32 * w0, c_end);
        WC_LAUNCH_CHECK();
        WC_CUDA(cudaEventRecord(ev_side, st_side));
    }
    RayInitArgs a{};
    a.cam = cam_params;
    a.pixel_ids = pix.p;
    a.origin_in = uniform_origin ? nullptr : origin.p;
    a.dir_in = uniform_origin ? nullptr : dir_in.p;
    a.nx = vol->nx;
    a.ny = vol->ny;
    a.nz = vol->nz;
    a.target = tgt.p;
    launch_pdl(k_init_rays, grid_for(n, 256), 256, 0, st, a, n, nullptr, dir.p, t_enter.p, t_exit.p, status.p, exited.p,
                                                  coarse_cell.p, fine_cell.p, coarse_tmax.p, fine_tmax.p, rgba.p,
                                                  depth.p);
    WC_LAUNCH_CHECK();
    // cache (cache.py:27-40, initial_capacity :122-125 with w*h == n):
    // unmap whatever the previous frame left resident (its slot count is
    // still in the control block)
    launch_pdl(k_cache_unmap, grid_for(slot_alloc, 256), 256, 0, st, block_of_slot.p, counters.p + C_PHYS, slot_of_block.p);
    WC_LAUNCH_CHECK();
    cap = std::max<int64_t>(1, init_cap <= 0 ? std::max<int64_t>(1024, 2 * n / 64) : init_cap);
    phys = std::min<int64_t>(cap, vol->n_blocks);
    reserve_slots(phys);  // no-op after creation (the session reserved the largest capacity)
    // Free slots' values are never read (a slot is written by its decode
    // before any lookup can reach it), so only the slot maps are reset.
    WC_CUDA(cudaMemsetAsync(block_of_slot.p, 0xFF, 4 * phys, st));
    WC_CUDA(cudaMemsetAsync(last_used.p, 0, 4 * phys, st));

    // initial active list (engine.py:331 on pass 0) and the device control block
    WC_CUDA(cudaMemsetAsync(counters.p, 0, 4 * C_COUNT, st));
    PredActive pa{status.p};
    scan_exclusive(pa, n, entry_off.p, counters.p + C_NACT, partials.p, st);
    launch_pdl(k_compact_index<PredActive>, grid_for(n, 256), 256, 0, st, pa, n, entry_off.p, act_list[0].p);
    WC_LAUNCH_CHECK();
    if ((++frame_no & 0x1FFFFu) == 0)  // device-derived scan epochs wrap: forget old status words
        WC_CUDA(cudaMemsetAsync(partials.p, 0, 4 * partials.n, st));
    launch_pdl(k_frame_start, 1, 1, 0, st, counters.p, n, speculation, max_spec, cap, phys, ceil_div(vol->n_blocks, 32),
                                   frame_no, fparams.p, eye[0], eye[1], eye[2], iso, base[0], base[1], base[2]);
    WC_LAUNCH_CHECK();
    pass_no = 0;
    hw = 0;
    pass_index = 0;
    n_act = -1;  // on the device until the first pass reads it
    frame_end = nullptr;
    for (double &m : stage_ms) m = 0.0;
    graph_ms = 0.0;
    for (auto &p : pass_stage_ms)
        for (double &m : p) m = 0.0;
    if (masks) WC_CUDA(cudaStreamWaitEvent(st, ev_side, 0));
    WC_CUDA(cudaEventRecord(ev_reset_end, st));
}

int64_t Session::active_count() {
    if (n_act < 0) {
        read_counters(0, C_COUNT);
        n_act = h_counters.p[C_NACT];
    }
    return n_act;
}

double Session::reset_device_ms() {
    float rms = 0.0f;
    if (cudaEventQuery(ev_reset_end) != cudaSuccess) return 0.0;
    WC_CUDA(cudaEventElapsedTime(&rms, ev_frame0, ev_reset_end));
    return rms;
}

Session::~Session() {
    drop_graphs();
    if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    if (st_side) {
        cudaStreamSynchronize(st_side);
        cudaStreamDestroy(st_side);
    }
    if (ev_side) cudaEventDestroy(ev_side);
    for (auto &e : ev_fork)
        if (e) cudaEventDestroy(e);
    if (st_copy) {
        cudaStreamSynchronize(st_copy);
        cudaStreamDestroy(st_copy);
    }
    for (int k = 0; k < kSnapRing; k++) {
        if (snap_ready[k]) cudaEventDestroy(snap_ready[k]);
        if (snap_done[k]) cudaEventDestroy(snap_done[k]);
    }
    if (ev_fb) cudaEventDestroy(ev_fb);
    if (ev_fb_done) cudaEventDestroy(ev_fb_done);
    if (ev_frame0) cudaEventDestroy(ev_frame0);
    if (ev_reset_end) cudaEventDestroy(ev_reset_end);
    for (auto &row : pass_ev)
        for (auto &e : row)
            if (e) cudaEventDestroy(e);
}

void Session::read_counters(int first, int count) {
    WC_CUDA(cudaMemcpyAsync(h_counters.p, counters.p + first, 4 * count, cudaMemcpyDeviceToHost, st));
    WC_CUDA(cudaStreamSynchronize(st));
}

// Physical slot storage for `need` slots (maps, values, eviction scratch).
// The session reserves, at creation, slots for the largest capacity the
// reference's growth rule can reach -- ceil(1.5 * active blocks) with at most
// min(8 N, n_blocks) active blocks per pass -- so a pass never allocates and
// the cache decisions can stay on the device.
void Session::reserve_slots(int64_t need) {
    if (need <= slot_alloc) return;
    drop_graphs();  // they hold the old buffers
    reserve_store(need, std::max<int64_t>({n, ceil_div(vol->n_blocks, 32), active_ids.n}), partials, st);
}

bool CacheStore::reserve_store(int64_t need, int64_t scan_n, DevBuf<uint32_t> &partials, cudaStream_t st) {
    if (need <= slot_alloc) return false;
    slot_values.grow(need * 64, st);
    block_of_slot.grow(need, st);
    last_used.grow(need, st);
    cand_key.alloc(need);
    cand_val.alloc(need);
    word_list.ensure(need);  // victim words <= resident slots
    const int64_t words = scan_scratch_words(std::max<int64_t>(scan_n, need));
    if (partials.n < words) {
        partials.ensure(words);
        WC_CUDA(cudaMemsetAsync(partials.p, 0, 4 * partials.n, st));
    }
    slot_alloc = need;
    return true;
}

bool CacheStore::prepare_regions(int64_t stamp, int64_t n_blocks, DevBuf<uint32_t> &partials, cudaStream_t st) {
    if (vict_regions >= stamp) return false;
    const int64_t nwords = ceil_div(n_blocks, 32);
    const int64_t r = std::max<int64_t>(stamp, std::max<int64_t>(8, 2 * vict_regions));
    vict_bm.alloc(r * nwords);
    WC_CUDA(cudaMemsetAsync(vict_bm.p, 0, 4 * r * nwords, st));
    vict_regions = r;
    vict_sum.alloc(ceil_div(r * nwords, 32));
    WC_CUDA(cudaMemsetAsync(vict_sum.p, 0, 4 * vict_sum.n, st));
    const int64_t words = scan_scratch_words(r * nwords);
    if (partials.n < words) {
        partials.ensure(words);
        WC_CUDA(cudaMemsetAsync(partials.p, 0, 4 * partials.n, st));
    }
    return true;
}

// cache.ensure_resident (cache.py:66-111): stamp hits, list misses
// (ascending), then growth / victims / decode, all sized on the device
void CacheStore::enqueue_lookup(uint32_t *ctl, const uint32_t *active_ids, int64_t nmax, int32_t stamp,
                                int64_t n_blocks, uint32_t *partials, cudaStream_t st) {
    // hits stamped and misses listed in ascending id order (cache.py:69-78)
    // in one scan + compaction pass; the growth / eviction decisions
    // (k_cache_plan) run as its epilogue while the stamp histogram is kept on
    // the device
    if (stamp < kHistBins)
        compact_dev(LookupStamp{active_ids, slot_of_block.p, last_used.p, stamp, ctl + C_COUNT}, active_ids,
                    ctl + C_NACTB, nmax, miss_ids.p, ctl + C_NMISS, partials, st,
                    CachePlanEpilogue{ctl, ctl + C_COUNT, stamp, n_blocks, slot_alloc});
    else
        compact_dev(LookupStamp{active_ids, slot_of_block.p, last_used.p, stamp, nullptr}, active_ids, ctl + C_NACTB,
                    nmax, miss_ids.p, ctl + C_NMISS, partials, st);
}

void CacheStore::enqueue_slow_plan(uint32_t *ctl, int32_t stamp, bool any_active, int64_t n_blocks, cudaStream_t st) {
    stamp_hist.ensure(stamp + 1);
    WC_CUDA(cudaMemsetAsync(stamp_hist.p, 0, 4 * (stamp + 1), st));
    if (any_active) {
        launch_pdl(k_stamp_hist, grid_for(slot_alloc, 256), 256, 4 * (size_t)stamp, st, block_of_slot.p, last_used.p,
                   ctl, stamp, stamp_hist.p);
        WC_LAUNCH_CHECK();
    }
    launch_pdl(k_cache_plan, 1, 1, 0, st, ctl, stamp_hist.p, stamp, n_blocks, slot_alloc, false);
    WC_LAUNCH_CHECK();
}

void CacheStore::enqueue_insert(uint32_t *ctl, int64_t nmax, int32_t stamp, const Volume *vol, uint32_t *partials,
                                cudaStream_t st) {
    const int64_t nwords = ceil_div(vol->n_blocks, 32);
    if (stamp >= 2) {  // victims in (last_used, block_id) order: one extraction over the stamp regions
        launch_pdl(k_mark_victims, grid_for(slot_alloc, 256), 256, 0, st, block_of_slot.p, last_used.p, ctl, stamp,
                   nwords, vict_bm.p, vict_sum.p);
        WC_LAUNCH_CHECK();
        bitmap_extract_listed(vict_bm.p, vict_sum.p, (int64_t)stamp * nwords, slot_alloc, nwords, nullptr, cand_key.p,
                              ctl + C_NCAND, true, word_list.p, ctl + C_NLIST, partials, st,
                              ctl + C_VSUM);  // clears the regions
        launch_pdl(k_evict, grid_for(slot_alloc, 256), 256, 0, st, cand_key.p, ctl + C_NEVICT, slot_of_block.p,
                   block_of_slot.p, cand_val.p);
        WC_LAUNCH_CHECK();
    }
    // the misses' records decoded straight into their slots (free slots
    // first, then the victims in order, cache.py:97-103); the kernel also
    // initialises the slots this pass's growth brought into use
    launch_pdl(k_decode_insert, grid_for(nmax * 32, kDecWarps * 32, WC_DEC_CTAS), kDecWarps * 32, 0, st,
               vol->payload.p, vol->qbits, vol->stride, miss_ids.p, ctl, cand_val.p, slot_values.p, block_of_slot.p,
               last_used.p, slot_of_block.p, stamp);
    WC_LAUNCH_CHECK();
}

cudaEvent_t *Session::pass_events(int64_t p) {
    if (p >= kMaxPassLog) return nullptr;
    if (!pass_ev[p][0])
        for (auto &e : pass_ev[p]) WC_CUDA(cudaEventCreate(&e));
    return pass_ev[p];
}

// Host-side preparation of pass p (allocations happen here, never inside a
// captured pass): the victim regions must hold one bitmap per stamp a
// candidate can carry.  Reallocation invalidates the captured pass graphs.
void Session::prepare_pass(int64_t p) {
    pass_events(p);
    if (prepare_regions(p + 1, vol->n_blocks, partials, st)) drop_graphs();
}

void Session::drop_graphs() {
    for (auto &g : graphs) cudaGraphExecDestroy(g.exec);
    graphs.clear();
}

// Pass p as a CUDA graph: captured once per (p, kernel variants) and then
// replayed every frame.  Everything that changes between frames is read on
// the device (control block, FrameParams, device-derived scan epochs), so a
// replay is exactly the enqueued pass.  Modes with host reads inside a pass
// (entry grouping, more passes than histogram bins) are enqueued directly.
Session::PassGraph *Session::graph_for(int64_t p) {
    for (auto &x : graphs)
        if (x.p == p) return &x;
    const long long launches0 = g_launches.load();
    cudaGraph_t graph = nullptr;
    WC_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
        enqueue_pass(p);
    } catch (...) {
        cudaStreamEndCapture(st, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    WC_CUDA(cudaStreamEndCapture(st, &graph));
    PassGraph pg{p, nullptr, g_launches.load() - launches0};
    g_launches -= pg.kernels;  // captured, not launched
    const cudaError_t e = cudaGraphInstantiate(&pg.exec, graph, 0);
    cudaGraphDestroy(graph);
    WC_CUDA(e);
    WC_CUDA(cudaGraphUpload(pg.exec, st));
    graphs.push_back(pg);
    return &graphs.back();
}

// Capture (and upload) the graphs of the first passes ahead of time, so that
// no frame's device timeline waits for the host to capture a pass it reaches
// for the first time.
void Session::precapture(int64_t passes) {
    if (!use_graphs || group_entries) return;
    for (int64_t p = 0; p < passes && p + 2 <= kHistBins && p < kMaxPassLog; p++) {
        prepare_pass(p);
        graph_for(p);
    }
}

void Session::launch_pass(int64_t p) {
    if (!use_graphs || group_entries || p + 2 > kHistBins || p >= kMaxPassLog) {
        enqueue_pass(p);
        return;
    }
    prepare_pass(p);
    PassGraph *g = graph_for(p);
    cudaEvent_t *ev = pass_events(p);
    WC_CUDA(cudaEventRecord(ev[0], st));
    WC_CUDA(cudaGraphLaunch(g->exec, st));
    WC_CUDA(cudaEventRecord(ev[kStages], st));
    pass_staged[p] = false;
    g_launches += g->kernels;
}

// One pass of render_passes (engine.py:326-382), enqueued without any host
// read: every size comes from the device control block (Counter).  p is the
// pass index since the last reset; its cache stamp is p + 1.
namespace {
// scan epochs of the pass derived on the device (the pass may be captured
// into a graph and replayed; see scan_epoch)
struct DeviceEpochs {
    DeviceEpochs(const uint32_t *d_frame, uint32_t salt) {
        t_epoch_frame = d_frame;
        t_epoch_salt = salt;
    }
    ~DeviceEpochs() { t_epoch_frame = nullptr; }
};
}  // namespace

void Session::enqueue_pass(int64_t p) {
    const int64_t nwords = ceil_div(vol->n_blocks, 32);
    const int32_t stamp = (int32_t)(p + 1);
    pass_no = stamp;
    uint32_t *ctl = counters.p;
    const DeviceEpochs epochs(ctl + C_FRAME, (uint32_t)(p % 256) * 16u);
    uint32_t *alist = act_list[p & 1].p;
    cudaEvent_t *ev = pass_events(p);
    // stage events only when the pass is launched directly (a captured pass
    // is timed as a whole, around its graph launch)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    WC_CUDA(cudaStreamIsCapturing(st, &cap));
    const bool capturing = cap != cudaStreamCaptureStatusNone;
    pass_staged[std::min<int64_t>(p, kMaxPassLog - 1)] = !capturing;
    static const bool ktime_on = getenv("WAVECAST_KTIME") != nullptr;
    struct KTimeScope {  // per-launch events while this pass is enqueued directly
        KTimeScope(bool on, cudaStream_t s, std::vector<KTime> *v, int64_t p) {
            if (!on) return;
            t_ktime_stream = s;
            t_ktime = v;
            ktime_tick("pass", (int)p);
        }
        ~KTimeScope() {
            t_ktime_stream = nullptr;
            t_ktime = nullptr;
        }
    } kscope((ktime_on || kernel_profile) && !capturing, st, &ktime, p);
    auto mark = [&](int k) {
        if (ev && !capturing) WC_CUDA(cudaEventRecord(ev[k], st));
    };
    prepare_pass(p);
    mark(0);

    // traverse_to_next_blocks + fused visibility marking (one of the two
    // kernels runs, by the device n_act)
    TraverseArgs ta{};
    ta.rays = RayView{uniform_origin ? nullptr : origin.p, dir.p, t_enter.p, fparams.p};
    ta.t_exit = t_exit.p;
    ta.exited = exited.p;
    ta.coarse_cell = coarse_cell.p;
    ta.fine_cell = fine_cell.p;
    ta.coarse_tmax = coarse_tmax.p;
    ta.fine_tmax = fine_tmax.p;
    ta.act_list = alist;
    ta.cell_mask = cell_mask.p;
    ta.coarse_bm = coarse_bm.p;
    ta.fdx = vol->bdx;
    ta.fdy = vol->bdy;
    ta.fdz = vol->bdz;
    ta.cdx = vol->cdx;
    ta.cdy = vol->cdy;
    ta.cdz = vol->cdz;
    ta.block_slots = block_slots.p;
    ta.ray_slots = ray_slots.p;
    ta.emitted = emitted.p;
    ta.vis_bm = vis_bm.p;
    ta.work = ctl + C_WORK;
    ta.long_q = long_q.p;
    ta.n_long = ctl + C_NLONG;
    ta.ctl = ctl;
    // C_WORK, C_NLONG and C_NITEMS are zero here (reset, or the last pass_end)
    launch_traverse(ta, n, 0, st);
    mark(1);
    // Forked pass (WC_PASS_FORK): the entry offsets and the raytrace entries
    // depend only on the traversal and mark_blocks, so they run on the side
    // stream (own scan scratch) while the cache lookup, eviction and decode
    // run on the session stream; the branches join before the raytrace.
    const bool fork = WC_PASS_FORK && !group_entries;
    if (fork) {
        WC_CUDA(cudaEventRecord(ev_fork[0], st));
        WC_CUDA(cudaStreamWaitEvent(st_side, ev_fork[0], 0));
        scan_exclusive_dev(LoadU32{emitted.p}, ctl + C_NACT, n, entry_off.p, ctl + C_NENT, partials_side.p, st_side);
    } else {
        // entry compaction: exclusive scan of per-ray emitted counts
        scan_exclusive_dev(LoadU32{emitted.p}, ctl + C_NACT, n, entry_off.p, ctl + C_NENT, partials.p, st);
    }
    // visible ids (ascending) + active marking, from the maintained
    // summaries: the cost follows the non-zero bitmap words
#if WC_MARK_FUSED
    if (vol->bdx % 32 == 0) {  // one launch: visible ids, ranks and active ids from the visibility bitmap
        mark_extract(vis_bm.p, nwords, vol->bdx / 32, vol->bdy, vol->bdz, vis_word_off.p, visible_ids.p, ctl + C_NVIS,
                     active_ids.p, ctl + C_NACTB, partials.p, st);
    } else
#endif
    {
        bitmap_extract_dense(vis_bm.p, nwords, vis_word_off.p, visible_ids.p, ctl + C_NVIS, false, partials.p, st);
        launch_mark_active(visible_ids.p, ctl + C_NVIS, vis_bm.p, vol->bdx, vol->bdy, vol->bdz, n, act_bm.p, st);
        bitmap_extract_dense(act_bm.p, nwords, nullptr, active_ids.p, ctl + C_NACTB, true, partials.p, st);  // clears act_bm
    }
    const FastDiv ra_bdv_x((uint32_t)vol->bdx), ra_bdv_xy((uint32_t)vol->bdx * (uint32_t)vol->bdy);
    const BuildEntriesArgs be{ctl, alist, emitted.p, entry_off.p, block_slots.p, vis_bm.p, vis_word_off.p,
                              ent_key.p, group_entries ? ent_val.p : nullptr, ent_ray.p, ent_blk.p,
                              block_slots.p, ray_slots.p};
    if (fork) {  // the entries, keyed by visible rank, on the side branch
        WC_CUDA(cudaEventRecord(ev_fork[1], st));
        WC_CUDA(cudaStreamWaitEvent(st_side, ev_fork[1], 0));
        launch_pdl(k_rt_entries, grid_for(n, 256), 256, 0, st_side, be);
        WC_LAUNCH_CHECK();
        WC_CUDA(cudaEventRecord(ev_fork[2], st_side));
    }
    // cache.ensure_resident (cache.py:66-111), sized on the device
    const int64_t nmax = active_ids.n - 1;  // upper bound of the active-block count
    enqueue_lookup(ctl, active_ids.p, nmax, stamp, vol->n_blocks, partials.p, st);
    mark(2);
    if (stamp >= kHistBins) {  // > kHistBins passes: histogram over all stamps through the host (rare)
        read_counters(0, C_COUNT);
        enqueue_slow_plan(ctl, stamp, h_counters.p[C_NACT] != 0, vol->n_blocks, st);
    }
    enqueue_insert(ctl, nmax, stamp, vol, partials.p, st);
    if (corrupt) WC_CUDA(cudaMemsetAsync(slot_values.p, 0, 4 * 64 * slot_alloc, st));  // engine.py:338-339
    mark(3);

    // the raytrace's inputs: entries (keyed by visible rank) and contributor rows
    if (fork) {
        launch_pdl(k_rt_contrib, grid_for(n, 256), 256, 0, st, visible_ids.p, ctl + C_NVIS, slot_of_block.p, vol->bdx,
                   vol->bdy, vol->bdz, ra_bdv_x, ra_bdv_xy, contrib.p, ctl + C_ERR);
        WC_LAUNCH_CHECK();
        WC_CUDA(cudaStreamWaitEvent(st, ev_fork[2], 0));  // join: the entries are built
    } else {
        launch_pdl(k_rt_prep, grid_for(2 * n, 256), 256, 0, st, be, visible_ids.p, ctl + C_NVIS, slot_of_block.p,
                   vol->bdx, vol->bdy, vol->bdz, ra_bdv_x, ra_bdv_xy, contrib.p, ctl + C_ERR);
        WC_LAUNCH_CHECK();
    }
    // build_rt_inputs grouping (debug views only: the raytrace is correct on
    // ray order; the radix sort needs the entry and visible counts on the host)
    if (group_entries) {
        read_counters(0, C_COUNT);
        const int64_t n_ent = h_counters.p[C_NENT], nvis = h_counters.p[C_NVIS];
        if (n_ent > 0) {
            radix_sort_pairs(ent_key.p, ent_val.p, n_ent, bits_for((uint64_t)(nvis - 1)), rs, st);
            launch_pdl(k_run_offsets, grid_for(n_ent, 256), 256, 0, st, ent_key.p, n_ent, nvis, block_ray_off.p);
            WC_LAUNCH_CHECK();
        }
    }
    mark(4);
    RaytraceArgs ra{};
    ra.visible_ids = visible_ids.p;
    ra.vis_bm = vis_bm.p;
    ra.d_nvis = ctl + C_NVIS;
    ra.ent_key = ent_key.p;
    ra.ent_val = ent_val.p;
    ra.ent_ray = ent_ray.p;
    ra.ent_blk = ent_blk.p;
    ra.identity = !group_entries;
    ra.d_n_ent = ctl + C_NENT;
    ra.contrib = contrib.p;
    ra.slot_values = slot_values.p;
    ra.bdx = vol->bdx;
    ra.bdy = vol->bdy;
    ra.bdv_x = FastDiv((uint32_t)vol->bdx);
    ra.bdv_xy = FastDiv((uint32_t)vol->bdx * (uint32_t)vol->bdy);
    ra.bdz = vol->bdz;
    ra.nx = vol->nx;
    ra.ny = vol->ny;
    ra.nz = vol->nz;
    ra.rays = ta.rays;
    ra.fp = fparams.p;
    ra.rgbz = rgbz.p;
#if WC_RT_FUSED
    if (true) {
        SplitArgs sa{};
        sa.a = ra;
        launch_pdl(k_rt_fused, grid_for(n, 128, WC_RTFIND_GRID), 128, 0, st, sa);
        WC_LAUNCH_CHECK();
    } else
#endif
    if (WC_SPLIT_RAYTRACE) {
        SplitArgs sa{};
        sa.a = ra;
        sa.item_cap = 10 * n;  // <= 10 dual cells per entry (monotone ray in a 4^3 region)
        sa.item_info = item_info.p;
        sa.item_corners = item_corners.p;
        sa.item_t = item_t.p;
        sa.best = best.p;
        sa.n_items = ctl + C_NITEMS;
        launch_pdl(k_rt_find, grid_for(n, 128, WC_RTFIND_GRID), 128, 0, st, sa);
        WC_LAUNCH_CHECK();
        launch_pdl(k_rt_solve, grid_for(sa.item_cap, 128, WC_RAYTRACE_MIN_CTAS), 128, 0, st, sa);
        WC_LAUNCH_CHECK();
        launch_pdl(k_rt_shade, grid_for(n, 128, WC_RTSHADE_GRID), 128, 0, st, sa);
        WC_LAUNCH_CHECK();
    } else {
#if !WC_SPLIT_RAYTRACE
        launch_pdl(k_raytrace, grid_for(n, 128, 16), 128, 0, st, ra);
        WC_LAUNCH_CHECK();
#endif
    }
    mark(5);
    // composite + compaction of the surviving rays (next pass's O_Act); the
    // device picks thread or warp per ray by the pass's n_spec
    launch_pdl(k_composite, grid_for((speculation && max_spec >= (int)kWarpCompositeSpec ? 32 : 1) * n, 256), 256, 0, st,
               ctl, alist, emitted.p, entry_off.p, rgbz.p, exited.p, status.p, rgba.p, depth.p, keep.p, tgt.p,
               pix.p);
    WC_LAUNCH_CHECK();
    // next pass's active list; the pass record and the next pass's counts
    // (pass_end) as its epilogue
    compact_dev(LoadU32{keep.p}, alist, ctl + C_NACT, n, act_list[(p + 1) & 1].p, ctl + C_NACT_NEXT, partials.p, st,
                PassEndEpilogue{ctl, plog.p + std::min<int64_t>(p, kMaxPassLog - 1) * L_COUNT, n, speculation,
                                max_spec});
    mark(6);
}

// WAVECAST_KTIME: device time of every launch since the last report, by
// pass and launch site (the stream has been synchronised by the caller).
// Readable kernel name: the demangled symbol without its return type,
// namespace and parameter list (template arguments kept).
static std::string kernel_name(const void *func) {
    if (!func) return "?";
    const char *raw = nullptr;
    if (cudaFuncGetName(&raw, func) != cudaSuccess || !raw) return "?";
    std::string s = raw;
    int status = 0;
    if (char *dm = abi::__cxa_demangle(raw, nullptr, nullptr, &status)) {
        if (status == 0) s = dm;
        free(dm);
    }
    if (s.rfind("void ", 0) == 0) s = s.substr(5);
    int depth = 0;
    for (size_t i = 0; i < s.size(); i++) {  // cut the parameter list (the first '(' outside <>)
        if (s[i] == '<') depth++;
        if (s[i] == '>') depth--;
        if (s[i] == '(' && depth == 0) {
            s = s.substr(0, i);
            break;
        }
    }
    for (size_t q; (q = s.find("wc::")) != std::string::npos;) s.erase(q, 4);
    return s;
}

void Session::ktime_report() {
    if (ktime.empty()) return;
    static const bool print = getenv("WAVECAST_KTIME") != nullptr;
    int pass = -1, k = 0;
    for (size_t i = 0; i < ktime.size(); i++) {
        const KTime &t = ktime[i];
        if (std::string(t.file) == "pass") {
            pass = t.line;
            k = 0;
            continue;
        }
        float ms = 0.0f;
        if (i > 0) cudaEventElapsedTime(&ms, ktime[i - 1].ev, t.ev);
        const char *base = strrchr(t.file, '/');
        if (print)
            fprintf(stderr, "[ktime] pass %d #%02d %s:%d %.1f us\n", pass, k++, base ? base + 1 : t.file, t.line,
                    ms * 1e3f);
        if (kernel_profile) {
            const std::string key = std::to_string(pass) + "\t" + kernel_name(t.func);
            auto it = std::find_if(kstats.begin(), kstats.end(), [&](const auto &e) { return e.first == key; });
            if (it == kstats.end()) {
                kstats.push_back({key, KStat{}});
                it = kstats.end() - 1;
            }
            it->second.calls++;
            it->second.ms += ms;
        }
    }
    for (auto &t : ktime) cudaEventDestroy(t.ev);
    ktime.clear();
}

std::string Session::kernel_profile_text() const {
    std::string out;
    char buf[64];
    for (const auto &e : kstats) {
        snprintf(buf, sizeof(buf), "\t%lld\t%.6f\n", (long long)e.second.calls, e.second.ms);
        out += e.first + buf;
    }
    return out;
}

void Session::check_device_errors() {
    if (h_counters.p[C_ERR]) throw InvariantError("visible block not resident");
    if (h_counters.p[C_ERR_BUDGET]) throw InvariantError("slot budget exceeded");
    if (h_counters.p[C_ERR_CAND]) throw InvariantError("cache: fewer eviction candidates than needed");
    if (h_counters.p[C_ERR_CAP]) throw InvariantError("cache: capacity beyond the reserved slots");
}

// PassStats of pass p from its device record (h_plog holds it) and events.
void Session::collect_pass(int64_t p, PassStatsC &stats) {
    const uint32_t *r = h_plog.p + std::min<int64_t>(p, kMaxPassLog - 1) * L_COUNT;
    double ms_pass = 0.0;
    if (cudaEvent_t *ev = pass_events(p)) {
        if (pass_staged[p]) {
            for (int k = 0; k < kStages; k++) {
                float ms = 0.0f;
                WC_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
                stage_ms[k] += ms;
                pass_stage_ms[p][k] = ms;
                ms_pass += ms;
            }
        } else {  // graph replay: the pass as a whole
            float ms = 0.0f;
            WC_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[kStages]));
            ms_pass = ms;
            for (int k = 0; k < kStages; k++) pass_stage_ms[p][k] = 0.0;
            graph_ms += ms;
        }
        last_kernel_ms = (float)ms_pass;
        frame_end = ev[kStages];
    }
    stats.pass_index = p;
    stats.n_active_before = r[L_NACT];
    stats.n_spec = r[L_NSPEC];
    stats.visible_blocks = r[L_NVIS];
    stats.active_blocks = r[L_NACTB];
    stats.new_decompressed = r[L_NMISS];
    stats.evicted = r[L_NEVICT];
    stats.cache_slots = r[L_CAP];
    stats.n_entries = r[L_NENT];
    stats.n_active_after = r[L_NAFTER];
    stats.utilization = (double)r[L_NENT] / (double)n;
    stats.completeness = (double)(n - (int64_t)r[L_NAFTER]) / (double)n;
    stats.duration = ms_pass * 1e-3;  // device time of the pass
    // host mirrors for the stage views (wc_session_sizes & co.)
    last_n_spec = r[L_NSPEC];
    last_slots_used = (int64_t)r[L_NACT] * r[L_NSPEC];
    last_nvis = r[L_NVIS];
    last_nactb = r[L_NACTB];
    last_nent = r[L_NENT];
    last_nlong = r[L_NLONG];
    cap = r[L_CAP];
    phys = r[L_PHYS];
    hw = r[L_HW];
    n_act = r[L_NAFTER];
    static const bool trace = getenv("WAVECAST_TRACE") != nullptr;
    if (trace)
        fprintf(stderr, "[wavecast] pass %lld n_act %u n_spec %u entries %u visible %u active %u miss %u evict %u "
                        "items %u after %u cap %u phys %u gpu %.3f ms\n",
                (long long)p, r[L_NACT], r[L_NSPEC], r[L_NENT], r[L_NVIS], r[L_NACTB], r[L_NMISS], r[L_NEVICT],
                r[L_NITEMS], r[L_NAFTER], r[L_CAP], r[L_PHYS], ms_pass);
}

// render_passes step (engine.py:326-382): one pass, then its stats.
bool Session::pass(PassStatsC &stats) {
    if (n_act < 0) {  // the count the reset left on the device
        read_counters(0, C_COUNT);
        n_act = h_counters.p[C_NACT];
    }
    if (n_act == 0) return false;
    launch_pass(pass_index);
    WC_CUDA(cudaMemcpyAsync(h_plog.p, plog.p, 4 * L_COUNT * std::min<int64_t>(pass_index + 1, kMaxPassLog),
                            cudaMemcpyDeviceToHost, st));
    read_counters(0, C_COUNT);
    ktime_report();
    check_device_errors();
    collect_pass(pass_index, stats);
    pass_index++;
    return true;
}

// A whole frame: passes are enqueued in batches (first as many as the last
// frame needed) and the host looks at the device only between batches.  A
// pass enqueued after the last one finds no active ray and does no work.
int64_t Session::run_frame(PassStatsC *out, int64_t max_out) {
    int64_t k = 0;
    int64_t batch = std::max<int64_t>(1, frame_passes_hint);
    for (;;) {
        const int64_t p0 = pass_index;
        batch = p0 < kMaxPassLog ? std::min<int64_t>(batch, kMaxPassLog - p0) : 1;  // one log row per pass
        for (int64_t b = 0; b < batch; b++) {
            const int64_t p = p0 + b;
            launch_pass(p);
            if (p == fb_snap_pass && fb_rgba) enqueue_fb_snapshot(p);
        }
        // render_to_host's zero-copy patch rides behind every batch (it writes
        // final values only, so an early one is merely redundant): the batch
        // that turns out to be the last needs no second round trip
        if (fb_snapped && fb_patch_rgba) {
            WC_CUDA(cudaStreamWaitEvent(st, ev_fb_done, 0));
            launch_pdl(k_patch_host, grid_for(n, 256), 256, 0, st, counters.p, snap_list.p, rgba.p, depth.p,
                       fb_patch_rgba, fb_patch_depth);
            WC_LAUNCH_CHECK();
        }
        WC_CUDA(cudaMemcpyAsync(h_plog.p, plog.p, 4 * L_COUNT * std::min<int64_t>(p0 + batch, kMaxPassLog),
                                cudaMemcpyDeviceToHost, st));
        read_counters(0, C_COUNT);
        ktime_report();
        check_device_errors();
        bool done = false;
        for (int64_t b = 0; b < batch; b++) {
            const int64_t p = p0 + b;
            if (h_plog.p[std::min<int64_t>(p, kMaxPassLog - 1) * L_COUNT + L_NACT] == 0) {
                done = true;
                break;
            }
            PassStatsC st_{};
            collect_pass(p, st_);
            if (p < kMaxPassLog) {
                nact_hist[p] = st_.n_active_before;
                pass_ms_hist[p] = st_.duration * 1e3;
            }
            if (out && k < max_out) out[k] = st_;
            k++;
            pass_index++;
        }
        if (done || h_counters.p[C_NACT] == 0) break;
        batch = 1;
    }
    n_act = 0;
    frame_passes_hint = std::max<int64_t>(1, k);
    return k;
}

float Session::frame_ms() {
    float ms = 0.0f;
    if (pass_index == 0 || !frame_end) return 0.0f;
    WC_CUDA(cudaEventElapsedTime(&ms, ev_frame0, frame_end));
    return ms;
}

// After pass p: remember the rays still active (only their pixels can
// change from here on) and start copying the whole framebuffer to the host on
// a second stream while the remaining passes run.
void Session::ensure_copy_stream() {
    if (st_copy) return;
    WC_CUDA(cudaStreamCreateWithFlags(&st_copy, cudaStreamNonBlocking));
    WC_CUDA(cudaEventCreate(&ev_fb));
    WC_CUDA(cudaEventCreate(&ev_fb_done));
}

void Session::enqueue_fb_snapshot(int64_t p) {
    ensure_copy_stream();
    if (!snap_list.p) {
        snap_list.alloc(n);
        patch.alloc(n);
    }
    launch_pdl(k_snapshot_list, grid_for(n, 256), 256, 0, st, counters.p, act_list[(p + 1) & 1].p, snap_list.p);
    WC_LAUNCH_CHECK();
    WC_CUDA(cudaEventRecord(ev_fb, st));
    WC_CUDA(cudaStreamWaitEvent(st_copy, ev_fb, 0));
    WC_CUDA(cudaMemcpyAsync(fb_rgba, rgba.p, 4 * n, cudaMemcpyDeviceToHost, st_copy));
    WC_CUDA(cudaMemcpyAsync(fb_depth, depth.p, 4 * n, cudaMemcpyDeviceToHost, st_copy));
    WC_CUDA(cudaEventRecord(ev_fb_done, st_copy));
    fb_snapped = true;
}

// Host patch of the pixels still active when the framebuffer copy started:
// a few persistent threads share the (ascending) patch list, so a copy
// started two passes before the end (~60K pixels at C3) is patched in well
// under its copy time.  Workers sleep on a condition variable between frames.
namespace {
struct PatchPool {
    std::vector<std::thread> workers;
    std::mutex m;
    std::condition_variable cv;
    uint64_t job = 0;
    bool stop = false;
    const uint4 *src = nullptr;
    uint32_t *rgba = nullptr;
    float *depth = nullptr;
    int64_t n = 0;
    int parts = 1;
    std::atomic<int> left{0};

    static void apply(const uint4 *q, int64_t b, int64_t e, uint32_t *rgba, float *depth) {
        for (int64_t i = b; i < e; i++) rgba[q[i].x] = q[i].y;
        for (int64_t i = b; i < e; i++) std::memcpy(depth + q[i].x, &q[i].z, 4);
    }
    void part(int k) { apply(src, n * k / parts, n * (k + 1) / parts, rgba, depth); }
    void run(const uint4 *q, int64_t count, uint32_t *rgba_, float *depth_) {
        const int want = count < 16384 ? 1 : (int)std::min<int64_t>(8, count / 8192);
        const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
        const int p = std::max(1, std::min(want, hw / 2));
        if (p == 1) {
            apply(q, 0, count, rgba_, depth_);
            return;
        }
        if ((int)workers.size() < p - 1) {
            for (int k = (int)workers.size(); k < p - 1; k++)
                workers.emplace_back([this, k] {
                    uint64_t seen = 0;
                    for (;;) {
                        std::unique_lock<std::mutex> lk(m);
                        cv.wait(lk, [&] { return stop || job != seen; });
                        if (stop) return;
                        seen = job;
                        const bool mine = k + 1 < parts;
                        lk.unlock();
                        if (mine) {
                            part(k + 1);
                            left.fetch_sub(1, std::memory_order_acq_rel);
                        }
                    }
                });
        }
        {
            std::lock_guard<std::mutex> lk(m);
            src = q;
            rgba = rgba_;
            depth = depth_;
            n = count;
            parts = p;
            left.store(p - 1, std::memory_order_release);
            job++;
        }
        cv.notify_all();
        part(0);
        while (left.load(std::memory_order_acquire) > 0) std::this_thread::yield();
    }
    ~PatchPool() {
        {
            std::lock_guard<std::mutex> lk(m);
            stop = true;
        }
        cv.notify_all();
        for (auto &t : workers) t.join();
    }
};
PatchPool &patch_pool() {
    static PatchPool p;
    return p;
}
std::mutex g_patch_mutex;  // one frame's patch at a time (sessions on several host threads)
}  // namespace

int64_t Session::render_to_host(const CameraParams *cam, double iso_, PassStatsC *out, int64_t max_out,
                                uint32_t *rgba_host, float *depth_host) {
    reset(cam, iso_);
    // Start the bulk copy after the pass that minimises (from the last
    // frame's pass times) the copy time left exposed after the frame plus the
    // host patching of the pixels still active then (~5 ns each); the first
    // frame of a session has no history and copies at the end.
    fb_snap_pass = -1;
    const double copy_ms = fb_copy_ms > 0.0 ? fb_copy_ms : 8.0 * (double)n / 50e6;
    // host patch cost per still-active pixel (ms): ~7 ns on one thread,
    // spread over the patch pool's threads for large patches
    const double patch_ms_per_px = zero_copy_patch ? 1e-6 : 3e-6;  // (measured at C3: the patch gather, its read-back and the threaded scatter of 60K pixels ~0.2 ms)
    int64_t last = 0;
    while (last < kMaxPassLog && nact_hist[last] > 0) last++;
    double best_cost = copy_ms, tail_ms = 0.0;
    for (int64_t p = last - 2; p >= 0; p--) {
        tail_ms += pass_ms_hist[p + 1];
        const double cost = std::max(0.0, copy_ms - tail_ms) + patch_ms_per_px * (double)nact_hist[p + 1];
        if (cost < best_cost) {
            best_cost = cost;
            fb_snap_pass = p;
        }
    }
    static const char *force_snap = getenv("WAVECAST_SNAP_PASS");  // diagnostic: copy after this pass
    if (force_snap && *force_snap) fb_snap_pass = atoi(force_snap);
    fb_rgba = rgba_host;
    fb_depth = depth_host;
    fb_snapped = false;
    // pinned (device-mapped) host buffers: the GPU writes the patch itself
    // once the bulk copy has landed; else gather, read back, patch on the host
    fb_patch_rgba = zero_copy_patch ? static_cast<uint32_t *>(mapped_device_ptr(rgba_host)) : nullptr;
    fb_patch_depth = fb_patch_rgba ? static_cast<float *>(mapped_device_ptr(depth_host)) : nullptr;
    if (!fb_patch_depth) fb_patch_rgba = nullptr;
    int64_t k = 0;
    const auto t0 = std::chrono::steady_clock::now();
    try {
        k = run_frame(out, max_out);
    } catch (...) {
        fb_rgba = nullptr;
        fb_patch_rgba = nullptr;
        fb_patch_depth = nullptr;
        if (st_copy) cudaStreamSynchronize(st_copy);
        throw;
    }
    fb_rgba = nullptr;
    fb_depth = nullptr;
    if (!fb_snapped) {  // no snapshot this frame: the whole framebuffer now
        fb_patch_rgba = nullptr;
        fb_patch_depth = nullptr;
        download_framebuffer(reinterpret_cast<uint8_t *>(rgba_host), depth_host);
        return k;
    }
    const int64_t nsnap = h_counters.p[C_NSNAP];  // read with the frame's last counters
    const bool zc = fb_patch_rgba != nullptr;  // patched by the GPU behind the last batch (run_frame)
    fb_patch_rgba = nullptr;
    fb_patch_depth = nullptr;
    if (nsnap > 0) {
        if (!zc) {
            launch_pdl(k_gather_patch, grid_for(nsnap, 256), 256, 0, st, counters.p, snap_list.p, rgba.p, depth.p,
                       patch.p);
            WC_LAUNCH_CHECK();
            h_patch.ensure_host(nsnap);
            WC_CUDA(cudaMemcpyAsync(h_patch.p, patch.p, sizeof(uint4) * nsnap, cudaMemcpyDeviceToHost, st));
        }
    }
    WC_CUDA(cudaStreamSynchronize(st));
    WC_CUDA(cudaEventSynchronize(ev_fb_done));  // the bulk copy has landed before it is patched
    float cms = 0.0f;
    if (cudaEventElapsedTime(&cms, ev_fb, ev_fb_done) == cudaSuccess && cms > 0.0f) fb_copy_ms = cms;
    const auto t2 = std::chrono::steady_clock::now();
    if (nsnap > 0 && !zc) {
        std::lock_guard<std::mutex> lk(g_patch_mutex);
        patch_pool().run(h_patch.p, nsnap, rgba_host, depth_host);
    }
    static const bool trace = getenv("WAVECAST_TRACE") != nullptr;
    if (trace) {
        const auto t3 = std::chrono::steady_clock::now();
        fprintf(stderr, "[wavecast] render_to_host: snap after pass %lld, %lld patched; frame+patch %.3f ms, scatter %.3f ms\n",
                (long long)fb_snap_pass, (long long)nsnap,
                std::chrono::duration<double>(t2 - t0).count() * 1e3,
                std::chrono::duration<double>(t3 - t2).count() * 1e3);
    }
    return k;
}

int64_t Session::snapshot_async(uint32_t *rgba_host, float *depth_host) {
    ensure_copy_stream();
    const int k = (int)(snap_seq % kSnapRing);
    if (!snap_ring[k].p) {
        snap_ring[k].alloc(2 * n);
        WC_CUDA(cudaEventCreateWithFlags(&snap_ready[k], cudaEventDisableTiming));
        WC_CUDA(cudaEventCreateWithFlags(&snap_done[k], cudaEventDisableTiming));
    } else {
        WC_CUDA(cudaStreamWaitEvent(st, snap_done[k], 0));  // the slot's previous host copy has landed
    }
    WC_CUDA(cudaMemcpyAsync(snap_ring[k].p, rgba.p, 4 * n, cudaMemcpyDeviceToDevice, st));
    WC_CUDA(cudaMemcpyAsync(snap_ring[k].p + n, depth.p, 4 * n, cudaMemcpyDeviceToDevice, st));
    WC_CUDA(cudaEventRecord(snap_ready[k], st));
    WC_CUDA(cudaStreamWaitEvent(st_copy, snap_ready[k], 0));
    WC_CUDA(cudaMemcpyAsync(rgba_host, snap_ring[k].p, 4 * n, cudaMemcpyDeviceToHost, st_copy));
    WC_CUDA(cudaMemcpyAsync(depth_host, snap_ring[k].p + n, 4 * n, cudaMemcpyDeviceToHost, st_copy));
    WC_CUDA(cudaEventRecord(snap_done[k], st_copy));
    return snap_seq++;
}

// The slot's event may since have been recorded for a later snapshot: the
// copy stream is in order, so that one completing implies this one did.
void Session::snapshot_wait(int64_t ticket) {
    if (ticket < 0 || ticket >= snap_seq) throw UsageError("no such snapshot");
    WC_CUDA(cudaEventSynchronize(snap_done[ticket % kSnapRing]));
}

void Session::sync_all() {
    WC_CUDA(cudaStreamSynchronize(st));
    if (st_copy) WC_CUDA(cudaStreamSynchronize(st_copy));
}

void Session::download_framebuffer(uint8_t *rgba_host, float *depth_host) {
    if (rgba_host) WC_CUDA(cudaMemcpyAsync(rgba_host, rgba.p, 4 * n, cudaMemcpyDeviceToHost, st));
    if (depth_host) WC_CUDA(cudaMemcpyAsync(depth_host, depth.p, 4 * n, cudaMemcpyDeviceToHost, st));
    WC_CUDA(cudaStreamSynchronize(st));
}

void Session::pack_framebuffer(uint32_t *dst, int64_t stride) {
    WC_CUDA(cudaMemcpyAsync(dst, rgba.p, 4 * n, cudaMemcpyDeviceToDevice, st));
    WC_CUDA(cudaMemcpyAsync(dst + stride, depth.p, 4 * n, cudaMemcpyDeviceToDevice, st));
}

__global__ void k_scatter_pixels(const uint32_t *packed, int64_t stride, const int64_t *ids, int64_t n, uint32_t *rgba,
                                 uint32_t *depth) {
    pdl_wait();
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = ids[j];
        if (p < 0) continue;
        const int64_t b = j / stride, i = j - b * stride;
        rgba[p] = packed[2 * stride * b + i];
        depth[p] = packed[2 * stride * b + stride + i];
    }
}

void scatter_pixels(const uint32_t *packed, int64_t stride, const int64_t *ids, int64_t n, uint32_t *rgba,
                    uint32_t *depth, cudaStream_t st) {
    if (n <= 0) return;
    launch_pdl(k_scatter_pixels, grid_for(n, 256), 256, 0, st, packed, stride, ids, n, rgba, depth);
    WC_LAUNCH_CHECK();
}

void Session::copy_framebuffer_device(void *rgba_dst, void *depth_dst) {
    if (rgba_dst) WC_CUDA(cudaMemcpyAsync(rgba_dst, rgba.p, 4 * n, cudaMemcpyDeviceToDevice, st));
    if (depth_dst) WC_CUDA(cudaMemcpyAsync(depth_dst, depth.p, 4 * n, cudaMemcpyDeviceToDevice, st));
    WC_CUDA(cudaStreamSynchronize(st));
}

}  // namespace wc
