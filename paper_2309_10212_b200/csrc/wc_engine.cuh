// wc_engine.cuh -- the per-pass wavefront session (engine.py:308-382).
#pragma once

#include <string>
#include <vector>

#include "wc_common.cuh"
#include "wc_prims.cuh"
#include "wc_volume.cuh"

namespace wc {

struct CameraParams {  // traversal.py:65-70, :111 (basis computed on the host)
    double eye[3], look[3], right[3], up[3];
    double tan_half;
    int32_t img_w, img_h;
};

struct PassStatsC {  // engine.py:66-77 PassStats (+ evicted, n_entries)
    int64_t pass_index, n_active_before, n_spec, visible_blocks, active_blocks, new_decompressed, evicted,
        cache_slots, n_entries, n_active_after;
    double utilization, completeness, duration;
};

constexpr int kHistBins = 64;  // stamp histogram bins kept after the counters (passes < 64)

// Device control block: every count a pass needs lives here, so a pass is
// enqueued without host round trips (each kernel reads its sizes).
enum Counter : int {
    C_NACT = 0,   // active rays of the current pass (engine.py:331)
    C_NENT,       // ray-block entries this pass
    C_NVIS,       // visible blocks
    C_NACTB,      // active blocks
    C_NMISS,      // cache misses
    C_NFREE,      // free slots (cap - hw)
    C_NCAND,      // eviction candidates listed (bucket extraction count)
    C_ERR,        // device-side invariant failure: visible block not resident
    C_HW,         // occupied cache slots: free slots are the suffix [hw, cap)
    C_WORK,       // persistent traversal work counter
    C_NITEMS,     // candidate cells listed by the two-phase raytrace
    C_NACT_NEXT,  // active rays after composite (next pass's n_act)
    C_NSPEC,      // n_spec of the current pass (engine.py:91-94)
    C_CAP,        // logical cache capacity (cache.py:74-75)
    C_PHYS,       // slots with initialised maps: min(cap, n_blocks)
    C_PHYS_OLD,   // C_PHYS before this pass's growth
    C_NEVICT,     // victims this pass
    C_LSTAR,      // last stamp bucket the victims reach (0xFFFFFFFF: none)
    C_HW_NEXT,    // occupied slots after this pass's inserts
    C_ERR_BUDGET, // device-side invariant failure: slot budget exceeded
    C_ERR_CAND,   // device-side invariant failure: fewer eviction candidates than needed
    C_ERR_CAP,    // logical capacity beyond the reserved slots (host must reserve more)
    C_NSNAP,      // rays still active when the framebuffer read-back started
    C_NLIST,      // non-zero bitmap words listed by bitmap_extract_listed
    C_FRAME,      // frame counter (device-derived scan epochs)
    C_VSUM,       // victim-region summary words to list this pass (0: no eviction)
    C_NLONG,      // rays handed from the thread-per-ray traversal to k_traverse_long this pass
    C_COUNT
};

// Per-pass record written on the device by pass_end (PassStats fields).
enum PassLog : int {
    L_NACT = 0, L_NSPEC, L_NVIS, L_NACTB, L_NMISS, L_NEVICT, L_CAP, L_NENT, L_NAFTER, L_NITEMS, L_PHYS, L_HW,
    L_NLONG,  // rays the thread-per-ray traversal handed to k_traverse_long
    L_COUNT
};

// Ray state as the kernels read it (origin per ray, or the shared eye).
struct RayView {
    const double *origin;  // nullable -> eye
    const double *dir, *t_enter;
    const double *eye;  // FrameParams (device): the camera eye of this frame
    double ex = 0.0, ey = 0.0, ez = 0.0;
    __device__ __forceinline__ void bind() {  // once per kernel: the eye into registers
        if (!origin) {
            ex = eye[0];
            ey = eye[1];
            ez = eye[2];
        }
    }
    __device__ __forceinline__ void load(int64_t r, double o[3], double d[3]) const {
        if (origin) {
            o[0] = origin[3 * r];
            o[1] = origin[3 * r + 1];
            o[2] = origin[3 * r + 2];
        } else {
            o[0] = ex;
            o[1] = ey;
            o[2] = ez;
        }
        d[0] = dir[3 * r];
        d[1] = dir[3 * r + 1];
        d[2] = dir[3 * r + 2];
    }
};

struct TraverseArgs {
    RayView rays;
    const double *t_exit;
    uint8_t *exited;
    uint32_t *coarse_cell, *fine_cell;
    double *coarse_tmax, *fine_tmax;
    const uint32_t *act_list;
    int64_t n_act;
    int n_spec;
    const uint32_t *coarse_bm;                // per-iso coarse range-test bitmap (k_iso_bitmap)
    const unsigned long long *cell_mask;  // per-iso fine tests, one word per coarse cell (k_iso_cell_mask)
    int fdx, fdy, fdz, cdx, cdy, cdz;
    FastDiv cdv_x, cdv_xy, fdv_x, fdv_xy;  // cdx, cdx cdy, fdx, fdx fdy (set by launch_traverse)
    double iso;
    uint32_t *block_slots, *ray_slots, *emitted, *vis_bm;
    uint32_t *work;        // persistent-kernel ray counter (zeroed per pass)
    // long-ray hand-off (nullable): thread-per-ray lanes still walking after
    // WC_DEFER_ITERS iterations save their iterator, queue the ray here and
    // k_traverse_long finishes it warp per ray (passes of <= WC_DEFER_MAX_ACT rays)
    uint32_t *long_q, *n_long;
    const uint32_t *ctl;   // control block: n_act and n_spec of the pass (Counter)
    // the kernel variant is chosen on the device from the pass's n_act:
    // warp per ray when n_act <= warp_max, thread per ray otherwise (both
    // kernels are launched; the other one returns at once)
    uint32_t warp_max;
    uint32_t warp_max_long;  // ... or n_act <= warp_max_long when n_spec >= WC_WARP_LONG_SPEC (long rays)
    bool warp_only;  // passes with more rays are another kernel's (k_traverse_q builds)
};

// Traversal kernel launch: both variants, the device picks by its n_act
// (variant 0); variant 1 / 2 forces thread-per-ray / warp-per-ray.
void launch_traverse(TraverseArgs ta, int64_t n_grid, int variant, cudaStream_t st);
// +octant active marking from the visible ids (engine.py:107-117)
void launch_mark_active(const uint32_t *visible_ids, const uint32_t *d_nvis, const uint32_t *vis_bm, int bdx, int bdy,
                        int bdz, int64_t n_max, uint32_t *act_bm, cudaStream_t st);
// per-iso coarse range-test bitmap (traversal.py:357)
void launch_iso_bitmap(const double2 *mm, int64_t n, double iso, uint32_t *bm, cudaStream_t st);

// BlockCache device state (cache.py:21-111): the slot pool, both maps, the
// miss / victim lists and the per-stamp victim regions, with the launches of
// one ensure_resident.  Used by the render session (one update per pass,
// control block shared with the pass) and by the standalone stage-level
// BlockCache (wc_cache_*).  Sizes live in the control block `ctl`.
struct CacheStore {
    int64_t slot_alloc = 0;  // allocated slots (the session reserves its largest capacity up front)
    DevBuf<float> slot_values;
    DevBuf<int32_t> block_of_slot, last_used, slot_of_block;
    DevBuf<uint32_t> miss_ids, cand_key, cand_val;
    DevBuf<uint32_t> vict_bm;    // per-stamp block bitmaps for victim selection
    DevBuf<uint32_t> vict_sum;   // summary of the victim regions
    DevBuf<uint32_t> word_list;  // non-zero words listed by bitmap_extract_listed
    int64_t vict_regions = 0;
    DevBuf<uint32_t> stamp_hist;  // > kHistBins passes only

    // slot storage for `need` slots (contents kept); scan scratch grown for
    // scans over `scan_n` elements.  True when buffers moved.
    bool reserve_store(int64_t need, int64_t scan_n, DevBuf<uint32_t> &partials, cudaStream_t st);
    // victim regions for stamps [0, stamp]; true when reallocated
    bool prepare_regions(int64_t stamp, int64_t n_blocks, DevBuf<uint32_t> &partials, cudaStream_t st);
    // stamp the hits, list the misses (ascending); with stamp < kHistBins the
    // growth / eviction plan runs as the epilogue of the miss compaction
    void enqueue_lookup(uint32_t *ctl, const uint32_t *active_ids, int64_t nmax, int32_t stamp, int64_t n_blocks,
                        uint32_t *partials, cudaStream_t st);
    // stamp >= kHistBins: the plan from a full recount of the stamps
    // (any_active: the pass has work; read on the host by the caller)
    void enqueue_slow_plan(uint32_t *ctl, int32_t stamp, bool any_active, int64_t n_blocks, cudaStream_t st);
    // victims in (last_used, block_id) order, eviction, decode into the slots
    void enqueue_insert(uint32_t *ctl, int64_t nmax, int32_t stamp, const Volume *vol, uint32_t *partials,
                        cudaStream_t st);
};

// Per-session device state.  Layout (N = rays in this session):
//   ray SoA: dir f64[N*3] (origin f64[N*3] only for arbitrary rays; camera
//   rays share `eye`), t_enter/t_exit f64[N], status/exited u8[N],
//   coarse/fine cell u32[N], coarse/fine tmax f64[N*3]          (122 B/ray)
//   act_list u32[N] x2 (ping-pong compacted active rays, ascending)
//   slots: block_slots/ray_slots u32[N] (prefix n_act*n_spec used)
//   entries: key/val/ray u32[N], rgbz float4[N]
//   bitmaps: vis/act u32[ceil(n_blocks/32)] (15.7 MB at 8.05B voxels)
//   cache: slot_values f32[phys*64], block_of_slot/last_used i32[phys],
//          slot_of_block i32[n_blocks]
//   framebuffer: rgba u32[N] (packed RGBA8), depth f32[N]
// Full-frame RGBA8 + depth on one GPU that every rank's session writes its
// final pixels into (multi-GPU frame assembly over peer memory): created
// (and owned) by rank 0, opened by the others through CUDA IPC handles.
struct FrameTarget {
    DevBuf<uint32_t> rgba;
    DevBuf<float> depth;
    uint32_t *p_rgba = nullptr;  // device addresses in this process (own or opened)
    float *p_depth = nullptr;
    bool opened = false;
    int64_t npix = 0;
    FrameTarget() = default;
    FrameTarget(const FrameTarget &) = delete;
    FrameTarget &operator=(const FrameTarget &) = delete;
    ~FrameTarget();
    void create(int64_t n);
    void ipc_handles(void *out) const;  // 2 x cudaIpcMemHandle_t (128 bytes)
    void open(const void *handles, int64_t n);
};

struct Session : CacheStore {
    Volume *vol = nullptr;
    cudaStream_t st = nullptr;
    int64_t n = 0;
    double iso = 0.0;
    int speculation = 1, max_spec = 64, corrupt = 0;
    double base[3] = {0.85, 0.85, 0.85};
    bool uniform_origin = true;
    // Stable sort of entries by block before the raytrace (build_rt_inputs,
    // engine.py:121-149).  Off by default: the thread-per-entry raytrace gets
    // its block locality from ray order + L1 (measured 1.70 vs 1.69 ms at C3)
    // and the sort costs 0.5 ms/frame; on for the reference PassBuffers views.
    bool group_entries = false;
    bool use_graphs = true;  // replay passes as captured CUDA graphs (WAVECAST_NO_GRAPHS=1: plain launches)
    double eye[3] = {0, 0, 0};

    DevBuf<double> origin, dir, t_enter, t_exit, coarse_tmax, fine_tmax;
    DevBuf<uint8_t> status, exited;
    DevBuf<uint32_t> coarse_cell, fine_cell;
    DevBuf<uint32_t> act_list[2], keep, emitted, entry_off, long_q;
    DevBuf<uint32_t> block_slots, ray_slots;
    DevBuf<uint32_t> ent_key, ent_val, ent_ray, ent_blk;
    DevBuf<float4> rgbz;
    DevBuf<int4> contrib;  // 8 contributor slots per visible block
    DevBuf<uint4> item_info;  // two-phase raytrace work list (SplitArgs)
    DevBuf<float4> item_corners;
    DevBuf<unsigned long long> best;
    DevBuf<double> item_t;
    DevBuf<uint32_t> vis_bm, act_bm, vis_word_off;
    DevBuf<uint32_t> coarse_bm;            // per-iso coarse range-test bitmap, rebuilt at every reset
    DevBuf<unsigned long long> cell_mask;  // per-iso fine range tests, 64 per coarse cell
    DevBuf<uint32_t> visible_ids, block_ray_off, active_ids;
    DevBuf<uint32_t> rgba;
    DevBuf<float> depth;
    // cache (cache.py)
    int64_t cap = 0, phys = 0, hw = 0;
    int32_t pass_no = 0;
    // scratch
    DevBuf<uint32_t> counters, partials, partials_side;
    PinnedBuf<uint32_t> h_counters;
    RadixScratch rs;
    cudaEvent_t ev_frame0 = nullptr, ev_reset_end = nullptr;
    cudaStream_t st_side = nullptr;  // reset: per-iso range tests overlapped with the ray setup
    cudaEvent_t ev_side = nullptr;
    cudaEvent_t ev_fork[3] = {};  // forked pass: after traverse, after mark_blocks, entries built
    static constexpr int kStages = 6;  // traverse, mark, cache, raytrace inputs (+ grouping), raytrace, composite
    double stage_ms[kStages] = {};
    static constexpr int kMaxPassLog = 128;
    double pass_stage_ms[kMaxPassLog][kStages] = {};  // per-pass stage device ms since reset
    bool pass_staged[kMaxPassLog] = {};  // pass timed per stage (launched directly) or as a whole (graph)
    double graph_ms = 0.0;               // device ms of the graph-replayed passes since reset
    DevBuf<uint32_t> pix;
    DevBuf<double> dir_in;
    CameraParams cam_params{};
    int64_t init_cap = 0;

    int64_t n_act = 0, pass_index = 0;
    int64_t frame_passes_hint = 1;  // passes to enqueue before the first host check of a frame
    int64_t nact_hist[kMaxPassLog] = {};  // active rays per pass of the last frame (variant guesses)
    double pass_ms_hist[kMaxPassLog] = {};  // device ms per pass of the last frame (read-back scheduling)
    DevBuf<uint32_t> plog;          // kMaxPassLog x L_COUNT per-pass records (device)
    PinnedBuf<uint32_t> h_plog;
    DevBuf<double> fparams;         // FrameParams: eye[3], iso, base colour[3] (written by k_frame_start)
    DevBuf<unsigned long long> tgt;  // frame target {rgba, depth} device addresses (0: none), set_frame_target
    uint32_t frame_no = 0;
    int64_t last_slots_used = 0, last_nvis = 0, last_nactb = 0, last_nent = 0, last_nlong = 0;
    int64_t last_n_spec = 1;
    float last_kernel_ms = 0.0f;
    std::vector<KTime> ktime;  // WAVECAST_KTIME: per-launch events of the directly enqueued passes
    void ktime_report();
    // per-kernel device time of the directly enqueued passes (graphs off),
    // accumulated while kernel_profile is on: "pass\tkernel\tcalls\tms" rows
    bool kernel_profile = false;
    struct KStat {
        int64_t calls = 0;
        double ms = 0.0;
    };
    std::vector<std::pair<std::string, KStat>> kstats;  // key "pass\tkernel"
    std::string kernel_profile_text() const;

    Session(Volume *v, const CameraParams *cam, const uint32_t *pixel_ids, int64_t n_rays, const double *origins,
            const double *dirs, double iso, int speculation, int max_spec, int64_t cache_capacity, int corrupt);
    ~Session();
    bool pass(PassStatsC &st);
    // a whole frame (passes until no ray is active), host-checked once per
    // batch of enqueued passes; stats of the passes that ran -> out
    int64_t run_frame(PassStatsC *out, int64_t max_out);
    // reset + run_frame with the framebuffer read back into pinned host
    // memory, the bulk of it overlapped with the tail passes
    int64_t render_to_host(const CameraParams *cam, double iso, PassStatsC *out, int64_t max_out,
                           uint32_t *rgba_host, float *depth_host);
    void reset(const CameraParams *cam, double iso);
    void reset_part(const CameraParams *cam, double iso, int64_t part, int64_t parts);
    void mask_buffers(int64_t parts, int64_t &chunk_words);  // sized for `parts` slices of chunk_words
    float frame_ms();  // device time from the last reset to the end of the last pass
    void download_framebuffer(uint8_t *rgba_host, float *depth_host);
    // Streamed per-pass snapshots (render_passes, Framebuffer.snapshot,
    // engine.py:62-63): a device-to-device copy of the framebuffer into a
    // ring slot on the session stream, then its copy to the caller's host
    // buffers on the copy stream, overlapped with the passes that follow.
    // Returns a ticket; snapshot_wait(ticket) blocks until that copy landed.
    int64_t snapshot_async(uint32_t *rgba_host, float *depth_host);
    void snapshot_wait(int64_t ticket);
    void sync_all();  // session and copy streams
    void copy_framebuffer_device(void *rgba_dst, void *depth_dst);
    // rgba words at dst[0, n), depth bits at dst[stride, stride + n) (stride
    // >= n), stream-ordered on the session stream (no host sync): the send
    // buffer of a tile gather
    void set_frame_target(const FrameTarget *t);
    void pack_framebuffer(uint32_t *dst, int64_t stride);

    double reset_device_ms();  // device time of the last reset, once it has run
    int64_t active_count();    // active rays now (read from the device after a reset)

   private:
    void read_counters(int first, int count);
    void enqueue_pass(int64_t p);
    void prepare_pass(int64_t p);
    void launch_pass(int64_t p);  // enqueue_pass through a cached CUDA graph
    void drop_graphs();
    struct PassGraph {
        int64_t p;
        cudaGraphExec_t exec;
        long long kernels;  // kernels per replay (the launch counter)
    };
    std::vector<PassGraph> graphs;
    PassGraph *graph_for(int64_t p);  // captured on first use
    static constexpr int64_t kPrecapturePasses = 8;
    void precapture(int64_t passes);
    void collect_pass(int64_t p, PassStatsC &stats);
    void check_device_errors();
    void reserve_slots(int64_t need);
    cudaEvent_t *pass_events(int64_t p);  // stage events of pass p (nullptr past kMaxPassLog)
    cudaEvent_t pass_ev[kMaxPassLog][kStages + 1] = {};
    cudaEvent_t frame_end = nullptr;      // end of the last pass that ran
    // overlapped read-back (render_to_host)
    void enqueue_fb_snapshot(int64_t p);
    cudaStream_t st_copy = nullptr;
    cudaEvent_t ev_fb = nullptr, ev_fb_done = nullptr;
    int64_t fb_snap_pass = -1;  // pass after which the bulk copy starts (-1: none)
    bool fb_snapped = false;
    double fb_copy_ms = 0.0;  // measured duration of the last bulk copy
    uint32_t *fb_rgba = nullptr;
    float *fb_depth = nullptr;
    DevBuf<uint32_t> snap_list;
    static constexpr int kSnapRing = 3;
    DevBuf<uint32_t> snap_ring[kSnapRing];  // rgba words (n) + depth bits (n) per slot
    cudaEvent_t snap_ready[kSnapRing] = {}, snap_done[kSnapRing] = {};
    int64_t snap_seq = 0;
    void ensure_copy_stream();
    DevBuf<uint4> patch;
    PinnedBuf<uint4> h_patch;
    // render_to_host patches pinned host framebuffers from the GPU (zero-copy
    // writes); WAVECAST_HOST_PATCH=1 patches on the host instead
    bool zero_copy_patch = getenv("WAVECAST_HOST_PATCH") == nullptr;
    uint32_t *fb_patch_rgba = nullptr;  // device addresses of this frame's mapped host framebuffer
    float *fb_patch_depth = nullptr;
};

// Finished tiles into the frame (multi-GPU gather): for every
// source b in [0, n / stride) and i < stride, pixel ids[b*stride + i] (< 0:
// padding) gets packed[2*stride*b + i] (RGBA8 word) and
// packed[2*stride*b + stride + i] (depth bits).
void scatter_pixels(const uint32_t *packed, int64_t stride, const int64_t *ids, int64_t n, uint32_t *rgba,
                    uint32_t *depth, cudaStream_t st);

// Brute-force oracle on the device (oracle.py:42-122): every ray marches all
// dual cells of the fully decoded volume.  d_values dense float32 x-fastest.
void reference_render_device(const float *d_values, int nx, int ny, int nz, const double *d_origin,
                             const double *d_dir, int64_t n, double iso, double br, double bg, double bb,
                             uint32_t *d_rgba, float *d_depth, cudaStream_t st);

// Ray setup alone (traversal.py:105-187) for parity tests.
void init_rays_device(const CameraParams *cam, const uint32_t *d_pixel_ids, int64_t n, const double *d_origin_in,
                      const double *d_dir_in, int nx, int ny, int nz, double *d_origin_out, double *d_dir,
                      double *t_enter, double *t_exit, uint8_t *status, uint8_t *exited, uint32_t *coarse_cell,
                      uint32_t *fine_cell, double *coarse_tmax, double *fine_tmax, cudaStream_t st);

}  // namespace wc
