// wc_prims.cuh -- device-wide data-parallel primitives (prims.py:13-40).
//
// exclusive_scan  -> scan_exclusive()  (single pass, decoupled look-back)
// compact         -> fused into callers via the scan offsets
// sort_by_key     -> radix_sort_pairs() (stable LSD, 8-bit digits, per-warp
//                    match_any ranking so equal keys keep input order)
// Bitmap ranking  -> bitmap_extract_listed() (ascending ids of set bits, from
//                    a summary maintained by the kernels that set them)
#pragma once

#include <type_traits>

#include "wc_common.cuh"

namespace wc {

#ifndef WC_SCAN_IPT
#define WC_SCAN_IPT 4
#endif
constexpr int kScanThreads = 256;
constexpr int kScanIPT = WC_SCAN_IPT;
constexpr int kScanTile = kScanThreads * kScanIPT;  // 2048 items per CTA

// Loaders: value of element i as uint32.
struct LoadU32 {
    const uint32_t *p;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return p[i]; }
};
struct LoadU8NonZero {
    const uint8_t *p;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return p[i] != 0; }
};
struct LoadPopc {
    const uint32_t *p;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return __popc(p[i]); }
};

// Scratch sizing for scan_exclusive over n elements.
inline int64_t scan_tiles(int64_t n) { return ceil_div(n < 1 ? 1 : n, kScanTile); }

// Block-wide exclusive scan of per-thread sums; returns this thread's
// exclusive prefix and writes the block total to *block_total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *smem_warp,
                                                         uint32_t *block_total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t w = lane < nw ? smem_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) smem_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    const uint32_t warp_prefix = warp ? smem_warp[warp - 1] : 0;
    if (block_total) *block_total = smem_warp[(blockDim.x >> 5) - 1];
    return warp_prefix + x - v;
}

// d_n (nullable): element count read on the device, capped by n (the
// launch-time upper bound), so a scan can follow a producer without a host
// round trip.
__device__ __forceinline__ int64_t scan_count(int64_t n, const uint32_t *d_n) {
    return d_n ? min(n, (int64_t)*d_n) : n;
}

// ---- single-pass scan (decoupled look-back) -----------------------------
// Each tile publishes its aggregate, then its inclusive prefix, in one
// 64-bit status word [epoch:30 | flag:2 | value:32]; successors look back
// over the status words with a warp.  The epoch tags every scan call, so
// the status array never needs clearing.  One launch per scan.
//
// Tile ids are dynamic tickets (an atomic counter in the scratch header), so
// a tile only ever waits on tiles whose CTAs are already running: forward
// progress does not depend on the hardware dispatching CTAs in blockIdx
// order, on how many CTAs fit per SM, or on other kernels sharing the GPU.
// Every CTA reads the element count before it takes its ticket, and the
// epilogue runs only once the last ticket is taken and the total is known,
// so an epilogue may rewrite the count the scan itself read.
constexpr uint32_t kFlagAggregate = 1, kFlagPrefix = 2;

// Host-issued epochs have bit 29 set; epochs derived on the device (below)
// have it clear, so the two never collide.
inline uint32_t next_scan_epoch() {
    static std::atomic<uint32_t> e{0};
    return ((e.fetch_add(1) + 1) & 0x1FFFFFFFu) | 0x20000000u;
}

// A scan inside a captured (replayed) pass must get a new epoch at every
// replay: it is then derived on the device from the frame counter and a
// per-call salt, (frame << 12) + salt.  The session sets the thread-local
// frame pointer and salt base while it enqueues a pass.
struct ScanEpoch {
    const uint32_t *d_frame;  // nullptr: `value` is the epoch
    uint32_t value;
};
inline thread_local const uint32_t *t_epoch_frame = nullptr;
inline thread_local uint32_t t_epoch_salt = 0;
inline ScanEpoch scan_epoch() {
    if (t_epoch_frame) return ScanEpoch{t_epoch_frame, (t_epoch_salt++) & 4095u};
    return ScanEpoch{nullptr, next_scan_epoch()};
}
__device__ __forceinline__ uint32_t resolve_epoch(const ScanEpoch e) {
    if (!e.d_frame) return e.value;
    const uint32_t v = ((*e.d_frame << 12) + e.value) & 0x1FFFFFFFu;
    return v ? v : 0x1FFFFFFFu;
}

// scratch words (uint32) a scan over n elements needs: a 64-bit header
// (ticket and done counters, zero between scans) + one status word per tile
inline int64_t scan_scratch_words(int64_t n) { return 2 * scan_tiles(n) + 8; }

// Scratch header: word 0 = ticket counter, word 1 = epilogue arrivals; both
// are zero between scans.
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
// Thread 0: this CTA's ticket (tile id), taken after the CTA has read its
// inputs' count.  The CTA holding the last ticket resets the counter for the
// next scan on this scratch (every ticket of the launch has been taken).
#ifndef WC_SCAN_TICKETS
#define WC_SCAN_TICKETS 1
#endif
// Thread 0: this CTA's ticket (tile id), taken after the CTA has read (and
// used) its inputs' count.  The CTA holding the last ticket resets the
// counter for the next scan on this scratch (every ticket of the launch has
// been taken).  A CTA loads the data of tile blockIdx.x while its ticket is in
// flight and reloads only when the ticket differs (dispatch out of blockIdx
// order), so the atomic's latency stays off the critical path.
__device__ __forceinline__ uint32_t take_ticket(uint64_t *scratch, bool &last_ticket) {
#if !WC_SCAN_TICKETS  // timing experiment only: tile id = blockIdx.x (assumes in-order dispatch)
    last_ticket = blockIdx.x == gridDim.x - 1;
    return blockIdx.x;
#endif
    uint32_t *c = reinterpret_cast<uint32_t *>(scratch);
    const uint32_t t = atomicAdd(c, 1u);
    last_ticket = t == gridDim.x - 1;
    if (last_ticket) *reinterpret_cast<volatile uint32_t *>(c) = 0u;
    return t;
}
// Thread 0: the epilogue runs once both the scan total is known (the last
// tile) and every CTA has read the count (the last ticket): the second of
// those two arrivals runs it and clears the arrival word.
__device__ __forceinline__ bool epilogue_arrive(uint64_t *scratch, uint32_t arrivals, uint32_t target = 2u) {
    uint32_t *c = reinterpret_cast<uint32_t *>(scratch) + 1;
    if (!arrivals) return false;
    if (atom_add_acq_rel(c, arrivals) + arrivals != target) return false;
    *reinterpret_cast<volatile uint32_t *>(c) = 0u;
    return true;
}
// the per-tile status words follow the header
__device__ __forceinline__ uint64_t *tile_status(uint64_t *scratch) { return scratch + 1; }

__device__ __forceinline__ void store_status(uint64_t *p, uint32_t epoch, uint32_t flag, uint32_t v) {
    atomicExch(reinterpret_cast<unsigned long long *>(p),
               ((unsigned long long)epoch << 34) | ((unsigned long long)flag << 32) | v);
}

// Sinks receive (element, its exclusive prefix, its loaded value).
struct SinkStore {  // out[i] = exclusive prefix
    uint32_t *out;
    __device__ __forceinline__ void operator()(int64_t i, uint32_t prefix, uint32_t) const { out[i] = prefix; }
};
struct SinkBits {  // word offsets + ascending ids of the set bits of bm
    const uint32_t *bm;
    uint32_t *word_offsets, *ids;
    __device__ __forceinline__ void operator()(int64_t i, uint32_t prefix, uint32_t) const {
        word_offsets[i] = prefix;
        uint32_t v = bm[i];
        while (v) {
            ids[prefix++] = (uint32_t)(i * 32 + __ffs(v) - 1);
            v &= v - 1;
        }
    }
};

// exclusive-scan consumer that compacts the ids whose predicate (the scan's
// 0/1 loaded value) holds
template <class Pred>
struct SinkCompact {
    Pred pred;
    const uint32_t *ids;
    uint32_t *out;
    __device__ __forceinline__ void operator()(int64_t i, uint32_t prefix, uint32_t v) const {
        if (v) out[prefix] = ids[i];
    }
};

// Loaders with per-CTA state (e.g. shared-memory bins) define cta_begin()
// (all threads, before the first load; the scan synchronises after it) and
// cta_end() (all threads, on every exit path, after the last load).  Such a
// loader runs only on the CTA's own tiles (no speculative load), but may be
// called twice per element by the same thread (chunk totals, then the tile):
// its side effects must be idempotent.
template <class L, class = void>
struct HasCtaHooks : std::false_type {};
template <class L>
struct HasCtaHooks<L, std::void_t<decltype(&L::cta_begin)>> : std::true_type {};

// Decoupled look-back of tile t (called by warp 0 of its CTA): publishes the
// tile's aggregate, sums predecessors back to the nearest published prefix,
// publishes the tile's inclusive prefix and returns its exclusive prefix.
__device__ __forceinline__ uint32_t tile_lookback(int64_t t, uint32_t agg, uint64_t *status, uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    uint32_t excl = 0;
    if (t == 0) {
        if (lane == 0) store_status(status, epoch, kFlagPrefix, agg);
        return 0;
    }
    if (lane == 0) store_status(status + t, epoch, kFlagAggregate, agg);
    for (int64_t pred = t - 1;; pred -= 32) {
        const int64_t idx = pred - lane;
        uint32_t flag = kFlagPrefix, val = 0;  // before tile 0: an implicit zero prefix
        if (idx >= 0) {
            unsigned long long w;
            do {
                w = *reinterpret_cast<volatile unsigned long long *>(status + idx);
                flag = (uint32_t)(w >> 34) == epoch ? (uint32_t)(w >> 32) & 3u : 0u;
            } while (flag == 0);
            val = (uint32_t)w;
        }
        const uint32_t pm = __ballot_sync(0xffffffffu, flag == kFlagPrefix);
        const int fp = pm ? __ffs(pm) - 1 : 31;  // nearest predecessor holding a prefix
        uint32_t c = lane <= fp ? val : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        excl += c;
        if (pm) break;
    }
    if (lane == 0) store_status(status + t, epoch, kFlagPrefix, excl + agg);
    return excl;
}

// The same look-back by the whole CTA (every thread calls it; blockDim.x a
// multiple of 32): a round reads the status words of the blockDim.x *
// WC_LOOKBACK_K nearest unread predecessors at once.  With one wave of ~1000
// tiles all publishing their aggregates together, the warp form needs a
// dependent L2 round trip per 32 predecessors (~30 for the last tile); this
// one needs one.  `sred`: 64 words of shared memory.
#ifndef WC_LOOKBACK_K
#define WC_LOOKBACK_K 4
#endif
#ifndef WC_LOOKBACK_CTA
#define WC_LOOKBACK_CTA 0  // measured slower at C3 (3.07 vs 2.97 ms; micro-benchmark: 23.5 vs 20.9 us per extraction)
#endif
__device__ __forceinline__ uint32_t tile_lookback_cta(int64_t t, uint32_t agg, uint64_t *status, uint32_t epoch,
                                                      uint32_t *sred) {
    constexpr int K = WC_LOOKBACK_K;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    if (t == 0) {
        if (tid == 0) store_status(status, epoch, kFlagPrefix, agg);
        return 0;
    }
    if (tid == 0) store_status(status + t, epoch, kFlagAggregate, agg);
    const int64_t span = (int64_t)blockDim.x * K;
    uint32_t excl = 0;
    for (int64_t hi = t - 1;; hi -= span) {
        // position p = k * blockDim.x + tid is predecessor hi - p (p = 0: the nearest)
        unsigned long long w[K];
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int64_t idx = hi - ((int64_t)k * blockDim.x + tid);
            // before tile 0: an implicit zero prefix
            w[k] = idx >= 0 ? *reinterpret_cast<volatile unsigned long long *>(status + idx)
                            : ((unsigned long long)epoch << 34) | ((unsigned long long)kFlagPrefix << 32);
        }
        uint32_t pmin = 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int64_t idx = hi - ((int64_t)k * blockDim.x + tid);
            uint32_t flag = (uint32_t)(w[k] >> 34) == epoch ? (uint32_t)(w[k] >> 32) & 3u : 0u;
            while (flag == 0) {
                w[k] = *reinterpret_cast<volatile unsigned long long *>(status + idx);
                flag = (uint32_t)(w[k] >> 34) == epoch ? (uint32_t)(w[k] >> 32) & 3u : 0u;
            }
            if (flag == kFlagPrefix) pmin = min(pmin, (uint32_t)(k * blockDim.x + tid));
        }
        pmin = __reduce_min_sync(0xffffffffu, pmin);
        if (lane == 0) sred[warp] = pmin;
        __syncthreads();
        uint32_t fp = sred[0];
        for (int i = 1; i < nwarps; i++) fp = min(fp, sred[i]);  // nearest predecessor holding a prefix
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < K; k++)
            if ((uint32_t)(k * blockDim.x + tid) <= fp) c += (uint32_t)w[k];
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) sred[32 + warp] = c;
        __syncthreads();
        for (int i = 0; i < nwarps; i++) excl += sred[32 + i];
        if (fp != 0xFFFFFFFFu) break;
    }
    if (tid == 0) store_status(status + t, epoch, kFlagPrefix, excl + agg);
    return excl;
}

// The grid is capped (scan_max_ctas) so that a scan sized for a large upper
// bound does not launch thousands of CTAs that find no work: with more tiles
// than CTAs, each CTA owns m consecutive tiles, publishes their total through
// the look-back, then scans them in order (loading each twice).
inline int64_t scan_max_ctas() { return (int64_t)num_sms() * 8; }
inline unsigned scan_grid(int64_t n_max) { return (unsigned)std::min<int64_t>(scan_tiles(n_max), scan_max_ctas()); }

// Epilogue of a scan: run once with the total, after every CTA has read the
// count (a control decision that would otherwise be a one-thread kernel).
struct NoEpilogue {
    __device__ __forceinline__ void operator()(uint32_t) const {}
};
template <class Epi>
struct EpiTraits {
    static constexpr bool none = false;
};
template <>
struct EpiTraits<NoEpilogue> {
    static constexpr bool none = true;
};

template <class Load, class Sink, class Epi = NoEpilogue>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_onepass(Load ld, Sink sink, int64_t n_max, const uint32_t *d_n, uint64_t *scratch, ScanEpoch ep,
                   uint32_t *d_total, Epi epi = Epi{}) {
    pdl_wait();
    __shared__ uint32_t sw[32];
    __shared__ uint32_t tile[kScanTile + 1];
    __shared__ uint32_t slb[64];
    __shared__ uint32_t s_excl, s_ticket, s_n, s_last_ticket;
    uint64_t *status = tile_status(scratch);
    const uint32_t epoch = resolve_epoch(ep);
    // A loader with per-CTA state flushes it at the CTA's end, and the
    // epilogue may read what it flushed: then every CTA arrives at its end
    // and the last of the gridDim.x arrivals runs the epilogue.
    constexpr bool kEndArrive = HasCtaHooks<Load>::value && !EpiTraits<Epi>::none;
    if (threadIdx.x == 0) s_n = (uint32_t)scan_count(n_max, d_n);
    if constexpr (HasCtaHooks<Load>::value) ld.cta_begin();
    __syncthreads();  // every CTA has read the count before it takes a ticket
    const int64_t n = s_n;
    // (32-bit divisions: counts < 2^32; a 64-bit one is a subroutine call)
    const int64_t ntiles = n > 0 ? (n - 1) / kScanTile + 1 : 1;
    const int64_t m = ((uint32_t)ntiles + gridDim.x - 1) / gridDim.x;  // tiles per CTA
    const int64_t last = (uint32_t)(ntiles - 1) / (uint32_t)m;
    bool lt = false;
    uint32_t tk = 0;
    if (threadIdx.x == 0) tk = take_ticket(scratch, lt);
    // speculative load of tile blockIdx.x while the ticket is in flight
    auto chunk_sum = [&](int64_t tt) {
        uint32_t acc = 0;
        const int64_t b0 = tt * m * kScanTile;
        for (int64_t i = b0 + threadIdx.x; i < min(n, b0 + m * kScanTile); i += kScanThreads) acc += ld(i);
        return acc;
    };
    auto load_tile = [&](int64_t tb) {
#pragma unroll
        for (int k = 0; k < kScanIPT; k++) {
            const int idx = k * kScanThreads + threadIdx.x;
            const int64_t i = tb + idx;
            tile[idx] = i < n ? ld(i) : 0;
        }
    };
    // (loaders with per-CTA state are not run speculatively: their side
    // effects then happen only in the tile's owner)
    const int64_t ts = HasCtaHooks<Load>::value ? -1 : (int64_t)blockIdx.x;
    uint32_t csum = 0;
    if (ts >= 0 && ts <= last) {
        if (m > 1)
            csum = chunk_sum(ts);
        else
            load_tile(ts * kScanTile);
    }
    if (threadIdx.x == 0) {
        s_ticket = tk;
        s_last_ticket = lt;
        // the holder of the last ticket arrives now unless it also holds the
        // last tile (which arrives once the total is known)
        if (!kEndArrive && !EpiTraits<Epi>::none && lt && (int64_t)tk != last && epilogue_arrive(scratch, 1u))
            epi(*reinterpret_cast<volatile uint32_t *>(d_total));
    }
    auto end_arrive = [&](bool total_known) {  // kEndArrive: after cta_end
        if (threadIdx.x == 0 && epilogue_arrive(scratch, 1u, gridDim.x)) epi(*reinterpret_cast<volatile uint32_t *>(d_total));
        (void)total_known;
    };
    __syncthreads();
    const int64_t t = s_ticket;
    if (t > last) {
        if constexpr (HasCtaHooks<Load>::value) ld.cta_end();  // the speculative loads' side effects
        if constexpr (kEndArrive) end_arrive(false);
        return;
    }
    if (t != ts) {  // dispatched out of order: the data of the ticket's tile
        if (m > 1)
            csum = chunk_sum(t);
        else
            load_tile(t * kScanTile);
    }
    const int64_t base = t * m * kScanTile;
    if (m > 1) {  // the chunk's total first, so successors can look back early
        uint32_t agg;
        block_exclusive_scan(csum, sw, &agg);
        uint32_t excl = 0;
        if (WC_LOOKBACK_CTA)
            excl = tile_lookback_cta(t, agg, status, epoch, slb);
        else if (threadIdx.x < 32)
            excl = tile_lookback(t, agg, status, epoch);
        if (threadIdx.x == 0) {
            s_excl = excl;
            if (t == last) {
                *d_total = excl + agg;
                if (!kEndArrive && !EpiTraits<Epi>::none && epilogue_arrive(scratch, 1u + s_last_ticket))
                    epi(excl + agg);
            }
        }
        __syncthreads();
        load_tile(base);  // the chunk's first tile
    }
    uint32_t running = 0;
    for (int64_t sub = 0; sub < m; sub++) {
        const int64_t tb = base + sub * kScanTile;
        if (sub > 0) load_tile(tb);  // sub-tile 0 is loaded above
        __syncthreads();
        uint32_t v[kScanIPT], s = 0;
#pragma unroll
        for (int k = 0; k < kScanIPT; k++) {
            v[k] = tile[threadIdx.x * kScanIPT + k];
            s += v[k];
        }
        uint32_t agg;
        uint32_t pre = block_exclusive_scan(s, sw, &agg);
        if (m == 1) {
            uint32_t excl = 0;
            if (WC_LOOKBACK_CTA)
                excl = tile_lookback_cta(t, agg, status, epoch, slb);
            else if (threadIdx.x < 32)
                excl = tile_lookback(t, agg, status, epoch);
            if (threadIdx.x == 0) {
                s_excl = excl;
                if (t == last) {
                    const uint32_t total = n > 0 ? excl + agg : 0u;
                    *d_total = total;
                    if (!kEndArrive && !EpiTraits<Epi>::none && epilogue_arrive(scratch, 1u + s_last_ticket))
                        epi(total);
                }
            }
        }
        __syncthreads();
        pre += s_excl + running;
#pragma unroll
        for (int k = 0; k < kScanIPT; k++) {
            tile[threadIdx.x * kScanIPT + k] = pre;
            pre += v[k];
        }
        if (threadIdx.x == kScanThreads - 1) tile[kScanTile] = pre;  // the tile's inclusive end
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kScanIPT; k++) {
            const int idx = k * kScanThreads + threadIdx.x;
            const int64_t i = tb + idx;
            if (i < n) sink(i, tile[idx], tile[idx + 1] - tile[idx]);
        }
        running += agg;
        __syncthreads();  // tile and sw are reused by the next tile
    }
    if constexpr (HasCtaHooks<Load>::value) ld.cta_end();
    if constexpr (kEndArrive) end_arrive(true);
}

// Exclusive scan of ld(0..n) into out[0..n); grand total into *d_total.
// `scratch` must hold scan_scratch_words(n) uint32 (zeroed once at allocation).
template <class Load>
void scan_exclusive(Load ld, int64_t n, uint32_t *out, uint32_t *d_total, uint32_t *scratch, cudaStream_t st) {
    if (n <= 0) {
        WC_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), st));
        return;
    }
    launch_pdl(k_scan_onepass<Load, SinkStore>, scan_grid(n), kScanThreads, 0, st, 
        ld, SinkStore{out}, n, nullptr, reinterpret_cast<uint64_t *>(scratch), scan_epoch(), d_total, NoEpilogue{});
    WC_LAUNCH_CHECK();
}

// Same with the element count on the device (<= n_max, the launch bound).
template <class Load>
void scan_exclusive_dev(Load ld, const uint32_t *d_n, int64_t n_max, uint32_t *out, uint32_t *d_total,
                        uint32_t *scratch, cudaStream_t st) {
    if (n_max <= 0) {
        WC_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), st));
        return;
    }
    launch_pdl(k_scan_onepass<Load, SinkStore>, scan_grid(n_max), kScanThreads, 0, st, 
        ld, SinkStore{out}, n_max, d_n, reinterpret_cast<uint64_t *>(scratch), scan_epoch(), d_total, NoEpilogue{});
    WC_LAUNCH_CHECK();
}

// Stable compaction of ids[i] for pred(i), i < *d_n (<= n_max), in one
// pass: out[...] in input order, count -> *d_total.
// (epi: optional epilogue run with the count, see NoEpilogue; n_max > 0)
template <class Pred, class Epi = NoEpilogue>
void compact_dev(Pred pred, const uint32_t *ids, const uint32_t *d_n, int64_t n_max, uint32_t *out,
                 uint32_t *d_total, uint32_t *scratch, cudaStream_t st, Epi epi = Epi{}) {
    if (n_max <= 0) {
        WC_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), st));
        return;
    }
    launch_pdl(k_scan_onepass<Pred, SinkCompact<Pred>, Epi>, scan_grid(n_max), kScanThreads, 0, st, pred,
               SinkCompact<Pred>{pred, ids, out}, n_max, d_n, reinterpret_cast<uint64_t *>(scratch), scan_epoch(),
               d_total, epi);
    WC_LAUNCH_CHECK();
}

// ------------------------------------------------------------ radix sort
constexpr int kSortThreads = 256;
constexpr int kSortIPT = 8;  // rounds of 32 items per warp
constexpr int kSortTile = kSortThreads * kSortIPT;
constexpr int kSortBins = 256;

struct RadixScratch {
    DevBuf<uint32_t> keys_alt, vals_alt, hist, hist_partials, total;
    void reserve(int64_t n);
};

// Stable sort of (keys, vals)[0..n) by the key bits [0, nbits).  Uses
// scratch.keys_alt/vals_alt as the ping-pong buffer; the sorted result is
// always left in (keys, vals).
void radix_sort_pairs(uint32_t *keys, uint32_t *vals, int64_t n, int nbits, RadixScratch &scratch,
                      cudaStream_t st);

// Bitmaps with a maintained summary: bit w of the summary is set whenever
// word w of the bitmap becomes non-zero, by the kernel that sets the bit
// (bitmap_set) or by a pass over the same ids, so an extraction never streams the whole
// bitmap: its cost follows the non-zero words.  Summaries are cleared by the
// extraction that reads them; bitmaps are cleared by it (clear = true) or by
// the caller after the ranks have been used.
__device__ __forceinline__ void bitmap_set_word(uint32_t *bm, uint32_t *summary, uint64_t word, uint32_t bits) {
    if (atomicOr(&bm[word], bits) == 0u) atomicOr(&summary[word >> 5], 1u << (word & 31));
}
__device__ __forceinline__ void bitmap_set(uint32_t *bm, uint32_t *summary, uint64_t word, uint32_t bit) {
    bitmap_set_word(bm, summary, word, 1u << bit);
}
// Ascending ids of the set bits of bm[0..nwords) -> ids, count -> *d_count,
// in one single-pass launch sized to one wave: each CTA owns a contiguous
// chunk of words (16 B loads, a contiguous run per thread), publishes its
// popcount through the decoupled look-back and writes its ids in order.
// word_offsets (nullable) receives the exclusive prefix of every non-zero
// word (bitmap rank: word_offsets[b >> 5] + popc(bm[b >> 5] & lowmask(b)));
// clear zeroes the non-zero words.  For bitmaps that live in L2 (set by
// atomics just before), the cost is one read of the bitmap plus the ids.
void bitmap_extract_dense(uint32_t *bm, int64_t nwords, uint32_t *word_offsets, uint32_t *ids, uint32_t *d_count,
                          bool clear, uint32_t *partials, cudaStream_t st);

// mark_blocks in one launch (engine.py:97-118): from the visibility bitmap
// vis (bdx % 32 == 0: a word never straddles an x-row), the ascending
// visible ids + the rank table vis_word_off, and the ascending ids of the
// active set -- the visible blocks and their existing +octant neighbours --
// computed word by word from vis itself (a block is active when it or its
// -x / -y / -z / ... neighbour is visible), so no active bitmap is built.
// Two look-backs (visible, active) run side by side; vis is left intact.
void mark_extract(const uint32_t *vis, int64_t nwords, int wx_words, int bdy, int bdz, uint32_t *vis_word_off,
                  uint32_t *vis_ids, uint32_t *d_nvis, uint32_t *act_ids, uint32_t *d_nact, uint32_t *partials,
                  cudaStream_t st);

// Ascending ids of the set bits of bm -> ids, count -> *d_count, from its
// summary (summary words [0, ceil(nwords_max / 32))):
//   1. a scan of the summary's popcounts lists the non-zero words in order
//      (and clears the summary);
//   2. a scan of those words' popcounts writes the ids: bit b of word w ->
//      (w % id_mod) * 32 + b, so concatenated bitmaps of id_mod words each
//      list (bitmap, id) pairs in order.
// nlist_max bounds the non-zero words (launch size of step 2).  word_offsets
// (nullable) receives the exclusive prefix of each non-zero word, so a set
// bit ranks as word_offsets[b >> 5] + popc(bm[b >> 5] & lowmask(b)); clear
// zeroes the listed words as they are read.  Scratch: word_list >= nlist_max
// words, partials >= scan_scratch_words(max(nlist_max, summary words)).
void bitmap_extract_listed(uint32_t *bm, uint32_t *summary, int64_t nwords_max, int64_t nlist_max, int64_t id_mod,
                           uint32_t *word_offsets, uint32_t *ids, uint32_t *d_count, bool clear, uint32_t *word_list,
                           uint32_t *d_nlist, uint32_t *partials, cudaStream_t st,
                           const uint32_t *d_nsummary = nullptr);  // summary words to scan, on the device (<= bound)

}  // namespace wc
