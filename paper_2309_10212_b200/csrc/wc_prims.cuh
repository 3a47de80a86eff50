// wc_prims.cuh -- device-wide data-parallel primitives (prims.py:13-40).
//
// exclusive_scan  -> scan_exclusive()  (3-phase reduce / scan-of-partials / scan)
// compact         -> fused into callers via the scan offsets
// sort_by_key     -> radix_sort_pairs() (stable LSD, 8-bit digits, per-warp
//                    match_any ranking so equal keys keep input order)
// Bitmap ranking  -> bitmap_extract() (ascending ids of set bits)
#pragma once

#include "wc_common.cuh"

namespace wc {

constexpr int kScanThreads = 256;
constexpr int kScanIPT = 8;
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

template <class Load>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_reduce(Load ld, int64_t n_max, const uint32_t *d_n, uint32_t *tile_sums) {
    __shared__ uint32_t sw[32];
    const int64_t n = scan_count(n_max, d_n);
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanIPT; k++) {
        const int64_t i = base + k * kScanThreads + threadIdx.x;  // striped: coalesced
        if (i < n) s += ld(i);
    }
    uint32_t tot;
    block_exclusive_scan(s, sw, &tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// Single CTA: exclusive scan of the tile sums in place; total -> *total.
__global__ void __launch_bounds__(1024) k_scan_partials(uint32_t *tile_sums, int64_t ntiles, uint32_t *total);

template <class Load>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_apply(Load ld, int64_t n_max, const uint32_t *d_n, const uint32_t *tile_offsets, uint32_t *out) {
    __shared__ uint32_t sw[32];
    __shared__ uint32_t tile[kScanTile];
    const int64_t n = scan_count(n_max, d_n);
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    if (base >= n) return;
#pragma unroll
    for (int k = 0; k < kScanIPT; k++) {
        const int idx = k * kScanThreads + threadIdx.x;
        const int64_t i = base + idx;
        tile[idx] = i < n ? ld(i) : 0;
    }
    __syncthreads();
    uint32_t v[kScanIPT], s = 0;
#pragma unroll
    for (int k = 0; k < kScanIPT; k++) {
        v[k] = tile[threadIdx.x * kScanIPT + k];
        s += v[k];
    }
    uint32_t pre = block_exclusive_scan(s, sw, nullptr) + tile_offsets[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanIPT; k++) {
        tile[threadIdx.x * kScanIPT + k] = pre;
        pre += v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanIPT; k++) {
        const int idx = k * kScanThreads + threadIdx.x;
        const int64_t i = base + idx;
        if (i < n) out[i] = tile[idx];
    }
}

// Exclusive scan of ld(0..n) into out[0..n); grand total into *d_total.
// `partials` must hold scan_tiles(n) uint32.
template <class Load>
void scan_exclusive(Load ld, int64_t n, uint32_t *out, uint32_t *d_total, uint32_t *partials,
                    cudaStream_t st) {
    if (n <= 0) {
        WC_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), st));
        return;
    }
    const int64_t nt = scan_tiles(n);
    k_scan_reduce<Load><<<(unsigned)nt, kScanThreads, 0, st>>>(ld, n, nullptr, partials);
    WC_LAUNCH_CHECK();
    k_scan_partials<<<1, 1024, 0, st>>>(partials, nt, d_total);
    WC_LAUNCH_CHECK();
    k_scan_apply<Load><<<(unsigned)nt, kScanThreads, 0, st>>>(ld, n, nullptr, partials, out);
    WC_LAUNCH_CHECK();
}

// Same with the element count on the device (<= n_max, the launch bound).
template <class Load>
void scan_exclusive_dev(Load ld, const uint32_t *d_n, int64_t n_max, uint32_t *out, uint32_t *d_total,
                        uint32_t *partials, cudaStream_t st) {
    if (n_max <= 0) {
        WC_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint32_t), st));
        return;
    }
    const int64_t nt = scan_tiles(n_max);
    k_scan_reduce<Load><<<(unsigned)nt, kScanThreads, 0, st>>>(ld, n_max, d_n, partials);
    WC_LAUNCH_CHECK();
    k_scan_partials<<<1, 1024, 0, st>>>(partials, nt, d_total);
    WC_LAUNCH_CHECK();
    k_scan_apply<Load><<<(unsigned)nt, kScanThreads, 0, st>>>(ld, n_max, d_n, partials, out);
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

// Ascending ids of the set bits of bm[0..nwords) -> out; count -> *d_count.
// word_offsets (nwords uint32) receives the exclusive popcount prefix and can
// later rank a set bit: rank(b) = word_offsets[b>>5] + popc(bm[b>>5] & lowmask).
void bitmap_extract(const uint32_t *bm, int64_t nwords, uint32_t *word_offsets, uint32_t *out,
                    uint32_t *d_count, uint32_t *partials, cudaStream_t st);

}  // namespace wc
