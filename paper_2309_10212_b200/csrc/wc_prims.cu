// wc_prims.cu -- scan / radix sort / bitmap extraction (prims.py:13-40).
#include "wc_prims.cuh"

namespace wc {

// ---------------------------------------------------------------- radix

__global__ void __launch_bounds__(kSortThreads)
    k_radix_hist(const uint32_t *keys, int64_t n, int shift, uint32_t mask, uint32_t *hist, int64_t ntiles) {
    __shared__ uint32_t h[kSortBins];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll
    for (int k = 0; k < kSortIPT; k++) {
        const int64_t i = base + k * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & mask], 1u);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];  // digit-major
}

// Stable scatter: warp w of the tile owns items [w*256, w*256+256), walked in
// 8 rounds of 32 consecutive items; __match_any_sync ranks equal digits
// within a round and a per-warp smem histogram carries counts across rounds.
__global__ void __launch_bounds__(kSortThreads)
    k_radix_scatter(const uint32_t *keys, const uint32_t *vals, uint32_t *keys_out, uint32_t *vals_out,
                    int64_t n, int shift, uint32_t mask, const uint32_t *hist_off, int64_t ntiles) {
    constexpr int kWarps = kSortThreads / 32;
    __shared__ uint32_t wh[kWarps][kSortBins];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = lane; d < kSortBins; d += 32) wh[warp][d] = 0;
    __syncwarp();
    const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)warp * (kSortIPT * 32);
    uint32_t k[kSortIPT], v[kSortIPT], rank[kSortIPT];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kSortIPT; r++) {
        const int64_t i = base + r * 32 + lane;
        const bool ok = i < n;
        k[r] = ok ? keys[i] : 0;
        v[r] = ok ? vals[i] : 0;
        const uint32_t dig = ok ? ((k[r] >> shift) & mask) : (0x10000u + lane);
        const uint32_t peers = __match_any_sync(0xffffffffu, dig);
        uint32_t prior = 0;
        if (ok) prior = wh[warp][dig];
        __syncwarp();
        rank[r] = prior + __popc(peers & lt);
        if (ok && (peers & lt) == 0) wh[warp][dig] = prior + __popc(peers);  // group leader
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix across warps per digit (in place), plus tile offset
    for (int d = threadIdx.x; d < kSortBins; d += kSortThreads) {
        uint32_t acc = hist_off[(int64_t)d * ntiles + blockIdx.x];
#pragma unroll
        for (int w = 0; w < kWarps; w++) {
            const uint32_t c = wh[w][d];
            wh[w][d] = acc;
            acc += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortIPT; r++) {
        const int64_t i = base + r * 32 + lane;
        if (i < n) {
            const uint32_t dig = (k[r] >> shift) & mask;
            const uint32_t pos = wh[warp][dig] + rank[r];
            keys_out[pos] = k[r];
            vals_out[pos] = v[r];
        }
    }
}

void RadixScratch::reserve(int64_t n) {
    if (keys_alt.n < n) {
        keys_alt.alloc(n);
        vals_alt.alloc(n);
    }
    const int64_t nt = ceil_div(n < 1 ? 1 : n, kSortTile);
    const int64_t hn = nt * kSortBins;
    if (hist.n < hn) {
        hist.alloc(hn);
        hist_partials.alloc(scan_scratch_words(hn));
        WC_CUDA(cudaMemset(hist_partials.p, 0, 4 * hist_partials.n));
    }
    if (!total.p) total.alloc(1);
}

void radix_sort_pairs(uint32_t *keys, uint32_t *vals, int64_t n, int nbits, RadixScratch &scratch,
                      cudaStream_t st) {
    if (n <= 1 || nbits <= 0) return;
    scratch.reserve(n);
    const int64_t nt = ceil_div(n, kSortTile);
    uint32_t *ka = keys, *va = vals, *kb = scratch.keys_alt.p, *vb = scratch.vals_alt.p;
    int passes = 0;
    for (int shift = 0; shift < nbits; shift += 8) {
        const int bits = (nbits - shift) < 8 ? (nbits - shift) : 8;
        const uint32_t mask = (1u << bits) - 1u;
        k_radix_hist<<<(unsigned)nt, kSortThreads, 0, st>>>(ka, n, shift, mask, scratch.hist.p, nt);
        WC_LAUNCH_CHECK();
        const int64_t hn = nt * kSortBins;
        scan_exclusive(LoadU32{scratch.hist.p}, hn, scratch.hist.p, scratch.total.p, scratch.hist_partials.p, st);
        k_radix_scatter<<<(unsigned)nt, kSortThreads, 0, st>>>(ka, va, kb, vb, n, shift, mask, scratch.hist.p, nt);
        WC_LAUNCH_CHECK();
        uint32_t *t = ka;
        ka = kb;
        kb = t;
        t = va;
        va = vb;
        vb = t;
        passes++;
    }
    if (passes & 1) {  // result sits in the scratch buffers: copy back
        WC_CUDA(cudaMemcpyAsync(keys, ka, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
        WC_CUDA(cudaMemcpyAsync(vals, va, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, st));
    }
}

// ----------------------------------------------------------- bitmap extract

void bitmap_extract(const uint32_t *bm, int64_t nwords, uint32_t *word_offsets, uint32_t *out,
                    uint32_t *d_count, uint32_t *partials, cudaStream_t st) {
    if (nwords <= 0) {
        WC_CUDA(cudaMemsetAsync(d_count, 0, sizeof(uint32_t), st));
        return;
    }
    // one pass: popcount scan of the words, ids written by each tile as
    // soon as its prefix is known
    k_scan_onepass<LoadPopc, SinkBits><<<(unsigned)scan_tiles(nwords), kScanThreads, 0, st>>>(
        LoadPopc{bm}, SinkBits{bm, word_offsets, out}, nwords, nullptr, reinterpret_cast<uint64_t *>(partials),
        scan_epoch(), d_count);
    WC_LAUNCH_CHECK();
}

void bitmap_extract_dev(const uint32_t *bm, const uint32_t *d_nwords, int64_t nwords_max, uint32_t *word_offsets,
                        uint32_t *out, uint32_t *d_count, uint32_t *partials, cudaStream_t st) {
    if (nwords_max <= 0) {
        WC_CUDA(cudaMemsetAsync(d_count, 0, sizeof(uint32_t), st));
        return;
    }
    k_scan_onepass<LoadPopc, SinkBits><<<(unsigned)scan_tiles(nwords_max), kScanThreads, 0, st>>>(
        LoadPopc{bm}, SinkBits{bm, word_offsets, out}, nwords_max, d_nwords, reinterpret_cast<uint64_t *>(partials),
        scan_epoch(), d_count);
    WC_LAUNCH_CHECK();
}

// ---- two-level extraction ----------------------------------------------

// summary bit w = (bm[w] != 0), warp per 32 words (one coalesced 128 B read)
__global__ void k_summarize(const uint32_t *__restrict__ bm, const uint32_t *d_nwords, int64_t nwords_max,
                            uint32_t *__restrict__ summary) {
    const int64_t n = d_nwords ? min(nwords_max, (int64_t)*d_nwords) : nwords_max;
    const int64_t ns = (nwords_max + 31) >> 5;  // every summary word (zero past n): no stale bits
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sidx = w0; sidx < ns; sidx += nw) {
        const int64_t w = sidx * 32 + lane;
        const uint32_t bits = __ballot_sync(0xffffffffu, w < n && bm[w] != 0u);
        if (lane == 0) summary[sidx] = bits;
    }
}

struct LoadPopcIdx {
    const uint32_t *bm, *idx;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const { return __popc(bm[idx[i]]); }
};

struct SinkBitsIdx {
    uint32_t *bm;
    const uint32_t *idx;
    uint32_t *word_offsets, *ids;
    int64_t id_mod;
    bool clear;
    __device__ __forceinline__ void operator()(int64_t i, uint32_t prefix) const {
        const uint32_t w = idx[i];
        uint32_t v = bm[w];
        if (word_offsets) word_offsets[w] = prefix;
        if (clear) bm[w] = 0u;
        const uint32_t base = (uint32_t)((w % id_mod) * 32);
        while (v) {
            ids[prefix++] = base + __ffs(v) - 1;
            v &= v - 1;
        }
    }
};

void bitmap_extract_sparse(uint32_t *bm, const uint32_t *d_nwords, int64_t nwords_max, int64_t id_mod,
                           uint32_t *word_offsets, uint32_t *ids, uint32_t *d_count, bool clear,
                           const SparseScratch &sc, uint32_t *partials, cudaStream_t st) {
    if (nwords_max <= 0) {
        WC_CUDA(cudaMemsetAsync(d_count, 0, sizeof(uint32_t), st));
        return;
    }
    const int64_t ns_max = (nwords_max + 31) / 32;
    k_summarize<<<grid_for(ns_max * 32, 256, 8), 256, 0, st>>>(bm, d_nwords, nwords_max, sc.summary);
    WC_LAUNCH_CHECK();
    k_scan_onepass<LoadPopc, SinkBits><<<(unsigned)scan_tiles(ns_max), kScanThreads, 0, st>>>(
        LoadPopc{sc.summary}, SinkBits{sc.summary, sc.word_list + nwords_max, sc.word_list}, ns_max, nullptr,
        reinterpret_cast<uint64_t *>(partials), scan_epoch(), sc.d_nlist);
    WC_LAUNCH_CHECK();
    k_scan_onepass<LoadPopcIdx, SinkBitsIdx><<<(unsigned)scan_tiles(nwords_max), kScanThreads, 0, st>>>(
        LoadPopcIdx{bm, sc.word_list}, SinkBitsIdx{bm, sc.word_list, word_offsets, ids, id_mod, clear}, nwords_max,
        sc.d_nlist, reinterpret_cast<uint64_t *>(partials), scan_epoch(), d_count);
    WC_LAUNCH_CHECK();
}

}  // namespace wc
