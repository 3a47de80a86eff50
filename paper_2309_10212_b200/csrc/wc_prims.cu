// wc_prims.cu -- scan / radix sort / bitmap extraction (prims.py:13-40).
#include "wc_prims.cuh"

namespace wc {

// ---------------------------------------------------------------- radix

__global__ void __launch_bounds__(kSortThreads)
    k_radix_hist(const uint32_t *keys, int64_t n, int shift, uint32_t mask, uint32_t *hist, int64_t ntiles) {
    pdl_wait();
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
    pdl_wait();
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
        launch_pdl(k_radix_hist, (unsigned)nt, kSortThreads, 0, st, ka, n, shift, mask, scratch.hist.p, nt);
        WC_LAUNCH_CHECK();
        const int64_t hn = nt * kSortBins;
        scan_exclusive(LoadU32{scratch.hist.p}, hn, scratch.hist.p, scratch.total.p, scratch.hist_partials.p, st);
        launch_pdl(k_radix_scatter, (unsigned)nt, kSortThreads, 0, st, ka, va, kb, vb, n, shift, mask, scratch.hist.p, nt);
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

// A thread owns kDenseQ16 16-byte groups (up to 16 words): all loads are
// issued before any is used and the words stay in registers for the id pass.
#ifndef WC_DENSE_Q16
#define WC_DENSE_Q16 4
#endif
#ifndef WC_DENSE_MIN_CTAS
#define WC_DENSE_MIN_CTAS 1
#endif
#ifndef WC_DENSE_CTAS_PER_SM
#define WC_DENSE_CTAS_PER_SM 8
#endif
constexpr int kDenseQ16 = WC_DENSE_Q16;
template <bool kClear>
__global__ void __launch_bounds__(256, WC_DENSE_MIN_CTAS) k_bitmap_dense(uint32_t *__restrict__ bm, int64_t nwords, int q16,
                                                      uint32_t *__restrict__ word_offsets, uint32_t *__restrict__ ids,
                                                      uint64_t *status, ScanEpoch ep, uint32_t *d_count) {
    pdl_wait();
    __shared__ uint32_t sw[32], slb[64];
    __shared__ uint32_t s_excl, s_ticket;
    const uint32_t epoch = resolve_epoch(ep);
    const int64_t chunk = 256LL * 4 * q16;
    const int64_t last = (nwords - 1) / chunk;
    bool lt = false;
    uint32_t tk = 0;
    if (threadIdx.x == 0) tk = take_ticket(status, lt);  // dynamic tile id (see k_scan_onepass)
    uint4 q[kDenseQ16];
    auto load = [&](int64_t tt) {
        const int64_t w0 = tt * chunk + (int64_t)threadIdx.x * 4 * q16;
#pragma unroll
        for (int j = 0; j < kDenseQ16; j++) {
            const int64_t w = w0 + 4 * j;
            q[j] = make_uint4(0u, 0u, 0u, 0u);
            if (j < q16) {
                if (w + 4 <= nwords) {
                    q[j] = *reinterpret_cast<const uint4 *>(bm + w);
                } else {
                    if (w < nwords) q[j].x = bm[w];
                    if (w + 1 < nwords) q[j].y = bm[w + 1];
                    if (w + 2 < nwords) q[j].z = bm[w + 2];
                }
            }
        }
    };
    load(blockIdx.x);  // speculative: the tile of blockIdx.x while the ticket is in flight
    if (threadIdx.x == 0) s_ticket = tk;
    __syncthreads();
    const int64_t t = s_ticket;
    if (t != (int64_t)blockIdx.x) load(t);
    const int64_t w0 = t * chunk + (int64_t)threadIdx.x * 4 * q16;
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < kDenseQ16; j++) cnt += __popc(q[j].x) + __popc(q[j].y) + __popc(q[j].z) + __popc(q[j].w);
    uint32_t agg;
    uint32_t pre = block_exclusive_scan(cnt, sw, &agg);
    uint32_t excl = 0;
    if (WC_LOOKBACK_CTA)
        excl = tile_lookback_cta(t, agg, tile_status(status), epoch, slb);
    else if (threadIdx.x < 32)
        excl = tile_lookback(t, agg, tile_status(status), epoch);
    if (threadIdx.x == 0) {
        s_excl = excl;
        if (t == last) *d_count = excl + agg;
    }
    __syncthreads();
    pre += s_excl;
    if (!cnt) return;
#pragma unroll
    for (int j = 0; j < kDenseQ16; j++) {
        const uint32_t wv[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
        for (int c = 0; c < 4; c++) {
            uint32_t v = wv[c];
            if (!v) continue;
            const int64_t w = w0 + 4 * j + c;
            if (word_offsets) word_offsets[w] = pre;
            if (kClear) bm[w] = 0u;
            const uint32_t base = (uint32_t)(w * 32);
            while (v) {
                ids[pre++] = base + __ffs(v) - 1;
                v &= v - 1;
            }
        }
    }
}

void bitmap_extract_dense(uint32_t *bm, int64_t nwords, uint32_t *word_offsets, uint32_t *ids, uint32_t *d_count,
                          bool clear, uint32_t *partials, cudaStream_t st) {
    if (nwords <= 0) {
        WC_CUDA(cudaMemsetAsync(d_count, 0, sizeof(uint32_t), st));
        return;
    }
    // about one wave of WC_DENSE_CTAS_PER_SM CTAs per SM, 1..kDenseQ16 16-byte groups per
    // thread (measured at C3: 8 x 4 beats 4 x 8, 2 x 16 and 8 x 1..3)
    // (larger bitmaps launch more waves)
    const int64_t q16 = std::min<int64_t>(kDenseQ16, std::max<int64_t>(1, ceil_div(nwords, (int64_t)num_sms() * WC_DENSE_CTAS_PER_SM * 256 * 4)));
    const unsigned grid = (unsigned)ceil_div(nwords, 256 * 4 * q16);
    if (clear)
        launch_pdl(k_bitmap_dense<true>, grid, 256, 0, st, bm, nwords, (int)q16, word_offsets, ids,
                                                  reinterpret_cast<uint64_t *>(partials), scan_epoch(), d_count);
    else
        launch_pdl(k_bitmap_dense<false>, grid, 256, 0, st, bm, nwords, (int)q16, word_offsets, ids,
                                                   reinterpret_cast<uint64_t *>(partials), scan_epoch(), d_count);
    WC_LAUNCH_CHECK();
}

#ifndef WC_MARK_Q16
#define WC_MARK_Q16 2  // words per thread / 4 (measured: 2 beats 4 and 1 over C3, C2 at max_spec 1 and an 8-way share)
#endif
constexpr int kMarkQ16 = WC_MARK_Q16;
template <int Q>
__global__ void __launch_bounds__(256, WC_DENSE_MIN_CTAS)
    k_mark_extract(const uint32_t *__restrict__ vis, int64_t nwords, int q16, int wx_words, int bdy, int bdz,
                   uint32_t *__restrict__ vis_word_off, uint32_t *__restrict__ vis_ids, uint32_t *d_nvis,
                   uint32_t *__restrict__ act_ids, uint32_t *d_nact, uint64_t *scratch, ScanEpoch ep) {
    pdl_wait();
    __shared__ uint32_t swv[32], swa[32];
    __shared__ uint32_t s_exv, s_exa, s_ticket;
    const uint32_t epoch = resolve_epoch(ep);
    // (32-bit index arithmetic: bitmaps of < 2^32 words; a 64-bit division
    // is a ~70-instruction subroutine call)
    const int64_t chunk = 256LL * 4 * q16;
    const int64_t ntiles = (int64_t)((uint32_t)(nwords - 1) / (uint32_t)chunk) + 1;
    const int64_t last = ntiles - 1;
    bool lt = false;
    uint32_t tk = 0;
    if (threadIdx.x == 0) tk = take_ticket(scratch, lt);
    uint32_t V[4 * Q], A[4 * Q];
    auto load_own = [&](int64_t tt) {
        const int64_t wb = tt * chunk + (int64_t)threadIdx.x * 4 * q16;
#pragma unroll
        for (int j = 0; j < Q; j++) {
            const int64_t w = wb + 4 * j;
            uint4 q = make_uint4(0u, 0u, 0u, 0u);
            if (j < q16) {
                if (w + 4 <= nwords) {
                    q = *reinterpret_cast<const uint4 *>(vis + w);
                } else {
                    if (w < nwords) q.x = vis[w];
                    if (w + 1 < nwords) q.y = vis[w + 1];
                    if (w + 2 < nwords) q.z = vis[w + 2];
                }
            }
            V[4 * j] = q.x, V[4 * j + 1] = q.y, V[4 * j + 2] = q.z, V[4 * j + 3] = q.w;
        }
    };
    load_own(blockIdx.x);  // speculative: the tile of blockIdx.x while the ticket is in flight
    if (threadIdx.x == 0) s_ticket = tk;
    __syncthreads();
    const int64_t t = s_ticket;
    if (t != (int64_t)blockIdx.x) load_own(t);
    const int64_t w0 = t * chunk + (int64_t)threadIdx.x * 4 * q16;
    const int nw = 4 * q16;  // this thread's words [w0, w0 + nw)
    const int64_t plane = (int64_t)wx_words * bdy;
    const bool aligned4 = (wx_words & 3) == 0 && (plane & 3) == 0;
    // row coordinates of each word (bitmasks over the thread's words)
    uint32_t m_wx = 0, m_by = 0, m_bz = 0;  // bit k: word k has x-word > 0 / y > 0 / z > 0
    {
        const uint32_t w0u = (uint32_t)w0, rowu = w0u / (uint32_t)wx_words;
        int64_t wx = w0u - rowu * (uint32_t)wx_words;
        int64_t by = rowu % (uint32_t)bdy, bz = rowu / (uint32_t)bdy;
#pragma unroll
        for (int k = 0; k < 4 * Q; k++) {
            m_wx |= (uint32_t)(wx > 0) << k;
            m_by |= (uint32_t)(by > 0) << k;
            m_bz |= (uint32_t)(bz > 0) << k;
            if (++wx == wx_words) {  // next x-row
                wx = 0;
                if (++by == bdy) {
                    by = 0;
                    ++bz;
                }
            }
        }
    }
    // x-dilation of a run of words S[1..nw] whose predecessor is S[0]
    auto load_run = [&](int64_t first, uint32_t S[4 * Q + 1]) {  // S[i] = vis[first - 1 + i]
        const bool vec = aligned4 && first >= 0 && first + 4 * Q <= nwords;
        S[0] = (first - 1 >= 0 && first - 1 < nwords) ? __ldg(vis + first - 1) : 0u;
        if (vec) {
#pragma unroll
            for (int j = 0; j < Q; j++) {
                const uint4 q = j < q16 ? __ldg(reinterpret_cast<const uint4 *>(vis + first + 4 * j)) : make_uint4(0, 0, 0, 0);
                S[1 + 4 * j] = q.x, S[2 + 4 * j] = q.y, S[3 + 4 * j] = q.z, S[4 + 4 * j] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4 * Q; k++) {
                const int64_t w = first + k;
                S[1 + k] = (k < nw && w >= 0 && w < nwords) ? __ldg(vis + w) : 0u;
            }
        }
    };
    auto dilate = [&](const uint32_t S[4 * Q + 1], uint32_t gate) {
#pragma unroll
        for (int k = 0; k < 4 * Q; k++)
            if ((gate >> k) & 1u) A[k] |= S[k + 1] | (S[k + 1] << 1) | (((m_wx >> k) & 1u) ? S[k] >> 31 : 0u);
    };
    {
        const uint32_t own = (1u << nw) - 1u;
        uint32_t S[4 * Q + 1];
        S[0] = (w0 - 1 >= 0 && w0 - 1 < nwords) ? __ldg(vis + w0 - 1) : 0u;
#pragma unroll
        for (int k = 0; k < 4 * Q; k++) {
            S[k + 1] = V[k];
            A[k] = 0u;
        }
        dilate(S, own);
        if (m_by & own) {
            load_run(w0 - wx_words, S);
            dilate(S, m_by & own);
        }
        if (m_bz & own) {
            load_run(w0 - plane, S);
            dilate(S, m_bz & own);
            if (m_by & m_bz & own) {
                load_run(w0 - plane - wx_words, S);
                dilate(S, m_by & m_bz & own);
            }
        }
#pragma unroll
        for (int k = 0; k < 4 * Q; k++)
            if (w0 + k >= nwords) A[k] = 0u;
    }
    (void)bdz;
    uint32_t cv = 0, ca = 0;
#pragma unroll
    for (int k = 0; k < 4 * Q; k++) {
        cv += __popc(V[k]);
        ca += __popc(A[k]);
    }
    uint32_t aggv, agga;
    uint32_t prev_v = block_exclusive_scan(cv, swv, &aggv);
    uint32_t prev_a = block_exclusive_scan(ca, swa, &agga);
    uint64_t *status_v = tile_status(scratch), *status_a = tile_status(scratch) + ntiles;
    if (threadIdx.x < 32) {
        const uint32_t e = tile_lookback(t, aggv, status_v, epoch);
        if (threadIdx.x == 0) {
            s_exv = e;
            if (t == last) *d_nvis = e + aggv;
        }
    } else if (threadIdx.x < 64) {
        const uint32_t e = tile_lookback(t, agga, status_a, epoch);
        if (threadIdx.x == 32) {
            s_exa = e;
            if (t == last) *d_nact = e + agga;
        }
    }
    __syncthreads();
    prev_v += s_exv;
    prev_a += s_exa;
#pragma unroll
    for (int k = 0; k < 4 * Q; k++) {
        uint32_t v = V[k], a = A[k];
        const int64_t w = w0 + k;
        if (v) {
            vis_word_off[w] = prev_v;
            const uint32_t base = (uint32_t)(w * 32);
            while (v) {
                vis_ids[prev_v++] = base + __ffs(v) - 1;
                v &= v - 1;
            }
        }
        if (a) {
            const uint32_t base = (uint32_t)(w * 32);
            while (a) {
                act_ids[prev_a++] = base + __ffs(a) - 1;
                a &= a - 1;
            }
        }
    }
}

void mark_extract(const uint32_t *vis, int64_t nwords, int wx_words, int bdy, int bdz, uint32_t *vis_word_off,
                  uint32_t *vis_ids, uint32_t *d_nvis, uint32_t *act_ids, uint32_t *d_nact, uint32_t *partials,
                  cudaStream_t st) {
    if (nwords <= 0) {
        WC_CUDA(cudaMemsetAsync(d_nvis, 0, sizeof(uint32_t), st));
        WC_CUDA(cudaMemsetAsync(d_nact, 0, sizeof(uint32_t), st));
        return;
    }
    const int64_t q16 = std::min<int64_t>(kMarkQ16, std::max<int64_t>(1, ceil_div(nwords, (int64_t)num_sms() * WC_DENSE_CTAS_PER_SM * 256 * 4)));
    const unsigned grid = (unsigned)ceil_div(nwords, 256 * 4 * q16);
    launch_pdl(k_mark_extract<kMarkQ16>, grid, 256, 0, st, vis, nwords, (int)q16, wx_words, bdy, bdz, vis_word_off,
               vis_ids, d_nvis, act_ids, d_nact, reinterpret_cast<uint64_t *>(partials), scan_epoch());
    WC_LAUNCH_CHECK();
}

// summary word i -> ascending indices of its set bits (the non-zero words of
// the bitmap), clearing the summary word
struct SinkList {
    uint32_t *summary, *list;
    __device__ __forceinline__ void operator()(int64_t i, uint32_t prefix, uint32_t) const {
        uint32_t v = summary[i];
        if (v) summary[i] = 0u;
        while (v) {
            list[prefix++] = (uint32_t)(i * 32 + __ffs(v) - 1);
            v &= v - 1;
        }
    }
};

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
    __device__ __forceinline__ void operator()(int64_t i, uint32_t prefix, uint32_t) const {
        const uint32_t w = idx[i];
        uint32_t v = bm[w];
        if (word_offsets) word_offsets[w] = prefix;
        if (clear) bm[w] = 0u;
        const uint32_t base = ((uint32_t)w % (uint32_t)id_mod) * 32u;  // (w < 2^32)
        while (v) {
            ids[prefix++] = base + __ffs(v) - 1;
            v &= v - 1;
        }
    }
};

void bitmap_extract_listed(uint32_t *bm, uint32_t *summary, int64_t nwords_max, int64_t nlist_max, int64_t id_mod,
                           uint32_t *word_offsets, uint32_t *ids, uint32_t *d_count, bool clear, uint32_t *word_list,
                           uint32_t *d_nlist, uint32_t *partials, cudaStream_t st, const uint32_t *d_nsummary) {
    const int64_t ns = ceil_div(nwords_max, 32);
    nlist_max = std::min(nlist_max, nwords_max);
    if (ns <= 0 || nlist_max <= 0) {
        WC_CUDA(cudaMemsetAsync(d_count, 0, sizeof(uint32_t), st));
        return;
    }
    launch_pdl(k_scan_onepass<LoadPopc, SinkList>, scan_grid(ns), kScanThreads, 0, st, 
        LoadPopc{summary}, SinkList{summary, word_list}, ns, d_nsummary, reinterpret_cast<uint64_t *>(partials),
        scan_epoch(), d_nlist, NoEpilogue{});
    WC_LAUNCH_CHECK();
    launch_pdl(k_scan_onepass<LoadPopcIdx, SinkBitsIdx>, scan_grid(nlist_max), kScanThreads, 0, st, 
        LoadPopcIdx{bm, word_list}, SinkBitsIdx{bm, word_list, word_offsets, ids, id_mod, clear}, nlist_max, d_nlist,
        reinterpret_cast<uint64_t *>(partials), scan_epoch(), d_count, NoEpilogue{});
    WC_LAUNCH_CHECK();
}

}  // namespace wc
