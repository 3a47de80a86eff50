// Micro-benchmark (experiment only, not part of the library): ways to turn a
// 15.7 MB visibility bitmap into ascending ids + word offsets.
//   W  warp look-back (the library's k_bitmap_dense)       W4 warp, 4 statuses per lane
//   C  whole-CTA look-back                                  N  no look-back (floor; wrong ids)
//   R  reduce-then-extract (two kernels, no look-back)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2309_10212_b200/csrc dense_micro.cu
#include "wc_prims.cuh"
#include <vector>
#include <random>
using namespace wc;

constexpr int Q16 = 4;
constexpr int64_t CHUNK = 256LL * 4 * Q16;

template <int MODE>  // 0 W, 1 W4, 2 C, 3 N
__global__ void __launch_bounds__(256) k_dense(uint32_t *bm, int64_t nwords, uint32_t *word_offsets, uint32_t *ids,
                                               uint64_t *status, uint32_t epoch, uint32_t *d_count) {
    __shared__ uint32_t sw[32], slb[64];
    __shared__ uint32_t s_excl, s_ticket;
    const int64_t last = (nwords - 1) / CHUNK;
    bool lt = false;
    uint32_t tk = 0;
    if (threadIdx.x == 0) tk = take_ticket(status, lt);
    uint4 q[Q16];
    auto load = [&](int64_t tt) {
        const int64_t w0 = tt * CHUNK + (int64_t)threadIdx.x * 4 * Q16;
#pragma unroll
        for (int j = 0; j < Q16; j++) {
            const int64_t w = w0 + 4 * j;
            q[j] = w + 4 <= nwords ? *reinterpret_cast<const uint4 *>(bm + w) : make_uint4(0, 0, 0, 0);
        }
    };
    load(blockIdx.x);
    if (threadIdx.x == 0) s_ticket = tk;
    __syncthreads();
    const int64_t t = s_ticket;
    if (t != (int64_t)blockIdx.x) load(t);
    const int64_t w0 = t * CHUNK + (int64_t)threadIdx.x * 4 * Q16;
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < Q16; j++) cnt += __popc(q[j].x) + __popc(q[j].y) + __popc(q[j].z) + __popc(q[j].w);
    uint32_t agg;
    uint32_t pre = block_exclusive_scan(cnt, sw, &agg);
    uint32_t excl = 0;
    uint64_t *st = tile_status(status);
    if (MODE == 0) {
        if (threadIdx.x < 32) excl = tile_lookback(t, agg, st, epoch);
    } else if (MODE == 1) {
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            if (t == 0) {
                if (lane == 0) store_status(st, epoch, kFlagPrefix, agg);
            } else {
                if (lane == 0) store_status(st + t, epoch, kFlagAggregate, agg);
                for (int64_t hi = t - 1;; hi -= 128) {
                    unsigned long long w[4];
                    uint32_t pmin = 0xFFFFFFFFu, f[4];
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const int64_t idx = hi - (k * 32 + lane);
                        w[k] = idx >= 0 ? *reinterpret_cast<volatile unsigned long long *>(st + idx)
                                        : ((unsigned long long)epoch << 34) | ((unsigned long long)kFlagPrefix << 32);
                    }
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const int64_t idx = hi - (k * 32 + lane);
                        f[k] = (uint32_t)(w[k] >> 34) == epoch ? (uint32_t)(w[k] >> 32) & 3u : 0u;
                        while (f[k] == 0) {
                            w[k] = *reinterpret_cast<volatile unsigned long long *>(st + idx);
                            f[k] = (uint32_t)(w[k] >> 34) == epoch ? (uint32_t)(w[k] >> 32) & 3u : 0u;
                        }
                        if (f[k] == kFlagPrefix) pmin = min(pmin, (uint32_t)(k * 32 + lane));
                    }
                    const uint32_t fp = __reduce_min_sync(0xffffffffu, pmin);
                    uint32_t c = 0;
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        if ((uint32_t)(k * 32 + lane) <= fp) c += (uint32_t)w[k];
                    excl += __reduce_add_sync(0xffffffffu, c);
                    if (fp != 0xFFFFFFFFu) break;
                }
                if (lane == 0) store_status(st + t, epoch, kFlagPrefix, excl + agg);
            }
        }
    } else if (MODE == 2) {
        excl = tile_lookback_cta(t, agg, st, epoch, slb);
    }
    if (threadIdx.x == 0) {
        s_excl = excl;
        if (t == last) *d_count = excl + agg;
    }
    __syncthreads();
    pre += s_excl;
    if (!cnt) return;
#pragma unroll
    for (int j = 0; j < Q16; j++) {
        const uint32_t wv[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
        for (int c = 0; c < 4; c++) {
            uint32_t v = wv[c];
            if (!v) continue;
            const int64_t w = w0 + 4 * j + c;
            word_offsets[w] = pre;
            const uint32_t base = (uint32_t)(w * 32);
            while (v) {
                ids[pre++] = base + __ffs(v) - 1;
                v &= v - 1;
            }
        }
    }
}

// R: counts per chunk, then extraction with the prefix summed by the whole CTA
__global__ void __launch_bounds__(256) k_count(const uint32_t *bm, int64_t nwords, uint32_t *counts) {
    __shared__ uint32_t sw[32];
    const int64_t w0 = blockIdx.x * CHUNK + (int64_t)threadIdx.x * 4 * Q16;
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < Q16; j++) {
        const int64_t w = w0 + 4 * j;
        const uint4 v = w + 4 <= nwords ? *reinterpret_cast<const uint4 *>(bm + w) : make_uint4(0, 0, 0, 0);
        cnt += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    uint32_t agg;
    block_exclusive_scan(cnt, sw, &agg);
    if (threadIdx.x == 0) counts[blockIdx.x] = agg;
}
__global__ void __launch_bounds__(256) k_extract(const uint32_t *bm, int64_t nwords, const uint32_t *counts,
                                                 uint32_t *word_offsets, uint32_t *ids, uint32_t *d_count) {
    __shared__ uint32_t sw[32], s_base;
    uint4 q[Q16];
    const int64_t w0 = blockIdx.x * CHUNK + (int64_t)threadIdx.x * 4 * Q16;
#pragma unroll
    for (int j = 0; j < Q16; j++) {
        const int64_t w = w0 + 4 * j;
        q[j] = w + 4 <= nwords ? *reinterpret_cast<const uint4 *>(bm + w) : make_uint4(0, 0, 0, 0);
    }
    uint32_t s = 0;
    for (int64_t i = threadIdx.x; i < blockIdx.x; i += 256) s += counts[i];
    s = __reduce_add_sync(0xffffffffu, s);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t b = 0;
        for (int i = 0; i < 8; i++) b += sw[i];
        s_base = b;
        if (blockIdx.x == gridDim.x - 1) *d_count = b + counts[blockIdx.x];
    }
    __syncthreads();
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < Q16; j++) cnt += __popc(q[j].x) + __popc(q[j].y) + __popc(q[j].z) + __popc(q[j].w);
    uint32_t agg;
    uint32_t pre = block_exclusive_scan(cnt, sw, &agg) + s_base;
    if (!cnt) return;
#pragma unroll
    for (int j = 0; j < Q16; j++) {
        const uint32_t wv[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
        for (int c = 0; c < 4; c++) {
            uint32_t v = wv[c];
            if (!v) continue;
            const int64_t w = w0 + 4 * j + c;
            word_offsets[w] = pre;
            const uint32_t base = (uint32_t)(w * 32);
            while (v) {
                ids[pre++] = base + __ffs(v) - 1;
                v &= v - 1;
            }
        }
    }
}

int main(int argc, char **argv) {
    const int64_t nwords = 3932160;  // C3: 126 M blocks
    const double density = argc > 1 ? atof(argv[1]) : 0.2;  // set bits per word
    std::vector<uint32_t> h(nwords, 0);
    std::mt19937_64 rng(1);
    const int64_t nbits = (int64_t)(density * nwords);
    for (int64_t i = 0; i < nbits; i++) {
        const uint64_t b = rng() % (uint64_t)(nwords * 32);
        h[b >> 5] |= 1u << (b & 31);
    }
    uint32_t *bm, *bm0, *wo, *ids, *cnt, *counts;
    uint64_t *status;
    cudaMalloc(&bm, 4 * nwords);
    cudaMalloc(&bm0, 4 * nwords);
    cudaMalloc(&wo, 4 * nwords);
    cudaMalloc(&ids, 4 * nwords * 32 / 8);
    cudaMalloc(&cnt, 4);
    cudaMalloc(&counts, 4 * 4096);
    cudaMalloc(&status, 8 * 8192);
    cudaMemset(status, 0, 8 * 8192);
    cudaMemcpy(bm0, h.data(), 4 * nwords, cudaMemcpyHostToDevice);
    const unsigned grid = (unsigned)((nwords + CHUNK - 1) / CHUNK);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[] = {"W warp", "W4 warp x4", "C cta", "N none", "R two-kernel"};
    uint32_t ref_count = 0;
    std::vector<uint32_t> ref_ids;
    for (int mode = 0; mode < 5; mode++) {
        float tot = 0;
        const int iters = 200;
        for (int it = 0; it < iters + 10; it++) {
            cudaMemcpyAsync(bm, bm0, 4 * nwords, cudaMemcpyDeviceToDevice);
            const uint32_t epoch = 1000 + mode * 1000 + it;
            cudaEventRecord(e0);
            switch (mode) {
                case 0: k_dense<0><<<grid, 256>>>(bm, nwords, wo, ids, status, epoch, cnt); break;
                case 1: k_dense<1><<<grid, 256>>>(bm, nwords, wo, ids, status, epoch, cnt); break;
                case 2: k_dense<2><<<grid, 256>>>(bm, nwords, wo, ids, status, epoch, cnt); break;
                case 3: k_dense<3><<<grid, 256>>>(bm, nwords, wo, ids, status, epoch, cnt); break;
                case 4:
                    k_count<<<grid, 256>>>(bm, nwords, counts);
                    k_extract<<<grid, 256>>>(bm, nwords, counts, wo, ids, cnt);
                    break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 10) tot += ms;
        }
        uint32_t c;
        cudaMemcpy(&c, cnt, 4, cudaMemcpyDeviceToHost);
        std::vector<uint32_t> hid(c);
        cudaMemcpy(hid.data(), ids, 4 * (size_t)c, cudaMemcpyDeviceToHost);
        if (mode == 0) {
            ref_count = c;
            ref_ids = hid;
        }
        const bool ok = mode == 3 || (c == ref_count && hid == ref_ids);
        printf("%-14s %8.2f us  count %u  %s  (%s)\n", names[mode], 1000.0 * tot / iters, c, ok ? "ids ok" : "IDS DIFFER",
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
