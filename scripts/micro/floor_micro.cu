// Micro-benchmark (experiment only): where the ~20 us of a one-wave bitmap
// extraction over 15.7 MB goes.  Each mode adds one ingredient.
//   E empty kernel                 R read + popc (one store per CTA)
//   T R + ticket atomic            L T + warp look-back (no id writes)
#include "wc_prims.cuh"
#include <vector>
using namespace wc;
constexpr int Q16 = 4;
constexpr int64_t CHUNK = 256LL * 4 * Q16;
template <int MODE>
__global__ void __launch_bounds__(256) k_floor(const uint32_t *bm, int64_t nwords, uint64_t *status, uint32_t epoch,
                                               uint32_t *out) {
    __shared__ uint32_t sw[32], s_t;
    if (MODE == 0) return;
    int64_t t = blockIdx.x;
    if (MODE >= 2) {
        bool lt;
        if (threadIdx.x == 0) s_t = take_ticket(status, lt);
        __syncthreads();
        t = s_t;
    }
    const int64_t w0 = t * CHUNK + (int64_t)threadIdx.x * 4 * Q16;
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < Q16; j++) {
        const int64_t w = w0 + 4 * j;
        const uint4 v = w + 4 <= nwords ? *reinterpret_cast<const uint4 *>(bm + w) : make_uint4(0, 0, 0, 0);
        cnt += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    }
    uint32_t agg;
    block_exclusive_scan(cnt, sw, &agg);
    uint32_t excl = 0;
    if (MODE == 3 && threadIdx.x < 32) excl = tile_lookback(t, agg, tile_status(status), epoch);
    if (threadIdx.x == 0) out[t] = agg + excl;
}
int main() {
    const int64_t nwords = 3932160;
    uint32_t *bm, *out;
    uint64_t *status;
    cudaMalloc(&bm, 4 * nwords);
    cudaMemset(bm, 0x11, 4 * nwords);
    cudaMalloc(&out, 4 * 8192);
    cudaMalloc(&status, 8 * 8192);
    cudaMemset(status, 0, 8 * 8192);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[] = {"E empty", "R read", "T ticket", "L lookback"};
    for (int q16 = 1; q16 <= 4; q16 *= 2) {
        (void)q16;
    }
    const unsigned grid = (unsigned)((nwords + CHUNK - 1) / CHUNK);
    for (int mode = 0; mode < 4; mode++) {
        float tot = 0, totg = 0;
        const int iters = 200;
        // (a) one launch timed alone; (b) 20 back-to-back launches in a graph
        for (int it = 0; it < iters + 10; it++) {
            cudaEventRecord(e0);
            const uint32_t ep = 100 + mode * 1000 + it;
            switch (mode) {
                case 0: k_floor<0><<<grid, 256>>>(bm, nwords, status, ep, out); break;
                case 1: k_floor<1><<<grid, 256>>>(bm, nwords, status, ep, out); break;
                case 2: k_floor<2><<<grid, 256>>>(bm, nwords, status, ep, out); break;
                case 3: k_floor<3><<<grid, 256>>>(bm, nwords, status, ep, out); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 10) tot += ms;
        }
        cudaStream_t s;
        cudaStreamCreate(&s);
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < 20; k++) {
            const uint32_t ep = 500000 + mode * 1000 + k;
            switch (mode) {
                case 0: k_floor<0><<<grid, 256, 0, s>>>(bm, nwords, status, ep, out); break;
                case 1: k_floor<1><<<grid, 256, 0, s>>>(bm, nwords, status, ep, out); break;
                case 2: k_floor<2><<<grid, 256, 0, s>>>(bm, nwords, status, ep, out); break;
                case 3: k_floor<3><<<grid, 256, 0, s>>>(bm, nwords, status, ep, out); break;
            }
        }
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&totg, e0, e1);
        printf("%-12s alone %7.2f us   in a 20-launch graph %7.2f us per launch  (%s)\n", names[mode],
               1000.0 * tot / iters, 1000.0 * totg / 20, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
