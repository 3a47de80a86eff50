// Micro-benchmark (experiment only): a chain of K tiny dependent kernels in a
// CUDA graph (with and without programmatic dependent launch) against one
// cooperative kernel with K grid-wide barriers.  Each step reads a counter
// written by the previous one (the pass pipeline's control-block pattern).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_step(unsigned *ctl, int k, bool pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    const unsigned v = ctl[k];
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl[k + 1] = v + 1;
}
__global__ void k_coop(unsigned *ctl, int K) {
    cg::grid_group g = cg::this_grid();
    for (int k = 0; k < K; k++) {
        const unsigned v = *(volatile unsigned *)(ctl + k);
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl[k + 1] = v + 1;
        g.sync();
    }
}
int main() {
    const int K = 16;
    unsigned *ctl;
    cudaMalloc(&ctl, 4 * (K + 2));
    cudaMemset(ctl, 0, 4 * (K + 2));
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int pdl = 0; pdl < 2; pdl++)
        for (int grid : {1, nsm, nsm * 4, nsm * 8}) {
            cudaGraph_t gr;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int k = 0; k < K; k++) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = grid;
                cfg.blockDim = 256;
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl;
                cudaLaunchKernelEx(&cfg, k_step, ctl, k, (bool)pdl);
            }
            cudaStreamEndCapture(s, &gr);
            cudaGraphInstantiate(&ge, gr, 0);
            for (int w = 0; w < 3; w++) cudaGraphLaunch(ge, s);
            cudaEventRecord(e0, s);
            for (int it = 0; it < 50; it++) cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("graph chain pdl=%d grid=%5d: %.2f us per kernel\n", pdl, grid, 1000.0 * ms / (50 * K));
        }
    for (int per : {1, 2, 4}) {
        int grid = nsm * per;
        void *args[] = {&ctl, (void *)&K};
        for (int w = 0; w < 3; w++) cudaLaunchCooperativeKernel((void *)k_coop, grid, 256, args, 0, s);
        cudaEventRecord(e0, s);
        for (int it = 0; it < 50; it++) cudaLaunchCooperativeKernel((void *)k_coop, grid, 256, args, 0, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("cooperative grid=%5d: %.2f us per grid sync (incl. launch / %d)  %s\n", grid, 1000.0 * ms / (50 * K), K,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
