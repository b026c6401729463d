// Micro-benchmark: cost of a cooperative grid-wide barrier vs a dependent kernel boundary in a
// CUDA graph (with and without programmatic dependent launch) on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_bench gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, int* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) atomicAdd(sink, 1);
        g.sync();
    }
}
__global__ void k_tiny(int* sink) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) atomicAdd(sink + blockIdx.x % 64, 1);
}

int main() {
    int* sink;
    cudaMalloc(&sink, 4096);
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int per : {1, 2, 4}) {
        const int iters = 2000;
        void* args[] = {(void*)&iters, (void*)&sink};
        dim3 grid(sms * per), block(256);
        cudaLaunchCooperativeKernel((void*)k_sync, grid, block, args, 0, s);  // warm
        cudaEventRecord(a, s);
        cudaLaunchCooperativeKernel((void*)k_sync, grid, block, args, 0, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid.sync with %d CTAs x 256: %.3f us per barrier\n", sms * per, 1e3 * ms / iters);
    }
    for (int pdl : {0, 1}) {
        for (int ctas : {64, sms * 4}) {
            const int n = 1000;
            cudaGraph_t g;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            for (int i = 0; i < n; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(ctas);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = pdl;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, k_tiny, sink);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphExec_t ge;
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
            cudaEventRecord(a, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("graph of dependent tiny kernels (%d CTAs, PDL %d): %.3f us per kernel\n", ctas, pdl, 1e3 * ms / n);
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
