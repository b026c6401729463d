// Microbenchmark: throughput of scalar FFMA vs packed FFMA2 (fma.rn.f32x2) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2(float a, float b) {
    unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
template <int MODE> __global__ void k(float* out, float s, int iters) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    if (MODE == 0) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f * i + 1.0f);  // imm form
    } else if (MODE == 1) {
        float c[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = out[i + 32];
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, c[i]);  // 3-reg form
    } else {
        unsigned long long A[8], C[8], S = f2(s, s);
#pragma unroll
        for (int i = 0; i < 8; ++i) { A[i] = f2(a[2 * i], a[2 * i + 1]); C[i] = f2(out[2 * i + 32], out[2 * i + 33]); }
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) A[i] = fma2(A[i], S, C[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(A[i])); a[2*i] = x; a[2*i+1] = y; }
    }
    float t = 0; for (int i = 0; i < 16; ++i) t += a[i];
    if (t == 12345.f) out[0] = t;
}
int main() {
    float* d; cudaMalloc(&d, 1 << 20); cudaMemset(d, 0, 1 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 4096, blocks = 148 * 8, thr = 256;
    for (int m = 0; m < 3; ++m) for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (m == 0) k<0><<<blocks, thr>>>(d, 0.999f, iters);
        if (m == 1) k<1><<<blocks, thr>>>(d, 0.999f, iters);
        if (m == 2) k<2><<<blocks, thr>>>(d, 0.999f, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 16 * iters * (double)blocks * thr;
        if (rep) printf("mode %d (%s): %.3f ms, %.1f TFLOP/s fp32\n", m, m == 0 ? "FFMA imm" : m == 1 ? "FFMA 3-reg" : "FFMA2", ms, fl / ms / 1e9);
    }
    return 0;
}
