// FP32 issue microbenchmark: FFMA (3-register form) vs FFMA2 (fma.rn.f32x2)
// chains, 8 independent chains per thread, many warps: reports FLOP/s.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
    u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__global__ void k1(float* out, float s, int iters) {
    float a[8], b = s * 1.0001f, c = s * 0.9999f;
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], c, b);
    }
    float t = 0; for (int i = 0; i < 8; ++i) t += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k2(float* out, float s, int iters) {
    u64 a[8];
    float2 bb = make_float2(s * 1.0001f, s * 1.0002f), cc = make_float2(s * 0.9999f, s * 0.9998f);
    u64 b = *(u64*)&bb, c = *(u64*)&cc;
    for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x + i, i); a[i] = *(u64*)&v; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = f2fma(a[i], b, c);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = f2fma(a[i], c, b);
    }
    float t = 0; for (int i = 0; i < 8; ++i) { float2 v = *(float2*)&a[i]; t += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 256 * 4 * 4);
    int iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        for (int which = 0; which < 2; ++which) {
            int blocks = 148 * 8, threads = 256;
            cudaEventRecord(e0);
            if (which == 0) k1<<<blocks, threads>>>(out, 1.0f, iters);
            else k2<<<blocks, threads>>>(out, 1.0f, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * blocks * threads * (double)iters * 16 * (which ? 2 : 1);
            printf("%s: %.3f ms, %.1f TFLOP/s fp32\n", which ? "FFMA2" : "FFMA ", ms, flops / ms / 1e9);
        }
    }
    return 0;
}
