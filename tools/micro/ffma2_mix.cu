// Does FFMA2 (fma.rn.f32x2) free issue slots?  Mixes of FP32 FMAs with
// integer ALU ops or shared-memory broadcast loads, same FLOPs per iteration:
//   A: 16 FFMA + 8 ALU      B: 8 FFMA2 + 8 ALU
//   C: 16 FFMA + 8 LDS.128  D: 8 FFMA2 + 8 LDS.128
// If FFMA2 takes one issue slot and two FMA-pipe cycles, B and D issue in
// ~16 slots where A and C need 24.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
    u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
template <int MODE>
__global__ void k(float* out, float s, int iters) {
    __shared__ float4 sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = make_float4(s, s + 1, s + 2, s + 3);
    __syncthreads();
    float a[16];
    u64 a2[8];
    unsigned ia[8];
    float4 acc4 = make_float4(0, 0, 0, 0);
    float b = s * 1.0001f, c = s * 0.9999f;
    float2 bb = make_float2(b, b), cc = make_float2(c, c);
    u64 b2 = *(u64*)&bb, c2 = *(u64*)&cc;
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x + i;
    for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x + i, i); a2[i] = *(u64*)&v; ia[i] = threadIdx.x * (i + 1); }
    int j = 0;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) a2[i] = f2fma(a2[i], b2, c2);
        }
        if (MODE < 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) ia[i] = (ia[i] ^ (unsigned)it) + 0x9e3779b9u;
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float4 t;
                unsigned addr = (unsigned)__cvta_generic_to_shared(&sm[(j + i) & 63]);
                asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w) : "r"(addr));
            }
            j += 3;
        }
    }
    float t = acc4.x;
    for (int i = 0; i < 16; ++i) t += a[i];
    for (int i = 0; i < 8; ++i) { float2 v = *(float2*)&a2[i]; t += v.x + v.y + (float)ia[i]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 256 * 4 * 4);
    int iters = 4096;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* nm[4] = {"16 FFMA + 8 ALU   ", "8 FFMA2 + 8 ALU   ", "16 FFMA + 8 LDS128", "8 FFMA2 + 8 LDS128"};
    for (int rep = 0; rep < 2; ++rep) {
        for (int which = 0; which < 4; ++which) {
            int blocks = 148 * 8, threads = 256;
            cudaEventRecord(e0);
            if (which == 0) k<0><<<blocks, threads>>>(out, 1.0f, iters);
            if (which == 1) k<1><<<blocks, threads>>>(out, 1.0f, iters);
            if (which == 2) k<2><<<blocks, threads>>>(out, 1.0f, iters);
            if (which == 3) k<3><<<blocks, threads>>>(out, 1.0f, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double warp_iters = (double)blocks * threads / 32 * iters;
            double cyc = ms * 1e-3 * 1.965e9 * 148 * 4;   // SMSP-cycles
            printf("%s: %.3f ms, %.2f SMSP-cycles per warp-iteration\n", nm[which], ms, cyc / warp_iters);
        }
    }
    return 0;
}
