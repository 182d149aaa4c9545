// Shared-memory / MIO instruction throughput on one SM pipe, per SM cycle:
// broadcast LDS.32 / .64 / .128, LDS.128 with 3 distinct addresses per warp,
// SHFL.IDX with a uniform source lane, and shared fp32 atomics (RED / ATOMS).
// Results feed the P2G design (lane = stencil node, particle records
// broadcast from shared memory).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
    __shared__ __align__(16) float sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = (float)i;
    __syncthreads();
    unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    const int lane = threadIdx.x & 31;
    unsigned x = 0;
    float fx = 0.f;
    int j = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const unsigned a = base + (((j + i) & 63) << 4);
            if (MODE == 0) {
                unsigned v; asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a)); x ^= v;
            } else if (MODE == 1) {
                unsigned v, w; asm volatile("ld.volatile.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v), "=r"(w) : "r"(a)); x ^= v ^ w;
            } else if (MODE == 2) {
                unsigned v0, v1, v2, v3;
                asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(a));
                x ^= v0 ^ v1 ^ v2 ^ v3;
            } else if (MODE == 3) {
                // 3 distinct 16-byte addresses (lane groups of 9 / 9 / 14), different banks
                const unsigned a3 = a + (unsigned)((lane / 9 > 2 ? 2 : lane / 9) << 4);
                unsigned v0, v1, v2, v3;
                asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(a3));
                x ^= v0 ^ v1 ^ v2 ^ v3;
            } else if (MODE == 4) {
                x ^= __shfl_sync(0xffffffffu, x + i, (j + i) & 31);
            } else if (MODE == 5) {
                // per-lane distinct addresses, conflict-free: red.shared.add.f32
                float* p = sm + ((lane + 32 * ((j + i) & 15)) & 4095);
                atomicAdd(p, 1.0f);
            } else if (MODE == 6) {
                // per-lane read-modify-write (LDS + FADD + STS)
                volatile float* p = sm + ((lane + 32 * ((j + i) & 15)) & 4095);
                *p = *p + 1.0f;
            }
        }
        j += 3;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)x + fx + sm[lane];
}
int main() {
    float* out; cudaMalloc(&out, 148 * 8 * 256 * 4 * 4);
    int iters = 2048;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* nm[7] = {"LDS.32 bcast ", "LDS.64 bcast ", "LDS.128 bcast", "LDS.128 3-addr", "SHFL.IDX     ",
                         "RED.shared.f32", "LDS+FADD+STS "};
    for (int rep = 0; rep < 2; ++rep) {
        for (int which = 0; which < 7; ++which) {
            int blocks = 148 * 8, threads = 256;
            cudaEventRecord(e0);
            switch (which) {
                case 0: k<0><<<blocks, threads>>>(out, iters); break;
                case 1: k<1><<<blocks, threads>>>(out, iters); break;
                case 2: k<2><<<blocks, threads>>>(out, iters); break;
                case 3: k<3><<<blocks, threads>>>(out, iters); break;
                case 4: k<4><<<blocks, threads>>>(out, iters); break;
                case 5: k<5><<<blocks, threads>>>(out, iters); break;
                case 6: k<6><<<blocks, threads>>>(out, iters); break;
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)blocks * threads / 32 * iters * 8;    // warp-level ops
            double smcyc = ms * 1e-3 * 1.965e9 * 148;
            printf("%s: %.3f ms, %.3f SM-cycles per warp op\n", nm[which], ms, smcyc / ops);
        }
    }
    return 0;
}
