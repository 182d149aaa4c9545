// Slab staging for the multi-GPU decomposition:
//
//   mlbm_halo_pack / mlbm_halo_unpack   ghost tile columns of a level's SoA
//       block <-> a contiguous NCCL buffer (collectives (i) and (ii): copy, or
//       add for the ghost-node partial sums)
//   mlbm_migrate_pack / mlbm_migrate_unpack   particles whose x left the slab
//       (collective (iii)): one stable partition of the particle rows into
//       keep / to-left / to-right with warp-ballot + block-scan compaction,
//       then the arrivals appended after the kept particles
//
// The partition keeps the original relative order inside each class (block
// counts, one exclusive scan, ballot ranks inside the warps), so a migration
// is deterministic.
#include "common.cuh"

namespace mlbm {

template <typename T>
__global__ void k_halo_pack(const T* __restrict__ src, int64_t stride, int nrows, int64_t lo, int64_t len,
                            T* __restrict__ buf) {
    const int64_t total = (int64_t)nrows * len;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / len, c = i - r * len;
        buf[i] = src[r * stride + lo + c];
    }
}

template <typename T>
__global__ void k_halo_unpack(const T* __restrict__ buf, T* __restrict__ dst, int64_t stride, int nrows,
                              int64_t lo, int64_t len, int add) {
    const int64_t total = (int64_t)nrows * len;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / len, c = i - r * len;
        T* d = &dst[r * stride + lo + c];
        *d = add ? *d + buf[i] : buf[i];
    }
}

// ---------------------------------------------------------------------------
constexpr int MIG_B = 256;

__device__ __forceinline__ int mig_class(double x, double lo, double hi, int has_l, int has_r) {
    if (x < lo && has_l) return 1;
    if (x >= hi && has_r) return 2;
    return 0;
}

// per block: counts of the three classes
__global__ void k_mig_count(int n, const double* __restrict__ x, double lo, double hi, int has_l, int has_r,
                            int32_t* __restrict__ bcount) {
    __shared__ int s[3];
    if (threadIdx.x < 3) s[threadIdx.x] = 0;
    __syncthreads();
    const int p = blockIdx.x * MIG_B + threadIdx.x;
    const int c = p < n ? mig_class(x[p], lo, hi, has_l, has_r) : -1;
    const unsigned b1 = __ballot_sync(0xffffffffu, c == 1), b2 = __ballot_sync(0xffffffffu, c == 2),
                   b0 = __ballot_sync(0xffffffffu, c == 0);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s[0], __popc(b0));
        atomicAdd(&s[1], __popc(b1));
        atomicAdd(&s[2], __popc(b2));
    }
    __syncthreads();
    if (threadIdx.x < 3) bcount[(int64_t)blockIdx.x * 3 + threadIdx.x] = s[threadIdx.x];
}

// exclusive scan of the block counts per class (one block), totals into counts[3]
__global__ void k_mig_scan(int nb, int32_t* __restrict__ bcount, int32_t* __restrict__ counts) {
    __shared__ int carry[3];
    __shared__ int warp_sum[3][32];
    if (threadIdx.x < 3) carry[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = 0; base < nb; base += blockDim.x) {
        const int b = base + threadIdx.x;
        int v[3], incl[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            v[k] = b < nb ? bcount[(int64_t)b * 3 + k] : 0;
            int t = v[k];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += u;
            }
            incl[k] = t;
            if (lane == 31) warp_sum[k][wid] = t;
        }
        __syncthreads();
        if (wid == 0) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                int t = lane < nw ? warp_sum[k][lane] : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, t, o);
                    if (lane >= o) t += u;
                }
                if (lane < nw) warp_sum[k][lane] = t;          // inclusive over warps
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int before = (wid ? warp_sum[k][wid - 1] : 0) + incl[k] - v[k];
            if (b < nb) bcount[(int64_t)b * 3 + k] = carry[k] + before;
        }
        __syncthreads();
        if (threadIdx.x < 3) carry[threadIdx.x] += warp_sum[threadIdx.x][nw - 1];
        __syncthreads();
    }
    if (threadIdx.x < 3) counts[threadIdx.x] = carry[threadIdx.x];
}

struct MigArgs {
    int n, dim, rows;
    const double* x;
    const void* p;
    const int32_t* pid;
    int64_t ps;
    double lo, hi, x0, gx;
    int has_l, has_r;
    double* xo[3];
    void* po[3];
    int32_t* io[3];
    int64_t os[3];
    int64_t cap;
    const int32_t* boff;
    int32_t* counts;
};

template <typename R>
__global__ void k_mig_scatter(MigArgs A) {
    __shared__ int wcnt[3][MIG_B / 32];
    const int p = blockIdx.x * MIG_B + threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int c = p < A.n ? mig_class(A.x[p], A.lo, A.hi, A.has_l, A.has_r) : -1;
    unsigned bal[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) bal[k] = __ballot_sync(0xffffffffu, c == k);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k) wcnt[k][wid] = __popc(bal[k]);
    }
    __syncthreads();
    if (c < 0) return;
    int off = A.boff[(int64_t)blockIdx.x * 3 + c];
    for (int w = 0; w < wid; ++w) off += wcnt[c][w];
    off += __popc(bal[c] & ((1u << lane) - 1u));
    if (c != 0 && off >= A.cap) {             // send buffer overflow: counted, not written
        return;
    }
    double* xo = A.xo[c];
    R* po = (R*)A.po[c];
    const int64_t os = A.os[c];
    for (int a = 0; a < A.dim; ++a) {
        double v = A.x[a * A.ps + p];
        if (c != 0 && a == 0) {               // leaving: global x, periodic wrap
            v += A.x0;
            if (v < 0.0) v += A.gx;
            else if (v >= A.gx) v -= A.gx;
        }
        xo[a * os + off] = v;
    }
    const R* pp = (const R*)A.p;
    for (int r = 0; r < A.rows; ++r) po[r * os + off] = pp[r * A.ps + p];
    A.io[c][off] = A.pid[p];
}

template <typename R>
__global__ void k_mig_append(int m, int dim, int rows, const double* __restrict__ xi, const R* __restrict__ pi,
                             const int32_t* __restrict__ ii, int64_t is, double x0, double gx, double local_len,
                             double* __restrict__ x, R* __restrict__ pp, int32_t* __restrict__ pid, int64_t ps,
                             int at) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int q = at + j;
    for (int a = 0; a < dim; ++a) {
        double v = xi[a * is + j];
        if (a == 0) {                          // global -> local box (ghosts wrap)
            v -= x0;
            if (v < 0.0) v += gx;
            if (v >= local_len) v -= gx;
        }
        x[a * ps + q] = v;
    }
    for (int r = 0; r < rows; ++r) pp[r * ps + q] = pi[r * is + j];
    pid[q] = ii[j];
}

}  // namespace mlbm

using namespace mlbm;

static int grid_for(int64_t total) {
    const int64_t g = (total + 255) / 256;
    return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

extern "C" int mlbm_halo_pack(const void* src, int64_t stride, int32_t nrows, int64_t lo, int64_t hi,
                              void* buf, int32_t elem_bytes, void* stream) {
    const int64_t len = hi - lo;
    if (len <= 0 || nrows <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int G = grid_for(len * nrows);
    if (elem_bytes == 8) k_halo_pack<double><<<G, 256, 0, s>>>((const double*)src, stride, nrows, lo, len, (double*)buf);
    else if (elem_bytes == 4) k_halo_pack<float><<<G, 256, 0, s>>>((const float*)src, stride, nrows, lo, len, (float*)buf);
    else if (elem_bytes == 1) k_halo_pack<uint8_t><<<G, 256, 0, s>>>((const uint8_t*)src, stride, nrows, lo, len, (uint8_t*)buf);
    else return -1;
    return launch_status(1);
}

extern "C" int mlbm_halo_unpack(const void* buf, void* dst, int64_t stride, int32_t nrows, int64_t lo,
                                int64_t hi, int32_t dtype, int32_t add, void* stream) {
    const int64_t len = hi - lo;
    if (len <= 0 || nrows <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int G = grid_for(len * nrows);
    if (dtype) k_halo_unpack<double><<<G, 256, 0, s>>>((const double*)buf, (double*)dst, stride, nrows, lo, len, add);
    else k_halo_unpack<float><<<G, 256, 0, s>>>((const float*)buf, (float*)dst, stride, nrows, lo, len, add);
    return launch_status(1);
}

extern "C" int64_t mlbm_migrate_ws_bytes(int32_t n) {
    const int64_t nb = ((int64_t)(n > 0 ? n : 1) + MIG_B - 1) / MIG_B;
    return nb * 3 * 4;
}

extern "C" int mlbm_migrate_count(int32_t n, const double* x, double lo, double hi, int32_t has_left,
                                  int32_t has_right, int32_t* counts, void* ws, int64_t ws_bytes,
                                  void* stream) {
    cudaStream_t s = as_stream(stream);
    if (n <= 0) {
        cudaMemsetAsync(counts, 0, 3 * sizeof(int32_t), s);
        return 0;
    }
    if (ws_bytes < mlbm_migrate_ws_bytes(n)) return -1;
    const int nb = (n + MIG_B - 1) / MIG_B;
    int32_t* bc = (int32_t*)ws;
    k_mig_count<<<nb, MIG_B, 0, s>>>(n, x, lo, hi, has_left, has_right, bc);
    k_mig_scan<<<1, 1024, 0, s>>>(nb, bc, counts);
    return launch_status(2);
}

extern "C" int mlbm_migrate_pack(int32_t dim, int32_t n, const double* x, const void* p, const int32_t* pid,
                                 int64_t ps, int32_t rows, int32_t dtype, double lo, double hi, double x0,
                                 double gx, int32_t has_left, int32_t has_right, double* x_keep,
                                 void* p_keep, int32_t* pid_keep, int64_t ks, double* x_left,
                                 void* p_left, int32_t* id_left, int64_t ls, double* x_right,
                                 void* p_right, int32_t* id_right, int64_t rs, const void* ws,
                                 int64_t ws_bytes, void* stream) {
    if (n <= 0) return 0;
    if (ws_bytes < mlbm_migrate_ws_bytes(n)) return -1;
    cudaStream_t s = as_stream(stream);
    const int nb = (n + MIG_B - 1) / MIG_B;
    MigArgs A;
    A.n = n; A.dim = dim; A.rows = rows; A.x = x; A.p = p; A.pid = pid; A.ps = ps;
    A.lo = lo; A.hi = hi; A.x0 = x0; A.gx = gx; A.has_l = has_left; A.has_r = has_right;
    A.xo[0] = x_keep; A.po[0] = p_keep; A.io[0] = pid_keep; A.os[0] = ks;
    A.xo[1] = x_left; A.po[1] = p_left; A.io[1] = id_left; A.os[1] = ls;
    A.xo[2] = x_right; A.po[2] = p_right; A.io[2] = id_right; A.os[2] = rs;
    A.cap = ((int64_t)1) << 62; A.boff = (const int32_t*)ws; A.counts = nullptr;
    if (dtype) k_mig_scatter<double><<<nb, MIG_B, 0, s>>>(A);
    else k_mig_scatter<float><<<nb, MIG_B, 0, s>>>(A);
    return launch_status(1);
}

extern "C" int mlbm_migrate_unpack(int32_t dim, int32_t m, const double* x_in, const void* p_in,
                                   const int32_t* id_in, int64_t in_stride, int32_t rows, int32_t dtype,
                                   double x0, double gx, double local_len, double* x, void* p,
                                   int32_t* pid, int64_t ps, int32_t at, void* stream) {
    if (m <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int G = (m + 255) / 256;
    if (dtype) k_mig_append<double><<<G, 256, 0, s>>>(m, dim, rows, x_in, (const double*)p_in, id_in, in_stride,
                                                      x0, gx, local_len, x, (double*)p, pid, ps, at);
    else k_mig_append<float><<<G, 256, 0, s>>>(m, dim, rows, x_in, (const float*)p_in, id_in, in_stride,
                                               x0, gx, local_len, x, (float*)p, pid, ps, at);
    return launch_status(1);
}
