// Shared device definitions: lattice tables (D2Q9 / D3Q27 with opposite
// directions adjacent), field layout, tile geometry, error record helpers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "mlbm_b200.h"

#define MLBM_HD __host__ __device__ __forceinline__

namespace mlbm {

constexpr double CS2 = 1.0 / 3.0;

template <int D> struct Geo;
template <> struct Geo<2> {
    static constexpr int Q = 9, NP = 4, T = 16, NB = 9, NS = 3, N3 = 2,
                         NM = 6, NF = 10, NC = 4, K = 9;
};
template <> struct Geo<3> {
    static constexpr int Q = 27, NP = 13, T = 64, NB = 27, NS = 6, N3 = 7,
                         NM = 10, NF = 15, NC = 8, K = 27;
};
// field indices: 0 drho | 1..D u | D+1..D+NS S | eps | f[D] | phi
template <int D> MLBM_HD constexpr int fi_u(int a) { return 1 + a; }
template <int D> MLBM_HD constexpr int fi_s(int k) { return 1 + D + k; }
template <int D> MLBM_HD constexpr int fi_eps() { return 1 + D + Geo<D>::NS; }
template <int D> MLBM_HD constexpr int fi_f(int a) { return 2 + D + Geo<D>::NS + a; }
template <int D> MLBM_HD constexpr int fi_phi() { return 2 + 2 * D + Geo<D>::NS; }

// S component index of (a <= b), row-major upper triangle
template <int D> MLBM_HD constexpr int sidx(int a, int b) {
    return a <= b ? a * D - a * (a - 1) / 2 + (b - a) : b * D - b * (b - 1) / 2 + (a - b);
}
template <int D> MLBM_HD constexpr int s_a(int k) {
    return D == 2 ? (k < 2 ? 0 : 1) : (k < 3 ? 0 : (k < 5 ? 1 : 2));
}
template <int D> MLBM_HD constexpr int s_b(int k) {
    return D == 2 ? (k == 0 ? 0 : 1) : (k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 2 : k == 3 ? 1 : 2);
}

// pair representatives; direction 2p+1 = rep p, 2p+2 = -rep p, 0 = rest
MLBM_HD constexpr int rep2(int p, int a) {
    return a == 0 ? (p == 0 ? 1 : p == 1 ? 0 : p == 2 ? 1 : -1)
                  : (p == 0 ? 0 : 1);
}
MLBM_HD constexpr int rep3(int p, int a) {
    // (1,0,0) (0,1,0) (0,0,1) (1,1,0) (1,0,1) (1,0,-1) (1,-1,0)
    // (0,1,1) (0,1,-1) (1,1,1) (1,1,-1) (1,-1,1) (1,-1,-1)
    return a == 0 ? (p == 0 ? 1 : p == 1 ? 0 : p == 2 ? 0 : p == 3 ? 1 : p == 4 ? 1 :
                     p == 5 ? 1 : p == 6 ? 1 : p == 7 ? 0 : p == 8 ? 0 : 1)
         : a == 1 ? (p == 0 ? 0 : p == 1 ? 1 : p == 2 ? 0 : p == 3 ? 1 : p == 4 ? 0 :
                     p == 5 ? 0 : p == 6 ? -1 : p == 7 ? 1 : p == 8 ? 1 : p == 9 ? 1 :
                     p == 10 ? 1 : -1)
                  : (p == 0 ? 0 : p == 1 ? 0 : p == 2 ? 1 : p == 3 ? 0 : p == 4 ? 1 :
                     p == 5 ? -1 : p == 6 ? 0 : p == 7 ? 1 : p == 8 ? -1 : p == 9 ? 1 :
                     p == 10 ? -1 : p == 11 ? 1 : -1);
}
template <int D> MLBM_HD constexpr int cvec(int i, int a) {
    return (a >= D || i == 0) ? 0
         : ((i & 1) ? (D == 2 ? rep2((i - 1) >> 1, a) : rep3((i - 1) >> 1, a))
                    : -(D == 2 ? rep2((i - 1) >> 1, a) : rep3((i - 1) >> 1, a)));
}
template <int D> MLBM_HD constexpr int opp(int i) {
    return i == 0 ? 0 : ((i & 1) ? i + 1 : i - 1);
}
template <int D> MLBM_HD constexpr double wdir(int i) {
    return D == 2
        ? (i == 0 ? 4.0 / 9.0 : (cvec<2>(i, 0) != 0 && cvec<2>(i, 1) != 0) ? 1.0 / 36.0 : 1.0 / 9.0)
        : ((cvec<3>(i, 0) != 0 ? 1.0 / 6.0 : 2.0 / 3.0) *
           (cvec<3>(i, 1) != 0 ? 1.0 / 6.0 : 2.0 / 3.0) *
           (cvec<3>(i, 2) != 0 ? 1.0 / 6.0 : 2.0 / 3.0));
}
// third-order index triples
template <int D> MLBM_HD constexpr int h3t(int t, int j) {
    // 2D: xxy xyy ; 3D: xxy xyy xxz xzz yzz yyz xyz
    return D == 2 ? (t == 0 ? (j < 2 ? 0 : 1) : (j < 1 ? 0 : 1))
        : (t == 0 ? (j < 2 ? 0 : 1) : t == 1 ? (j < 1 ? 0 : 1) : t == 2 ? (j < 2 ? 0 : 2) :
           t == 3 ? (j < 1 ? 0 : 2) : t == 4 ? (j < 1 ? 1 : 2) : t == 5 ? (j < 2 ? 1 : 2) : j);
}
template <int D> MLBM_HD constexpr double h2v(int i, int a, int b) {
    return (double)(cvec<D>(i, a) * cvec<D>(i, b)) - (a == b ? CS2 : 0.0);
}
template <int D> MLBM_HD constexpr double h3v(int i, int t) {
    // c_a c_b c_g - cs2 (c_a d_bg + c_b d_ag + c_g d_ab)
    return (double)(cvec<D>(i, h3t<D>(t, 0)) * cvec<D>(i, h3t<D>(t, 1)) * cvec<D>(i, h3t<D>(t, 2)))
         - CS2 * ((h3t<D>(t, 1) == h3t<D>(t, 2) ? cvec<D>(i, h3t<D>(t, 0)) : 0) +
                  (h3t<D>(t, 0) == h3t<D>(t, 2) ? cvec<D>(i, h3t<D>(t, 1)) : 0) +
                  (h3t<D>(t, 0) == h3t<D>(t, 1) ? cvec<D>(i, h3t<D>(t, 2)) : 0));
}

// neighbour-tile offset index (ox+1) + 3 (oy+1) + 9 (oz+1)
template <int D> MLBM_HD constexpr int nb_index(int ox, int oy, int oz) {
    return (ox + 1) + 3 * (oy + 1) + (D == 3 ? 9 * (oz + 1) : 0);
}
template <int D> MLBM_HD int local_of(int lx, int ly, int lz) {
    return lx + 4 * ly + (D == 3 ? 16 * lz : 0);
}

template <typename R> struct FieldsT {
    R* p;
    int64_t s;
    MLBM_HD R& at(int k, int64_t c) const { return p[k * s + c]; }
};
template <typename R> MLBM_HD FieldsT<R> fields_of(mlbm_fields_t f) {
    return FieldsT<R>{(R*)f.ptr, f.stride};
}

__device__ __forceinline__ void report_error(mlbm_error_t* err, int code, int level,
                                             int x, int y, int z, int detail = 0) {
    if (!err) return;
    int prev = atomicCAS(&err->code, 0, code);
    if (prev == 0 || prev == code) {
        int k = atomicAdd(&err->count, 1);
        if (prev == 0 && k == 0) { err->level = level; err->detail = detail; }
        if (k < 5) { err->cells[k][0] = x; err->cells[k][1] = y; err->cells[k][2] = z; }
    }
}

// live tiles of a level: the device count when present, else n_tiles
__device__ __forceinline__ int live_tiles(const mlbm_level_t& lv) {
    return lv.counts ? __ldg(lv.counts) : lv.n_tiles;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// returns the number of kernels launched (>= 0) or -cudaError
inline int launch_status(int launched = 1) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? launched : -(int)e;
}

}  // namespace mlbm
