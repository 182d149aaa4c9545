// One-launch block-maintenance pass (reference adapt.py:54-230, 374-389).
//
// All bitmap passes of GridAdaptor.update that do not depend on the rebuild
// run in ONE cooperative kernel separated by grid barriers:
//
//   A  seeds <- static mask; invariants of the current topology (coverage,
//      two-tile rings); cur[0] = leaf(kind[0])
//   B  seeds |= particle tiles (domain check); particles in level-0 leaves
//   C  des[0] = align_up(seeds); cur[1] = leaf(kind[1]) | parents(cur[0])
//   D/E per level l >= 1: par = parents(des[l-1]); des[l] = align_up(dilate2(par))
//      (top level: all ones); cur[l+1]
//   F  eff[0] = hysteresis(des[0], cur[0])          (int16 streaks)
//   G/H per level l >= 1: par = parents(eff[l-1]);
//      eff[l] = hysteresis(des[l], cur[l], guard = dilate2(par), par)
//   I  own[l] = eff[l] & ~parents(eff[l-1])
//   J  storage = dilate2(own); new kind = own ? leaf : storage ? border : 0;
//      changed[l] |= new kind != kind
//
// Integer-only, bit-exact with the reference bitmap algorithm.  The grid
// barrier needs co-resident blocks: the kernel is launched cooperatively
// with at most the occupancy-limited number of blocks.
#include <algorithm>
#include <cstdlib>
#include <cooperative_groups.h>
#include "common.cuh"

#ifndef MLBM_NO_CG_GRID_SYNC
#define MLBM_CG_GRID_SYNC 1
#endif

namespace mlbm {

struct AdaptArgs {
    int32_t dim, levels;
    int32_t tdims[MLBM_MAX_LEVELS][3];
    int32_t periodic[3];
    const uint8_t* kind[MLBM_MAX_LEVELS];
    uint8_t* des[MLBM_MAX_LEVELS];
    uint8_t* cur[MLBM_MAX_LEVELS];
    uint8_t* eff[MLBM_MAX_LEVELS];
    uint8_t* par[MLBM_MAX_LEVELS];
    uint8_t* own[MLBM_MAX_LEVELS];
    uint8_t* nkind[MLBM_MAX_LEVELS];
    uint8_t* stor[MLBM_MAX_LEVELS];
    int16_t* streak[MLBM_MAX_LEVELS];
    uint8_t* seeds;
    const uint8_t* static_tiles;
    const double* x;
    int64_t xs;
    int32_t n;
    int32_t* status;        // [levels] changed, [levels..+2] violations
    mlbm_error_t* err;
    unsigned int* bar;      // 2 words, zero-initialised once
    unsigned long long* ts; // optional stage timestamps (block 0), may be null
    int32_t* ext_count;     // particles outside level-0 leaves counted by G2P with the seeds (or null)
    int32_t* win;           // [2][levels][6] tile windows (lo xyz, hi xyz; see k_adapt_pass) or null
};

__device__ __forceinline__ int64_t gi3(const int* d, int x, int y, int z) {
    return ((int64_t)x * d[1] + y) * d[2] + z;
}
// tile grids hold < 2^31 tiles (mlbm_adapt_pass refuses larger): 32-bit division only
__device__ __forceinline__ void dec3(const int* d, int64_t g, int& x, int& y, int& z) {
    const unsigned gg = (unsigned)g, d1 = (unsigned)d[1], d2 = (unsigned)d[2];
    const unsigned q = gg / d2;
    z = (int)(gg - q * d2);
    const unsigned r = q / d1;
    y = (int)(q - r * d1);
    x = (int)r;
}

// Tile window of one level in a pass: every bitmap of the level is zero
// outside it (the arrays start zeroed and no pass writes outside its window;
// windows never shrink).  n = number of tiles in it.
struct Win {
    int lo[3], ext[3];
    int64_t n;
};
__device__ __forceinline__ int64_t win_tile(const Win& w, const int* d, int64_t i, int (&c)[3]) {
    dec3(w.ext, i, c[0], c[1], c[2]);
    c[0] += w.lo[0]; c[1] += w.lo[1]; c[2] += w.lo[2];
    return gi3(d, c[0], c[1], c[2]);
}

__device__ void grid_barrier(unsigned int* bar) {
#ifdef MLBM_CG_GRID_SYNC
    (void)bar;
    cooperative_groups::this_grid().sync();
    return;
#endif
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* vgen = bar + 1;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(&bar[1], 1u);
        } else {
            while (*vgen == g) { }
        }
        __threadfence();
    }
    __syncthreads();
}

// wrapped / clipped coordinates of the window c-r..c+r along one axis (-1 = outside)
__device__ __forceinline__ void axis_window(int c, int r, int n, int per, int (&o)[5]) {
    for (int k = 0; k < 2 * r + 1; ++k) {
        int v = c - r + k;
        if (per) { v = v < 0 ? v + n : (v >= n ? v - n : v); }
        else if (v < 0 || v >= n) v = -1;
        o[k] = v;
    }
}

// any of src over the Chebyshev window [c - r, c + r] (wrap / clip per axis)
__device__ bool window_any(const uint8_t* src, const int* d, int dim, const int* per, const int (&c)[3],
                           int r) {
    int wx[5], wy[5], wz[5] = {c[2], -1, -1, -1, -1};
    axis_window(c[0], r, d[0], per[0], wx);
    axis_window(c[1], r, d[1], per[1], wy);
    const int nz = dim == 3 ? 2 * r + 1 : 1;
    if (dim == 3) axis_window(c[2], r, d[2], per[2], wz);
    for (int iz = 0; iz < nz; ++iz) {
        if (wz[iz] < 0) continue;
        for (int iy = 0; iy < 2 * r + 1; ++iy) {
            if (wy[iy] < 0) continue;
            for (int ix = 0; ix < 2 * r + 1; ++ix)
                if (wx[ix] >= 0 && src[gi3(d, wx[ix], wy[iy], wz[iz])]) return true;
        }
    }
    return false;
}

// align_up(dilate_r(src)) at tile c: any over the parent-group window
__device__ bool group_window_any(const uint8_t* src, const int* d, int dim, const int* per,
                                 const int (&c)[3], int r) {
    int g0[3] = {c[0] & ~1, c[1] & ~1, dim == 3 ? (c[2] & ~1) : c[2]};
    const int lz = dim == 3 ? -r : 0, hz = dim == 3 ? r + 1 : 0;
    for (int dz = lz; dz <= hz; ++dz) {
        int z = g0[2] + dz;
        if (dim == 3) {
            if (per[2]) z = (z % d[2] + d[2]) % d[2];
            else if (z < 0 || z >= d[2]) continue;
        }
        for (int dy = -r; dy <= r + 1; ++dy) {
            int y = g0[1] + dy;
            if (per[1]) y = (y % d[1] + d[1]) % d[1];
            else if (y < 0 || y >= d[1]) continue;
            for (int dx = -r; dx <= r + 1; ++dx) {
                int x = g0[0] + dx;
                if (per[0]) x = (x % d[0] + d[0]) % d[0];
                else if (x < 0 || x >= d[0]) continue;
                if (src[gi3(d, x, y, z)]) return true;
            }
        }
    }
    return false;
}

// any over the 2^dim children of parent tile c (child grid dims dc)
__device__ bool children_any(const uint8_t* src, const int* dc, int dim, const int (&c)[3]) {
    for (int k = 0; k < (1 << dim); ++k) {
        const int x = 2 * c[0] + (k & 1), y = 2 * c[1] + ((k >> 1) & 1),
                  z = dim == 3 ? 2 * c[2] + ((k >> 2) & 1) : c[2];
        if (src[gi3(dc, x, y, z)]) return true;
    }
    return false;
}

// Hysteresis of one level (adapt.py:140-181): one thread per tile; the 2^dim
// tiles of a sibling group sit in consecutive lanes, so "all siblings may
// coarsen" is a 2^dim-lane AND over shuffles.
__device__ void effective_stage(const AdaptArgs& A, int l, bool with_guard, int64_t tid, int64_t nth,
                                const Win& W) {
    const int* d = A.tdims[l];
    const int dim = A.dim;
    bool grouped = true;
    for (int a = 0; a < dim; ++a) grouped &= (d[a] % 2) == 0;
    // sibling groups of the window (its bounds are group-aligned when grouped)
    int gd[3] = {W.ext[0], W.ext[1], W.ext[2]}, g0[3] = {W.lo[0], W.lo[1], W.lo[2]};
    if (grouped)
        for (int a = 0; a < dim; ++a) { gd[a] = W.ext[a] / 2; g0[a] = W.lo[a] / 2; }
    const int K = grouped ? (1 << dim) : 1;
    const int64_t total = (int64_t)gd[0] * gd[1] * gd[2] * K;
    const uint8_t* par = A.par[l];
    const int lane = threadIdx.x & 31;
    for (int64_t base = tid - lane; base < total; base += nth) {      // warp-uniform trip count
        const int64_t t = base + lane;
        const bool valid = t < total;
        int64_t g = 0;
        bool cand = false, avail = false;
        int c[3] = {0, 0, 0};
        if (valid) {
            const int64_t j = t >> (K == 8 ? 3 : K == 4 ? 2 : 0);
            const int k = (int)(t - j * K);
            int x[3];
            dec3(gd, j, x[0], x[1], x[2]);
            for (int a = 0; a < 3; ++a)
                c[a] = (grouped && a < dim) ? 2 * (g0[a] + x[a]) + ((k >> a) & 1) : g0[a] + x[a];
            g = gi3(d, c[0], c[1], c[2]);
            cand = A.cur[l][g] && !A.des[l][g];
            const int16_t sv = cand ? (int16_t)(A.streak[l][g] + 1) : (int16_t)0;
            A.streak[l][g] = sv;
            bool guard = false;
            if (with_guard && cand && sv >= 2) guard = window_any(par, d, dim, A.periodic, c, 2);
            avail = cand && sv >= 2 && !guard;
        }
        bool all = avail;
        for (int off = 1; off < K; off <<= 1) all &= __shfl_xor_sync(0xffffffffu, all, off) != 0;
        if (valid) {
            const bool act = grouped ? all : false;
            const bool pp = with_guard ? par[g] != 0 : false;
            A.eff[l][g] = (A.des[l][g] || (A.cur[l][g] && !act) || pp) ? 1 : 0;
        }
    }
}

// OR of src over the radius-2 window along one axis (wrap / clip)
__device__ __forceinline__ bool axis_or2(const uint8_t* src, const int* d, const int* per, const int (&c)[3],
                                         int axis) {
    const int n = d[axis];
    bool any = false;
#pragma unroll
    for (int k = -2; k <= 2; ++k) {
        int v = c[axis] + k;
        if (per[axis]) { v %= n; if (v < 0) v += n; }
        else if (v < 0 || v >= n) continue;
        int q[3] = {c[0], c[1], c[2]};
        q[axis] = v;
        any |= src[gi3(d, q[0], q[1], q[2])] != 0;
    }
    return any;
}

// OR of src over the sibling-group window [g0 - 2, g0 + 3] (g0 = c & ~1)
// along one axis (wrap / clip): one factor of group_window_any(r = 2)
__device__ __forceinline__ bool axis_group_or2(const uint8_t* src, const int* d, const int* per,
                                               const int (&c)[3], int axis) {
    const int n = d[axis], g0 = c[axis] & ~1;
    bool any = false;
#pragma unroll
    for (int k = -2; k <= 3; ++k) {
        int v = g0 + k;
        if (per[axis]) { v %= n; if (v < 0) v += n; }
        else if (v < 0 || v >= n) continue;
        int q[3] = {c[0], c[1], c[2]};
        q[axis] = v;
        any |= src[gi3(d, q[0], q[1], q[2])] != 0;
    }
    return any;
}

// Branchless, fully unrolled radius-2 windows: out-of-domain taps are
// redirected to the centre tile and masked, so all 25 / 125 accesses issue
// back to back (memory-level parallelism instead of a serial loop).
__device__ __forceinline__ void window_axes(const int* d, const int* per, const int (&c)[3], int dim,
                                            int (&w)[3][5], unsigned (&ok)[3]) {
    for (int a = 0; a < 3; ++a) {
        ok[a] = 0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            int v = c[a] + k - 2;
            bool in = true;
            if (a < dim) {
                if (per[a]) v = v < 0 ? v + d[a] : (v >= d[a] ? v - d[a] : v);
                else if (v < 0 || v >= d[a]) { in = false; v = c[a]; }
            } else {
                v = c[a];
                in = k == 2;
            }
            w[a][k] = v;
            if (in) ok[a] |= 1u << k;
        }
    }
}

// number of absent (kind == 0) tiles in the radius-2 window
template <bool UNUSED>
__device__ __forceinline__ int window_count(const uint8_t* kind, const int* d, int dim, const int* per,
                                            const int (&c)[3]) {
    int w[3][5];
    unsigned ok[3];
    window_axes(d, per, c, dim, w, ok);
    int miss = 0;
#pragma unroll
    for (int iz = 0; iz < 5; ++iz)
#pragma unroll
        for (int iy = 0; iy < 5; ++iy)
#pragma unroll
            for (int ix = 0; ix < 5; ++ix) {
                const bool in = ((ok[2] >> iz) & (ok[1] >> iy) & (ok[0] >> ix)) & 1u;
                const uint8_t k = kind[gi3(d, w[0][ix], w[1][iy], w[2][iz])];
                miss += (in && k == 0) ? 1 : 0;
            }
    return miss;
}

__device__ __forceinline__ bool window_any2(const uint8_t* src, const int* d, int dim, const int* per,
                                            const int (&c)[3]) {
    int w[3][5];
    unsigned ok[3];
    window_axes(d, per, c, dim, w, ok);
    int any = 0;
#pragma unroll
    for (int iz = 0; iz < 5; ++iz)
#pragma unroll
        for (int iy = 0; iy < 5; ++iy)
#pragma unroll
            for (int ix = 0; ix < 5; ++ix) {
                const bool in = ((ok[2] >> iz) & (ok[1] >> iy) & (ok[0] >> ix)) & 1u;
                any |= (in && src[gi3(d, w[0][ix], w[1][iy], w[2][iz])]) ? 1 : 0;
            }
    return any != 0;
}

__device__ __forceinline__ void window_mark(uint8_t* dst, const int* d, int dim, const int* per,
                                            const int (&c)[3]) {
    int w[3][5];
    unsigned ok[3];
    window_axes(d, per, c, dim, w, ok);
#pragma unroll
    for (int iz = 0; iz < 5; ++iz)
#pragma unroll
        for (int iy = 0; iy < 5; ++iy)
#pragma unroll
            for (int ix = 0; ix < 5; ++ix) {
                const bool in = ((ok[2] >> iz) & (ok[1] >> iy) & (ok[0] >> ix)) & 1u;
                if (in) dst[gi3(d, w[0][ix], w[1][iy], w[2][iz])] = 1;
            }
}

// Warp-cooperative window pass: the warp scans 32 tiles per iteration, and
// for every selected tile (ballot) its (2r+1)^dim window is split over the
// lanes.  op(l, window_tile_index) is called once per in-domain window tile.
template <typename Sel, typename Op>
__device__ __forceinline__ void warp_window_pass(const int* d, int dim, const int* per, int64_t n, int r,
                                                 Sel sel, Op op) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int w = 2 * r + 1, nwin = dim == 3 ? w * w * w : w * w;
    for (int64_t base = wid * 32; base < n; base += nw * 32) {
        const int64_t g = base + lane;
        unsigned m = __ballot_sync(0xffffffffu, g < n && sel(g));
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const int64_t t = base + src;
            int c[3];
            dec3(d, t, c[0], c[1], c[2]);
            for (int k = lane; k < nwin; k += 32) {
                int o[3] = {k % w - r, (k / w) % w - r, dim == 3 ? k / (w * w) - r : 0};
                int q[3];
                bool in = true;
                for (int a = 0; a < 3; ++a) {
                    int v = c[a] + o[a];
                    if (a < dim) {
                        if (per[a]) v = v < 0 ? v + d[a] : (v >= d[a] ? v - d[a] : v);
                        else if (v < 0 || v >= d[a]) in = false;
                    }
                    q[a] = v;
                }
                if (in) op(gi3(d, q[0], q[1], q[2]));
            }
        }
    }
}

__device__ __forceinline__ void stamp(const AdaptArgs& A, int k) {
    if (A.ts && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        A.ts[k] = t;
    }
}
#define STAMP_BARRIER(k) do { grid_barrier(A.bar); stamp(A, k); } while (0)

#ifndef WIN_MARGIN
#define WIN_MARGIN 8      // tiles added around the inputs of a level's window
#endif
#ifndef ADAPT_MINB
#define ADAPT_MINB 2      // 64 registers, 2 x 512 threads per SM (explicit 1 lets ptxas take 69)
#endif
__global__ void __launch_bounds__(512, ADAPT_MINB) k_adapt_pass(AdaptArgs A) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const int dim = A.dim, L = A.levels;
    const int* d0 = A.tdims[0];
    const int64_t n0 = (int64_t)d0[0] * d0[1] * d0[2];
    // tile windows of this pass (every block derives the same ones): the last
    // pass's window, the bounding box of the kinds it produced widened by
    // WIN_MARGIN tiles, and the parent footprint of the finer level's window
    // widened the same way — wider than any chain of stages reaches from a
    // non-zero input (seeds within 1 tile of a leaf, group alignment 1,
    // dilations 2 + 2 + 3).  The top level, periodic axes and win = null
    // span the whole grid.
    __shared__ Win W[MLBM_MAX_LEVELS];
    if (threadIdx.x == 0) {
        for (int l = 0; l < L; ++l) {
            const int* d = A.tdims[l];
            bool grouped = true;
            for (int a = 0; a < dim; ++a) grouped &= (d[a] % 2) == 0;
            int lo[3], hi[3];
            for (int a = 0; a < 3; ++a) {
                lo[a] = 0; hi[a] = d[a] - 1;
                if (a >= dim || !A.win || l == L - 1 || A.periodic[a]) continue;
                const int* cw = A.win + l * 6;
                const int* nx = A.win + (L + l) * 6;
                int wl = cw[a], wh = cw[3 + a];                   // empty: wl > wh
                if (nx[a] <= nx[3 + a]) { wl = min(wl, nx[a] - WIN_MARGIN); wh = max(wh, nx[3 + a] + WIN_MARGIN); }
                if (l > 0 && W[l - 1].n > 0) {
                    wl = min(wl, (W[l - 1].lo[a] >> 1) - WIN_MARGIN);
                    wh = max(wh, ((W[l - 1].lo[a] + W[l - 1].ext[a] - 1) >> 1) + WIN_MARGIN);
                }
                if (grouped) { wl &= ~1; wh |= 1; }
                lo[a] = max(wl, 0);
                hi[a] = min(wh, d[a] - 1);
            }
            int64_t n = 1;
            for (int a = 0; a < 3; ++a) {
                W[l].lo[a] = lo[a];
                W[l].ext[a] = hi[a] >= lo[a] ? hi[a] - lo[a] + 1 : 0;
                n *= W[l].ext[a];
            }
            W[l].n = n;
        }
    }
    __syncthreads();
    stamp(A, 0);

    // ---- A: seeds <- static, invariants of the current topology, cur[0]
    if (dim == 3 && (d0[2] & 15) == 0 && L <= 5) {
        // 16 consecutive z tiles of one (x, y) row per trip: level-0 kinds and
        // cur[0] as 16-byte vectors, level l's 16 >> l covering kinds as bytes
        int viol = 0;
        for (int64_t q = tid; q < (n0 >> 4); q += nth) {
            const int64_t g = q << 4;
            int x[3];
            dec3(d0, g, x[0], x[1], x[2]);
            const uint4 k0 = *reinterpret_cast<const uint4*>(A.kind[0] + g);
            const unsigned kw[4] = {k0.x, k0.y, k0.z, k0.w};
            unsigned cw[4], nw[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                cw[i] = __vcmpeq4(kw[i], 0x01010101u) & 0x01010101u;     // leaf bytes -> 1
                nw[i] = cw[i];                                          // per-tile leaf count
            }
            *reinterpret_cast<uint4*>(A.cur[0] + g) = make_uint4(cw[0], cw[1], cw[2], cw[3]);
            for (int l = 1; l < L; ++l) {
                const uint8_t* kl = A.kind[l] + gi3(A.tdims[l], x[0] >> l, x[1] >> l, x[2] >> l);
#pragma unroll
                for (int z = 0; z < 16; ++z)
                    if (kl[z >> l] == 1) nw[z >> 2] += 1u << (8 * (z & 3));
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) viol += __popc(__vcmpne4(nw[i], 0x01010101u)) >> 3;
        }
        if (viol) atomicAdd(&A.status[L], viol);
    } else {
        for (int64_t g = tid; g < n0; g += nth) {
            A.cur[0][g] = A.kind[0][g] == 1;
            int x[3];
            dec3(d0, g, x[0], x[1], x[2]);
            int cnt = 0;
            for (int l = 0; l < L; ++l) {
                int c[3];
                for (int a = 0; a < 3; ++a) c[a] = a < dim ? x[a] >> l : 0;
                cnt += A.kind[l][gi3(A.tdims[l], c[0], c[1], c[2])] == 1;
            }
            if (cnt != 1) atomicAdd(&A.status[L], 1);
        }
    }
    // two-tile rings of the current leaves (sparse_grid.py:320-337): the
    // absent tiles inside dilate2(leaf) are counted; the dilation is done as
    // three separable radius-2 ORs spread over phases A (x -> stor), C
    // (y -> nkind) and F (z + count), in buffers that are free until I/J
    for (int l = 0; l < L; ++l) {
        const int* d = A.tdims[l];
        const uint8_t* kind = A.kind[l];
        const int nx = d[0], per0 = A.periodic[0];
        for (int64_t i = tid; i < W[l].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[l], d, i, c);
            bool any = false;
#pragma unroll
            for (int k = -2; k <= 2; ++k) {
                int v = c[0] + k;
                if (per0) { v %= nx; if (v < 0) v += nx; }
                else if (v < 0 || v >= nx) continue;
                any |= kind[gi3(d, v, c[1], c[2])] == 1;
            }
            A.stor[l][g] = any;
        }
    }
    // ---- B (same stage): particle seeds (seeds are all-zero on entry, they are
    //      cleared at the end of every pass) + particles in level-0 leaves
    constexpr int PU = 4;                       // particles per thread per trip (loads first)
    for (int64_t p0 = tid; p0 < A.n; p0 += PU * nth) {
        double v[PU][3];
#pragma unroll
        for (int u = 0; u < PU; ++u) {
            const int64_t p = p0 + u * nth;
#pragma unroll
            for (int a = 0; a < 3; ++a) v[u][a] = (p < A.n && a < dim) ? __ldg(&A.x[a * A.xs + p]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < PU; ++u) {
            const int64_t p = p0 + u * nth;
            if (p >= A.n) break;
            int t[3] = {0, 0, 0};
            bool bad = false;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (a >= dim) break;
                const int64_t c = (int64_t)floor(v[u][a]);
                const int64_t tt = c >= 0 ? c / 4 : -((-c + 3) / 4);
                if (tt < 0 || tt >= d0[a] || !(v[u][a] == v[u][a])) bad = true;
                t[a] = (int)tt;
            }
            if (bad) {
                report_error(A.err, MLBM_ERR_DOMAIN, 0, t[0], t[1], t[2]);
                atomicAdd(&A.status[L + 2], 1);
                continue;
            }
            const int64_t g = gi3(d0, t[0], t[1], t[2]);
            A.seeds[g] = 1;
            if (A.kind[0][g] != 1) atomicAdd(&A.status[L + 2], 1);
        }
    }
    if (A.ext_count && tid == 0) {
        // the seeds came from G2P: its leaf-invariant count joins status[L+2]
        atomicAdd(&A.status[L + 2], *A.ext_count);
        *A.ext_count = 0;
    }
    STAMP_BARRIER(2);
    if (A.win && blockIdx.x == 0 && threadIdx.x == 0) {
        // this pass's windows; the kinds' bounding boxes are collected anew in J
        for (int l = 0; l < L; ++l)
            for (int a = 0; a < 3; ++a) {
                A.win[l * 6 + a] = W[l].lo[a];
                A.win[l * 6 + 3 + a] = W[l].lo[a] + W[l].ext[a] - 1;
                A.win[(L + l) * 6 + a] = 0x7fffffff;
                A.win[(L + l) * 6 + 3 + a] = -0x7fffffff;
            }
    }

    // ---- C: des[0], cur[1]
    if (L == 1) {
        for (int64_t g = tid; g < n0; g += nth) A.des[0][g] = 1;
    } else {
        for (int64_t i = tid; i < W[0].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[0], d0, i, c);
            int g0[3] = {c[0] & ~1, c[1] & ~1, dim == 3 ? (c[2] & ~1) : c[2]};
            bool any = false;
            for (int k = 0; k < (1 << dim) && !any; ++k) {
                const int x = g0[0] + (k & 1), y = g0[1] + ((k >> 1) & 1),
                          z = dim == 3 ? g0[2] + ((k >> 2) & 1) : g0[2];
                const int64_t gg = gi3(d0, x, y, z);
                any = A.seeds[gg] != 0 || (A.static_tiles && A.static_tiles[gg]);
            }
            A.des[0][g] = any;
        }
        const int* d1 = A.tdims[1];
        for (int64_t i = tid; i < W[1].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[1], d1, i, c);
            A.cur[1][g] = (A.kind[1][g] == 1) || children_any(A.cur[0], d0, dim, c);
        }
    }
    {
        int miss = 0;
        for (int l = 0; l < L; ++l) {
            const int* d = A.tdims[l];
            for (int64_t i = tid; i < W[l].n; i += nth) {
                int c[3];
                const int64_t g = win_tile(W[l], d, i, c);
                const bool any = axis_or2(A.stor[l], d, A.periodic, c, 1);
                if (dim == 3) A.nkind[l][g] = any;
                else miss += any && A.kind[l][g] == 0;
            }
        }
        for (int off = 16; off > 0; off >>= 1) miss += __shfl_down_sync(0xffffffffu, miss, off);
        if ((threadIdx.x & 31) == 0 && miss) atomicAdd(&A.status[L + 1], miss);
    }
    STAMP_BARRIER(3);

    // ---- D/E: desired coverage of coarser levels (the top level is all ones
    //      and needs neither its parents bitmap nor a barrier)
    for (int l = 1; l < L; ++l) {
        const int* d = A.tdims[l];
        if (l == L - 1) {
            const int64_t n = (int64_t)d[0] * d[1] * d[2];
            for (int64_t g = tid; g < n; g += nth) A.des[l][g] = 1;
            break;
        }
        for (int64_t i = tid; i < W[l].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[l], d, i, c);
            A.par[l][g] = children_any(A.des[l - 1], A.tdims[l - 1], dim, c);
        }
        if (l + 1 < L) {
            const int* dn = A.tdims[l + 1];
            for (int64_t i = tid; i < W[l + 1].n; i += nth) {
                int c[3];
                const int64_t g = win_tile(W[l + 1], dn, i, c);
                A.cur[l + 1][g] = (A.kind[l + 1][g] == 1) || children_any(A.cur[l], d, dim, c);
            }
        }
        STAMP_BARRIER(4);
        // des[l] = align_up(dilate2(par)): the group window [g0 - 2, g0 + 3]
        // (g0 = c & ~1) per axis, as separable ORs x -> own, y -> stor,
        // z -> des (own and stor are free here: stor's ring data was consumed
        // in C, own is written in I)
        for (int64_t i = tid; i < W[l].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[l], d, i, c);
            A.own[l][g] = axis_group_or2(A.par[l], d, A.periodic, c, 0);
        }
        grid_barrier(A.bar);
        for (int64_t i = tid; i < W[l].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[l], d, i, c);
            const bool any = axis_group_or2(A.own[l], d, A.periodic, c, 1);
            if (dim == 3) A.stor[l][g] = any;
            else A.des[l][g] = any;
        }
        if (dim == 3) {
            grid_barrier(A.bar);
            for (int64_t i = tid; i < W[l].n; i += nth) {
                int c[3];
                const int64_t g = win_tile(W[l], d, i, c);
                A.des[l][g] = axis_group_or2(A.stor[l], d, A.periodic, c, 2);
            }
        }
        STAMP_BARRIER(5);
    }

    // ---- F/G/H: hysteresis per level (+ the z pass of the ring check)
    if (dim == 3) {
        int miss = 0;
        for (int l = 0; l < L; ++l) {
            const int* d = A.tdims[l];
            for (int64_t i = tid; i < W[l].n; i += nth) {
                int c[3];
                const int64_t g = win_tile(W[l], d, i, c);
                if (A.kind[l][g] != 0) continue;
                miss += axis_or2(A.nkind[l], d, A.periodic, c, 2);
            }
        }
        for (int off = 16; off > 0; off >>= 1) miss += __shfl_down_sync(0xffffffffu, miss, off);
        if ((threadIdx.x & 31) == 0 && miss) atomicAdd(&A.status[L + 1], miss);
    }
    effective_stage(A, 0, false, tid, nth, W[0]);
    STAMP_BARRIER(6);
    for (int l = 1; l < L; ++l) {
        const int* d = A.tdims[l];
        for (int64_t i = tid; i < W[l].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[l], d, i, c);
            A.par[l][g] = children_any(A.eff[l - 1], A.tdims[l - 1], dim, c);
        }
        STAMP_BARRIER(7);
        // the top level's hysteresis is a no-op (des = 1: no candidate, its
        // streaks stay 0) and its effective coverage is all ones
        // (adapt.py:180-181): skipped, phase I reads eff[L-1] as 1
        if (l < L - 1) {
            effective_stage(A, l, true, tid, nth, W[l]);
            STAMP_BARRIER(8);
        }
    }
    // par[l] now holds parents(eff[l-1]) for every l >= 1

    // ---- I/J: own = eff & ~parents(eff[l-1]); storage = dilate2(own) as three
    //      separable radius-2 ORs (x into stor, y into des, z on the fly);
    //      new kinds, no-op flags (adapt.py:184-225); seeds cleared
    for (int l = 0; l < L; ++l) {
        const int* d = A.tdims[l];
        const int per0 = A.periodic[0], nx = d[0];
        for (int64_t i = tid; i < W[l].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[l], d, i, c);
            A.own[l][g] = (l == L - 1 || A.eff[l][g]) && !(l > 0 && A.par[l][g]);
            bool any = false;
#pragma unroll
            for (int k = -2; k <= 2; ++k) {
                int v = c[0] + k;
                if (per0) { v %= nx; if (v < 0) v += nx; }
                else if (v < 0 || v >= nx) continue;
                const int64_t q = gi3(d, v, c[1], c[2]);
                any |= (l == L - 1 || A.eff[l][q]) && !(l > 0 && A.par[l][q]);
            }
            A.stor[l][g] = any;
        }
    }
    {
        // all seeds cleared (not only the window's: a seed of a particle far
        // from every leaf must not survive into a later window), 16 B per store
        uint4* s16 = reinterpret_cast<uint4*>(A.seeds);      // torch allocations: 512 B aligned
        const int64_t n16 = n0 >> 4;
        for (int64_t g = tid; g < n16; g += nth) s16[g] = make_uint4(0u, 0u, 0u, 0u);
        for (int64_t g = (n16 << 4) + tid; g < n0; g += nth) A.seeds[g] = 0;
    }
    STAMP_BARRIER(10);
    if (dim == 3) {
        for (int l = 0; l < L; ++l) {
            const int* d = A.tdims[l];
            for (int64_t i = tid; i < W[l].n; i += nth) {
                int c[3];
                const int64_t g = win_tile(W[l], d, i, c);
                A.des[l][g] = axis_or2(A.stor[l], d, A.periodic, c, 1);
            }
        }
        grid_barrier(A.bar);
    }
    for (int l = 0; l < L; ++l) {
        const int* d = A.tdims[l];
        bool changed = false;
        int cnt = 0, fresh = 0;
        int blo[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff}, bhi[3] = {-0x7fffffff, -0x7fffffff, -0x7fffffff};
        for (int64_t i = tid; i < W[l].n; i += nth) {
            int c[3];
            const int64_t g = win_tile(W[l], d, i, c);
            uint8_t k;
            if (A.own[l][g]) k = 1;
            else {
                const bool dil = dim == 3 ? axis_or2(A.des[l], d, A.periodic, c, 2)
                                          : axis_or2(A.stor[l], d, A.periodic, c, 1);
                k = dil ? 2 : 0;
            }
            A.nkind[l][g] = k;
            const uint8_t old = A.kind[l][g];
            changed |= k != old;
            cnt += k != 0;
            fresh += (k != 0 && old == 0);
            if (k) {
                for (int a = 0; a < 3; ++a) { blo[a] = min(blo[a], c[a]); bhi[a] = max(bhi[a], c[a]); }
            }
        }
        if (A.win && l < L - 1) {
            // bounding box of the new kinds: the next pass's window input
            for (int a = 0; a < 3; ++a) {
                const int wl = __reduce_min_sync(0xffffffffu, blo[a]);
                const int wh = __reduce_max_sync(0xffffffffu, bhi[a]);
                if ((threadIdx.x & 31) == 0 && wl <= wh) {
                    atomicMin(&A.win[(L + l) * 6 + a], wl);
                    atomicMax(&A.win[(L + l) * 6 + 3 + a], wh);
                }
            }
        }
        if (__syncthreads_or(changed) && threadIdx.x == 0) atomicOr(&A.status[l], 1);
        for (int off = 16; off > 0; off >>= 1) {
            cnt += __shfl_down_sync(0xffffffffu, cnt, off);
            fresh += __shfl_down_sync(0xffffffffu, fresh, off);
        }
        if ((threadIdx.x & 31) == 0) {
            if (cnt) atomicAdd(&A.status[L + 4 + l], cnt);
            if (fresh) atomicAdd(&A.status[2 * L + 4 + l], fresh);
        }
    }
    if (A.ts) STAMP_BARRIER(11);
}

}  // namespace mlbm

using namespace mlbm;

extern "C" unsigned long long* mlbm_adapt_timestamps_ptr();
int mlbm_adapt_bits_launch(const mlbm_hier_t* h, uint8_t* const* nkind, int16_t* const* streak,
                           uint8_t* seeds, const uint8_t* static_tiles, const double* x, int64_t xs,
                           int32_t n, int32_t* status, mlbm_error_t* err, int64_t seeds_bytes,
                           void* stream);

// optional stage timestamps (tools/adapt_bench.py): a caller-owned buffer of
// 64 uint64 set once; the library never allocates
static unsigned long long* g_ts_last = nullptr;
extern "C" unsigned long long* mlbm_adapt_timestamps_ptr() { return g_ts_last; }
extern "C" int mlbm_adapt_set_timestamps(unsigned long long* buf) {
    g_ts_last = buf;
    return 0;
}

extern "C" int mlbm_adapt_pass(const mlbm_hier_t* h, uint8_t* const* des, uint8_t* const* cur,
                               uint8_t* const* eff, uint8_t* const* par, uint8_t* const* own,
                               uint8_t* const* nkind, uint8_t* const* stor, int16_t* const* streak,
                               uint8_t* seeds,
                               const uint8_t* static_tiles, const double* x, int64_t xs, int32_t n,
                               int32_t* ext_count, int32_t* win,
                               int32_t* status, mlbm_error_t* err, unsigned int* bar, void* stream) {
    // MLBM_ADAPT_PATH=bits selects the bit-packed single-CTA pass
    // (adapt_bits.cu) when the hierarchy's bitmaps fit in shared memory.  It
    // is bit-exact but slower on B200 (one SM against 148: 74 us vs 52 us on
    // C2), so the cooperative byte pass is the default.
    const char* path = getenv("MLBM_ADAPT_PATH");
    if (path && path[0] == 'b' && !ext_count) {
        int64_t n0 = 1;
        for (int a = 0; a < h->dim; ++a) n0 *= h->finest[a] / 4;
        const int r = mlbm_adapt_bits_launch(h, nkind, streak, seeds, static_tiles, x, xs, n, status, err,
                                             n0, stream);
        if (r != 0) return r;
    }
    AdaptArgs A;
    A.dim = h->dim;
    A.levels = h->levels;
    for (int l = 0; l < h->levels; ++l) {
        for (int a = 0; a < 3; ++a) A.tdims[l][a] = a < h->dim ? (h->finest[a] >> l) / 4 : 1;
        A.kind[l] = h->kind[l];
        A.des[l] = des[l];
        A.cur[l] = cur[l];
        A.eff[l] = eff[l];
        A.par[l] = par[l];
        A.own[l] = own[l];
        A.nkind[l] = nkind[l];
        A.stor[l] = stor[l];
        A.streak[l] = streak[l];
    }
    for (int a = 0; a < 3; ++a) A.periodic[a] = h->periodic[a];
    A.seeds = seeds;
    A.static_tiles = static_tiles;
    A.x = x;
    A.xs = xs;
    A.n = n;
    A.ext_count = ext_count;
    A.win = ext_count ? win : nullptr;       // windows need G2P's seeds (within a tile of a leaf)
    A.status = status;
    A.err = err;
    A.bar = bar;
    A.ts = g_ts_last;
    static int grid_sms = 0, grid_per = 1;
    int grid = 0;
    if (grid_sms == 0) {
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_adapt_pass, 512, 0);
        grid_sms = sms;
        grid_per = std::max(per, 1);
    }
    // small tile grids (C2: 32K level-0 tiles) are barrier-latency bound: one
    // CTA per SM; large ones (C4: 7.1M) need every resident warp for memory
    // parallelism: up to the occupancy limit, ~8 tiles per thread per stage
    int64_t n0 = 1;
    for (int a = 0; a < h->dim; ++a) n0 *= (h->finest[a] / 4);
    if (n0 >= ((int64_t)1 << 31)) return -(int)cudaErrorInvalidValue;   // 32-bit tile indices (dec3)
    const int64_t want = (n0 + (int64_t)grid_sms * 512 * 8 - 1) / ((int64_t)grid_sms * 512 * 8);
    grid = grid_sms * (int)std::max<int64_t>(1, std::min<int64_t>(want, grid_per));
    if (const char* g = getenv("MLBM_ADAPT_GRID")) {          // tuning experiments
        const int v = atoi(g);
        if (v > 0 && v <= grid_sms * grid_per) grid = v;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_adapt_pass, A);
    if (e != cudaSuccess) return -(int)e;
    return launch_status(1);
}
