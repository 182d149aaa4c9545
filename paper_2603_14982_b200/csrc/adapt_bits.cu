// Bit-packed block-maintenance pass (reference adapt.py:54-230, 374-389) for
// tile hierarchies whose bitmaps fit in one CTA's shared memory.
//
// The tile bitmaps of every level are packed 32 tiles per word along the
// fastest memory axis of the kind grids (z in 3D, y in 2D), so every bitmap
// operation of the pass is word-parallel:
//   dilate (Chebyshev radius 2)  funnel shifts along the row + OR of 5 (or 25) rows
//   align_up / parents           pair-OR of bits + row pairs (+ even-bit compaction)
//   sibling-group AND            pair-AND of bits + row pairs
// and the whole pass — invariants of the current topology, desired / current
// coverage, int16 hysteresis streaks, effective coverage, ownership, storage
// and the new kind grids — runs in ONE CTA separated by __syncthreads
// (~16 block barriers instead of grid barriers).  Particle seeds come from a
// multi-CTA pre-kernel that ORs tile bits with one atomic per run of equal
// words in a warp (particles are sorted by tile).  Bit-exact with the byte
// algorithm of adapt.cu (tests/test_gpu_adapt.py runs both).
#include <algorithm>
#include <cstdlib>
#include "common.cuh"

namespace mlbm {
namespace ab {

constexpr int MAXL = MLBM_MAX_LEVELS;
enum { S_LEAF, S_PRES, S_DES, S_CUR, S_EFF, S_PAR, S_OWN, S_T1, S_T2, NSET };
constexpr int THREADS = 1024;
struct T3 { int v[3]; };

// canonical axes: A0 = x (slowest in memory), A1 = y in 3D / unit dummy in 2D,
// R = z in 3D / y in 2D (fastest, the packed row axis)
struct Lvl {
    int n0, n1, nr, W;      // extents, words per row
    int nw, off;            // words of the level, offset inside a set
    uint32_t tail;          // valid bits of a row's last word
};

struct BitArgs {
    int dim, L, nwt;
    int per0, per1, perr;
    int grouped[MAXL];
    Lvl lv[MAXL];
    const uint8_t* kind[MAXL];
    uint8_t* nkind[MAXL];
    int16_t* streak[MAXL];
    uint32_t* seeds;            // level-0 words (row layout); cleared here
    const uint8_t* static_tiles;
    int32_t* status;
    unsigned long long* ts;     // optional phase timestamps (thread 0)
};

__device__ __forceinline__ uint32_t row_mask(const Lvl& g, int w) { return w == g.W - 1 ? g.tail : 0xffffffffu; }

// word index (within the level) of the row offset by (d0, d1), or -1
__device__ __forceinline__ int row_nb(const Lvl& g, int per0, int per1, int i, int d0, int d1) {
    const int row = i / g.W, w = i - row * g.W;
    int a0 = row / g.n1, a1 = row - a0 * g.n1;
    a0 += d0;
    a1 += d1;
    if (per0) { a0 %= g.n0; if (a0 < 0) a0 += g.n0; } else if (a0 < 0 || a0 >= g.n0) return -1;
    if (per1) { a1 %= g.n1; if (a1 < 0) a1 += g.n1; } else if (a1 < 0 || a1 >= g.n1) return -1;
    return (a0 * g.n1 + a1) * g.W + w;
}

// bits of the row shifted so that bit i holds row bit (32 w + i + k), wrap / clip
__device__ __forceinline__ uint32_t rshift(const uint32_t* s, const Lvl& g, int perr, int i, int k) {
    const int row = i / g.W, w = i - row * g.W;
    const uint32_t* rw = s + row * g.W;
    if (g.nr < 32) {
        const uint32_t v = rw[0];
        uint32_t out = 0;
        for (int b = 0; b < g.nr; ++b) {
            int j = b + k;
            if (perr) { j %= g.nr; if (j < 0) j += g.nr; } else if (j < 0 || j >= g.nr) continue;
            out |= ((v >> j) & 1u) << b;
        }
        return out;
    }
    const uint32_t cur = rw[w];
    if (k == 0) return cur;
    if (k > 0) {
        const int wn = w + 1 < g.W ? w + 1 : (perr ? 0 : -1);
        const uint32_t nx = wn >= 0 ? rw[wn] : 0u;
        return (cur >> k) | (nx << (32 - k));
    }
    const int wp = w > 0 ? w - 1 : (perr ? g.W - 1 : -1);
    const uint32_t pv = wp >= 0 ? rw[wp] : 0u;
    return (cur << (-k)) | (pv >> (32 + k));
}

// pair-OR / pair-AND along the row (bits 2j, 2j+1), result on both bits
__device__ __forceinline__ uint32_t pair_or(uint32_t v) { uint32_t m = (v | (v >> 1)) & 0x55555555u; return m | (m << 1); }
__device__ __forceinline__ uint32_t pair_and(uint32_t v) { uint32_t m = (v & (v >> 1)) & 0x55555555u; return m | (m << 1); }
// OR of bit pairs compacted to 16 bits
__device__ __forceinline__ uint32_t compress_or(uint32_t c) {
    uint32_t m = (c | (c >> 1)) & 0x55555555u;
    m = (m | (m >> 1)) & 0x33333333u;
    m = (m | (m >> 2)) & 0x0F0F0F0Fu;
    m = (m | (m >> 4)) & 0x00FF00FFu;
    m = (m | (m >> 8)) & 0x0000FFFFu;
    return m;
}
// each of the low 16 bits doubled
__device__ __forceinline__ uint32_t spread2(uint32_t x) {
    x &= 0xFFFFu;
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x | (x << 1);
}

__device__ __forceinline__ void tstamp(const BitArgs& A, int k) {
    if (A.ts && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        A.ts[k] = t;
    }
}

struct Ctx {
    const BitArgs& A;
    uint32_t* sm;
    __device__ uint32_t* set(int s, int l) const { return sm + s * A.nwt + A.lv[l].off; }
};

// dst = OR over the radius-2 row window (R axis)
__device__ void dil_r(const Ctx& C, int l, int src, int dst) {
    const Lvl& g = C.A.lv[l];
    const uint32_t* s = C.set(src, l);
    uint32_t* d = C.set(dst, l);
    for (int i = threadIdx.x; i < g.nw; i += THREADS) {
        uint32_t v = 0;
#pragma unroll
        for (int k = -2; k <= 2; ++k) v |= rshift(s, g, C.A.perr, i, k);
        d[i] = v & row_mask(g, i % g.W);
    }
}
// dst = OR over the radius-2 window of rows (A0 x A1)
__device__ void dil_a(const Ctx& C, int l, int src, int dst) {
    const Lvl& g = C.A.lv[l];
    const uint32_t* s = C.set(src, l);
    uint32_t* d = C.set(dst, l);
    const int r1 = g.n1 > 1 ? 2 : 0;
    for (int i = threadIdx.x; i < g.nw; i += THREADS) {
        uint32_t v = 0;
        for (int d0 = -2; d0 <= 2; ++d0)
            for (int d1 = -r1; d1 <= r1; ++d1) {
                const int j = row_nb(g, C.A.per0, C.A.per1, i, d0, d1);
                if (j >= 0) v |= s[j];
            }
        d[i] = v;
    }
}
// dst = align_up(src): OR over the 2^dim sibling group, on every member
__device__ void align_up(const Ctx& C, int l, int src, int dst) {
    const Lvl& g = C.A.lv[l];
    const uint32_t* s = C.set(src, l);
    uint32_t* d = C.set(dst, l);
    for (int i = threadIdx.x; i < g.nw; i += THREADS) {
        const int row = i / g.W, a0 = row / g.n1, a1 = row - a0 * g.n1;
        uint32_t v = 0;
        for (int k0 = 0; k0 < 2; ++k0)
            for (int k1 = 0; k1 < (g.n1 > 1 ? 2 : 1); ++k1) {
                const int j = row_nb(g, 0, 0, i, ((a0 & ~1) | k0) - a0, g.n1 > 1 ? ((a1 & ~1) | k1) - a1 : 0);
                if (j >= 0) v |= s[j];
            }
        d[i] = pair_or(v) & row_mask(g, i % g.W);
    }
}
// dst(level lp) = parents(src(level lp - 1)) [| also_or(level lp) when also >= 0]
__device__ void parents(const Ctx& C, int lp, int src, int dst, int also) {
    const Lvl& gp = C.A.lv[lp];
    const Lvl& gc = C.A.lv[lp - 1];
    const uint32_t* s = C.set(src, lp - 1);
    uint32_t* d = C.set(dst, lp);
    const uint32_t* o = also >= 0 ? C.set(also, lp) : nullptr;
    for (int i = threadIdx.x; i < gp.nw; i += THREADS) {
        const int prow = i / gp.W, pw = i - prow * gp.W;
        const int p0 = prow / gp.n1, p1 = prow - p0 * gp.n1;
        uint32_t v = 0;
        for (int k0 = 0; k0 < 2; ++k0)
            for (int k1 = 0; k1 < (gc.n1 > 1 ? 2 : 1); ++k1) {
                const int c0 = 2 * p0 + k0, c1 = gc.n1 > 1 ? 2 * p1 + k1 : 0;
                const uint32_t* cr = s + (c0 * gc.n1 + c1) * gc.W;
                if (gc.nr >= 64) v |= compress_or(cr[2 * pw]) | (compress_or(cr[2 * pw + 1]) << 16);
                else v |= compress_or(cr[0]);      // child row of <= 32 bits -> <= 16 parent bits
            }
        if (o) v |= o[i];
        d[i] = v & row_mask(gp, pw);
    }
}

// bits of the level-l leaf bitmap at level-0 resolution for level-0 word i0
__device__ __forceinline__ uint32_t leaf_at0(const Ctx& C, int l, int i0) {
    const Lvl& g0 = C.A.lv[0];
    const Lvl& g = C.A.lv[l];
    const int row = i0 / g0.W, w = i0 - row * g0.W;
    const int a0 = row / g0.n1, a1 = row - a0 * g0.n1;
    const int r0 = a0 >> l, r1 = g.n1 > 1 ? (a1 >> l) : 0;
    const uint32_t* lr = C.set(S_LEAF, l) + (r0 * g.n1 + r1) * g.W;
    const int start = (32 * w) >> l;                  // first level-l bit of this word
    const int cnt = (g0.nr < 32 ? g0.nr : 32) >> l;   // level-l bits covered
    uint32_t v = (lr[start >> 5] >> (start & 31));
    v &= cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
    for (int k = 0; k < l; ++k) v = spread2(v);
    return v;
}

__global__ void __launch_bounds__(THREADS) k_adapt_bits(BitArgs A) {
    extern __shared__ uint32_t smem_bits[];
    const Ctx C{A, smem_bits};
    const int L = A.L, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NWARP = THREADS / 32;
    tstamp(A, 0);

    // ---- 1: leaf / present bits of every level (warp per word, lane per tile;
    //         8 words per trip so the byte loads overlap), seeds | static -> T2
    constexpr int UL = 8;
    for (int l = 0; l < L; ++l) {
        const Lvl& g = A.lv[l];
        uint32_t* lf = C.set(S_LEAF, l);
        uint32_t* pr = C.set(S_PRES, l);
        const uint8_t* kd = A.kind[l];
        const bool st = l == 0 && A.static_tiles;
        for (int i0 = warp; i0 < g.nw; i0 += NWARP * UL) {
            uint8_t k[UL], sv[UL];
#pragma unroll
            for (int u = 0; u < UL; ++u) {
                const int i = i0 + u * NWARP;
                k[u] = 0;
                sv[u] = 0;
                if (i < g.nw) {
                    const int row = i / g.W, r = 32 * (i - row * g.W) + lane;
                    if (r < g.nr) {
                        k[u] = kd[(int64_t)row * g.nr + r];
                        if (st) sv[u] = A.static_tiles[(int64_t)row * g.nr + r];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < UL; ++u) {
                const int i = i0 + u * NWARP;
                if (i >= g.nw) break;
                const uint32_t bl = __ballot_sync(0xffffffffu, k[u] == 1);
                const uint32_t bp = __ballot_sync(0xffffffffu, k[u] != 0);
                const uint32_t bs = __ballot_sync(0xffffffffu, sv[u] != 0);
                if (lane == 0) {
                    lf[i] = bl;
                    pr[i] = bp;
                    if (l == 0) C.set(S_T2, 0)[i] = A.seeds[i] | bs;
                }
            }
        }
    }
    __syncthreads(); tstamp(A, 1);

    // ---- 2: coverage (each finest tile a leaf of exactly one level); ring
    //         check R pass (dilate2(leaf) -> T1)
    {
        const Lvl& g0 = A.lv[0];
        int viol = 0;
        for (int i = threadIdx.x; i < g0.nw; i += THREADS) {
            uint32_t ones = 0, twos = 0;
            for (int l = 0; l < L; ++l) {
                const uint32_t b = leaf_at0(C, l, i);
                twos |= ones & b;
                ones |= b;
            }
            viol += __popc(row_mask(g0, i % g0.W) & ~(ones & ~twos));
        }
        if (viol) atomicAdd(&A.status[L], viol);
    }
    for (int l = 0; l < L; ++l) dil_r(C, l, S_LEAF, S_T1);
    __syncthreads(); tstamp(A, 2);
    for (int l = 0; l < L; ++l) dil_a(C, l, S_T1, S_OWN);
    __syncthreads(); tstamp(A, 3);
    // ---- 3: ring count; des[0] = align_up(seeds); cur[0] = leaf[0]
    {
        int miss = 0;
        for (int l = 0; l < L; ++l) {
            const Lvl& g = A.lv[l];
            const uint32_t* dl = C.set(S_OWN, l);
            const uint32_t* pr = C.set(S_PRES, l);
            for (int i = threadIdx.x; i < g.nw; i += THREADS) miss += __popc(dl[i] & ~pr[i]);
        }
        if (miss) atomicAdd(&A.status[L + 1], miss);
    }
    {
        const Lvl& g0 = A.lv[0];
        if (L == 1) {
            for (int i = threadIdx.x; i < g0.nw; i += THREADS) C.set(S_DES, 0)[i] = row_mask(g0, i % g0.W);
        } else {
            align_up(C, 0, S_T2, S_DES);
        }
        for (int i = threadIdx.x; i < g0.nw; i += THREADS) C.set(S_CUR, 0)[i] = C.set(S_LEAF, 0)[i];
    }
    __syncthreads(); tstamp(A, 4);
    // ---- 4: desired / current coverage of the coarser levels
    for (int l = 1; l < L; ++l) {
        parents(C, l, S_DES, S_PAR, -1);
        parents(C, l, S_CUR, S_CUR, S_LEAF);
        __syncthreads(); tstamp(A, 5);
        const Lvl& g = A.lv[l];
        if (l == L - 1) {
            for (int i = threadIdx.x; i < g.nw; i += THREADS) C.set(S_DES, l)[i] = row_mask(g, i % g.W);
            __syncthreads(); tstamp(A, 6);
        } else {
            dil_r(C, l, S_PAR, S_T1);
            __syncthreads(); tstamp(A, 7);
            dil_a(C, l, S_T1, S_T2);
            __syncthreads(); tstamp(A, 8);
            align_up(C, l, S_T2, S_DES);
            __syncthreads(); tstamp(A, 9);
        }
    }
    // ---- 5: hysteresis per level (adapt.py:140-181)
    for (int l = 0; l < L; ++l) {
        const Lvl& g = A.lv[l];
        const bool guard = l > 0;
        if (guard) {
            parents(C, l, S_EFF, S_PAR, -1);
            __syncthreads(); tstamp(A, 10);
            dil_r(C, l, S_PAR, S_T1);
            __syncthreads(); tstamp(A, 11);
            dil_a(C, l, S_T1, S_T2);
            __syncthreads(); tstamp(A, 12);
        }
        // streaks (warp per word; 4 words per trip so the int16 loads overlap)
        const uint32_t* cur = C.set(S_CUR, l);
        const uint32_t* des = C.set(S_DES, l);
        const uint32_t* gw = C.set(S_T2, l);
        uint32_t* av = C.set(S_T1, l);
        int16_t* strk = A.streak[l];
        constexpr int U = 8;
        for (int i0 = warp; i0 < g.nw; i0 += NWARP * U) {
            int16_t so[U];
            bool cand[U], in[U];
            int64_t lin[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * NWARP;
                in[u] = false;
                cand[u] = false;
                so[u] = 0;
                lin[u] = 0;
                if (i < g.nw) {
                    const int row = i / g.W, w = i - row * g.W, r = 32 * w + lane;
                    in[u] = r < g.nr;
                    lin[u] = (int64_t)row * g.nr + r;
                    cand[u] = in[u] && (((cur[i] & ~des[i]) >> lane) & 1u);
                    if (in[u]) so[u] = strk[lin[u]];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * NWARP;
                if (i >= g.nw) break;
                const int16_t sn = cand[u] ? (int16_t)(so[u] + 1) : (int16_t)0;
                if (in[u] && sn != so[u]) strk[lin[u]] = sn;
                const bool gd = guard && ((gw[i] >> lane) & 1u);
                const uint32_t b = __ballot_sync(0xffffffffu, cand[u] && sn >= 2 && !gd);
                if (lane == 0) av[i] = b;
            }
        }
        __syncthreads(); tstamp(A, 13);
        // group-all and effective coverage
        uint32_t* eff = C.set(S_EFF, l);
        const uint32_t* par = C.set(S_PAR, l);
        for (int i = threadIdx.x; i < g.nw; i += THREADS) {
            uint32_t act = 0;
            if (A.grouped[l]) {
                const int row = i / g.W, a0 = row / g.n1, a1 = row - a0 * g.n1;
                act = 0xffffffffu;
                for (int k0 = 0; k0 < 2; ++k0)
                    for (int k1 = 0; k1 < (g.n1 > 1 ? 2 : 1); ++k1) {
                        const int j = row_nb(g, 0, 0, i, ((a0 & ~1) | k0) - a0,
                                             g.n1 > 1 ? ((a1 & ~1) | k1) - a1 : 0);
                        act &= j >= 0 ? pair_and(av[j]) : 0u;
                    }
            }
            uint32_t e = des[i] | (cur[i] & ~act);
            if (guard) e |= par[i];
            eff[i] = e & row_mask(g, i % g.W);
        }
        __syncthreads(); tstamp(A, 14);
    }
    // top level: eff = all ones after its own parents were taken (adapt.py:180-181)
    {
        const Lvl& g = A.lv[L - 1];
        for (int i = threadIdx.x; i < g.nw; i += THREADS) C.set(S_EFF, L - 1)[i] = row_mask(g, i % g.W);
    }
    __syncthreads(); tstamp(A, 15);
    // ---- 6: own = eff & ~parents(eff[l-1]); storage = dilate2(own)
    for (int l = 0; l < L; ++l) {
        const Lvl& g = A.lv[l];
        uint32_t* own = C.set(S_OWN, l);
        const uint32_t* eff = C.set(S_EFF, l);
        const uint32_t* par = C.set(S_PAR, l);
        for (int i = threadIdx.x; i < g.nw; i += THREADS) own[i] = l > 0 ? (eff[i] & ~par[i]) : eff[i];
    }
    __syncthreads(); tstamp(A, 16);
    for (int l = 0; l < L; ++l) dil_r(C, l, S_OWN, S_T1);
    __syncthreads(); tstamp(A, 17);
    for (int l = 0; l < L; ++l) dil_a(C, l, S_T1, S_T2);
    __syncthreads(); tstamp(A, 18);
    // ---- 7: new kinds (stores only: the old kinds are the leaf / present
    //         bits), no-op flags and counts by popcount; seeds cleared
    for (int l = 0; l < L; ++l) {
        const Lvl& g = A.lv[l];
        const uint32_t* own = C.set(S_OWN, l);
        const uint32_t* sto = C.set(S_T2, l);
        const uint32_t* lf = C.set(S_LEAF, l);
        const uint32_t* pr = C.set(S_PRES, l);
        int changed = 0, cnt = 0, fresh = 0;
        for (int i = threadIdx.x; i < g.nw; i += THREADS) {
            const uint32_t m = row_mask(g, i % g.W);
            const uint32_t o = own[i] & m, p = (o | sto[i]) & m;
            changed |= (o != lf[i]) || (p != pr[i]);
            cnt += __popc(p);
            fresh += __popc(p & ~pr[i]);
        }
        uint8_t* nk = A.nkind[l];
        for (int i = warp; i < g.nw; i += NWARP) {
            const int row = i / g.W, r = 32 * (i - row * g.W) + lane;
            if (r < g.nr)
                nk[(int64_t)row * g.nr + r] = ((own[i] >> lane) & 1u) ? 1 : (((sto[i] >> lane) & 1u) ? 2 : 0);
        }
        changed = __syncthreads_or(changed);
        if (threadIdx.x == 0 && changed) atomicOr(&A.status[l], 1);
        for (int off = 16; off > 0; off >>= 1) {
            cnt += __shfl_down_sync(0xffffffffu, cnt, off);
            fresh += __shfl_down_sync(0xffffffffu, fresh, off);
        }
        if (lane == 0) {
            if (cnt) atomicAdd(&A.status[L + 4 + l], cnt);
            if (fresh) atomicAdd(&A.status[2 * L + 4 + l], fresh);
        }
    }
    for (int i = threadIdx.x; i < A.lv[0].nw; i += THREADS) A.seeds[i] = 0;
}

// particle seeds (adapt.py:54-65) as level-0 bits + domain check + particles
// in level-0 leaves.  One atomicOr per run of equal words within a warp.
__global__ void k_seed_bits(int dim, int n, const double* x, int64_t xs, Lvl g0, T3 t0,
                            const uint8_t* kind0, uint32_t* seeds, int32_t* status, int L,
                            mlbm_error_t* err) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int word = -1;
    uint32_t bit = 0;
    int notleaf = 0, bad = 0;
    if (p < n) {
        int t[3] = {0, 0, 0};
        bool out = false;
        for (int a = 0; a < dim; ++a) {
            const double v = x[a * xs + p];
            const int64_t c = (int64_t)floor(v);
            const int64_t tt = c >= 0 ? c / 4 : -((-c + 3) / 4);
            if (tt < 0 || tt >= t0.v[a] || !(v == v)) out = true;
            t[a] = (int)tt;
        }
        if (out) {
            report_error(err, MLBM_ERR_DOMAIN, 0, t[0], t[1], t[2]);
            bad = 1;
        } else {
            const int64_t lin = ((int64_t)t[0] * t0.v[1] + t[1]) * t0.v[2] + t[2];
            const int64_t row = lin / g0.nr, r = lin - row * g0.nr;
            word = (int)(row * g0.W + (r >> 5));
            bit = 1u << (r & 31);
            notleaf = kind0[lin] != 1;
        }
    }
    // OR the bits of lanes with the same word; the lowest such lane writes
    const unsigned same = __match_any_sync(0xffffffffu, word);
    const uint32_t acc = __reduce_or_sync(same, bit);
    if (word >= 0 && lane == __ffs(same) - 1) atomicOr(&seeds[word], acc);
    const int c = __reduce_add_sync(0xffffffffu, notleaf + bad);
    if (lane == 0 && c) atomicAdd(&status[L + 2], c);
}

}  // namespace ab
}  // namespace mlbm

using namespace mlbm;

static unsigned long long* g_bits_ts = nullptr;
extern "C" unsigned long long* mlbm_adapt_bits_ts_ptr() { return g_bits_ts; }
extern "C" int mlbm_adapt_bits_set_timestamps(unsigned long long* buf) {
    g_bits_ts = buf;
    return 0;
}

// host side: geometry, eligibility, launch (called from mlbm_adapt_pass)
int mlbm_adapt_bits_launch(const mlbm_hier_t* h, uint8_t* const* nkind, int16_t* const* streak,
                                      uint8_t* seeds, const uint8_t* static_tiles, const double* x,
                                      int64_t xs, int32_t n, int32_t* status, mlbm_error_t* err,
                                      int64_t seeds_bytes, void* stream) {
    using namespace mlbm::ab;
    BitArgs A{};
    A.dim = h->dim;
    A.L = h->levels;
    const int dim = h->dim;
    int off = 0;
    for (int l = 0; l < h->levels; ++l) {
        int td[3];
        for (int a = 0; a < 3; ++a) td[a] = a < dim ? (h->finest[a] >> l) / 4 : 1;
        Lvl& g = A.lv[l];
        g.n0 = td[0];
        g.n1 = dim == 3 ? td[1] : 1;
        g.nr = dim == 3 ? td[2] : td[1];
        if (!(g.nr < 32 || g.nr % 32 == 0)) return 0;                  // not packable
        g.W = (g.nr + 31) / 32;
        g.tail = g.nr % 32 ? ((1u << (g.nr % 32)) - 1u) : 0xffffffffu;
        g.nw = g.n0 * g.n1 * g.W;
        g.off = off;
        off += g.nw;
        bool grp = true;
        for (int a = 0; a < dim; ++a) grp &= td[a] % 2 == 0;
        A.grouped[l] = grp;
        A.kind[l] = h->kind[l];
        A.nkind[l] = nkind[l];
        A.streak[l] = streak[l];
    }
    A.nwt = off;
    A.per0 = h->periodic[0];
    A.per1 = dim == 3 ? h->periodic[1] : 0;
    A.perr = dim == 3 ? h->periodic[2] : h->periodic[1];
    const size_t smem = (size_t)NSET * A.nwt * sizeof(uint32_t);
    if (smem > 200 * 1024 || (int64_t)A.lv[0].nw * 4 > seeds_bytes) return 0;
    A.seeds = (uint32_t*)seeds;
    A.static_tiles = static_tiles;
    A.status = status;
    A.ts = g_bits_ts;       // caller-owned (mlbm_adapt_bits_set_timestamps), may be null
    if (A.ts) cudaMemsetAsync(A.ts, 0, 64 * sizeof(unsigned long long), as_stream(stream));
    cudaStream_t s = as_stream(stream);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_adapt_bits, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    int launches = 0;
    if (n > 0) {
        T3 t0{{(h->finest[0]) / 4, dim > 1 ? (h->finest[1]) / 4 : 1, dim == 3 ? (h->finest[2]) / 4 : 1}};
        k_seed_bits<<<(n + 255) / 256, 256, 0, s>>>(dim, n, x, xs, A.lv[0], t0, h->kind[0], A.seeds,
                                                   status, h->levels, err);
        ++launches;
    }
    k_adapt_bits<<<1, THREADS, smem, s>>>(A);
    ++launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return -(int)e;
    return launches;               // > 0: handled; 0: not eligible (byte path)
}
