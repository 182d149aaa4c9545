// HOME-LBM level kernels for sm_100a.
//
//   mlbm_level_step  — fused pull-stream + moment BGK collide + boundaries
//                      (reference solver.py:336-481, one call per level step)
//   mlbm_downward    — I^d fill from the coarser level (solver.py:501-526)
//   mlbm_upward      — I^u fill from the finer level   (solver.py:536-560)
//
// Level step design: one 4^D tile per thread group, one thread
// per cell.  Each cell turns its own moments into Hermite coefficients and
// reconstructs its Q populations in opposite pairs (shared even/odd parts),
// pushing the ones that stay inside the tile into a shared-memory buffer
// fbuf[dir][cell].  Populations entering the tile from its 3^D-1 neighbour
// tiles are reconstructed by a static halo work list (sorted by direction so
// warps stay convergent).  After one barrier each cell pulls its Q incoming
// populations, accumulates the bare moments in the shifted form
// (g = f - w, drho = rho - 1), collides, and the BC tiles apply the
// outlet/inlet passes in reference face order through shared memory.
#include <algorithm>
#include "common.cuh"
#include "exchange.cuh"

namespace mlbm {

// ---------------------------------------------------------------------------
// compile-time halo tables.  The (4+2)^D box around a tile minus the tile is
// the halo: HB cells, each staged once (its Hermite coefficients) in shared
// memory.  Items are the (halo cell, direction, destination) pulls that enter
// the tile, sorted by direction so warps stay convergent.
template <int D> struct HaloTable {
    static constexpr int HB = D == 2 ? 20 : 152;     // halo cells
    static constexpr int N = D == 2 ? 44 : 728;      // halo items
    uint32_t cell[HB];                               // nbi | srcl << 5
    uint32_t item[N];                                // h | dir << 8 | dstl << 13 | nbi << 19
};

template <int D> constexpr int box_halo_index(int bx, int by, int bz) {
    // halo cells enumerated in box order (bx fastest), skipping the tile
    int h = 0;
    for (int z = (D == 3 ? -1 : 0); z <= (D == 3 ? 4 : 0); ++z)
        for (int y = -1; y <= 4; ++y)
            for (int x = -1; x <= 4; ++x) {
                const bool inside = x >= 0 && x < 4 && y >= 0 && y < 4 && (D == 2 || (z >= 0 && z < 4));
                if (inside) continue;
                if (x == bx && y == by && z == bz) return h;
                ++h;
            }
    return -1;
}

template <int D> constexpr HaloTable<D> make_halo_table() {
    HaloTable<D> h{};
    int nh = 0;
    for (int z = (D == 3 ? -1 : 0); z <= (D == 3 ? 4 : 0); ++z)
        for (int y = -1; y <= 4; ++y)
            for (int x = -1; x <= 4; ++x) {
                const bool inside = x >= 0 && x < 4 && y >= 0 && y < 4 && (D == 2 || (z >= 0 && z < 4));
                if (inside) continue;
                const int b[3] = {x, y, z};
                int o[3] = {0, 0, 0}, s[3] = {0, 0, 0};
                for (int a = 0; a < 3; ++a) {
                    o[a] = b[a] < 0 ? -1 : (b[a] > 3 ? 1 : 0);
                    s[a] = b[a] - 4 * o[a];
                }
                const int nbi = nb_index<D>(o[0], o[1], o[2]);
                const int srcl = s[0] + 4 * s[1] + (D == 3 ? 16 * s[2] : 0);
                h.cell[nh++] = (uint32_t)nbi | ((uint32_t)srcl << 5);
            }
    int n = 0;
    constexpr int T = Geo<D>::T;
    for (int i = 1; i < Geo<D>::Q; ++i) {
        for (int x = 0; x < T; ++x) {
            int l[3] = {x & 3, (x >> 2) & 3, D == 3 ? (x >> 4) & 3 : 0};
            int s[3] = {0, 0, 0};
            bool outside = false;
            for (int a = 0; a < 3; ++a) {
                s[a] = l[a] - cvec<D>(i, a);
                if (s[a] < 0 || s[a] > 3) outside = true;
            }
            if (!outside) continue;
            const int hidx = box_halo_index<D>(s[0], s[1], s[2]);
            int o[3] = {0, 0, 0};
            for (int a = 0; a < 3; ++a) o[a] = s[a] < 0 ? -1 : (s[a] > 3 ? 1 : 0);
            const int nbi = nb_index<D>(o[0], o[1], o[2]);
            h.item[n++] = (uint32_t)hidx | ((uint32_t)i << 8) | ((uint32_t)x << 13) | ((uint32_t)nbi << 19);
        }
    }
    return h;
}

// items of direction i: tile cells whose pull source lies outside the tile
template <int D> constexpr int halo_count(int i) {
    int inside = 1;
    for (int a = 0; a < D; ++a) inside *= 4 - (cvec<D>(i, a) != 0 ? 1 : 0);
    return Geo<D>::T - inside;
}
template <int D> constexpr int halo_offset(int i) {
    int o = 0;
    for (int j = 1; j < i; ++j) o += halo_count<D>(j);
    return o;
}

constexpr HaloTable<2> k_halo2 = make_halo_table<2>();
constexpr HaloTable<3> k_halo3 = make_halo_table<3>();
// in global memory, read through L1 with __ldg: lanes index consecutive
// entries (coalesced); a __constant__ table would serialise the divergent
// per-lane indices in the constant cache
__device__ const HaloTable<2> g_halo2 = k_halo2;
__device__ const HaloTable<3> g_halo3 = k_halo3;

template <int D> __device__ __forceinline__ uint32_t halo_item(int k) {
    if constexpr (D == 2) return __ldg(&g_halo2.item[k]); else return __ldg(&g_halo3.item[k]);
}
template <int D> __device__ __forceinline__ uint32_t halo_cell(int k) {
    if constexpr (D == 2) return __ldg(&g_halo2.cell[k]); else return __ldg(&g_halo3.cell[k]);
}

// ---------------------------------------------------------------------------
// Hermite coefficients of one cell (shifted form):
//   g_i = f_i - w_i = w_i [ dr + sum H2_ab(c_i) B_ab + sum c_a A_a + sum H3_t(c_i) G_t ]
template <int D, typename R> struct Coef {
    R dr;
    R A[D];
    R B[Geo<D>::NS];
    R G[Geo<D>::N3];
};

template <int D, typename R>
__device__ __forceinline__ void make_coef(const R (&m)[Geo<D>::NM], R h3xyz, Coef<D, R>& c) {
    constexpr int NS = Geo<D>::NS;
    const R rho = R(1) + m[0];
    c.dr = m[0];
    R u[D];
#pragma unroll
    for (int a = 0; a < D; ++a) { u[a] = m[1 + a]; c.A[a] = R(3) * rho * u[a]; }
#pragma unroll
    for (int k = 0; k < NS; ++k)
        c.B[k] = (s_a<D>(k) == s_b<D>(k) ? R(4.5) : R(9)) * rho * m[1 + D + k];
#pragma unroll
    for (int t = 0; t < Geo<D>::N3; ++t) {
        const int a = h3t<D>(t, 0), b = h3t<D>(t, 1), g = h3t<D>(t, 2);
        const R Sab = m[1 + D + sidx<D>(a, b)], Sag = m[1 + D + sidx<D>(a, g)],
                Sbg = m[1 + D + sidx<D>(b, g)];
        const R gam = Sab * u[g] + Sag * u[b] + Sbg * u[a] - R(2) * u[a] * u[b] * u[g];
        const R coef = (D == 3 && t == 6) ? h3xyz : R(13.5);
        c.G[t] = coef * rho * gam;
    }
}

template <int D, int I, typename R>
__device__ __forceinline__ R even_part(const Coef<D, R>& c) {
    R e = c.dr;
#pragma unroll
    for (int k = 0; k < Geo<D>::NS; ++k) e += R(h2v<D>(I, s_a<D>(k), s_b<D>(k))) * c.B[k];
    return e;
}
template <int D, int I, typename R>
__device__ __forceinline__ R odd_part(const Coef<D, R>& c) {
    R o = R(0);
#pragma unroll
    for (int a = 0; a < D; ++a)
        if (cvec<D>(I, a) != 0) o += R(cvec<D>(I, a)) * c.A[a];
#pragma unroll
    for (int t = 0; t < Geo<D>::N3; ++t)
        if (h3v<D>(I, t) != 0.0) o += R(h3v<D>(I, t)) * c.G[t];
    return o;
}
template <int D, int I, typename R>
__device__ __forceinline__ R g_dir(const Coef<D, R>& c) {
    return R(wdir<D>(I)) * (even_part<D, I>(c) + odd_part<D, I>(c));
}

// runtime-direction reconstruct (halo items, special cells): switch over I
template <int D, typename R, int I = 0>
__device__ __forceinline__ R g_dir_rt(int i, const Coef<D, R>& c) {
    if constexpr (I + 1 >= Geo<D>::Q) {
        return g_dir<D, I>(c);
    } else {
        if (i == I) return g_dir<D, I>(c);
        return g_dir_rt<D, R, I + 1>(i, c);
    }
}

// coefficient slot layout: dr | A[D] | B[NS] | G[N3]
template <int D> struct CoefSlots {
    static constexpr int DR = 0, A = 1, B = 1 + D, G = 1 + D + Geo<D>::NS, N = 1 + D + Geo<D>::NS + Geo<D>::N3;
};

template <int D, typename R>
__device__ __forceinline__ void store_coef(const Coef<D, R>& c, R* hc, int h, int HB) {
    using CS = CoefSlots<D>;
    hc[CS::DR * HB + h] = c.dr;
#pragma unroll
    for (int a = 0; a < D; ++a) hc[(CS::A + a) * HB + h] = c.A[a];
#pragma unroll
    for (int k = 0; k < Geo<D>::NS; ++k) hc[(CS::B + k) * HB + h] = c.B[k];
#pragma unroll
    for (int t = 0; t < Geo<D>::N3; ++t) hc[(CS::G + t) * HB + h] = c.G[t];
}

// g_I of a staged halo cell, reading only the coefficients direction I needs
template <int D, int I, typename R>
__device__ __forceinline__ R g_dir_staged(const R* hc, int h, int HB) {
    using CS = CoefSlots<D>;
    R e = hc[CS::DR * HB + h];
#pragma unroll
    for (int k = 0; k < Geo<D>::NS; ++k) {
        constexpr int dummy = 0; (void)dummy;
        const double hv = h2v<D>(I, s_a<D>(k), s_b<D>(k));
        if (hv != 0.0) e += R(hv) * hc[(CS::B + k) * HB + h];
    }
    R o = R(0);
#pragma unroll
    for (int a = 0; a < D; ++a)
        if (cvec<D>(I, a) != 0) o += R(cvec<D>(I, a)) * hc[(CS::A + a) * HB + h];
#pragma unroll
    for (int t = 0; t < Geo<D>::N3; ++t)
        if (h3v<D>(I, t) != 0.0) o += R(h3v<D>(I, t)) * hc[(CS::G + t) * HB + h];
    return R(wdir<D>(I)) * (e + o);
}

template <int D, typename R, int I = 1>
__device__ __forceinline__ R g_dir_staged_rt(int i, const R* hc, int h, int HB) {
    if constexpr (I + 1 >= Geo<D>::Q) {
        return g_dir_staged<D, I>(hc, h, HB);
    } else {
        if (i == I) return g_dir_staged<D, I>(hc, h, HB);
        return g_dir_staged_rt<D, R, I + 1>(i, hc, h, HB);
    }
}

template <int D, typename R>
__device__ __forceinline__ void load_moments(const FieldsT<R>& f, int64_t cell,
                                             R (&m)[Geo<D>::NM]) {
#pragma unroll
    for (int k = 0; k < Geo<D>::NM; ++k) m[k] = __ldg(&f.at(k, cell));
}

// ---------------------------------------------------------------------------
struct StepArgs {
    mlbm_level_t lv;
    mlbm_fields_t src, dst;
    mlbm_collide_t cp;
    mlbm_bc_t bc;
    mlbm_error_t* err;
    ExchArgs ex;          // mode 5 only: the level-0 exchange between stream and collide
};

template <int D, int I, typename R>
__device__ __forceinline__ void accumulate(R g, R& dr, R (&mm)[D], R (&pi)[Geo<D>::NS]) {
    dr += g;
#pragma unroll
    for (int a = 0; a < D; ++a)
        if (cvec<D>(I, a) != 0) mm[a] += R(cvec<D>(I, a)) * g;
#pragma unroll
    for (int k = 0; k < Geo<D>::NS; ++k) {
        const double h = h2v<D>(I, s_a<D>(k), s_b<D>(k));
        if (h != 0.0) pi[k] += R(h) * g;
    }
}

template <int D, typename R, int P = 0>
__device__ __forceinline__ void push_pairs(const Coef<D, R>& c, R* fb, int lc, const int (&l)[3]) {
    if constexpr (P < Geo<D>::NP) {
        constexpr int I = 2 * P + 1, J = 2 * P + 2;
        constexpr int T = Geo<D>::T;
        const R e = even_part<D, I>(c), o = odd_part<D, I>(c);
        const R w = R(wdir<D>(I));
        const R gp = w * (e + o), gm = w * (e - o);
        constexpr int c0 = cvec<D>(I, 0), c1 = cvec<D>(I, 1), c2 = cvec<D>(I, 2);
        // +c lands at l + c, -c at l - c
        const bool inp = (unsigned)(l[0] + c0) < 4u && (unsigned)(l[1] + c1) < 4u &&
                         (D == 2 || (unsigned)(l[2] + c2) < 4u);
        const bool inm = (unsigned)(l[0] - c0) < 4u && (unsigned)(l[1] - c1) < 4u &&
                         (D == 2 || (unsigned)(l[2] - c2) < 4u);
        constexpr int doff = c0 + 4 * c1 + (D == 3 ? 16 * c2 : 0);
        if (inp) fb[I * T + lc + doff] = gp;
        if (inm) fb[J * T + lc - doff] = gm;
        push_pairs<D, R, P + 1>(c, fb, lc, l);
    }
}

template <int D, typename R, bool SPECIAL, int I = 0>
__device__ __forceinline__ void pull_all(const R* fb, int lc, uint64_t mask,
                                         const Coef<D, R>& own, R& dr, R (&mm)[D],
                                         R (&pi)[Geo<D>::NS]) {
    if constexpr (I < Geo<D>::Q) {
        constexpr int T = Geo<D>::T;
        R g = fb[I * T + lc];
        if constexpr (SPECIAL) {
            if ((mask >> I) & 1ull) g = g_dir<D, opp<D>(I)>(own);
            else if ((mask >> (32 + I)) & 1ull) g = g_dir<D, I>(own);
        }
        accumulate<D, I>(g, dr, mm, pi);
        pull_all<D, R, SPECIAL, I + 1>(fb, lc, mask, own, dr, mm, pi);
    }
}

template <int D, typename R>
__device__ __forceinline__ void halo_stage(const FieldsT<R>& src, R* hc, const int* snb, int lc, R h3xyz) {
    constexpr int T = Geo<D>::T, HB = HaloTable<D>::HB;
    for (int h = lc; h < HB; h += T) {
        const uint32_t hcell = halo_cell<D>(h);
        const int ns = snb[hcell & 31];
        if (ns < 0) continue;        // absent neighbour: its pulls are special-cased
        R m[Geo<D>::NM];
        load_moments<D, R>(src, (int64_t)ns * T + (int)(hcell >> 5), m);
        Coef<D, R> c;
        make_coef<D, R>(m, h3xyz, c);
        store_coef<D, R>(c, hc, h, HB);
    }
}

// 3D: warp PAR of the tile handles direction 2p+1+PAR of every pair p, one
// compile-time-specialised direction at a time (no divergence, only the
// coefficients that direction needs are read)
template <int D, typename R, int PAR, int P = 0>
__device__ __forceinline__ void halo_items_dir(R* fb, const R* hc, const int* snb, int lane) {
    if constexpr (P < Geo<D>::NP) {
        constexpr int I = 2 * P + 1 + PAR;
        constexpr int T = Geo<D>::T, HB = HaloTable<D>::HB;
        constexpr int OFF = halo_offset<D>(I), CNT = halo_count<D>(I);
#pragma unroll
        for (int j = lane; j < CNT; j += 32) {
            const uint32_t it = halo_item<D>(OFF + j);
            const int h = it & 255, dstl = (it >> 13) & 63, nbi = (it >> 19) & 31;
            if (snb[nbi] >= 0) fb[I * T + dstl] = g_dir_staged<D, I>(hc, h, HB);
        }
        halo_items_dir<D, R, PAR, P + 1>(fb, hc, snb, lane);
    }
}

template <int D, typename R>
__device__ __forceinline__ void halo_items(R* fb, const R* hc, const int* snb, int lc) {
    if constexpr (D == 3) {
        if (lc < 32) halo_items_dir<D, R, 0>(fb, hc, snb, lc);
        else halo_items_dir<D, R, 1>(fb, hc, snb, lc - 32);
        return;
    }
    constexpr int T = Geo<D>::T, HB = HaloTable<D>::HB, NH = HaloTable<D>::N;
    for (int k = lc; k < NH; k += T) {
        const uint32_t it = halo_item<D>(k);
        const int h = it & 255, dir = (it >> 8) & 31, dstl = (it >> 13) & 63;
        if (snb[halo_cell<D>(h) & 31] < 0) continue;
        fb[dir * T + dstl] = g_dir_staged_rt<D, R>(dir, hc, h, HB);
    }
}

// ===========================================================================
// D3Q27 stream by sum factorisation.  D3Q27 is the tensor
// product {-1,0,1}^3 and the reconstruction basis is separable:
//   g(c) = w1(cx) w1(cy) w1(cz) sum_{n} a[nx][ny][nz] h_nx(cx) h_ny(cy) h_nz(cz)
// with h0 = 1, h1 = c, h2 = c^2 - 1/3 and the 17 coefficients of make_coef
// placed at their multi-indices (|n| <= 3).  All 27 populations of a cell cost
// three 1D passes (~110 flops instead of 13 pairs x ~22); the bare moments of
// the 27 pulled populations are the transposed passes (~66 adds).  Halo faces,
// edges and corners are evaluated straight from the neighbour's moments in
// registers: a face cell contracts its normal axis first and then does a 2D
// pass over the 9 in-plane directions (no coefficient staging in shared memory).
namespace tp {

MLBM_HD constexpr double hp(int n, int c) { return n == 0 ? 1.0 : n == 1 ? (double)c : (double)(c * c) - CS2; }
MLBM_HD constexpr double w1(int c) { return c == 0 ? 2.0 / 3.0 : 1.0 / 6.0; }
MLBM_HD constexpr bool has3(int nx, int ny, int nz) { return nx + ny + nz <= 3; }
// D3Q27 direction index of velocity c (common.cuh ordering): 5-bit entries
// k = (cx+1) + 3 (cy+1) + 9 (cz+1) packed in three words, so a call with
// unrolled (compile-time) arguments folds to a constant and a runtime call
// costs a few integer ops (no search over the 27 directions)
MLBM_HD constexpr int dir3(int cx, int cy, int cz) {
    const int k = (cx + 1) + 3 * (cy + 1) + 9 * (cz + 1);
    const unsigned long long w = k < 12 ? 0x691158e16656614ull : (k < 24 ? 0x49597958e370402ull : 0x4dfaull);
    return (int)((w >> (5 * (k % 12))) & 31ull);
}
// multiply by a compile-time Hermite value without rounding-neutral folds lost
template <typename R> __device__ __forceinline__ R hmul(double h, R x) {
    return h == 1.0 ? x : (h == -1.0 ? -x : R(h) * x);
}
// running sum whose "first" flag resolves at compile time after unrolling
template <typename R> struct Acc {
    R s;
    bool z = true;
    __device__ __forceinline__ void add(R t) { if (z) { s = t; z = false; } else s += t; }
};

template <typename R>
__device__ __forceinline__ void tcoef(const Coef<3, R>& c, R (&a)[3][3][3]) {
    a[0][0][0] = c.dr;
    a[1][0][0] = c.A[0];
    a[0][1][0] = c.A[1];
    a[0][0][1] = c.A[2];
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        int n[3] = {0, 0, 0};
        ++n[s_a<3>(k)];
        ++n[s_b<3>(k)];
        a[n[0]][n[1]][n[2]] = c.B[k];
    }
#pragma unroll
    for (int t = 0; t < 7; ++t) {
        int n[3] = {0, 0, 0};
        ++n[h3t<3>(t, 0)];
        ++n[h3t<3>(t, 1)];
        ++n[h3t<3>(t, 2)];
        a[n[0]][n[1]][n[2]] = c.G[t];
    }
}

template <typename R>
__device__ __forceinline__ void load_tcoef(const FieldsT<R>& f, int64_t cell, R h3xyz, R (&a)[3][3][3]) {
    R m[10];
    load_moments<3, R>(f, cell, m);
    Coef<3, R> c;
    make_coef<3, R>(m, h3xyz, c);
    tcoef<R>(c, a);
}

// all 27 populations g[cx+1][cy+1][cz+1]
template <typename R>
__device__ __forceinline__ void recon_all(const R (&a)[3][3][3], R (&g)[3][3][3]) {
    Acc<R> P[3][3][3];   // [nx][ny][cz+1]
#pragma unroll
    for (int nx = 0; nx < 3; ++nx)
#pragma unroll
        for (int ny = 0; ny < 3; ++ny)
#pragma unroll
            for (int cz = -1; cz <= 1; ++cz)
#pragma unroll
                for (int nz = 0; nz < 3; ++nz) {
                    if (!has3(nx, ny, nz) || hp(nz, cz) == 0.0) continue;
                    P[nx][ny][cz + 1].add(hmul<R>(hp(nz, cz), a[nx][ny][nz]));
                }
    Acc<R> Q[3][3][3];   // [nx][cy+1][cz+1]
#pragma unroll
    for (int nx = 0; nx < 3; ++nx)
#pragma unroll
        for (int cy = -1; cy <= 1; ++cy)
#pragma unroll
            for (int cz = 0; cz < 3; ++cz)
#pragma unroll
                for (int ny = 0; ny < 3; ++ny) {
                    if (P[nx][ny][cz].z || hp(ny, cy) == 0.0) continue;
                    Q[nx][cy + 1][cz].add(hmul<R>(hp(ny, cy), P[nx][ny][cz].s));
                }
#pragma unroll
    for (int cx = -1; cx <= 1; ++cx)
#pragma unroll
        for (int cy = 0; cy < 3; ++cy)
#pragma unroll
            for (int cz = 0; cz < 3; ++cz) {
                Acc<R> s;
#pragma unroll
                for (int nx = 0; nx < 3; ++nx) {
                    if (Q[nx][cy][cz].z || hp(nx, cx) == 0.0) continue;
                    s.add(hmul<R>(hp(nx, cx), Q[nx][cy][cz].s));
                }
                g[cx + 1][cy][cz] = R(w1(cx) * w1(cy - 1) * w1(cz - 1)) * s.s;
            }
}

// bare moments of 27 pulled populations: dr, m_a, Pi_ab = sum H2_ab g
template <typename R>
__device__ __forceinline__ void moments_of(const R (&g)[3][3][3], R& dr, R (&mm)[3], R (&pi)[6]) {
    R X[3][3][3];        // [n][cy][cz] = sum_cx cx^n g
#pragma unroll
    for (int cy = 0; cy < 3; ++cy)
#pragma unroll
        for (int cz = 0; cz < 3; ++cz) {
            const R s = g[2][cy][cz] + g[0][cy][cz];
            X[0][cy][cz] = s + g[1][cy][cz];
            X[1][cy][cz] = g[2][cy][cz] - g[0][cy][cz];
            X[2][cy][cz] = s;
        }
    R Y[3][3][3];        // [nx][ny][cz], nx + ny <= 2
#pragma unroll
    for (int nx = 0; nx < 3; ++nx)
#pragma unroll
        for (int cz = 0; cz < 3; ++cz) {
            const R s = X[nx][2][cz] + X[nx][0][cz];
            Y[nx][0][cz] = s + X[nx][1][cz];
            if (nx <= 1) Y[nx][1][cz] = X[nx][2][cz] - X[nx][0][cz];
            if (nx == 0) Y[nx][2][cz] = s;
        }
    R M[3][3][3];        // [nx][ny][nz], |n| <= 2
#pragma unroll
    for (int nx = 0; nx < 3; ++nx)
#pragma unroll
        for (int ny = 0; ny < 3; ++ny) {
            if (nx + ny > 2) continue;
            const R s = Y[nx][ny][2] + Y[nx][ny][0];
            M[nx][ny][0] = s + Y[nx][ny][1];
            if (nx + ny <= 1) M[nx][ny][1] = Y[nx][ny][2] - Y[nx][ny][0];
            if (nx + ny == 0) M[nx][ny][2] = s;
        }
    dr = M[0][0][0];
    mm[0] = M[1][0][0];
    mm[1] = M[0][1][0];
    mm[2] = M[0][0][1];
    const R third = dr * R(CS2);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        int n[3] = {0, 0, 0};
        ++n[s_a<3>(k)];
        ++n[s_b<3>(k)];
        const R v = M[n[0]][n[1]][n[2]];
        pi[k] = s_a<3>(k) == s_b<3>(k) ? v - third : v;
    }
}

template <int A, int NA, int NU, int NV>
MLBM_HD constexpr int pidx(int which) {   // multi-index of (nA along A, nU along U, nV along V)
    constexpr int U = A == 0 ? 1 : 0, V = A == 2 ? 1 : 2;
    return which == A ? NA : which == U ? NU : NV;
}

// face cell with normal axis A: 9 in-plane populations gf[cu+1][cv+1] for the
// inward velocity cA = +-1 (runtime); U < V are the in-plane axes
template <int A, typename R>
__device__ __forceinline__ void face_eval(const R (&a)[3][3][3], R cA, R (&gf)[3][3]) {
    constexpr int U = A == 0 ? 1 : 0, V = A == 2 ? 1 : 2;
    Acc<R> b[3][3];      // [nu][nv]
#pragma unroll
    for (int nu = 0; nu < 3; ++nu)
#pragma unroll
        for (int nv = 0; nv < 3; ++nv)
#pragma unroll
            for (int na = 0; na < 3; ++na) {
                int n[3];
                n[A] = na; n[U] = nu; n[V] = nv;
                if (!has3(n[0], n[1], n[2])) continue;
                const R x = a[n[0]][n[1]][n[2]];
                b[nu][nv].add(na == 0 ? x : (na == 1 ? cA * x : R(2.0 / 3.0) * x));
            }
    Acc<R> P[3][3];      // [nu][cv+1]
#pragma unroll
    for (int nu = 0; nu < 3; ++nu)
#pragma unroll
        for (int cv = -1; cv <= 1; ++cv)
#pragma unroll
            for (int nv = 0; nv < 3; ++nv) {
                if (b[nu][nv].z || hp(nv, cv) == 0.0) continue;
                P[nu][cv + 1].add(hmul<R>(hp(nv, cv), b[nu][nv].s));
            }
#pragma unroll
    for (int cu = -1; cu <= 1; ++cu)
#pragma unroll
        for (int cv = 0; cv < 3; ++cv) {
            Acc<R> s;
#pragma unroll
            for (int nu = 0; nu < 3; ++nu) {
                if (P[nu][cv].z || hp(nu, cu) == 0.0) continue;
                s.add(hmul<R>(hp(nu, cu), P[nu][cv].s));
            }
            gf[cu + 1][cv] = R(w1(1) * w1(cu) * w1(cv - 1)) * s.s;
        }
}

// edge cell with free axis E: the 3 populations ge[cE+1] for inward velocities
// cP, cQ = +-1 (runtime) on the two fixed axes P < Q
template <int E, typename R>
__device__ __forceinline__ void edge_eval(const R (&a)[3][3][3], R cP, R cQ, R (&ge)[3]) {
    constexpr int P = E == 0 ? 1 : 0, Q = E == 2 ? 1 : 2;
    const R hpq[3] = {R(1), cP, R(2.0 / 3.0)};
    const R hqq[3] = {R(1), cQ, R(2.0 / 3.0)};
    Acc<R> b[3];
#pragma unroll
    for (int ne = 0; ne < 3; ++ne)
#pragma unroll
        for (int np = 0; np < 3; ++np)
#pragma unroll
            for (int nq = 0; nq < 3; ++nq) {
                int n[3];
                n[E] = ne; n[P] = np; n[Q] = nq;
                if (!has3(n[0], n[1], n[2])) continue;
                R x = a[n[0]][n[1]][n[2]];
                if (np) x *= hpq[np];
                if (nq) x *= hqq[nq];
                b[ne].add(x);
            }
#pragma unroll
    for (int ce = -1; ce <= 1; ++ce) {
        Acc<R> s;
#pragma unroll
        for (int ne = 0; ne < 3; ++ne) {
            if (b[ne].z || hp(ne, ce) == 0.0) continue;
            s.add(hmul<R>(hp(ne, ce), b[ne].s));
        }
        ge[ce + 1] = R(w1(1) * w1(1) * w1(ce)) * s.s;
    }
}

template <typename R>
__device__ __forceinline__ R corner_eval(const R (&a)[3][3][3], R cx, R cy, R cz) {
    const R hx[3] = {R(1), cx, R(2.0 / 3.0)}, hy[3] = {R(1), cy, R(2.0 / 3.0)}, hz[3] = {R(1), cz, R(2.0 / 3.0)};
    Acc<R> s;
#pragma unroll
    for (int nx = 0; nx < 3; ++nx)
#pragma unroll
        for (int ny = 0; ny < 3; ++ny)
#pragma unroll
            for (int nz = 0; nz < 3; ++nz) {
                if (!has3(nx, ny, nz)) continue;
                R x = a[nx][ny][nz];
                if (nx) x *= hx[nx];
                if (ny) x *= hy[ny];
                if (nz) x *= hz[nz];
                s.add(x);
            }
    return R(w1(1) * w1(1) * w1(1)) * s.s;
}

// direction index of a velocity with one runtime-signed component
template <int A> MLBM_HD int dir_sel(bool neg, int cu, int cv) {
    // component along A is -1 if neg else +1; cu, cv along the other two axes
    constexpr int U = A == 0 ? 1 : 0, V = A == 2 ? 1 : 2;
    int cp[3], cm[3];
    cp[A] = 1; cm[A] = -1; cp[U] = cm[U] = cu; cp[V] = cm[V] = cv;
    return neg ? dir3(cm[0], cm[1], cm[2]) : dir3(cp[0], cp[1], cp[2]);
}

constexpr bool dir3_table_ok() {
    for (int i = 0; i < 27; ++i)
        if (dir3(cvec<3>(i, 0), cvec<3>(i, 1), cvec<3>(i, 2)) != i) return false;
    return true;
}
static_assert(dir3_table_ok(), "packed D3Q27 direction table");

// runtime-velocity direction index (unrolled compare over the 26 moving directions)
MLBM_HD int dir_rt(int cx, int cy, int cz) { return dir3(cx, cy, cz); }

// slot of velocity c in the push/pull buffer: the buffer is private to the
// kernel, so it is indexed by the velocity's digits rather than by the D3Q27
// direction number (no table lookup for runtime velocities)
MLBM_HD constexpr int kidx(int cx, int cy, int cz) { return (cx + 1) + 3 * (cy + 1) + 9 * (cz + 1); }

template <int A, typename R>
__device__ __forceinline__ void face_body(const FieldsT<R>& src, R* fb, const int* snb, int f, R h3xyz) {
    constexpr int T = 64, U = A == 0 ? 1 : 0, V = A == 2 ? 1 : 2;
    constexpr int SA = A == 0 ? 1 : A == 1 ? 4 : 16, SU = U == 0 ? 1 : 4, SV = V == 1 ? 4 : 16;
    const int side = (f >> 4) & 1, u = f & 3, v = (f >> 2) & 3;
    int o[3] = {0, 0, 0};
    o[A] = side ? 1 : -1;
    const int ns = snb[nb_index<3>(o[0], o[1], o[2])];
    if (ns < 0) return;
    const int srcl = (side ? 0 : 3) * SA + u * SU + v * SV;
    R a[3][3][3];
    load_tcoef<R>(src, (int64_t)ns * T + srcl, h3xyz, a);
    R gf[3][3];
    face_eval<A, R>(a, side ? R(-1) : R(1), gf);
    const int base = (side ? 3 : 0) * SA;
#pragma unroll
    for (int cu = -1; cu <= 1; ++cu)
#pragma unroll
        for (int cv = -1; cv <= 1; ++cv) {
            const int lu = u + cu, lv = v + cv;
            if ((unsigned)lu > 3u || (unsigned)lv > 3u) continue;
            constexpr int KA = A == 0 ? 1 : A == 1 ? 3 : 9, KU = U == 0 ? 1 : 3, KV = V == 1 ? 3 : 9;
            const int k = (side ? 0 : 2) * KA + (cu + 1) * KU + (cv + 1) * KV;   // c_A = -1 / +1
            fb[k * T + base + lu * SU + lv * SV] = gf[cu + 1][cv + 1];
        }
}

template <int E, typename R>
__device__ __forceinline__ void edge_body(const FieldsT<R>& src, R* fb, const int* snb, int e, R h3xyz) {
    constexpr int T = 64, P = E == 0 ? 1 : 0, Q = E == 2 ? 1 : 2;
    constexpr int SE = E == 0 ? 1 : E == 1 ? 4 : 16, SP = P == 0 ? 1 : 4, SQ = Q == 1 ? 4 : 16;
    const int combo = (e >> 2) & 3, t = e & 3, sp = combo & 1, sq = combo >> 1;
    int o[3];
    o[E] = 0; o[P] = sp ? 1 : -1; o[Q] = sq ? 1 : -1;
    const int ns = snb[nb_index<3>(o[0], o[1], o[2])];
    if (ns < 0) return;
    const int srcl = t * SE + (sp ? 0 : 3) * SP + (sq ? 0 : 3) * SQ;
    R a[3][3][3];
    load_tcoef<R>(src, (int64_t)ns * T + srcl, h3xyz, a);
    const int cP = sp ? -1 : 1, cQ = sq ? -1 : 1;
    R ge[3];
    edge_eval<E, R>(a, R(cP), R(cQ), ge);
    const int base = (sp ? 3 : 0) * SP + (sq ? 3 : 0) * SQ;
#pragma unroll
    for (int ce = -1; ce <= 1; ++ce) {
        const int le = t + ce;
        if ((unsigned)le > 3u) continue;
        int c[3];
        c[E] = ce; c[P] = cP; c[Q] = cQ;
        fb[kidx(c[0], c[1], c[2]) * T + base + le * SE] = ge[ce + 1];
    }
}

// own push + halo of one tile (all 64 threads of the tile group call it)
template <typename R>
__device__ __forceinline__ void stream_push(const FieldsT<R>& src, R* fb, const int* snb, int64_t cell,
                                            int lc, bool valid, R h3xyz) {
    constexpr int T = 64;
    const int l[3] = {lc & 3, (lc >> 2) & 3, (lc >> 4) & 3};
    if (valid) {
        R a[3][3][3], g[3][3][3];
        load_tcoef<R>(src, cell, h3xyz, a);
        recon_all<R>(a, g);
        bool okm[3], okp[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) { okm[q] = l[q] > 0; okp[q] = l[q] < 3; }
#pragma unroll
        for (int cx = -1; cx <= 1; ++cx)
#pragma unroll
            for (int cy = -1; cy <= 1; ++cy)
#pragma unroll
                for (int cz = -1; cz <= 1; ++cz) {
                    const bool in = (cx < 0 ? okm[0] : cx > 0 ? okp[0] : true) &&
                                    (cy < 0 ? okm[1] : cy > 0 ? okp[1] : true) &&
                                    (cz < 0 ? okm[2] : cz > 0 ? okp[2] : true);
                    if (in) fb[kidx(cx, cy, cz) * T + lc + cx + 4 * cy + 16 * cz] = g[cx + 1][cy + 1][cz + 1];
                }
        // ---- halo faces: 96 cells; warp-uniform normal axis per round
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int f = lc + 64 * r;
            if (f >= 96) break;
            const int A = f >> 5;
            if (A == 0) face_body<0, R>(src, fb, snb, f, h3xyz);
            else if (A == 1) face_body<1, R>(src, fb, snb, f, h3xyz);
            else face_body<2, R>(src, fb, snb, f, h3xyz);
        }
        // ---- halo edges: 48 cells (free axis E, 4 sign combos, 4 positions)
        if (lc < 48) {
            const int E = lc >> 4;
            if (E == 0) edge_body<0, R>(src, fb, snb, lc, h3xyz);
            else if (E == 1) edge_body<1, R>(src, fb, snb, lc, h3xyz);
            else edge_body<2, R>(src, fb, snb, lc, h3xyz);
        } else if (lc < 56) {
            // ---- halo corners: 8 cells, one population each
            const int k = lc - 48, sx = k & 1, sy = (k >> 1) & 1, sz = k >> 2;
            const int ns = snb[nb_index<3>(sx ? 1 : -1, sy ? 1 : -1, sz ? 1 : -1)];
            if (ns >= 0) {
                load_tcoef<R>(src, (int64_t)ns * T + (sx ? 0 : 3) + 4 * (sy ? 0 : 3) + 16 * (sz ? 0 : 3),
                              h3xyz, a);
                const int cx = sx ? -1 : 1, cy = sy ? -1 : 1, cz = sz ? -1 : 1;
                const R gc = corner_eval<R>(a, R(cx), R(cy), R(cz));
                const int dir = kidx(cx, cy, cz);
                fb[dir * T + (sx ? 3 : 0) + 4 * (sy ? 3 : 0) + 16 * (sz ? 3 : 0)] = gc;
            }
        }
    }
}

// pull the 27 incoming populations of a cell and form the bare moments;
// special cells replace bounce-back / self-source directions by their own
template <typename R>
__device__ __forceinline__ void stream_pull(const FieldsT<R>& src, const R* fb, int64_t cell, int lc,
                                            bool special, uint64_t mask, R h3xyz, R& dr, R (&mm)[3],
                                            R (&pi)[6]) {
    constexpr int T = 64;
    R g[3][3][3];
#pragma unroll
    for (int cx = -1; cx <= 1; ++cx)
#pragma unroll
        for (int cy = -1; cy <= 1; ++cy)
#pragma unroll
            for (int cz = -1; cz <= 1; ++cz) g[cx + 1][cy + 1][cz + 1] = fb[kidx(cx, cy, cz) * T + lc];
    if (special) {
        R a[3][3][3], own[3][3][3];
        load_tcoef<R>(src, cell, h3xyz, a);
        recon_all<R>(a, own);
#pragma unroll
        for (int cx = -1; cx <= 1; ++cx)
#pragma unroll
            for (int cy = -1; cy <= 1; ++cy)
#pragma unroll
                for (int cz = -1; cz <= 1; ++cz) {
                    constexpr int dummy = 0; (void)dummy;
                    const int I = dir3(cx, cy, cz);
                    if ((mask >> I) & 1ull) g[cx + 1][cy + 1][cz + 1] = own[1 - cx][1 - cy][1 - cz];
                    else if ((mask >> (32 + I)) & 1ull) g[cx + 1][cy + 1][cz + 1] = own[cx + 1][cy + 1][cz + 1];
                }
    }
    moments_of<R>(g, dr, mm, pi);
}

}  // namespace tp

// mode 0 fused stream+collide+bc, 1 stream only, 2 collide+bc of dst's bare
// moments, 3 collide only (collide_kernel), 4 boundaries only (boundary_kernel)
#ifndef LEVEL_TPC3
#define LEVEL_TPC3 2
#endif
template <int D, typename R> struct LevelCfg {
    static constexpr int TPC = D == 2 ? 8 : (sizeof(R) == 4 ? LEVEL_TPC3 : 1);   // tiles per CTA
    static constexpr int THREADS = TPC * Geo<D>::T;
};

#ifndef LEVEL_MINB
#define LEVEL_MINB (16 / LEVEL_TPC3)      // 1024 resident threads per SM (64 registers, 8 B of stack):
                                          // C4 level-0 stream 0.794 -> 0.773 ms against 7 CTAs at 72
                                          // registers; 6 CTAs: 0.84 (tools/lib_ab.sh)
#endif
template <int D, typename R, int MODE>
__global__ void __launch_bounds__(LevelCfg<D, R>::THREADS,
                                  (D == 3 && sizeof(R) == 4 && (MODE <= 1 || MODE == 5)) ? LEVEL_MINB : 1)
level_kernel(const StepArgs A) {
    constexpr int T = Geo<D>::T, Q = Geo<D>::Q, NS = Geo<D>::NS, NM = Geo<D>::NM;
    constexpr int TPC = LevelCfg<D, R>::TPC;
    constexpr int HB = HaloTable<D>::HB, NCO = CoefSlots<D>::N;
    __shared__ R fbuf_all[TPC][Q * T];
    // halo coefficient staging: 2D only (3D evaluates its halo in registers)
    constexpr bool STREAM = MODE <= 1 || MODE == 5;      // pull-stream first
    constexpr bool HC = STREAM && D == 2;
    __shared__ R hcoef_all[HC ? TPC : 1][HC ? NCO * HB : 1];
    __shared__ int snb_all[TPC][Geo<D>::NB];

    const int grp = threadIdx.x / T, lc = threadIdx.x % T;
    (void)hcoef_all;
    const int tile = A.lv.first + blockIdx.x * TPC + grp;
    const bool valid = tile < live_tiles(A.lv);
    R* fb = fbuf_all[grp];
    int* snb = snb_all[grp];
    const FieldsT<R> src = fields_of<R>(A.src), dst = fields_of<R>(A.dst);
    const R h3xyz = R(A.cp.h3_xyz);

    if (STREAM && valid && lc < Geo<D>::NB) snb[lc] = A.lv.nbr[(int64_t)tile * Geo<D>::NB + lc];

    const int64_t cell = (int64_t)tile * T + lc;
    int l[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    uint8_t cf = MLBM_CF_ACTIVE, tf = MLBM_TF_PLAIN;
    int gx[3] = {0, 0, 0};
    if (valid) {
        tf = A.lv.tile_flags[tile];
        cf = (tf & MLBM_TF_PLAIN) ? (uint8_t)MLBM_CF_ACTIVE : A.lv.cell_flags[cell];
#pragma unroll
        for (int a = 0; a < D; ++a) gx[a] = A.lv.tile_xyz[tile * 3 + a] * 4 + l[a];
    }
    // modes 2-4 read dst's moments (and the force / eps rows): issued before
    // the block vote so their latency overlaps it (the collide was
    // latency-bound: 18 long-scoreboard stalls per issue)
    R pre[STREAM ? 1 : NM + D + 1];
    if constexpr (!STREAM) {
        if (valid) {
#pragma unroll
            for (int k = 0; k < NM; ++k) pre[k] = dst.at(k, cell);
            if (MODE != 4 && A.cp.force_mode != 0) {
#pragma unroll
                for (int a = 0; a < D; ++a) pre[NM + a] = dst.at(fi_f<D>(a), cell);
            }
            if (MODE != 4 && A.cp.tau_mode == 1) pre[NM + D] = dst.at(fi_eps<D>(), cell);
        }
    }
    const int any_bc = __syncthreads_or(valid && (tf & MLBM_TF_BC));
    const bool active = cf & MLBM_CF_ACTIVE;
    // boundary_kernel touches the outlet / inlet layers only (block-uniform)
    if constexpr (MODE == 4) {
        if (!any_bc) return;
    }

    R dr, mm[D], pi[NS];
    if constexpr (STREAM && D == 3) {
        // eps / phi ride along to the write tree: fetch them now so the
        // loads overlap the stream instead of stalling the epilogue
        R eps_c = R(0), phi_c = R(0);
        if (MODE == 1 && valid) { eps_c = src.at(fi_eps<D>(), cell); phi_c = src.at(fi_phi<D>(), cell); }
        tp::stream_push<R>(src, fb, snb, cell, lc, valid, h3xyz);
        __syncthreads();
        dr = R(0);
#pragma unroll
        for (int a = 0; a < D; ++a) mm[a] = R(0);
#pragma unroll
        for (int k = 0; k < NS; ++k) pi[k] = R(0);
        if (valid) {
            const bool special = cf & MLBM_CF_SPECIAL;
            R mm3[3], pi6[6];
            tp::stream_pull<R>(src, fb, cell, lc, special, special ? A.lv.dir_masks[cell] : 0ull, h3xyz,
                               dr, mm3, pi6);
#pragma unroll
            for (int a = 0; a < D; ++a) mm[a] = mm3[a];
#pragma unroll
            for (int k = 0; k < NS; ++k) pi[k] = pi6[k];
        }
        if constexpr (MODE == 1) {
            if (valid) {
                dst.at(0, cell) = dr;
#pragma unroll
                for (int a = 0; a < D; ++a) dst.at(1 + a, cell) = mm[a];
#pragma unroll
                for (int k = 0; k < NS; ++k) dst.at(1 + D + k, cell) = pi[k];
                dst.at(fi_eps<D>(), cell) = eps_c;
                dst.at(fi_phi<D>(), cell) = phi_c;
            }
            return;
        }
    } else if constexpr (STREAM) {
        Coef<D, R> own;
        if (valid) {
            R m[NM];
            load_moments<D, R>(src, cell, m);
            make_coef<D, R>(m, h3xyz, own);
            push_pairs<D, R>(own, fb, lc, l);
            fb[lc] = R(wdir<D>(0)) * even_part<D, 0>(own);
            halo_stage<D, R>(src, hcoef_all[grp], snb, lc, h3xyz);
        }
        __syncthreads();
        if (valid) halo_items<D, R>(fb, hcoef_all[grp], snb, lc);
        __syncthreads();
        dr = R(0);
#pragma unroll
        for (int a = 0; a < D; ++a) mm[a] = R(0);
#pragma unroll
        for (int k = 0; k < NS; ++k) pi[k] = R(0);
        if (valid) {
            const bool special = cf & MLBM_CF_SPECIAL;
            if (special) pull_all<D, R, true>(fb, lc, A.lv.dir_masks[cell], own, dr, mm, pi);
            else pull_all<D, R, false>(fb, lc, 0ull, own, dr, mm, pi);
        }
        if constexpr (MODE == 1) {
            if (valid) {
                dst.at(0, cell) = dr;
#pragma unroll
                for (int a = 0; a < D; ++a) dst.at(1 + a, cell) = mm[a];
#pragma unroll
                for (int k = 0; k < NS; ++k) dst.at(1 + D + k, cell) = pi[k];
                dst.at(fi_eps<D>(), cell) = src.at(fi_eps<D>(), cell);
                dst.at(fi_phi<D>(), cell) = src.at(fi_phi<D>(), cell);
            }
            return;
        }
    } else {   // MODE 2, 3, 4 read the bare (2, 3) or collided (4) moments of dst
        if (valid) {
            dr = pre[0];
#pragma unroll
            for (int a = 0; a < D; ++a) mm[a] = pre[1 + a];
#pragma unroll
            for (int k = 0; k < NS; ++k) pi[k] = pre[1 + D + k];
        }
    }

    // mode 5: every cell's eps (raw eta, the read tree's phi) staged per tile
    // for the exchange's grad eps (in-tile neighbours from shared memory)
    __shared__ R seps_all[MODE == 5 ? TPC : 1][MODE == 5 ? T : 1];
    if constexpr (MODE == 5) {
        if (valid)
            seps_all[grp][lc] = eps_of<D, R>((const R*)A.ex.ras, A.ex.rs, fields_of<R>(A.ex.r_tree), cell,
                                             R(A.ex.eps_min));
        __syncthreads();
    }

    // ---- collide (solver.py:394-453) -------------------------------------
    R out[NM];
    if (MODE == 4 && valid) {
        out[0] = dr;
#pragma unroll
        for (int a = 0; a < D; ++a) out[1 + a] = mm[a];
#pragma unroll
        for (int k = 0; k < NS; ++k) out[1 + D + k] = pi[k];
    }
    R eps5 = R(1);
    if (MODE != 4 && valid) {
        const R rho = R(1) + dr;
        if (active && !(rho > R(0) && isfinite((double)rho)))
            report_error(A.err, MLBM_ERR_DENSITY, A.lv.level, gx[0], gx[1], gx[2]);
        R F[D];
        if constexpr (MODE == 5) {
            // the coupling hook between stream and collide (coupling.py:403-446):
            // fractions, drag, grad eps, mixture force and the MPM grid update of
            // this cell from its bare post-stream moments (in registers)
            R u5[D];
#pragma unroll
            for (int a = 0; a < D; ++a) u5[a] = mm[a] / rho;
            exchange_cell<D, R>(A.ex, cell, gx, rho, u5, F, eps5, seps_all[grp]);
        } else if (A.cp.force_mode == 0) {
            const R sc = R(1 << A.lv.level);
#pragma unroll
            for (int a = 0; a < D; ++a) F[a] = rho * (R(A.cp.gravity[a]) * sc);
        } else {
#pragma unroll
            for (int a = 0; a < D; ++a) {
                if constexpr (STREAM) F[a] = dst.at(fi_f<D>(a), cell);
                else F[a] = pre[NM + a];
            }
        }
        R eps_d = R(1);
        if (MODE != 5 && A.cp.tau_mode == 1) {
            if constexpr (STREAM) eps_d = dst.at(fi_eps<D>(), cell);
            else eps_d = pre[NM + D];
        }
        const R tau = MODE == 5 ? eps5 * R(A.cp.tau0)
                    : A.cp.tau_mode == 0 ? R(A.cp.tau)
                    : A.cp.tau_mode == 1 ? eps_d * R(A.cp.tau0)
                                         : ((const R*)A.cp.tau_ptr)[cell];
        const R inv_rho = R(1) / rho;
        R us[D];
#pragma unroll
        for (int a = 0; a < D; ++a) us[a] = (mm[a] + R(0.5) * F[a]) * inv_rho;
        const R inv_tau = R(1) / tau;
        const R fcoef = (R(2) * tau - R(1)) / (R(2) * tau) * inv_rho;
        out[0] = dr;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const int a = s_a<D>(k), b = s_b<D>(k);
            out[1 + D + k] = (R(1) - inv_tau) * (pi[k] * inv_rho) + inv_tau * us[a] * us[b] +
                             fcoef * (F[a] * us[b] + F[b] * us[a]);
        }
#pragma unroll
        for (int a = 0; a < D; ++a) out[1 + a] = us[a] + R(0.5) * F[a] * inv_rho;
        if (!active) {
#pragma unroll
            for (int k = 0; k < NM; ++k) out[k] = src.at(k, cell);
        } else {
            bool bad = false;
#pragma unroll
            for (int a = 0; a < D; ++a) bad |= !isfinite((double)out[1 + a]);
            if (bad) report_error(A.err, MLBM_ERR_VELOCITY, A.lv.level, gx[0], gx[1], gx[2]);
        }
    }

    // ---- boundaries (solver.py:460-481), face order x-,x+,y-,y+,z-,z+ ------
    if (MODE != 3 && any_bc) {   // block-uniform
        __syncthreads();
        R* mb = fb;   // reuse: [NM][T]
        if (valid) {
#pragma unroll
            for (int k = 0; k < NM; ++k) mb[k * T + lc] = out[k];
        }
        __syncthreads();
        const bool bct = valid && (tf & MLBM_TF_BC);
        for (int face = 0; face < 2 * D; ++face) {
            const int kind = A.bc.face[face];
            if (kind != MLBM_FACE_OUTLET) continue;   // uniform
            const int axis = face >> 1, side = face & 1;
            const int edge = side == 0 ? 0 : A.lv.cells[axis] - 1;
            R nv[NM];
            bool on = bct && gx[axis] == edge;
            if (on) {
                const int inner = lc + (side == 0 ? 1 : -1) * (axis == 0 ? 1 : axis == 1 ? 4 : 16);
                const R sgn = side == 0 ? R(-1) : R(1);
                R un = sgn * mb[(1 + axis) * T + inner];
                un = un > R(0) ? un : R(0);
                un = un < R(1) ? un : R(1);
#pragma unroll
                for (int k = 0; k < NM; ++k) {
                    const R v = mb[k * T + lc];
                    nv[k] = v - un * (v - mb[k * T + inner]);
                }
            }
            __syncthreads();
            if (on) {
#pragma unroll
                for (int k = 0; k < NM; ++k) mb[k * T + lc] = nv[k];
            }
            __syncthreads();
        }
        if (A.bc.face[0] == MLBM_FACE_LOG_INLET && bct && gx[0] == 0) {
            const double ypos = (double)gx[1] * (double)(1 << A.lv.level);
            const double arg = 1.0 + A.bc.inlet_beta * (ypos - A.bc.inlet_y0);
            const double uxv = ypos >= A.bc.inlet_y0 ? A.bc.inlet_u0 * log(arg > 1.0 ? arg : 1.0) : 0.0;
            mb[lc] = R(A.bc.rho0 - 1.0);
#pragma unroll
            for (int a = 0; a < D; ++a) mb[(1 + a) * T + lc] = a == 0 ? R(uxv) : R(0);
#pragma unroll
            for (int k = 0; k < NS; ++k) mb[(1 + D + k) * T + lc] = k == 0 ? R(uxv * uxv) : R(0);
        }
        __syncthreads();
        if (valid) {
#pragma unroll
            for (int k = 0; k < NM; ++k) out[k] = mb[k * T + lc];
        }
    }

    if (valid && (MODE != 4 || (tf & MLBM_TF_BC))) {
#pragma unroll
        for (int k = 0; k < NM; ++k) dst.at(k, cell) = out[k];
        if constexpr (MODE == 5) {
            dst.at(fi_phi<D>(), cell) = src.at(fi_phi<D>(), cell);   // eps: written by the exchange
        } else if ((MODE == 0 || !active) && MODE != 4) {
            dst.at(fi_eps<D>(), cell) = src.at(fi_eps<D>(), cell);
            dst.at(fi_phi<D>(), cell) = src.at(fi_phi<D>(), cell);
        }
    }
}

template <int D, typename R>
int launch_level(const StepArgs& a, int mode, cudaStream_t s) {
    constexpr int TPC = LevelCfg<D, R>::TPC, NT = LevelCfg<D, R>::THREADS;
    const int blocks = (a.lv.n_tiles - a.lv.first + TPC - 1) / TPC;
    if (blocks == 0) return 0;
    switch (mode) {
    case 0: level_kernel<D, R, 0><<<blocks, NT, 0, s>>>(a); break;
    case 1: level_kernel<D, R, 1><<<blocks, NT, 0, s>>>(a); break;
    case 2: level_kernel<D, R, 2><<<blocks, NT, 0, s>>>(a); break;
    case 3: level_kernel<D, R, 3><<<blocks, NT, 0, s>>>(a); break;
    case 4: level_kernel<D, R, 4><<<blocks, NT, 0, s>>>(a); break;
    default: level_kernel<D, R, 5><<<blocks, NT, 0, s>>>(a); break;
    }
    return launch_status(1);
}

// ---------------------------------------------------------------------------
// One target per 16-lane group, lane q < n_m + 2 interpolates field q: the
// 2^D gathers of all fields of a target are in flight at once (the per-target
// loop of 12 x 8 dependent-address loads was latency-bound at ~12 % warps
// active); the S rescale takes u from lanes 1..D of the group by shuffles.
template <int D, typename R>
__global__ void __launch_bounds__(128) downward_kernel(int n, const int32_t* __restrict__ n_dev,
                                                       const int32_t* __restrict__ targets,
                                                       const int32_t* __restrict__ srcs,
                                                       FieldsT<R> olda, FieldsT<R> newa, FieldsT<R> dst,
                                                       int step, R kappa) {
    // one thread per target cell: consecutive targets of a warp read each
    // row at neighbouring coarse cells and write it at neighbouring fine cells
    // (coalesced), where a 16-lane group per target touched 16 rows of one
    // cell per instruction (one sector per lane: l1tex-bound, 0.4 ms per C4
    // launch)
    constexpr int NC = Geo<D>::NC, T = Geo<D>::T, NM = Geo<D>::NM, NS = Geo<D>::NS;
    constexpr int NV = NM + 2;   // moments + eps + phi
    const int live = n_dev ? __ldg(n_dev) : n;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < live; j += gridDim.x * blockDim.x) {
        const int tgt = targets[j];
        const int lc = tgt % T;
        const int par[3] = {lc & 1, (lc >> 2) & 1, (lc >> 4) & 1};
        int sk[NC];
        R wk[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            sk[k] = __ldg(&srcs[(int64_t)j * NC + k]);
            R w = R(1);
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int o = (k >> a) & 1;
                const R fr = par[a] ? R(0.5) : R(0);
                w *= o ? fr : R(1) - fr;
            }
            wk[k] = w;
        }
        R v[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int fk = q < NM ? q : (q == NM ? fi_eps<D>() : fi_phi<D>());
            R val = R(0);
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                if (sk[k] < 0) continue;
                R x = olda.at(fk, sk[k]);
                if (step == 2) x = R(0.5) * (x + newa.at(fk, sk[k]));
                val += x * wk[k];
            }
            v[q] = val;
        }
        // S rescale: v_S = kappa (v_S - u_a u_b) + u_a u_b
#pragma unroll
        for (int k = 0; k < NS; ++k) {
            const R eq = v[1 + s_a<D>(k)] * v[1 + s_b<D>(k)];
            v[1 + D + k] = kappa * (v[1 + D + k] - eq) + eq;
        }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const int fk = q < NM ? q : (q == NM ? fi_eps<D>() : fi_phi<D>());
            dst.at(fk, tgt) = v[q];
        }
    }
}

template <int D, typename R>
__global__ void upward_kernel(int n, const int32_t* __restrict__ n_dev, const int32_t* __restrict__ targets,
                              const int32_t* __restrict__ srcs, FieldsT<R> fine,
                              FieldsT<R> dst, int average, R kappa) {
    constexpr int NC = Geo<D>::NC, NS = Geo<D>::NS;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= (n_dev ? __ldg(n_dev) : n)) return;
    const int tgt = targets[j];
    constexpr int NV = Geo<D>::NM + 2;
    R v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int fk = q < Geo<D>::NM ? q : (q == Geo<D>::NM ? fi_eps<D>() : fi_phi<D>());
        if (average) {
            R acc = R(0);
#pragma unroll
            for (int k = 0; k < NC; ++k) acc += fine.at(fk, srcs[(int64_t)j * NC + k]);
            v[q] = acc / R(NC);
        } else {
            v[q] = fine.at(fk, srcs[(int64_t)j * NC]);
        }
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const R eq = v[1 + s_a<D>(k)] * v[1 + s_b<D>(k)];
        v[1 + D + k] = kappa * (v[1 + D + k] - eq) + eq;
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        const int fk = q < Geo<D>::NM ? q : (q == Geo<D>::NM ? fi_eps<D>() : fi_phi<D>());
        dst.at(fk, tgt) = v[q];
    }
}

}  // namespace mlbm

using namespace mlbm;

extern "C" int mlbm_level_step(const mlbm_level_t* lv, mlbm_fields_t src, mlbm_fields_t dst,
                               int32_t dtype, int32_t mode, const mlbm_collide_t* cp,
                               const mlbm_bc_t* bc, mlbm_error_t* err, void* stream) {
    if (!lv || !cp || !bc || mode < 0 || mode > 4) return -1;
    StepArgs a{*lv, src, dst, *cp, *bc, err, ExchArgs{}};
    cudaStream_t s = as_stream(stream);
    if (lv->dim == 2) return dtype ? launch_level<2, double>(a, mode, s) : launch_level<2, float>(a, mode, s);
    if (lv->dim == 3) return dtype ? launch_level<3, double>(a, mode, s) : launch_level<3, float>(a, mode, s);
    return -1;
}

extern "C" int mlbm_downward(int32_t dim, int32_t n, const int32_t* n_dev, const int32_t* targets,
                             const int32_t* src,
                             const int32_t* tile_xyz, mlbm_fields_t olda, mlbm_fields_t newa,
                             mlbm_fields_t dst, int32_t dtype, int32_t step, double kappa,
                             void* stream) {
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    static int sms = 0;
    if (!sms) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev); }
    const int B = 128;
    const int G = (int)std::min<int64_t>(((int64_t)n + B - 1) / B, (int64_t)sms * 16);
    (void)tile_xyz;
#define DOWN(D, R) downward_kernel<D, R><<<G, B, 0, s>>>(n, n_dev, targets, src, \
        fields_of<R>(olda), fields_of<R>(newa), fields_of<R>(dst), step, R(kappa))
    if (dim == 2) { if (dtype) DOWN(2, double); else DOWN(2, float); }
    else if (dim == 3) { if (dtype) DOWN(3, double); else DOWN(3, float); }
    else return -1;
#undef DOWN
    return launch_status(1);
}

extern "C" int mlbm_upward(int32_t dim, int32_t n, const int32_t* n_dev, const int32_t* targets,
                           const int32_t* src,
                           mlbm_fields_t fine, mlbm_fields_t dst, int32_t dtype,
                           int32_t average, double kappa, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int B = 128, G = (n + B - 1) / B;
#define UP(D, R) upward_kernel<D, R><<<G, B, 0, s>>>(n, n_dev, targets, src, fields_of<R>(fine), \
        fields_of<R>(dst), average, R(kappa))
    if (dim == 2) { if (dtype) UP(2, double); else UP(2, float); }
    else if (dim == 3) { if (dtype) UP(3, double); else UP(3, float); }
    else return -1;
#undef UP
    return launch_status(1);
}

extern "C" int mlbm_level0_coupled(const mlbm_level_t* lv, mlbm_fields_t src, mlbm_fields_t dst,
                                   mlbm_fields_t tree0, mlbm_fields_t tree1, int32_t dtype,
                                   const mlbm_collide_t* cp, const mlbm_bc_t* bc, void* ras, int64_t rs,
                                   double eps_min, double nu, double d_p, double re_min, double dt,
                                   double rho0, const double* g_fluid, const double* g_sed,
                                   const int32_t* faces, double floor_friction, mlbm_error_t* err,
                                   void* stream) {
    if (!lv || !cp || !bc || lv->level != 0) return -1;
    StepArgs a{*lv, src, dst, *cp, *bc, err, ExchArgs{}};
    ExchArgs& A = a.ex;
    A.lv = *lv; A.w_tree = dst; A.r_tree = src; A.tree0 = tree0; A.tree1 = tree1;
    A.ras = ras; A.rs = rs; A.eps_min = eps_min; A.nu = nu; A.d_p = d_p; A.re_min = re_min;
    A.dt = dt; A.rho0 = rho0;
    for (int q = 0; q < 3; ++q) { A.g_fluid[q] = g_fluid[q]; A.g_sed[q] = g_sed[q]; }
    for (int f = 0; f < 6; ++f) A.face[f] = faces[f];
    A.floor_friction = floor_friction;
    A.mode = 1;
    cudaStream_t s = as_stream(stream);
    if (lv->dim == 2) return dtype ? launch_level<2, double>(a, 5, s) : launch_level<2, float>(a, 5, s);
    if (lv->dim == 3) return dtype ? launch_level<3, double>(a, 5, s) : launch_level<3, float>(a, 5, s);
    return -1;
}
