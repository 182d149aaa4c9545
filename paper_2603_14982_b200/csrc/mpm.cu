// MPM sand + fluid-sediment exchange kernels (sm_100a).
//
//   mlbm_p2g        — stencil + Kirchhoff stress + P2G scatter fused with the
//                     fraction rasterisation (granular.py:137-178, 260-310;
//                     coupling.py:96-131)
//   mlbm_exchange   — per level-0 cell: eps, cell velocity, Di Felice drag +
//                     limiter, grad eps, mixture force (written into both
//                     trees), MPM grid update with wall / sticky projection
//                     (coupling.py:134-197, 379-446; granular.py:313-341)
//   mlbm_g2p        — gather, advect, deformation update, SVD, Drucker-Prager
//                     return map (granular.py:344-412)
//   mlbm_stress_raster / mlbm_powder — entrainment source and powder
//                     transport (coupling.py:200-322, 483-498)
//   mlbm_diag_level / mlbm_diag_particles — diagnostics (coupling.py:500-531)
//
// Particle positions are always float64 (sub-cell offsets at x ~ 1e3 need
// ~1e-8 absolute resolution); everything else follows the run dtype.
#include <algorithm>
#include <cstdlib>
#include <cuda_pipeline.h>
#include "common.cuh"
#include "exchange.cuh"

namespace mlbm {

// raster row layout over level-0 cells

// particle row layout (after the float64 positions): v[D] C[D*D] F[D*D] m V0 vc
// TAU: the Kirchhoff stress tau(F) (granular.py:260-279, symmetric, NS rows)
// of the particle's current F, written by G2P from its own decomposition of the
// updated F (and by mlbm_particle_stress when F is set from outside), so P2G and
// the entrainment raster read it instead of re-decomposing F
template <int D> struct PRows {
    static constexpr int V = 0, C = D, F = D + D * D, M = D + 2 * D * D, V0 = M + 1, VC = M + 2,
                         TAU = M + 3, N = M + 3 + D * (D + 1) / 2;
};

struct TopoL0 {
    int32_t cells[3], tiles[3], periodic[3];
    const int32_t* tile_map;
};


// periodic wrap of a coordinate that is almost always within one period of
// the domain (stencil / box nodes): compare-and-add, modulo only otherwise
__device__ __forceinline__ int wrap_near(int c, int n) {
    if (c < 0) c += n;
    else if (c >= n) c -= n;
    if ((unsigned)c >= (unsigned)n) c = ((c % n) + n) % n;
    return c;
}

// coordinates of entry i of a node box with extents ext (x fastest): the
// divisions run in fp32 (i < 2^20, ext <= 2^10: (i + 0.5) / e is at least
// 0.5 / e away from an integer, far above the reciprocal's rounding error)
template <int D>
__device__ __forceinline__ void box_coord(int i, const int (&lo)[3], const int (&ext)[3], int (&c)[3]) {
    c[0] = c[1] = c[2] = 0;
    int r = i;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        if (a == D - 1) { c[a] = lo[a] + r; break; }
        const int q = (int)(((float)r + 0.5f) * __frcp_rn((float)ext[a]));
        c[a] = lo[a] + (r - q * ext[a]);
        r = q;
    }
}

template <int D>
__device__ __forceinline__ int64_t node_index(const TopoL0& t, int (&c)[3], bool& bad) {
    for (int a = 0; a < D; ++a) {
        if (t.periodic[a]) c[a] = wrap_near(c[a], t.cells[a]);
        else if (c[a] < 0 || c[a] >= t.cells[a]) { bad = true; return -1; }
    }
    const int s = t.tile_map[g3(t.tiles, c[0] >> 2, c[1] >> 2, D == 3 ? c[2] >> 2 : 0)];
    if (s < 0) { bad = true; return -1; }
    return (int64_t)s * Geo<D>::T + local_of<D>(c[0] & 3, c[1] & 3, c[2] & 3);
}

// -- small dense linear algebra --------------------------------------------
template <typename R> __device__ __forceinline__ R rsqrt_(R x) { return R(1) / sqrt(x); }

// 2x2 closed form (granular.py:181-213)
template <typename R>
__device__ void svd2(const R (&F)[4], R (&U)[4], R (&s)[2], R (&V)[4]) {
    const R a = F[0], b = F[1], c = F[2], d = F[3];
    const R e = R(0.5) * (a + d), f = R(0.5) * (a - d), g = R(0.5) * (c + b), h = R(0.5) * (c - b);
    const R q = hypot(e, h), r = hypot(f, g);
    const R a1 = atan2(g, f), a2 = atan2(h, e);
    const R tu = R(0.5) * (a1 + a2), tv = R(0.5) * (a1 - a2);
    const R cu = cos(tu), su = sin(tu), cv = cos(tv), sv = sin(tv);
    U[0] = cu; U[1] = -su; U[2] = su; U[3] = cu;
    V[0] = cv; V[1] = -sv; V[2] = sv; V[3] = cv;
    s[0] = q + r;
    s[1] = q - r;
}

// 3x3 rotation-variant SVD: Jacobi on F^T F, Gram-Schmidt for U,
// det U = det V = +1, sign on the smallest singular value.
template <typename R>
__device__ void svd3(const R (&F)[9], R (&U)[9], R (&s)[3], R (&V)[9]) {
    R A[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            R acc = R(0);
            for (int k = 0; k < 3; ++k) acc += F[k * 3 + i] * F[k * 3 + j];
            A[i * 3 + j] = acc;
        }
    for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? R(1) : R(0);
    for (int sweep = 0; sweep < 10; ++sweep) {
        const R off = A[1] * A[1] + A[2] * A[2] + A[5] * A[5];
        const R dia = A[0] * A[0] + A[4] * A[4] + A[8] * A[8];
        if (!(off > dia * R(sizeof(R) == 8 ? 1e-34 : 1e-16))) break;
        for (int pq = 0; pq < 3; ++pq) {
            const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2;
            const R apq = A[p * 3 + q];
            if (apq == R(0)) continue;
            const R theta = (A[q * 3 + q] - A[p * 3 + p]) / (R(2) * apq);
            const R t = (theta >= R(0) ? R(1) : R(-1)) / (fabs(theta) + sqrt(theta * theta + R(1)));
            const R c = rsqrt_(t * t + R(1)), sn = t * c;
            // A <- J^T A J
            for (int k = 0; k < 3; ++k) {
                const R akp = A[k * 3 + p], akq = A[k * 3 + q];
                A[k * 3 + p] = c * akp - sn * akq;
                A[k * 3 + q] = sn * akp + c * akq;
            }
            for (int k = 0; k < 3; ++k) {
                const R apk = A[p * 3 + k], aqk = A[q * 3 + k];
                A[p * 3 + k] = c * apk - sn * aqk;
                A[q * 3 + k] = sn * apk + c * aqk;
            }
            for (int k = 0; k < 3; ++k) {
                const R vkp = V[k * 3 + p], vkq = V[k * 3 + q];
                V[k * 3 + p] = c * vkp - sn * vkq;
                V[k * 3 + q] = sn * vkp + c * vkq;
            }
        }
    }
    // sort eigenvalues descending (columns of V)
    R lam[3] = {A[0], A[4], A[8]};
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2 - i; ++j)
            if (lam[j] < lam[j + 1]) {
                const R tl = lam[j]; lam[j] = lam[j + 1]; lam[j + 1] = tl;
                for (int k = 0; k < 3; ++k) {
                    const R tv = V[k * 3 + j]; V[k * 3 + j] = V[k * 3 + j + 1]; V[k * 3 + j + 1] = tv;
                }
            }
    // det V = +1
    const R detV = V[0] * (V[4] * V[8] - V[5] * V[7]) - V[1] * (V[3] * V[8] - V[5] * V[6]) +
                   V[2] * (V[3] * V[7] - V[4] * V[6]);
    if (detV < R(0)) for (int k = 0; k < 3; ++k) V[k * 3 + 2] = -V[k * 3 + 2];
    // B = F V
    R B[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            R acc = R(0);
            for (int k = 0; k < 3; ++k) acc += F[i * 3 + k] * V[k * 3 + j];
            B[i * 3 + j] = acc;
        }
    // u0
    R n0 = sqrt(B[0] * B[0] + B[3] * B[3] + B[6] * B[6]);
    R u0[3];
    if (n0 > R(0)) { u0[0] = B[0] / n0; u0[1] = B[3] / n0; u0[2] = B[6] / n0; }
    else { u0[0] = R(1); u0[1] = R(0); u0[2] = R(0); }
    R b1[3] = {B[1], B[4], B[7]};
    R d01 = u0[0] * b1[0] + u0[1] * b1[1] + u0[2] * b1[2];
    for (int k = 0; k < 3; ++k) b1[k] -= d01 * u0[k];
    R n1 = sqrt(b1[0] * b1[0] + b1[1] * b1[1] + b1[2] * b1[2]);
    R u1[3];
    if (n1 > R(0) && n1 > n0 * R(sizeof(R) == 8 ? 1e-14 : 1e-6)) {
        for (int k = 0; k < 3; ++k) u1[k] = b1[k] / n1;
    } else {
        // any unit vector orthogonal to u0
        R e[3] = {R(0), R(0), R(0)};
        int m = fabs(u0[0]) < fabs(u0[1]) ? (fabs(u0[0]) < fabs(u0[2]) ? 0 : 2) : (fabs(u0[1]) < fabs(u0[2]) ? 1 : 2);
        e[m] = R(1);
        R dd = u0[0] * e[0] + u0[1] * e[1] + u0[2] * e[2];
        for (int k = 0; k < 3; ++k) e[k] -= dd * u0[k];
        R ne = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
        for (int k = 0; k < 3; ++k) u1[k] = e[k] / ne;
    }
    R u2[3] = {u0[1] * u1[2] - u0[2] * u1[1], u0[2] * u1[0] - u0[0] * u1[2], u0[0] * u1[1] - u0[1] * u1[0]};
    for (int k = 0; k < 3; ++k) { U[k * 3 + 0] = u0[k]; U[k * 3 + 1] = u1[k]; U[k * 3 + 2] = u2[k]; }
    s[0] = u0[0] * B[0] + u0[1] * B[3] + u0[2] * B[6];
    s[1] = u1[0] * B[1] + u1[1] * B[4] + u1[2] * B[7];
    s[2] = u2[0] * B[2] + u2[1] * B[5] + u2[2] * B[8];
}

template <int D, typename R>
__device__ __forceinline__ void svd(const R (&F)[D * D], R (&U)[D * D], R (&s)[D], R (&V)[D * D]) {
    if constexpr (D == 2) svd2<R>(F, U, s, V); else svd3<R>(F, U, s, V);
}

// Cyclic Jacobi on a symmetric 3x3 (entries a00 a01 a02 a11 a12 a22), only the
// touched entries updated.  Returns eigenvalues lam and eigenvectors as the
// columns of Q (Q diag(lam) Q^T = a).
template <typename R>
__device__ __forceinline__ void sym_eig3(R a00, R a01, R a02, R a11, R a12, R a22, R (&lam)[3],
                                         R (&Q)[9]) {
    R A[3][3] = {{a00, a01, a02}, {a01, a11, a12}, {a02, a12, a22}};
#pragma unroll
    for (int i = 0; i < 9; ++i) Q[i] = (i % 4 == 0) ? R(1) : R(0);
#ifndef MLBM_JACOBI_TOL32
#define MLBM_JACOBI_TOL32 1e-13   // off-diagonal ~3e-7 relative: fp32 round-off level
#endif
    const R tol = R(sizeof(R) == 8 ? 1e-32 : MLBM_JACOBI_TOL32);
#pragma unroll 1
    for (int sweep = 0; sweep < 8; ++sweep) {
        const R off = A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2];
        const R dia = A[0][0] * A[0][0] + A[1][1] * A[1][1] + A[2][2] * A[2][2];
        if (!(off > dia * tol)) break;
#pragma unroll
        for (int pq = 0; pq < 3; ++pq) {
            const int p = pq == 2 ? 1 : 0, q = pq == 0 ? 1 : 2, r = 3 - p - q;
            const R apq = A[p][q];
            if (apq == R(0)) continue;
            R t, c;
            if constexpr (sizeof(R) == 4) {
                // fp32: the angle only steers the sweep (apq is zeroed
                // explicitly), so it takes the approximate divide / square
                // root; the rotation itself stays orthogonal to round-off:
                // c = 1 / sqrt(1 + t^2) by rsqrt + one Newton step, s = t c
                const float theta = __fdividef(A[q][q] - A[p][p], 2.f * apq);
                const float at = fabsf(theta);
                t = at < 1e18f ? __fdividef(1.f, at + __fsqrt_rz(fmaf(theta, theta, 1.f))) : 0.5f / at;
                t = theta >= 0.f ? t : -t;
                const float x = fmaf(t, t, 1.f);
                const float r0 = rsqrtf(x);
                c = r0 * fmaf(-0.5f * x * r0, r0, 1.5f);
            } else {
                const R theta = (A[q][q] - A[p][p]) / (R(2) * apq);
                t = (theta >= R(0) ? R(1) : R(-1)) / (fabs(theta) + sqrt(theta * theta + R(1)));
                c = R(1) / sqrt(t * t + R(1));
            }
            const R sn = t * c;
            A[p][p] -= t * apq;
            A[q][q] += t * apq;
            A[p][q] = A[q][p] = R(0);
            const R arp = A[r][p], arq = A[r][q];
            A[r][p] = A[p][r] = c * arp - sn * arq;
            A[r][q] = A[q][r] = sn * arp + c * arq;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const R vkp = Q[k * 3 + p], vkq = Q[k * 3 + q];
                Q[k * 3 + p] = c * vkp - sn * vkq;
                Q[k * 3 + q] = sn * vkp + c * vkq;
            }
        }
    }
    lam[0] = A[0][0];
    lam[1] = A[1][1];
    lam[2] = A[2][2];
}

// principal stretches of F from b = F F^T (left vectors U = Q); the sign of
// det F goes on the smallest value (the rotation-variant SVD convention)
template <typename R>
__device__ __forceinline__ void left_stretch3(const R (&F)[9], R (&U)[9], R (&s)[3]) {
    const R b00 = F[0] * F[0] + F[1] * F[1] + F[2] * F[2];
    const R b01 = F[0] * F[3] + F[1] * F[4] + F[2] * F[5];
    const R b02 = F[0] * F[6] + F[1] * F[7] + F[2] * F[8];
    const R b11 = F[3] * F[3] + F[4] * F[4] + F[5] * F[5];
    const R b12 = F[3] * F[6] + F[4] * F[7] + F[5] * F[8];
    const R b22 = F[6] * F[6] + F[7] * F[7] + F[8] * F[8];
    R lam[3];
    sym_eig3<R>(b00, b01, b02, b11, b12, b22, lam, U);
    int imin = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        s[i] = sqrt(lam[i] > R(0) ? lam[i] : R(0));
        if (lam[i] < lam[imin]) imin = i;
    }
    const R det = F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
                  F[2] * (F[3] * F[7] - F[4] * F[6]);
    if (det < R(0)) s[imin] = -s[imin];
}

struct MatParams {
    double lam, mu, alpha, floor_friction;
    double kdg2, kdg3;      // (d lam + 2 mu) / (2 mu) for d = 2, 3 (host-computed)
    int snow;               // 0 Drucker-Prager sand, 1 NACC snow
    double M, beta, xi, alpha_soft;
};
static inline MatParams mat_params(double lam, double mu, double alpha, const mlbm_snow_t* sn = nullptr) {
    MatParams m{lam, mu, alpha, 0.0, mu != 0.0 ? (2.0 * lam + 2.0 * mu) / (2.0 * mu) : 0.0,
                mu != 0.0 ? (3.0 * lam + 2.0 * mu) / (2.0 * mu) : 0.0, 0, 0.0, 0.0, 0.0, 0.0};
    if (sn) { m.snow = 1; m.M = sn->M; m.beta = sn->beta; m.xi = sn->xi; m.alpha_soft = sn->alpha_soft; }
    return m;
}

// NACC return map + the paper's softening law in principal log-strain space
// (Hencky elasticity, p = -kappa tr e, s = 2 mu dev e): the device statement of
// oracle/mpm.py:nacc_return_map (parity unpinned).  qs: the
// hardening state (q >= 0, or -(q + 1) once the particle has cracked)
template <int D, typename R>
__device__ __forceinline__ void nacc_return(R (&e)[D], R& qs, const MatParams& mp) {
    const R kappa = R(mp.lam) + R(2.0 * mp.mu / D);
    const bool cracked = qs < R(0);
    const R q = cracked ? -qs - R(1) : qs;
    const R beta = cracked ? R(0) : R(mp.beta);
    const R p0 = kappa * (R(1e-5) + sinh(R(mp.xi) * (q > R(0) ? q : R(0))));
    R ev = R(0);
#pragma unroll
    for (int a = 0; a < D; ++a) ev += e[a];
    R eh[D], n2 = R(0);
#pragma unroll
    for (int a = 0; a < D; ++a) { eh[a] = e[a] - ev / R(D); n2 += eh[a] * eh[a]; }
    const R sn = R(2.0 * mp.mu) * sqrt(n2);
    const R cs = sqrt(R(6 - D) / R(2));
    const R p_tr = -kappa * ev, q_tr = cs * sn;
    const R M2 = R(mp.M * mp.M);
    const R yp = M2 * (p_tr + beta * p0) * (p_tr - p0);
    const R y = (R(1) + R(2) * beta) * q_tr * q_tr + yp;
    R dlogjp = R(0);
    const R ytol = R(1e-12) * fmax(p0 * p0 * M2, R(1e-30));
    if (p_tr > p0) {                          // compressive tip
        const R ev1 = -p0 / kappa;
#pragma unroll
        for (int a = 0; a < D; ++a) e[a] = ev1 / R(D);
        dlogjp = ev - ev1;
    } else if (p_tr < -beta * p0) {           // tensile tip
        const R ev2 = beta * p0 / kappa;
#pragma unroll
        for (int a = 0; a < D; ++a) e[a] = ev2 / R(D);
        dlogjp = ev - ev2;
    } else if (y > ytol) {                    // deviatoric return at fixed p
        const R snew = sqrt(fmax(-yp, R(0)) / (R(1) + R(2) * beta)) / cs;
        const R scale = sn > R(0) ? snew / sn : R(0);
#pragma unroll
        for (int a = 0; a < D; ++a) e[a] = eh[a] * scale + ev / R(D);
        // hardening: the surface point on the line from the centre (p_c, 0)
        const R pc = (R(1) - beta) * p0 / R(2);
        R d0 = pc - p_tr, d1 = -q_tr;
        R nr = sqrt(d0 * d0 + d1 * d1);
        nr = nr > R(0) ? nr : R(1);
        d0 /= nr;
        d1 /= nr;
        R A = M2 * d0 * d0 + (R(1) + R(2) * beta) * d1 * d1;
        const R B = M2 * d0 * (R(2) * pc - p0 + beta * p0);
        const R C = M2 * (pc + beta * p0) * (pc - p0);
        const R disc = sqrt(fmax(B * B - R(4) * A * C, R(0)));
        A = A > R(0) ? A : R(1);
        const R p1 = pc + (-B + disc) / (R(2) * A) * d0;
        const R p2 = pc + (-B - disc) / (R(2) * A) * d0;
        const R px = (p_tr - pc) * (p1 - pc) > R(0) ? p1 : p2;
        dlogjp = ev + px / kappa;
    }
    R qn = q + (cracked ? R(1) : -R(mp.alpha_soft)) * (-dlogjp);
    const bool newly = !cracked && qn <= R(0);
    if (cracked || newly) qn = qn > R(0) ? qn : R(0);
    if (newly) qn = R(0);
    qs = (cracked || newly) ? -qn - R(1) : qn;
}

// tau = U diag(2 mu eps + lam tr) U^T  (granular.py:260-279)
template <int D, typename R>
__device__ void kirchhoff(const R (&F)[D * D], const MatParams& mp, R (&tau)[D * D]) {
    R U[D * D], s[D];
    if constexpr (D == 3) {
        left_stretch3<R>(F, U, s);
    } else {
        R V[D * D];
        svd<D, R>(F, U, s, V);
    }
    R e[D], tr = R(0);
#pragma unroll
    for (int a = 0; a < D; ++a) { e[a] = log(s[a] > R(1e-12) ? s[a] : R(1e-12)); tr += e[a]; }
    R tp[D];
#pragma unroll
    for (int a = 0; a < D; ++a) tp[a] = R(2.0 * mp.mu) * e[a] + R(mp.lam) * tr;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            R acc = R(0);
#pragma unroll
            for (int k = 0; k < D; ++k) acc += U[i * D + k] * tp[k] * U[j * D + k];
            tau[i * D + j] = acc;
        }
}

// the stored Kirchhoff stress of particle p as a full D x D matrix
template <int D, typename R>
__device__ __forceinline__ void load_tau(const R* pp, int64_t ps, int p, R (&tau)[D * D]) {
#pragma unroll
    for (int k = 0; k < Geo<D>::NS; ++k) {
        const R t = pp[(PRows<D>::TAU + k) * ps + p];
        tau[s_a<D>(k) * D + s_b<D>(k)] = t;
        tau[s_b<D>(k) * D + s_a<D>(k)] = t;
    }
}

// tau = U diag(2 mu e + lam tr e) U^T from left vectors U and log stretches e
template <int D, typename R>
__device__ __forceinline__ void store_tau(R* pw, int64_t ps, int p, const R (&U)[D * D], const R (&e)[D],
                                          const MatParams& mp) {
    R tr = R(0);
#pragma unroll
    for (int a = 0; a < D; ++a) tr += e[a];
    R tp[D];
#pragma unroll
    for (int a = 0; a < D; ++a) tp[a] = R(2.0 * mp.mu) * e[a] + R(mp.lam) * tr;
#pragma unroll
    for (int k = 0; k < Geo<D>::NS; ++k) {
        const int i = s_a<D>(k), j = s_b<D>(k);
        R acc = R(0);
#pragma unroll
        for (int q = 0; q < D; ++q) acc += U[i * D + q] * tp[q] * U[j * D + q];
        pw[(PRows<D>::TAU + k) * ps + p] = acc;
    }
}

// B-spline stencil of one particle (granular.py:137-178)
template <int D, typename R> struct Stencil {
    int base[3];
    R w[D][3], dw[D][3];
    R frac[D];
};
template <int D, typename R>
__device__ __forceinline__ void make_stencil(const double (&x)[D], Stencil<D, R>& st) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const double b = floor(x[a] - 0.5);
        st.base[a] = (int)b;
        const R f = R(x[a] - b);
        st.frac[a] = f;
        st.w[a][0] = R(0.5) * (R(1.5) - f) * (R(1.5) - f);
        st.w[a][1] = R(0.75) - (f - R(1)) * (f - R(1));
        st.w[a][2] = R(0.5) * (f - R(0.5)) * (f - R(0.5));
        st.dw[a][0] = f - R(1.5);
        st.dw[a][1] = R(-2) * (f - R(1));
        st.dw[a][2] = f - R(0.5);
    }
    if (D == 2) st.base[2] = 0;
}

// register-resident pick of a per-axis stencil value (a dynamic index into
// the w / dw arrays would force them into local memory)
template <typename R>
__device__ __forceinline__ R sel3(const R (&v)[3], int o) {
    return o == 0 ? v[0] : (o == 1 ? v[1] : v[2]);
}

struct PartArgs {
    int32_t dim, n;
    const double* x;     // [D][n]
    double* xw;          // writable positions (g2p)
    void* p;             // [PRows::N][n] of R
    int64_t ps;          // stride of p and x
    void* pw;            // g2p output rows (may alias p)
    const int32_t* pid;  // g2p: particle ids in / out (may be null)
    int32_t* pidw;
    // g2p: the level-0 seed tiles of the next adapt pass (adapt.py:54-65) from
    // the new positions, and the count of particles outside level-0 leaves of
    // the current topology (adapt.py:374-389); null: not written
    uint8_t* seeds;
    const uint8_t* kind0;
    int32_t* nonleaf;
};

template <typename R> __device__ __forceinline__ void aadd(R* a, R v) { atomicAdd(a, v); }

// ---------------------------------------------------------------------------
template <int D, typename R>
__global__ void __launch_bounds__(128) k_p2g(PartArgs P, TopoL0 t0, MatParams mp, R* ras, int64_t rs,
                                             mlbm_error_t* err) {
    constexpr int K = Geo<D>::K;
    using RW = Rows<D>;
    using PR = PRows<D>;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P.n) return;
    const R* pp = (const R*)P.p;
    double x[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = P.x[a * P.ps + p];
    Stencil<D, R> st;
    make_stencil<D, R>(x, st);
    R v[D], C[D * D];
#pragma unroll
    for (int a = 0; a < D; ++a) v[a] = pp[(PR::V + a) * P.ps + p];
#pragma unroll
    for (int k = 0; k < D * D; ++k) C[k] = pp[(PR::C + k) * P.ps + p];
    const R m = pp[PR::M * P.ps + p], V0 = pp[PR::V0 * P.ps + p];
    R tau[D * D];
    load_tau<D, R>(pp, P.ps, p, tau);
    const R ap = D == 2 ? R(2) * sqrt(V0 / R(3.14159265358979323846))
                        : R(3.14159265358979323846) * pow(R(3) * V0 / (R(4) * R(3.14159265358979323846)), R(2.0 / 3.0));
    bool bad = false;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const int o[3] = {k % 3, (k / 3) % 3, k / 9};
        int c[3] = {st.base[0] + o[0], st.base[1] + o[1], D == 3 ? st.base[2] + o[2] : 0};
        const int64_t ni = node_index<D>(t0, c, bad);
        if (ni < 0) continue;
        R w = R(1), gr[D];
#pragma unroll
        for (int a = 0; a < D; ++a) { w *= sel3<R>(st.w[a], o[a]); gr[a] = R(1); }
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = 0; b < D; ++b) gr[b] *= (a == b) ? sel3<R>(st.dw[a], o[a]) : sel3<R>(st.w[a], o[a]);
        R dpos[D];
#pragma unroll
        for (int a = 0; a < D; ++a) dpos[a] = R((double)(st.base[a] + o[a]) - x[a]);
        const R wm = w * m;
        aadd(&ras[RW::MASS * rs + ni], wm);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            R aff = v[a];
#pragma unroll
            for (int b = 0; b < D; ++b) aff += C[a * D + b] * dpos[b];
            aadd(&ras[(RW::MOM + a) * rs + ni], wm * aff);
            R fa = R(0);
#pragma unroll
            for (int b = 0; b < D; ++b) fa += V0 * tau[a * D + b] * gr[b];
            aadd(&ras[(RW::FINT + a) * rs + ni], -fa);
            aadd(&ras[(RW::VMOM + a) * rs + ni], wm * v[a]);
        }
        aadd(&ras[RW::ETA * rs + ni], w * V0);
        aadd(&ras[RW::AREA * rs + ni], w * ap);
    }
    if (bad) report_error(err, MLBM_ERR_STENCIL, 0, st.base[0], st.base[1], st.base[2]);
}

// ---------------------------------------------------------------------------
#ifndef EXCH_MINB
#define EXCH_MINB 16
#endif
template <int D, typename R>
__global__ void __launch_bounds__(128, sizeof(R) == 4 ? EXCH_MINB : 1) k_exchange(ExchArgs A) {
    constexpr int T = Geo<D>::T;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)live_tiles(A.lv) * T) return;
    const int slot = (int)(c / T), lc = (int)(c % T);
    const int l3[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    int g[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) g[a] = A.lv.tile_xyz[slot * 3 + a] * 4 + l3[a];
    if (A.mode == 1) {
        // the bare post-stream moments of the write tree
        const FieldsT<R> wt = fields_of<R>(A.w_tree);
        const R rho = R(1) + wt.at(0, c);
        R u[D], force[D], eps;
        for (int a = 0; a < D; ++a) u[a] = wt.at(1 + a, c) / rho;
        exchange_cell<D, R>(A, c, g, rho, u, force, eps);
    } else {
        R fs[D];
        for (int a = 0; a < D; ++a) fs[a] = ((const R*)A.ras)[(Rows<D>::FS + a) * A.rs + c];
        grid_update_cell<D, R>(A, c, g, fs);
    }
}

// ---------------------------------------------------------------------------
// The reference's standalone coupling functions (coupling.py:96-197,379-401)
// as per-cell passes over the level-0 raster, sharing the device functions of
// the fused k_exchange (difelice_cell, limit_drag_cell, grad_cell):
//   FRACTIONS      eta_eff, eps, v_cell from the accumulated P2G rows and phi (a0)
//   DRAG           f_s and rel = u - v_cell from eps, area, rho (a0), u rows
//   LIMIT          the smooth limiter on the FS rows (rho a0, u rows, dt)
//   GRAD_EPS       out rows = central differences of a0 (or of the EPS row)
//   MIXTURE_FORCE  GRAD rows = (rho - rho0)/eps grad eps, out = GRAD + rho g - f_s
struct CoupleArgs {
    mlbm_level_t lv;
    void* ras;
    int64_t rs;
    const void* a0;
    const void* u;
    int64_t us;
    void* out;
    int64_t os;
    double eps_min, nu, d_p, re_min, dt, rho0, g[3];
    int32_t op;
};

template <int D, typename R>
__global__ void k_coupling_op(CoupleArgs A) {
    constexpr int T = Geo<D>::T;
    using RW = Rows<D>;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)live_tiles(A.lv) * T) return;
    R* ras = (R*)A.ras;
    const int64_t rs = A.rs;
    const R* a0 = (const R*)A.a0;
    const R* u = (const R*)A.u;
    R* out = (R*)A.out;
    if (A.op == MLBM_COUPLE_FRACTIONS) {
        const R mass = ras[RW::MASS * rs + c];
        const R phi = a0 ? a0[c] : R(0);
        R eta = ras[RW::ETA * rs + c] - phi;
        eta = eta > R(0) ? eta : R(0);
        R e = R(1) - eta - phi;
        e = e < R(A.eps_min) ? R(A.eps_min) : (e > R(1) ? R(1) : e);
        ras[RW::ETAE * rs + c] = eta;
        ras[RW::EPS * rs + c] = e;
        for (int a = 0; a < D; ++a)
            ras[(RW::VMOM + a) * rs + c] = mass > R(0) ? ras[(RW::VMOM + a) * rs + c] / mass : R(0);
        return;
    }
    if (A.op == MLBM_COUPLE_DRAG || A.op == MLBM_COUPLE_LIMIT) {
        const R rho = a0[c];
        R rel[D], sp2 = R(0);
        for (int a = 0; a < D; ++a) {
            rel[a] = u[a * A.us + c] - ras[(RW::VMOM + a) * rs + c];
            sp2 += rel[a] * rel[a];
        }
        const R speed = sqrt(sp2);
        R fs[D];
        if (A.op == MLBM_COUPLE_DRAG) {
            difelice_cell<D, R>(ras[RW::EPS * rs + c], rho, rel, speed, ras[RW::AREA * rs + c], R(A.d_p),
                                R(A.nu), R(A.re_min), fs);
            for (int a = 0; a < D; ++a) ras[(RW::REL + a) * rs + c] = rel[a];
        } else {
            for (int a = 0; a < D; ++a) fs[a] = ras[(RW::FS + a) * rs + c];
            limit_drag_cell<D, R>(fs, rho, ras[RW::MASS * rs + c], speed, R(A.dt));
        }
        for (int a = 0; a < D; ++a) ras[(RW::FS + a) * rs + c] = fs[a];
        return;
    }
    const int slot = (int)(c / T), lc = (int)(c % T);
    const int l3[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    int g[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) g[a] = A.lv.tile_xyz[slot * 3 + a] * 4 + l3[a];
    const R* fld = (A.op == MLBM_COUPLE_GRAD_EPS && a0) ? a0 : ras + RW::EPS * rs;
    R grad[D];
    grad_cell<D, R>(A.lv, g, c, [&](int64_t ni) { return fld[ni]; }, grad);
    if (A.op == MLBM_COUPLE_GRAD_EPS) {
        for (int a = 0; a < D; ++a) out[a * A.os + c] = grad[a];
        return;
    }
    const R rho = a0[c];
    const R coefg = (rho - R(A.rho0)) / ras[RW::EPS * rs + c];
    for (int a = 0; a < D; ++a) {
        const R gt = coefg * grad[a];
        ras[(RW::GRAD + a) * rs + c] = gt;
        out[a * A.os + c] = gt + rho * R(A.g[a]) - ras[(RW::FS + a) * rs + c];
    }
}

// granular.stencil (granular.py:137-178) per particle: flat node index, weight,
// weight gradient and node offset for each of the 3^D nodes (node k: offsets
// k % 3, (k / 3) % 3, k / 9, the reference's _OFF_X/_OFF_Y order); a node
// outside a non-periodic domain or not stored at level 0 is a stencil fault
template <int D, typename R>
__global__ void k_stencil(int n, const double* __restrict__ x, int64_t ps, TopoL0 t0, int32_t* idx,
                          R* w, R* grad, R* dpos, int64_t os, mlbm_error_t* err) {
    constexpr int K = Geo<D>::K;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    double xp[3] = {0, 0, 0}, f[3] = {0, 0, 0}, wa[3][3], da[3][3];
    int base[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) {
        xp[a] = x[a * ps + p];
        const double b = floor(xp[a] - 0.5);
        base[a] = (int)b;
        f[a] = xp[a] - b;
        wa[a][0] = 0.5 * (1.5 - f[a]) * (1.5 - f[a]);
        wa[a][1] = 0.75 - (f[a] - 1.0) * (f[a] - 1.0);
        wa[a][2] = 0.5 * (f[a] - 0.5) * (f[a] - 0.5);
        da[a][0] = f[a] - 1.5;
        da[a][1] = -2.0 * (f[a] - 1.0);
        da[a][2] = f[a] - 0.5;
    }
    bool bad = false;
    for (int k = 0; k < K; ++k) {
        const int o[3] = {k % 3, (k / 3) % 3, D == 3 ? k / 9 : 0};
        int c[3] = {0, 0, 0};
        for (int a = 0; a < D; ++a) c[a] = base[a] + o[a];
        const int64_t ni = node_index<D>(t0, c, bad);
        idx[(int64_t)k * os + p] = (int32_t)ni;
        double ww = 1.0;
        for (int a = 0; a < D; ++a) ww *= wa[a][o[a]];
        w[(int64_t)k * os + p] = R(ww);
        for (int b = 0; b < D; ++b) {
            double gb = da[b][o[b]];
            for (int e = 0; e < D; ++e) if (e != b) gb *= wa[e][o[e]];
            grad[((int64_t)b * K + k) * os + p] = R(gb);
            dpos[((int64_t)b * K + k) * os + p] = R((double)(base[b] + o[b]) - xp[b]);
        }
    }
    if (bad) report_error(err, MLBM_ERR_STENCIL, 0, base[0], base[1], base[2]);
}

// Kirchhoff stress rows from F for every particle (granular.py:260-279): the
// initial state and any F set from outside G2P
template <int D, typename R>
__global__ void k_particle_stress(int n, R* pp, int64_t ps, MatParams mp) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    R F[D * D], tau[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) F[k] = pp[(PRows<D>::F + k) * ps + p];
    kirchhoff<D, R>(F, mp, tau);
#pragma unroll
    for (int k = 0; k < Geo<D>::NS; ++k) pp[(PRows<D>::TAU + k) * ps + p] = tau[s_a<D>(k) * D + s_b<D>(k)];
}

// ---------------------------------------------------------------------------
// fp32: 7 resident CTAs per SM (72 registers, 80 B of stack) — C4 G2P 4.07 ms
// against 4.13 at 8 CTAs (64 registers) and 4.20 at 6 (80 registers)
// (tools/lib_ab.sh); 5 CTAs at 96 registers were 17 % slower on C3
#ifndef G2P_MINB
#define G2P_MINB 7
#endif
#ifndef G2P_BT
#define G2P_BT 128      // particles (threads) per block: one node box per block
#endif
#ifndef G2P_EARLY
#define G2P_EARLY 0     // 1: ride-along rows loaded before the node-box staging (measured +4 % on C4)
#endif
#ifndef G2P_ASYNC
#define G2P_ASYNC 1     // ride-along rows copied to shared memory asynchronously (cp.async) before the staging
#endif
// MAT: 0 elastic (plastic = 0), 1 Drucker-Prager sand, 2 NACC snow — one
// instantiation per model, so the kernel holds only its own return map (G2P
// stalled on instruction fetch: 2.7 no-instruction stalls per issue with
// both return maps in one kernel)
template <int D, typename R, int MAT>
__global__ void __launch_bounds__(G2P_BT, sizeof(R) == 4 ? G2P_MINB : 1) k_g2p(PartArgs P, TopoL0 t0, MatParams mp, const R* ras, int64_t rs,
                                             double dt, int32_t* clamped, mlbm_error_t* err) {
    constexpr bool plastic = MAT != 0;
    constexpr int K = Geo<D>::K;
    using RW = Rows<D>;
    using PR = PRows<D>;
    constexpr int MAXB = sizeof(R) == 4 ? 512 : 256;
    // grid velocities of the block's node box staged in shared memory (sorted
    // particles: the 128 particles of a block span a few cells); absent nodes
    // hold NaN so a particle touching one reports the stencil error
    __shared__ R svel[D][MAXB];
    __shared__ int s_lo[3], s_hi[3];
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = p < P.n;
    const R* pp = (const R*)P.p;
    R* pw = (R*)P.pw;
#if G2P_ASYNC && !G2P_EARLY
    // the rows that only ride along (F, vc, m, V0, id) are copied into shared
    // memory by cp.async (LDGSTS) now: their latency overlaps the node-box
    // staging and its barriers without holding registers (the register form,
    // G2P_EARLY, measured slower at the 64-register bound)
    constexpr int NPRE = D * D + 3;
    __shared__ R spre[NPRE][G2P_BT];
    __shared__ int32_t spid[G2P_BT];
    const bool copy_rows = pw != pp;
    if (live) {
#pragma unroll
        for (int k = 0; k < D * D; ++k)
            __pipeline_memcpy_async(&spre[k][threadIdx.x], &pp[(PR::F + k) * P.ps + p], sizeof(R));
        __pipeline_memcpy_async(&spre[D * D][threadIdx.x], &pp[PR::VC * P.ps + p], sizeof(R));
        if (copy_rows) {
            __pipeline_memcpy_async(&spre[D * D + 1][threadIdx.x], &pp[PR::M * P.ps + p], sizeof(R));
            __pipeline_memcpy_async(&spre[D * D + 2][threadIdx.x], &pp[PR::V0 * P.ps + p], sizeof(R));
        }
        if (P.pidw) __pipeline_memcpy_async(&spid[threadIdx.x], &P.pid[p], sizeof(int32_t));
    }
    __pipeline_commit();
#endif
    double x[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = live ? P.x[a * P.ps + p] : 0.5 * t0.cells[a];
    Stencil<D, R> st;
    make_stencil<D, R>(x, st);
#if G2P_EARLY
    // rows that only ride along (F, vc, m, V0, id): issued before the node-box
    // staging so their latency overlaps it and the gather
    R Fpre[D * D];
    const bool copy_rows = pw != pp;
#pragma unroll
    for (int k = 0; k < D * D; ++k) Fpre[k] = live ? pp[(PR::F + k) * P.ps + p] : R(1);
    const R vc_pre = live ? pp[PR::VC * P.ps + p] : R(0);
    const R m_pre = copy_rows && live ? pp[PR::M * P.ps + p] : R(0);
    const R v0_pre = copy_rows && live ? pp[PR::V0 * P.ps + p] : R(0);
    const int32_t id_pre = P.pidw && live ? P.pid[p] : 0;
#endif
    if (threadIdx.x < 3) { s_lo[threadIdx.x] = 0x7fffffff; s_hi[threadIdx.x] = -0x7fffffff; }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int l2 = __reduce_min_sync(0xffffffffu, live ? st.base[a] : 0x7fffffff);
        const int h2 = __reduce_max_sync(0xffffffffu, live ? st.base[a] + 2 : -0x7fffffff);
        if ((threadIdx.x & 31) == 0 && l2 <= h2) { atomicMin(&s_lo[a], l2); atomicMax(&s_hi[a], h2); }
    }
    __syncthreads();
    int blo[3] = {0, 0, 0}, bext[3] = {1, 1, 1}, nbox = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) { blo[a] = s_lo[a]; bext[a] = s_hi[a] - s_lo[a] + 1; nbox *= bext[a]; }
    const bool use_box = nbox > 0 && nbox <= MAXB;      // block-uniform
    if (use_box) {
        for (int i = threadIdx.x; i < nbox; i += blockDim.x) {
            int c[3];
            box_coord<D>(i, blo, bext, c);
            bool nb = false;
            const int64_t ni = node_index<D>(t0, c, nb);
#pragma unroll
            for (int a = 0; a < D; ++a) svel[a][i] = ni >= 0 ? ras[(RW::VEL + a) * rs + ni] : R(NAN);
        }
    }
    __syncthreads();
    if (!live) return;
#if G2P_ASYNC && !G2P_EARLY
    __pipeline_wait_prior(0);                 // this thread's own copies (no other thread reads them)
    R Fpre[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) Fpre[k] = spre[k][threadIdx.x];
    const R vc_pre = spre[D * D][threadIdx.x];
    const R m_pre = copy_rows ? spre[D * D + 1][threadIdx.x] : R(0);
    const R v0_pre = copy_rows ? spre[D * D + 2][threadIdx.x] : R(0);
    const int32_t id_pre = P.pidw ? spid[threadIdx.x] : 0;
#elif !G2P_EARLY
    // rows that only ride along (F, vc, m, V0, id): loaded now so their
    // latency overlaps the gather instead of stalling the epilogue
    R Fpre[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) Fpre[k] = pp[(PR::F + k) * P.ps + p];
    const R vc_pre = pp[PR::VC * P.ps + p];
    const bool copy_rows = pw != pp;
    const R m_pre = copy_rows ? pp[PR::M * P.ps + p] : R(0);
    const R v0_pre = copy_rows ? pp[PR::V0 * P.ps + p] : R(0);
    const int32_t id_pre = P.pidw ? P.pid[p] : 0;
#endif
    R v[D], B[D * D];
#pragma unroll
    for (int a = 0; a < D; ++a) v[a] = R(0);
#pragma unroll
    for (int k = 0; k < D * D; ++k) B[k] = R(0);
    bool bad = false;
    if (use_box) {
        R dp[D][3];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int o = 0; o < 3; ++o) dp[a][o] = R(o) - st.frac[a];
        int pb = 0, oy[3] = {0, 0, 0}, oz[3] = {0, 0, 0};
        {
            int m = 1;
#pragma unroll
            for (int a = 0; a < D; ++a) { pb += (st.base[a] - blo[a]) * m; m *= bext[a]; }
#pragma unroll
            for (int o = 0; o < 3; ++o) { oy[o] = o * bext[0]; oz[o] = D == 3 ? o * bext[0] * bext[1] : 0; }
        }
        if constexpr (D == 3) {
            // sum factorisation over the tensor-product stencil: z, then y,
            // then x contractions of the 27 node velocities (v and the APIC
            // moments B = sum w v dx^T: 93 instead of 135 FMAs per component)
            R wz[3], wdz[3], wy[3], wdy[3], wx[3], wdx[3];
#pragma unroll
            for (int o = 0; o < 3; ++o) {
                wx[o] = st.w[0][o]; wdx[o] = st.w[0][o] * dp[0][o];
                wy[o] = st.w[1][o]; wdy[o] = st.w[1][o] * dp[1][o];
                wz[o] = st.w[2][o]; wdz[o] = st.w[2][o] * dp[2][o];
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                R T0[3], Ty[3], Tz[3];
#pragma unroll
                for (int ox = 0; ox < 3; ++ox) {
                    R t0 = R(0), ty = R(0), tz = R(0);
#pragma unroll
                    for (int oyy = 0; oyy < 3; ++oyy) {
                        const int b0 = pb + ox + oy[oyy];
                        const R g0 = svel[a][b0 + oz[0]], g1 = svel[a][b0 + oz[1]], g2 = svel[a][b0 + oz[2]];
                        const R s0 = wz[0] * g0 + wz[1] * g1 + wz[2] * g2;
                        const R s1 = wdz[0] * g0 + wdz[1] * g1 + wdz[2] * g2;
                        t0 += wy[oyy] * s0;
                        ty += wdy[oyy] * s0;
                        tz += wy[oyy] * s1;
                    }
                    T0[ox] = t0; Ty[ox] = ty; Tz[ox] = tz;
                }
                v[a] = wx[0] * T0[0] + wx[1] * T0[1] + wx[2] * T0[2];
                B[a * 3 + 0] = wdx[0] * T0[0] + wdx[1] * T0[1] + wdx[2] * T0[2];
                B[a * 3 + 1] = wx[0] * Ty[0] + wx[1] * Ty[1] + wx[2] * Ty[2];
                B[a * 3 + 2] = wx[0] * Tz[0] + wx[1] * Tz[1] + wx[2] * Tz[2];
            }
        } else {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int o[3] = {k % 3, (k / 3) % 3, D == 3 ? k / 9 : 0};
            const int bi = pb + o[0] + oy[o[1]] + oz[o[2]];
            R w = st.w[0][o[0]];
#pragma unroll
            for (int a = 1; a < D; ++a) w *= st.w[a][o[a]];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const R wg = w * svel[a][bi];
                v[a] += wg;
#pragma unroll
                for (int b = 0; b < D; ++b) B[a * D + b] += wg * dp[b][o[b]];
            }
        }
        }
#pragma unroll
        for (int a = 0; a < D; ++a) bad |= isnan((double)v[a]);
    } else {
    // per-axis node coordinates of the 3^D stencil: tile coordinate (-1 when
    // outside a non-periodic box) and in-tile offset; the 27 tile-map reads
    // hit L1 (at most 2^D distinct tiles)
    int tix[3][3], loc[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int o = 0; o < 3; ++o) {
            if (a >= D) { tix[a][o] = 0; loc[a][o] = 0; continue; }
            int c = st.base[a] + o;
            const int nc = t0.cells[a];
            if (t0.periodic[a]) c = c < 0 ? c + nc : (c >= nc ? c - nc : c);
            const bool in = c >= 0 && c < nc;
            tix[a][o] = in ? c >> 2 : -1;
            loc[a][o] = c & 3;
        }
    R dp[D][3];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int o = 0; o < 3; ++o) dp[a][o] = R(o) - st.frac[a];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int o[3] = {k % 3, (k / 3) % 3, D == 3 ? k / 9 : 0};
        const int tx = tix[0][o[0]], ty = tix[1][o[1]], tz = tix[2][o[2]];
        if ((tx | ty | tz) < 0) { bad = true; continue; }
        const int sl = __ldg(&t0.tile_map[((int64_t)tx * t0.tiles[1] + ty) * t0.tiles[2] + tz]);
        if (sl < 0) { bad = true; continue; }
        const int64_t ni = (int64_t)sl * Geo<D>::T + local_of<D>(loc[0][o[0]], loc[1][o[1]], loc[2][o[2]]);
        R w = st.w[0][o[0]];
#pragma unroll
        for (int a = 1; a < D; ++a) w *= st.w[a][o[a]];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const R wg = w * ras[(RW::VEL + a) * rs + ni];
            v[a] += wg;
#pragma unroll
            for (int b = 0; b < D; ++b) B[a * D + b] += wg * dp[b][o[b]];
        }
    }
    }
    if (bad) report_error(err, MLBM_ERR_STENCIL, 0, st.base[0], st.base[1], st.base[2]);
    R C[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) C[k] = R(4) * B[k];
    int ncl = 0;
    double xnew[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double xn = x[a] + dt * (double)v[a];
        const double dim = (double)t0.cells[a];
        if (t0.periodic[a]) {
            xn = fmod(xn, dim);
            if (xn < 0) xn += dim;
            if (xn >= dim) xn -= dim;
        } else {
            if (xn < 2.0 || xn > dim - 2.0) ++ncl;
            xn = xn < 2.0 ? 2.0 : (xn > dim - 2.0 ? dim - 2.0 : xn);
        }
        P.xw[a * P.ps + p] = xn;
        xnew[a] = xn;
        pw[(PR::V + a) * P.ps + p] = v[a];
    }
    if (ncl) atomicAdd(clamped, ncl);
    if (P.seeds) {
        // seeds of the adapt pass that follows (its particle stage reads no
        // positions then): tile of floor(x) // 4 of the new position
        int tc[3] = {0, 0, 0};
        bool bad_x = false;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const double xv = xnew[a];
            const int c = (int)floor(xv);
            if (!(xv == xv) || c < 0 || c >= t0.cells[a]) bad_x = true;
            tc[a] = c >> 2;
        }
        if (bad_x) {
            report_error(err, MLBM_ERR_DOMAIN, 0, tc[0], tc[1], tc[2]);
            atomicAdd(P.nonleaf, 1);
        } else {
            const int64_t g = g3(t0.tiles, tc[0], tc[1], tc[2]);
            P.seeds[g] = 1;
            if (P.kind0[g] != 1) atomicAdd(P.nonleaf, 1);
        }
    }
    {
        R vmax = R(0);
#pragma unroll
        for (int a = 0; a < D; ++a) vmax = fabs(v[a]) > vmax ? fabs(v[a]) : vmax;
        if (!((double)vmax * dt < 0.5)) atomicOr(clamped + 1, 1);   // cfl_check (granular.py:428-432)
    }
    R F[D * D], Fn[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) { F[k] = Fpre[k]; pw[(PR::C + k) * P.ps + p] = C[k]; }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            R acc = R(0);
#pragma unroll
            for (int k = 0; k < D; ++k) acc += ((i == k ? R(1) : R(0)) + R(dt) * C[i * D + k]) * F[k * D + j];
            Fn[i * D + j] = acc;
        }
    if constexpr (plastic) {
        R U[D * D], s[D], V[D * D];
        bool fast = false;
        if constexpr (D == 3) {
            left_stretch3<R>(Fn, U, s);
            fast = fabs(s[0]) > R(1e-6) && fabs(s[1]) > R(1e-6) && fabs(s[2]) > R(1e-6);
        }
        if (!fast) svd<D, R>(Fn, U, s, V);
        const R vc = vc_pre;
        R en[D], se[D];
        if constexpr (MAT == 2) {
            // NACC snow with the paper's softening law; vc is the hardening state
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const R sa = s[a] < R(0.05) ? R(0.05) : (s[a] > R(4) ? R(4) : s[a]);
                en[a] = log(sa);
            }
            R qs = vc;
            nacc_return<D, R>(en, qs, mp);
            pw[PR::VC * P.ps + p] = qs;
#pragma unroll
            for (int a = 0; a < D; ++a) se[a] = exp(en[a]);
        } else {
            R e[D], tr = R(0);
#pragma unroll
            for (int a = 0; a < D; ++a) {
                R sa = s[a] < R(0.05) ? R(0.05) : (s[a] > R(4) ? R(4) : s[a]);
                e[a] = log(sa) + vc / R(D);
                tr += e[a];
            }
            R eh[D], nrm2 = R(0);
#pragma unroll
            for (int a = 0; a < D; ++a) { eh[a] = e[a] - tr / R(D); nrm2 += eh[a] * eh[a]; }
            const R nrm = sqrt(nrm2);
            const R dg = nrm + R(D == 3 ? mp.kdg3 : mp.kdg2) * tr * R(mp.alpha);
            if (tr > R(0)) {
#pragma unroll
                for (int a = 0; a < D; ++a) en[a] = R(0);
            } else if (nrm > R(0) && dg > R(0)) {
                const R sc = dg / nrm;
#pragma unroll
                for (int a = 0; a < D; ++a) en[a] = e[a] - sc * eh[a];
            } else {
#pragma unroll
                for (int a = 0; a < D; ++a) en[a] = e[a];
            }
            R sum = R(0);
#pragma unroll
            for (int a = 0; a < D; ++a) { sum += en[a]; se[a] = exp(en[a]); }
            pw[PR::VC * P.ps + p] = tr - sum;
        }
        // F_new has left vectors U and stretches exp(en): its Kirchhoff stress
        // (what the next P2G would get from an SVD of F_new) is U diag(2 mu en
        // + lam tr en) U^T
        store_tau<D, R>(pw, P.ps, p, U, en, mp);
        if (fast) {
            // F_new = U diag(s_new / s) U^T F  ( = U diag(s_new) V^T )
            R M[D * D], G[D * D];
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    R acc = R(0);
#pragma unroll
                    for (int k = 0; k < D; ++k) acc += U[i * D + k] * (se[k] / s[k]) * U[j * D + k];
                    M[i * D + j] = acc;
                }
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    R acc = R(0);
#pragma unroll
                    for (int k = 0; k < D; ++k) acc += M[i * D + k] * Fn[k * D + j];
                    G[i * D + j] = acc;
                }
#pragma unroll
            for (int k = 0; k < D * D; ++k) Fn[k] = G[k];
        } else {
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    R acc = R(0);
#pragma unroll
                    for (int k = 0; k < D; ++k) acc += U[i * D + k] * se[k] * V[j * D + k];
                    Fn[i * D + j] = acc;
                }
        }
    }
    if constexpr (!plastic) {
        // elastic: decompose the updated F for its stress
        R U[D * D], s[D], e[D];
        if constexpr (D == 3) {
            left_stretch3<R>(Fn, U, s);
        } else {
            R V[D * D];
            svd<D, R>(Fn, U, s, V);
        }
#pragma unroll
        for (int a = 0; a < D; ++a) e[a] = log(s[a] > R(1e-12) ? s[a] : R(1e-12));
        store_tau<D, R>(pw, P.ps, p, U, e, mp);
    }
#pragma unroll
    for (int k = 0; k < D * D; ++k) pw[(PR::F + k) * P.ps + p] = Fn[k];
    if (copy_rows) {
        if (!plastic) pw[PR::VC * P.ps + p] = vc_pre;
        pw[PR::M * P.ps + p] = m_pre;
        pw[PR::V0 * P.ps + p] = v0_pre;
    }
    if (P.pidw) P.pidw[p] = id_pre;
}

// ---------------------------------------------------------------------------
// entrainment stress raster (coupling.py:283-294) with post-G2P positions
template <int D, typename R>
__global__ void k_stress_raster(PartArgs P, TopoL0 t0, MatParams mp, R* ras, int64_t rs, mlbm_error_t* err) {
    constexpr int K = Geo<D>::K, NS = Geo<D>::NS;
    using RW = Rows<D>;
    using PR = PRows<D>;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P.n) return;
    const R* pp = (const R*)P.p;
    double x[D];
    for (int a = 0; a < D; ++a) x[a] = P.x[a * P.ps + p];
    Stencil<D, R> st;
    make_stencil<D, R>(x, st);
    R tau[D * D];
    load_tau<D, R>(pp, P.ps, p, tau);
    const R V0 = pp[PR::V0 * P.ps + p];
    bool bad = false;
    for (int k = 0; k < K; ++k) {
        const int o[3] = {k % 3, (k / 3) % 3, k / 9};
        int c[3] = {st.base[0] + o[0], st.base[1] + o[1], D == 3 ? st.base[2] + o[2] : 0};
        const int64_t ni = node_index<D>(t0, c, bad);
        if (ni < 0) continue;
        R w = V0;
        for (int a = 0; a < D; ++a) w *= sel3<R>(st.w[a], o[a]);
        for (int q = 0; q < NS; ++q) aadd(&ras[(RW::SIG + q) * rs + ni], w * tau[s_a<D>(q) * D + s_b<D>(q)]);
    }
    if (bad) report_error(err, MLBM_ERR_STENCIL, 0, st.base[0], st.base[1], st.base[2]);
}

// renormalised multilinear sample of NC level-0 fields at one position
// (coupling.py:200-227); the corner lookups are shared by the NC fields and
// each field's sum runs in the reference's corner order
template <int D, typename R, int NC>
__device__ void sample_lin_n(const R* const (&f)[NC], const double (&pos)[D], const mlbm_level_t& lv,
                             double (&out)[NC]) {
    constexpr int T = Geo<D>::T;
    // per axis: the two corner coordinates (wrapped / clamped), their tile
    // and in-tile parts and weights; the 2^D corners only combine them, and
    // a corner in the same tile as corner 0 reuses its slot (no lookup)
    int tp[3][2] = {{0, 0}, {0, 0}, {0, 0}}, lp[3][2] = {{0, 0}, {0, 0}, {0, 0}};
    double wt[3][2];
    unsigned same = 0u;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const double fl = floor(pos[a]);
        const int b = (int)fl;
        const double fr = pos[a] - fl;
        wt[a][0] = 1.0 - fr;
        wt[a][1] = fr;
#pragma unroll
        for (int o = 0; o < 2; ++o) {
            int v = b + o;
            if (lv.periodic[a]) v = wrap_near(v, lv.cells[a]);
            else v = v < 0 ? 0 : (v >= lv.cells[a] ? lv.cells[a] - 1 : v);
            tp[a][o] = v >> 2;
            lp[a][o] = v & 3;
        }
        if (tp[a][0] == tp[a][1]) same |= 1u << a;
    }
    const int s0 = lv.tile_map[g3(lv.tiles, tp[0][0], tp[1][0], tp[2][0])];
    double acc[NC], ws = 0.0;
#pragma unroll
    for (int q = 0; q < NC; ++q) acc[q] = 0.0;
#pragma unroll
    for (int k = 0; k < (1 << D); ++k) {
        const int ox = k & 1, oy = (k >> 1) & 1, oz = D == 3 ? (k >> 2) & 1 : 0;
        double w = 1.0;
        w *= wt[0][ox];
        w *= wt[1][oy];
        if (D == 3) w *= wt[2][oz];
        const int s = (k & ~(int)same) == 0 ? s0 : lv.tile_map[g3(lv.tiles, tp[0][ox], tp[1][oy], tp[2][oz])];
        if (s < 0) continue;
        const int64_t ni = (int64_t)s * T + local_of<D>(lp[0][ox], lp[1][oy], lp[2][oz]);
#pragma unroll
        for (int q = 0; q < NC; ++q) acc[q] += w * (double)f[q][ni];
        ws += w;
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) out[q] = ws > 0.0 ? (double)R(acc[q] / ws) : (double)R(acc[q]);
}

struct PowderArgs {
    mlbm_level_t lv;
    mlbm_fields_t src, dst;   // last read / write trees of level 0
    void* ras;
    int64_t rs;
    void* tmp;                // [n0] scratch (advected phi)
    double diffusion, sign, dt, entrain, eta_surface;
    int32_t with_source;
    const void* source;       // optional explicit per-cell source (powder_step's `source`)
    const uint8_t* active;    // optional per tile: phi non-zero within its 3^D tile neighbourhood
};

// Face neighbour (axis a, side sgn: +1 / -1) of cell lc of tile slot with the
// coordinate conventions of the level-0 face stencils (coupling.py:300-316):
// periodic axes wrap, other axes clamp (the neighbour of a boundary cell is
// the cell itself); absent tiles -> returns -1.  In-tile neighbours need no
// lookup; the others read one entry of the tile's neighbour table.
template <int D>
__device__ __forceinline__ int64_t face_nbr(const mlbm_level_t& lv, int slot, int lc, int a, int sgn) {
    constexpr int T = Geo<D>::T;
    int l[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    const int la = l[a] + sgn;
    if (la >= 0 && la <= 3) {
        l[a] = la;
        return (int64_t)slot * T + local_of<D>(l[0], l[1], l[2]);
    }
    // leaves the tile: a domain face clamps (non-periodic), else the neighbour tile
    const int ta = lv.tile_xyz[slot * 3 + a] + sgn;
    if (!lv.periodic[a] && (ta < 0 || ta >= lv.tiles[a])) return (int64_t)slot * T + lc;
    int o[3] = {0, 0, 0};
    o[a] = sgn;
    const int ns = lv.nbr[(int64_t)slot * Geo<D>::NB + nb_index<D>(o[0], o[1], o[2])];
    if (ns < 0) return -1;
    l[a] = la & 3;
    return (int64_t)ns * T + local_of<D>(l[0], l[1], l[2]);
}

// Cell at offset o (|o_a| <= 1) from cell lc of tile slot: periodic axes
// wrap, a position outside a non-periodic domain or in an absent tile -> -1
// (the 3^D neighbourhood of the entrainment-surface flags).
template <int D>
__device__ __forceinline__ int64_t cell_nbr(const mlbm_level_t& lv, int slot, int lc, const int (&o)[3]) {
    constexpr int T = Geo<D>::T;
    int l[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    int to[3] = {0, 0, 0};
    bool inside = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int la = l[a] + o[a];
        to[a] = la < 0 ? -1 : (la > 3 ? 1 : 0);
        l[a] = la & 3;
        if (to[a] != 0) {
            inside = false;
            const int ta = lv.tile_xyz[slot * 3 + a] + to[a];
            if (!lv.periodic[a] && (ta < 0 || ta >= lv.tiles[a])) return -1;
        }
    }
    const int ns = inside ? slot : lv.nbr[(int64_t)slot * Geo<D>::NB + nb_index<D>(to[0], to[1], to[2])];
    if (ns < 0) return -1;
    return (int64_t)ns * T + local_of<D>(l[0], l[1], l[2]);
}

// The backtrace of one RK3 step moves less than a tile (|u| dt < 1 cell), so a
// cell whose tile has phi = 0 in all its 3^D neighbour tiles advects exactly 0:
// those cells skip the velocity sampling (the result is bit-identical).
template <int D, typename R>
__global__ void k_phi_tiles(mlbm_level_t lv, mlbm_fields_t src, uint8_t* __restrict__ tflag) {
    constexpr int T = Geo<D>::T;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= live_tiles(lv)) return;
    const FieldsT<R> f = fields_of<R>(src);
    const R* phi = &f.at(fi_phi<D>(), (int64_t)t * T);
    uint8_t nz = 0;
    for (int i = 0; i < T && !nz; ++i) nz = phi[i] != R(0);
    tflag[t] = nz;
}

template <int D>
__global__ void k_phi_region(mlbm_level_t lv, const uint8_t* __restrict__ tflag, uint8_t* __restrict__ active) {
    constexpr int NB = Geo<D>::NB;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= live_tiles(lv)) return;
    uint8_t a = 0;
    for (int k = 0; k < NB && !a; ++k) {
        const int s = lv.nbr[(int64_t)t * NB + k];
        a = s >= 0 ? tflag[s] : 0;
    }
    active[t] = a;
}

template <int D, typename R>
__global__ void k_powder_advect(PowderArgs A) {
    constexpr int T = Geo<D>::T;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)live_tiles(A.lv) * T) return;
    const FieldsT<R> src = fields_of<R>(A.src), dst = fields_of<R>(A.dst);
    const int slot = (int)(c / T), lc = (int)(c % T);
    if (A.active && !A.active[slot]) {       // no powder within reach: exactly 0
        ((R*)A.tmp)[c] = R(0);
        return;
    }
    const int l3[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    double pos[D];
    for (int a = 0; a < D; ++a) pos[a] = (double)(A.lv.tile_xyz[slot * 3 + a] * 4 + l3[a]);
    const R* u[D];
    for (int a = 0; a < D; ++a) u[a] = &dst.at(1 + a, 0);
    double k1[D], k2[D], k3[D], q[D];
    // k1 samples at the cell's own (integer) position: weight 1 on the cell,
    // exact zeros elsewhere, so the renormalised sample is the cell value
    for (int a = 0; a < D; ++a) k1[a] = (double)u[a][c];
    for (int a = 0; a < D; ++a) q[a] = pos[a] - 0.5 * A.dt * k1[a];
    sample_lin_n<D, R, D>(u, q, A.lv, k2);
    for (int a = 0; a < D; ++a) q[a] = pos[a] - 0.75 * A.dt * k2[a];
    sample_lin_n<D, R, D>(u, q, A.lv, k3);
    for (int a = 0; a < D; ++a) q[a] = pos[a] - A.dt * (2.0 * k1[a] + 3.0 * k2[a] + 4.0 * k3[a]) / 9.0;
    const R* ph[1] = {&src.at(fi_phi<D>(), 0)};
    double phv[1];
    sample_lin_n<D, R, 1>(ph, q, A.lv, phv);
    ((R*)A.tmp)[c] = R(phv[0]);
}

// 3D advection with the tile's velocities and phi staged in shared memory:
// one CTA per level-0 tile, the 6^3 cells of the tile and its one-cell halo
// (coordinates wrapped / clamped and looked up exactly as sample_lin_n does)
// loaded once, then every cell's three trilinear samples read shared memory —
// the same corners, weights, order and renormalisation as k_powder_advect, so
// the result is bit-identical.  A sample whose corners leave the halo (a
// backtrace longer than one cell) falls back to sample_lin_n.
template <typename R>
__device__ __forceinline__ bool sample_halo(const R* const (&f)[3], int nc, const uint8_t* pres,
                                            const double (&pos)[3], const int (&h0)[3], double (&out)[3]) {
    int hb[3];
    double wt[3][2];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double fl = floor(pos[a]);
        const double fr = pos[a] - fl;
        wt[a][0] = 1.0 - fr;
        wt[a][1] = fr;
        hb[a] = (int)fl - h0[a];
        if (hb[a] < 0 || hb[a] > 4) return false;
    }
    double acc[3] = {0.0, 0.0, 0.0}, ws = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int ox = k & 1, oy = (k >> 1) & 1, oz = (k >> 2) & 1;
        double w = 1.0;
        w *= wt[0][ox];
        w *= wt[1][oy];
        w *= wt[2][oz];
        const int h = (hb[0] + ox) + 6 * (hb[1] + oy) + 36 * (hb[2] + oz);
        if (!pres[h]) continue;
        for (int q = 0; q < nc; ++q) acc[q] += w * (double)f[q][h];
        ws += w;
    }
    for (int q = 0; q < nc; ++q) out[q] = ws > 0.0 ? (double)R(acc[q] / ws) : (double)R(acc[q]);
    return true;
}

template <typename R>
__global__ void __launch_bounds__(64) k_powder_advect_tile(PowderArgs A) {
    constexpr int T = 64, NH = 216;
    const int slot = blockIdx.x;
    if (slot >= live_tiles(A.lv)) return;
    const int lc = threadIdx.x;
    const int64_t c = (int64_t)slot * T + lc;
    if (A.active && !A.active[slot]) {       // no powder within reach: exactly 0 (block-uniform)
        ((R*)A.tmp)[c] = R(0);
        return;
    }
    __shared__ R su[3][NH], sph[NH];
    __shared__ uint8_t spres[NH];
    const FieldsT<R> src = fields_of<R>(A.src), dst = fields_of<R>(A.dst);
    const mlbm_level_t& lv = A.lv;
    int h0[3];                               // global cell of halo index 0
#pragma unroll
    for (int a = 0; a < 3; ++a) h0[a] = lv.tile_xyz[slot * 3 + a] * 4 - 1;
    for (int h = threadIdx.x; h < NH; h += T) {
        int v[3] = {h0[0] + h % 6, h0[1] + (h / 6) % 6, h0[2] + h / 36};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if (lv.periodic[a]) v[a] = wrap_near(v[a], lv.cells[a]);
            else v[a] = v[a] < 0 ? 0 : (v[a] >= lv.cells[a] ? lv.cells[a] - 1 : v[a]);
        }
        const int s = lv.tile_map[g3(lv.tiles, v[0] >> 2, v[1] >> 2, v[2] >> 2)];
        spres[h] = s >= 0;
        if (s >= 0) {
            const int64_t ni = (int64_t)s * T + local_of<3>(v[0] & 3, v[1] & 3, v[2] & 3);
#pragma unroll
            for (int a = 0; a < 3; ++a) su[a][h] = dst.at(1 + a, ni);
            sph[h] = src.at(fi_phi<3>(), ni);
        }
    }
    __syncthreads();
    const int l3[3] = {lc & 3, (lc >> 2) & 3, (lc >> 4) & 3};
    double pos[3];
    for (int a = 0; a < 3; ++a) pos[a] = (double)(h0[a] + 1 + l3[a]);
    const R* u[3] = {su[0], su[1], su[2]};
    const R* ug[3];
    for (int a = 0; a < 3; ++a) ug[a] = &dst.at(1 + a, 0);
    double k1[3], k2[3], k3[3], q[3];
    const int own = (l3[0] + 1) + 6 * (l3[1] + 1) + 36 * (l3[2] + 1);
    for (int a = 0; a < 3; ++a) k1[a] = (double)su[a][own];
    for (int a = 0; a < 3; ++a) q[a] = pos[a] - 0.5 * A.dt * k1[a];
    if (!sample_halo<R>(u, 3, spres, q, h0, k2)) sample_lin_n<3, R, 3>(ug, q, lv, k2);
    for (int a = 0; a < 3; ++a) q[a] = pos[a] - 0.75 * A.dt * k2[a];
    if (!sample_halo<R>(u, 3, spres, q, h0, k3)) sample_lin_n<3, R, 3>(ug, q, lv, k3);
    for (int a = 0; a < 3; ++a) q[a] = pos[a] - A.dt * (2.0 * k1[a] + 3.0 * k2[a] + 4.0 * k3[a]) / 9.0;
    const R* ph[3] = {sph, sph, sph};
    double phv[3];
    if (!sample_halo<R>(ph, 1, spres, q, h0, phv)) {
        const R* pg[1] = {&src.at(fi_phi<3>(), 0)};
        double pv[1];
        sample_lin_n<3, R, 1>(pg, q, lv, pv);
        phv[0] = pv[0];
    }
    ((R*)A.tmp)[c] = R(phv[0]);
}

template <int D, typename R>
__global__ void k_powder_diffuse(PowderArgs A) {
    constexpr int T = Geo<D>::T, NS = Geo<D>::NS;
    using RW = Rows<D>;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= (int64_t)live_tiles(A.lv) * T) return;
    const FieldsT<R> dst = fields_of<R>(A.dst);
    const R* adv = (const R*)A.tmp;
    const R* ras = (const R*)A.ras;
    const int64_t rs = A.rs;
    const int slot = (int)(c / T), lc = (int)(c % T);
    R lap = R(-2 * D) * adv[c];
    bool has_empty = false;
    const R eta_c = A.with_source ? ras[RW::ETAE * rs + c] : R(0);
    // only a cell with 0 < eta < eta_surface can be a source: the others skip
    // the neighbours' eta and their own velocity / stress rows (q = 0 either way)
    const bool cand = A.with_source && eta_c > R(0) && eta_c < R(A.eta_surface);
    for (int a = 0; a < D; ++a)
        for (int sgn = 0; sgn < 2; ++sgn) {
            const int64_t nb = face_nbr<D>(A.lv, slot, lc, a, sgn == 0 ? 1 : -1);
            const int64_t ni = nb >= 0 ? nb : c;
            lap += adv[ni];
            if (cand) {
                if (nb < 0) has_empty = true;
                else if (ras[RW::ETAE * rs + ni] < R(1e-3)) has_empty = true;
            }
        }
    R out = adv[c] + R(A.sign * A.diffusion * A.dt) * lap;
    if (A.with_source) {
        R q = R(0);
        if (cand && has_empty) {
            R sp2 = R(0), v[D];
            for (int a = 0; a < D; ++a) { v[a] = ras[(RW::VMOM + a) * rs + c]; sp2 += v[a] * v[a]; }
            const R speed = sqrt(sp2);
            if (speed > R(0)) {
                R vsv = R(0);
                for (int k = 0; k < NS; ++k) {
                    const int a = s_a<D>(k), b = s_b<D>(k);
                    vsv += (a == b ? R(1) : R(2)) * v[a] * v[b] * ras[(RW::SIG + k) * rs + c];
                }
                q = R(A.entrain) * fabs(vsv) / speed;
            }
        }
        out += R(A.dt) * q;
    }
    if (A.source) out += R(A.dt) * ((const R*)A.source)[c];
    dst.at(fi_phi<D>(), c) = out;
}

// ---------------------------------------------------------------------------
// diagnostics: out[0..D-1] += vol * sum rho u (leaf), out[D] += vol * sum phi,
// out[D+1] = min eps (leaf); warp shuffles -> shared memory -> one double
// atomic per block and value
template <int NV>
__device__ __forceinline__ void block_sum_atomic(double (&acc)[NV], double* out) {
    __shared__ double red[NV][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        double v = acc[k];
        for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
        if (lane == 0) red[k][wid] = v;
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double v = lane < nw ? red[k][lane] : 0.0;
            for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
            if (lane == 0 && v != 0.0) atomicAdd(&out[k], v);
        }
    }
}

__device__ __forceinline__ void atomic_min_double(double* addr, double v) {
    unsigned long long* a = (unsigned long long*)addr;
    unsigned long long old = *a, assumed;
    do {
        assumed = old;
        if (__longlong_as_double(assumed) <= v) break;
        old = atomicCAS(a, assumed, __double_as_longlong(v));
    } while (assumed != old);
}

template <int D, typename R>
__global__ void k_diag_level(mlbm_level_t lv, mlbm_fields_t f, double vol, double* out) {
    constexpr int T = Geo<D>::T;
    double acc[D + 1];
    for (int k = 0; k <= D; ++k) acc[k] = 0.0;
    double emin = 1e300;
    const FieldsT<R> a = fields_of<R>(f);
    const int64_t n = (int64_t)live_tiles(lv) * T;
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;                 // 4 cells per trip: loads overlap
    for (int64_t c0 = (int64_t)lv.first * T + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c0 < n;
         c0 += U * st) {
        bool lf[U];
        R r0[U], uu[U][D], ph[U], ep[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t c = c0 + u * st;
            lf[u] = c < n && (lv.cell_flags[c] & MLBM_CF_LEAF);
            if (lf[u]) {
                r0[u] = a.at(0, c);
#pragma unroll
                for (int k = 0; k < D; ++k) uu[u][k] = a.at(1 + k, c);
                ph[u] = a.at(fi_phi<D>(), c);
                ep[u] = a.at(fi_eps<D>(), c);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!lf[u]) continue;
            const double rho = 1.0 + (double)r0[u];
            for (int k = 0; k < D; ++k) acc[k] += vol * rho * (double)uu[u][k];
            acc[D] += vol * (double)ph[u];
            emin = fmin(emin, (double)ep[u]);
        }
    }
    // block min, then one compare-and-swap per block (not per warp)
    __shared__ double smin[32];
    for (int off = 16; off > 0; off >>= 1) emin = fmin(emin, __shfl_down_sync(0xffffffffu, emin, off));
    if ((threadIdx.x & 31) == 0) smin[threadIdx.x >> 5] = emin;
    block_sum_atomic<D + 1>(acc, out);          // contains __syncthreads
    if (threadIdx.x == 0) {
        double m = smin[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, smin[w]);
        if (m < 1e300 && m < *(volatile double*)&out[D + 1]) atomic_min_double(&out[D + 1], m);
    }
}

// out[0..D-1] += sum m v ; out[D..2D-1] += sum fs (level-0 cells)
template <int D, typename R>
__global__ void __launch_bounds__(256, 4) k_diag_particles(PartArgs P, const R* ras, int64_t rs, int64_t n0,
                                 const int32_t* live, double* out) {
    using PR = PRows<D>;
    if (live) n0 = min(n0, (int64_t)live[0] * Geo<D>::T);
    double acc[2 * D];
    for (int k = 0; k < 2 * D; ++k) acc[k] = 0.0;
    const R* pp = (const R*)P.p;
    const int64_t m = P.n > n0 ? P.n : n0;
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    constexpr int U = 4;                 // 4 elements per trip: loads overlap
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < m; i0 += U * st) {
        R mv[U], vv[U][D], fv[U][D];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + u * st;
            mv[u] = R(0);
#pragma unroll
            for (int a = 0; a < D; ++a) { vv[u][a] = R(0); fv[u][a] = R(0); }
            if (i < P.n) {
                mv[u] = pp[PR::M * P.ps + i];
#pragma unroll
                for (int a = 0; a < D; ++a) vv[u][a] = pp[(PR::V + a) * P.ps + i];
            }
            if (ras && i < n0) {
#pragma unroll
                for (int a = 0; a < D; ++a) fv[u][a] = ras[(Rows<D>::FS + a) * rs + i];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int a = 0; a < D; ++a) {
                acc[a] += (double)mv[u] * (double)vv[u][a];
                acc[D + a] += (double)fv[u][a];
            }
    }
    block_sum_atomic<2 * D>(acc, out);
}

// ---------------------------------------------------------------------------
// particle sort by (level-0 tile slot, cell) of the stencil base cell
template <int D>
__global__ void k_sort_keys(int n, const double* x, int64_t ps, TopoL0 t0, uint32_t* keys, int32_t* vals) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int c[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) {
        int b = (int)floor(x[a * ps + p] - 0.5);
        if (t0.periodic[a]) b = wrap_near(b, t0.cells[a]);
        else b = b < 0 ? 0 : (b >= t0.cells[a] ? t0.cells[a] - 1 : b);
        c[a] = b;
    }
    const int s = t0.tile_map[g3(t0.tiles, c[0] >> 2, c[1] >> 2, D == 3 ? c[2] >> 2 : 0)];
    keys[p] = s < 0 ? 0xffffffffu : (uint32_t)s * Geo<D>::T + local_of<D>(c[0] & 3, c[1] & 3, c[2] & 3);
    vals[p] = p;
}

template <typename R>
__global__ void k_gather_particles(int n, int nrows, const int32_t* __restrict__ perm,
                                   const double* __restrict__ x, int dim, const R* __restrict__ pdat,
                                   const int32_t* __restrict__ pid, int64_t ps, double* __restrict__ xo,
                                   R* __restrict__ po, int32_t* __restrict__ pido) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int j = perm[i];
    for (int a = 0; a < dim; ++a) xo[a * ps + i] = x[a * ps + j];
    // rows in batches of 8: the (non-aliasing) loads of a batch are in flight
    // together instead of one row's latency at a time
    int r = 0;
    for (; r + 8 <= nrows; r += 8) {
        R v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = pdat[(r + k) * ps + j];
#pragma unroll
        for (int k = 0; k < 8; ++k) po[(r + k) * ps + i] = v[k];
    }
    for (; r < nrows; ++r) po[r * ps + i] = pdat[r * ps + j];
    pido[i] = pid[j];
}

// P2G with per-block shared-memory accumulation over the bounding box of
// the block's (sorted) particles; blocks whose box does not fit fall back to
// global atomics.  Same arithmetic per contribution as k_p2g.
template <int D, typename R> struct P2GSmem {
    static constexpr int NV = 3 + 3 * D;                        // mass, mom, fint, eta, area, vmom
    static constexpr int MAXN = sizeof(R) == 4 ? 512 : 256;
};

template <int D, typename R>
__global__ void __launch_bounds__(256) k_p2g_smem(PartArgs P, TopoL0 t0, MatParams mp, R* ras, int64_t rs,
                                                  mlbm_error_t* err) {
    constexpr int K = Geo<D>::K;
    constexpr int NV = P2GSmem<D, R>::NV, MAXN = P2GSmem<D, R>::MAXN;
    using RW = Rows<D>;
    using PR = PRows<D>;
    __shared__ R acc[NV * MAXN];
    __shared__ int s_lo[3], s_hi[3];
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = p < P.n;
    const R* pp = (const R*)P.p;
    double x[D];
    Stencil<D, R> st;
    if (valid) {
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = P.x[a * P.ps + p];
        make_stencil<D, R>(x, st);
    }
    if (threadIdx.x < 3) { s_lo[threadIdx.x] = 0x7fffffff; s_hi[threadIdx.x] = -0x7fffffff; }
    __syncthreads();
    if (valid) {
#pragma unroll
        for (int a = 0; a < D; ++a) { atomicMin(&s_lo[a], st.base[a]); atomicMax(&s_hi[a], st.base[a] + 2); }
    }
    __syncthreads();
    int ext[3] = {1, 1, 1}, lo[3] = {0, 0, 0};
    int nbox = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) { lo[a] = s_lo[a]; ext[a] = s_hi[a] - s_lo[a] + 1; nbox *= ext[a]; }
    const bool use_smem = nbox <= MAXN && nbox > 0;
    if (use_smem) {
        for (int i = threadIdx.x; i < NV * nbox; i += blockDim.x) acc[(i / nbox) * MAXN + i % nbox] = R(0);
    }
    __syncthreads();
    if (valid) {
        R v[D], C[D * D];
#pragma unroll
        for (int a = 0; a < D; ++a) v[a] = pp[(PR::V + a) * P.ps + p];
#pragma unroll
        for (int k = 0; k < D * D; ++k) C[k] = pp[(PR::C + k) * P.ps + p];
        const R m = pp[PR::M * P.ps + p], V0 = pp[PR::V0 * P.ps + p];
        R tau[D * D];
        load_tau<D, R>(pp, P.ps, p, tau);
        const R ap = D == 2 ? R(2) * sqrt(V0 / R(3.14159265358979323846))
                            : R(3.14159265358979323846) * pow(R(3) * V0 / (R(4) * R(3.14159265358979323846)), R(2.0 / 3.0));
        bool bad = false;
        // sorted neighbours share their stencil: stagger the node order per
        // lane so that lanes of one cell hit different shared-memory words
        const int k0 = (threadIdx.x & 31) % K;
#pragma unroll 1
        for (int kk = 0; kk < K; ++kk) {
            const int k = (kk + k0) % K;
            const int o[3] = {k % 3, (k / 3) % 3, k / 9};
            R w = R(1), gr[D];
#pragma unroll
            for (int a = 0; a < D; ++a) { w *= sel3<R>(st.w[a], o[a]); gr[a] = R(1); }
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = 0; b < D; ++b) gr[b] *= (a == b) ? sel3<R>(st.dw[a], o[a]) : sel3<R>(st.w[a], o[a]);
            R dpos[D];
#pragma unroll
            for (int a = 0; a < D; ++a) dpos[a] = R((double)(st.base[a] + o[a]) - x[a]);
            const R wm = w * m;
            R val[NV];
            val[0] = wm;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                R aff = v[a];
#pragma unroll
                for (int b = 0; b < D; ++b) aff += C[a * D + b] * dpos[b];
                val[1 + a] = wm * aff;
                R fa = R(0);
#pragma unroll
                for (int b = 0; b < D; ++b) fa += V0 * tau[a * D + b] * gr[b];
                val[1 + D + a] = -fa;
                val[3 + 2 * D + a] = wm * v[a];
            }
            val[1 + 2 * D] = w * V0;
            val[2 + 2 * D] = w * ap;
            if (use_smem) {
                int li = 0;
#pragma unroll
                for (int a = D - 1; a >= 0; --a) li = li * ext[a] + (st.base[a] + o[a] - lo[a]);
#pragma unroll
                for (int q = 0; q < NV; ++q) atomicAdd(&acc[q * MAXN + li], val[q]);
            } else {
                int c[3] = {st.base[0] + o[0], st.base[1] + o[1], D == 3 ? st.base[2] + o[2] : 0};
                const int64_t ni = node_index<D>(t0, c, bad);
                if (ni < 0) continue;
                // row order of the raster: mass, mom, fint, eta, area, vmom
#pragma unroll
                for (int q = 0; q < NV; ++q) aadd(&ras[q * rs + ni], val[q]);
            }
        }
        if (bad) report_error(err, MLBM_ERR_STENCIL, 0, st.base[0], st.base[1], st.base[2]);
    }
    if (!use_smem) return;
    __syncthreads();
    for (int i = threadIdx.x; i < nbox; i += blockDim.x) {
        if (acc[i] == R(0) && acc[(2 * D + 2) * MAXN + i] == R(0)) {
            // no mass and no area landed here: every row is zero
            continue;
        }
        int c[3] = {0, 0, 0};
        int r = i;
#pragma unroll
        for (int a = 0; a < D; ++a) { c[a] = lo[a] + r % ext[a]; r /= ext[a]; }
        bool bad = false;
        const int64_t ni = node_index<D>(t0, c, bad);
        if (ni < 0) { report_error(err, MLBM_ERR_STENCIL, 0, c[0], c[1], c[2]); continue; }
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const R vq = acc[q * MAXN + i];
            if (vq != R(0)) aadd(&ras[q * rs + ni], vq);
        }
    }
}

// ---------------------------------------------------------------------------
// Warp-cooperative P2G for sorted particles.  Each lane owns up to NPL nodes of
// the warp's node bounding box and accumulates all 3+3D rows for them in
// registers while the warp's 32 particles are broadcast one by one (shuffles);
// a warp whose box exceeds 32*NPL nodes scatters per particle instead.
// Contribution algebra (granular.py:282-310) with dpos = o - f:
//   mass  w m          mom_a  w (q_a + sum_b P_ab o_b),  q = m v - m C f,  P = m C
//   fint_a -sum_b S_ab grad_b (S = V0 tau)   eta w V0   area w a_p   vmom_a w m v_a
template <int D, typename R, int NPL>
__global__ void __launch_bounds__(128, 4) k_p2g_warp(PartArgs P, TopoL0 t0, MatParams mp, R* ras, int64_t rs,
                                                  mlbm_error_t* err) {
    constexpr int NV = 3 + 3 * D;
    using PR = PRows<D>;
    const int lane = threadIdx.x & 31;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = p < P.n;
    const R* pp = (const R*)P.p;
    // ---- per-particle quantities
    int base[3] = {0, 0, 0};
    R f[D], m = R(0), V0 = R(0), ap = R(0), mv[D], q[D], PC[D * D], S[D * (D + 1) / 2];
#pragma unroll
    for (int a = 0; a < D; ++a) { f[a] = R(0); mv[a] = R(0); q[a] = R(0); }
#pragma unroll
    for (int k = 0; k < D * D; ++k) PC[k] = R(0);
#pragma unroll
    for (int k = 0; k < D * (D + 1) / 2; ++k) S[k] = R(0);
    if (valid) {
        double x[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            x[a] = P.x[a * P.ps + p];
            const double b = floor(x[a] - 0.5);
            base[a] = (int)b;
            f[a] = R(x[a] - b);
        }
        m = pp[PR::M * P.ps + p];
        V0 = pp[PR::V0 * P.ps + p];
        R v[D], C[D * D];
#pragma unroll
        for (int a = 0; a < D; ++a) v[a] = pp[(PR::V + a) * P.ps + p];
#pragma unroll
        for (int k = 0; k < D * D; ++k) C[k] = pp[(PR::C + k) * P.ps + p];
        R tau[D * D];
        load_tau<D, R>(pp, P.ps, p, tau);
        ap = D == 2 ? R(2) * sqrt(V0 / R(3.14159265358979323846))
                    : R(3.14159265358979323846) * pow(R(3) * V0 / (R(4) * R(3.14159265358979323846)), R(2.0 / 3.0));
#pragma unroll
        for (int a = 0; a < D; ++a) {
            mv[a] = m * v[a];
            R cf = R(0);
#pragma unroll
            for (int b = 0; b < D; ++b) { PC[a * D + b] = m * C[a * D + b]; cf += C[a * D + b] * f[b]; }
            q[a] = m * (v[a] - cf);
        }
        int k = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a; b < D; ++b) S[k++] = V0 * tau[a * D + b];
    }
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    if (vmask == 0) return;
    // Warp-uniform segmentation of the sorted particles: a segment grows
    // while the bounding box of its stencils stays within 32*NPL nodes.
    int j0 = 0;
    while (j0 < 32) {
        if (!((vmask >> j0) & 1u)) { ++j0; continue; }
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
#pragma unroll
        for (int a = 0; a < D; ++a) {
            lo[a] = __shfl_sync(0xffffffffu, base[a], j0);
            hi[a] = lo[a] + 2;
        }
        int j1 = j0 + 1;
        while (j1 < 32) {
            if (!((vmask >> j1) & 1u)) { ++j1; continue; }
            int nl[3], nh[3], nb = 1;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int b = __shfl_sync(0xffffffffu, base[a], j1);
                nl[a] = min(lo[a], b);
                nh[a] = max(hi[a], b + 2);
                nb *= nh[a] - nl[a] + 1;
            }
            if (nb > 32 * NPL) break;
#pragma unroll
            for (int a = 0; a < D; ++a) { lo[a] = nl[a]; hi[a] = nh[a]; }
            ++j1;
        }
        int ext[3] = {1, 1, 1}, nbox = 1;
#pragma unroll
        for (int a = 0; a < D; ++a) { ext[a] = hi[a] - lo[a] + 1; nbox *= ext[a]; }
        R acc[NPL][NV];
        int nc[NPL][3];
#pragma unroll
        for (int r = 0; r < NPL; ++r) {
            int li = lane + 32 * r;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (a < D) { nc[r][a] = lo[a] + li % ext[a]; li /= ext[a]; } else nc[r][a] = 0;
            }
#pragma unroll
            for (int qv = 0; qv < NV; ++qv) acc[r][qv] = R(0);
        }
        for (int j = j0; j < j1; ++j) {
            if (!((vmask >> j) & 1u)) continue;
            int bj[3];
            R fj[D], mj, V0j, apj, mvj[D], qj[D], Pj[D * D], Sj[D * (D + 1) / 2];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                bj[a] = __shfl_sync(0xffffffffu, base[a], j);
                fj[a] = __shfl_sync(0xffffffffu, f[a], j);
                mvj[a] = __shfl_sync(0xffffffffu, mv[a], j);
                qj[a] = __shfl_sync(0xffffffffu, q[a], j);
            }
#pragma unroll
            for (int k = 0; k < D * D; ++k) Pj[k] = __shfl_sync(0xffffffffu, PC[k], j);
#pragma unroll
            for (int k = 0; k < D * (D + 1) / 2; ++k) Sj[k] = __shfl_sync(0xffffffffu, S[k], j);
            mj = __shfl_sync(0xffffffffu, m, j);
            V0j = __shfl_sync(0xffffffffu, V0, j);
            apj = __shfl_sync(0xffffffffu, ap, j);
            R W[D][3], DW[D][3];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const R fa = fj[a];
                W[a][0] = R(0.5) * (R(1.5) - fa) * (R(1.5) - fa);
                W[a][1] = R(0.75) - (fa - R(1)) * (fa - R(1));
                W[a][2] = R(0.5) * (fa - R(0.5)) * (fa - R(0.5));
                DW[a][0] = fa - R(1.5);
                DW[a][1] = R(-2) * (fa - R(1));
                DW[a][2] = fa - R(0.5);
            }
#pragma unroll
            for (int r = 0; r < NPL; ++r) {
                int o[3] = {0, 0, 0};
                bool in = lane + 32 * r < nbox;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    o[a] = nc[r][a] - bj[a];
                    in &= (unsigned)o[a] < 3u;
                }
                if (!in) continue;
                R wa[D], dwa[D];
#pragma unroll
                for (int a = 0; a < D; ++a) { wa[a] = sel3<R>(W[a], o[a]); dwa[a] = sel3<R>(DW[a], o[a]); }
                R w = R(1);
#pragma unroll
                for (int a = 0; a < D; ++a) w *= wa[a];
                R gr[D];
#pragma unroll
                for (int b = 0; b < D; ++b) {
                    R g = dwa[b];
#pragma unroll
                    for (int a = 0; a < D; ++a) if (a != b) g *= wa[a];
                    gr[b] = g;
                }
                acc[r][0] += w * mj;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    R mo = qj[a];
#pragma unroll
                    for (int b = 0; b < D; ++b) mo += Pj[a * D + b] * R(o[b]);
                    acc[r][1 + a] += w * mo;
                    R fa = R(0);
#pragma unroll
                    for (int b = 0; b < D; ++b) {
                        const int sk = a <= b ? a * D - a * (a - 1) / 2 + (b - a) : b * D - b * (b - 1) / 2 + (a - b);
                        fa += Sj[sk] * gr[b];
                    }
                    acc[r][1 + D + a] -= fa;
                    acc[r][3 + 2 * D + a] += w * mvj[a];
                }
                acc[r][1 + 2 * D] += w * V0j;
                acc[r][2 + 2 * D] += w * apj;
            }
        }
#pragma unroll
        for (int r = 0; r < NPL; ++r) {
            if (lane + 32 * r >= nbox) continue;
            if (acc[r][0] == R(0) && acc[r][2 + 2 * D] == R(0)) continue;
            int c[3] = {nc[r][0], nc[r][1], nc[r][2]};
            bool bad = false;
            const int64_t ni = node_index<D>(t0, c, bad);
            if (ni < 0) { report_error(err, MLBM_ERR_STENCIL, 0, nc[r][0], nc[r][1], nc[r][2]); continue; }
#pragma unroll
            for (int qv = 0; qv < NV; ++qv)
                if (acc[r][qv] != R(0)) aadd(&ras[qv * rs + ni], acc[r][qv]);
        }
        j0 = j1;
    }
}

// ---------------------------------------------------------------------------
// Cell-cooperative P2G for sorted particles (smem mode 3).  Within a warp, the
// particles of one cell share their 3^D stencil nodes: lane k < 3^D owns node
// k of the current cell and accumulates all 3+3D rows in registers while the
// cell's particles are broadcast; at each cell change the lanes flush into a
// block-wide shared-memory box (one conflict-free RED per lane and row), and
// the block box is flushed to HBM once.  No coverage tests, no idle-node work.
// min resident 64-thread blocks per SM for the fp32 P2G (9: up to 112
// registers; 1-3 % faster than 10 at 96 registers, profiles/r1_p2g_box_sweep.txt)
#ifndef P2G2_MIN_BLOCKS
#define P2G2_MIN_BLOCKS 9
#endif
#ifndef P2G2_MAXN
#define P2G2_MAXN 144
#endif
// node-box capacity of the stress raster (its box spans only the particles
// near an entrainment surface)
#ifndef STRESS_MAXN
#define STRESS_MAXN 64      // 144 (the P2G box): +0.08 ms on C4 (occupancy); 48-72 alike
#endif
#ifndef P2G2_NW
#define P2G2_NW 2
#endif
#ifndef P2G2_ROUNDS
#define P2G2_ROUNDS 1
#endif
// 3D fp32 P2G node arithmetic on register pairs (FFMA2 / FMUL2: one issue slot
// for two lanes of fp32 math; tools/micro/ffma2_mix.cu)
#ifndef P2G2_PAIRED
#define P2G2_PAIRED 1
#endif
// rounds of a dense-sampling block (mode 5): C4 P2G 5.60 / 5.41 / 5.43 / 5.51 ms
// at 4 / 8 / 12 / 16 rounds, 5.89 at 2 (tools/p2g_sweep.sh)
#ifndef P2G2_ROUNDS_DENSE
#define P2G2_ROUNDS_DENSE 8
#endif
template <int D, typename R>
__global__ void __launch_bounds__(128) k_p2g_cell(PartArgs P, TopoL0 t0, MatParams mp, R* ras, int64_t rs,
                                                  mlbm_error_t* err) {
    constexpr int K = Geo<D>::K, NV = 3 + 3 * D, NS = D * (D + 1) / 2;
    constexpr int MAXN = sizeof(R) == 4 ? 512 : 256;
    using PR = PRows<D>;
    __shared__ R sacc[NV * MAXN];
    __shared__ int s_lo[3], s_hi[3];
    // per-warp particle slabs: one 32-float record per particle, broadcast to
    // the node lanes with uniform-address vector loads (fp32 only)
    constexpr bool SLAB = sizeof(R) == 4;
    constexpr int REC = 32;
    __shared__ __align__(16) float slab[SLAB ? 4 : 1][SLAB ? 32 * REC : 1];
    const int lane = threadIdx.x & 31;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = p < P.n;
    const R* pp = (const R*)P.p;
    int base[3] = {0, 0, 0};
    R f[D], m = R(0), V0 = R(0), ap = R(0), mv[D], q[D], PC[D * D], S[NS];
#pragma unroll
    for (int a = 0; a < D; ++a) { f[a] = R(0); mv[a] = R(0); q[a] = R(0); }
#pragma unroll
    for (int k = 0; k < D * D; ++k) PC[k] = R(0);
#pragma unroll
    for (int k = 0; k < NS; ++k) S[k] = R(0);
    if (valid) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const double x = P.x[a * P.ps + p];
            const double b = floor(x - 0.5);
            base[a] = (int)b;
            f[a] = R(x - b);
        }
        m = pp[PR::M * P.ps + p];
        V0 = pp[PR::V0 * P.ps + p];
        R v[D], C[D * D];
#pragma unroll
        for (int a = 0; a < D; ++a) v[a] = pp[(PR::V + a) * P.ps + p];
#pragma unroll
        for (int k = 0; k < D * D; ++k) C[k] = pp[(PR::C + k) * P.ps + p];
        R tau[D * D];
        load_tau<D, R>(pp, P.ps, p, tau);
        ap = D == 2 ? R(2) * sqrt(V0 / R(3.14159265358979323846))
                    : R(3.14159265358979323846) * pow(R(3) * V0 / (R(4) * R(3.14159265358979323846)), R(2.0 / 3.0));
#pragma unroll
        for (int a = 0; a < D; ++a) {
            mv[a] = m * v[a];
            R cf = R(0);
#pragma unroll
            for (int b = 0; b < D; ++b) { PC[a * D + b] = m * C[a * D + b]; cf += C[a * D + b] * f[b]; }
            q[a] = m * (v[a] - cf);
        }
        int k = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a; b < D; ++b) S[k++] = V0 * tau[a * D + b];
    }
    if constexpr (SLAB) {
        float* rec = &slab[threadIdx.x >> 5][lane * REC];
        int o2 = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) rec[o2++] = __int_as_float(a < D ? base[a] : 0);
#pragma unroll
        for (int a = 0; a < D; ++a) rec[o2++] = (float)f[a];
#pragma unroll
        for (int a = 0; a < D; ++a) rec[o2++] = (float)mv[a];
#pragma unroll
        for (int a = 0; a < D; ++a) rec[o2++] = (float)q[a];
#pragma unroll
        for (int kk = 0; kk < D * D; ++kk) rec[o2++] = (float)PC[kk];
#pragma unroll
        for (int kk = 0; kk < NS; ++kk) rec[o2++] = (float)S[kk];
        rec[o2++] = (float)m;
        rec[o2++] = (float)V0;
        rec[o2++] = (float)ap;
        __syncwarp();
    }
    // block node box (shared-memory accumulation when it fits)
    if (threadIdx.x < 3) { s_lo[threadIdx.x] = 0x7fffffff; s_hi[threadIdx.x] = -0x7fffffff; }
    __syncthreads();
    if (valid) {
#pragma unroll
        for (int a = 0; a < D; ++a) { atomicMin(&s_lo[a], base[a]); atomicMax(&s_hi[a], base[a] + 2); }
    }
    __syncthreads();
    int lo[3] = {0, 0, 0}, ext[3] = {1, 1, 1}, nbox = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) { lo[a] = s_lo[a]; ext[a] = s_hi[a] - s_lo[a] + 1; nbox *= ext[a]; }
    const bool use_smem = nbox > 0 && nbox <= MAXN;
    if (use_smem)
        for (int i = threadIdx.x; i < NV * nbox; i += blockDim.x) sacc[(i / nbox) * MAXN + i % nbox] = R(0);
    __syncthreads();

    const int o[3] = {lane % 3, (lane / 3) % 3, D == 3 ? (lane / 9) % 3 : 0};
    const bool node_lane = lane < K;
    const unsigned vmask = __ballot_sync(0xffffffffu, valid);
    R acc[NV];
#pragma unroll
    for (int qv = 0; qv < NV; ++qv) acc[qv] = R(0);
    int cur[3] = {0, 0, 0};
    bool have = false;
    bool bad = false;
    auto flush = [&]() {
        if (!have || !node_lane) return;
        if (acc[0] == R(0) && acc[2 + 2 * D] == R(0)) return;
        int c[3] = {cur[0] + o[0], cur[1] + o[1], D == 3 ? cur[2] + o[2] : 0};
        if (use_smem) {
            int li = 0;
#pragma unroll
            for (int a = D - 1; a >= 0; --a) li = li * ext[a] + (c[a] - lo[a]);
#pragma unroll
            for (int qv = 0; qv < NV; ++qv) atomicAdd(&sacc[qv * MAXN + li], acc[qv]);
        } else {
            const int64_t ni = node_index<D>(t0, c, bad);
            if (ni >= 0) {
#pragma unroll
                for (int qv = 0; qv < NV; ++qv) aadd(&ras[qv * rs + ni], acc[qv]);
            }
        }
    };
    for (int j = 0; j < 32; ++j) {
        if (!((vmask >> j) & 1u)) continue;
        int bj[3];
        R fj[D], mvj[D], qj[D], Pj[D * D], Sj[NS], mj, V0j, apj;
        if constexpr (SLAB) {
            float r[REC];
            const float4* rp = reinterpret_cast<const float4*>(&slab[threadIdx.x >> 5][j * REC]);
#pragma unroll
            for (int v4 = 0; v4 < REC / 4; ++v4) {
                const float4 t = rp[v4];
                r[4 * v4] = t.x; r[4 * v4 + 1] = t.y; r[4 * v4 + 2] = t.z; r[4 * v4 + 3] = t.w;
            }
            int o2 = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a) bj[a] = __float_as_int(r[o2++]);
#pragma unroll
            for (int a = 0; a < D; ++a) fj[a] = r[o2++];
#pragma unroll
            for (int a = 0; a < D; ++a) mvj[a] = r[o2++];
#pragma unroll
            for (int a = 0; a < D; ++a) qj[a] = r[o2++];
#pragma unroll
            for (int kk = 0; kk < D * D; ++kk) Pj[kk] = r[o2++];
#pragma unroll
            for (int kk = 0; kk < NS; ++kk) Sj[kk] = r[o2++];
            mj = r[o2++];
            V0j = r[o2++];
            apj = r[o2++];
        } else {
#pragma unroll
            for (int a = 0; a < 3; ++a) bj[a] = a < D ? __shfl_sync(0xffffffffu, base[a], j) : 0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                fj[a] = __shfl_sync(0xffffffffu, f[a], j);
                mvj[a] = __shfl_sync(0xffffffffu, mv[a], j);
                qj[a] = __shfl_sync(0xffffffffu, q[a], j);
            }
#pragma unroll
            for (int kk = 0; kk < D * D; ++kk) Pj[kk] = __shfl_sync(0xffffffffu, PC[kk], j);
#pragma unroll
            for (int kk = 0; kk < NS; ++kk) Sj[kk] = __shfl_sync(0xffffffffu, S[kk], j);
            mj = __shfl_sync(0xffffffffu, m, j);
            V0j = __shfl_sync(0xffffffffu, V0, j);
            apj = __shfl_sync(0xffffffffu, ap, j);
        }
        if (!have || bj[0] != cur[0] || bj[1] != cur[1] || (D == 3 && bj[2] != cur[2])) {
            flush();
#pragma unroll
            for (int qv = 0; qv < NV; ++qv) acc[qv] = R(0);
#pragma unroll
            for (int a = 0; a < 3; ++a) cur[a] = bj[a];
            have = true;
        }
        R wa[D], dwa[D];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const R fa = fj[a];
            wa[a] = o[a] == 0 ? R(0.5) * (R(1.5) - fa) * (R(1.5) - fa)
                  : (o[a] == 1 ? R(0.75) - (fa - R(1)) * (fa - R(1)) : R(0.5) * (fa - R(0.5)) * (fa - R(0.5)));
            dwa[a] = o[a] == 0 ? fa - R(1.5) : (o[a] == 1 ? R(-2) * (fa - R(1)) : fa - R(0.5));
        }
        R w = R(1);
#pragma unroll
        for (int a = 0; a < D; ++a) w *= wa[a];
        acc[0] += w * mj;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            R mo = qj[a];
#pragma unroll
            for (int b = 0; b < D; ++b) mo += Pj[a * D + b] * R(o[b]);
            acc[1 + a] += w * mo;
            R fa = R(0);
#pragma unroll
            for (int b = 0; b < D; ++b) {
                R g = dwa[b];
#pragma unroll
                for (int e = 0; e < D; ++e) if (e != b) g *= wa[e];
                const int sk = a <= b ? a * D - a * (a - 1) / 2 + (b - a) : b * D - b * (b - 1) / 2 + (a - b);
                fa += Sj[sk] * g;
            }
            acc[1 + D + a] -= fa;
            acc[3 + 2 * D + a] += w * mvj[a];
        }
        acc[1 + 2 * D] += w * V0j;
        acc[2 + 2 * D] += w * apj;
    }
    flush();
    if (bad) report_error(err, MLBM_ERR_STENCIL, 0, cur[0], cur[1], cur[2]);
    if (!use_smem) return;
    __syncthreads();
    for (int i = threadIdx.x; i < nbox; i += blockDim.x) {
        if (sacc[i] == R(0) && sacc[(2 + 2 * D) * MAXN + i] == R(0)) continue;
        int c[3] = {0, 0, 0};
        int r = i;
#pragma unroll
        for (int a = 0; a < D; ++a) { c[a] = lo[a] + r % ext[a]; r /= ext[a]; }
        bool b2 = false;
        const int64_t ni = node_index<D>(t0, c, b2);
        if (ni < 0) { report_error(err, MLBM_ERR_STENCIL, 0, c[0], c[1], c[2]); continue; }
#pragma unroll
        for (int qv = 0; qv < NV; ++qv) {
            const R vq = sacc[qv * MAXN + i];
            if (vq != R(0)) aadd(&ras[qv * rs + ni], vq);
        }
    }
}

// ---------------------------------------------------------------------------
// Cell-cooperative P2G, fp32, atomic-free in shared memory (smem mode 4).
// Same decomposition as k_p2g_cell (lane k owns stencil node k of the current
// cell; particles of a warp broadcast from a per-warp record slab), but
//  * every warp owns a private copy of the block's node box, so the per-cell
//    flushes are plain read-add-write (shared-memory fp32 atomics lower to a
//    compare-and-swap loop on this architecture); the NW copies are summed
//    once when the box is written to HBM;
//  * the lane's B-spline weights are per-lane quadratics c0 + c1 f + c2 f^2
//    (coefficients fixed by the lane's node offset), no selects per particle.
// per-particle P2G record (fp32): base[3] f[D] m V0 ap q[D] mv[D] S[NS] PC[D*D]
// (granular.py:282-310: APIC affine momentum, V0 * Kirchhoff stress, area)
template <int D>
__device__ __forceinline__ void p2g_record(const PartArgs& P, const MatParams& mp, int p, bool valid,
                                           float* rec) {
    constexpr int NS = D * (D + 1) / 2;
    using PR = PRows<D>;
    const float* pp = (const float*)P.p;
    int base[3] = {0, 0, 0};
        float f[D], m = 0.f, V0 = 0.f, ap = 0.f, mv[D], q[D], PC[D * D], S[NS];
#pragma unroll
        for (int a = 0; a < D; ++a) { f[a] = 0.f; mv[a] = 0.f; q[a] = 0.f; }
#pragma unroll
        for (int k = 0; k < D * D; ++k) PC[k] = 0.f;
#pragma unroll
        for (int k = 0; k < NS; ++k) S[k] = 0.f;
        if (valid) {
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const double x = P.x[a * P.ps + p];
                const double b = floor(x - 0.5);
                base[a] = (int)b;
                f[a] = (float)(x - b);
            }
            m = pp[PR::M * P.ps + p];
            V0 = pp[PR::V0 * P.ps + p];
            float v[D], C[D * D];
#pragma unroll
            for (int a = 0; a < D; ++a) v[a] = pp[(PR::V + a) * P.ps + p];
#pragma unroll
            for (int k = 0; k < D * D; ++k) C[k] = pp[(PR::C + k) * P.ps + p];
            float tau[D * D];
            load_tau<D, float>(pp, P.ps, p, tau);
            ap = D == 2 ? 2.f * sqrtf(V0 / 3.14159265358979323846f)
                        : [](float c) { return 3.14159265358979323846f * c * c; }(
                              cbrtf(3.f * V0 / (4.f * 3.14159265358979323846f)));   // pi (3V/4pi)^(2/3)
#pragma unroll
            for (int a = 0; a < D; ++a) {
                mv[a] = m * v[a];
                float cf = 0.f;
#pragma unroll
                for (int b = 0; b < D; ++b) { PC[a * D + b] = m * C[a * D + b]; cf += C[a * D + b] * f[b]; }
                q[a] = m * (v[a] - cf);
            }
            int k = 0;
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = a; b < D; ++b) S[k++] = V0 * tau[a * D + b];
        }
        // record: base[3] f[D] m V0 ap q[D] mv[D] S[NS] PC[D*D]
        int o2 = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) rec[o2++] = __int_as_float(a < D ? base[a] : 0);
#pragma unroll
        for (int a = 0; a < D; ++a) rec[o2++] = f[a];
        rec[o2++] = m;
        rec[o2++] = V0;
        rec[o2++] = ap;
#pragma unroll
        for (int a = 0; a < D; ++a) rec[o2++] = q[a];
#pragma unroll
        for (int a = 0; a < D; ++a) rec[o2++] = mv[a];
#pragma unroll
        for (int kk = 0; kk < NS; ++kk) rec[o2++] = S[kk];
#pragma unroll
        for (int kk = 0; kk < D * D; ++kk) rec[o2++] = PC[kk];
    }

// The 3D record of p2g_record (base[3] f[3] m V0 ap q[3] mv[3] S[6] PC[9])
// permuted for the paired node arithmetic of k_p2g_cell2: every operand pair
// of an FFMA2 sits in an aligned register pair of one 128-bit load (28 floats,
// seven broadcast loads):
//   (fx fy) fz q2 | (m V0)(ap mv0) | (mv1 mv2)(q0 q1) | (PC00 PC10)(PC01 PC11) |
//   (PC02 PC12) PC20 PC21 | PC22 -S22 (-S00 -S01) | (-S01 -S11)(-S02 -S12)
__device__ __forceinline__ void p2g_pair_record(const float (&r)[32], float (&p)[28]) {
    constexpr int F = 3, M = 6, Q = 9, MV = 12, S = 15, PC = 21;
    const float q[28] = {r[F], r[F + 1], r[F + 2], r[Q + 2],
                         r[M], r[M + 1], r[M + 2], r[MV],
                         r[MV + 1], r[MV + 2], r[Q], r[Q + 1],
                         r[PC + 0], r[PC + 3], r[PC + 1], r[PC + 4],
                         r[PC + 2], r[PC + 5], r[PC + 6], r[PC + 7],
                         r[PC + 8], -r[S + 5], -r[S + 0], -r[S + 1],
                         -r[S + 1], -r[S + 3], -r[S + 2], -r[S + 4]};
#pragma unroll
    for (int k = 0; k < 28; ++k) p[k] = q[k];
}

// Sum the NW per-warp node-box copies and add the node totals into the
// raster rows (one atomic per touched node and non-zero row).  STRESS = 0:
// the P2G rows (a node is touched iff its mass or area is non-zero); STRESS =
// 1: rows 0..NV-2 are written and row NV-1 counts the particles that touched
// the node (an untouched node is neither written nor checked).
template <int D, int NV, int STRESS>
__device__ __forceinline__ void p2g_box_merge(const float* sacc, int NW, int MAXN, int nbox,
                                              const int (&lo)[3], const int (&ext)[3], const TopoL0& t0,
                                              float* ras, int64_t rs, mlbm_error_t* err) {
    for (int i = threadIdx.x; i < nbox; i += blockDim.x) {
        float tot[NV];
#pragma unroll
        for (int qv = 0; qv < NV; ++qv) {
            float v = sacc[qv * MAXN + i];
            for (int w2 = 1; w2 < NW; ++w2) v += sacc[(w2 * NV + qv) * MAXN + i];
            tot[qv] = v;
        }
        if (STRESS ? tot[NV - 1] == 0.f : (tot[0] == 0.f && tot[2 + 2 * D] == 0.f)) continue;
        int c[3];
        box_coord<D>(i, lo, ext, c);
        bool b2 = false;
        const int64_t ni = node_index<D>(t0, c, b2);
        if (ni < 0) { report_error(err, MLBM_ERR_STENCIL, 0, c[0], c[1], c[2]); continue; }
#pragma unroll
        for (int qv = 0; qv < NV - STRESS; ++qv)
            if (tot[qv] != 0.f) atomicAdd(&ras[qv * rs + ni], tot[qv]);
    }
}

// Node boxes of the fp32 P2G kernel (k_p2g_cell2): the block's
// box over all its rounds (use_smem: every warp accumulates into its own copy
// of it), or, when it overflows P2G2_MAXN nodes, each warp's fixed window (its
// middle particle's tile in x, y; the z layer pair its particles vote for) —
// runs outside it take global atomics.  Zeroes the copies in use.
template <int D, int NW, int ROUNDS, int NV>
__device__ __forceinline__ void p2g2_boxes(const PartArgs& P, float* sacc, int p0, int (&lo)[3],
                                           int (&ext)[3], int& nbox, bool& use_smem, bool& warp_box) {
    constexpr int MAXN = P2G2_MAXN, BT = 32 * NW;
    __shared__ int s_lo[3], s_hi[3];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // block node box over all rounds
    if (threadIdx.x < 3) { s_lo[threadIdx.x] = 0x7fffffff; s_hi[threadIdx.x] = -0x7fffffff; }
    __syncthreads();
    int wl[3] = {0, 0, 0}, wh[3] = {0, 0, 0};        // this warp's node box
    // the warp's fixed window for blocks whose box overflows: the tile (x, y)
    // of its middle particle, and in z the layer pair the warp's particles
    // vote for; runs outside it (drifted particles) take global atomics
    int bm[3] = {0, 0, 0};
    int zup = 0, zdown = 0;
    {
        const int pm = min(p0 + (wid * ROUNDS + ROUNDS / 2) * 32 + 16, P.n - 1);
#pragma unroll
        for (int a = 0; a < D; ++a) bm[a] = (int)floor(P.x[a * P.ps + pm] - 0.5);
    }
    {
        int bl[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff}, bh[3] = {-0x7fffffff, -0x7fffffff, -0x7fffffff};
#pragma unroll
        for (int r = 0; r < ROUNDS; ++r) {
            const int p = p0 + (wid * ROUNDS + r) * 32 + lane;   // this warp's chunk r
            int bz = bm[D - 1];
            if (p < P.n) {
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const int b = (int)floor(P.x[a * P.ps + p] - 0.5);
                    bl[a] = min(bl[a], b);
                    bh[a] = max(bh[a], b + 2);
                    if (a == D - 1) bz = b;
                }
            }
            zup += __popc(__ballot_sync(0xffffffffu, bz == bm[D - 1] + 1));
            zdown += __popc(__ballot_sync(0xffffffffu, bz == bm[D - 1] - 1));
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const int l2 = __reduce_min_sync(0xffffffffu, bl[a]);
            const int h2 = __reduce_max_sync(0xffffffffu, bh[a]);
            wl[a] = l2;
            wh[a] = h2;
            if (lane == 0 && l2 <= h2) { atomicMin(&s_lo[a], l2); atomicMax(&s_hi[a], h2); }
        }
    }
    __syncthreads();
    lo[0] = lo[1] = lo[2] = 0;
    ext[0] = ext[1] = ext[2] = 1;
    nbox = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) { lo[a] = s_lo[a]; ext[a] = s_hi[a] - s_lo[a] + 1; nbox *= ext[a]; }
    use_smem = nbox > 0 && nbox <= MAXN;                   // block-uniform
    // a block whose box is too large (particles drifted since the last sort, a
    // tile run ends) accumulates per warp in its own copy over a fixed window
    // (the warp's tile in x, y; two z layers); runs outside it add to HBM
    // directly
    warp_box = !use_smem;
    if (warp_box) {
        constexpr int EX = D == 3 ? 6 : 10, EZ = D == 3 ? 4 : 1;
        static_assert(EX * EX * EZ <= MAXN, "warp window fits a per-warp copy");
        if constexpr (D == 3) {
            lo[0] = bm[0] & ~3; lo[1] = bm[1] & ~3; lo[2] = zup >= zdown ? bm[2] : bm[2] - 1;
            ext[0] = EX; ext[1] = EX; ext[2] = EZ;
        } else {
            lo[0] = (bm[0] & ~3) - 2; lo[1] = (bm[1] & ~3) - 2;
            ext[0] = EX; ext[1] = EX;
        }
        nbox = EX * EX * EZ;
        float4* s4 = reinterpret_cast<float4*>(sacc + wid * NV * MAXN);
        for (int i = lane; i < NV * MAXN / 4; i += 32) s4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (use_smem) {
        // zero the [NW * NV rows][nbox] box copies as float4, iterating over a
        // power-of-two padded row (no integer division)
        constexpr int RP = MAXN / 4 <= 32 ? 32 : (MAXN / 4 <= 64 ? 64 : 128);
        static_assert(MAXN / 4 <= RP, "row padding");
        const int n4 = (nbox + 3) >> 2;
        float4* s4 = reinterpret_cast<float4*>(sacc);
        for (int i = threadIdx.x; i < NW * NV * RP; i += BT) {
            const int row = i / RP, c4 = i % RP;
            if (c4 < n4) s4[row * (MAXN / 4) + c4] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __syncthreads();
}

// Flush of the fp32 P2G node boxes into the raster rows: a warp window (the
// warp's own copy, lanes striding over it) or the block box (sum of the NW
// copies, after a block barrier).
template <int D, int NW, int NV>
__device__ __forceinline__ void p2g2_merge(const float* sacc, const int (&lo)[3], const int (&ext)[3], int nbox,
                                           bool use_smem, bool warp_box, const TopoL0& t0, float* ras,
                                           int64_t rs, mlbm_error_t* err) {
    constexpr int MAXN = P2G2_MAXN;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (warp_box) {
        __syncwarp();
        const float* wa = sacc + wid * NV * MAXN;
        for (int i = lane; i < nbox; i += 32) {
            float tot[NV];
#pragma unroll
            for (int qv = 0; qv < NV; ++qv) tot[qv] = wa[qv * MAXN + i];
            if (tot[0] == 0.f && tot[2 + 2 * D] == 0.f) continue;
            int c[3];
            box_coord<D>(i, lo, ext, c);
            bool b2 = false;
            const int64_t ni = node_index<D>(t0, c, b2);
            if (ni < 0) { report_error(err, MLBM_ERR_STENCIL, 0, c[0], c[1], c[2]); continue; }
#pragma unroll
            for (int qv = 0; qv < NV; ++qv)
                if (tot[qv] != 0.f) atomicAdd(&ras[qv * rs + ni], tot[qv]);
        }
        return;
    }
    if (!use_smem) return;
    __syncthreads();
    p2g_box_merge<D, NV, 0>(sacc, NW, MAXN, nbox, lo, ext, t0, ras, rs, err);
}

template <int D, int NW, int ROUNDS>
__global__ void __launch_bounds__(32 * NW, P2G2_MIN_BLOCKS) k_p2g_cell2(PartArgs P, TopoL0 t0, MatParams mp, float* ras,
                                                       int64_t rs, mlbm_error_t* err) {
    constexpr int K = Geo<D>::K, NV = 3 + 3 * D, NS = D * (D + 1) / 2;
    constexpr int MAXN = P2G2_MAXN, REC = 32, BT = 32 * NW;
    extern __shared__ __align__(16) float p2g_smem[];
    float* sacc = p2g_smem;                                  // [NW][NV][MAXN]
    float* slab = p2g_smem + NW * NV * MAXN;                 // [NW][REC / 4][32] float4
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int p0 = blockIdx.x * (BT * ROUNDS);
    int lo[3], ext[3], nbox;
    bool use_smem, warp_box;
    p2g2_boxes<D, NW, ROUNDS, NV>(P, sacc, p0, lo, ext, nbox, use_smem, warp_box);

    const int o[3] = {lane % 3, (lane / 3) % 3, D == 3 ? (lane / 9) % 3 : 0};
    const bool node_lane = lane < K;
    float c0[D], c1[D], c2[D], d0[D], d1[D], of[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int oa = o[a];
        c2[a] = oa == 1 ? -1.f : 0.5f;
        c1[a] = oa == 0 ? -1.5f : (oa == 1 ? 2.f : -0.5f);
        c0[a] = oa == 0 ? 1.125f : (oa == 1 ? -0.25f : 0.125f);
        d1[a] = oa == 1 ? -2.f : 1.f;
        d0[a] = oa == 0 ? -1.5f : (oa == 1 ? 2.f : -0.5f);
        of[a] = (float)oa;
    }
    constexpr bool PAIRED = D == 3 && P2G2_PAIRED;
    // lane constants of the paired arithmetic (x / y weights and derivatives
    // in one pair each; z scalar)
    const float2 pC2xy = make_float2(c2[0], c2[D > 1 ? 1 : 0]), pC1xy = make_float2(c1[0], c1[D > 1 ? 1 : 0]),
                 pC0xy = make_float2(c0[0], c0[D > 1 ? 1 : 0]);
    const float2 pD1xy = make_float2(d1[0], d1[D > 1 ? 1 : 0]), pD0xy = make_float2(d0[0], d0[D > 1 ? 1 : 0]);
    const float2 pO0 = make_float2(of[0], of[0]), pO1 = make_float2(of[D > 1 ? 1 : 0], of[D > 1 ? 1 : 0]),
                 pO2 = make_float2(of[D - 1], of[D - 1]);
    float* wacc = sacc + wid * NV * MAXN;
    float* wslab = &slab[wid * 32 * REC];
    float acc[NV];
    int cur[3] = {0, 0, 0};
    bool bad = false;
    constexpr int OF = 3, OM = 3 + D, OQ = 6 + D, OMV = 6 + 2 * D, OS = 6 + 3 * D, OP = 6 + 3 * D + NS;
    constexpr int NREC4 = (OP + D * D + 3) / 4;
#pragma unroll 1
    for (int rd = 0; rd < ROUNDS; ++rd) {
        // warp w owns the consecutive chunks w * ROUNDS .. w * ROUNDS + ROUNDS - 1:
        // its particles are contiguous in the sorted order, so its node box
        // stays small when the block box overflows (-1 % on C4 against
        // interleaved chunks; a sliding per-warp box instead of the per-run
        // atomic fallback measured +9 %)
        const int pw = p0 + (wid * ROUNDS + rd) * 32;     // first particle of this warp's chunk
        const int nj = min(32, P.n - pw);
        if (nj <= 0) break;                               // warp-uniform
        const int p = pw + lane;
        int base[3];
        {
            // the record is built in registers and stored chunk-major
            // ([chunk][lane] float4): the 128-bit stores are conflict-free (a
            // lane-major 128 B record stride is an 8-way conflict) and the
            // broadcast reads of particle j sit at constant offsets from j
            float rec[REC];
#pragma unroll
            for (int k = 0; k < REC; ++k) rec[k] = 0.f;
            p2g_record<D>(P, mp, p, lane < nj, rec);
            float4* w4 = reinterpret_cast<float4*>(wslab) + lane;
            if constexpr (PAIRED) {
                float pr[28];
                p2g_pair_record(rec, pr);
#pragma unroll
                for (int v4 = 0; v4 < 7; ++v4)
                    w4[v4 * 32] = make_float4(pr[4 * v4], pr[4 * v4 + 1], pr[4 * v4 + 2], pr[4 * v4 + 3]);
            } else {
#pragma unroll
                for (int v4 = 0; v4 < NREC4; ++v4)
                    w4[v4 * 32] = make_float4(rec[4 * v4], rec[4 * v4 + 1], rec[4 * v4 + 2], rec[4 * v4 + 3]);
            }
#pragma unroll
            for (int a = 0; a < 3; ++a) base[a] = __float_as_int(rec[a]);
        }
        __syncwarp();
        // runs of equal stencil base (particles sorted by cell)
        bool start = lane < nj;
        {
            bool same = lane > 0;
#pragma unroll
            for (int a = 0; a < D; ++a) same &= __shfl_up_sync(0xffffffffu, base[a], 1) == base[a];
            start &= !same;
        }
        unsigned runs = __ballot_sync(0xffffffffu, start);
        while (runs) {
            const int j0 = __ffs(runs) - 1;
            runs &= runs - 1;
            const int j1 = runs ? __ffs(runs) - 1 : nj;
    #pragma unroll
            for (int a = 0; a < 3; ++a) cur[a] = __shfl_sync(0xffffffffu, a < D ? base[a] : 0, j0);
    #pragma unroll
            for (int qv = 0; qv < NV; ++qv) acc[qv] = 0.f;
            if constexpr (PAIRED) {
                // rows: (m V0) (ap mv0) (mv1 mv2) (mom0 mom1) mom2; the force
                // rows as (b = 1, b = 0) pair partial sums + the b = 2 term
                const float2 z2 = make_float2(0.f, 0.f);
                float2 aMV = z2, aA = z2, aV = z2, aM = z2, aF0 = z2, aF1 = z2, aF2 = z2;
                float aM2 = 0.f, aG0 = 0.f, aG1 = 0.f, aG2 = 0.f;
                for (int j = j0; j < j1; ++j) {
                    const float4* rp = reinterpret_cast<const float4*>(wslab) + j;
                    float4 t[7];
    #pragma unroll
                    for (int v4 = 0; v4 < 7; ++v4) t[v4] = rp[v4 * 32];
                    const float2 Fxy = make_float2(t[0].x, t[0].y);
                    const float fz = t[0].z;
                    const float2 Wxy = __ffma2_rn(__ffma2_rn(pC2xy, Fxy, pC1xy), Fxy, pC0xy);
                    const float wz = fmaf(fmaf(c2[2], fz, c1[2]), fz, c0[2]);
                    const float2 T = make_float2(Wxy.y * wz, Wxy.x * wz);         // (wy wz, wx wz)
                    const float2 G01 = __fmul2_rn(__ffma2_rn(pD1xy, Fxy, pD0xy), T);  // (g0, g1)
                    const float2 W2 = make_float2(T.x * Wxy.x, T.y * Wxy.y);       // (w, w)
                    const float g2 = (Wxy.x * Wxy.y) * fmaf(d1[2], fz, d0[2]);
                    aMV = __ffma2_rn(W2, make_float2(t[1].x, t[1].y), aMV);
                    aA = __ffma2_rn(W2, make_float2(t[1].z, t[1].w), aA);
                    aV = __ffma2_rn(W2, make_float2(t[2].x, t[2].y), aV);
                    float2 mo = __ffma2_rn(make_float2(t[3].x, t[3].y), pO0, make_float2(t[2].z, t[2].w));
                    mo = __ffma2_rn(make_float2(t[3].z, t[3].w), pO1, mo);
                    mo = __ffma2_rn(make_float2(t[4].x, t[4].y), pO2, mo);
                    aM = __ffma2_rn(W2, mo, aM);
                    float mo2 = fmaf(t[4].z, of[0], t[0].w);
                    mo2 = fmaf(t[4].w, of[1], mo2);
                    mo2 = fmaf(t[5].x, of[2], mo2);
                    aM2 = fmaf(W2.x, mo2, aM2);
                    aF0 = __ffma2_rn(make_float2(t[5].z, t[5].w), G01, aF0);
                    aF1 = __ffma2_rn(make_float2(t[6].x, t[6].y), G01, aF1);
                    aF2 = __ffma2_rn(make_float2(t[6].z, t[6].w), G01, aF2);
                    aG0 = fmaf(t[6].z, g2, aG0);
                    aG1 = fmaf(t[6].w, g2, aG1);
                    aG2 = fmaf(t[5].y, g2, aG2);
                }
                acc[0] = aMV.x;
                acc[1] = aM.x; acc[2] = aM.y; acc[3] = aM2;
                acc[4] = aF0.x + aF0.y + aG0; acc[5] = aF1.x + aF1.y + aG1; acc[6] = aF2.x + aF2.y + aG2;
                acc[7] = aMV.y; acc[8] = aA.x;
                acc[9] = aA.y; acc[10] = aV.x; acc[11] = aV.y;
            } else
            for (int j = j0; j < j1; ++j) {
                const float4* rp = reinterpret_cast<const float4*>(wslab) + j;
                float r[4 * NREC4];
    #pragma unroll
                for (int v4 = 0; v4 < NREC4; ++v4) {
                    const float4 t = rp[v4 * 32];
                    r[4 * v4] = t.x; r[4 * v4 + 1] = t.y; r[4 * v4 + 2] = t.z; r[4 * v4 + 3] = t.w;
                }
                float wa[D], dwa[D];
    #pragma unroll
                for (int a = 0; a < D; ++a) {
                    const float fa = r[OF + a];
                    wa[a] = fmaf(fmaf(c2[a], fa, c1[a]), fa, c0[a]);
                    dwa[a] = fmaf(d1[a], fa, d0[a]);
                }
                float w = wa[0];
    #pragma unroll
                for (int a = 1; a < D; ++a) w *= wa[a];
                float g[D];
    #pragma unroll
                for (int b = 0; b < D; ++b) {
                    float gb = dwa[b];
    #pragma unroll
                    for (int e = 0; e < D; ++e) if (e != b) gb *= wa[e];
                    g[b] = gb;
                }
                acc[0] = fmaf(w, r[OM], acc[0]);
                acc[1 + 2 * D] = fmaf(w, r[OM + 1], acc[1 + 2 * D]);
                acc[2 + 2 * D] = fmaf(w, r[OM + 2], acc[2 + 2 * D]);
    #pragma unroll
                for (int a = 0; a < D; ++a) {
                    float mo = r[OQ + a];
    #pragma unroll
                    for (int b = 0; b < D; ++b) mo = fmaf(r[OP + a * D + b], of[b], mo);
                    acc[1 + a] = fmaf(w, mo, acc[1 + a]);
                    float fa = acc[1 + D + a];
    #pragma unroll
                    for (int b = 0; b < D; ++b) {
                        const int sk = a <= b ? a * D - a * (a - 1) / 2 + (b - a) : b * D - b * (b - 1) / 2 + (a - b);
                        fa = fmaf(-r[OS + sk], g[b], fa);
                    }
                    acc[1 + D + a] = fa;
                    acc[3 + 2 * D + a] = fmaf(w, r[OMV + a], acc[3 + 2 * D + a]);
                }
            }
            bool inbox = true;                                   // warp-uniform
            if (warp_box) {
    #pragma unroll
                for (int a = 0; a < D; ++a) inbox &= cur[a] >= lo[a] && cur[a] + 2 < lo[a] + ext[a];
            }
            if (node_lane && (acc[0] != 0.f || acc[2 + 2 * D] != 0.f)) {
                int c[3] = {cur[0] + o[0], cur[1] + o[1], D == 3 ? cur[2] + o[2] : 0};
                if (inbox) {
                    int li = 0;
    #pragma unroll
                    for (int a = D - 1; a >= 0; --a) li = li * ext[a] + (c[a] - lo[a]);
    #pragma unroll
                    for (int qv = 0; qv < NV; ++qv) wacc[qv * MAXN + li] += acc[qv];
                } else {
                    const int64_t ni = node_index<D>(t0, c, bad);
                    if (ni >= 0) {
    #pragma unroll
                        for (int qv = 0; qv < NV; ++qv) atomicAdd(&ras[qv * rs + ni], acc[qv]);
                    }
                }
            }
            __syncwarp();
        }
        __syncwarp();                                     // slab reused next round
    }
    if (bad) report_error(err, MLBM_ERR_STENCIL, 0, cur[0], cur[1], cur[2]);
    p2g2_merge<D, NW, NV>(sacc, lo, ext, nbox, use_smem, warp_box, t0, ras, rs, err);
}

// Entrainment stress raster (coupling.py:283-294) in the P2G layout: sum over
// particles of V0 w_i tau (NS rows of RW::SIG) with post-G2P positions.  Lane
// k = stencil node k of the current run of particles with equal stencil base;
// records (base, f, V0 tau) are broadcast from a per-warp slab; per-warp node
// box copies in shared memory, merged once into HBM (no per-particle atomics).
// surf (optional, [n0] 0/1): the raster is only READ at entrainment surface
// cells (k_powder_diffuse), so a run none of whose 27 nodes is a surface cell
// is skipped before its particles' Kirchhoff stress is evaluated; the sums at
// surface nodes are unchanged (same runs, same order).  Every run's nodes are
// still checked for storage (stencil errors as in the reference).
template <int D, int NW>
__global__ void __launch_bounds__(32 * NW) k_stress_cell2(PartArgs P, TopoL0 t0, MatParams mp, float* ras,
                                                          int64_t rs, const float* __restrict__ surf,
                                                          mlbm_error_t* err) {
    constexpr int K = Geo<D>::K, NS = D * (D + 1) / 2, NV = NS + 1;
    constexpr int MAXN = STRESS_MAXN, REC = 16, BT = 32 * NW;
    using PR = PRows<D>;
    using RW = Rows<D>;
    extern __shared__ __align__(16) float p2g_smem[];
    float* sacc = p2g_smem;                                  // [NW][NV][MAXN]
    float* slab = p2g_smem + NW * NV * MAXN;                 // [NW][REC / 4][32] float4
    __shared__ int s_lo[3], s_hi[3];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int p = blockIdx.x * BT + threadIdx.x;
    const int pw = blockIdx.x * BT + wid * 32;
    const int nj = max(0, min(32, P.n - pw));
    const bool valid = lane < nj;
    if (threadIdx.x < 3) { s_lo[threadIdx.x] = 0x7fffffff; s_hi[threadIdx.x] = -0x7fffffff; }
    int base[3] = {0, 0, 0};
    float f[D];
#pragma unroll
    for (int a = 0; a < D; ++a) f[a] = 0.f;
    if (valid) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const double x = P.x[a * P.ps + p];
            const double b = floor(x - 0.5);
            base[a] = (int)b;
            f[a] = (float)(x - b);
        }
    }
    // a particle's stencil is the 3^D node box centred on its nearest node
    // m = floor(x + 1/2) = base + 1; need[m] marks boxes that contain an
    // entrainment surface cell (k_surface_need), so one lookup per particle
    // decides whether its stress is rasterised at all
    bool need = false;
    bool bad = false;
    if (valid) {
        int m[3] = {base[0] + 1, base[1] + 1, D == 3 ? base[2] + 1 : 0};
        const int64_t ni = node_index<D>(t0, m, bad);
        need = ni >= 0 && (surf == nullptr || surf[ni] != 0.f);
    }
    const int o[3] = {lane % 3, (lane / 3) % 3, D == 3 ? (lane / 9) % 3 : 0};
    const bool node_lane = lane < K;
    // runs of equal stencil base among the needed particles
    bool start = need;
    {
        bool same = lane > 0;
#pragma unroll
        for (int a = 0; a < D; ++a) same &= __shfl_up_sync(0xffffffffu, base[a], 1) == base[a];
        same &= __shfl_up_sync(0xffffffffu, (int)need, 1) != 0;
        start &= !same;
    }
    const unsigned need_runs = __ballot_sync(0xffffffffu, start);
    const unsigned need_parts = __ballot_sync(0xffffffffu, need);
    const int bad_at[3] = {base[0] + 1, base[1] + 1, base[2] + (D == 3 ? 1 : 0)};
    // block node box over the particles of needed runs
    __syncthreads();
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int l2 = __reduce_min_sync(0xffffffffu, need ? base[a] : 0x7fffffff);
        const int h2 = __reduce_max_sync(0xffffffffu, need ? base[a] + 2 : -0x7fffffff);
        if (lane == 0 && l2 <= h2) { atomicMin(&s_lo[a], l2); atomicMax(&s_hi[a], h2); }
    }
    // per-particle record of needed particles: base[3] f[D] V0 tau[NS]
    float* wslab = &slab[wid * 32 * REC];
    if (need) {
        const float* pp = (const float*)P.p;
        float tau[D * D];
        load_tau<D, float>(pp, P.ps, p, tau);
        const float V0 = pp[PR::V0 * P.ps + p];
        float r[REC];
#pragma unroll
        for (int k = 0; k < REC; ++k) r[k] = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) r[a] = __int_as_float(a < D ? base[a] : 0);
#pragma unroll
        for (int a = 0; a < D; ++a) r[3 + a] = f[a];
        int k = 0;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a; b < D; ++b) r[3 + D + (k++)] = V0 * tau[a * D + b];
        // chunk-major records ([chunk][lane] float4): conflict-free 128-bit
        // stores, broadcast reads at constant offsets from the particle
        float4* w4 = reinterpret_cast<float4*>(wslab) + lane;
#pragma unroll
        for (int v4 = 0; v4 < 3; ++v4)
            w4[v4 * 32] = make_float4(r[4 * v4], r[4 * v4 + 1], r[4 * v4 + 2], r[4 * v4 + 3]);
    }
    __syncthreads();
    const int any_need = __syncthreads_or(need_runs != 0u);
    if (bad) report_error(err, MLBM_ERR_STENCIL, 0, bad_at[0], bad_at[1], bad_at[2]);
    if (!any_need) return;                                   // block-uniform
    int lo[3] = {0, 0, 0}, ext[3] = {1, 1, 1}, nbox = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) { lo[a] = s_lo[a]; ext[a] = s_hi[a] - s_lo[a] + 1; nbox *= ext[a]; }
    const bool use_smem = nbox > 0 && nbox <= MAXN;
    if (use_smem) {
        constexpr int RP = MAXN / 4 <= 32 ? 32 : (MAXN / 4 <= 64 ? 64 : 128);
        const int n4 = (nbox + 3) >> 2;
        float4* s4 = reinterpret_cast<float4*>(sacc);
        for (int i = threadIdx.x; i < NW * NV * RP; i += BT) {
            const int row = i / RP, c4 = i % RP;
            if (c4 < n4) s4[row * (MAXN / 4) + c4] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __syncthreads();

    float c0[D], c1[D], c2[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const int oa = o[a];
        c2[a] = oa == 1 ? -1.f : 0.5f;
        c1[a] = oa == 0 ? -1.5f : (oa == 1 ? 2.f : -0.5f);
        c0[a] = oa == 0 ? 1.125f : (oa == 1 ? -0.25f : 0.125f);
    }
    float* wacc = sacc + wid * NV * MAXN;
    unsigned runs = need_runs;
    while (runs) {
        const int j0 = __ffs(runs) - 1;
        runs &= runs - 1;
        // the run ends at the next run start or at the first non-needed lane
        const unsigned after = ~((2u << j0) - 1u);
        const unsigned stop = (need_runs | ~need_parts) & after;
        const int j1 = stop ? __ffs(stop) - 1 : 32;
        int cur[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) cur[a] = __shfl_sync(0xffffffffu, a < D ? base[a] : 0, j0);
        float acc[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = 0.f;
        for (int j = j0; j < j1; ++j) {
            const float4* rp = reinterpret_cast<const float4*>(wslab) + j;
            float r[12];
#pragma unroll
            for (int v4 = 0; v4 < 3; ++v4) {
                const float4 t = rp[v4 * 32];
                r[4 * v4] = t.x; r[4 * v4 + 1] = t.y; r[4 * v4 + 2] = t.z; r[4 * v4 + 3] = t.w;
            }
            float w = 1.f;
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const float fa = r[3 + a];
                w *= fmaf(fmaf(c2[a], fa, c1[a]), fa, c0[a]);
            }
#pragma unroll
            for (int q = 0; q < NS; ++q) acc[q] = fmaf(w, r[3 + D + q], acc[q]);
            acc[NS] += 1.f;
        }
        if (node_lane) {
            int c[3] = {cur[0] + o[0], cur[1] + o[1], D == 3 ? cur[2] + o[2] : 0};
            if (use_smem) {
                int li = 0;
#pragma unroll
                for (int a = D - 1; a >= 0; --a) li = li * ext[a] + (c[a] - lo[a]);
#pragma unroll
                for (int q = 0; q < NV; ++q) wacc[q * MAXN + li] += acc[q];
            } else {
                bool b2 = false;
                const int64_t ni = node_index<D>(t0, c, b2);
                if (ni >= 0) {
#pragma unroll
                    for (int q = 0; q < NS; ++q) atomicAdd(&ras[(RW::SIG + q) * rs + ni], acc[q]);
                }
            }
        }
        __syncwarp();
    }
    if (!use_smem) return;
    __syncthreads();
    p2g_box_merge<D, NV, 1>(sacc, NW, MAXN, nbox, lo, ext, t0, ras + (int64_t)RW::SIG * rs, rs, err);
}

// entrainment surface cells of level 0 (the source condition of
// k_powder_diffuse, coupling.py:300-316, without the speed test): 0 < eta <
// eta_surface and an absent / empty (eta < 1e-3) face neighbour.  Every
// surface cell marks need = 1 on the stored cells of its 3^D neighbourhood,
// i.e. on every nearest node whose stencil box contains it, and 2 on itself
// (need zeroed by the caller)
template <int D, typename R>
__global__ void __launch_bounds__(256) k_surface_need(mlbm_level_t lv, const R* __restrict__ ras, int64_t rs,
                                                      double eta_surface, float* __restrict__ need) {
    // one tile per T threads: the surface cells mark the tile's 6^D window
    // (tile + one-cell halo) in shared memory — no per-offset neighbour
    // lookups, no atomics — and the marked window cells are then written
    // once: the tile's own cells by plain stores, the halo cells (owned by
    // neighbour tiles, which may store 2 there) by an integer atomicMax of 1
    constexpr int T = Geo<D>::T, TPB = 256 / T, W6 = D == 3 ? 216 : 36;
    using RW = Rows<D>;
    __shared__ uint8_t win_all[TPB][W6];
    const int grp = threadIdx.x / T, lc = threadIdx.x % T;
    const int slot = blockIdx.x * TPB + grp;
    const bool valid = slot < live_tiles(lv);
    uint8_t* win = win_all[grp];
    for (int i = lc; i < W6; i += T) win[i] = 0;
    const int l[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    bool surf = false;
    if (valid) {
        const int64_t c = (int64_t)slot * T + lc;
        const R eta_c = ras[RW::ETAE * rs + c];
        if (eta_c > R(0) && eta_c < R(eta_surface)) {
            for (int a = 0; a < D; ++a)
                for (int sgn = 0; sgn < 2; ++sgn) {
                    const int64_t nb = face_nbr<D>(lv, slot, lc, a, sgn == 0 ? 1 : -1);
                    if (nb < 0 || ras[RW::ETAE * rs + nb] < R(1e-3)) surf = true;
                }
        }
    }
    const int wc = (l[0] + 1) + 6 * (l[1] + 1) + (D == 3 ? 36 * (l[2] + 1) : 0);
    __syncthreads();
    if (surf) {
#pragma unroll
        for (int k = 0; k < Geo<D>::K; ++k) {
            const int o[3] = {k % 3 - 1, (k / 3) % 3 - 1, D == 3 ? k / 9 - 1 : 0};
            win[wc + o[0] + 6 * o[1] + (D == 3 ? 36 * o[2] : 0)] = 1;
        }
    }
    const int any = __syncthreads_or(surf);
    if (!any) return;                                    // block-uniform
    if (surf) win[wc] = 2;                               // 2 on the surface cell itself
    __syncthreads();
    if (!valid) return;
    for (int i = lc; i < W6; i += T) {
        const uint8_t v = win[i];
        if (!v) continue;
        const int w[3] = {i % 6 - 1, (i / 6) % 6 - 1, D == 3 ? i / 36 - 1 : 0};
        int to[3] = {0, 0, 0}, ll[3] = {0, 0, 0};
        bool inside = true;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            to[a] = w[a] < 0 ? -1 : (w[a] > 3 ? 1 : 0);
            ll[a] = w[a] & 3;
            inside &= to[a] == 0;
        }
        if (inside) {
            need[(int64_t)slot * T + local_of<D>(ll[0], ll[1], ll[2])] = (float)v;
        } else {
            // a position outside a non-periodic domain or in an absent tile has
            // no neighbour slot (-1)
            const int ns = lv.nbr[(int64_t)slot * Geo<D>::NB + nb_index<D>(to[0], to[1], to[2])];
            if (ns >= 0)
                atomicMax(reinterpret_cast<int*>(&need[(int64_t)ns * T + local_of<D>(ll[0], ll[1], ll[2])]),
                          __float_as_int(1.f));
        }
    }
}

}  // namespace mlbm

using namespace mlbm;

static inline int nblk(int64_t n, int b) { return (int)((n + b - 1) / b); }
static TopoL0 topo0(const mlbm_level_t* lv) {
    TopoL0 t;
    for (int a = 0; a < 3; ++a) { t.cells[a] = lv->cells[a]; t.tiles[a] = lv->tiles[a]; t.periodic[a] = lv->periodic[a]; }
    t.tile_map = lv->tile_map;
    return t;
}

extern "C" int mlbm_raster_rows(int32_t dim) { return dim == 2 ? Rows<2>::N : Rows<3>::N; }
extern "C" int mlbm_particle_rows(int32_t dim) { return dim == 2 ? PRows<2>::N : PRows<3>::N; }

extern "C" int mlbm_p2g(const mlbm_level_t* lv0, int32_t n, const double* x, void* p, int64_t ps,
                        double lam, double mu, double alpha, void* ras, int64_t rs, int32_t dtype,
                        int32_t smem, mlbm_error_t* err, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    PartArgs P{lv0->dim, n, x, nullptr, p, ps, nullptr, nullptr, nullptr};
    MatParams mp = mat_params(lam, mu, alpha);
    const TopoL0 t = topo0(lv0);
    if ((smem == 4 || smem == 5) && dtype == 0) {
        // 4: one round of 32 * NW particles per block; 5: two rounds sharing
        // the block's node box (dense sampling, >= 8 per cell: 256 sorted
        // particles span <= 32 cells, whose box fits P2G2_MAXN)
        constexpr int NW = P2G2_NW;
        const int sh = (NW * (3 + 3 * 3) * P2G2_MAXN + NW * 32 * 32) * (int)sizeof(float);
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_p2g_cell2<3, NW, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
            cudaFuncSetAttribute(k_p2g_cell2<2, NW, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
            cudaFuncSetAttribute(k_p2g_cell2<3, NW, P2G2_ROUNDS_DENSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
            cudaFuncSetAttribute(k_p2g_cell2<2, NW, P2G2_ROUNDS_DENSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
            attr = true;
        }
        if (smem == 5) {
            constexpr int R2 = P2G2_ROUNDS_DENSE;
            if (lv0->dim == 2) k_p2g_cell2<2, NW, R2><<<nblk(n, 32 * NW * R2), 32 * NW, sh, s>>>(P, t, mp, (float*)ras, rs, err);
            else k_p2g_cell2<3, NW, R2><<<nblk(n, 32 * NW * R2), 32 * NW, sh, s>>>(P, t, mp, (float*)ras, rs, err);
        } else {
            if (lv0->dim == 2) k_p2g_cell2<2, NW, 1><<<nblk(n, 32 * NW), 32 * NW, sh, s>>>(P, t, mp, (float*)ras, rs, err);
            else k_p2g_cell2<3, NW, 1><<<nblk(n, 32 * NW), 32 * NW, sh, s>>>(P, t, mp, (float*)ras, rs, err);
        }
        return launch_status(1);
    }
    if (smem == 5) smem = 3;
    if (smem == 4) smem = 3;
#define P2G(D, R) do { if (smem == 3) k_p2g_cell<D, R><<<nblk(n, 128), 128, 0, s>>>(P, t, mp, (R*)ras, rs, err); \
                       else if (smem == 2) k_p2g_warp<D, R, 3><<<nblk(n, 128), 128, 0, s>>>(P, t, mp, (R*)ras, rs, err); \
                       else if (smem) k_p2g_smem<D, R><<<nblk(n, 256), 256, 0, s>>>(P, t, mp, (R*)ras, rs, err); \
                       else k_p2g<D, R><<<nblk(n, 128), 128, 0, s>>>(P, t, mp, (R*)ras, rs, err); } while (0)
    if (lv0->dim == 2) { if (dtype) P2G(2, double); else P2G(2, float); }
    else { if (dtype) P2G(3, double); else P2G(3, float); }
#undef P2G
    return launch_status(1);
}

// ---------------------------------------------------------------------------
// Particle sort by (level-0 tile slot, cell) without a library sort: a
// bucketed counting sort keyed by the live tile slot —
//   k_sort_keys     key = slot * T + cell of the stencil base (invalid: last bucket)
//   k_slot_hist     per-slot counts (atomics; sorted input hits few addresses)
//   scan            exclusive scan of the slot counts (the compaction scan of
//                   topology.cu, mlbm_scan_i32)
//   k_slot_scatter  particles into their slot's range
//   k_cell_sort     one CTA per slot: counting sort of its range by cell
//                   (shared-memory histogram + scan over the 4^D cells)
//   k_gather        every particle row into the sorted order
// Order inside a cell: by the particle's index before the sort (deterministic).
extern "C" int mlbm_scan_i32(int32_t n, int32_t* data, int32_t* total, void* ws, int64_t ws_bytes,
                             void* stream);
extern "C" int64_t mlbm_scan_ws_bytes(int32_t n);

// warp-aggregated: lanes with the same slot (sorted input: usually the whole
// warp) share one atomic; a lane's rank is its order among them
__global__ void k_slot_hist(int n, const uint32_t* __restrict__ keys, int tshift, int nslot,
                            int32_t* __restrict__ hist) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t k = p < n ? keys[p] : 0xfffffffeu;
    const int slot = k == 0xffffffffu ? nslot - 1 : (int)(k >> tshift);
    const unsigned peers = __match_any_sync(0xffffffffu, p < n ? slot : -1);
    const int lane = threadIdx.x & 31;
    if (p < n && (__ffs(peers) - 1) == lane) atomicAdd(&hist[slot], __popc(peers));
}

__global__ void k_slot_scatter(int n, const uint32_t* __restrict__ keys, int tshift, int nslot,
                               const int32_t* __restrict__ start, int32_t* __restrict__ fill,
                               int32_t* __restrict__ perm, uint8_t* __restrict__ cell) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t k = p < n ? keys[p] : 0xfffffffeu;
    const bool bad = k == 0xffffffffu;
    const int slot = bad ? nslot - 1 : (int)(k >> tshift);
    const unsigned peers = __match_any_sync(0xffffffffu, p < n ? slot : -1);
    const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
    int base = 0;
    if (p < n && lane == leader) base = atomicAdd(&fill[slot], __popc(peers));
    base = __shfl_sync(peers, base, leader);
    if (p >= n) return;
    const int pos = start[slot] + base + __popc(peers & ((1u << lane) - 1u));
    perm[pos] = p;
    cell[pos] = bad ? 0 : (uint8_t)(k & ((1u << tshift) - 1u));
}

template <int T>
__global__ void k_cell_sort(int nslot, const int32_t* __restrict__ start, const int32_t* __restrict__ perm_in,
                            const uint8_t* __restrict__ cell, int32_t* __restrict__ perm_out, int n) {
    __shared__ int cnt[T], off[T];
    const int slot = blockIdx.x;
    const int a = start[slot], b = slot + 1 < nslot ? start[slot + 1] : n;
    if (b - a <= 1) {
        if (b - a == 1 && threadIdx.x == 0) perm_out[a] = perm_in[a];
        return;
    }
    for (int c = threadIdx.x; c < T; c += blockDim.x) cnt[c] = 0;
    __syncthreads();
    for (int i = a + threadIdx.x; i < b; i += blockDim.x) atomicAdd(&cnt[cell[i]], 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int c = 0; c < T; ++c) { off[c] = t; t += cnt[c]; cnt[c] = 0; }
    }
    __syncthreads();
    for (int i = a + threadIdx.x; i < b; i += blockDim.x) {
        const int c = cell[i];
        perm_out[a + off[c] + atomicAdd(&cnt[c], 1)] = perm_in[i];
    }
    __syncthreads();
    // deterministic order: each cell's particles by their index before the
    // sort (insertion sort of a few entries per cell, one thread per cell)
    for (int c = threadIdx.x; c < T; c += blockDim.x) {
        const int lo = a + off[c], hi = lo + cnt[c];
        for (int i = lo + 1; i < hi; ++i) {
            const int v = perm_out[i];
            int j = i - 1;
            while (j >= lo && perm_out[j] > v) { perm_out[j + 1] = perm_out[j]; --j; }
            perm_out[j + 1] = v;
        }
    }
}

static int64_t al256(int64_t v) { return (v + 255) & ~(int64_t)255; }

extern "C" int64_t mlbm_sort_ws_bytes(int64_t n, int64_t n_slots) {
    if (n < 1) n = 1;
    const int64_t ns = n_slots + 1;
    // keys, perm, perm2 (n int32 each), cell (n bytes), hist, fill (ns int32), scan ws
    return 3 * al256(4 * n) + al256(n) + 2 * al256(4 * ns) + al256(mlbm_scan_ws_bytes((int32_t)ns)) + 256;
}

extern "C" int mlbm_particle_sort(const mlbm_level_t* lv0, int32_t n, const double* x, const void* p,
                                  const int32_t* pid, int64_t ps, double* x_out, void* p_out,
                                  int32_t* pid_out, int32_t dtype, void* ws, int64_t ws_bytes,
                                  void* stream) {
    if (n <= 0) return 0;
    const int nslot = lv0->n_tiles + 1;           // capacity slots + the invalid bucket
    if (ws_bytes < mlbm_sort_ws_bytes(n, lv0->n_tiles)) return -1;
    char* w = (char*)ws;
    uint32_t* keys = (uint32_t*)w;                 w += al256(4 * (int64_t)n);
    int32_t* perm = (int32_t*)w;                   w += al256(4 * (int64_t)n);
    int32_t* perm2 = (int32_t*)w;                  w += al256(4 * (int64_t)n);
    uint8_t* cell = (uint8_t*)w;                   w += al256(n);
    int32_t* hist = (int32_t*)w;                   w += al256(4 * (int64_t)nslot);
    int32_t* fill = (int32_t*)w;                   w += al256(4 * (int64_t)nslot);
    void* sws = w;
    const int64_t sws_b = mlbm_scan_ws_bytes(nslot);
    cudaStream_t s = as_stream(stream);
    const TopoL0 t = topo0(lv0);
    const int tshift = lv0->dim == 2 ? 4 : 6;
    if (lv0->dim == 2) k_sort_keys<2><<<nblk(n, 256), 256, 0, s>>>(n, x, ps, t, keys, perm2);
    else k_sort_keys<3><<<nblk(n, 256), 256, 0, s>>>(n, x, ps, t, keys, perm2);
    cudaMemsetAsync(hist, 0, 2 * al256(4 * (int64_t)nslot), s);       // hist + fill
    k_slot_hist<<<nblk(n, 256), 256, 0, s>>>(n, keys, tshift, nslot, hist);
    const int ks = mlbm_scan_i32(nslot, hist, nullptr, sws, sws_b, s);
    if (ks < 0) return ks;
    k_slot_scatter<<<nblk(n, 256), 256, 0, s>>>(n, keys, tshift, nslot, hist, fill, perm, cell);
    if (lv0->dim == 2) k_cell_sort<16><<<nslot, 128, 0, s>>>(nslot, hist, perm, cell, perm2, n);
    else k_cell_sort<64><<<nslot, 128, 0, s>>>(nslot, hist, perm, cell, perm2, n);
    const int rows = lv0->dim == 2 ? PRows<2>::N : PRows<3>::N;
    if (dtype) k_gather_particles<double><<<nblk(n, 256), 256, 0, s>>>(n, rows, perm2, x, lv0->dim, (const double*)p, pid, ps, x_out, (double*)p_out, pid_out);
    else k_gather_particles<float><<<nblk(n, 256), 256, 0, s>>>(n, rows, perm2, x, lv0->dim, (const float*)p, pid, ps, x_out, (float*)p_out, pid_out);
    return launch_status(6 + ks);
}

extern "C" int mlbm_exchange(const mlbm_level_t* lv0, mlbm_fields_t w_tree, mlbm_fields_t r_tree,
                             mlbm_fields_t tree0, mlbm_fields_t tree1, void* ras, int64_t rs,
                             double eps_min, double nu, double d_p, double re_min, double dt,
                             double rho0, const double* g_fluid, const double* g_sed,
                             const int32_t* faces, double floor_friction, int32_t mode,
                             int32_t dtype, void* stream) {
    const int T = lv0->dim == 2 ? 16 : 64;
    const int64_t n = (int64_t)lv0->n_tiles * T;
    if (n == 0) return 0;
    ExchArgs A;
    A.lv = *lv0; A.w_tree = w_tree; A.r_tree = r_tree; A.tree0 = tree0; A.tree1 = tree1;
    A.ras = ras; A.rs = rs; A.eps_min = eps_min; A.nu = nu; A.d_p = d_p; A.re_min = re_min;
    A.dt = dt; A.rho0 = rho0;
    for (int a = 0; a < 3; ++a) { A.g_fluid[a] = g_fluid[a]; A.g_sed[a] = g_sed[a]; }
    for (int f = 0; f < 6; ++f) A.face[f] = faces[f];
    A.floor_friction = floor_friction;
    A.mode = mode;
    cudaStream_t s = as_stream(stream);
#define EX(D, R) k_exchange<D, R><<<nblk(n, 128), 128, 0, s>>>(A)
    if (lv0->dim == 2) { if (dtype) EX(2, double); else EX(2, float); }
    else { if (dtype) EX(3, double); else EX(3, float); }
#undef EX
    return launch_status(1);
}

extern "C" int mlbm_g2p(const mlbm_level_t* lv0, int32_t n, const double* x_in, double* x_out,
                        const void* p_in, void* p_out, const int32_t* pid_in, int32_t* pid_out,
                        int64_t ps, double lam, double mu, double alpha, const mlbm_snow_t* snow,
                        const void* ras, int64_t rs,
                        double dt, int32_t plastic, int32_t dtype, int32_t* clamped,
                        uint8_t* seeds, const uint8_t* kind0, int32_t* nonleaf,
                        mlbm_error_t* err, void* stream) {
    if (n <= 0) return 0;
    if (seeds && (!kind0 || !nonleaf)) return -1;
    cudaStream_t s = as_stream(stream);
    PartArgs P{lv0->dim, n, x_in, x_out, (void*)p_in, ps, p_out, pid_in, pid_in ? pid_out : nullptr,
               seeds, kind0, nonleaf};
    MatParams mp = mat_params(lam, mu, alpha, snow);
    const TopoL0 t = topo0(lv0);
    const int mat = !plastic ? 0 : (mp.snow ? 2 : 1);
#define G2P(D, R) do { if (mat == 0) k_g2p<D, R, 0><<<nblk(n, G2P_BT), G2P_BT, 0, s>>>(P, t, mp, (const R*)ras, rs, dt, clamped, err); \
                       else if (mat == 1) k_g2p<D, R, 1><<<nblk(n, G2P_BT), G2P_BT, 0, s>>>(P, t, mp, (const R*)ras, rs, dt, clamped, err); \
                       else k_g2p<D, R, 2><<<nblk(n, G2P_BT), G2P_BT, 0, s>>>(P, t, mp, (const R*)ras, rs, dt, clamped, err); } while (0)
    if (lv0->dim == 2) { if (dtype) G2P(2, double); else G2P(2, float); }
    else { if (dtype) G2P(3, double); else G2P(3, float); }
#undef G2P
    return launch_status(1);
}

static int stress_raster_impl(const mlbm_level_t* lv0, int32_t n, const double* x, const void* p,
                              int64_t ps, double lam, double mu, double alpha, void* ras, int64_t rs,
                              int32_t dtype, const float* surf, mlbm_error_t* err, cudaStream_t s) {
    PartArgs P{lv0->dim, n, x, nullptr, (void*)p, ps, nullptr, nullptr, nullptr};
    MatParams mp = mat_params(lam, mu, alpha);
    const TopoL0 t = topo0(lv0);
    if (dtype == 0 && !getenv("MLBM_STRESS_ATOMIC")) {
        // fp32: the P2G layout (sorted particles, per-warp node boxes)
        constexpr int NW = P2G2_NW;
        const int sh = (NW * 7 * STRESS_MAXN + NW * 32 * 16) * (int)sizeof(float);   // NV <= 7
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_stress_cell2<3, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
            cudaFuncSetAttribute(k_stress_cell2<2, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh);
            attr = true;
        }
        if (lv0->dim == 2) k_stress_cell2<2, NW><<<nblk(n, 32 * NW), 32 * NW, sh, s>>>(P, t, mp, (float*)ras, rs, surf, err);
        else k_stress_cell2<3, NW><<<nblk(n, 32 * NW), 32 * NW, sh, s>>>(P, t, mp, (float*)ras, rs, surf, err);
        return 1;
    }
#define SR(D, R) k_stress_raster<D, R><<<nblk(n, 128), 128, 0, s>>>(P, t, mp, (R*)ras, rs, err)
    if (lv0->dim == 2) { if (dtype) SR(2, double); else SR(2, float); }
    else { if (dtype) SR(3, double); else SR(3, float); }
#undef SR
    return 1;
}

extern "C" int mlbm_stress_raster(const mlbm_level_t* lv0, int32_t n, const double* x, const void* p,
                                  int64_t ps, double lam, double mu, double alpha, void* ras, int64_t rs,
                                  int32_t dtype, mlbm_error_t* err, void* stream) {
    if (n <= 0) return 0;
    const int k = stress_raster_impl(lv0, n, x, p, ps, lam, mu, alpha, ras, rs, dtype, nullptr, err,
                                     as_stream(stream));
    return launch_status(k);
}

extern "C" int mlbm_stress_raster_surface(const mlbm_level_t* lv0, int32_t n, const double* x,
                                          const void* p, int64_t ps, double lam, double mu, double alpha,
                                          void* ras, int64_t rs, double eta_surface, void* surf,
                                          int32_t dtype, mlbm_error_t* err, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    if (dtype != 0)   // fp64 (parity runs): the full raster
        return launch_status(stress_raster_impl(lv0, n, x, p, ps, lam, mu, alpha, ras, rs, dtype, nullptr,
                                                err, s));
    const int T = lv0->dim == 2 ? 16 : 64;
    const int64_t ncell = (int64_t)lv0->n_tiles * T;
    if (ncell > 0) {
        cudaMemsetAsync(surf, 0, (size_t)ncell * sizeof(float), s);
        if (lv0->dim == 2) k_surface_need<2, float><<<nblk(lv0->n_tiles, 16), 256, 0, s>>>(*lv0, (const float*)ras, rs, eta_surface, (float*)surf);
        else k_surface_need<3, float><<<nblk(lv0->n_tiles, 4), 256, 0, s>>>(*lv0, (const float*)ras, rs, eta_surface, (float*)surf);
    }
    const int k = stress_raster_impl(lv0, n, x, p, ps, lam, mu, alpha, ras, rs, dtype, (const float*)surf,
                                     err, s);
    return launch_status(k + (ncell > 0 ? 1 : 0));
}

extern "C" int mlbm_powder(const mlbm_level_t* lv0, mlbm_fields_t src, mlbm_fields_t dst, void* ras,
                           int64_t rs, void* tmp, uint8_t* tile_ws, double diffusion, double sign,
                           double dt, double entrain, double eta_surface, int32_t with_source,
                           int32_t dtype, void* stream) {
    const int T = lv0->dim == 2 ? 16 : 64;
    const int64_t n = (int64_t)lv0->n_tiles * T;
    if (n == 0) return 0;
    PowderArgs A{*lv0, src, dst, ras, rs, tmp, diffusion, sign, dt, entrain, eta_surface, with_source,
                 nullptr, tile_ws ? tile_ws + lv0->n_tiles : nullptr};
    cudaStream_t s = as_stream(stream);
    const int nt = lv0->n_tiles;
    int k = 2;
    if (tile_ws) {
        k += 2;
        if (lv0->dim == 2) {
            if (dtype) k_phi_tiles<2, double><<<nblk(nt, 128), 128, 0, s>>>(*lv0, src, tile_ws);
            else k_phi_tiles<2, float><<<nblk(nt, 128), 128, 0, s>>>(*lv0, src, tile_ws);
            k_phi_region<2><<<nblk(nt, 128), 128, 0, s>>>(*lv0, tile_ws, tile_ws + nt);
        } else {
            if (dtype) k_phi_tiles<3, double><<<nblk(nt, 128), 128, 0, s>>>(*lv0, src, tile_ws);
            else k_phi_tiles<3, float><<<nblk(nt, 128), 128, 0, s>>>(*lv0, src, tile_ws);
            k_phi_region<3><<<nblk(nt, 128), 128, 0, s>>>(*lv0, tile_ws, tile_ws + nt);
        }
    }
#define PW(D, R) do { if (D == 3) k_powder_advect_tile<R><<<nt, 64, 0, s>>>(A); \
                      else k_powder_advect<D, R><<<nblk(n, 128), 128, 0, s>>>(A); \
                      k_powder_diffuse<D, R><<<nblk(n, 128), 128, 0, s>>>(A); } while (0)
    if (lv0->dim == 2) { if (dtype) PW(2, double); else PW(2, float); }
    else { if (dtype) PW(3, double); else PW(3, float); }
#undef PW
    return launch_status(k);
}

// fp32 fluid diagnostics, 4 consecutive cells per thread: the flags as one
// 32-bit load, each field row as one 16-byte load (same sums as k_diag_level
// up to the summation order)
template <int D>
__global__ void __launch_bounds__(256) k_diag_level4(mlbm_level_t lv, mlbm_fields_t f, double vol, double* out) {
    constexpr int T = Geo<D>::T;
    double acc[D + 1];
#pragma unroll
    for (int k = 0; k <= D; ++k) acc[k] = 0.0;
    double emin = 1e300;
    const float* p = (const float*)f.ptr;
    const int64_t s = f.stride;
    const int64_t n4 = (int64_t)live_tiles(lv) * (T / 4);
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = (int64_t)lv.first * (T / 4) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += st) {
        const int64_t c = q * 4;
        const unsigned fl = *reinterpret_cast<const unsigned*>(lv.cell_flags + c);
        if (!(fl & 0x01010101u * MLBM_CF_LEAF)) continue;
        const float4 r4 = *reinterpret_cast<const float4*>(p + c);
        float4 u4[D];
#pragma unroll
        for (int a = 0; a < D; ++a) u4[a] = *reinterpret_cast<const float4*>(p + (1 + a) * s + c);
        const float4 ph4 = *reinterpret_cast<const float4*>(p + fi_phi<D>() * s + c);
        const float4 ep4 = *reinterpret_cast<const float4*>(p + fi_eps<D>() * s + c);
        const float rr[4] = {r4.x, r4.y, r4.z, r4.w}, ph[4] = {ph4.x, ph4.y, ph4.z, ph4.w},
                    ep[4] = {ep4.x, ep4.y, ep4.z, ep4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (!((fl >> (8 * u)) & MLBM_CF_LEAF)) continue;
            const double rho = 1.0 + (double)rr[u];
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const float ua = u == 0 ? u4[a].x : u == 1 ? u4[a].y : u == 2 ? u4[a].z : u4[a].w;
                acc[a] += vol * rho * (double)ua;
            }
            acc[D] += vol * (double)ph[u];
            emin = fmin(emin, (double)ep[u]);
        }
    }
    __shared__ double smin[32];
    for (int off = 16; off > 0; off >>= 1) emin = fmin(emin, __shfl_down_sync(0xffffffffu, emin, off));
    if ((threadIdx.x & 31) == 0) smin[threadIdx.x >> 5] = emin;
    block_sum_atomic<D + 1>(acc, out);          // contains __syncthreads
    if (threadIdx.x == 0) {
        double m = smin[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, smin[w]);
        if (m < 1e300 && m < *(volatile double*)&out[D + 1]) atomic_min_double(&out[D + 1], m);
    }
}

extern "C" int mlbm_diag_level(const mlbm_level_t* lv, mlbm_fields_t f, double vol, int32_t dtype,
                               double* out, void* stream) {
    const int T = lv->dim == 2 ? 16 : 64;
    const int64_t n = (int64_t)lv->n_tiles * T;
    if (n == 0) return 0;
    cudaStream_t s = as_stream(stream);
    static int sms = 0;
    if (!sms) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev); }
    const int gb = (int)std::min<int64_t>(nblk(n, 256 * 4), (int64_t)sms * 4);
    if (dtype == 0 && f.stride % 4 == 0) {
        const int gb4 = (int)std::min<int64_t>(nblk(n / 4, 256), (int64_t)sms * 8);
        if (lv->dim == 2) k_diag_level4<2><<<gb4, 256, 0, s>>>(*lv, f, vol, out);
        else k_diag_level4<3><<<gb4, 256, 0, s>>>(*lv, f, vol, out);
        return launch_status(1);
    }
#define DG(D, R) k_diag_level<D, R><<<gb, 256, 0, s>>>(*lv, f, vol, out)
    if (lv->dim == 2) { if (dtype) DG(2, double); else DG(2, float); }
    else { if (dtype) DG(3, double); else DG(3, float); }
#undef DG
    return launch_status(1);
}

// fp32 particle diagnostics, 4 consecutive particles / cells per thread with
// 16-byte row loads (same sums as k_diag_particles up to the summation order)
template <int D>
__global__ void __launch_bounds__(256) k_diag_particles4(PartArgs P, const float* ras, int64_t rs, int64_t n0,
                                                          const int32_t* live, double* out) {
    using PR = PRows<D>;
    if (live) n0 = min(n0, (int64_t)live[0] * Geo<D>::T);
    double acc[2 * D];
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) acc[k] = 0.0;
    const float* pp = (const float*)P.p;
    const int64_t st = (int64_t)gridDim.x * blockDim.x;
    const int64_t np4 = P.n / 4, nc4 = n0 / 4;
    const int64_t m4 = np4 > nc4 ? np4 : nc4;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m4; q += st) {
        const int64_t i = q * 4;
        if (q < np4) {
            const float4 m = *reinterpret_cast<const float4*>(pp + PR::M * P.ps + i);
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const float4 v = *reinterpret_cast<const float4*>(pp + (PR::V + a) * P.ps + i);
                acc[a] += (double)m.x * (double)v.x + (double)m.y * (double)v.y + (double)m.z * (double)v.z +
                          (double)m.w * (double)v.w;
            }
        }
        if (ras && q < nc4) {
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const float4 f = *reinterpret_cast<const float4*>(ras + (Rows<D>::FS + a) * rs + i);
                acc[D + a] += (double)f.x + (double)f.y + (double)f.z + (double)f.w;
            }
        }
    }
    // the ragged ends (n, n0 not multiples of 4)
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g < P.n - np4 * 4) {
        const int64_t i = np4 * 4 + g;
        const double m = pp[PR::M * P.ps + i];
#pragma unroll
        for (int a = 0; a < D; ++a) acc[a] += m * (double)pp[(PR::V + a) * P.ps + i];
    }
    if (ras && g < n0 - nc4 * 4) {
        const int64_t i = nc4 * 4 + g;
#pragma unroll
        for (int a = 0; a < D; ++a) acc[D + a] += (double)ras[(Rows<D>::FS + a) * rs + i];
    }
    block_sum_atomic<2 * D>(acc, out);
}

extern "C" int mlbm_diag_particles(int32_t dim, int32_t n, const void* p, int64_t ps, const void* ras,
                                   int64_t rs, int64_t n0, const int32_t* live, int32_t dtype,
                                   double* out, void* stream) {
    const int64_t m = n > n0 ? n : n0;
    if (m == 0) return 0;
    PartArgs P{dim, n, nullptr, nullptr, (void*)p, ps, nullptr, nullptr, nullptr};
    cudaStream_t s = as_stream(stream);
    static int sms = 0;
    if (!sms) { int dev = 0; cudaGetDevice(&dev); cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev); }
    const int gb = (int)std::min<int64_t>(nblk(m, 256 * 4), (int64_t)sms * 4);
    if (dtype == 0 && ps % 4 == 0 && rs % 4 == 0) {
        const int gb4 = (int)std::max<int64_t>(1, std::min<int64_t>(nblk(m / 4, 256), (int64_t)sms * 8));
        if (dim == 2) k_diag_particles4<2><<<gb4, 256, 0, s>>>(P, (const float*)ras, rs, n0, live, out);
        else k_diag_particles4<3><<<gb4, 256, 0, s>>>(P, (const float*)ras, rs, n0, live, out);
        return launch_status(1);
    }
#define DP(D, R) k_diag_particles<D, R><<<gb, 256, 0, s>>>(P, (const R*)ras, rs, n0, live, out)
    if (dim == 2) { if (dtype) DP(2, double); else DP(2, float); }
    else { if (dtype) DP(3, double); else DP(3, float); }
#undef DP
    return launch_status(1);
}

extern "C" int mlbm_coupling_op(const mlbm_level_t* lv0, int32_t op, void* ras, int64_t rs, const void* a0,
                                const void* u, int64_t us, void* out, int64_t os, double eps_min,
                                double nu, double d_p, double re_min, double dt, double rho0,
                                const double* g, int32_t dtype, void* stream) {
    if (op < MLBM_COUPLE_FRACTIONS || op > MLBM_COUPLE_MIXTURE_FORCE) return -1;
    const int T = lv0->dim == 2 ? 16 : 64;
    const int64_t n = (int64_t)lv0->n_tiles * T;
    if (n == 0) return 0;
    CoupleArgs A{*lv0, ras, rs, a0, u, us, out, os, eps_min, nu, d_p, re_min, dt, rho0,
                 {g ? g[0] : 0.0, g ? g[1] : 0.0, g ? g[2] : 0.0}, op};
    cudaStream_t s = as_stream(stream);
#define CO(D, R) k_coupling_op<D, R><<<nblk(n, 128), 128, 0, s>>>(A)
    if (lv0->dim == 2) { if (dtype) CO(2, double); else CO(2, float); }
    else { if (dtype) CO(3, double); else CO(3, float); }
#undef CO
    return launch_status(1);
}

extern "C" int mlbm_stencil(const mlbm_level_t* lv0, int32_t n, const double* x, int64_t ps, int32_t* idx,
                            void* w, void* grad, void* dpos, int64_t os, int32_t dtype, mlbm_error_t* err,
                            void* stream) {
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    const TopoL0 t = topo0(lv0);
#define ST(D, R) k_stencil<D, R><<<nblk(n, 128), 128, 0, s>>>(n, x, ps, t, idx, (R*)w, (R*)grad, (R*)dpos, os, err)
    if (lv0->dim == 2) { if (dtype) ST(2, double); else ST(2, float); }
    else { if (dtype) ST(3, double); else ST(3, float); }
#undef ST
    return launch_status(1);
}

extern "C" int mlbm_powder_step(const mlbm_level_t* lv0, mlbm_fields_t src, mlbm_fields_t dst, void* tmp,
                                double diffusion, double sign, double dt, const void* source,
                                int32_t dtype, void* stream) {
    const int T = lv0->dim == 2 ? 16 : 64;
    const int64_t n = (int64_t)lv0->n_tiles * T;
    if (n == 0) return 0;
    PowderArgs A{*lv0, src, dst, nullptr, 0, tmp, diffusion, sign, dt, 0.0, 0.0, 0, source, nullptr};
    cudaStream_t s = as_stream(stream);
#define PW(D, R) do { k_powder_advect<D, R><<<nblk(n, 128), 128, 0, s>>>(A); \
                      k_powder_diffuse<D, R><<<nblk(n, 128), 128, 0, s>>>(A); } while (0)
    if (lv0->dim == 2) { if (dtype) PW(2, double); else PW(2, float); }
    else { if (dtype) PW(3, double); else PW(3, float); }
#undef PW
    return launch_status(2);
}

extern "C" int mlbm_particle_stress(int32_t dim, int32_t n, void* p, int64_t ps, double lam, double mu,
                                    double alpha, int32_t dtype, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    const MatParams mp = mat_params(lam, mu, alpha);
#define PSK(D, R) k_particle_stress<D, R><<<nblk(n, 128), 128, 0, s>>>(n, (R*)p, ps, mp)
    if (dim == 2) { if (dtype) PSK(2, double); else PSK(2, float); }
    else if (dim == 3) { if (dtype) PSK(3, double); else PSK(3, float); }
    else return -1;
#undef PSK
    return launch_status(1);
}
