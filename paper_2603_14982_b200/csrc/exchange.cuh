// Per-cell fluid-sediment exchange of level 0 (coupling.py:96-197,379-446;
// granular.py:313-341), shared by the exchange kernel (mpm.cu:k_exchange), the
// standalone coupling seams (mpm.cu:k_coupling_op) and the fused level-0
// stream + exchange + collide kernel (lbm.cu:level_kernel mode 5).
#pragma once
#include "common.cuh"

namespace mlbm {

// level-0 raster rows (one [N][n0] block of the run dtype)
template <int D> struct Rows {
    static constexpr int MASS = 0, MOM = 1, FINT = 1 + D, ETA = 1 + 2 * D, AREA = 2 + 2 * D,
                         VMOM = 3 + 2 * D, VEL = 3 + 3 * D, FS = 3 + 4 * D, EPS = 3 + 5 * D,
                         GRAD = 4 + 5 * D, REL = 4 + 6 * D, SIG = 4 + 7 * D,
                         // eta_eff = max(eta - phi, 0) (coupling.py:127) in its own
                         // row: k_exchange's neighbour eps reads the raw ETA row
                         ETAE = 4 + 7 * D + Geo<D>::NS,
                         N = 5 + 7 * D + Geo<D>::NS, NACC = 3 + 3 * D;
};

MLBM_HD int64_t g3(const int* d, int x, int y, int z) { return ((int64_t)x * d[1] + y) * d[2] + z; }

struct ExchArgs {
    mlbm_level_t lv;          // level 0
    mlbm_fields_t w_tree, r_tree;   // level-0 write (post-stream) / read trees
    mlbm_fields_t tree0, tree1;     // both trees (eps / force written into both)
    void* ras;
    int64_t rs;
    double eps_min, nu, d_p, re_min, dt, rho0;
    double g_fluid[3], g_sed[3];
    int32_t face[6];
    double floor_friction;
    int32_t mode;             // 1 exchange (drag + force + grid update), 0 grid update only
};

template <int D, typename R>
__device__ __forceinline__ R eps_of(const R* ras, int64_t rs, const FieldsT<R>& rt, int64_t c, R eps_min) {
    const R phi = rt.at(fi_phi<D>(), c);
    R eta = ras[Rows<D>::ETA * rs + c] - phi;
    eta = eta > R(0) ? eta : R(0);
    R e = R(1) - eta - phi;
    e = e < eps_min ? eps_min : (e > R(1) ? R(1) : e);
    return e;
}

// Di Felice drag on the sediment of one cell (coupling.py:134-156): rel =
// u - v_cell, Re = max(eps |rel| d_p / nu, re_min), C_d, chi, f_s
template <int D, typename R>
__device__ __forceinline__ void difelice_cell(R eps, R rho, const R (&rel)[D], R speed, R area, R d_p,
                                              R nu, R re_min, R (&fs)[D]) {
    for (int a = 0; a < D; ++a) fs[a] = R(0);
    if (!(area > R(0) && speed > R(0))) return;
    R re = eps * speed * d_p / nu;
    re = re > re_min ? re : re_min;
    const R cd = (R(0.63) + R(4.8) / sqrt(re)) * (R(0.63) + R(4.8) / sqrt(re));
    const R lg = R(1.5) - log10(re);
    const R chi = R(3.7) - R(0.65) * exp(R(-0.5) * lg * lg);
    const R coef = R(0.5) * cd * pow(eps, -chi) * rho * area * speed;
    for (int a = 0; a < D; ++a) fs[a] = coef * rel[a];
}

// smooth drag limiter (CoupledSim._limit_drag, coupling.py:379-401)
template <int D, typename R>
__device__ __forceinline__ void limit_drag_cell(R (&fs)[D], R rho, R mass, R speed, R dt) {
    R mag2 = R(0);
    for (int a = 0; a < D; ++a) mag2 += fs[a] * fs[a];
    const R mag = sqrt(mag2);
    if (!(mag > R(0))) return;
    const R inv_m = R(1) / rho + R(1) / (mass > R(1e-12) ? mass : R(1e-12));
    const R beta = mag * dt * inv_m / (speed > R(1e-14) ? speed : R(1e-14));
    R over = beta - R(0.5);
    over = over > R(0) ? over : R(0);
    const R real = (beta < R(0.5) ? beta : R(0.5)) + over / (R(1) + over);
    const R scale = real / (beta > R(1e-14) ? beta : R(1e-14));
    for (int a = 0; a < D; ++a) fs[a] *= scale;
}

// central differences of a level-0 cell field (coupling.py:159-182): the
// neighbour wraps (periodic) or clamps to the domain; a neighbour that is
// not stored counts as the cell itself.  val(ni) returns the field at cell ni.
template <int D, typename R, typename F>
__device__ __forceinline__ void grad_cell(const mlbm_level_t& lv, const int (&g)[3], int64_t c, F val,
                                          R (&grad)[D]) {
    constexpr int T = Geo<D>::T;
    for (int a = 0; a < D; ++a) {
        R pm[2];
        for (int sgn = 0; sgn < 2; ++sgn) {
            int nb[3] = {g[0], g[1], g[2]};
            nb[a] += sgn == 0 ? 1 : -1;
            if (lv.periodic[a]) nb[a] = (nb[a] + lv.cells[a]) % lv.cells[a];
            else nb[a] = nb[a] < 0 ? 0 : (nb[a] >= lv.cells[a] ? lv.cells[a] - 1 : nb[a]);
            // a neighbour in the cell's own tile needs no tile-map lookup
            const bool same = (nb[a] >> 2) == (g[a] >> 2);
            const int s = same ? (int)(c / T)
                               : lv.tile_map[g3(lv.tiles, nb[0] >> 2, nb[1] >> 2, D == 3 ? nb[2] >> 2 : 0)];
            const int64_t ni = s >= 0 ? (int64_t)s * T + local_of<D>(nb[0] & 3, nb[1] & 3, nb[2] & 3) : c;
            pm[sgn] = val(ni);
        }
        grad[a] = R(0.5) * (pm[0] - pm[1]);
    }
}


// MPM grid update of one node (granular.py:313-341): v = (mom + dt (f_int +
// f_s)) / m + dt g on massive nodes, wall bands of 2 nodes with Coulomb
// friction, sticky solids; written to the VEL rows
template <int D, typename R>
__device__ __forceinline__ void grid_update_cell(const ExchArgs& A, int64_t c, const int (&g)[3],
                                                 const R (&fs)[D]) {
    using RW = Rows<D>;
    R* ras = (R*)A.ras;
    const int64_t rs = A.rs;
    const R mass = ras[RW::MASS * rs + c];
    R vel[D];
    if (mass > R(0)) {
        const R inv_m = R(1) / mass;
        for (int a = 0; a < D; ++a)
            vel[a] = (ras[(RW::MOM + a) * rs + c] + R(A.dt) * (ras[(RW::FINT + a) * rs + c] + fs[a])) * inv_m
                     + R(A.dt) * R(A.g_sed[a]);
    } else {
        for (int a = 0; a < D; ++a) vel[a] = R(0);
    }
    for (int f = 0; f < 2 * D; ++f) {
        if (A.face[f] != MLBM_FACE_WALL) continue;
        const int axis = f >> 1;
        const bool lo = (f & 1) == 0;
        const bool in_band = lo ? g[axis] <= 1 : g[axis] >= A.lv.cells[axis] - 2;
        if (!in_band) continue;
        const R sgn = lo ? R(1) : R(-1);
        const R vn = sgn * vel[axis];
        if (!(vn < R(0))) continue;
        R vt2 = R(0);
        for (int b = 0; b < D; ++b) if (b != axis) vt2 += vel[b] * vel[b];
        const R vtn = sqrt(vt2);
        R scale = R(1) - R(A.floor_friction) * (-vn) / (vtn > R(1e-14) ? vtn : R(1e-14));
        scale = scale > R(0) ? scale : R(0);
        vel[axis] = R(0);
        for (int b = 0; b < D; ++b) if (b != axis) vel[b] *= scale;
    }
    if (A.lv.cell_flags[c] & MLBM_CF_SOLID)
        for (int a = 0; a < D; ++a) vel[a] = R(0);
    for (int a = 0; a < D; ++a) ras[(RW::VEL + a) * rs + c] = vel[a];
}

// The exchange of one level-0 cell from its bare post-stream density and
// velocity: eps from the rasterised fractions and the read tree's phi, Di Felice
// drag + limiter, grad eps, the mixture force (into both trees' f rows, eps
// into both trees), the raster rows the MPM and powder steps read, and the
// grid update.  Returns the lattice force and eps of the cell.
template <int D, typename R>
__device__ __forceinline__ void exchange_cell(const ExchArgs& A, int64_t c, const int (&g)[3], R rho,
                                              const R (&u)[D], R (&force)[D], R& eps_out,
                                              const R* seps = nullptr) {
    using RW = Rows<D>;
    R* ras = (R*)A.ras;
    const int64_t rs = A.rs;
    const FieldsT<R> rt = fields_of<R>(A.r_tree);
    const R eps_min = R(A.eps_min);
    const R mass = ras[RW::MASS * rs + c];
    // seps (optional): the eps of every cell of this cell's tile, staged by the
    // caller (fused level kernel): in-tile neighbours of grad eps read it
    const R eps = seps ? seps[c % Geo<D>::T] : eps_of<D, R>(ras, rs, rt, c, eps_min);
    R eta = ras[RW::ETA * rs + c] - rt.at(fi_phi<D>(), c);
    eta = eta > R(0) ? eta : R(0);
    R vcell[D];
    for (int a = 0; a < D; ++a) vcell[a] = mass > R(0) ? ras[(RW::VMOM + a) * rs + c] / mass : R(0);
    R rel[D], sp2 = R(0);
    for (int a = 0; a < D; ++a) {
        rel[a] = u[a] - vcell[a];
        sp2 += rel[a] * rel[a];
    }
    const R speed = sqrt(sp2);
    const R area = ras[RW::AREA * rs + c];
    R fs[D];
    difelice_cell<D, R>(eps, rho, rel, speed, area, R(A.d_p), R(A.nu), R(A.re_min), fs);
    if (area > R(0) && speed > R(0)) limit_drag_cell<D, R>(fs, rho, mass, speed, R(A.dt));
    // grad eps: the neighbours' eps from the raw eta (never overwritten here)
    R grad[D];
    if (seps) {
        const int64_t tile0 = c - c % Geo<D>::T;
        grad_cell<D, R>(A.lv, g, c, [&](int64_t ni) {
            return (ni - tile0 >= 0 && ni - tile0 < Geo<D>::T) ? seps[ni - tile0]
                                                               : eps_of<D, R>(ras, rs, rt, ni, eps_min);
        }, grad);
    } else {
        grad_cell<D, R>(A.lv, g, c, [&](int64_t ni) { return eps_of<D, R>(ras, rs, rt, ni, eps_min); },
                        grad);
    }
    const R coefg = (rho - R(A.rho0)) / eps;
    const FieldsT<R> t0 = fields_of<R>(A.tree0), t1 = fields_of<R>(A.tree1);
    for (int a = 0; a < D; ++a) {
        const R gt = coefg * grad[a];
        force[a] = gt + rho * R(A.g_fluid[a]) - fs[a];
        t0.at(fi_f<D>(a), c) = force[a];
        t1.at(fi_f<D>(a), c) = force[a];
        ras[(RW::GRAD + a) * rs + c] = gt;
        ras[(RW::REL + a) * rs + c] = rel[a];
        ras[(RW::FS + a) * rs + c] = fs[a];
        ras[(RW::VMOM + a) * rs + c] = vcell[a];   // becomes the cell velocity
    }
    t0.at(fi_eps<D>(), c) = eps;
    t1.at(fi_eps<D>(), c) = eps;
    ras[RW::EPS * rs + c] = eps;
    ras[RW::ETAE * rs + c] = eta;                  // eta_eff (ETA stays raw: neighbours read it)
    eps_out = eps;
    grid_update_cell<D, R>(A, c, g, fs);
}

}  // namespace mlbm
