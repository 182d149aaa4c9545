// Sparse tile hierarchy on the GPU: compaction into sorted slots, neighbour
// tables, per-cell classification (interfaces / BC / solid / bounce-back
// masks), interface stencils, the bitmap passes of block maintenance, data
// migration and new-cell initialisation.
//
// Reference seams: sparse_grid.py:183-200 (rebuild_level), 210-282 (rasters),
// 304-363 (validation, dilation), 439-544 (interfaces); solver.py:159-273
// (solid raster, _LevelTables); adapt.py:54-389 (GridAdaptor).
//
// Integer work only (except migration / init): every pass is a coalesced
// sweep over a dense uint8 tile grid or over the stored cells, bit-exact with
// the reference by construction (no floating point decides topology).
#include "common.cuh"

namespace mlbm {

MLBM_HD int64_t gidx3(const int* d, int x, int y, int z) {
    return ((int64_t)x * d[1] + y) * d[2] + z;
}
MLBM_HD void gdec3(const int* d, int64_t g, int& x, int& y, int& z) {
    z = (int)(g % d[2]);
    g /= d[2];
    y = (int)(g % d[1]);
    x = (int)(g / d[1]);
}
struct I3 { int v[3]; };
MLBM_HD I3 tdims_of(const mlbm_hier_t& h, int l) {
    I3 r;
    for (int a = 0; a < 3; ++a) r.v[a] = a < h.dim ? (h.finest[a] >> l) / 4 : 1;
    return r;
}
MLBM_HD I3 cdims_of(const mlbm_hier_t& h, int l) {
    I3 r;
    for (int a = 0; a < 3; ++a) r.v[a] = a < h.dim ? (h.finest[a] >> l) : 1;
    return r;
}

__device__ bool solid_at(const mlbm_solid_t& s, int dim, const int (&g)[3]) {
    for (int b = 0; b < s.n_boxes; ++b) {
        bool in = true;
        for (int a = 0; a < dim; ++a)
            in &= (double)g[a] >= s.boxes[b][a] && (double)g[a] < s.boxes[b][3 + a];
        if (in) return true;
    }
    if (s.heightmap) {
        int hx = g[0] < 0 ? 0 : (g[0] >= s.hm_dims[0] ? s.hm_dims[0] - 1 : g[0]);
        float h;
        if (dim == 2) h = s.heightmap[hx];
        else {
            int hz = g[2] < 0 ? 0 : (g[2] >= s.hm_dims[1] ? s.hm_dims[1] - 1 : g[2]);
            h = s.heightmap[(int64_t)hx * s.hm_dims[1] + hz];
        }
        if (h > 0.f && (float)g[1] < h) return true;
    }
    return false;
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Stable stream compaction (no library scan): the flagged indices of [0, n) in
// increasing order get consecutive positions.
//   k_flag_count   per block of CB * CI elements: warp ballots + popc, one
//                  block sum
//   k_scan_blocks  one block: exclusive scan of the block sums (+ total)
//   k_flag_scatter per block again: for each of the CI element strips the
//                  ballot rank inside the warp + the warps before it (shared
//                  scan) + the block offset give every flagged element its
//                  position, and the writer functor is called for every element
constexpr int CB = 256, CI = 4;          // 1024 elements per block
constexpr int CPB = CB * CI;

template <typename F>
__global__ void k_flag_count(int64_t n, F flag, int32_t* __restrict__ bsum) {
    __shared__ int ws[CB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * CPB;
    int c = 0;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
        const int64_t g = base + k * CB + threadIdx.x;
        c += __popc(__ballot_sync(0xffffffffu, g < n && flag(g)));
    }
    if (lane == 0) ws[wid] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < CB / 32; ++w) t += ws[w];
        bsum[blockIdx.x] = t;
    }
}

__global__ void k_scan_blocks(int nb, int32_t* __restrict__ bsum, int32_t* __restrict__ total) {
    __shared__ int wsum[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int base = 0; base < nb; base += blockDim.x) {
        const int b = base + threadIdx.x;
        const int v = b < nb ? bsum[b] : 0;
        int t = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        if (lane == 31) wsum[wid] = t;
        __syncthreads();
        if (wid == 0) {
            int q = lane < nw ? wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, q, o);
                if (lane >= o) q += u;
            }
            if (lane < nw) wsum[lane] = q;
        }
        __syncthreads();
        if (b < nb) bsum[b] = carry + (wid ? wsum[wid - 1] : 0) + t - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += wsum[nw - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

template <typename F, typename W>
__global__ void k_flag_scatter(int64_t n, F flag, const int32_t* __restrict__ boff, W write) {
    __shared__ int wsum[CB / 32];
    __shared__ int strip_total;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * CPB;
    int run = boff[blockIdx.x];
#pragma unroll 1
    for (int k = 0; k < CI; ++k) {
        const int64_t g = base + k * CB + threadIdx.x;
        const bool f = g < n && flag(g);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        int before = 0;
        for (int w = 0; w < wid; ++w) before += wsum[w];
        if (threadIdx.x == 0) {
            int t = 0;
            for (int w = 0; w < CB / 32; ++w) t += wsum[w];
            strip_total = t;
        }
        const int pos = run + before + __popc(bal & ((1u << lane) - 1u));
        if (g < n) write(g, f, pos);
        __syncthreads();
        run += strip_total;
        __syncthreads();
    }
}

static inline int flag_blocks(int64_t n) { return (int)((n + CPB - 1) / CPB); }

struct KindFlag {
    const uint8_t* kind;
    __device__ bool operator()(int64_t g) const { return kind[g] != 0; }
};

struct TileWriter {
    I3 td;
    const uint8_t* kind;
    const int32_t* old_map;
    int32_t* tile_map;
    int32_t* tile_xyz;
    uint8_t* tile_kind;
    int32_t* old_slot;
    int32_t cap;
    int32_t* counts;
    __device__ void operator()(int64_t g, bool f, int slot) const {
        if (f && slot < cap) {
            tile_map[g] = slot;
            int x, y, z;
            gdec3(td.v, g, x, y, z);
            tile_xyz[slot * 3 + 0] = x;
            tile_xyz[slot * 3 + 1] = y;
            tile_xyz[slot * 3 + 2] = z;
            tile_kind[slot] = kind[g];
            const int os = old_map ? old_map[g] : -1;
            old_slot[slot] = os;
            if (os < 0) atomicAdd(&counts[1], 1);
        } else {
            tile_map[g] = -1;
        }
    }
};

struct IfaceFlag {      // interface target: a live cell with the ghost bit
    mlbm_level_t lv;       // live tile count on the device (lv.counts)
    int T;
    uint8_t bit;
    __device__ bool operator()(int64_t g) const {
        return g < (int64_t)live_tiles(lv) * T && (lv.cell_flags[g] & bit);
    }
};

struct ChangedFlag {     // a tile whose kind differs between two kind grids
    const uint8_t* a;
    const uint8_t* b;
    __device__ bool operator()(int64_t g) const { return a[g] != b[g]; }
};

struct TargetWriter {
    int32_t* targets;
    __device__ void operator()(int64_t g, bool f, int pos) const {
        if (f) targets[pos] = (int32_t)g;
    }
};

__global__ void k_zero_i32(int32_t* p, int n) {
    if (threadIdx.x < n) p[threadIdx.x] = 0;
}

static int64_t align256(int64_t v) { return (v + 255) & ~(int64_t)255; }

// ---------------------------------------------------------------------------
// neighbours
template <int D>
__global__ void k_neighbors(mlbm_level_t lv, int32_t* nbr) {
    constexpr int NB = Geo<D>::NB;
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= (int64_t)live_tiles(lv) * NB) return;
    const int t = (int)(j / NB), k = (int)(j % NB);
    const int o[3] = {k % 3 - 1, (k / 3) % 3 - 1, D == 3 ? k / 9 - 1 : 0};
    int c[3];
    for (int a = 0; a < 3; ++a) {
        c[a] = lv.tile_xyz[t * 3 + a] + o[a];
        if (a >= D) continue;
        if (lv.periodic[a]) c[a] = (c[a] + lv.tiles[a]) % lv.tiles[a];
        else if (c[a] < 0 || c[a] >= lv.tiles[a]) { nbr[j] = -1; return; }
    }
    nbr[j] = lv.tile_map[gidx3(lv.tiles, c[0], c[1], c[2])];
}

// ---------------------------------------------------------------------------
// owner level of a level-l cell position (finest leaf wins, corner sample)
__device__ int owner_of(const mlbm_hier_t& h, int l, const int (&c)[3]) {
    for (int lp = 0; lp < h.levels; ++lp) {
        const I3 td = tdims_of(h, lp);
        int p[3];
        for (int a = 0; a < 3; ++a) {
            if (a >= h.dim) { p[a] = 0; continue; }
            const int s = lp >= l ? (c[a] >> (lp - l)) : (c[a] << (l - lp));
            p[a] = s >> 2;
        }
        if (h.kind[lp][gidx3(td.v, p[0], p[1], p[2])] == 1) return lp;
    }
    return -1;
}

// incremental classification after a topology change: a tile whose tile
// neighbourhood saw no kind change at any level (dirty == 0) keeps its
// classification, copied from its old slot
struct ClassifyPrev {
    const uint8_t* dirty;      // the level's tile grid, or null: classify every tile
    const int32_t* old_slot;   // new slot -> old slot (null: unchanged slots)
    const uint8_t* cf;         // old cell flags / masks / tile flags
    const uint64_t* masks;
    const uint8_t* tf;
};

template <int D>
__global__ void __launch_bounds__(Geo<D>::T) k_classify(mlbm_level_t lv, mlbm_hier_t h, mlbm_bc_t bc,
                                                     mlbm_solid_t solid, uint8_t* cell_flags,
                                                     uint64_t* dir_masks, uint8_t* tile_flags,
                                                     int32_t* counts, mlbm_error_t* err,
                                                     ClassifyPrev prev, const int32_t* list,
                                                     const int32_t* n_list) {
    constexpr int T = Geo<D>::T, NB = Geo<D>::NB, Q = Geo<D>::Q;
    const int lc = threadIdx.x;
    const int level = lv.level;
    // one tile per block, or (list) a persistent loop over the dirty tiles the
    // copy kernel listed
    for (int it = blockIdx.x;; it += gridDim.x) {
    int tile;
    if (list) {
        if (it >= __ldg(n_list)) break;         // block-uniform
        tile = list[it];
    } else {
        if (it >= live_tiles(lv)) break;        // block-uniform
        tile = it;
    }
    if (prev.dirty && !list) {
        const int t3[3] = {lv.tile_xyz[tile * 3], lv.tile_xyz[tile * 3 + 1], lv.tile_xyz[tile * 3 + 2]};
        const int os = prev.old_slot ? prev.old_slot[tile] : tile;
        if (os >= 0 && !prev.dirty[gidx3(lv.tiles, t3[0], t3[1], t3[2])]) {   // block-uniform
            const int64_t oc = (int64_t)os * T + lc, nc = (int64_t)tile * T + lc;
            const uint8_t f = prev.cf[oc];
            cell_flags[nc] = f;
            dir_masks[nc] = prev.masks[oc];
            const int nid = __syncthreads_count(f & MLBM_CF_GHOST_D);
            const int niu = __syncthreads_count(f & MLBM_CF_GHOST_U);
            if (lc == 0) {
                if (nid) atomicAdd(&counts[0], nid);
                if (niu) atomicAdd(&counts[1], niu);
                tile_flags[tile] = prev.tf[os];
            }
            continue;
        }
    }
    __shared__ int snb[NB];
    if (lc < NB) snb[lc] = lv.nbr[(int64_t)tile * NB + lc];
    const int tx[3] = {lv.tile_xyz[tile * 3], lv.tile_xyz[tile * 3 + 1], lv.tile_xyz[tile * 3 + 2]};
    const uint8_t tkind = h.kind[level][gidx3(lv.tiles, tx[0], tx[1], tx[2])];
    const int l[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    int g[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) g[a] = tx[a] * 4 + l[a];
    // rim: some in-domain neighbour tile is absent
    // per neighbour-tile offset: 1 = outside a non-periodic axis, 2 = outside
    // through a wall face (bounce-back), 4 = stored (read by the pull scan)
    __shared__ uint8_t sstate[NB];
    if (lc < NB) {
        const int o[3] = {lc % 3 - 1, (lc / 3) % 3 - 1, D == 3 ? lc / 9 - 1 : 0};
        uint8_t st = 0;
        for (int a = 0; a < D; ++a) {
            if (lv.periodic[a] || o[a] == 0) continue;
            const int t = tx[a] + o[a];
            if (t < 0) { st |= 1; if (bc.face[2 * a] == MLBM_FACE_WALL) st |= 2; }
            else if (t >= lv.tiles[a]) { st |= 1; if (bc.face[2 * a + 1] == MLBM_FACE_WALL) st |= 2; }
        }
        if (!(st & 1) && lv.nbr[(int64_t)tile * NB + lc] >= 0) st |= 4;
        sstate[lc] = st;
    }
    bool gapnb = false;
    if (lc < NB) {
        const int o[3] = {lc % 3 - 1, (lc / 3) % 3 - 1, D == 3 ? lc / 9 - 1 : 0};
        bool indom = true;
        for (int a = 0; a < D; ++a) {
            const int c = tx[a] + o[a];
            if (!lv.periodic[a] && (c < 0 || c >= lv.tiles[a])) indom = false;
        }
        gapnb = indom && lv.nbr[(int64_t)tile * NB + lc] < 0;
    }
    const int rim = __syncthreads_or(gapnb);

    int gf[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) gf[a] = g[a] << level;
    // solids can only bounce a pull if one lies within one cell of the tile:
    // boxes are tested against the dilated tile box, the heightmap by its
    // maximum over the dilated footprint (a tile on a periodic seam is always
    // scanned)
    bool near = false;
    if (solid.near[level]) {
        near = solid.near[level][gidx3(lv.tiles, tx[0], tx[1], tx[2])] != 0;   // static map
    } else if (solid.n_boxes > 0 || solid.heightmap != nullptr) {
        bool seam = false;
        for (int a = 0; a < D; ++a)
            seam |= lv.periodic[a] && (tx[a] == 0 || tx[a] == lv.tiles[a] - 1);
        const int sc = 1 << level;
        int lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};      // finest, [lo, hi)
        for (int a = 0; a < D; ++a) { lo[a] = (tx[a] * 4 - 1) * sc; hi[a] = (tx[a] * 4 + 5) * sc; }
        bool mine = seam;
        if (lc == 0 && !seam) {
            for (int b = 0; b < solid.n_boxes && !mine; ++b) {
                bool in = true;
                for (int a = 0; a < D; ++a)
                    in &= solid.boxes[b][a] < (double)hi[a] && solid.boxes[b][3 + a] > (double)lo[a];
                mine |= in;
            }
        }
        if (solid.heightmap && !seam && !mine) {
            // footprint columns (x, z) strided over the block; heights clamp
            // at the map edges exactly as solid_at does
            const int nx = hi[0] - lo[0], nz = D == 3 ? hi[2] - lo[2] : 1;
            float hmax = 0.f;
            for (int i = lc; i < nx * nz; i += T) {
                const int cx = lo[0] + i % nx, cz = D == 3 ? lo[2] + i / nx : 0;
                const int hx = cx < 0 ? 0 : (cx >= solid.hm_dims[0] ? solid.hm_dims[0] - 1 : cx);
                float h;
                if (D == 2) h = solid.heightmap[hx];
                else {
                    const int hz = cz < 0 ? 0 : (cz >= solid.hm_dims[1] ? solid.hm_dims[1] - 1 : cz);
                    h = solid.heightmap[(int64_t)hx * solid.hm_dims[1] + hz];
                }
                hmax = h > hmax ? h : hmax;
            }
            mine |= hmax > 0.f && (float)lo[1] < hmax;
        }
        near = __syncthreads_or(mine);
    }
    const bool solid_c = near && solid_at(solid, D, gf);
    bool bcl = false;
    for (int f = 0; f < 2 * D; ++f) {
        const int k = bc.face[f];
        if (k != MLBM_FACE_OUTLET && k != MLBM_FACE_LOG_INLET) continue;
        const int axis = f >> 1;
        if (g[axis] == ((f & 1) ? lv.cells[axis] - 1 : 0)) bcl = true;
    }
    bool id = false, iu = false;
    // owner level of every cell within 2 of the tile (8^D box, smem), taken
    // only in absent in-domain neighbour tiles (-1 elsewhere: no effect)
    constexpr int W = D == 3 ? 512 : 64;
    __shared__ int8_t sown[W];
    if (rim) {                                   // block-uniform
        for (int i = lc; i < W; i += T) {
            const int m[3] = {i & 7, (i >> 3) & 7, D == 3 ? i >> 6 : 2};
            int o[3] = {0, 0, 0}, cc[3] = {0, 0, 0};
            bool indom = true;
            for (int a = 0; a < D; ++a) {
                const int u = tx[a] * 4 + m[a] - 2;     // unwrapped cell
                o[a] = (m[a] < 2) ? -1 : (m[a] >= 6 ? 1 : 0);
                int c = u;
                if (lv.periodic[a]) c = (c + lv.cells[a]) % lv.cells[a];
                else if (c < 0 || c >= lv.cells[a]) indom = false;
                cc[a] = c;
            }
            const int k = (o[0] + 1) + 3 * (o[1] + 1) + (D == 3 ? 9 * (o[2] + 1) : 0);
            int8_t v = -1;
            if (indom && snb[k] < 0) v = (int8_t)owner_of(h, level, cc);
            sown[i] = v;
        }
        __syncthreads();
        // id: a coarser owner within Chebyshev 2; iu: a finer owner within 1 —
        // box dilations of two indicator bits, done separably over the window
        // (x over the tile's 4 columns, then y, then z) instead of a 5^D scan
        // per cell
        __shared__ uint8_t sx[D == 3 ? 4 * 8 * 8 : 4 * 8], sy[D == 3 ? 4 * 4 * 8 : 16];
        auto bits = [&](int i) -> uint8_t {
            const int own = sown[i];
            return (uint8_t)((own > level ? 1 : 0) | (own >= 0 && own < level ? 2 : 0));
        };
        for (int i = lc; i < (D == 3 ? 256 : 32); i += T) {            // x pass
            const int x = i & 3, y = (i >> 2) & 7, z = D == 3 ? i >> 5 : 0;
            const int row = 8 * y + 64 * z;
            uint8_t v = 0;
#pragma unroll
            for (int dx = -2; dx <= 2; ++dx) {
                const uint8_t q = bits(row + x + 2 + dx);
                v |= (q & 1) | ((dx >= -1 && dx <= 1) ? (q & 2) : 0);
            }
            sx[i] = v;
        }
        __syncthreads();
        for (int i = lc; i < (D == 3 ? 128 : 16); i += T) {            // y pass
            const int x = i & 3, y = (i >> 2) & 3, z = D == 3 ? i >> 4 : 0;
            uint8_t v = 0;
#pragma unroll
            for (int dy = -2; dy <= 2; ++dy) {
                const uint8_t q = sx[x + 4 * (y + 2 + dy) + 32 * z];
                v |= (q & 1) | ((dy >= -1 && dy <= 1) ? (q & 2) : 0);
            }
            sy[i] = v;
        }
        __syncthreads();
        uint8_t v = 0;
        if constexpr (D == 3) {
#pragma unroll
            for (int dz = -2; dz <= 2; ++dz) {
                const uint8_t q = sy[l[0] + 4 * l[1] + 16 * (l[2] + 2 + dz)];
                v |= (q & 1) | ((dz >= -1 && dz <= 1) ? (q & 2) : 0);
            }
        } else {
            v = sy[l[0] + 4 * l[1]];
        }
        id = v & 1;
        iu = (v & 2) != 0;
        if (id && iu) report_error(err, MLBM_ERR_TOPOLOGY, level, g[0], g[1], g[2], 1);
        if (id && level == h.levels - 1) report_error(err, MLBM_ERR_TOPOLOGY, level, g[0], g[1], g[2], 2);
        if (iu && level == 0) report_error(err, MLBM_ERR_TOPOLOGY, level, g[0], g[1], g[2], 3);
    }
    const bool active = !(id || iu || bcl || solid_c);
    uint64_t mask = 0;
    // masks can only be non-zero next to an absent tile, the domain edge or a
    // solid: plain interior tiles skip the 26-direction scan (block-uniform)
    bool edge = false;
    for (int a = 0; a < D; ++a)
        edge |= !lv.periodic[a] && (tx[a] == 0 || tx[a] == lv.tiles[a] - 1);
    const bool need = rim || edge || near;
    if (need) {
        // neighbour tile of the pull source from the smem neighbour slots (no
        // tile-map reads); out-of-domain = neighbour tile outside a
        // non-periodic axis
        const bool has_solids = near;      // no solid within one cell: none to test
#pragma unroll
        for (int i = 1; i < Q; ++i) {
            int o[3] = {0, 0, 0};
#pragma unroll
            for (int a = 0; a < D; ++a) {
                const int sa = l[a] - cvec<D>(i, a);
                o[a] = sa < 0 ? -1 : (sa > 3 ? 1 : 0);
            }
            const uint8_t st = sstate[nb_index<D>(o[0], o[1], o[2])];
            const bool oob = st & 1;
            bool bb = st & 2;
            const bool stored = st & 4;
            if (!oob) {
                if (has_solids) {
                    int sf[3] = {0, 0, 0};
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        int sa = g[a] - cvec<D>(i, a);
                        if (lv.periodic[a]) sa = (sa + lv.cells[a]) % lv.cells[a];
                        sf[a] = sa << level;
                    }
                    if (solid_at(solid, D, sf)) bb = true;
                }
            }
            if (bb) mask |= 1ull << i;
            else if (oob || !stored) {
                mask |= 1ull << (32 + i);
                if (active) report_error(err, MLBM_ERR_TOPOLOGY, level, g[0], g[1], g[2], 4);
            }
        }
    }
    uint8_t f = 0;
    if (active) f |= MLBM_CF_ACTIVE;
    if (solid_c) f |= MLBM_CF_SOLID;
    if (id) f |= MLBM_CF_GHOST_D;
    if (iu) f |= MLBM_CF_GHOST_U;
    if (bcl) f |= MLBM_CF_BC;
    if (mask) f |= MLBM_CF_SPECIAL;
    if (tkind == 1) f |= MLBM_CF_LEAF;
    const int64_t cell = (int64_t)tile * T + lc;
    cell_flags[cell] = f;
    dir_masks[cell] = mask;
    const int nid = __syncthreads_count(id), niu = __syncthreads_count(iu);
    if (lc == 0 && nid) atomicAdd(&counts[0], nid);
    if (lc == 0 && niu) atomicAdd(&counts[1], niu);
    const int plain = __syncthreads_and(active && mask == 0);
    const int anybc = __syncthreads_or(bcl);
    if (lc == 0)
        tile_flags[tile] = (plain ? MLBM_TF_PLAIN : 0) | (anybc ? MLBM_TF_BC : 0) |
                           (tkind == 1 ? MLBM_TF_LEAF : 0);
    __syncthreads();                            // shared staging reused by the next tile
    }
}

// incremental classification, clean tiles: one warp per tile copies the
// flags / masks / tile flag from the old slot (coalesced rows instead of one
// 64-thread block per tile) and lists the dirty / fresh tiles for k_classify
template <int D>
__global__ void __launch_bounds__(256) k_classify_copy(mlbm_level_t lv, uint8_t* cell_flags,
                                                       uint64_t* dir_masks, uint8_t* tile_flags,
                                                       int32_t* counts, ClassifyPrev prev,
                                                       int32_t* list, int32_t* n_list) {
    constexpr int T = Geo<D>::T;
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    const int ntl = live_tiles(lv);
    int nid = 0, niu = 0;
    for (int tile = warp; tile < ntl; tile += nw) {
        const int os = prev.old_slot ? prev.old_slot[tile] : tile;
        bool dirty = os < 0;
        if (!dirty) {
            const int* t3 = lv.tile_xyz + tile * 3;
            dirty = prev.dirty[gidx3(lv.tiles, t3[0], t3[1], t3[2])] != 0;
        }
        if (dirty) {                              // warp-uniform
            if (lane == 0) list[atomicAdd(n_list, 1)] = tile;
            continue;
        }
        for (int c = lane; c < T; c += 32) {
            const int64_t oc = (int64_t)os * T + c, nc = (int64_t)tile * T + c;
            const uint8_t f = prev.cf[oc];
            cell_flags[nc] = f;
            dir_masks[nc] = prev.masks[oc];
            nid += (f & MLBM_CF_GHOST_D) ? 1 : 0;
            niu += (f & MLBM_CF_GHOST_U) ? 1 : 0;
        }
        if (lane == 0) tile_flags[tile] = prev.tf[os];
    }
    nid = __reduce_add_sync(0xffffffffu, nid);
    niu = __reduce_add_sync(0xffffffffu, niu);
    if (lane == 0 && nid) atomicAdd(&counts[0], nid);
    if (lane == 0 && niu) atomicAdd(&counts[1], niu);
}

// ---------------------------------------------------------------------------
// interfaces

template <int D>
__global__ void k_iface_stencil(mlbm_level_t lv, mlbm_level_t other, int which, const int32_t* counts,
                                const int32_t* targets, int32_t* src, mlbm_error_t* err) {
    constexpr int T = Geo<D>::T, NC = Geo<D>::NC;
    // grid-stride over the device count (the grid is sized for the SMs, not
    // for the capacity bound: most of a capacity-sized grid would exit at once)
    const int nt = __ldg(counts);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < nt; j += gridDim.x * blockDim.x) {
    const int c = targets[j];
    const int slot = c / T, lc = c % T;
    const int l[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    int g[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) g[a] = lv.tile_xyz[slot * 3 + a] * 4 + l[a];
    for (int k = 0; k < NC; ++k) {
        int cc[3] = {0, 0, 0};
        bool wpos = true;
        for (int a = 0; a < D; ++a) {
            const int o = (k >> a) & 1;
            int v;
            if (which == 0) {
                v = (g[a] >> 1) + o;
                if (o == 1 && !(g[a] & 1)) wpos = false;
            } else {
                v = g[a] * 2 + o;
            }
            const int dimc = other.cells[a];
            if (other.periodic[a]) v = (v % dimc + dimc) % dimc;
            else v = v < 0 ? 0 : (v >= dimc ? dimc - 1 : v);
            cc[a] = v;
        }
        const int s = other.tile_map[gidx3(other.tiles, cc[0] >> 2, cc[1] >> 2, D == 3 ? cc[2] >> 2 : 0)];
        int idx = -1;
        if (s >= 0) idx = s * T + local_of<D>(cc[0] & 3, cc[1] & 3, cc[2] & 3);
        else if ((which == 0 && wpos) || which == 1)
            report_error(err, MLBM_ERR_TOPOLOGY, lv.level, g[0], g[1], g[2], which == 0 ? 5 : 6);
        src[(int64_t)j * NC + k] = idx;
    }
    }
}

// ---------------------------------------------------------------------------
// block maintenance bitmaps
template <typename R>
__global__ void k_seed(int dim, int n, const R* x, int64_t xs, I3 t0, uint8_t* seeds, mlbm_error_t* err) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int t[3] = {0, 0, 0};
    bool bad = false;
    for (int a = 0; a < dim; ++a) {
        const double v = (double)x[a * xs + p];
        const int64_t c = (int64_t)floor(v);
        const int64_t tt = c >= 0 ? c / 4 : -((-c + 3) / 4);
        if (tt < 0 || tt >= t0.v[a] || !(v == v)) bad = true;
        t[a] = (int)tt;
    }
    if (bad) { report_error(err, MLBM_ERR_DOMAIN, 0, t[0], t[1], t[2]); return; }
    seeds[gidx3(t0.v, t[0], t[1], t[2])] = 1;
}

__global__ void k_bitmap_op(int op, int dim, I3 d, const uint8_t* in, uint8_t* out) {
    // grid over the output (parents: parent grid; else same grid)
    I3 od = d;
    if (op == 1) for (int a = 0; a < dim; ++a) od.v[a] = d.v[a] / 2;
    const int64_t n = (int64_t)od.v[0] * od.v[1] * od.v[2];
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n) return;
    int x[3];
    gdec3(od.v, g, x[0], x[1], x[2]);
    switch (op) {
    case 0:
    case 1: {
        int b[3];
        for (int a = 0; a < 3; ++a) b[a] = a < dim ? (op == 0 ? (x[a] & ~1) : 2 * x[a]) : x[a];
        uint8_t any = 0;
        for (int k = 0; k < (1 << dim); ++k) {
            int c[3] = {b[0] + (k & 1), b[1] + ((k >> 1) & 1), dim == 3 ? b[2] + ((k >> 2) & 1) : b[2]};
            any |= in[gidx3(d.v, c[0], c[1], c[2])] ? 1 : 0;
        }
        out[g] = any;
        break;
    }
    case 2: out[g] = (out[g] | (in[g] ? 1 : 0)); break;
    case 3: out[g] = (out[g] && !in[g]) ? 1 : 0; break;
    case 4: out[g] = in[g] ? 1 : 0; break;
    case 5: out[g] = 1; break;
    case 6: out[g] = in[g] == 1 ? 1 : 0; break;
    case 7: out[g] = in[g] != 0 ? 1 : 0; break;
    case 8: out[g] = out[g] != in[g] ? 1 : 0; break;        // differs (out: a raw copy)
    case 9: out[g] = in[g]; break;                          // raw copy
    case 10: {                                              // out |= in at the parent tile
        I3 pd = d;
        for (int a = 0; a < dim; ++a) pd.v[a] = d.v[a] / 2;
        int q[3] = {x[0], x[1], x[2]};
        for (int a = 0; a < dim; ++a) q[a] >>= 1;
        out[g] = out[g] | (in[gidx3(pd.v, q[0], q[1], q[2])] ? 1 : 0);
        break;
    }
    }
}

__global__ void k_dilate_axis(I3 d, int axis, int periodic, int r, const uint8_t* in, uint8_t* out) {
    const int64_t n = (int64_t)d.v[0] * d.v[1] * d.v[2];
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n) return;
    int x[3];
    gdec3(d.v, g, x[0], x[1], x[2]);
    const int N = d.v[axis];
    uint8_t any = 0;
    for (int k = -r; k <= r && !any; ++k) {
        int c = x[axis] + k;
        if (periodic) c = ((c % N) + N) % N;
        else if (c < 0 || c >= N) continue;
        int y[3] = {x[0], x[1], x[2]};
        y[axis] = c;
        any = in[gidx3(d.v, y[0], y[1], y[2])] ? 1 : 0;
    }
    out[g] = any;
}

// one thread per sibling group (grouped) or per tile (top level)
__global__ void k_effective(int dim, I3 d, int grouped, const uint8_t* des, const uint8_t* cur,
                            const uint8_t* guard, const uint8_t* par_prev, int16_t* streak,
                            uint8_t* eff) {
    I3 gd = d;
    if (grouped) for (int a = 0; a < dim; ++a) gd.v[a] = d.v[a] / 2;
    const int64_t n = (int64_t)gd.v[0] * gd.v[1] * gd.v[2];
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    int x[3];
    gdec3(gd.v, j, x[0], x[1], x[2]);
    const int K = grouped ? (1 << dim) : 1;
    int64_t gi[8];
    bool cand[8], avail[8];
    bool all = true;
    for (int k = 0; k < K; ++k) {
        int c[3];
        for (int a = 0; a < 3; ++a) c[a] = (grouped && a < dim) ? 2 * x[a] + ((k >> a) & 1) : x[a];
        const int64_t g = gidx3(d.v, c[0], c[1], c[2]);
        gi[k] = g;
        cand[k] = cur[g] && !des[g];
        const int16_t s = cand[k] ? (int16_t)(streak[g] + 1) : (int16_t)0;
        streak[g] = s;
        avail[k] = cand[k] && s >= 2 && !(guard && guard[g]);
        all &= avail[k];
    }
    for (int k = 0; k < K; ++k) {
        const int64_t g = gi[k];
        const bool act = grouped ? (avail[k] && all) : false;
        eff[g] = (des[g] || (cur[g] && !act) || (par_prev && par_prev[g])) ? 1 : 0;
    }
}

__global__ void k_plan(int64_t n, const uint8_t* own, const uint8_t* storage, const uint8_t* old_kind,
                       uint8_t* new_kind, int32_t* changed) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n) return;
    const uint8_t k = own[g] ? 1 : (storage[g] ? 2 : 0);
    new_kind[g] = k;
    if (k != old_kind[g]) atomicOr(changed, 1);
}

__global__ void k_coverage(mlbm_hier_t h, int32_t* viol) {
    const I3 t0 = tdims_of(h, 0);
    const int64_t n = (int64_t)t0.v[0] * t0.v[1] * t0.v[2];
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n) return;
    int x[3];
    gdec3(t0.v, g, x[0], x[1], x[2]);
    int cnt = 0;
    for (int l = 0; l < h.levels; ++l) {
        const I3 td = tdims_of(h, l);
        int c[3];
        for (int a = 0; a < 3; ++a) c[a] = a < h.dim ? x[a] >> l : 0;
        cnt += h.kind[l][gidx3(td.v, c[0], c[1], c[2])] == 1;
    }
    if (cnt != 1) atomicAdd(&viol[0], 1);
}

__global__ void k_ring_viol(int64_t n, const uint8_t* dil, const uint8_t* kind, int32_t* viol) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g < n && dil[g] && kind[g] == 0) atomicAdd(&viol[1], 1);
}

template <typename R>
__global__ void k_particle_leaf(int dim, int n, const R* x, int64_t xs, I3 t0, const uint8_t* kind0,
                                int32_t* viol) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int t[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) {
        const int64_t c = (int64_t)floor((double)x[a * xs + p]);
        t[a] = (int)(c >= 0 ? c / 4 : -((-c + 3) / 4));
        if (t[a] < 0 || t[a] >= t0.v[a]) { atomicAdd(&viol[2], 1); return; }
    }
    if (kind0[gidx3(t0.v, t[0], t[1], t[2])] != 1) atomicAdd(&viol[2], 1);
}

// ---------------------------------------------------------------------------
// migration + new-cell init (adapt.py:259-372)
template <int D, typename R>
__global__ void k_migrate(int64_t ncells, const int32_t* n_dev, const int32_t* old_slot, FieldsT<R> o0,
                          FieldsT<R> o1, FieldsT<R> n0, FieldsT<R> n1) {
    constexpr int T = Geo<D>::T, NF = Geo<D>::NF;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= ncells || (n_dev && c >= (int64_t)__ldg(n_dev) * T)) return;
    const int os = old_slot[c / T];
    const int64_t oc = (int64_t)os * T + c % T;
    const bool two = n1.p != nullptr;          // second tree optional (latest-only rebuild)
#pragma unroll
    for (int k = 0; k < NF; ++k) {
        const R def = k == fi_eps<D>() ? R(1) : R(0);
        n0.at(k, c) = os >= 0 ? o0.at(k, oc) : def;
        if (two) n1.at(k, c) = os >= 0 ? o1.at(k, oc) : def;
    }
}

// the same migration in 16-byte vectors (V = 4 floats or 2 doubles): thread i
// moves vector i % nvec of row i / nvec; a tile's cells are contiguous in both
// layouts, so a vector never straddles tiles (T / PER vectors per tile)
template <int D, typename R, typename V>
__global__ void k_migrate_vec(int64_t nvec_row, const int32_t* n_dev, const int32_t* old_slot,
                              const V* __restrict__ o0, const V* __restrict__ o1, V* __restrict__ n0,
                              V* __restrict__ n1, int64_t stride_vec) {
    constexpr int T = Geo<D>::T, NF = Geo<D>::NF, PER = (int)(sizeof(V) / sizeof(R)), TV = T / PER;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t row = i / nvec_row, v = i - row * nvec_row;
    if (row >= NF) return;
    if (n_dev && v >= (int64_t)__ldg(n_dev) * TV) return;
    const int os = __ldg(&old_slot[v / TV]);
    const int64_t ov = (int64_t)os * TV + v % TV;
    V d0, d1;
    if (os >= 0) {
        d0 = o0[row * stride_vec + ov];
        if (n1) d1 = o1[row * stride_vec + ov];
    } else {
        const R def = row == fi_eps<D>() ? R(1) : R(0);
        R* a = reinterpret_cast<R*>(&d0);
#pragma unroll
        for (int k = 0; k < PER; ++k) a[k] = def;
        d1 = d0;
    }
    n0[row * stride_vec + v] = d0;
    if (n1) n1[row * stride_vec + v] = d1;
}

// copy the live cells (device count) of both trees' field blocks in 16-byte
// vectors (V = 4 floats or 2 doubles); rows are capacity-strided and hold
// whole tiles (16 / 64 cells), so the live range is a whole number of vectors
template <int D, typename R, typename V>
__global__ void k_copy_live(int64_t nvec_row, const int32_t* n_dev, int nf, const V* __restrict__ s0,
                            const V* __restrict__ s1, V* __restrict__ d0, V* __restrict__ d1,
                            int64_t stride_vec) {
    constexpr int T = Geo<D>::T, PER = (int)(sizeof(V) / sizeof(R));
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t row = i / nvec_row, v = i - row * nvec_row;
    if (row >= nf) return;
    if (n_dev && v >= (int64_t)__ldg(n_dev) * (T / PER)) return;
    d0[row * stride_vec + v] = s0[row * stride_vec + v];
    if (d1) d1[row * stride_vec + v] = s1[row * stride_vec + v];
}

MLBM_HD double kap_down(double tf, double tc, int conv) { return conv == 0 ? tf / (2.0 * tc) : 2.0 * tc / tf; }
MLBM_HD double kap_up(double tf, double tc, int conv) { return conv == 0 ? 2.0 * tc / tf : tc / (2.0 * tf); }

template <int D, typename R>
__device__ void init_new_cell(const mlbm_hier_t& oh, int level, const int32_t* tile_xyz, int64_t c,
                              const FieldsT<R>& n0, const FieldsT<R>& n1, const double* taus, int conv,
                              int32_t* viol) {
    constexpr int T = Geo<D>::T, NC = Geo<D>::NC, NS = Geo<D>::NS, NM = Geo<D>::NM;
    const int slot = (int)(c / T), lc = (int)(c % T);
    const int l3[3] = {lc & 3, (lc >> 2) & 3, D == 3 ? (lc >> 4) & 3 : 0};
    int g[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) g[a] = tile_xyz[slot * 3 + a] * 4 + l3[a];
    const FieldsT<R> dstt[2] = {n0, n1};
    // coarser: nearest level with a complete stencil
    for (int sl = level + 1; sl < oh.levels; ++sl) {
        if (oh.n_tiles[sl] == 0) continue;
        const int r = sl - level;
        const I3 cd = cdims_of(oh, sl), td = tdims_of(oh, sl);
        int idx[NC];
        R w[NC];
        bool ok = true;
        for (int k = 0; k < NC; ++k) {
            int cc[3] = {0, 0, 0};
            double wk = 1.0;
            for (int a = 0; a < D; ++a) {
                const int o = (k >> a) & 1;
                const double fr = (double)(g[a] & ((1 << r) - 1)) / (double)(1 << r);
                int v = (g[a] >> r) + o;
                if (oh.periodic[a]) v = ((v % cd.v[a]) + cd.v[a]) % cd.v[a];
                else v = v < 0 ? 0 : (v >= cd.v[a] ? cd.v[a] - 1 : v);
                cc[a] = v;
                wk *= o ? fr : 1.0 - fr;
            }
            const int s = oh.tile_map[sl][gidx3(td.v, cc[0] >> 2, cc[1] >> 2, D == 3 ? cc[2] >> 2 : 0)];
            idx[k] = s >= 0 ? s * T + local_of<D>(cc[0] & 3, cc[1] & 3, cc[2] & 3) : 0;
            w[k] = R(wk);
            if (wk > 0.0 && s < 0) ok = false;
        }
        if (!ok) continue;
        for (int t = 0; t < 2; ++t) {
            if (dstt[t].p == nullptr) continue;   // latest-only rebuild
            const FieldsT<R> src{(R*)oh.fields[t][sl], oh.stride[sl]};
            R v[NM + 2];
            for (int q = 0; q < NM + 2; ++q) {
                const int fk = q < NM ? q : (q == NM ? fi_eps<D>() : fi_phi<D>());
                R acc = R(0);
                for (int k = 0; k < NC; ++k) acc += src.at(fk, idx[k]) * w[k];
                v[q] = acc;
            }
            for (int lvl = sl; lvl > level; --lvl) {
                const R kap = R(kap_down(taus[lvl - 1], taus[lvl], conv));
                for (int k = 0; k < NS; ++k) {
                    const R eq = v[1 + s_a<D>(k)] * v[1 + s_b<D>(k)];
                    v[1 + D + k] = kap * (v[1 + D + k] - eq) + eq;
                }
            }
            for (int q = 0; q < NM + 2; ++q) {
                const int fk = q < NM ? q : (q == NM ? fi_eps<D>() : fi_phi<D>());
                dstt[t].at(fk, c) = v[q];
            }
        }
        return;
    }
    // finer: coincident cell of the nearest old finer level
    for (int sl = level - 1; sl >= 0; --sl) {
        if (oh.n_tiles[sl] == 0) continue;
        const int sh = level - sl;
        const I3 td = tdims_of(oh, sl);
        int cc[3] = {0, 0, 0};
        for (int a = 0; a < D; ++a) cc[a] = g[a] << sh;
        const int s = oh.tile_map[sl][gidx3(td.v, cc[0] >> 2, cc[1] >> 2, D == 3 ? cc[2] >> 2 : 0)];
        if (s < 0) continue;
        const int64_t si = (int64_t)s * T + local_of<D>(cc[0] & 3, cc[1] & 3, cc[2] & 3);
        for (int t = 0; t < 2; ++t) {
            if (dstt[t].p == nullptr) continue;   // latest-only rebuild
            const FieldsT<R> src{(R*)oh.fields[t][sl], oh.stride[sl]};
            R v[NM + 2];
            for (int q = 0; q < NM + 2; ++q) {
                const int fk = q < NM ? q : (q == NM ? fi_eps<D>() : fi_phi<D>());
                v[q] = src.at(fk, si);
            }
            for (int lvl = sl; lvl < level; ++lvl) {
                const R kap = R(kap_up(taus[lvl], taus[lvl + 1], conv));
                for (int k = 0; k < NS; ++k) {
                    const R eq = v[1 + s_a<D>(k)] * v[1 + s_b<D>(k)];
                    v[1 + D + k] = kap * (v[1 + D + k] - eq) + eq;
                }
            }
            for (int q = 0; q < NM + 2; ++q) {
                const int fk = q < NM ? q : (q == NM ? fi_eps<D>() : fi_phi<D>());
                dstt[t].at(fk, c) = v[q];
            }
        }
        return;
    }
    atomicAdd(viol, 1);
}

// fresh tiles only: each warp reads the old slots of 32 consecutive tiles
// (one coalesced load), then initialises the cells of its fresh ones — the
// kept tiles (nearly all) cost one load instead of 64 idle threads
template <int D, typename R>
__global__ void __launch_bounds__(256) k_init_new(mlbm_hier_t oh, int level, const int32_t* tile_xyz,
                                                  const int32_t* old_slot, int n_tiles, const int32_t* n_dev,
                                                  FieldsT<R> n0, FieldsT<R> n1, const double* taus, int conv,
                                                  int32_t* viol) {
    constexpr int T = Geo<D>::T;
    const int n = n_dev ? min(n_tiles, __ldg(n_dev)) : n_tiles;
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    for (int s0 = warp * 32; s0 < n; s0 += nwarps * 32) {
        const int sl = s0 + lane;
        unsigned fresh = __ballot_sync(0xffffffffu, sl < n && old_slot[sl] < 0);
        while (fresh) {
            const int j = __ffs(fresh) - 1;
            fresh &= fresh - 1;
            for (int lc = lane; lc < T; lc += 32)
                init_new_cell<D, R>(oh, level, tile_xyz, (int64_t)(s0 + j) * T + lc, n0, n1, taus, conv, viol);
        }
    }
}

// the static near-solid map of one level (the same test as k_classify's
// inline scan, one thread per tile of the whole tile grid)
template <int D>
__global__ void k_solid_near(mlbm_level_t lv, mlbm_solid_t solid, uint8_t* near) {
    const int64_t n = (int64_t)lv.tiles[0] * lv.tiles[1] * lv.tiles[2];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int tx[3];
    gdec3(lv.tiles, t, tx[0], tx[1], tx[2]);
    bool seam = false;
    for (int a = 0; a < D; ++a) seam |= lv.periodic[a] && (tx[a] == 0 || tx[a] == lv.tiles[a] - 1);
    const int sc = 1 << lv.level;
    int lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
    for (int a = 0; a < D; ++a) { lo[a] = (tx[a] * 4 - 1) * sc; hi[a] = (tx[a] * 4 + 5) * sc; }
    bool mine = seam;
    for (int b = 0; b < solid.n_boxes && !mine; ++b) {
        bool in = true;
        for (int a = 0; a < D; ++a) in &= solid.boxes[b][a] < (double)hi[a] && solid.boxes[b][3 + a] > (double)lo[a];
        mine |= in;
    }
    if (solid.heightmap && !mine) {
        const int nx = hi[0] - lo[0], nz = D == 3 ? hi[2] - lo[2] : 1;
        float hmax = 0.f;
        for (int i = 0; i < nx * nz; ++i) {
            const int cx = lo[0] + i % nx, cz = D == 3 ? lo[2] + i / nx : 0;
            const int hx = cx < 0 ? 0 : (cx >= solid.hm_dims[0] ? solid.hm_dims[0] - 1 : cx);
            float h;
            if (D == 2) h = solid.heightmap[hx];
            else {
                const int hz = cz < 0 ? 0 : (cz >= solid.hm_dims[1] ? solid.hm_dims[1] - 1 : cz);
                h = solid.heightmap[(int64_t)hx * solid.hm_dims[1] + hz];
            }
            hmax = h > hmax ? h : hmax;
        }
        mine |= hmax > 0.f && (float)lo[1] < hmax;
    }
    near[t] = mine ? 1 : 0;
}

}  // namespace mlbm

using namespace mlbm;

static inline int blocks_for(int64_t n, int b) { return (int)((n + b - 1) / b); }

extern "C" int64_t mlbm_ws_bytes(int64_t n) {
    if (n < 1) n = 1;
    // [n flag bytes (interfaces)][block sums]
    return align256(4 * n) + align256(4 * (int64_t)flag_blocks(n)) + 256;
}

extern "C" int mlbm_compact_tiles(int32_t dim, const int32_t tiles[3], const uint8_t* kind,
                                  const int32_t* old_map, int32_t* tile_map, int32_t* tile_xyz,
                                  uint8_t* tile_kind, int32_t* old_slot, int32_t capacity,
                                  int32_t* counts, void* ws, int64_t ws_bytes, void* stream) {
    (void)dim;
    const int64_t n = (int64_t)tiles[0] * tiles[1] * tiles[2];
    if (n <= 0 || ws_bytes < mlbm_ws_bytes(n)) return -1;
    cudaStream_t s = as_stream(stream);
    int32_t* bsum = (int32_t*)((char*)ws + align256(4 * n));
    const int nb = flag_blocks(n);
    const KindFlag fl{kind};
    // counts[0] = stored tiles (the scan total), counts[1] = fresh tiles
    k_zero_i32<<<1, 32, 0, s>>>(counts, 2);
    k_flag_count<<<nb, CB, 0, s>>>(n, fl, bsum);
    k_scan_blocks<<<1, 1024, 0, s>>>(nb, bsum, counts);
    I3 td{{tiles[0], tiles[1], tiles[2]}};
    const TileWriter tw{td, kind, old_map, tile_map, tile_xyz, tile_kind, old_slot, capacity, counts};
    k_flag_scatter<<<nb, CB, 0, s>>>(n, fl, bsum, tw);
    return launch_status(4);
}

extern "C" int mlbm_build_neighbors(const mlbm_level_t* lv, int32_t* nbr, void* stream) {
    const int NB = lv->dim == 2 ? 9 : 27;
    const int64_t n = (int64_t)lv->n_tiles * NB;
    if (n == 0) return 0;
    cudaStream_t s = as_stream(stream);
    if (lv->dim == 2) k_neighbors<2><<<blocks_for(n, 256), 256, 0, s>>>(*lv, nbr);
    else k_neighbors<3><<<blocks_for(n, 256), 256, 0, s>>>(*lv, nbr);
    return launch_status(1);
}

extern "C" int mlbm_classify_level(const mlbm_level_t* lv, const mlbm_hier_t* h, const mlbm_bc_t* bc,
                                   const mlbm_solid_t* solid, uint8_t* cell_flags, uint64_t* dir_masks,
                                   uint8_t* tile_flags, int32_t* counts, mlbm_error_t* err,
                                   const uint8_t* dirty, const int32_t* old_slot, const uint8_t* old_cf,
                                   const uint64_t* old_masks, const uint8_t* old_tf, int32_t* work,
                                   void* stream) {
    if (lv->n_tiles == 0) return 0;
    if (dirty && (!old_cf || !old_masks || !old_tf)) return -1;
    cudaStream_t s = as_stream(stream);
    if (counts) cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), s);
    const ClassifyPrev prev{dirty, old_slot, old_cf, old_masks, old_tf};
    const int T = lv->dim == 2 ? 16 : 64;
    int32_t* list = nullptr;
    int32_t* n_list = nullptr;
    int grid = lv->n_tiles;
    if (dirty && work) {
        // clean tiles copied by warps, the dirty ones listed and classified by
        // a persistent grid
        n_list = work;
        list = work + 1;
        cudaMemsetAsync(n_list, 0, sizeof(int32_t), s);
        const int cb = (int)std::min<int64_t>(((int64_t)lv->n_tiles + 7) / 8, 148 * 8);
        if (lv->dim == 2)
            k_classify_copy<2><<<cb, 256, 0, s>>>(*lv, cell_flags, dir_masks, tile_flags, counts, prev, list, n_list);
        else
            k_classify_copy<3><<<cb, 256, 0, s>>>(*lv, cell_flags, dir_masks, tile_flags, counts, prev, list, n_list);
        grid = std::min(lv->n_tiles, 148 * (2048 / T));
    }
    if (lv->dim == 2)
        k_classify<2><<<grid, 16, 0, s>>>(*lv, *h, *bc, *solid, cell_flags, dir_masks,
                                          tile_flags, counts, err, prev, list, n_list);
    else
        k_classify<3><<<grid, 64, 0, s>>>(*lv, *h, *bc, *solid, cell_flags, dir_masks,
                                          tile_flags, counts, err, prev, list, n_list);
    return launch_status(1);
}

extern "C" int mlbm_copy(void* dst, const void* src, int64_t bytes, void* stream) {
    if (bytes <= 0) return 0;
    const cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, as_stream(stream));
    return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" int mlbm_build_interface(const mlbm_level_t* lv, const mlbm_level_t* other, int32_t which,
                                    int32_t* targets, int32_t* src, int32_t* counts,
                                    mlbm_error_t* err, void* ws, int64_t ws_bytes, void* stream) {
    const int T = lv->dim == 2 ? 16 : 64;
    const int64_t n = (int64_t)lv->n_tiles * T;
    if (n == 0) return 0;
    if (ws_bytes < mlbm_ws_bytes(n)) return -1;
    cudaStream_t s = as_stream(stream);
    char* w = (char*)ws;
    int32_t* bsum = (int32_t*)(w + align256(4 * n));
    const int nb = flag_blocks(n);
    // the flags are read straight from the cell flags (no flag array pass);
    // the live count is a device value: kernels launched over the capacity
    // read it themselves
    const uint8_t bit = which == 0 ? MLBM_CF_GHOST_D : MLBM_CF_GHOST_U;
    const IfaceFlag fl{*lv, T, bit};
    k_flag_count<<<nb, CB, 0, s>>>(n, fl, bsum);
    k_scan_blocks<<<1, 1024, 0, s>>>(nb, bsum, counts);
    k_flag_scatter<<<nb, CB, 0, s>>>(n, fl, bsum, TargetWriter{targets});
    const int gs = (int)std::min<int64_t>(blocks_for(n, 128), 148 * 16);
    if (lv->dim == 2)
        k_iface_stencil<2><<<gs, 128, 0, s>>>(*lv, *other, which, counts, targets, src, err);
    else
        k_iface_stencil<3><<<gs, 128, 0, s>>>(*lv, *other, which, counts, targets, src, err);
    return launch_status(5);
}

extern "C" int mlbm_seed_tiles(int32_t dim, int32_t n, const void* x, int64_t xstride, int32_t dtype,
                               const int32_t tiles0[3], uint8_t* seeds, mlbm_error_t* err,
                               void* stream) {
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    I3 t0{{tiles0[0], tiles0[1], tiles0[2]}};
    if (dtype) k_seed<double><<<blocks_for(n, 256), 256, 0, s>>>(dim, n, (const double*)x, xstride, t0, seeds, err);
    else k_seed<float><<<blocks_for(n, 256), 256, 0, s>>>(dim, n, (const float*)x, xstride, t0, seeds, err);
    return launch_status(1);
}

extern "C" int mlbm_bitmap_op(int32_t op, int32_t dim, const int32_t dims[3], const uint8_t* in,
                              uint8_t* out, void* stream) {
    I3 d{{dims[0], dims[1], dims[2]}};
    int64_t n = (int64_t)dims[0] * dims[1] * dims[2];
    if (op == 1) { n = 1; for (int a = 0; a < 3; ++a) n *= a < dim ? dims[a] / 2 : dims[a]; }
    if (n <= 0) return 0;
    k_bitmap_op<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(op, dim, d, in, out);
    return launch_status(1);
}

extern "C" int mlbm_dilate(int32_t dim, const int32_t dims[3], const int32_t periodic[3], int32_t r,
                           const uint8_t* in, uint8_t* out, uint8_t* tmp, void* stream) {
    I3 d{{dims[0], dims[1], dims[2]}};
    const int64_t n = (int64_t)dims[0] * dims[1] * dims[2];
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int B = blocks_for(n, 256);
    if (dim == 2) {
        k_dilate_axis<<<B, 256, 0, s>>>(d, 0, periodic[0], r, in, tmp);
        k_dilate_axis<<<B, 256, 0, s>>>(d, 1, periodic[1], r, tmp, out);
    } else {
        k_dilate_axis<<<B, 256, 0, s>>>(d, 0, periodic[0], r, in, out);
        k_dilate_axis<<<B, 256, 0, s>>>(d, 1, periodic[1], r, out, tmp);
        k_dilate_axis<<<B, 256, 0, s>>>(d, 2, periodic[2], r, tmp, out);
    }
    return launch_status(dim);
}

extern "C" int mlbm_effective_level(int32_t dim, const int32_t dims[3], const uint8_t* des,
                                    const uint8_t* cur, const uint8_t* guard, const uint8_t* par_prev,
                                    int16_t* streak, uint8_t* eff, void* stream) {
    I3 d{{dims[0], dims[1], dims[2]}};
    bool grouped = true;
    for (int a = 0; a < dim; ++a) grouped &= (dims[a] % 2) == 0;
    int64_t n = 1;
    for (int a = 0; a < 3; ++a) n *= (grouped && a < dim) ? dims[a] / 2 : dims[a];
    if (n <= 0) return 0;
    k_effective<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(dim, d, grouped ? 1 : 0, des, cur, guard,
                                                                  par_prev, streak, eff);
    return launch_status(1);
}

extern "C" int mlbm_plan_level(int32_t n, const uint8_t* own, const uint8_t* storage,
                               const uint8_t* old_kind, uint8_t* new_kind, int32_t* changed,
                               void* stream) {
    if (n <= 0) return 0;
    k_plan<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(n, own, storage, old_kind, new_kind, changed);
    return launch_status(1);
}

extern "C" int mlbm_check_coverage(const mlbm_hier_t* h, int32_t* viol, void* stream) {
    const I3 t0 = tdims_of(*h, 0);
    const int64_t n = (int64_t)t0.v[0] * t0.v[1] * t0.v[2];
    k_coverage<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(*h, viol);
    return launch_status(1);
}

extern "C" int mlbm_count_ring_violations(int64_t n, const uint8_t* dil, const uint8_t* kind,
                                          int32_t* viol, void* stream) {
    if (n <= 0) return 0;
    k_ring_viol<<<blocks_for(n, 256), 256, 0, as_stream(stream)>>>(n, dil, kind, viol);
    return launch_status(1);
}

extern "C" int mlbm_check_particles(int32_t dim, int32_t n, const void* x, int64_t xstride, int32_t dtype,
                                    const int32_t tiles0[3], const uint8_t* kind0, int32_t* viol,
                                    void* stream) {
    if (n <= 0) return 0;
    I3 t0{{tiles0[0], tiles0[1], tiles0[2]}};
    cudaStream_t s = as_stream(stream);
    if (dtype) k_particle_leaf<double><<<blocks_for(n, 256), 256, 0, s>>>(dim, n, (const double*)x, xstride, t0, kind0, viol);
    else k_particle_leaf<float><<<blocks_for(n, 256), 256, 0, s>>>(dim, n, (const float*)x, xstride, t0, kind0, viol);
    return launch_status(1);
}

extern "C" int mlbm_migrate_level(int32_t dim, int32_t n_new_tiles, const int32_t* n_dev,
                                  const int32_t* old_slot,
                                  mlbm_fields_t old0, mlbm_fields_t old1, mlbm_fields_t new0,
                                  mlbm_fields_t new1, int32_t dtype, void* stream) {
    const int T = dim == 2 ? 16 : 64;
    const int64_t n = (int64_t)n_new_tiles * T;
    if (n == 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int es = dtype ? 8 : 4;
    const bool same = old0.stride == new0.stride &&
                      (!new1.ptr || (old1.stride == old0.stride && new1.stride == old0.stride));
    if (same && (old0.stride * es) % 16 == 0) {
        // 16-byte vectors (C4: 391 -> 297 us per call against the per-cell kernel)
        const int nf = dim == 2 ? Geo<2>::NF : Geo<3>::NF;
        const int64_t nvec = n * es / 16, stride_vec = old0.stride * es / 16, total = nvec * nf;
#define MIGV(D, R, V) k_migrate_vec<D, R, V><<<blocks_for(total, 256), 256, 0, s>>>(nvec, n_dev, old_slot, \
        (const V*)old0.ptr, (const V*)old1.ptr, (V*)new0.ptr, (V*)new1.ptr, stride_vec)
        if (dim == 2) { if (dtype) MIGV(2, double, double2); else MIGV(2, float, float4); }
        else { if (dtype) MIGV(3, double, double2); else MIGV(3, float, float4); }
#undef MIGV
        return launch_status(1);
    }
#define MIG(D, R) k_migrate<D, R><<<blocks_for(n, 256), 256, 0, s>>>(n, n_dev, old_slot, fields_of<R>(old0), \
        fields_of<R>(old1), fields_of<R>(new0), fields_of<R>(new1))
    if (dim == 2) { if (dtype) MIG(2, double); else MIG(2, float); }
    else { if (dtype) MIG(3, double); else MIG(3, float); }
#undef MIG
    return launch_status(1);
}

extern "C" int mlbm_copy_live_fields(int32_t dim, int32_t cap_tiles, const int32_t* n_dev,
                                     mlbm_fields_t src0, mlbm_fields_t src1, mlbm_fields_t dst0,
                                     mlbm_fields_t dst1, int32_t dtype, void* stream) {
    if (cap_tiles <= 0) return 0;
    if (dst0.stride != src0.stride || (dst1.ptr && (src1.stride != src0.stride || dst1.stride != src0.stride)))
        return -1;
    const int es = dtype ? 8 : 4;
    if ((src0.stride * es) % 16 != 0) return -1;
    const int T = dim == 2 ? 16 : 64;
    const int nf = dim == 2 ? Geo<2>::NF : Geo<3>::NF;
    const int64_t nvec = (int64_t)cap_tiles * T * es / 16, stride_vec = src0.stride * es / 16;
    const int64_t total = nvec * nf;
    cudaStream_t s = as_stream(stream);
#define CPY(D, R, V) k_copy_live<D, R, V><<<blocks_for(total, 256), 256, 0, s>>>(nvec, n_dev, nf, \
        (const V*)src0.ptr, (const V*)src1.ptr, (V*)dst0.ptr, (V*)dst1.ptr, stride_vec)
    if (dim == 2) { if (dtype) CPY(2, double, double2); else CPY(2, float, float4); }
    else { if (dtype) CPY(3, double, double2); else CPY(3, float, float4); }
#undef CPY
    return launch_status(1);
}

extern "C" int mlbm_init_new_cells(const mlbm_hier_t* old_h, const mlbm_hier_t* nh, int32_t level,
                                   const int32_t* tile_xyz, const int32_t* old_slot, int32_t n_tiles,
                                   const int32_t* n_dev,
                                   mlbm_fields_t new0, mlbm_fields_t new1, const double* taus,
                                   int32_t conv, int32_t dtype, int32_t* viol, void* stream) {
    const int T = old_h->dim == 2 ? 16 : 64;
    const int64_t n = (int64_t)n_tiles * T;
    if (n == 0) return 0;
    cudaStream_t s = as_stream(stream);
    (void)nh;
    const int64_t blocks = std::min<int64_t>(((int64_t)n_tiles + 255) / 256, 148 * 16);
#define INI(D, R) k_init_new<D, R><<<(unsigned)blocks, 256, 0, s>>>(*old_h, level, tile_xyz, old_slot, \
        n_tiles, n_dev, fields_of<R>(new0), fields_of<R>(new1), taus, conv, viol)
    if (old_h->dim == 2) { if (dtype) INI(2, double); else INI(2, float); }
    else { if (dtype) INI(3, double); else INI(3, float); }
#undef INI
    return launch_status(1);
}

// ---------------------------------------------------------------------------
// buffer initialisation inside the step (no framework fill kernels in the
// captured graphs): byte memset on the stream, typed fill for non-zero values
namespace mlbm {
template <typename T>
__global__ void k_fill(T* p, int64_t n, T v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}
}  // namespace mlbm

extern "C" int mlbm_memset(void* p, int32_t value, int64_t bytes, void* stream) {
    if (bytes <= 0) return 0;
    const cudaError_t e = cudaMemsetAsync(p, value, (size_t)bytes, as_stream(stream));
    return e == cudaSuccess ? 0 : -(int)e;
}

extern "C" int mlbm_fill(void* p, int64_t n, int32_t kind, double value, void* stream) {
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    const int B = 256;
    const int G = (int)std::min<int64_t>((n + B - 1) / B, 148 * 8);
    switch (kind) {
    case 0: k_fill<uint8_t><<<G, B, 0, s>>>((uint8_t*)p, n, (uint8_t)value); break;
    case 1: k_fill<int32_t><<<G, B, 0, s>>>((int32_t*)p, n, (int32_t)value); break;
    case 2: k_fill<float><<<G, B, 0, s>>>((float*)p, n, (float)value); break;
    case 3: k_fill<double><<<G, B, 0, s>>>((double*)p, n, value); break;
    default: return -1;
    }
    return launch_status(1);
}

// exclusive scan of n int32 in place (the compaction scan; used by the particle
// sort): per-block sums of the 1024-element blocks, one scan of the sums, and
// the block-local scan applied
namespace mlbm {
__global__ void k_block_sum(int n, const int32_t* __restrict__ v, int32_t* __restrict__ bsum) {
    __shared__ int ws[CB / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * CPB;
    int c = 0;
#pragma unroll
    for (int k = 0; k < CI; ++k) {
        const int64_t g = base + k * CB + threadIdx.x;
        c += g < n ? v[g] : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if (lane == 0) ws[wid] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < CB / 32; ++w) t += ws[w];
        bsum[blockIdx.x] = t;
    }
}
__global__ void k_block_apply(int n, int32_t* __restrict__ v, const int32_t* __restrict__ boff) {
    __shared__ int wsum[CB / 32];
    __shared__ int strip_total;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * CPB;
    int run = boff[blockIdx.x];
#pragma unroll 1
    for (int k = 0; k < CI; ++k) {
        const int64_t g = base + k * CB + threadIdx.x;
        const int x = g < n ? v[g] : 0;
        int t = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += u;
        }
        if (lane == 31) wsum[wid] = t;
        __syncthreads();
        int before = 0;
        for (int w = 0; w < wid; ++w) before += wsum[w];
        if (threadIdx.x == 0) {
            int tt = 0;
            for (int w = 0; w < CB / 32; ++w) tt += wsum[w];
            strip_total = tt;
        }
        if (g < n) v[g] = run + before + t - x;
        __syncthreads();
        run += strip_total;
        __syncthreads();
    }
}
}  // namespace mlbm

extern "C" int64_t mlbm_scan_ws_bytes(int32_t n) {
    return align256(4 * (int64_t)flag_blocks(n > 0 ? n : 1)) + 256;
}

extern "C" int mlbm_scan_i32(int32_t n, int32_t* data, int32_t* total, void* ws, int64_t ws_bytes,
                             void* stream) {
    if (n <= 0) return 0;
    if (ws_bytes < mlbm_scan_ws_bytes(n)) return -1;
    cudaStream_t s = as_stream(stream);
    const int nb = flag_blocks(n);
    int32_t* bsum = (int32_t*)ws;
    k_block_sum<<<nb, CB, 0, s>>>(n, data, bsum);
    k_scan_blocks<<<1, 1024, 0, s>>>(nb, bsum, total);
    k_block_apply<<<nb, CB, 0, s>>>(n, data, bsum);
    return 3;
}

extern "C" int mlbm_solid_near(const mlbm_level_t* lv, const mlbm_solid_t* solid, uint8_t* near, void* stream) {
    const int64_t n = (int64_t)lv->tiles[0] * lv->tiles[1] * lv->tiles[2];
    if (n <= 0) return 0;
    cudaStream_t s = as_stream(stream);
    mlbm_solid_t sl = *solid;
    for (int l = 0; l < MLBM_MAX_LEVELS; ++l) sl.near[l] = nullptr;
    if (lv->dim == 2) k_solid_near<2><<<blocks_for(n, 128), 128, 0, s>>>(*lv, sl, near);
    else k_solid_near<3><<<blocks_for(n, 128), 128, 0, s>>>(*lv, sl, near);
    return launch_status(1);
}

// ---------------------------------------------------------------------------
// Dirty tiles of an incremental classification, sparse: the tiles whose kind
// changed at one level (compacted list), and for every level the tiles within
// one tile of the region each changed tile covers (marked by scatter).
extern "C" int mlbm_changed_tiles(int64_t n, const uint8_t* old_kind, const uint8_t* new_kind,
                                  int32_t* list, int32_t* count, void* ws, int64_t ws_bytes,
                                  void* stream) {
    if (n <= 0) return 0;
    if (ws_bytes < mlbm_ws_bytes(n)) return -1;
    cudaStream_t s = as_stream(stream);
    int32_t* bsum = (int32_t*)((char*)ws + align256(4 * n));
    const int nb = flag_blocks(n);
    const ChangedFlag fl{old_kind, new_kind};
    k_flag_count<<<nb, CB, 0, s>>>(n, fl, bsum);
    k_scan_blocks<<<1, 1024, 0, s>>>(nb, bsum, count);
    k_flag_scatter<<<nb, CB, 0, s>>>(n, fl, bsum, TargetWriter{list});
    return launch_status(3);
}

namespace mlbm {
__global__ void k_mark_dirty(mlbm_hier_t h, int m, const int32_t* __restrict__ list,
                             const int32_t* __restrict__ count, uint8_t* d0, uint8_t* d1, uint8_t* d2,
                             uint8_t* d3, uint8_t* d4, uint8_t* d5) {
    uint8_t* dirty[6] = {d0, d1, d2, d3, d4, d5};
    const int dim = h.dim;
    const int nc = *count;
    const I3 dm = tdims_of(h, m);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)nc * h.levels;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(i / h.levels), l = (int)(i % h.levels);
        if (!dirty[l]) continue;
        int t[3];
        gdec3(dm.v, list[j], t[0], t[1], t[2]);
        const I3 dl = tdims_of(h, l);
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};       // level-l tiles, inclusive, before dilation
        for (int a = 0; a < 3; ++a) {
            if (a >= dim) continue;
            if (m >= l) { lo[a] = t[a] << (m - l); hi[a] = ((t[a] + 1) << (m - l)) - 1; }
            else { lo[a] = t[a] >> (l - m); hi[a] = lo[a]; }
            lo[a] -= 1;
            hi[a] += 1;
        }
        for (int z = lo[2]; z <= hi[2]; ++z)
            for (int y = lo[1]; y <= hi[1]; ++y)
                for (int x = lo[0]; x <= hi[0]; ++x) {
                    int c[3] = {x, y, z};
                    bool in = true;
                    for (int a = 0; a < 3; ++a) {
                        if (a >= dim) { c[a] = 0; continue; }
                        if (h.periodic[a]) c[a] = (c[a] % dl.v[a] + dl.v[a]) % dl.v[a];
                        else in &= c[a] >= 0 && c[a] < dl.v[a];
                    }
                    if (in) dirty[l][gidx3(dl.v, c[0], c[1], c[2])] = 1;
                }
    }
}
}  // namespace mlbm

extern "C" int mlbm_mark_dirty(const mlbm_hier_t* h, int32_t level, const int32_t* list,
                               const int32_t* count, uint8_t* const* dirty, void* stream) {
    uint8_t* d[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    for (int l = 0; l < h->levels && l < 6; ++l) d[l] = dirty[l];
    k_mark_dirty<<<148 * 4, 128, 0, as_stream(stream)>>>(*h, level, list, count, d[0], d[1], d[2], d[3],
                                                         d[4], d[5]);
    return launch_status(1);
}
