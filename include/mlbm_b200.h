/*
 * mlbm_b200.h — C ABI of the B200-native hot path of arXiv 2603.14982's
 * adaptive multi-level HOME-LBM <-> MPM coupled solver.
 *
 * Every entry point is extern "C", takes device pointers + sizes + a CUDA
 * stream (as void*), never allocates persistently (scratch comes from a
 * caller-provided workspace), is asynchronous on the given stream and returns
 * an int status (>= 0: number of kernels launched, < 0: bad argument / launch
 * failure, -cudaError).  Numerical
 * failures (divergence, topology violations) are written to a device-side
 * mlbm_error_t record that the host reads after the step.
 *
 * Each entry names the reference Python seam it replaces
 * (paths relative to the reference package root pkg/src/mlbm/).
 *
 * Data layout:
 *   - tiles of 4^dim cells; within-tile cell index lx + 4 ly + 16 lz
 *   - per level, tiles stored in sorted (x, y, z) slot order; cell = slot*4^dim + local
 *   - fields: structure of arrays, field k at base + k*stride (elements);
 *     order drho, u[dim], S[dim(dim+1)/2] (xx,xy,(xz),yy,(yz),(zz)), eps, f[dim], phi
 *     (drho = rho - 1 is the stored density: the shifted form keeps fp32 exact enough)
 *   - dtype 0 = float32, 1 = float64
 */
#ifndef MLBM_B200_H
#define MLBM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLBM_MAX_LEVELS 6
#define MLBM_MAX_BOXES 16

/* face order x_min, x_max, y_min, y_max, z_min, z_max */
enum { MLBM_FACE_PERIODIC = 0, MLBM_FACE_WALL = 1, MLBM_FACE_OUTLET = 2,
       MLBM_FACE_LOG_INLET = 3 };

/* cell flag bits */
enum { MLBM_CF_ACTIVE = 1, MLBM_CF_SOLID = 2, MLBM_CF_GHOST_D = 4,
       MLBM_CF_GHOST_U = 8, MLBM_CF_BC = 16, MLBM_CF_SPECIAL = 32,
       MLBM_CF_LEAF = 64 };

/* tile flag bits */
enum { MLBM_TF_PLAIN = 1,      /* every cell active and non-special */
       MLBM_TF_BC = 2,         /* holds an outlet / inlet layer cell */
       MLBM_TF_LEAF = 4 };

/* error codes in mlbm_error_t.code (first error wins) */
enum { MLBM_OK = 0, MLBM_ERR_DENSITY = 1, MLBM_ERR_VELOCITY = 2,
       MLBM_ERR_TOPOLOGY = 3, MLBM_ERR_STENCIL = 4, MLBM_ERR_DOMAIN = 5 };

typedef struct {
    int32_t code;
    int32_t level;
    int32_t count;
    int32_t cells[5][3];
    int32_t detail;
} mlbm_error_t;

/* One level of the sparse tile hierarchy (device pointers). */
typedef struct {
    int32_t dim;
    int32_t level;
    int32_t cells[3];           /* cells per axis at this level (1 for unused z) */
    int32_t tiles[3];           /* tiles per axis */
    int32_t periodic[3];
    int32_t n_tiles;
    const int32_t* tile_map;    /* dense tile grid -> slot or -1, index (x*ty + y)*tz + z */
    const int32_t* tile_xyz;    /* [n_tiles][3] */
    const int32_t* nbr;         /* [n_tiles][3^dim], offset index ox + 3 oy + 9 oz, o = d+1 */
    const uint8_t* cell_flags;  /* [n_tiles * 4^dim] MLBM_CF_* */
    const uint64_t* dir_masks;  /* [n_tiles * 4^dim] bit i: bounce-back dir i; bit 32+i: self source */
    const uint8_t* tile_flags;  /* [n_tiles] MLBM_TF_* */
    const int32_t* counts;      /* device: [0] live tiles, [1] |I^d|, [2] |I^u| (or NULL:
                                 * n_tiles is exact).  With counts, n_tiles is the
                                 * allocated capacity and sizes the launch grids, so a
                                 * captured CUDA graph survives topology changes. */
    int32_t first;              /* first slot the level step / diagnostics process
                                 * (slots [first, live)); 0 except for slab ranks, whose
                                 * x-sorted slots start with a ghost tile column */
} mlbm_level_t;

typedef struct {
    void* ptr;                  /* field 0 */
    int64_t stride;             /* elements between consecutive fields */
} mlbm_fields_t;

typedef struct {
    int32_t face[6];
    double inlet_u0, inlet_beta, inlet_y0;
    double rho0;
} mlbm_bc_t;

typedef struct {
    int32_t n_boxes;
    double boxes[MLBM_MAX_BOXES][6];   /* lo[3], hi[3] in finest units (2D: lo x,y,_ hi x,y,_) */
    const float* heightmap;            /* finest (x[, z]) heights or NULL */
    int32_t hm_dims[2];
    /* per level (or NULL): 1 where a solid lies within one cell of the tile
     * (mlbm_solid_near, computed once: the geometry is static) */
    const uint8_t* near[MLBM_MAX_LEVELS];
} mlbm_solid_t;

typedef struct {
    double tau;                 /* level relaxation time */
    double gravity[3];          /* lattice gravity (force = rho g 2^level) */
    double h3_xyz;              /* 3D Hermite coefficient of Gamma_xyz */
    int32_t force_mode;         /* 0: gravity; 1: per-cell f fields of dst */
    int32_t tau_mode;           /* 0: scalar tau; 1: tau0 * eps field of dst; 2: tau_ptr[cell] */
    double tau0;
    const void* tau_ptr;        /* per-cell relaxation times (tau_mode 2), run dtype */
} mlbm_collide_t;

/* ---- LBM level kernels ------------------------------------------------- */

/* mode: 0 fused stream+collide+boundary (solver.py:483-488),
 *       1 stream only   (solver.py:336-381 stream_kernel),
 *       2 collide+boundary (solver.py:394-453 collide_kernel +
 *         solver.py:460-481 boundary_kernel), 3 collide only, 4 boundary only. */
int mlbm_level_step(const mlbm_level_t* lv, mlbm_fields_t src, mlbm_fields_t dst,
                    int32_t dtype, int32_t mode, const mlbm_collide_t* cp,
                    const mlbm_bc_t* bc, mlbm_error_t* err, void* stream);

/* I^d fill (solver.py:501-526 downward_kernel): targets [n], src [n][2^dim]
 * coarse cell indices (-1 where the weight is zero).  step 1 or 2.  n is the
 * launch capacity; n_dev (device, may be NULL) the live count. */
int mlbm_downward(int32_t dim, int32_t n, const int32_t* n_dev, const int32_t* targets,
                  const int32_t* src,
                  const int32_t* fine_tile_xyz,
                  mlbm_fields_t olda, mlbm_fields_t newa, mlbm_fields_t dst,
                  int32_t dtype, int32_t step, double kappa, void* stream);

/* I^u fill (solver.py:536-560 upward_kernel): src [n][2^dim], column 0 is the
 * coincident child; average != 0 uses the 2^dim mean. */
int mlbm_upward(int32_t dim, int32_t n, const int32_t* n_dev, const int32_t* targets,
                const int32_t* src,
                mlbm_fields_t fine, mlbm_fields_t dst, int32_t dtype,
                int32_t average, double kappa, void* stream);

/* ---- tile hierarchy ------------------------------------------------------ */

/* Whole-hierarchy view passed to the topology / adapt / migration kernels.
 * kind[l]: dense tile grid of level l (index (x*ty + y)*tz + z): 0 absent,
 * 1 leaf, 2 border.  tile_map[l]: dense grid -> slot or -1.  fields[t][l]:
 * field base of tree t at level l (only used by migration). */
typedef struct {
    int32_t dim, levels;
    int32_t finest[3];          /* finest cells per axis (unused axes = 4) */
    int32_t periodic[3];
    const uint8_t* kind[MLBM_MAX_LEVELS];
    const int32_t* tile_map[MLBM_MAX_LEVELS];
    void* fields[2][MLBM_MAX_LEVELS];
    int64_t stride[MLBM_MAX_LEVELS];
    int32_t n_tiles[MLBM_MAX_LEVELS];
} mlbm_hier_t;

/* bytes of scratch for the scans / selections over n items */
int64_t mlbm_ws_bytes(int64_t n);

/* ---- topology (sparse_grid.py:183-200 rebuild_level, 210-282 rasters) ---- */

/* Compacts a level's kind grid into sorted slots (x, y, z lexicographic =
 * reference sorted(coords) order).  Writes tile_map, tile_xyz[n][3],
 * tile_kind[n], old_slot[n] (slot of the same tile in old_map or -1) and
 * counts[0] = n tiles, counts[1] = fresh tiles; slots >= capacity are not written. */
int mlbm_compact_tiles(int32_t dim, const int32_t tiles[3], const uint8_t* kind,
                       const int32_t* old_map, int32_t* tile_map, int32_t* tile_xyz,
                       uint8_t* tile_kind, int32_t* old_slot, int32_t capacity, int32_t* counts,
                       void* ws, int64_t ws_bytes, void* stream);

/* 3^dim neighbour slots per tile with periodic wrap (-1 absent / outside). */
int mlbm_build_neighbors(const mlbm_level_t* lv, int32_t* nbr, void* stream);

/* Per-cell classification of one level (sparse_grid.py:468-544
 * classify_interfaces, solver.py:177-273 _LevelTables): I^d / I^u ghosts,
 * BC layer, solid, active, per-direction bounce-back / self-source masks,
 * tile flags.  counts[0] += |I^d|, counts[1] += |I^u|; violations -> err.
 * Incremental (dirty non-NULL, over the level's tile grid): a tile not marked
 * dirty copies its flags / masks / tile flag from the old arrays at
 * old_slot[tile] (NULL: the same slot) instead of being classified; dirty =
 * the tiles within one tile of a kind change at any level (mlbm_bitmap_op).
 * work (optional, incremental only): int32 [1 + n_tiles]; with it the clean
 * tiles are copied one warp per tile and only the listed dirty tiles are
 * classified (persistent grid); NULL: one block per tile. */
/* the static near-solid map of one level over its whole tile grid (1 where a
 * solid box or the heightmap reaches within one cell of the tile; periodic
 * seams always 1), read by mlbm_classify_level instead of rescanning the
 * geometry at every rebuild */
int mlbm_solid_near(const mlbm_level_t* lv, const mlbm_solid_t* solid, uint8_t* near, void* stream);

int mlbm_classify_level(const mlbm_level_t* lv, const mlbm_hier_t* h,
                        const mlbm_bc_t* bc, const mlbm_solid_t* solid,
                        uint8_t* cell_flags, uint64_t* dir_masks, uint8_t* tile_flags,
                        int32_t* counts, mlbm_error_t* err, const uint8_t* dirty,
                        const int32_t* old_slot, const uint8_t* old_cf,
                        const uint64_t* old_masks, const uint8_t* old_tf, int32_t* work,
                        void* stream);
/* the tiles of a level whose kind differs between two kind grids (stable
 * compaction; count[0] = how many; ws: mlbm_ws_bytes(n)), and the scatter of
 * the dirty maps of mlbm_classify_level: for every changed tile of `level` and
 * every level l with dirty[l] non-NULL, the level-l tiles within one tile of the
 * region it covers are marked 1 (dirty maps zeroed by the caller) */
int mlbm_changed_tiles(int64_t n, const uint8_t* old_kind, const uint8_t* new_kind, int32_t* list,
                       int32_t* count, void* ws, int64_t ws_bytes, void* stream);
int mlbm_mark_dirty(const mlbm_hier_t* h, int32_t level, const int32_t* list,
                    const int32_t* count, uint8_t* const* dirty, void* stream);
/* device-to-device copy on the stream */
int mlbm_copy(void* dst, const void* src, int64_t bytes, void* stream);

/* Compacts the I^d (which = 0) / I^u (which = 1) cells of `lv` in cell order
 * and builds their 2^dim stencils into the coarser / finer level `other`
 * (sparse_grid.py:439-465, 500-543).  counts[0] = n. */
int mlbm_build_interface(const mlbm_level_t* lv, const mlbm_level_t* other, int32_t which,
                         int32_t* targets, int32_t* src, int32_t* counts,
                         mlbm_error_t* err, void* ws, int64_t ws_bytes, void* stream);

/* ---- block maintenance (adapt.py) --------------------------------------- */

/* seeds |= tile of floor(x) (adapt.py:54-65); x is [n][dim] SoA (x + a*xstride). */
int mlbm_seed_tiles(int32_t dim, int32_t n, const void* x, int64_t xstride, int32_t dtype,
                    const int32_t tiles0[3], uint8_t* seeds, mlbm_error_t* err, void* stream);

/* out = op(in) over a level's tile grid (dims = child grid for group ops):
 * op 0 align_up (adapt.py:77-81), 1 parents (adapt.py:84-87; out on the parent
 * grid), 2 or-into (out |= in), 3 and-not (out &= ~in), 4 copy, 5 fill ones,
 * 6 leaf-of-kind (out = kind == 1), 7 non-zero, 8 differs (out = out != in),
 * 9 raw copy, 10 or-parent (out |= in at the parent tile; dims = child grid). */
int mlbm_bitmap_op(int32_t op, int32_t dim, const int32_t dims[3], const uint8_t* in,
                   uint8_t* out, void* stream);

/* Chebyshev dilation by r tiles, separable, periodic per axis
 * (sparse_grid.py:358-363); tmp has the grid's size. */
int mlbm_dilate(int32_t dim, const int32_t dims[3], const int32_t periodic[3], int32_t r,
                const uint8_t* in, uint8_t* out, uint8_t* tmp, void* stream);

/* One level of adapt.py:152-182 (_effective_cumulative):
 * cand = cur & ~des; streak = cand ? streak + 1 : 0;
 * avail = streak >= 2 & cand & ~guard; act = avail on complete sibling groups;
 * eff = des | (cur & ~act) | par_prev (par_prev may be NULL). */
int mlbm_effective_level(int32_t dim, const int32_t dims[3], const uint8_t* des,
                         const uint8_t* cur, const uint8_t* guard, const uint8_t* par_prev,
                         int16_t* streak, uint8_t* eff, void* stream);

/* adapt.py:184-194 + no-op test: own = eff & ~par_finer; storage = dilate(own, 2);
 * new kind = own ? 1 : storage ? 2 : 0; changed[0] |= (new kind != old kind).
 * `storage` is the already-dilated own bitmap. */
int mlbm_plan_level(int32_t n, const uint8_t* own, const uint8_t* storage,
                    const uint8_t* old_kind, uint8_t* new_kind, int32_t* changed,
                    void* stream);

/* The whole per-update bitmap pass in ONE cooperative launch (grid barriers
 * between the stages of adapt.py:54-194 + 374-389): seeds, desired / current
 * cumulative coverage, int16 hysteresis, plan, no-op flags status[0..L-1],
 * invariant counts status[L..L+2] of the current topology (ring violations
 * are counted as (leaf, absent neighbour) pairs), and per level the tile count
 * status[L+4+l] and fresh-tile count status[2L+4+l] of the new plan.  Per-level buffer
 * arrays have h->levels entries; bar: 2 zero-initialised words.  Seeds come either
 * from the n positions x (stride xs) or, with n = 0 and ext_count non-NULL, from
 * mlbm_g2p of the same step (seeds filled, *ext_count = its leaf-invariant count,
 * consumed and reset to 0 here).  seeds are all zero again on return.
 * win (optional, int32 [2][levels][6], caller-owned, used only with ext_count):
 * per level the tile window of the last pass (lo xyz, hi xyz inclusive; empty
 * when lo > hi) and the bounding box of its non-zero kinds; the pass works
 * inside max(last window, kinds box + 8 tiles, parent footprint of the finer
 * window + 8 tiles) and writes both back (the top level, periodic axes and
 * win = NULL span the whole grid).  Every bitmap buffer must be zero outside
 * the windows: start from zeroed buffers and never shrink a window. */
int mlbm_adapt_pass(const mlbm_hier_t* h, uint8_t* const* des, uint8_t* const* cur,
                    uint8_t* const* eff, uint8_t* const* par, uint8_t* const* own,
                    uint8_t* const* nkind, uint8_t* const* stor, int16_t* const* streak,
                    uint8_t* seeds, const uint8_t* static_tiles, const double* x, int64_t xs,
                    int32_t n, int32_t* ext_count, int32_t* win, int32_t* status, mlbm_error_t* err,
                    unsigned int* bar, void* stream);
/* optional stage timestamps of the adapt passes into a caller-owned buffer of 64
 * uint64 (NULL: off); the library never allocates */
int mlbm_adapt_set_timestamps(unsigned long long* buf);
int mlbm_adapt_bits_set_timestamps(unsigned long long* buf);

/* Invariants (adapt.py:374-389): leaf coverage of every finest tile exactly
 * once, two-tile rings, particles inside level-0 leaves -> viol[0..2]. */
int mlbm_check_coverage(const mlbm_hier_t* h, int32_t* viol, void* stream);
int mlbm_count_ring_violations(int64_t n, const uint8_t* dilated_leaf, const uint8_t* kind,
                                int32_t* viol, void* stream);
int mlbm_check_particles(int32_t dim, int32_t n, const void* x, int64_t xstride,
                         int32_t dtype, const int32_t tiles0[3], const uint8_t* kind0,
                         int32_t* viol, void* stream);

/* Data migration after a rebuild (adapt.py:259-283): both trees, surviving
 * tiles bitwise, fresh tiles get drho = 0, eps = 1, others 0.  A null second
 * tree (new1.ptr == NULL) migrates only the first (the coupled step's level 0,
 * whose other tree is rewritten before it is read); mlbm_init_new_cells and
 * mlbm_copy_live_fields accept the same. */
int mlbm_migrate_level(int32_t dim, int32_t n_new_tiles, const int32_t* n_dev,
                       const int32_t* old_slot,
                       mlbm_fields_t old0, mlbm_fields_t old1, mlbm_fields_t new0,
                       mlbm_fields_t new1, int32_t dtype, void* stream);

/* Copy the live cells (device count n_dev, capacity cap_tiles) of two field
 * blocks into two others of the same stride: the migrated scratch blocks back
 * into the trees after a rebuild (adapt.py:266-279 replaces the arrays; the
 * device trees keep their pointers so captured graphs stay valid). */
int mlbm_copy_live_fields(int32_t dim, int32_t cap_tiles, const int32_t* n_dev,
                          mlbm_fields_t src0, mlbm_fields_t src1, mlbm_fields_t dst0,
                          mlbm_fields_t dst1, int32_t dtype, void* stream);

/* New-cell initialisation (adapt.py:301-372): for every cell of a fresh
 * tile of level `level` (new topology `nh`), interpolate from the nearest old
 * coarser level whose stencil is complete (S chain down), else copy the
 * coincident old finer cell (S chain up).  taus[] per level, conv 0 derived /
 * 1 paper_literal.  Unfilled cells counted into viol[0]. */
int mlbm_init_new_cells(const mlbm_hier_t* old_h, const mlbm_hier_t* nh, int32_t level,
                        const int32_t* tile_xyz, const int32_t* old_slot, int32_t n_tiles,
                        const int32_t* n_dev,
                        mlbm_fields_t new0, mlbm_fields_t new1, const double* taus,
                        int32_t conv, int32_t dtype, int32_t* viol, void* stream);

/* ---- MPM + coupling (granular.py, coupling.py) -------------------------- */

/* row counts of the level-0 raster and of the particle state */
int mlbm_raster_rows(int32_t dim);
int mlbm_particle_rows(int32_t dim);

/* Kirchhoff stress rows tau(F) = U diag(2 mu ln s + lam tr ln s) U^T
 * (granular.py:260-279) of every particle from its F rows.  mlbm_g2p keeps them
 * current (from its own decomposition of the updated F); call this once after
 * F is set from outside (initial state, user edits).  mlbm_p2g and the stress
 * rasters read these rows. */
int mlbm_particle_stress(int32_t dim, int32_t n, void* p, int64_t ps, double lam, double mu,
                         double alpha, int32_t dtype, void* stream);

/* stencil + Kirchhoff stress + P2G scatter fused with rasterize_fractions
 * (granular.py:137-178, 260-310; coupling.py:96-131).  x: float64 [dim][ps];
 * p: run-dtype particle rows [rows][ps]; ras: zeroed accumulator rows. */
int mlbm_p2g(const mlbm_level_t* lv0, int32_t n, const double* x, void* p, int64_t ps,
             double lam, double mu, double alpha, void* ras, int64_t rs, int32_t dtype,
             int32_t smem, mlbm_error_t* err, void* stream);

/* MPM particle sort (no reference counterpart — ordering only, SURVEY.md
 * §2.3 K7): a bucketed counting sort by (level-0 tile slot, cell) of the
 * stencil base cell — slot histogram, exclusive scan (mlbm_scan_i32), scatter
 * into the slot ranges, one CTA per slot sorting its range by cell — then every
 * particle row (positions, state rows, ids) gathered into the _out buffers.
 * ws: mlbm_sort_ws_bytes(n, lv0->n_tiles) bytes (the level's slot capacity).
 * In mlbm_p2g, smem = 1 accumulates per block in shared memory over the
 * block's bounding box; smem = 2 accumulates per warp in registers (nodes
 * owned by lanes, particles broadcast by shuffles); smem = 3 lets lane k own
 * stencil node k of the current cell and flushes per cell into a block box;
 * smem = 4 (fp32 only, the default for fp32 runs; fp64 falls back to 3) keeps
 * one box copy per warp so the per-cell flushes need no shared-memory atomics
 * — all four need sorted input. */
int64_t mlbm_sort_ws_bytes(int64_t n, int64_t n_slots);
int mlbm_particle_sort(const mlbm_level_t* lv0, int32_t n, const double* x, const void* p,
                       const int32_t* pid, int64_t ps, double* x_out, void* p_out,
                       int32_t* pid_out, int32_t dtype, void* ws, int64_t ws_bytes,
                       void* stream);

/* per level-0 cell: eps, Di Felice drag + limiter, grad eps, mixture force
 * (written into both trees), MPM grid update with wall / sticky projection
 * (coupling.py:134-197, 379-446; granular.py:313-341).  mode 1: full exchange;
 * mode 0: grid update only, with the drag already in the FS rows. */
int mlbm_exchange(const mlbm_level_t* lv0, mlbm_fields_t w_tree, mlbm_fields_t r_tree,
                  mlbm_fields_t tree0, mlbm_fields_t tree1, void* ras, int64_t rs,
                  double eps_min, double nu, double d_p, double re_min, double dt,
                  double rho0, const double* g_fluid, const double* g_sed,
                  const int32_t* faces, double floor_friction, int32_t mode,
                  int32_t dtype, void* stream);

/* the coupled level-0 phase in ONE kernel (level_kernel mode 5): pull-stream of
 * src into registers, then per cell the exchange of mlbm_exchange (mode 1) on
 * those bare moments (eps and force into both trees' rows, the raster rows, the
 * MPM grid update), then the collide with that force and tau = eps tau0 and the
 * boundary passes into dst (coupling.py:403-446 between solver.py:336 and
 * :394 / :460).  P2G must have filled ras; G2P reads its VEL rows after. */
int mlbm_level0_coupled(const mlbm_level_t* lv, mlbm_fields_t src, mlbm_fields_t dst,
                        mlbm_fields_t tree0, mlbm_fields_t tree1, int32_t dtype,
                        const mlbm_collide_t* cp, const mlbm_bc_t* bc, void* ras, int64_t rs,
                        double eps_min, double nu, double d_p, double re_min, double dt,
                        double rho0, const double* g_fluid, const double* g_sed,
                        const int32_t* faces, double floor_friction, mlbm_error_t* err,
                        void* stream);

/* gather, advect (wrap / clamp to [2, dim-2]), F update, SVD + Drucker-Prager
 * (granular.py:344-412), reading the (sorted) _in rows and writing the _out rows
 * (in place when they alias); the tau rows get the Kirchhoff stress of the new F.
 * clamped[0] += clamped coordinates; clamped[1] |= CFL violation (max |v| dt >= 0.5,
 * granular.py:428-432).  seeds (optional, level-0 tile grid bytes, all zero on
 * entry): seeds[tile of floor(x_new) // 4] = 1 for the adapt pass that follows
 * (adapt.py:54-65), with nonleaf[0] += particles whose tile is not a level-0 leaf
 * of kind0 (adapt.py:374-389) and MLBM_ERR_DOMAIN for a non-finite position;
 * mlbm_adapt_pass then runs with n = 0 and ext_count = nonleaf. */
/* NACC snow (absent from the reference, oracle/mpm.py:
 * nacc_return_map is the specification): critical-state slope M, cohesion beta,
 * hardening factor xi, softening coefficient alpha_soft.  With snow non-NULL,
 * mlbm_g2p's return map is NACC on the Hencky elasticity (lam, mu) and the
 * vol_corr row holds the hardening state (q >= 0; -(q + 1) once cracked). */
typedef struct {
    double M, beta, xi, alpha_soft;
} mlbm_snow_t;

int mlbm_g2p(const mlbm_level_t* lv0, int32_t n, const double* x_in, double* x_out,
             const void* p_in, void* p_out, const int32_t* pid_in, int32_t* pid_out,
             int64_t ps, double lam, double mu, double alpha, const mlbm_snow_t* snow,
             const void* ras, int64_t rs,
             double dt, int32_t plastic, int32_t dtype, int32_t* clamped,
             uint8_t* seeds, const uint8_t* kind0, int32_t* nonleaf, mlbm_error_t* err,
             void* stream);

/* entrainment stress raster (coupling.py:283-294) and powder transport
 * (coupling.py:230-272, 275-322, 483-498). tmp: [n0] run-dtype scratch. */
int mlbm_stress_raster(const mlbm_level_t* lv0, int32_t n, const double* x, const void* p,
                       int64_t ps, double lam, double mu, double alpha, void* ras, int64_t rs,
                       int32_t dtype, mlbm_error_t* err, void* stream);
/* fp32: the stress raster restricted to the entrainment surface (the only
 * cells k_powder reads it at).  surf [n0] floats receives 2 on surface cells
 * (0 < eta < eta_surface with an absent / empty face neighbour) and 1 on the
 * other cells of their 3^D neighbourhoods; particles whose nearest node has
 * surf == 0 (no surface cell in their stencil) are skipped, so the sums at
 * surface cells equal mlbm_stress_raster's.  fp64: the full raster. */
int mlbm_stress_raster_surface(const mlbm_level_t* lv0, int32_t n, const double* x,
                               const void* p, int64_t ps, double lam, double mu, double alpha,
                               void* ras, int64_t rs, double eta_surface, void* surf,
                               int32_t dtype, mlbm_error_t* err, void* stream);
/* tile_ws (optional, 2 x lv0->n_tiles bytes): per tile whether phi is non-zero
 * within its 3^dim tile neighbourhood; cells of inactive tiles skip the RK3
 * velocity sampling (their advected value is exactly 0). */
int mlbm_powder(const mlbm_level_t* lv0, mlbm_fields_t src, mlbm_fields_t dst, void* ras,
                int64_t rs, void* tmp, uint8_t* tile_ws, double diffusion, double sign,
                double dt, double entrain, double eta_surface, int32_t with_source,
                int32_t dtype, void* stream);

/* The reference's standalone coupling functions as per-cell passes over the
 * level-0 raster (the fused mlbm_exchange runs the same device code):
 *   MLBM_COUPLE_FRACTIONS     rasterize_fractions' finish (coupling.py:96-131): a0 = phi;
 *                             ETAE = max(eta - phi, 0), EPS = clip(1 - eta_eff - phi,
 *                             eps_min, 1), VMOM <- v_cell = sum w m v / mass
 *   MLBM_COUPLE_DRAG          difelice_drag (coupling.py:134-156): a0 = rho, u = velocity
 *                             rows [dim][us]; FS, REL rows (no limiter)
 *   MLBM_COUPLE_LIMIT         CoupledSim._limit_drag (coupling.py:379-401) on the FS rows
 *   MLBM_COUPLE_GRAD_EPS      grad_eps (coupling.py:159-182) of a0 (NULL: the EPS row) into
 *                             out [dim][os]
 *   MLBM_COUPLE_MIXTURE_FORCE mixture_force (coupling.py:185-197): a0 = rho; GRAD rows,
 *                             out [dim][os] = force on the fluid (g = lattice gravity) */
enum { MLBM_COUPLE_FRACTIONS = 0, MLBM_COUPLE_DRAG = 1, MLBM_COUPLE_LIMIT = 2,
       MLBM_COUPLE_GRAD_EPS = 3, MLBM_COUPLE_MIXTURE_FORCE = 4 };
int mlbm_coupling_op(const mlbm_level_t* lv0, int32_t op, void* ras, int64_t rs, const void* a0,
                     const void* u, int64_t us, void* out, int64_t os, double eps_min,
                     double nu, double d_p, double re_min, double dt, double rho0,
                     const double* g, int32_t dtype, void* stream);

/* granular.stencil (granular.py:137-178): for particle p and node k of its 3^dim
 * stencil (offsets k % 3, (k / 3) % 3, k / 9): idx[k][os] flat level-0 cell, w[k][os]
 * weight, grad[b][k][os] dw/dx_b, dpos[b][k][os] node - particle.  Nodes outside a
 * non-periodic domain or not stored at level 0 -> idx -1 and MLBM_ERR_STENCIL. */
int mlbm_stencil(const mlbm_level_t* lv0, int32_t n, const double* x, int64_t ps, int32_t* idx,
                 void* w, void* grad, void* dpos, int64_t os, int32_t dtype, mlbm_error_t* err,
                 void* stream);

/* powder_step (coupling.py:230-272): RK3 semi-Lagrangian backtrace of src's phi
 * row along dst's velocity rows, 2*dim-point diffusion (sign = +1 stable, -1 the
 * printed form), + dt * source[c] when source is non-NULL; writes dst's phi row.
 * tmp: [n0] run-dtype scratch. */
int mlbm_powder_step(const mlbm_level_t* lv0, mlbm_fields_t src, mlbm_fields_t dst, void* tmp,
                     double diffusion, double sign, double dt, const void* source,
                     int32_t dtype, void* stream);

/* diagnostics (coupling.py:500-531): out[0..dim-1] += vol sum rho u, out[dim] +=
 * vol sum phi, out[dim+1] = min(out[dim+1], eps) over leaf cells;
 * particles: out[0..dim-1] += sum m v, out[dim..2dim-1] += sum fs over the first
 * min(n0, live[0] * tile cells) raster cells (live may be NULL: n0 cells). */
int mlbm_diag_level(const mlbm_level_t* lv, mlbm_fields_t f, double vol, int32_t dtype,
                    double* out, void* stream);
int mlbm_diag_particles(int32_t dim, int32_t n, const void* p, int64_t ps, const void* ras,
                        int64_t rs, int64_t n0, const int32_t* live, int32_t dtype,
                        double* out, void* stream);

/* ---- slab staging for the multi-GPU decomposition ------ */

/* ghost / edge tile columns of a SoA block <-> a contiguous NCCL buffer:
 * buf[r][c - lo] = src[r * stride + c] for r < nrows, lo <= c < hi (elem_bytes
 * 1, 4 or 8); unpack copies back, or adds (add = 1: the ghost-node partial sums
 * of collective (ii); dtype 0 f32, 1 f64). */
int mlbm_halo_pack(const void* src, int64_t stride, int32_t nrows, int64_t lo, int64_t hi,
                   void* buf, int32_t elem_bytes, void* stream);
int mlbm_halo_unpack(const void* buf, void* dst, int64_t stride, int32_t nrows, int64_t lo,
                     int64_t hi, int32_t dtype, int32_t add, void* stream);

/* particle migration (collective (iii)): a stable partition of the n particles
 * (float64 x [dim][ps], run-dtype rows [rows][ps], ids) into keep (x[0] in
 * [lo, hi) or no neighbour that side), to-left and to-right, with warp-ballot +
 * block-scan compaction.  mlbm_migrate_count writes counts[3] = keep, left, right
 * and the per-block offsets into ws (mlbm_migrate_ws_bytes(n)); mlbm_migrate_pack
 * (same ws, after the host sized the buffers from counts) scatters every class
 * in order: keep to the _keep buffers (row stride ks), the leavers to the _left /
 * _right buffers (row strides ls / rs: one contiguous message per direction)
 * with x[0] shifted by x0 into global coordinates and wrapped into [0, gx). */
int64_t mlbm_migrate_ws_bytes(int32_t n);
int mlbm_migrate_count(int32_t n, const double* x, double lo, double hi, int32_t has_left,
                       int32_t has_right, int32_t* counts, void* ws, int64_t ws_bytes,
                       void* stream);
int mlbm_migrate_pack(int32_t dim, int32_t n, const double* x, const void* p, const int32_t* pid,
                      int64_t ps, int32_t rows, int32_t dtype, double lo, double hi, double x0,
                      double gx, int32_t has_left, int32_t has_right, double* x_keep,
                      void* p_keep, int32_t* pid_keep, int64_t ks, double* x_left,
                      void* p_left, int32_t* id_left, int64_t ls, double* x_right,
                      void* p_right, int32_t* id_right, int64_t rs, const void* ws,
                      int64_t ws_bytes, void* stream);
/* arrivals (m received records, stride in_stride) appended at particle index at:
 * x[0] mapped from global coordinates into the local box [0, local_len) */
int mlbm_migrate_unpack(int32_t dim, int32_t m, const double* x_in, const void* p_in,
                        const int32_t* id_in, int64_t in_stride, int32_t rows, int32_t dtype,
                        double x0, double gx, double local_len, double* x, void* p,
                        int32_t* pid, int64_t ps, int32_t at, void* stream);

/* exclusive scan of n int32 in place (block sums, one scan of the sums, block
 * scans; no library scan), total (optional) = the sum; ws: mlbm_scan_ws_bytes */
int64_t mlbm_scan_ws_bytes(int32_t n);
int mlbm_scan_i32(int32_t n, int32_t* data, int32_t* total, void* ws, int64_t ws_bytes,
                  void* stream);

/* buffer initialisation on the stream (used inside the captured step graphs
 * instead of framework fill kernels): mlbm_memset = cudaMemsetAsync of bytes;
 * mlbm_fill writes n elements of kind 0 u8, 1 i32, 2 f32, 3 f64 = value. */
int mlbm_memset(void* p, int32_t value, int64_t bytes, void* stream);
int mlbm_fill(void* p, int64_t n, int32_t kind, double value, void* stream);

#ifdef __cplusplus
}
#endif
#endif
