/*
 * tilu.h -- C ABI of the B200 (sm_100a) surrogate ILU(0) smoother library (libtilu.so).
 *
 * The drop-in boundary for the hot path of arXiv 2210.15280's matrix-free ILU(0)
 * smoother (reference: /root/reference/pkg/src/tetilu, "tetilu").  The reference's
 * path is pure Python + Numba; the entry points below are what its Python layer
 * would bind through ctypes in place of the Numba kernels (INTEGRATION.md shows the
 * binding).  Every function states the reference interface it replaces.
 *
 * Conventions (reference geometry.py:188-215, _kernels.py:1-7):
 *   - n = 2^level; a macro-tet vector is fp64[grid] with grid = (n+1)(n+2)(n+3)/6,
 *     full-lattice rank order (z, then y, then x), ZERO outside the interior
 *     (x,y,z >= 1, x+y+z <= n-1).  Batches of independent macro-tets are stored
 *     back to back: fp64[ntets][grid].
 *   - Vector pointers passed to tilu_* compute calls are DEVICE pointers; the plan
 *     descriptor's coefficient arrays are HOST pointers (copied at plan creation).
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*, NULL = legacy
 *     default stream) and is asynchronous with respect to the host.
 *   - Status codes instead of exceptions: 0 = ok, see TILU_E* below;
 *     tilu_last_error() returns a thread-local message for the last failure.
 *   - A plan is immutable after creation.  Concurrent calls on one plan from
 *     several streams are allowed (scratch is stream-ordered per call).
 */
#ifndef TILU_H
#define TILU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TILU_OK 0
#define TILU_EINVAL 1       /* bad argument / shape (reference: ValueError) */
#define TILU_ECUDA 2        /* CUDA launch or runtime failure */
#define TILU_ENOMEM 3       /* device allocation failed */
#define TILU_EUNSUPPORTED 4 /* configuration outside the compiled kernels (e.g. kx+1 > 9) */
#define TILU_EPIVOT 5       /* zero pivot in the factorization (reference: PivotBreakdown) */

/* plan flags */
#define TILU_VARIANT_V1 1 /* boundary-band rows from the exact factor store (surrogate.py:258, use_store) */
#define TILU_VARIANT_V2 2 /* surrogate everywhere, boundary-pointing entries vanish */
#define TILU_FAST 0x1     /* fused (FMA) substitution + residual: <= 1e-12 rel. vs the reference,
                             not bitwise.  Default: exact reference operation order. */
#define TILU_SCHED_SIMPLE 0x2 /* force the reference-layout wavefront kernels (no plane layout) */
#define TILU_SCHED_PLANE 0x4  /* single tets: plane-layout band kernels at every level >= 3 (default: >= 5) */
#define TILU_SCHED_BATCH 0x8  /* single tets: never the plane kernels (interleaved dataflow kernels instead) */

typedef struct tilu_plan tilu_plan_t;

/* Everything a reference SurrogateILU (surrogate.py:232-263) + its cell operator hold. */
typedef struct {
    int level;                  /* refinement level L, 2 <= L <= 10 */
    int kx1, ky1, kz1;          /* coefficient extents = effective degrees + 1; 1 <= kx1 <= 9 */
    int variant;                /* TILU_VARIANT_V1 or TILU_VARIANT_V2 */
    const double *lcoefs;       /* [7][kx1][ky1][kz1]  SurrogateILU._lcoefs (surrogate.py:250-251) */
    const double *dcoefs;       /* [kx1][ky1][kz1]     SurrogateILU._dcoefs (surrogate.py:252) */
    const int64_t *band_ranks;  /* [nband] sorted      SurrogateILU._band_ranks (V1; may be NULL for V2) */
    int64_t nband;
    const double *store_rows;   /* [nband][9]          SurrogateILU._store_rows (V1) */
    const double *arow;         /* [15] constant operator stencil (StencilSource.data, assembly.py:173-206),
                                   or NULL when arows_dev / acoefs is given */
    const double *arows_dev;    /* DEVICE [grid][15] per-point stencil rows (assembly.py:208-221), or NULL */
    const double *acoefs;       /* [15][akx1][aky1][akz1] SurrogateOperator._acoefs (surrogate.py:344-358),
                                   or NULL: residual from arow / arows_dev */
    int akx1, aky1, akz1;
    const double *factors;      /* [grid][9] CellILU rows (ilu.py:210-227) for the stored-factor sweep,
                                   or NULL */
    int flags;                  /* TILU_FAST | TILU_SCHED_SIMPLE */
    /* Separable scalar coefficient on the unit macro-tet (config 3), rows evaluated on the fly
       instead of read (takes precedence over arow / arows_dev): HOST [3][4n+1] tables
       c1*gx(c/4n), gy(c/4n), gz(c/4n); k = c0 + (hx*gy)*gz; W = n^2 |micro-tet| (stencil.py SeparableK).
       NULL: not used. */
    const double *sepk_tables;
    double sepk_c0, sepk_w;
    const double *factors_dev;  /* DEVICE [grid][9] CellILU rows, e.g. written by tilu_factorize_device (used
                                   when `factors` is NULL; caller-owned, must outlive the plan), or NULL */
} tilu_desc_t;

/* Build a device plan: uploads coefficients, band rows and stencil, precomputes the
 * per-row forward-difference seed tables.  Replaces SurrogateILU.__init__
 * (surrogate.py:235-252) + CellILU.__init__ (ilu.py:216-223) on the device side. */
int tilu_plan_create(const tilu_desc_t *desc, tilu_plan_t **out);
void tilu_plan_destroy(tilu_plan_t *plan);

/* In place w <- (L D L^T)^{-1} w on ntets vectors sharing the plan.
 * Replaces SurrogateILU.solve_into (surrogate.py:258-263) =
 * _kernels.surrogate_forward (_kernels.py:323-367) + surrogate_backward (:370-431). */
int tilu_solve_into(const tilu_plan_t *plan, double *w, int ntets, void *stream);

/* Forward (L) or backward (D^-1, L^T) half of solve_into alone.
 * Replaces _kernels.surrogate_forward / surrogate_backward. */
int tilu_surrogate_forward(const tilu_plan_t *plan, double *w, int ntets, void *stream);
int tilu_surrogate_backward(const tilu_plan_t *plan, double *w, int ntets, void *stream);

/* w = f - A u on interior rows, 0 elsewhere; optional rnorm2 (DEVICE, [ntets]) = ||w||^2.
 * Replaces Hierarchy._cell_stage's residual (multigrid.py:420-427) in stencil form
 * (_kernels.stencil_apply, _kernels.py:243-267) or SurrogateOperator.residual_into
 * (surrogate.py:356-358 -> _kernels.surrogate_apply_residual, _kernels.py:444-483). */
int tilu_residual(const tilu_plan_t *plan, const double *u, const double *f, double *w, int ntets,
                  double *rnorm2, void *stream);

/* out = A u on interior rows (_kernels.stencil_apply, _kernels.py:243-267). */
int tilu_stencil_apply(const tilu_plan_t *plan, const double *u, double *out, int ntets, void *stream);

/* `sweeps` smoothing steps u <- u + (L D L^T)^{-1}(f - A u) on every tet of the batch,
 * i.e. `sweeps` calls of the single-tet all-Dirichlet cell stage (multigrid.py:414-429 via
 * Hierarchy.smooth, :431-442).  u is updated in place; boundary entries are never written.
 * rnorm2 (DEVICE, [sweeps][ntets], may be NULL) receives ||f - A u||^2 before each sweep.
 * Kernels: one tet from level 5 up -> plane-layout band kernels (the plan keeps a plane workspace of
 * four vectors between calls; calls from several streams are serialised on it); several tets ->
 * interleaved dataflow kernels; otherwise the reference-layout kernels.  All bitwise equal in exact
 * mode. */
int tilu_sweep(const tilu_plan_t *plan, double *u, const double *f, int ntets, int sweeps,
               double *rnorm2, void *stream);

/* Packed (interleaved) layout for batches of macro-tets sharing one plan: groups of GW = 32 * T
 * tets (T = 2 for ntets > 32, else 1), group g = fp64 [grid][GW] (tet-minor), i.e. one lattice
 * point of a group is 256 / 512 contiguous bytes.  tilu_packed_size() = doubles of a packed vector
 * for ntets; tilu_pack/unpack convert from/to the reference layout [ntets][grid] (padding tets are
 * zero).  tilu_sweep_packed() runs `sweeps` fused sweeps on packed u, f with caller-owned scratch
 * w_p of tilu_packed_scratch_size() doubles, zero-initialised before its first use (it keeps its
 * own state across calls: a header plus the two work vectors; reuse it only with the same plan and
 * ntets, or zero it again).  tilu_sweep() uses this path internally for ntets >= 2; single tets from
 * level 5 up run on the plane-layout band kernels (see TILU_SCHED_PLANE / TILU_SCHED_BATCH). */
int64_t tilu_packed_size(const tilu_plan_t *plan, int ntets);
int64_t tilu_packed_scratch_size(const tilu_plan_t *plan, int ntets);
int tilu_pack(const tilu_plan_t *plan, const double *src, double *dst, int ntets, void *stream);
int tilu_unpack(const tilu_plan_t *plan, const double *src, double *dst, int ntets, void *stream);
int tilu_sweep_packed(const tilu_plan_t *plan, double *u_p, const double *f_p, double *w_p, int ntets, int sweeps,
                      double *rnorm2, void *stream);

/* Stored-factor comparison (plan built with desc.factors): CellILU.solve_into (ilu.py:225-227)
 * = _kernels.ilu_forward (_kernels.py:150-166) + ilu_backward (:169-192), and the sweep. */
int tilu_stored_solve_into(const tilu_plan_t *plan, double *w, int ntets, void *stream);
int tilu_stored_sweep(const tilu_plan_t *plan, double *u, const double *f, int ntets, int sweeps,
                      double *rnorm2, void *stream);

/* Host-side setup kernel: streaming two-layer LDL^T ILU(0) factorization.
 * Replaces _kernels.factorize_stream (_kernels.py:39-143), same arguments:
 * rowoff [(n+1)*(n+1)], arows [1][15] (aconst) or [grid][15], full_store [grid][9] (if do_full),
 * collect_ranks [ncollect] sorted, collect_out [ncollect][9].  Returns 0 or 1 + rank of the
 * first vanishing pivot.  HOST pointers; runs on the calling CPU thread. */
int64_t tilu_factorize_stream(int n, const int64_t *rowoff, const double *arows, int aconst,
                              double *full_store, int do_full, const int64_t *collect_ranks,
                              int64_t ncollect, double *collect_out, double pivot_eps);

/* On-device streaming factorization: the same factorization as tilu_factorize_stream
 * (_kernels.factorize_stream, _kernels.py:39-143; factorize_tet ilu.py:139-175 with full_store=True),
 * computed by a hyperplane-wavefront kernel, bitwise equal to the host routine.  Exactly one operator
 * source: arows_dev (DEVICE [grid][15] per-point rows), arow (HOST [15] constant row) or
 * sepk_tables_dev (DEVICE [3][4n+1], config 3's separable coefficient evaluated on the fly).
 * store_dev: DEVICE [grid][9] factor rows (L_w..L_be, D, 1/D; ilu.py:32), interior rows written, the
 * rest untouched.  *status_host = 0, or 1 + rank of the first vanishing pivot (|D| < pivot_eps; the
 * call then returns TILU_EPIVOT).  Synchronises `stream` before returning. */
int tilu_factorize_device(int level, const double *arows_dev, const double *arow, const double *sepk_tables_dev,
                          double sepk_c0, double sepk_w, double *store_dev, double pivot_eps,
                          int64_t *status_host, void *stream);
/* out_dev[i][0..8] = store_dev[ranks_dev[i]][0..8]: the sampled / band rows the fit and the V1 store
 * take from the factorization (factorize_stream's collect_ranks / collect_out).  DEVICE pointers. */
int tilu_gather_rows(const double *store_dev, const int64_t *ranks_dev, int64_t count, double *out_dev,
                     void *stream);

/* Multigrid transfers on one macro-tet lattice, vectors in the reference layout, DEVICE:
 * r_coarse = P^T r_fine on interior coarse points, 0 elsewhere (Hierarchy.restrict / v_cycle,
 * multigrid.py:383-388, 476-480; P = build_prolongation, multigrid.py:241-277; the fine level is
 * coarse_level + 1, r_fine zero outside its interior); u_fine += P e_coarse on interior fine points
 * (multigrid.py:482); y = M x for the coarsest-level inverse (Hierarchy.coarse_solve, :445-457). */
int tilu_mg_restrict(int coarse_level, const double *r_fine, double *r_coarse, void *stream);
int tilu_mg_prolong_add(int coarse_level, const double *e_coarse, double *u_fine, void *stream);
int tilu_dense_mv(int m, const double *M, const double *x, double *y, void *stream);

/* Interface stages of the hybrid multi-tet smoother (Hierarchy._interface_stage,
 * multigrid.py:400-412).  DEVICE pointers unless stated.
 * tilu_csr_residual_rows: r[i] = f[ids[i]] - sum_k data[k] u[indices[k]] over row i of a CSR row subset
 *   (the rows `ids` of the global matrix, global column indices), in scipy's csr_matvec order.
 * tilu_csr_tri_solve_blocks: nblocks independent CSR blocks stored back to back (rows roff[b]..roff[b+1]-1,
 *   block-local int32 column indices): z = (lower | upper triangle incl. diagonal)^{-1} b per block
 *   (_kernels.csr_lower_solve / csr_upper_solve, _kernels.py:490-519), then u[ids[row]] += z[row].  The
 *   schedule (loff [nblocks+1] -> lptr [nlevels_total+1] -> perm, block-local rows grouped by dependency
 *   level) comes from tilu_csr_levels (HOST pointers; returns the level count of one block, -1 on a bad
 *   argument).
 * tilu_csr_matvec: y = M x or y += M x (accumulate) for a CSR matrix in scipy's csr_matvec order -- the
 *   transfers P e and P^T r (P^T passed as CSR) of a macro-mesh hierarchy (multigrid.py:377-388). */
int tilu_csr_matvec(int64_t nrows, const int64_t *indptr, const int64_t *indices, const double *data,
                    const double *x, double *y, int accumulate, void *stream);
int tilu_csr_levels(int m, const int64_t *indptr, const int *indices, int upper, int *level);
int tilu_csr_residual_rows(int64_t nrows, const int64_t *indptr, const int64_t *indices, const double *data,
                           const int64_t *ids, const double *u, const double *f, double *r, void *stream);
int tilu_csr_tri_solve_blocks(int nblocks, const int64_t *roff, const int64_t *indptr, const int *indices,
                              const double *data, const int64_t *loff, const int64_t *lptr, const int *perm,
                              int upper, const double *b, double *z, const int64_t *ids, double *u, void *stream);

/* Host-side setup: rows [grid][15] (interior rows written, others untouched) of a separable scalar
 * coefficient on the unit macro-tet from its [3][4n+1] tables -- bitwise the reference's per-point
 * assembly stencil_source (assembly.py:208-221) for that coefficient.  HOST pointers. */
int tilu_sepk_rows(int level, const double *tables, double c0, double w, double *rows);

/* Introspection. */
const char *tilu_last_error(void);
int tilu_version(void);
/* Number of kernels the last compute call on this thread enqueued (bench accounting). */
int tilu_last_launch_count(void);
/* Per-kernel device timing for benchmarks: while enabled, every kernel the library launches is
 * bracketed by CUDA events on its stream.  tilu_profile_read() synchronises the recorded events
 * and returns, for up to `cap` kernel families, the name, launch count and summed milliseconds;
 * it returns the number of families.  tilu_profile_reset() clears the table. */
void tilu_profile_enable(int on);
void tilu_profile_reset(void);
int tilu_profile_read(char *names /* cap * 64 bytes */, int *counts, double *ms, int cap);

/* Band tasks of the single-tet plane kernels at a level (n = 2^level): codes (b << 16) | c for band b
 * (diagonals s = 2 + 4b .. 5 + 4b) and 32-row chunk c (rows z = 1 + 32c .. 32 + 32c), in the forward
 * pass's topological order (the backward pass takes them reversed).  Writes up to cap codes and
 * returns the task count (introspection and tests; no device work). */
int tilu_plane_tasks(int level, int *out, int cap);

/* Plan geometry: grid size and interior DoF count. */
int64_t tilu_plan_grid_size(const tilu_plan_t *plan);
int64_t tilu_plan_interior_size(const tilu_plan_t *plan);

#ifdef __cplusplus
}
#endif
#endif /* TILU_H */
