/*
 * tilu_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, serial, fp64, no FMA contraction) of the hot path
 * of the tetilu reference (arXiv 2210.15280): the surrogate ILU(0) smoothing
 * sweep on the interior of one refined macro-tetrahedron.  It exists to check
 * the CUDA product and to time a CPU baseline; nothing in the product links or
 * calls it (only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg load it).
 *
 * Every function follows the operation order of the reference Numba kernel it
 * cites (file:line into /root/reference/pkg/src/tetilu/) so that results are
 * bit-identical; this is pinned by tests/test_oracle_golden.py against golden
 * vectors produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).
 *
 * Layout conventions (reference geometry.py:188-215): full-lattice rank of
 * (x,y,z) is rowoff[z*(n+1)+y] + x with rows ordered (z, then y, then x); all
 * vectors are zero outside the interior x,y,z>=1, x+y+z<=n-1.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXK 16 /* kx+1 <= MAXK */

/* _kernels.py:12-15: lattice displacement of the lower directions w s se bnw bn bc be */
static const int DX[7] = {-1, 0, 1, -1, 0, 0, 1};
static const int DY[7] = {0, -1, -1, 1, 1, 0, 0};
static const int DZ[7] = {0, 0, 0, -1, -1, -1, -1};

static int64_t num_points(int64_t m) { return m < 0 ? 0 : (m + 1) * (m + 2) * (m + 3) / 6; }

/* geometry.py:201-215 rank_tables: rowoff[z][y], -1 outside the lattice. */
void oracle_rank_tables(int n, int64_t *rowoff /* (n+1)*(n+1) */)
{
    int64_t tot = num_points(n);
    for (int z = 0; z <= n; ++z) {
        int64_t zoff = tot - num_points(n - z);
        for (int y = 0; y <= n; ++y)
            rowoff[(int64_t)z * (n + 1) + y] =
                (y <= n - z) ? zoff + (int64_t)y * (n - z + 1) - (int64_t)y * (y - 1) / 2 : -1;
    }
}

static inline int is_interior(int x, int y, int z, int n) /* _kernels.py:22-24 */
{
    return x >= 1 && y >= 1 && z >= 1 && x + y + z <= n - 1;
}

static inline int64_t find_rank(const int64_t *ranks, int64_t nr, int64_t v) /* _kernels.py:27-36 */
{
    int64_t lo = 0, hi = nr;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (ranks[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* NDDF helpers, _kernels.py:274-316.  coefs is [M][ni][nj][nk] C-order. */
static void collapse_z(const double *coefs, int m, int ni, int nj, int nk, double zval, double *bxy)
{
    const double *c = coefs + (int64_t)m * ni * nj * nk;
    for (int i = 0; i < ni; ++i)
        for (int j = 0; j < nj; ++j) {
            const double *cij = c + ((int64_t)i * nj + j) * nk;
            double acc = cij[nk - 1];
            for (int k = nk - 2; k >= 0; --k) acc = acc * zval + cij[k];
            bxy[i * nj + j] = acc;
        }
}

static void collapse_y(const double *bxy, int ni, int nj, double yval, double *ax)
{
    for (int i = 0; i < ni; ++i) {
        double acc = bxy[i * nj + nj - 1];
        for (int j = nj - 2; j >= 0; --j) acc = acc * yval + bxy[i * nj + j];
        ax[i] = acc;
    }
}

static double horner1(const double *ax, int ni, double xval)
{
    double acc = ax[ni - 1];
    for (int i = ni - 2; i >= 0; --i) acc = acc * xval + ax[i];
    return acc;
}

static void seed_diffs(const double *ax, int ni, int64_t x0, int step, double h, int count, double *out)
{
    for (int t = 0; t < count; ++t) out[t] = horner1(ax, ni, (double)(x0 + (int64_t)t * step) * h);
    for (int o = 1; o < count; ++o)
        for (int t = count - 1; t >= o; --t) out[t] = out[t] - out[t - 1];
}

static inline void march(double *d, int count)
{
    for (int j = 0; j < count - 1; ++j) d[j] += d[j + 1];
}

/* _kernels.py:323-367 surrogate_forward */
void oracle_surrogate_forward(int n, const int64_t *rowoff, double h, const double *lcoefs,
                              int kx1, int ky1, int kz1, double *w, int use_store,
                              const int64_t *band_ranks, int64_t nband, const double *store_rows)
{
    const int N1 = n + 1;
    double bxy[7][MAXK * MAXK], ax[7][MAXK], diffs[7][MAXK];
#define RO(z, y) rowoff[(int64_t)(z) * N1 + (y)]
    for (int z = 1; z < n - 2; ++z) {
        double zv = (double)z * h;
        for (int m = 0; m < 7; ++m) collapse_z(lcoefs, m, kx1, ky1, kz1, zv, bxy[m]);
        for (int y = 1; y < n - 1 - z; ++y) {
            double yv = (double)y * h;
            int64_t base = RO(z, y);
            int xe = n - 1 - z - y;
            int cnt = kx1 < xe ? kx1 : xe;
            for (int m = 0; m < 7; ++m) {
                collapse_y(bxy[m], kx1, ky1, yv, ax[m]);
                seed_diffs(ax[m], kx1, 1, 1, h, cnt, diffs[m]);
            }
            int band_row = (z == 1 || y == 1);
            for (int x = 1; x <= xe; ++x) {
                int64_t r = base + x;
                double acc = w[r];
                const int64_t q[7] = {r - 1, RO(z, y - 1) + x, RO(z, y - 1) + x + 1,
                                      RO(z - 1, y + 1) + x - 1, RO(z - 1, y + 1) + x,
                                      RO(z - 1, y) + x, RO(z - 1, y) + x + 1};
                if (use_store && (band_row || x == 1 || x + y + z == n - 1)) {
                    const double *s = store_rows + 9 * find_rank(band_ranks, nband, r);
                    for (int m = 0; m < 7; ++m) acc -= s[m] * w[q[m]];
                } else {
                    for (int m = 0; m < 7; ++m) acc -= diffs[m][0] * w[q[m]];
                }
                w[r] = acc;
                for (int m = 0; m < 7; ++m) march(diffs[m], cnt);
            }
        }
    }
#undef RO
}

/* _kernels.py:434-441 _lq */
static inline double lq(int m, int qx, int qy, int qz, int n, double dval, int use_store,
                        const int64_t *band_ranks, int64_t nband, const double *store_rows, int64_t q)
{
    if (!is_interior(qx, qy, qz, n)) return 0.0;
    if (use_store && (qx == 1 || qy == 1 || qz == 1 || qx + qy + qz == n - 1))
        return store_rows[9 * find_rank(band_ranks, nband, q) + m];
    return dval;
}

/* _kernels.py:370-431 surrogate_backward */
void oracle_surrogate_backward(int n, const int64_t *rowoff, double h, const double *lcoefs,
                               const double *dcoefs, int kx1, int ky1, int kz1, double *w,
                               int use_store, const int64_t *band_ranks, int64_t nband,
                               const double *store_rows)
{
    const int N1 = n + 1;
    double bxy[7][MAXK * MAXK], ax[7][MAXK], diffs[7][MAXK];
    double dbxy[MAXK * MAXK], dax[MAXK], ddiffs[MAXK];
#define RO(z, y) rowoff[(int64_t)(z) * N1 + (y)]
    for (int z = n - 3; z >= 1; --z) {
        for (int m = 0; m < 7; ++m) collapse_z(lcoefs, m, kx1, ky1, kz1, (double)(z - DZ[m]) * h, bxy[m]);
        collapse_z(dcoefs, 0, kx1, ky1, kz1, (double)z * h, dbxy);
        for (int y = n - 2 - z; y >= 1; --y) {
            int64_t base = RO(z, y);
            int xe = n - 1 - z - y;
            int cnt = kx1 < xe ? kx1 : xe;
            int dcnt = cnt;
            for (int m = 0; m < 7; ++m) {
                collapse_y(bxy[m], kx1, ky1, (double)(y - DY[m]) * h, ax[m]);
                seed_diffs(ax[m], kx1, xe - DX[m], -1, h, cnt, diffs[m]);
            }
            collapse_y(dbxy, kx1, ky1, (double)y * h, dax);
            seed_diffs(dax, kx1, xe, -1, h, dcnt, ddiffs);
            for (int x = xe; x >= 1; --x) {
                int64_t r = base + x;
                double inv_d;
                if (use_store && (z == 1 || y == 1 || x == 1 || x + y + z == n - 1))
                    inv_d = store_rows[9 * find_rank(band_ranks, nband, r) + 8];
                else
                    inv_d = ddiffs[0];
                double acc = inv_d * w[r];
                int64_t q;
                q = r + 1;
                acc -= lq(0, x + 1, y, z, n, diffs[0][0], use_store, band_ranks, nband, store_rows, q) * w[q];
                q = RO(z, y + 1) + x;
                acc -= lq(1, x, y + 1, z, n, diffs[1][0], use_store, band_ranks, nband, store_rows, q) * w[q];
                q = RO(z, y + 1) + x - 1;
                acc -= lq(2, x - 1, y + 1, z, n, diffs[2][0], use_store, band_ranks, nband, store_rows, q) * w[q];
                q = RO(z + 1, y - 1) + x + 1;
                acc -= lq(3, x + 1, y - 1, z + 1, n, diffs[3][0], use_store, band_ranks, nband, store_rows, q) * w[q];
                q = RO(z + 1, y - 1) + x;
                acc -= lq(4, x, y - 1, z + 1, n, diffs[4][0], use_store, band_ranks, nband, store_rows, q) * w[q];
                q = RO(z + 1, y) + x;
                acc -= lq(5, x, y, z + 1, n, diffs[5][0], use_store, band_ranks, nband, store_rows, q) * w[q];
                q = RO(z + 1, y) + x - 1;
                acc -= lq(6, x - 1, y, z + 1, n, diffs[6][0], use_store, band_ranks, nband, store_rows, q) * w[q];
                w[r] = acc;
                for (int m = 0; m < 7; ++m) march(diffs[m], cnt);
                march(ddiffs, dcnt);
            }
        }
    }
#undef RO
}

/* surrogate.py:258-263 SurrogateILU.solve_into */
void oracle_solve_into(int n, const int64_t *rowoff, double h, const double *lcoefs,
                       const double *dcoefs, int kx1, int ky1, int kz1, double *w, int use_store,
                       const int64_t *band_ranks, int64_t nband, const double *store_rows)
{
    oracle_surrogate_forward(n, rowoff, h, lcoefs, kx1, ky1, kz1, w, use_store, band_ranks, nband, store_rows);
    oracle_surrogate_backward(n, rowoff, h, lcoefs, dcoefs, kx1, ky1, kz1, w, use_store, band_ranks, nband,
                              store_rows);
}

/* _kernels.py:243-267 stencil_apply: out = A u on interior rows (arows [1][15] if aconst) */
void oracle_stencil_apply(int n, const int64_t *rowoff, const double *arows, int aconst,
                          const double *u, double *out)
{
    const int N1 = n + 1;
#define RO(z, y) rowoff[(int64_t)(z) * N1 + (y)]
    for (int z = 1; z < n - 2; ++z)
        for (int y = 1; y < n - 1 - z; ++y) {
            int64_t base = RO(z, y);
            for (int x = 1; x < n - z - y; ++x) {
                int64_t r = base + x;
                const double *row = aconst ? arows : arows + 15 * r;
                double acc = row[7] * u[r];
                acc += row[0] * u[r - 1];
                acc += row[1] * u[RO(z, y - 1) + x];
                acc += row[2] * u[RO(z, y - 1) + x + 1];
                acc += row[3] * u[RO(z - 1, y + 1) + x - 1];
                acc += row[4] * u[RO(z - 1, y + 1) + x];
                acc += row[5] * u[RO(z - 1, y) + x];
                acc += row[6] * u[RO(z - 1, y) + x + 1];
                acc += row[8] * u[r + 1];
                acc += row[9] * u[RO(z, y + 1) + x];
                acc += row[10] * u[RO(z, y + 1) + x - 1];
                acc += row[11] * u[RO(z + 1, y - 1) + x + 1];
                acc += row[12] * u[RO(z + 1, y - 1) + x];
                acc += row[13] * u[RO(z + 1, y) + x];
                acc += row[14] * u[RO(z + 1, y) + x - 1];
                out[r] = acc;
            }
        }
#undef RO
}

/* _kernels.py:444-483 surrogate_apply_residual: w = f - A u with 15 NDDF marchers */
void oracle_surrogate_apply_residual(int n, const int64_t *rowoff, double h, const double *acoefs,
                                     int kx1, int ky1, int kz1, const double *u, const double *f,
                                     double *w)
{
    const int N1 = n + 1;
    double (*bxy)[MAXK * MAXK] = malloc(sizeof(double) * 15 * MAXK * MAXK);
    double ax[15][MAXK], diffs[15][MAXK];
#define RO(z, y) rowoff[(int64_t)(z) * N1 + (y)]
    for (int z = 1; z < n - 2; ++z) {
        double zv = (double)z * h;
        for (int m = 0; m < 15; ++m) collapse_z(acoefs, m, kx1, ky1, kz1, zv, bxy[m]);
        for (int y = 1; y < n - 1 - z; ++y) {
            double yv = (double)y * h;
            int64_t base = RO(z, y);
            int xe = n - 1 - z - y;
            int cnt = kx1 < xe ? kx1 : xe;
            for (int m = 0; m < 15; ++m) {
                collapse_y(bxy[m], kx1, ky1, yv, ax[m]);
                seed_diffs(ax[m], kx1, 1, 1, h, cnt, diffs[m]);
            }
            for (int x = 1; x <= xe; ++x) {
                int64_t r = base + x;
                double acc = f[r] - diffs[7][0] * u[r];
                acc -= diffs[0][0] * u[r - 1];
                acc -= diffs[1][0] * u[RO(z, y - 1) + x];
                acc -= diffs[2][0] * u[RO(z, y - 1) + x + 1];
                acc -= diffs[3][0] * u[RO(z - 1, y + 1) + x - 1];
                acc -= diffs[4][0] * u[RO(z - 1, y + 1) + x];
                acc -= diffs[5][0] * u[RO(z - 1, y) + x];
                acc -= diffs[6][0] * u[RO(z - 1, y) + x + 1];
                acc -= diffs[8][0] * u[r + 1];
                acc -= diffs[9][0] * u[RO(z, y + 1) + x];
                acc -= diffs[10][0] * u[RO(z, y + 1) + x - 1];
                acc -= diffs[11][0] * u[RO(z + 1, y - 1) + x + 1];
                acc -= diffs[12][0] * u[RO(z + 1, y - 1) + x];
                acc -= diffs[13][0] * u[RO(z + 1, y) + x];
                acc -= diffs[14][0] * u[RO(z + 1, y) + x - 1];
                w[r] = acc;
                for (int m = 0; m < 15; ++m) march(diffs[m], cnt);
            }
        }
    }
#undef RO
    free(bxy);
}

/* _kernels.py:150-166 ilu_forward; factors is [grid][9] = L_w..L_be, D, 1/D */
void oracle_ilu_forward(int n, const int64_t *rowoff, const double *factors, double *w)
{
    const int N1 = n + 1;
#define RO(z, y) rowoff[(int64_t)(z) * N1 + (y)]
    for (int z = 1; z < n - 2; ++z)
        for (int y = 1; y < n - 1 - z; ++y) {
            int64_t base = RO(z, y);
            for (int x = 1; x < n - z - y; ++x) {
                int64_t r = base + x;
                const double *F = factors + 9 * r;
                double acc = w[r];
                acc -= F[0] * w[r - 1];
                acc -= F[1] * w[RO(z, y - 1) + x];
                acc -= F[2] * w[RO(z, y - 1) + x + 1];
                acc -= F[3] * w[RO(z - 1, y + 1) + x - 1];
                acc -= F[4] * w[RO(z - 1, y + 1) + x];
                acc -= F[5] * w[RO(z - 1, y) + x];
                acc -= F[6] * w[RO(z - 1, y) + x + 1];
                w[r] = acc;
            }
        }
#undef RO
}

/* _kernels.py:169-192 ilu_backward */
void oracle_ilu_backward(int n, const int64_t *rowoff, const double *factors, double *w)
{
    const int N1 = n + 1;
#define RO(z, y) rowoff[(int64_t)(z) * N1 + (y)]
    for (int z = n - 3; z >= 1; --z)
        for (int y = n - 2 - z; y >= 1; --y) {
            int64_t base = RO(z, y);
            for (int x = n - 1 - z - y; x >= 1; --x) {
                int64_t r = base + x, q;
                double acc = factors[9 * r + 8] * w[r];
                q = r + 1;                       acc -= factors[9 * q + 0] * w[q];
                q = RO(z, y + 1) + x;            acc -= factors[9 * q + 1] * w[q];
                q = RO(z, y + 1) + x - 1;        acc -= factors[9 * q + 2] * w[q];
                q = RO(z + 1, y - 1) + x + 1;    acc -= factors[9 * q + 3] * w[q];
                q = RO(z + 1, y - 1) + x;        acc -= factors[9 * q + 4] * w[q];
                q = RO(z + 1, y) + x;            acc -= factors[9 * q + 5] * w[q];
                q = RO(z + 1, y) + x - 1;        acc -= factors[9 * q + 6] * w[q];
                w[r] = acc;
            }
        }
#undef RO
}

/* ------------------------------------------------------------------------ */
/* Sweep drivers: one smoothing step of the single-tet, all-Dirichlet cell    */
/* stage (multigrid.py:414-429) in its stencil form: r = A u (stencil_apply),  */
/* w[interior] = f - r, solve_into(w), u[interior] += w.                       */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n;
    double h;
    const int64_t *rowoff;
    const double *lcoefs, *dcoefs;
    int kx1, ky1, kz1;
    int use_store;
    const int64_t *band_ranks;
    int64_t nband;
    const double *store_rows;
    const double *arows;
    int aconst;
    const double *acoefs; /* non-NULL: surrogate-A residual (a_mode='surrogate') */
    int akx1, aky1, akz1;
    const double *factors; /* non-NULL: stored-factor CellILU sweep instead of surrogate */
} oracle_cell_t;

static void sweep_one(const oracle_cell_t *c, double *u, const double *f, double *w, double *tmp,
                      int64_t grid, double *rnorm2)
{
    int n = c->n;
    const int N1 = n + 1;
    memset(w, 0, sizeof(double) * grid);
    if (c->acoefs) {
        oracle_surrogate_apply_residual(n, c->rowoff, c->h, c->acoefs, c->akx1, c->aky1, c->akz1, u, f, w);
    } else {
        oracle_stencil_apply(n, c->rowoff, c->arows, c->aconst, u, tmp);
        for (int z = 1; z < n - 2; ++z)
            for (int y = 1; y < n - 1 - z; ++y) {
                int64_t base = c->rowoff[(int64_t)z * N1 + y];
                for (int x = 1; x < n - z - y; ++x) w[base + x] = f[base + x] - tmp[base + x];
            }
    }
    if (rnorm2) {
        double s = 0.0;
        for (int64_t i = 0; i < grid; ++i) s += w[i] * w[i];
        *rnorm2 = s;
    }
    if (c->factors) {
        oracle_ilu_forward(n, c->rowoff, c->factors, w);
        oracle_ilu_backward(n, c->rowoff, c->factors, w);
    } else {
        oracle_solve_into(n, c->rowoff, c->h, c->lcoefs, c->dcoefs, c->kx1, c->ky1, c->kz1, w, c->use_store,
                          c->band_ranks, c->nband, c->store_rows);
    }
    for (int z = 1; z < n - 2; ++z)
        for (int y = 1; y < n - 1 - z; ++y) {
            int64_t base = c->rowoff[(int64_t)z * N1 + y];
            for (int x = 1; x < n - z - y; ++x) u[base + x] += w[base + x];
        }
}

/* `sweeps` smoothing steps on one tet; rnorm2 (optional, length sweeps) gets ||f - A u||^2 before each. */
int oracle_sweeps(int n, double h, const int64_t *rowoff, const double *lcoefs, const double *dcoefs,
                  int kx1, int ky1, int kz1, int use_store, const int64_t *band_ranks, int64_t nband,
                  const double *store_rows, const double *arows, int aconst, const double *acoefs,
                  int akx1, int aky1, int akz1, const double *factors, double *u, const double *f,
                  int sweeps, double *rnorm2)
{
    oracle_cell_t c = {n, h, rowoff, lcoefs, dcoefs, kx1, ky1, kz1, use_store, band_ranks, nband,
                       store_rows, arows, aconst, acoefs, akx1, aky1, akz1, factors};
    int64_t grid = num_points(n);
    double *w = malloc(sizeof(double) * grid), *tmp = calloc(grid, sizeof(double));
    if (!w || !tmp) { free(w); free(tmp); return 1; }
    for (int s = 0; s < sweeps; ++s) sweep_one(&c, u, f, w, tmp, grid, rnorm2 ? rnorm2 + s : NULL);
    free(w);
    free(tmp);
    return 0;
}

/* Independent macro-tets sharing one surrogate (config 4): u, f are [ntets][grid]; one
 * OpenMP thread per tet (the reference runs one serial Numba call per tet).  Returns the
 * thread count used. */
int oracle_sweeps_many(int n, double h, const int64_t *rowoff, const double *lcoefs,
                       const double *dcoefs, int kx1, int ky1, int kz1, int use_store,
                       const int64_t *band_ranks, int64_t nband, const double *store_rows,
                       const double *arows, int aconst, double *u, const double *f, int ntets,
                       int sweeps, int nthreads)
{
    int64_t grid = num_points(n);
    int used = 1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
    {
#pragma omp single
        used = omp_get_num_threads();
    }
#endif
    int err = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err)
    for (int t = 0; t < ntets; ++t)
        err |= oracle_sweeps(n, h, rowoff, lcoefs, dcoefs, kx1, ky1, kz1, use_store, band_ranks, nband,
                             store_rows, arows, aconst, NULL, 0, 0, 0, NULL, u + (int64_t)t * grid,
                             f + (int64_t)t * grid, sweeps, NULL);
    return err ? -1 : used;
}
