// Reference-layout kernels ("simple" schedule): setup-time seed tables, the residual /
// stencil-apply kernels, and hyperplane-wavefront triangular sweeps that work directly on
// the reference's full-lattice vectors.
//
// Wavefront schedule: t = x + 2y + 3z is the minimal hyperplane satisfying all seven lower
// offsets; a row (z, y) is live for xe consecutive steps, one thread owns it and
// keeps its forward-difference table in registers, so the per-row seeding and march order of
// the reference (_kernels.py:323-431) are reproduced exactly and the result is bitwise equal
// to the serial lexicographic sweep.  One CTA per macro-tet, one __syncthreads() per step.
// These kernels are the drop-in path for solve_into on reference-layout vectors and the
// fallback for shapes the plane-layout fast path does not cover.
#include "tilu_common.cuh"
#include "tilu_plan.cuh"
#include "tilu_sepk_dev.cuh"

namespace tilu {

// ----------------------------------------------------------------------------------------------
// Seed tables: per row, the forward-difference table each marcher starts from.
// Forward: 7 L polynomials at (x0=1, step=+1).  Backward: the 7 L polynomials on the
// direction-shifted rows (q = p - d_m) at (x0 = xe - DX[m], step = -1), plus 1/D at (xe, -1).
// (_kernels.py:331-342 and :381-395.)
// ----------------------------------------------------------------------------------------------
__global__ void k_seed(PlanDev P, const double *__restrict__ lcoefs, const double *__restrict__ dcoefs,
                       double *__restrict__ seedF, double *__restrict__ seedB)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int slot = blockIdx.y;  // 0..6 fwd L, 7..13 bwd L, 14 bwd D
    if (r >= P.nrows) return;
    const RowInfo ri = P.rows[r];
    const int K = P.kx1;
    const int cnt = K < ri.xe ? K : ri.xe;
    double ax[16], tab[16];
    if (slot < 7) {
        collapse_zy(lcoefs, slot, K, P.ky1, P.kz1, dmul((double)ri.z, P.h), dmul((double)ri.y, P.h), ax);
        seed_table(ax, K, 1, 1, P.h, cnt, tab);
        double *o = seedF + ((int64_t)r * 7 + slot) * K;
        for (int j = 0; j < K; ++j) o[j] = tab[j];
    } else if (slot < 14) {
        const int m = slot - 7;
        collapse_zy(lcoefs, m, K, P.ky1, P.kz1, dmul((double)(ri.z - kDZ[m]), P.h),
                    dmul((double)(ri.y - kDY[m]), P.h), ax);
        seed_table(ax, K, ri.xe - kDX[m], -1, P.h, cnt, tab);
        double *o = seedB + ((int64_t)r * 8 + m) * K;
        for (int j = 0; j < K; ++j) o[j] = tab[j];
    } else {
        collapse_zy(dcoefs, 0, K, P.ky1, P.kz1, dmul((double)ri.z, P.h), dmul((double)ri.y, P.h), ax);
        seed_table(ax, K, ri.xe, -1, P.h, cnt, tab);
        double *o = seedB + ((int64_t)r * 8 + 7) * K;
        for (int j = 0; j < K; ++j) o[j] = tab[j];
    }
}

// Operator surrogate seeds (15 marchers, x0 = 1, step = +1; _kernels.py:453-465).
__global__ void k_seed_op(PlanDev P, const double *__restrict__ acoefs, int ky1, int kz1,
                          double *__restrict__ seedA)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = blockIdx.y;
    if (r >= P.nrows) return;
    const RowInfo ri = P.rows[r];
    const int K = P.akx1;
    const int cnt = K < ri.xe ? K : ri.xe;
    double ax[16], tab[16];
    collapse_zy(acoefs, m, K, ky1, kz1, dmul((double)ri.z, P.h), dmul((double)ri.y, P.h), ax);
    seed_table(ax, K, 1, 1, P.h, cnt, tab);
    double *o = seedA + ((int64_t)r * 15 + m) * K;
    for (int j = 0; j < K; ++j) o[j] = tab[j];
}

// ----------------------------------------------------------------------------------------------
// Residual w = f - A u on interior rows (stencil_apply order, _kernels.py:243-267, then
// w[interior] = f - out as in multigrid.py:420-427).  One CTA per (row, tet); per-row sum of
// squares into part[tet][row] for a deterministic norm.
// ----------------------------------------------------------------------------------------------
// AMODE: 0 = per-point rows, 1 = constant row, 2 = separable coefficient rows evaluated on the fly.
template <bool EXACT, int AMODE, bool APPLY_ONLY>
__global__ void __launch_bounds__(128) k_residual(PlanDev P, const double *__restrict__ uall,
                                                  const double *__restrict__ fall, double *__restrict__ wall,
                                                  double *__restrict__ part)
{
    const int r = blockIdx.x;
    const int tet = blockIdx.y;
    const double *u = uall + (int64_t)tet * P.grid;
    const double *f = fall ? fall + (int64_t)tet * P.grid : nullptr;
    double *w = wall + (int64_t)tet * P.grid;
    const RowInfo ri = P.rows[r];
    const int n = P.n, z = ri.z, y = ri.y;
    const int64_t base = P.rowbase[r];
    const int64_t rs = row_offset(n, z, y - 1), rn = row_offset(n, z, y + 1);
    const int64_t rbn = row_offset(n, z - 1, y + 1), rbc = row_offset(n, z - 1, y);
    const int64_t rts = row_offset(n, z + 1, y - 1), rtc = row_offset(n, z + 1, y);
    double ss = 0.0;
    for (int x = 1 + threadIdx.x; x <= ri.xe; x += blockDim.x) {
        const int64_t p = base + x;
        TILU_CHECK(p >= 0 && p < P.grid && rs + x + 1 < P.grid && rtc + x < P.grid, "residual point", p, P.grid);
        double sa[15];
        if (AMODE == 2) sepk_point(P, x, y, z, sa);
        const double *a = AMODE == 2 ? sa : AMODE == 1 ? P.arow : P.arows + 15 * p;
        double acc = EXACT ? dmul(a[7], u[p]) : a[7] * u[p];
        acc = madd<EXACT>(acc, a[0], u[p - 1]);
        acc = madd<EXACT>(acc, a[1], u[rs + x]);
        acc = madd<EXACT>(acc, a[2], u[rs + x + 1]);
        acc = madd<EXACT>(acc, a[3], u[rbn + x - 1]);
        acc = madd<EXACT>(acc, a[4], u[rbn + x]);
        acc = madd<EXACT>(acc, a[5], u[rbc + x]);
        acc = madd<EXACT>(acc, a[6], u[rbc + x + 1]);
        acc = madd<EXACT>(acc, a[8], u[p + 1]);
        acc = madd<EXACT>(acc, a[9], u[rn + x]);
        acc = madd<EXACT>(acc, a[10], u[rn + x - 1]);
        acc = madd<EXACT>(acc, a[11], u[rts + x + 1]);
        acc = madd<EXACT>(acc, a[12], u[rts + x]);
        acc = madd<EXACT>(acc, a[13], u[rtc + x]);
        acc = madd<EXACT>(acc, a[14], u[rtc + x - 1]);
        if (APPLY_ONLY) {
            w[p] = acc;
        } else {
            const double v = dsub(f[p], acc);
            w[p] = v;
            ss = fma(v, v, ss);
        }
    }
    if (part) {
        __shared__ double red[128];
        red[threadIdx.x] = ss;
        __syncthreads();
        for (int s = 64; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) part[(int64_t)tet * P.nrows + r] = red[0];
    }
}

// Operator-surrogate residual (_kernels.py:444-483): w = f - A u with all 15 stencil weights
// marched along x.  One thread per (row, tet); the row is sequential because of the march.
template <int K>
__global__ void __launch_bounds__(128) k_residual_sop(PlanDev P, const double *__restrict__ uall,
                                                      const double *__restrict__ fall, double *__restrict__ wall,
                                                      double *__restrict__ part)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int tet = blockIdx.y;
    if (r >= P.nrows) return;
    const double *u = uall + (int64_t)tet * P.grid;
    const double *f = fall + (int64_t)tet * P.grid;
    double *w = wall + (int64_t)tet * P.grid;
    const RowInfo ri = P.rows[r];
    const int n = P.n, z = ri.z, y = ri.y;
    const int64_t base = P.rowbase[r];
    const int64_t rs = row_offset(n, z, y - 1), rn = row_offset(n, z, y + 1);
    const int64_t rbn = row_offset(n, z - 1, y + 1), rbc = row_offset(n, z - 1, y);
    const int64_t rts = row_offset(n, z + 1, y - 1), rtc = row_offset(n, z + 1, y);
    double d[15][K];
    const double *s = P.seedA + (int64_t)r * 15 * K;
#pragma unroll
    for (int m = 0; m < 15; ++m)
#pragma unroll
        for (int j = 0; j < K; ++j) d[m][j] = s[m * K + j];
    double ss = 0.0;
    for (int x = 1; x <= ri.xe; ++x) {
        const int64_t p = base + x;
        double acc = dsub(f[p], dmul(d[7][0], u[p]));
        acc = dsub(acc, dmul(d[0][0], u[p - 1]));
        acc = dsub(acc, dmul(d[1][0], u[rs + x]));
        acc = dsub(acc, dmul(d[2][0], u[rs + x + 1]));
        acc = dsub(acc, dmul(d[3][0], u[rbn + x - 1]));
        acc = dsub(acc, dmul(d[4][0], u[rbn + x]));
        acc = dsub(acc, dmul(d[5][0], u[rbc + x]));
        acc = dsub(acc, dmul(d[6][0], u[rbc + x + 1]));
        acc = dsub(acc, dmul(d[8][0], u[p + 1]));
        acc = dsub(acc, dmul(d[9][0], u[rn + x]));
        acc = dsub(acc, dmul(d[10][0], u[rn + x - 1]));
        acc = dsub(acc, dmul(d[11][0], u[rts + x + 1]));
        acc = dsub(acc, dmul(d[12][0], u[rts + x]));
        acc = dsub(acc, dmul(d[13][0], u[rtc + x]));
        acc = dsub(acc, dmul(d[14][0], u[rtc + x - 1]));
        w[p] = acc;
        ss = fma(acc, acc, ss);
#pragma unroll
        for (int m = 0; m < 15; ++m) march<K>(d[m]);
    }
    if (part) part[(int64_t)tet * P.nrows + r] = ss;
}

// Deterministic per-tet sum of the per-row partials: out[tet] = sum_r part[tet][r].
__global__ void __launch_bounds__(256) k_reduce_rows(const double *__restrict__ part, int nrows,
                                                     double *__restrict__ out)
{
    const int tet = blockIdx.x;
    double s = 0.0;
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) s += part[(int64_t)tet * nrows + r];
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[tet] = red[0];
}

// ----------------------------------------------------------------------------------------------
// Band-store index of interior point (x, y, z) (V1).  Band = x|y|z == 1 or x+y+z == n-1
// (surrogate.py:223-229); within a row the band points are ordered by x, so the reference's
// binary search (_kernels.py:27-36) becomes bandoff[row] + offset.
// ----------------------------------------------------------------------------------------------
__device__ __forceinline__ bool in_band(int x, int y, int z, int xe) { return z == 1 || y == 1 || x == 1 || x == xe; }
__device__ __forceinline__ int band_index(const PlanDev &P, int row, int x, int y, int z, int xe)
{
    return P.bandoff[row] + ((z == 1 || y == 1) ? x - 1 : (x == 1 ? 0 : 1));
}

// ----------------------------------------------------------------------------------------------
// Forward substitution (unit lower L), wavefront over t = x + 2y + 3z ascending.
// state: [ntets][nrows][7][K] per-row difference tables kept across steps.
// ----------------------------------------------------------------------------------------------
template <int K, bool EXACT, bool STORED>
__global__ void __launch_bounds__(256) k_fwd_simple(PlanDev P, double *__restrict__ wall, double *__restrict__ stall)
{
    const int tet = blockIdx.x;
    double *w = wall + (int64_t)tet * P.grid;
    double *st = STORED ? nullptr : stall + (int64_t)tet * P.nrows * 7 * K;
    const int n = P.n;
    for (int t = P.tmin; t <= P.tmax; ++t) {
        for (int r = threadIdx.x; r < P.nrows; r += blockDim.x) {
            const RowInfo ri = P.rows[r];
            const int x = t - ri.t0 + 1;
            if (x < 1 || x > ri.xe) continue;
            const int z = ri.z, y = ri.y;
            const int64_t p = P.rowbase[r] + x;
            const int64_t rs = row_offset(n, z, y - 1), rb = row_offset(n, z - 1, y + 1), rc = row_offset(n, z - 1, y);
            const double wn[7] = {w[p - 1], w[rs + x], w[rs + x + 1], w[rb + x - 1], w[rb + x], w[rc + x], w[rc + x + 1]};
            double L[7];
            double d[7][K];
            if (STORED) {
#pragma unroll
                for (int m = 0; m < 7; ++m) L[m] = P.factors[9 * p + m];
            } else {
                const double *src = (x == 1) ? P.seedF + (int64_t)r * 7 * K : st + (int64_t)r * 7 * K;
#pragma unroll
                for (int m = 0; m < 7; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = src[m * K + j];
                if (P.variant == 1 && in_band(x, y, z, ri.xe)) {
                    const double *s = P.store + 9 * (int64_t)band_index(P, r, x, y, z, ri.xe);
#pragma unroll
                    for (int m = 0; m < 7; ++m) L[m] = s[m];
                } else {
#pragma unroll
                    for (int m = 0; m < 7; ++m) L[m] = d[m][0];
                }
            }
            double acc = w[p];
#pragma unroll
            for (int m = 0; m < 7; ++m) acc = msub<EXACT>(acc, L[m], wn[m]);
            w[p] = acc;
            if (!STORED) {
                double *dst = st + (int64_t)r * 7 * K;
#pragma unroll
                for (int m = 0; m < 7; ++m) {
                    march<K>(d[m]);
#pragma unroll
                    for (int j = 0; j < K; ++j) dst[m * K + j] = d[m][j];
                }
            }
        }
        __syncthreads();
    }
}

// L value of direction m at the shifted source point q (_kernels.py:434-441 _lq).
__device__ __forceinline__ double lq_value(const PlanDev &P, int m, int qx, int qy, int qz, double dval)
{
    const int n = P.n;
    if (!interior(qx, qy, qz, n)) return 0.0;
    if (P.variant == 1) {
        const int xe = n - 1 - qz - qy;
        if (in_band(qx, qy, qz, xe)) return P.store[9 * (int64_t)band_index(P, row_id(n, qz, qy), qx, qy, qz, xe) + m];
    }
    return dval;
}

// Backward pass (D^{-1} scaling + L^T solve), descending t, fused with u[p] += w[p]
// (multigrid.py:429).  uall may be nullptr (plain solve_into).
template <int K, bool EXACT, bool STORED>
__global__ void __launch_bounds__(256) k_bwd_simple(PlanDev P, double *__restrict__ wall, double *__restrict__ stall,
                                                    double *__restrict__ uall)
{
    const int tet = blockIdx.x;
    double *w = wall + (int64_t)tet * P.grid;
    double *u = uall ? uall + (int64_t)tet * P.grid : nullptr;
    double *st = STORED ? nullptr : stall + (int64_t)tet * P.nrows * 8 * K;
    const int n = P.n;
    for (int t = P.tmax; t >= P.tmin; --t) {
        for (int r = threadIdx.x; r < P.nrows; r += blockDim.x) {
            const RowInfo ri = P.rows[r];
            const int x = t - ri.t0 + 1;
            if (x < 1 || x > ri.xe) continue;
            const int z = ri.z, y = ri.y;
            const int64_t p = P.rowbase[r] + x;
            const int64_t rn = row_offset(n, z, y + 1), rts = row_offset(n, z + 1, y - 1), rtc = row_offset(n, z + 1, y);
            const int64_t q[7] = {p + 1, rn + x, rn + x - 1, rts + x + 1, rts + x, rtc + x, rtc + x - 1};
            double Lq[7], inv_d;
            double d[8][K];
            if (STORED) {
                inv_d = P.factors[9 * p + 8];
#pragma unroll
                for (int m = 0; m < 7; ++m) Lq[m] = P.factors[9 * q[m] + m];
            } else {
                const double *src = (x == ri.xe) ? P.seedB + (int64_t)r * 8 * K : st + (int64_t)r * 8 * K;
#pragma unroll
                for (int m = 0; m < 8; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = src[m * K + j];
                inv_d = (P.variant == 1 && in_band(x, y, z, ri.xe))
                            ? P.store[9 * (int64_t)band_index(P, r, x, y, z, ri.xe) + 8]
                            : d[7][0];
                Lq[0] = lq_value(P, 0, x + 1, y, z, d[0][0]);
                Lq[1] = lq_value(P, 1, x, y + 1, z, d[1][0]);
                Lq[2] = lq_value(P, 2, x - 1, y + 1, z, d[2][0]);
                Lq[3] = lq_value(P, 3, x + 1, y - 1, z + 1, d[3][0]);
                Lq[4] = lq_value(P, 4, x, y - 1, z + 1, d[4][0]);
                Lq[5] = lq_value(P, 5, x, y, z + 1, d[5][0]);
                Lq[6] = lq_value(P, 6, x - 1, y, z + 1, d[6][0]);
            }
            double acc = EXACT ? dmul(inv_d, w[p]) : inv_d * w[p];
#pragma unroll
            for (int m = 0; m < 7; ++m) acc = msub<EXACT>(acc, Lq[m], w[q[m]]);
            w[p] = acc;
            if (u) u[p] = dadd(u[p], acc);
            if (!STORED) {
                double *dst = st + (int64_t)r * 8 * K;
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    march<K>(d[m]);
#pragma unroll
                    for (int j = 0; j < K; ++j) dst[m * K + j] = d[m][j];
                }
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------------------------
// Host-side launchers (called from tilu_abi.cu).
// ----------------------------------------------------------------------------------------------
void launch_seed(const PlanDev &P, const double *lcoefs, const double *dcoefs, double *seedF, double *seedB,
                 cudaStream_t s)
{
    dim3 grid((P.nrows + 127) / 128, 15);
    k_seed<<<grid, 128, 0, s>>>(P, lcoefs, dcoefs, seedF, seedB);
}

void launch_seed_op(const PlanDev &P, const double *acoefs, int ky1, int kz1, double *seedA, cudaStream_t s)
{
    dim3 grid((P.nrows + 127) / 128, 15);
    k_seed_op<<<grid, 128, 0, s>>>(P, acoefs, ky1, kz1, seedA);
}

void launch_residual(const PlanDev &P, bool exact, const double *u, const double *f, double *w, double *part,
                     int ntets, bool apply_only, cudaStream_t s)
{
    dim3 grid(P.nrows, ntets);
    const int am = P.sepk ? 2 : P.arow ? 1 : 0;
#define TILU_RES(E, M, A) k_residual<E, M, A><<<grid, 128, 0, s>>>(P, u, f, w, A ? nullptr : part)
    if (apply_only) {
        if (am == 2) TILU_RES(true, 2, true);
        else if (am == 1) TILU_RES(true, 1, true);
        else TILU_RES(true, 0, true);
    } else if (exact) {
        if (am == 2) TILU_RES(true, 2, false);
        else if (am == 1) TILU_RES(true, 1, false);
        else TILU_RES(true, 0, false);
    } else {
        if (am == 2) TILU_RES(false, 2, false);
        else if (am == 1) TILU_RES(false, 1, false);
        else TILU_RES(false, 0, false);
    }
#undef TILU_RES
}

template <int K>
static void launch_sop_k(const PlanDev &P, const double *u, const double *f, double *w, double *part, int ntets,
                         cudaStream_t s)
{
    dim3 grid((P.nrows + 127) / 128, ntets);
    k_residual_sop<K><<<grid, 128, 0, s>>>(P, u, f, w, part);
}

bool launch_residual_sop(const PlanDev &P, const double *u, const double *f, double *w, double *part, int ntets,
                         cudaStream_t s)
{
    switch (P.akx1) {
    case 1: launch_sop_k<1>(P, u, f, w, part, ntets, s); return true;
    case 2: launch_sop_k<2>(P, u, f, w, part, ntets, s); return true;
    case 3: launch_sop_k<3>(P, u, f, w, part, ntets, s); return true;
    case 4: launch_sop_k<4>(P, u, f, w, part, ntets, s); return true;
    case 5: launch_sop_k<5>(P, u, f, w, part, ntets, s); return true;
    case 6: launch_sop_k<6>(P, u, f, w, part, ntets, s); return true;
    case 7: launch_sop_k<7>(P, u, f, w, part, ntets, s); return true;
    case 8: launch_sop_k<8>(P, u, f, w, part, ntets, s); return true;
    case 9: launch_sop_k<9>(P, u, f, w, part, ntets, s); return true;
    default: return false;
    }
}

void launch_reduce_rows(const double *part, int nrows, double *out, int ntets, cudaStream_t s)
{
    k_reduce_rows<<<ntets, 256, 0, s>>>(part, nrows, out);
}

template <int K, bool EXACT, bool STORED>
static void launch_pair_k(const PlanDev &P, double *w, double *state, double *u, int ntets, int which,
                          cudaStream_t s)
{
    if (which & 1) k_fwd_simple<K, EXACT, STORED><<<ntets, 256, 0, s>>>(P, w, state);
    if (which & 2) k_bwd_simple<K, EXACT, STORED><<<ntets, 256, 0, s>>>(P, w, state, u);
}

template <bool EXACT, bool STORED>
static bool launch_pair_e(const PlanDev &P, double *w, double *state, double *u, int ntets, int which,
                          cudaStream_t s)
{
    if (STORED) { launch_pair_k<1, EXACT, true>(P, w, state, u, ntets, which, s); return true; }
    switch (P.kx1) {
    case 1: launch_pair_k<1, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    case 2: launch_pair_k<2, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    case 3: launch_pair_k<3, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    case 4: launch_pair_k<4, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    case 5: launch_pair_k<5, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    case 6: launch_pair_k<6, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    case 7: launch_pair_k<7, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    case 8: launch_pair_k<8, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    case 9: launch_pair_k<9, EXACT, STORED>(P, w, state, u, ntets, which, s); return true;
    default: return false;
    }
}

// which: 1 = forward, 2 = backward, 3 = both.  u != nullptr fuses the update into backward.
bool launch_simple_solve(const PlanDev &P, bool exact, bool stored, double *w, double *state, double *u, int ntets,
                         int which, cudaStream_t s)
{
    if (exact) return stored ? launch_pair_e<true, true>(P, w, state, u, ntets, which, s)
                             : launch_pair_e<true, false>(P, w, state, u, ntets, which, s);
    return stored ? launch_pair_e<false, true>(P, w, state, u, ntets, which, s)
                  : launch_pair_e<false, false>(P, w, state, u, ntets, which, s);
}

}  // namespace tilu
