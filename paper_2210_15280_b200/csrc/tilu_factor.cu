// On-device streaming LDL^T ILU(0) factorization of one macro-tet interior (replaces the
// reference's _kernels.factorize_stream, _kernels.py:39-143, whose host restatement is
// tilu_factorize.cpp) and the gather of the sampled / band factor rows.
//
// The eight stencil equations of a point read the factor rows of its seven lower neighbours
// (w s se in the same z-layer, bnw bn bc be in the layer below), i.e. the dependency pattern of the
// forward substitution, so the hyperplanes t = x + 2y + 3z are independent sets.  One
// persistent, co-resident grid (cooperative launch) walks the hyperplanes with a grid barrier between
// them: a thread owns lattice rows (z, y) and at step t factors its point x = t - 2y - 3z, keeping its
// own previous point (the w neighbour) in registers and reading the other six neighbour rows from the
// factor store in L2 (ld.relaxed.gpu: never a stale L1 line).  Rows are dealt to threads so that one
// warp holds 32 consecutive y of one z-layer: its loads of a neighbour row class walk parallel rows.
//
// Arithmetic: per point exactly the reference's sequence (association, IEEE division, no FMA: this
// library is built with -fmad=false and the products below are written with __dmul_rn / __dsub_rn), so
// the factor rows are bitwise those of tilu_factorize_stream and of the reference; a point depends only
// on lexicographically earlier points, hence the first vanishing pivot (smallest rank) is the
// reference's (atomicMin over the failing ranks; later points may see garbage, their ranks are larger).
//
// Operator rows: per-point rows [grid][15] (device), one constant row, or config 3's separable
// coefficient evaluated on the fly (tilu_sepk.h) -- no 2.7 GB row array at level 9.
#include <algorithm>

#include <cstdio>

#include "tilu.h"
#include "tilu_common.cuh"
#include "tilu_plan.cuh"
#include "tilu_sepk_dev.cuh"

namespace tilu {
void prof_begin(cudaStream_t s);
void prof_end(const char *name, cudaStream_t s);
int abi_fail(int code, const char *fmt, ...);
void abi_count_launches(int k);

namespace fac {

struct Args {
    int n;
    int amode;             // 0 per-point rows, 1 constant row, 2 separable coefficient on the fly
    const double *arows;   // [grid][15] (amode 0)
    double arow[15];       // amode 1
    const double *sepk;    // [3][4n+1] (amode 2)
    double c0, w;
    double *store;         // [grid][9]: L_w L_s L_se L_bnw L_bn L_bc L_be D 1/D (ilu.py:32)
    double eps;
    unsigned long long *status;  // [0] = min failing rank + 1 (init ~0ull); [1] = barrier counter
    int nrows;
};

__device__ __forceinline__ unsigned ld_acq(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier on a monotonically increasing counter (every CTA is resident: cooperative launch).
__device__ __forceinline__ void grid_barrier(unsigned *ctr, unsigned &target)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        target += gridDim.x;
        __threadfence();
        atomicAdd(ctr, 1u);
        while ((int)(ld_acq(ctr) - target) < 0) {
        }
        __threadfence();
    }
    __syncthreads();
}

// factor value q of interior point `rank`, or the neutral row (L = 0, D = 1) outside the interior
// (_kernels.py:52-57: beta / gamma are initialised neutral and only interior points are written)
__device__ __forceinline__ double fv(const double *store, bool in, int64_t rank, int q)
{
    TILU_CHECK(!in || rank >= 0, "factor neighbour rank", rank, q);
    return in ? ld_rlx(store + 9 * rank + q) : (q == 7 ? 1.0 : 0.0);
}

// Row of thread slot i: rows are enumerated per z-layer in blocks of 32 consecutive y (one warp).
// rowmap[i] = (z << 16) | y, or -1 for a padding slot.
__global__ void __launch_bounds__(256) k_factor(const Args A, const int *__restrict__ rowmap, int nslots)
{
    const int n = A.n;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthreads = gridDim.x * blockDim.x;
    unsigned *ctr = reinterpret_cast<unsigned *>(A.status + 1);
    unsigned target = 0;
    // rows of this thread (slot tid, tid + nthreads, ...): at most MAXR
    constexpr int MAXR = 8;
    int rz[MAXR], ry[MAXR];
    double pw[MAXR][4];  // own previous point: values 2, 4, 6, 7 (b_se, b_bn, b_be, d_c)
    int nr = 0;
    for (int i = tid; i < nslots && nr < MAXR; i += nthreads) {
        const int code = rowmap[i];
        if (code < 0) continue;
        rz[nr] = code >> 16;
        ry[nr] = code & 0xffff;
        ++nr;
    }
    const int tmin = 6, tmax = 3 * (n - 3) + 3;  // t = x + 2y + 3z over the interior (x, y, z >= 1, x+y+z <= n-1)
    for (int t = tmin; t <= tmax; ++t) {
#pragma unroll 1
        for (int j = 0; j < nr; ++j) {
            const int z = rz[j], y = ry[j];
            const int x = t - 2 * y - 3 * z;
            const int xe = n - 1 - y - z;
            if (x < 1 || x > xe) continue;
            const int64_t base = row_offset(n, z, y);
            const int64_t rank = base + x;
            TILU_CHECK(rank > 0 && rank < num_points(n) && y >= 1 && z >= 1 && y + z <= n - 2, "factor point", rank, t);
            double a[15];
            if (A.amode == 2) {
                const int T4 = 4 * n + 1;
                double hx[7], gy[7], gz[7];
                sepk_window(A.sepk, 4 * x, hx);
                sepk_window(A.sepk + T4, 4 * y, gy);
                sepk_window(A.sepk + 2 * T4, 4 * z, gz);
                sepk_row(hx, gy, gz, A.c0, A.w, a);
            } else if (A.amode == 1) {
#pragma unroll
                for (int q = 0; q < 8; ++q) a[q] = A.arow[q];
            } else {
                const double *r = A.arows + 15 * rank;
#pragma unroll
                for (int q = 0; q < 8; ++q) a[q] = __ldg(r + q);
            }
            // interior-restricted lower stencil (_kernels.py:70-77)
            const bool i_w = x >= 2, i_s = y >= 2, i_se = y >= 2;          // (x+1, y-1, z): x+1+y-1+z <= n-1
            const bool i_bnw = z >= 2 && x >= 2, i_bn = z >= 2, i_bc = z >= 2, i_be = z >= 2;
            const double a_w = i_w ? a[0] : 0.0, a_s = i_s ? a[1] : 0.0, a_se = i_se ? a[2] : 0.0;
            const double a_bnw = i_bnw ? a[3] : 0.0, a_bn = i_bn ? a[4] : 0.0, a_bc = i_bc ? a[5] : 0.0;
            const double a_be = i_be ? a[6] : 0.0, a_c = a[7];
            // neighbour ranks: beta (layer z) ls = (x, y-1), lse = (x+1, y-1); gamma (layer z-1)
            // l = (x, y), lnw = (x-1, y+1), ln = (x, y+1), le = (x+1, y)
            const int64_t r_s = row_offset(n, z, y - 1) + x, r_se = r_s + 1;
            const int64_t g_l = row_offset(n, z - 1, y) + x, g_e = g_l + 1;
            const int64_t g_n = row_offset(n, z - 1, y + 1) + x, g_nw = g_n - 1;
            // gamma neighbours are interior when z >= 2 (their x + y + z sums are <= n - 1 by construction)
            const bool in_gl = z >= 2, in_ge = z >= 2, in_gn = z >= 2, in_gnw = z >= 2 && x >= 2;
            const bool in_s = y >= 2, in_se = y >= 2, in_w = x >= 2;
            const double g_c = fv(A.store, in_gl, g_l, 7);
            const double s4 = fv(A.store, in_s, r_s, 4), s7 = fv(A.store, in_s, r_s, 7);
            const double nw2 = fv(A.store, in_gnw, g_nw, 2), nw7 = fv(A.store, in_gnw, g_nw, 7);
            const double e0 = fv(A.store, in_ge, g_e, 0), e7 = fv(A.store, in_ge, g_e, 7);
            const double n0 = fv(A.store, in_gn, g_n, 0), n1 = fv(A.store, in_gn, g_n, 1);
            const double n2 = fv(A.store, in_gn, g_n, 2), n7 = fv(A.store, in_gn, g_n, 7);
            const double se0 = fv(A.store, in_se, r_se, 0), se3 = fv(A.store, in_se, r_se, 3);
            const double se4 = fv(A.store, in_se, r_se, 4), se7 = fv(A.store, in_se, r_se, 7);
            const double w2 = in_w ? pw[j][0] : 0.0, w4 = in_w ? pw[j][1] : 0.0;
            const double w6 = in_w ? pw[j][2] : 0.0, w7 = in_w ? pw[j][3] : 1.0;
            // _kernels.py:87-110, same association: (b * g) * v, left-to-right subtraction
            const double b_bc = __ddiv_rn(a_bc, g_c);
            const double bcg = dmul(b_bc, g_c);
            const double b_s = __ddiv_rn(dsub(a_s, dmul(bcg, s4)), s7);
            const double b_bnw = __ddiv_rn(dsub(a_bnw, dmul(bcg, nw2)), nw7);
            const double b_be = __ddiv_rn(dsub(a_be, dmul(bcg, e0)), e7);
            const double bnwg = dmul(b_bnw, nw7), bsb = dmul(b_s, s7), beg = dmul(b_be, e7);
            const double b_w = __ddiv_rn(dsub(dsub(dsub(a_w, dmul(bcg, w6)), dmul(bnwg, w4)), dmul(bsb, w2)), w7);
            const double b_bn = __ddiv_rn(dsub(dsub(dsub(a_bn, dmul(bcg, n1)), dmul(beg, n2)), dmul(bnwg, n0)), n7);
            const double b_se = __ddiv_rn(dsub(dsub(dsub(a_se, dmul(bcg, se3)), dmul(beg, se4)), dmul(bsb, se0)), se7);
            double d_c = dsub(a_c, dmul(dmul(b_bc, b_bc), g_c));
            d_c = dsub(d_c, dmul(dmul(b_be, b_be), e7));
            d_c = dsub(d_c, dmul(dmul(b_bnw, b_bnw), nw7));
            d_c = dsub(d_c, dmul(dmul(b_bn, b_bn), n7));
            d_c = dsub(d_c, dmul(dmul(b_se, b_se), se7));
            d_c = dsub(d_c, dmul(dmul(b_s, b_s), s7));
            d_c = dsub(d_c, dmul(dmul(b_w, b_w), w7));
            if (fabs(d_c) < A.eps) atomicMin(A.status, (unsigned long long)(rank + 1));
            double *o = A.store + 9 * rank;
            st_rlx(o + 0, b_w);
            st_rlx(o + 1, b_s);
            st_rlx(o + 2, b_se);
            st_rlx(o + 3, b_bnw);
            st_rlx(o + 4, b_bn);
            st_rlx(o + 5, b_bc);
            st_rlx(o + 6, b_be);
            st_rlx(o + 7, d_c);
            st_rlx(o + 8, __ddiv_rn(1.0, d_c));
            pw[j][0] = b_se;
            pw[j][1] = b_bn;
            pw[j][2] = b_be;
            pw[j][3] = d_c;
        }
        grid_barrier(ctr, target);
    }
}

__global__ void k_gather_rows(const double *__restrict__ store, const int64_t *__restrict__ ranks, int64_t count,
                              double *__restrict__ out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count * 9) return;
    TILU_CHECK(ranks[i / 9] >= 0, "gather rank", ranks[i / 9], i);
    out[i] = store[9 * ranks[i / 9] + i % 9];
}

__global__ void k_fill_rowmap(int n, int *rowmap, int nslots)
{
    // slots: for z = 1..n-3, ceil((n-2-z)/32) warps of 32 consecutive y (y = 1 .. n-2-z)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nslots) return;
    int rem = i >> 5, z = 1;
    for (; z <= n - 3; ++z) {
        const int wz = (n - 2 - z + 31) / 32;
        if (rem < wz) break;
        rem -= wz;
    }
    const int y = 1 + 32 * rem + (i & 31);
    rowmap[i] = (z <= n - 3 && y <= n - 2 - z) ? ((z << 16) | y) : -1;
}

}  // namespace fac
}  // namespace tilu

using namespace tilu;

extern "C" int tilu_factorize_device(int level, const double *arows_dev, const double *arow_host,
                                     const double *sepk_tables_dev, double sepk_c0, double sepk_w,
                                     double *store_dev, double pivot_eps, int64_t *status_host, void *stream)
{
    if (level < 2 || level > 10 || !store_dev || !status_host) return abi_fail(TILU_EINVAL, "factorize_device: bad argument");
    const int nsrc = (arows_dev != nullptr) + (arow_host != nullptr) + (sepk_tables_dev != nullptr);
    if (nsrc != 1) return abi_fail(TILU_EINVAL, "factorize_device: exactly one of arows_dev, arow, sepk_tables_dev");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int n = 1 << level;
    *status_host = 0;
    if (n < 4) return TILU_OK;
    fac::Args A{};
    A.n = n;
    A.amode = sepk_tables_dev ? 2 : (arow_host ? 1 : 0);
    A.arows = arows_dev;
    if (arow_host)
        for (int q = 0; q < 15; ++q) A.arow[q] = arow_host[q];
    A.sepk = sepk_tables_dev;
    A.c0 = sepk_c0;
    A.w = sepk_w;
    A.store = store_dev;
    A.eps = pivot_eps;
    int nslots = 0;
    for (int z = 1; z <= n - 3; ++z) nslots += 32 * ((n - 2 - z + 31) / 32);
    A.nrows = nslots;
    if (nslots == 0) return TILU_OK;

    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fac::k_factor, 256, 0) != cudaSuccess || per < 1 || sms < 1)
        return abi_fail(TILU_ECUDA, "factorize_device: occupancy query failed: %s", cudaGetErrorString(cudaGetLastError()));
    int ctas = std::min(sms * per, (nslots + 255) / 256);
    if ((int64_t)ctas * 256 * 8 < nslots) return abi_fail(TILU_EUNSUPPORTED, "factorize_device: level %d needs more resident threads", level);

    unsigned long long *status = nullptr;
    int *rowmap = nullptr;
    if (cudaMallocAsync(&status, 2 * sizeof(unsigned long long), s) != cudaSuccess ||
        cudaMallocAsync(&rowmap, (size_t)nslots * sizeof(int), s) != cudaSuccess) {
        cudaGetLastError();
        if (status) cudaFreeAsync(status, s);
        return abi_fail(TILU_ENOMEM, "factorize_device: scratch allocation failed");
    }
    const unsigned long long init[2] = {~0ull, 0ull};
    cudaMemcpyAsync(status, init, sizeof(init), cudaMemcpyHostToDevice, s);
    A.status = status;
    prof_begin(s);
    fac::k_fill_rowmap<<<(nslots + 255) / 256, 256, 0, s>>>(n, rowmap, nslots);
    void *params[] = {(void *)&A, (void *)&rowmap, (void *)&nslots};
    cudaError_t e = cudaLaunchCooperativeKernel((const void *)fac::k_factor, dim3(ctas), dim3(256), params, 0, s);
    prof_end("factorize", s);
    abi_count_launches(2);
    unsigned long long st[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(st, status, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(status, s);
    cudaFreeAsync(rowmap, s);
    if (e != cudaSuccess) return abi_fail(TILU_ECUDA, "factorize_device: %s", cudaGetErrorString(e));
    if (st[0] != ~0ull) {
        *status_host = (int64_t)st[0];
        return abi_fail(TILU_EPIVOT, "factorize_device: vanishing pivot at rank %lld", (long long)st[0] - 1);
    }
    return TILU_OK;
}

extern "C" int tilu_gather_rows(const double *store_dev, const int64_t *ranks_dev, int64_t count, double *out_dev,
                                void *stream)
{
    if (count < 0 || (count > 0 && (!store_dev || !ranks_dev || !out_dev))) return abi_fail(TILU_EINVAL, "gather_rows: bad argument");
    if (count == 0) return TILU_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    prof_begin(s);
    fac::k_gather_rows<<<(unsigned)((count * 9 + 255) / 256), 256, 0, s>>>(store_dev, ranks_dev, count, out_dev);
    prof_end("gather_rows", s);
    abi_count_launches(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return abi_fail(TILU_ECUDA, "gather_rows: %s", cudaGetErrorString(e));
    return TILU_OK;
}
