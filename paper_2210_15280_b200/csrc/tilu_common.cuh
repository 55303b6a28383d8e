// Shared device helpers for the sm_100a surrogate ILU(0) smoother kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Debug build (-DTILU_DEBUG_BOUNDS, tools/build_variant.py bounds -DTILU_DEBUG_BOUNDS): global-memory
// indices of every kernel family are range-checked; a violation prints and traps.  Off (no code) in
// the product build.
#ifdef TILU_DEBUG_BOUNDS
#include <cstdio>
#define TILU_CHECK(cond, what, a, b)                                                                  \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("tilu bounds: %s (%lld, %lld) block %d thread %d\n", what, (long long)(a), (long long)(b), \
                   blockIdx.x, threadIdx.x);                                                          \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define TILU_CHECK(cond, what, a, b) ((void)0)
#endif

namespace tilu {

// Unfused IEEE fp64 ops.  The reference Numba kernels contract nothing; the
// forward-difference (NDDF) seeding must reproduce their rounding bit for bit, and in exact
// mode so must the substitution and residual.  __d*_rn are never contracted into DFMA.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// acc - a*b: reference order (separately rounded product) or one fused DFMA (fast mode).
template <bool EXACT>
__device__ __forceinline__ double msub(double acc, double a, double b)
{
    if (EXACT) return dsub(acc, dmul(a, b));
    return fma(-a, b, acc);
}
template <bool EXACT>
__device__ __forceinline__ double madd(double acc, double a, double b)
{
    if (EXACT) return dadd(acc, dmul(a, b));
    return fma(a, b, acc);
}

// Handoff accesses of the data-is-the-flag protocol (a value produced by another warp / CTA during
// the same kernel, polled until it is no longer the sentinel): morally strong relaxed accesses at
// GPU scope -- single-copy atomic and eventually visible under the PTX memory model -- issued as
// asm volatile so the compiler never caches a polled value in a register or drops / merges a
// store.  They compile to the same LDG/STG.E.STRONG.GPU as ld.global.cg / a plain store (the L1
// is bypassed either way); no ordering with other addresses is needed (each value is its own flag).
__device__ __forceinline__ double ld_rlx(const double *p)
{
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_rlx2(const double *p)
{
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_rlx(double *p, double v)
{
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v));
}
__device__ __forceinline__ void st_rlx2(double *p, double a, double b)
{
    asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b));
}

__host__ __device__ __forceinline__ int64_t num_points(int64_t m)
{
    return m < 0 ? 0 : (m + 1) * (m + 2) * (m + 3) / 6;
}

// Full-lattice rank of row (z, y) at x = 0 (geometry.py:188-215 rank_tables).
__host__ __device__ __forceinline__ int64_t row_offset(int n, int z, int y)
{
    const int64_t zoff = num_points(n) - num_points(n - z);
    return zoff + (int64_t)y * (n - z + 1) - (int64_t)y * (y - 1) / 2;
}

// Index of interior row (z, y) in (z, y) lexicographic order.
__host__ __device__ __forceinline__ int row_id(int n, int z, int y)
{
    return (z - 1) * (n - 2) - (z - 1) * z / 2 + (y - 1);
}

__host__ __device__ __forceinline__ bool interior(int x, int y, int z, int n)
{
    return x >= 1 && y >= 1 && z >= 1 && x + y + z <= n - 1;
}

// Lower-direction displacements w s se bnw bn bc be (_kernels.py:12-15).
__device__ __constant__ static const int kDX[7] = {-1, 0, 1, -1, 0, 0, 1};
__device__ __constant__ static const int kDY[7] = {0, -1, -1, 1, 1, 0, 0};
__device__ __constant__ static const int kDZ[7] = {0, 0, 0, -1, -1, -1, -1};

// Horner in z of table m ([M][kx1][ky1][kz1]) then in y, giving the x-polynomial ax[0..kx1-1]
// (_kernels.py:274-292 _collapse_z / _collapse_y), exact order.
__device__ __forceinline__ void collapse_zy(const double *__restrict__ coefs, int m, int kx1, int ky1, int kz1,
                                            double zval, double yval, double *ax)
{
    const double *c = coefs + (int64_t)m * kx1 * ky1 * kz1;
    for (int i = 0; i < kx1; ++i) {
        double accy = 0.0;
        for (int j = ky1 - 1; j >= 0; --j) {
            const double *cij = c + ((int64_t)i * ky1 + j) * kz1;
            double bz = cij[kz1 - 1];
            for (int k = kz1 - 2; k >= 0; --k) bz = dadd(dmul(bz, zval), cij[k]);
            accy = (j == ky1 - 1) ? bz : dadd(dmul(accy, yval), bz);
        }
        ax[i] = accy;
    }
}

// Difference table of the x-polynomial at x0, x0+step, ... (count points), zero-padded to kx1
// entries (_kernels.py:295-310 _horner1 / _seed_diffs).
__device__ __forceinline__ void seed_table(const double *ax, int kx1, int x0, int step, double h, int count,
                                           double *out)
{
    for (int t = 0; t < count; ++t) {
        const double xv = dmul((double)(x0 + t * step), h);
        double acc = ax[kx1 - 1];
        for (int i = kx1 - 2; i >= 0; --i) acc = dadd(dmul(acc, xv), ax[i]);
        out[t] = acc;
    }
    for (int o = 1; o < count; ++o)
        for (int t = count - 1; t >= o; --t) out[t] = dsub(out[t], out[t - 1]);
    for (int t = count; t < kx1; ++t) out[t] = 0.0;
}

// One forward-difference step d[j] += d[j+1] (_kernels.py:313-316).  Marching all K-1 entries
// instead of count-1 never changes an entry that is read before the row ends (the value used at
// step s depends only on d[0..s] with s < count), so the fixed-width march is bitwise safe.
template <int K>
__device__ __forceinline__ void march(double *d)
{
#pragma unroll
    for (int j = 0; j < K - 1; ++j) d[j] = dadd(d[j], d[j + 1]);
}

}  // namespace tilu
