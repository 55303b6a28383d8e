// Grid transfers of the multigrid cycle around the smoother on one macro-tet:
// the linear-interpolation prolongation P of multigrid.py:241-277 (build_prolongation: coinciding
// vertices copy, edge midpoints average their two coarse endpoints) applied matrix-free on the
// lattice, P^T for the restriction (Hierarchy.restrict / v_cycle, multigrid.py:383-388, 476-480), and
// the dense apply of the coarsest-level inverse (Hierarchy.coarse_solve, multigrid.py:445-457).
//
// A fine point f = 2C + d with d one of the 14 stencil directions is the midpoint of the coarse edge
// (C, C + d) (the parity classes of _PARITY_ENDPOINTS, multigrid.py:230-238), so P^T gathers, per
// coarse point, the coinciding fine point (weight 1) and its 14 fine neighbours (weight 1/2) -- the
// same 15-point shape as the operator stencil.  scipy's csc (P^T) product accumulates a coarse
// entry over ascending fine index, i.e. over the offsets in (dz, dy, dx) order, which the restriction
// kernel repeats; the csr (P) product of an odd point is 0.5 e_a + 0.5 e_b.  Vectors are the
// reference layout (full-lattice rank order, zero outside the interior).
#include <cstdio>

#include "tilu.h"
#include "tilu_common.cuh"

namespace tilu {
void prof_begin(cudaStream_t s);
void prof_end(const char *name, cudaStream_t s);
int abi_fail(int code, const char *fmt, ...);
void abi_count_launches(int k);

namespace mg {

__device__ __forceinline__ int64_t rank_of(int n, int x, int y, int z) { return row_offset(n, z, y) + x; }

// offsets (dx, dy, dz) in ascending (dz, dy, dx) order = ascending fine rank; weight 1 for (0,0,0)
__device__ __constant__ static const signed char kOff[15][3] = {
    {0, 0, -1}, {1, 0, -1}, {-1, 1, -1}, {0, 1, -1},                    // dz = -1: bc be bnw bn
    {0, -1, 0}, {1, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {1, 0, 0}, {-1, 1, 0}, {0, 1, 0},  // dz = 0
    {0, -1, 1}, {1, -1, 1}, {-1, 0, 1}, {0, 0, 1}};                     // dz = +1: ts tse tw tc

// rc = P^T r on interior coarse points, 0 elsewhere.  grid (yc, zc), threads over xc.
__global__ void __launch_bounds__(128) k_restrict(int nc, const double *__restrict__ rf, double *__restrict__ rc)
{
    const int zc = blockIdx.y, yc = blockIdx.x;
    if (yc + zc > nc) return;
    const int nf = 2 * nc;
    const int64_t cb = row_offset(nc, zc, yc);
    for (int xc = threadIdx.x; xc <= nc - yc - zc; xc += blockDim.x) {
        double acc = 0.0;
        if (interior(xc, yc, zc, nc)) {
#pragma unroll
            for (int d = 0; d < 15; ++d) {
                const int dx = kOff[d][0], dy = kOff[d][1], dz = kOff[d][2];
                TILU_CHECK(2 * xc + dx >= 0 && 2 * yc + dy >= 0 && 2 * zc + dz >= 0 &&
                               2 * (xc + yc + zc) + dx + dy + dz <= nf, "restrict fine point", xc, d);
                const double v = rf[rank_of(nf, 2 * xc + dx, 2 * yc + dy, 2 * zc + dz)];
                acc = dadd(acc, (dx | dy | dz) ? dmul(0.5, v) : v);
            }
        }
        rc[cb + xc] = acc;
    }
}

// u += P e on interior fine points.  grid (yf, zf), threads over xf.
__global__ void __launch_bounds__(128) k_prolong_add(int nc, const double *__restrict__ ec, double *__restrict__ uf)
{
    const int nf = 2 * nc;
    const int zf = blockIdx.y + 1, yf = blockIdx.x + 1;
    if (yf + zf > nf - 2) return;
    const int64_t fb = row_offset(nf, zf, yf);
    for (int xf = 1 + threadIdx.x; xf <= nf - 1 - yf - zf; xf += blockDim.x) {
        const int px = xf & 1, py = yf & 1, pz = zf & 1;
        double add;
        if (!(px | py | pz)) {
            add = ec[rank_of(nc, xf >> 1, yf >> 1, zf >> 1)];
        } else {
            // endpoint maps of the parity class (multigrid.py:230-238): a + b = fine coordinate
            int ax, ay, az;
            const int code = px + 2 * py + 4 * pz;
            switch (code) {
            case 1: ax = -1, ay = 0, az = 0; break;
            case 2: ax = 0, ay = -1, az = 0; break;
            case 4: ax = 0, ay = 0, az = -1; break;
            case 3: ax = 1, ay = -1, az = 0; break;
            case 5: ax = 1, ay = 0, az = -1; break;
            case 6: ax = 0, ay = 1, az = -1; break;
            default: ax = -1, ay = 1, az = -1; break;
            }
            const int hx = (xf + ax) >> 1, hy = (yf + ay) >> 1, hz = (zf + az) >> 1;
            TILU_CHECK(hx >= 0 && hy >= 0 && hz >= 0 && hx + hy + hz <= nc && hx - ax >= 0 && hy - ay >= 0 && hz - az >= 0 &&
                           hx + hy + hz - ax - ay - az <= nc, "prolong coarse endpoints", xf, code);
            const double ea = ec[rank_of(nc, hx, hy, hz)];
            const double eb = ec[rank_of(nc, hx - ax, hy - ay, hz - az)];
            add = dadd(dmul(0.5, ea), dmul(0.5, eb));
        }
        uf[fb + xf] = dadd(uf[fb + xf], add);
    }
}

// y = M x, M row-major [m][m]; one warp per row, fixed lane-strided order + shuffle tree.
__global__ void __launch_bounds__(128) k_dense_mv(int m, const double *__restrict__ M, const double *__restrict__ x,
                                                  double *__restrict__ y)
{
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= m) return;
    double acc = 0.0;
    for (int j = lane; j < m; j += 32) acc = fma(M[(int64_t)row * m + j], x[j], acc);
    for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) y[row] = acc;
}

}  // namespace mg
}  // namespace tilu

using namespace tilu;

extern "C" int tilu_mg_restrict(int coarse_level, const double *r_fine, double *r_coarse, void *stream)
{
    if (coarse_level < 1 || coarse_level > 9 || !r_fine || !r_coarse) return abi_fail(TILU_EINVAL, "mg_restrict: bad argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nc = 1 << coarse_level;
    prof_begin(s);
    mg::k_restrict<<<dim3(nc + 1, nc + 1), 128, 0, s>>>(nc, r_fine, r_coarse);
    prof_end("mg_restrict", s);
    abi_count_launches(1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TILU_OK : abi_fail(TILU_ECUDA, "mg_restrict: %s", cudaGetErrorString(e));
}

extern "C" int tilu_mg_prolong_add(int coarse_level, const double *e_coarse, double *u_fine, void *stream)
{
    if (coarse_level < 1 || coarse_level > 9 || !e_coarse || !u_fine) return abi_fail(TILU_EINVAL, "mg_prolong_add: bad argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nc = 1 << coarse_level, nf = 2 * nc;
    if (nf < 4) return TILU_OK;
    prof_begin(s);
    mg::k_prolong_add<<<dim3(nf - 3, nf - 3), 128, 0, s>>>(nc, e_coarse, u_fine);
    prof_end("mg_prolong", s);
    abi_count_launches(1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TILU_OK : abi_fail(TILU_ECUDA, "mg_prolong_add: %s", cudaGetErrorString(e));
}

extern "C" int tilu_dense_mv(int m, const double *M, const double *x, double *y, void *stream)
{
    if (m < 0 || (m > 0 && (!M || !x || !y))) return abi_fail(TILU_EINVAL, "dense_mv: bad argument");
    if (m == 0) return TILU_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    prof_begin(s);
    mg::k_dense_mv<<<(m + 3) / 4, 128, 0, s>>>(m, M, x, y);
    prof_end("mg_coarse", s);
    abi_count_launches(1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TILU_OK : abi_fail(TILU_ECUDA, "dense_mv: %s", cudaGetErrorString(e));
}
