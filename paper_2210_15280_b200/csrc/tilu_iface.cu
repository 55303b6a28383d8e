// Interface stages of the hybrid multi-tet smoother: the vertex / edge / face
// primitive blocks that macro-tets share are smoothed by CSR triangular substitution
// (Hierarchy._interface_stage, multigrid.py:400-412 -> _kernels.csr_lower_solve / csr_upper_solve,
// _kernels.py:490-519) on the residual r = f - A u restricted to the blocks' rows.
//
// Blocks of one primitive kind are independent (the stage computes r once, then every block solves
// its own rows: block Jacobi across blocks, Gauss-Seidel inside), so one CTA takes one block and
// walks its dependency levels (level of a row = 1 + max level of the rows it reads; computed once on
// the host by tilu_csr_levels) with a CTA barrier between levels.  Per row the arithmetic is the
// reference's: acc = b_i, acc -= a_ij z_j over the strictly lower (upper) entries in CSR order,
// z_i = acc / a_ii -- bitwise equal for any schedule.  The residual rows repeat scipy's csr_matvec
// order (sum from 0 over the row's entries, then f - sum).
#include <algorithm>
#include <cstdio>
#include <vector>

#include "tilu.h"
#include "tilu_common.cuh"

namespace tilu {
void prof_begin(cudaStream_t s);
void prof_end(const char *name, cudaStream_t s);
int abi_fail(int code, const char *fmt, ...);
void abi_count_launches(int k);

namespace iface {

__global__ void __launch_bounds__(128) k_residual_rows(int64_t nrows, const int64_t *__restrict__ indptr,
                                                       const int64_t *__restrict__ indices,
                                                       const double *__restrict__ data, const int64_t *__restrict__ ids,
                                                       const double *__restrict__ u, const double *__restrict__ f,
                                                       double *__restrict__ r)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    double sum = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) sum = dadd(sum, dmul(data[k], u[indices[k]]));
    r[i] = dsub(f[ids[i]], sum);
}

// y = M x (accumulate = 0) or y += M x (accumulate = 1) for a CSR matrix, one thread per row, the row's products
// summed from 0 in index order (scipy's csr_matvec; for M = P^T stored as CSR that is csc_matvec's ascending
// fine-index accumulation): the transfers of a macro-mesh hierarchy (Hierarchy.restrict / prolongate,
// multigrid.py:377-388 with the caller's build_prolongation matrices).
__global__ void __launch_bounds__(128) k_csr_matvec(int64_t nrows, const int64_t *__restrict__ indptr,
                                                    const int64_t *__restrict__ indices, const double *__restrict__ data,
                                                    const double *__restrict__ x, double *__restrict__ y, int accumulate)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    double sum = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) sum = dadd(sum, dmul(data[k], x[indices[k]]));
    y[i] = accumulate ? dadd(y[i], sum) : sum;
}

// One CTA per block.  Rows of block b: roff[b] .. roff[b+1]-1 of the concatenated block CSR (block-local
// column indices).  Schedule: levels loff[b] .. loff[b+1]-1; level l holds rows perm[lptr[l] .. lptr[l+1]-1]
// (block-local row numbers).  After the solve u[ids[row]] += z[row].
__global__ void __launch_bounds__(128) k_tri_solve_blocks(const int64_t *__restrict__ roff, const int64_t *__restrict__ indptr,
                                                          const int *__restrict__ indices, const double *__restrict__ data,
                                                          const int64_t *__restrict__ loff, const int64_t *__restrict__ lptr,
                                                          const int *__restrict__ perm, int upper,
                                                          const double *__restrict__ b, double *z,
                                                          const int64_t *__restrict__ ids, double *u)
{
    const int blk = blockIdx.x;
    const int64_t r0 = roff[blk], m = roff[blk + 1] - r0;
    double *zb = z + r0;
    for (int64_t l = loff[blk]; l < loff[blk + 1]; ++l) {
        for (int64_t q = lptr[l] + threadIdx.x; q < lptr[l + 1]; q += blockDim.x) {
            const int i = perm[q];
            double acc = b[r0 + i], diag = 0.0;
            TILU_CHECK(i >= 0 && i < m, "tri solve row", i, blk);
            for (int64_t k = indptr[r0 + i]; k < indptr[r0 + i + 1]; ++k) {
                const int j = indices[k];
                TILU_CHECK(j >= 0 && j < m, "tri solve column", j, blk);
                if (upper ? (j > i) : (j < i)) acc = dsub(acc, dmul(data[k], zb[j]));
                else if (j == i) diag = data[k];
            }
            zb[i] = __ddiv_rn(acc, diag);
        }
        __syncthreads();
    }
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const int64_t g = ids[r0 + i];
        u[g] = dadd(u[g], zb[i]);
    }
}

}  // namespace iface
}  // namespace tilu

using namespace tilu;

// Host helper: dependency level of every row of one CSR block for the lower (upper = 0) or upper
// substitution; returns the number of levels.  level[i] in 0 .. nlevels-1.
extern "C" int tilu_csr_levels(int m, const int64_t *indptr, const int *indices, int upper, int *level)
{
    if (m < 0 || (m > 0 && (!indptr || !indices || !level))) return -1;
    int nl = 0;
    if (!upper) {
        for (int i = 0; i < m; ++i) {
            int lv = 0;
            for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
                if (indices[k] < i) lv = std::max(lv, level[indices[k]] + 1);
            level[i] = lv;
            nl = std::max(nl, lv + 1);
        }
    } else {
        for (int i = m - 1; i >= 0; --i) {
            int lv = 0;
            for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k)
                if (indices[k] > i) lv = std::max(lv, level[indices[k]] + 1);
            level[i] = lv;
            nl = std::max(nl, lv + 1);
        }
    }
    return nl;
}

extern "C" int tilu_csr_residual_rows(int64_t nrows, const int64_t *indptr, const int64_t *indices, const double *data,
                                      const int64_t *ids, const double *u, const double *f, double *r, void *stream)
{
    if (nrows < 0 || (nrows > 0 && (!indptr || !indices || !data || !ids || !u || !f || !r)))
        return abi_fail(TILU_EINVAL, "csr_residual_rows: bad argument");
    if (nrows == 0) return TILU_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    prof_begin(s);
    iface::k_residual_rows<<<(unsigned)((nrows + 127) / 128), 128, 0, s>>>(nrows, indptr, indices, data, ids, u, f, r);
    prof_end("iface_residual", s);
    abi_count_launches(1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TILU_OK : abi_fail(TILU_ECUDA, "csr_residual_rows: %s", cudaGetErrorString(e));
}

extern "C" int tilu_csr_matvec(int64_t nrows, const int64_t *indptr, const int64_t *indices, const double *data,
                               const double *x, double *y, int accumulate, void *stream)
{
    if (nrows < 0 || (nrows > 0 && (!indptr || !indices || !data || !x || !y)))
        return abi_fail(TILU_EINVAL, "csr_matvec: bad argument");
    if (nrows == 0) return TILU_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    prof_begin(s);
    iface::k_csr_matvec<<<(unsigned)((nrows + 127) / 128), 128, 0, s>>>(nrows, indptr, indices, data, x, y, accumulate);
    prof_end("csr_matvec", s);
    abi_count_launches(1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TILU_OK : abi_fail(TILU_ECUDA, "csr_matvec: %s", cudaGetErrorString(e));
}

extern "C" int tilu_csr_tri_solve_blocks(int nblocks, const int64_t *roff, const int64_t *indptr, const int *indices,
                                         const double *data, const int64_t *loff, const int64_t *lptr, const int *perm,
                                         int upper, const double *b, double *z, const int64_t *ids, double *u,
                                         void *stream)
{
    if (nblocks < 0 || (nblocks > 0 && (!roff || !indptr || !indices || !data || !loff || !lptr || !perm || !b || !z || !ids || !u)))
        return abi_fail(TILU_EINVAL, "csr_tri_solve_blocks: bad argument");
    if (nblocks == 0) return TILU_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    prof_begin(s);
    iface::k_tri_solve_blocks<<<nblocks, 128, 0, s>>>(roff, indptr, indices, data, loff, lptr, perm, upper, b, z, ids, u);
    prof_end(upper ? "iface_upper" : "iface_lower", s);
    abi_count_launches(1);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TILU_OK : abi_fail(TILU_ECUDA, "csr_tri_solve_blocks: %s", cudaGetErrorString(e));
}
