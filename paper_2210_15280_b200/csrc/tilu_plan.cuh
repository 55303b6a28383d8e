// Device-side plan layout shared by all kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tilu.h"

namespace tilu {

// Per-row metadata, rows in (z, y) lexicographic order (row_id()).
struct RowInfo {
    int z, y, xe, t0;  // t0 = first hyperplane step of the row: 1 + 2y + 3z (x = 1)
};

// POD view passed by value to kernels.
struct PlanDev {
    int level, n;
    int64_t grid;
    int nrows;
    int kx1, ky1, kz1;
    int variant;  // 1 = V1, 2 = V2
    double h;
    int tmin, tmax;                  // hyperplane t = x + 2y + 3z over the interior
    const RowInfo *rows;             // [nrows]
    const int64_t *rowbase;          // [nrows] rank of (0, y, z)
    const int *bandoff;              // [nrows] first band entry of the row (V1)
    const double *store;             // [nband][9] (V1)
    const double *seedF;             // [nrows][7][kx1]  forward-difference tables, forward pass
    const double *seedB;             // [nrows][8][kx1]  backward pass: 7 shifted L + 1/D
    const double *arow;              // [15] constant stencil or nullptr
    const double *arows;             // [grid][15] per-point rows or nullptr
    const double *sepk;              // [3][4n+1] separable-coefficient tables (rows on the fly) or nullptr
    double sepk_c0, sepk_w;
    const double *seedA;             // [nrows][15][akx1] operator-surrogate tables or nullptr
    int akx1;
    const double *factors;           // [grid][9] stored ILU rows or nullptr
    int64_t nband_dbg;               // band entries (debug bounds checks)
    // Per-point coefficient tables of the batched path (shared by every tet of a batch; built once
    // per plan on first use, bit-identical to the on-the-fly NDDF + band evaluation):
    const double *coefF;             // [grid][8]: L_0..L_6 at p (forward), 0
    const double *coefB;             // [grid][8]: L_0..L_6 at q_m = p - d_m (0 outside), 1/D at p
    // Batched row order: (z << 10) | y for every interior row, sorted by the wavefront step of its
    // first point t = 2y + 3z (ties by z).  Every forward dependency of a row has a smaller t, so
    // the order is topological; the backward pass walks it reversed.
    const int *order;
};

}  // namespace tilu

struct tilu_plan {
    tilu::PlanDev dev;
    const void *bsched;  // non-null: the batched (packed) path supports this level
    double harow[15];  // host copy of the constant stencil (batched kernel parameters)
    int flags;
    int64_t interior;
    int64_t nband;
    int ky1a, kz1a;
    void *coef;  // coefficient tables (2 x [grid][8] doubles), lazily built; freed with the plan
    void *plane;  // plane-layout workspace of the single-tet path (tilu_plane.cu), lazily built
    // owned device allocations
    const double *zrow;  // DEVICE [15] zeros: the operator row of solve_into routed through a sweep (r = f exactly)
    void *allocs[20];
    int nallocs;
};
