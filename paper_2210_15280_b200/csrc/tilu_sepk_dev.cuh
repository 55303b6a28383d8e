// Device side of the on-the-fly rows of a separable scalar coefficient (config 3): the generated
// program tilu_sepk.h evaluated with unfused IEEE ops (bitwise the host builder / reference rows).
#pragma once
#include "tilu_common.cuh"

#define TILU_SEPK_MUL(a, b) ::tilu::dmul((a), (b))
#define TILU_SEPK_ADD(a, b) ::tilu::dadd((a), (b))
#define TILU_SEPK_HD __device__ __forceinline__
#include "tilu_sepk.h"

namespace tilu {

// v[i] = tab[c + i - 3], i = 0..6 (tables hold 4n + 1 abscissae; c = 4 * coordinate, 1 <= coordinate <= n - 3)
__device__ __forceinline__ void sepk_window(const double *__restrict__ tab, int c, double (&v)[7])
{
    TILU_CHECK(c >= 4, "sepk window", c, 0);
#pragma unroll
    for (int i = 0; i < 7; ++i) v[i] = __ldg(tab + c + i - 3);
}

// The 15 row entries of interior point (x, y, z).
__device__ __forceinline__ void sepk_point(const PlanDev &P, int x, int y, int z, double (&a)[15])
{
    const int T = 4 * P.n + 1;
    double hx[7], gy[7], gz[7];
    sepk_window(P.sepk, 4 * x, hx);
    sepk_window(P.sepk + T, 4 * y, gy);
    sepk_window(P.sepk + 2 * T, 4 * z, gz);
    sepk_row(hx, gy, gz, P.sepk_c0, P.sepk_w, a);
}

}  // namespace tilu
