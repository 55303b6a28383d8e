// Host-side setup: the per-point operator rows of a separable scalar coefficient on the unit
// macro-tet (config 3's k(x) = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z)), from the generated
// program tilu_sepk.h -- the same rows, bitwise, as the reference's per-point numpy assembly
// (stencil_source, assembly.py:208-221; pinned by tests/test_sepk.py), in seconds instead of the
// reference's ~28 min at level 9.  Compiled with -ffp-contract=off: nothing is fused.
#include <cstdint>
#include <cstring>

#include "tilu.h"
#include "tilu_sepk.h"

extern "C" int tilu_sepk_rows(int level, const double *tables, double c0, double w, double *rows)
{
    if (level < 2 || level > 10 || !tables || !rows) return TILU_EINVAL;
    const int n = 1 << level;
    const int T = 4 * n + 1;
    const double *hxT = tables, *gyT = tables + T, *gzT = tables + 2 * T;
    auto num_points = [](int64_t m) { return m < 0 ? (int64_t)0 : (m + 1) * (m + 2) * (m + 3) / 6; };
    for (int z = 1; z <= n - 3; ++z) {
        double gz[7];
        for (int i = 0; i < 7; ++i) gz[i] = gzT[4 * z + i - 3];
        const int64_t zoff = num_points(n) - num_points(n - z);
        for (int y = 1; y <= n - 2 - z; ++y) {
            double gy[7];
            for (int i = 0; i < 7; ++i) gy[i] = gyT[4 * y + i - 3];
            const int64_t base = zoff + (int64_t)y * (n - z + 1) - (int64_t)y * (y - 1) / 2;
            for (int x = 1; x <= n - 1 - z - y; ++x) {
                double hx[7], a[15];
                for (int i = 0; i < 7; ++i) hx[i] = hxT[4 * x + i - 3];
                tilu::sepk_row(hx, gy, gz, c0, w, a);
                std::memcpy(rows + 15 * (base + x), a, sizeof(a));
            }
        }
    }
    return TILU_OK;
}
