// Host-side setup: streaming two-layer LDL^T ILU(0) factorization of one macro-tet
// interior (arXiv 2210.15280, Alg. 1).  Replaces the reference Numba kernel
// _kernels.factorize_stream (/root/reference/pkg/src/tetilu/_kernels.py:39-143).
//
// Only the current (beta) and previous (gamma) z-layer are kept: two triangles of
// (n+1)(n+2)/2 stencils x 8 values, initialised to the neutral row L = 0, D = 1 so
// boundary neighbours drop out (ilu.py:43-78).  The eight stencil equations at
// each point are evaluated in the reference's exact order and association
// (no FMA: this TU is compiled with -ffp-contract=off), so the factor rows, and
// therefore the sampled least-squares targets, are bitwise identical to the
// reference's (pinned by tests/test_setup_parity.py).
#include <cmath>
#include <cstdint>
#include <vector>

#include "tilu.h"

namespace {

struct Layer {
    // value q of triangle slot s
    std::vector<double> v;
    explicit Layer(int64_t tri) : v(static_cast<size_t>(tri) * 8, 0.0) {}
    double &at(int64_t s, int q) { return v[static_cast<size_t>(s) * 8 + q]; }
    void reset_neutral(int64_t tri) {
        for (int64_t s = 0; s < tri; ++s) {
            for (int q = 0; q < 7; ++q) at(s, q) = 0.0;
            at(s, 7) = 1.0;
        }
    }
};

inline bool inside(int x, int y, int z, int n) { return x >= 1 && y >= 1 && z >= 1 && x + y + z <= n - 1; }

}  // namespace

extern "C" int64_t tilu_factorize_stream(int n, const int64_t *rowoff, const double *arows, int aconst,
                                         double *full_store, int do_full, const int64_t *collect_ranks,
                                         int64_t ncollect, double *collect_out, double pivot_eps)
{
    const int64_t tri = static_cast<int64_t>(n + 1) * (n + 2) / 2;
    std::vector<int64_t> loff(n + 2);
    for (int y = 0; y <= n + 1; ++y) loff[y] = static_cast<int64_t>(y) * (n + 1) - static_cast<int64_t>(y) * (y - 1) / 2;
    Layer cur(tri), prev(tri);  // beta, gamma
    cur.reset_neutral(tri);
    prev.reset_neutral(tri);

    int64_t cptr = 0;
    for (int z = 1; z < n - 2; ++z) {
        for (int y = 1; y < n - 1 - z; ++y) {
            const int64_t base = rowoff[static_cast<int64_t>(z) * (n + 1) + y];
            for (int x = 1; x < n - z - y; ++x) {
                const int64_t rank = base + x;
                const double *row = aconst ? arows : arows + 15 * rank;
                // interior-restricted lower stencil (entries toward the boundary vanish)
                const double a_w = inside(x - 1, y, z, n) ? row[0] : 0.0;
                const double a_s = inside(x, y - 1, z, n) ? row[1] : 0.0;
                const double a_se = inside(x + 1, y - 1, z, n) ? row[2] : 0.0;
                const double a_bnw = inside(x - 1, y + 1, z - 1, n) ? row[3] : 0.0;
                const double a_bn = inside(x, y + 1, z - 1, n) ? row[4] : 0.0;
                const double a_bc = inside(x, y, z - 1, n) ? row[5] : 0.0;
                const double a_be = inside(x + 1, y, z - 1, n) ? row[6] : 0.0;
                const double a_c = row[7];

                const int64_t l = loff[y] + x, lw = l - 1, ls = loff[y - 1] + x, lse = ls + 1;
                const int64_t lnw = loff[y + 1] + x - 1, ln = lnw + 1, le = l + 1;
                double *B = cur.v.data(), *G = prev.v.data();
#define BV(s, q) B[(s) * 8 + (q)]
#define GV(s, q) G[(s) * 8 + (q)]
                const double g_c = GV(l, 7);
                const double b_bc = a_bc / g_c;
                const double b_s = (a_s - b_bc * g_c * BV(ls, 4)) / BV(ls, 7);
                const double b_bnw = (a_bnw - b_bc * g_c * GV(lnw, 2)) / GV(lnw, 7);
                const double b_be = (a_be - b_bc * g_c * GV(le, 0)) / GV(le, 7);
                const double b_w = (a_w - b_bc * g_c * BV(lw, 6) - b_bnw * GV(lnw, 7) * BV(lw, 4) -
                                    b_s * BV(ls, 7) * BV(lw, 2)) / BV(lw, 7);
                const double b_bn = (a_bn - b_bc * g_c * GV(ln, 1) - b_be * GV(le, 7) * GV(ln, 2) -
                                     b_bnw * GV(lnw, 7) * GV(ln, 0)) / GV(ln, 7);
                const double b_se = (a_se - b_bc * g_c * BV(lse, 3) - b_be * GV(le, 7) * BV(lse, 4) -
                                     b_s * BV(ls, 7) * BV(lse, 0)) / BV(lse, 7);
                const double d_c = a_c - b_bc * b_bc * g_c - b_be * b_be * GV(le, 7) -
                                   b_bnw * b_bnw * GV(lnw, 7) - b_bn * b_bn * GV(ln, 7) -
                                   b_se * b_se * BV(lse, 7) - b_s * b_s * BV(ls, 7) - b_w * b_w * BV(lw, 7);
                if (std::fabs(d_c) < pivot_eps) return rank + 1;
                const double vals[8] = {b_w, b_s, b_se, b_bnw, b_bn, b_bc, b_be, d_c};
                for (int q = 0; q < 8; ++q) BV(l, q) = vals[q];
#undef BV
#undef GV
                if (do_full) {
                    double *F = full_store + 9 * rank;
                    for (int q = 0; q < 8; ++q) F[q] = vals[q];
                    F[8] = 1.0 / d_c;
                }
                if (cptr < ncollect && collect_ranks[cptr] == rank) {
                    double *C = collect_out + 9 * cptr;
                    for (int q = 0; q < 8; ++q) C[q] = vals[q];
                    C[8] = 1.0 / d_c;
                    ++cptr;
                }
            }
        }
        // next layer: gamma <- beta, beta <- neutral
        prev.v.swap(cur.v);
        cur.reset_neutral(tri);
    }
    return 0;
}
