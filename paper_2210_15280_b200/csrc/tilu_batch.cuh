// Batched (interleaved-tets) sweep: kernel arguments.
#pragma once
#include <stdint.h>

namespace tilu {

constexpr int BW = 8;              // compute warps per CTA (rows of one z-layer in flight)
constexpr int NT = (BW + 1) * 32;  // + one sync warp (progress mirror, off the compute path)
constexpr int MAXR = 512;          // rows per layer supported (level <= 9)
constexpr int GSTRIDE = MAXR + 4;  // ints per (group, layer) in the global progress array

struct BatchArgs {
    double *u;        // packed [G][grid][32]
    const double *f;  // packed
    double *w;        // packed scratch, zero on the lattice boundary
    int G, ntets;
    int *ticket;      // CTA ticket counter (zeroed per pass)
    int *gprog;       // [G][n-3][GSTRIDE] per-row progress (points done), zeroed per pass
    double *part;     // [G][n-3][32] residual partial sums or nullptr
    int max_ticket;   // debug: CTAs with a larger ticket exit at once (-1 = off)
    double arow[15];  // constant stencil (kernel-parameter constant bank: DMUL operands, no registers)
};

}  // namespace tilu
