// Batched (interleaved-tets) sweep: schedule tables and kernel arguments.
#pragma once
#include <stdint.h>

namespace tilu {

constexpr int BW = 8;  // warps per CTA = rows of one z-layer in flight

// Per z-layer forward schedule: point (x, y) runs at global step O + A*(y-1) + x - 1.
struct LayerSched {
    int A;   // row skew (>= 2, A * BW >= longest row)
    int B;   // synchronisation window = A - 1 steps
    int O;   // step of the layer's first point
    int T0;  // first step (= O)
    int T1;  // last step
};

struct BatchArgs {
    double *u;        // packed [G][grid][32]
    const double *f;  // packed
    double *w;        // packed scratch, zero on the lattice boundary
    int G, ntets;
    const LayerSched *sched;  // [n-3]
    int Tmax, D;
    int *flags;   // [G][n-3] progress counters (-1 = nothing done)
    int *ticket;  // CTA ticket counter (starts at -1)
    double *part; // [G][n-3][32] residual partial sums or nullptr
};

}  // namespace tilu
