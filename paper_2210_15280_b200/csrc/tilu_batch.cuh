// Batched (interleaved-tets) sweep: schedule tables and kernel arguments.
#pragma once
#include <stdint.h>

#include <vector>

namespace tilu {

constexpr int BW = 8;        // compute warps per CTA = rows of one z-layer in flight
constexpr int NT = (BW + 1) * 32;  // + one sync warp (progress wait / publish off the compute path)
constexpr int BWIN = 4;      // synchronisation window (steps between CTA barriers)
constexpr int PF = 1;        // load prefetch distance (points)
constexpr int RING = 4;      // register ring slots (== BWIN: static slot indices in the unrolled window)
static_assert(RING == BWIN && PF < RING, "ring layout");
// min. start offset of consecutive rows of a layer: window + 1 + PF

// Per-row schedule (indexed by row_id(n, z, y)): the forward step of point (x, y, z) is
// start + x - 1; next / prev = the neighbouring rows (same layer) owned by the same warp, 0 = none.
struct RowSched {
    int start, next, prev;
};

// Per z-layer: first / last forward step and each warp's first / last row (0 = none).
struct LayerSched {
    int T0, T1;
    int first[BW], last[BW];
};

struct BatchArgs {
    double *u;        // packed [G][grid][32]
    const double *f;  // packed
    double *w;        // packed scratch, zero on the lattice boundary
    int G, ntets;
    const LayerSched *sched;  // [n-3]
    const RowSched *rows;     // [nrows]
    int Tmax, D;
    int *flags;    // [G][n-3] progress counters (-1 = nothing done)
    int *ticket;   // CTA ticket counter (starts at -1)
    double *part;  // [G][n-3][32] residual partial sums or nullptr
    unsigned long long *trace;  // debug: per CTA [ticket][4] globaltimer stamps (start, first window open,
                                //        end, windows) or nullptr
    int max_ticket;   // debug: CTAs with a larger ticket exit at once (-1 = off)
    double arow[15];  // constant stencil (kernel-parameter constant bank: DMUL operands, no registers)
};

// Host: greedy list schedule of one level (tilu_batch.cu header comment).
void batch_schedule(int n, int bwin, int pf, std::vector<LayerSched> &layers, std::vector<RowSched> &rows, int &Tmax,
                    int &D);

}  // namespace tilu
