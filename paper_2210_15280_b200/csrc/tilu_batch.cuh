// Batched (interleaved-tets) sweep: kernel arguments.
#pragma once
#include <stdint.h>

namespace tilu {

constexpr int MAXR = 512;  // rows per layer supported (level <= 9; row order packs y, z in 10 bits)

struct BatchArgs {
    double *u;                // packed [G][grid][32 * tpl]
    const double *f;          // packed
    double *wa;               // w_f: packed, 0 on the lattice boundary, sentinel on the interior
    double *wb;               // w_b: packed, 0 on the lattice boundary
    int G, ntets;
    int tpl;                  // tets per lane: groups of 32 * tpl tets, layout [G][grid][32 * tpl]
    int *ticket;              // row ticket counter (zeroed per pass)
    int *done;                // warps finished (backward pass; zeroed per pass)
    int nwarps;               // warps in the (persistent) grid
    unsigned long long *hdr;  // scratch header: == key when w_f is armed
    unsigned long long key;
    double *part;             // [G][nrows][32 * tpl] per-row residual partial sums or nullptr
    int max_ticket;           // debug: warps stop after this ticket (-1 = off)
    double arow[15];          // constant stencil (kernel-parameter constant bank: DMUL operands, no registers)
};

}  // namespace tilu
