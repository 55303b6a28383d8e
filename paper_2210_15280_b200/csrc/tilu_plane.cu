// Plane-layout fast path for one large macro-tetrahedron (configs 1, 2, 3, 5: a single tet whose
// sweep must be parallelised inside the tet).
//
// Geometry.  A lattice row (z, y) of length xe = n-1-y-z lies on the anti-diagonal s = y + z, and
// every row of one diagonal has the same length xe(s) = n-1-s.  With the skewed coordinate
// tau = x + z, the forward dependencies of point (x, y, z) (_kernels.py:323-367, offsets
// w s se bnw bn bc be) are
//     own row            (tau-1, z)                      -> register
//     same diagonal s    (tau-2, z-1), (tau-1, z-1)      -> lane z-1 of the same warp, 1-2 steps ago
//     diagonal s-1       (tau, z), (tau+1, z), (tau-1, z-1), (tau, z-1)
// so a warp whose 32 lanes own 32 consecutive rows z0..z0+31 of one diagonal, lane z processing
// x = tau - z at step tau, resolves every same-diagonal dependency through shuffles with no slack,
// and needs the previous diagonal two steps ahead.
//
// Layout ("plane"): fp64 [s][tau][z] with z fastest (ZP doubles per (s, tau) line), zero outside
// the interior.  The 32 lanes of a warp touch 32 consecutive doubles of one (s, tau) line per
// stream per step, so every stream is one 256-byte coalesced segment, and the 15 stencil
// neighbours of the residual come from three lines (s-1, s, s+1) at tau-2..tau+2.
//
// Bands.  A CTA (PW warps) processes one band task: PW consecutive diagonals s0..s0+PW-1 of one
// 32-row chunk c.  Warp k owns diagonal s0+k and hands its values to warp k+1 through a
// shared-memory ring (data is the flag: a signalling-NaN sentinel marks an empty slot; the
// consumer re-arms the slot after reading it, the producer waits for an armed slot).  Across
// bands (the band's first diagonal needs the previous band's last one) and across chunks (lane 0
// needs row z0-1 of the chunk below) the values travel through global memory with the same
// sentinel protocol on the handoff positions only:
//   forward : W (w_f, full plane, written by the forward pass).  Handoff positions are the last
//             diagonal of every band and the rows z = 0 mod 32.  The backward pass reads w_f and
//             re-arms those positions.
//   backward: B (w_b, handoff positions only: the first diagonal of every band and the rows
//             z = 1 mod 32, z > 32).  The forward pass re-arms them.
// Persistent CTAs take band tasks from one global ticket in a topological order (every task a
// band depends on has a smaller ticket), so a CTA only waits for tasks held by running CTAs:
// deadlock-free for any residency.
//
// Per lane the arithmetic is exactly the reference's serial sequence for its row (NDDF seed table
// in registers, marched after every point; residual in stencil_apply order; substitution in
// reference order), so the exact mode is bitwise equal to the reference; the fast mode uses FMA
// and puts the newest operand (own row) last.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "tilu_common.cuh"
#include "tilu_plan.cuh"

namespace tilu {
void prof_begin(cudaStream_t s);
void prof_end(const char *name, cudaStream_t s);

namespace pl {

constexpr int PW = 4;    // diagonals (warps) per band
constexpr int GS = 4;    // unroll factor == global handoff prefetch distance (steps)
constexpr int TG = 8;    // steps staged by one pair of TMA tensor copies
constexpr int NG = 2;    // TMA ring depth (groups of TG steps) per warp
constexpr int HR = 16;   // shared-memory handoff ring depth (steps)
constexpr int WIN = 34;  // doubles per staged line: z0-1 .. z0+32
// one staged group: forward u box [3 planes s-1..s+1][TG+2 lines][WIN] + f box [TG][WIN];
// backward w_f box [TG][WIN] + u box [TG][WIN]
// (tensor copies need 128-byte aligned shared-memory destinations)
constexpr int FOFF = (3 * (TG + 2) * WIN * 8 + 127) / 128 * 128 / 8;  // doubles: f box offset in a slot
constexpr int SLOT = (FOFF * 8 + TG * WIN * 8 + 127) / 128 * 128;
constexpr int TR = 4 + 3 * PW;  // trace record: start ns, end ns, sm, cta, per warp: cycles total / slow path / waits
constexpr long long kSentP = 0x7FF4DEADBEEF0002ll;  // signalling NaN: "not produced yet"

struct Geo {
    int n, TP, ZP;
};
__host__ __device__ __forceinline__ int64_t pidx(const Geo &g, int s, int tau, int z)
{
    return ((int64_t)s * g.TP + tau) * g.ZP + z;
}
__host__ inline Geo make_geo(int n)
{
    const int nch = std::max(1, (n - 3 + 31) / 32);
    return Geo{n, n + 40, 32 * nch + 4};
}
__host__ inline int64_t plane_elems(const Geo &g) { return (int64_t)(g.n + 1) * g.TP * g.ZP; }

// TMA tensor maps over the planes ([s][tau][z], z fastest; out-of-range boxes are zero-filled):
// u3 = u, box (WIN, TG+2, 3); f1 = f, box (WIN, TG, 1); w1 = w_f, box (WIN, TG, 1); u1 = u, box (WIN, TG, 1).
struct Maps {
    CUtensorMap u3, f1, w1, u1;
};

struct Args {
    double *u;             // plane
    const double *f;       // plane
    double *W;             // plane: w_f (handoff positions armed with the sentinel before the forward pass)
    double *B;             // plane: w_b handoff positions (re-armed by the forward pass)
    const int *tasks;      // (b << 16) | c, topological order of the forward pass
    int ntasks;
    int *ticket;           // zeroed per pass
    double *part;          // [ntasks][PW * 32] residual partial sums (forward) or nullptr
    long long *trace;      // TILU_PLANE_TRACE: [ntasks][4] = start ns, end ns, sm id, CTA (or nullptr)
    Geo g;
    double arow[15];       // constant stencil (kernel-parameter bank)
};

// ---- small PTX helpers ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mb_expect(uint64_t *b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(b))
        : "memory");
}
__device__ __forceinline__ double sentv() { return __longlong_as_double(kSentP); }
__device__ __forceinline__ bool is_sent(double v) { return __double_as_longlong(v) == kSentP; }
__device__ __forceinline__ double lds_vol(const double *p)
{
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(su32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void sts(double *p, double v)
{
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(su32(p)), "d"(v) : "memory");
}
__device__ __forceinline__ double ldg_cg(const double *p) { return __ldcg(p); }
__device__ __forceinline__ long long gtimer()
{
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int smid()
{
    int v;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
    return v;
}

// Warp-uniform wait until no lane holds the sentinel (global value re-read from L2).  A dependency
// bug must fail loudly instead of hanging the device: trap after ~2^26 re-reads.
__device__ __forceinline__ void ready_g(double &v, const double *p, bool mine)
{
    long long spins = 0;
    while (__any_sync(0xffffffffu, mine && is_sent(v))) {
        __nanosleep(40);
        if (mine) v = ldg_cg(p);
        if (++spins > (1ll << 26)) __trap();
    }
}
// Shared-memory handoff: take the value of slot p (wait until produced), re-arm the slot.
__device__ __forceinline__ double take_s(double *p)
{
    double v = lds_vol(p);
    long long spins = 0;
    while (__any_sync(0xffffffffu, is_sent(v))) {
        v = lds_vol(p);
        if (++spins > (1ll << 28)) __trap();
    }
    sts(p, sentv());
    return v;
}
__device__ __forceinline__ void put_s(double *p, double v)
{
    long long spins = 0;
    while (__any_sync(0xffffffffu, !is_sent(lds_vol(p)))) {
        if (++spins > (1ll << 28)) __trap();
    }
    sts(p, v);
}

__device__ __forceinline__ bool band_pt(int x, int y, int z, int xe) { return z == 1 || y == 1 || x == 1 || x == xe; }
__device__ __forceinline__ int band_off(int x, int y, int z) { return (z == 1 || y == 1) ? x - 1 : (x == 1 ? 0 : 1); }

// Shared memory of one CTA.
struct Smem {
    alignas(128) unsigned char tbuf[PW][NG][SLOT];  // TMA ring (groups of TG steps)
    double hring[PW][HR][32];                       // handoff ring k: written by warp k-1, read by warp k
    uint64_t mbar[PW][NG];
    int task;
};

// Predicated global load (no branch): v = p ? *ptr : other.
__device__ __forceinline__ double ld_if(bool p, const double *ptr, double other)
{
    double v = other;
    asm("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q ld.global.nc.f64 %0, [%1];\n}" : "+d"(v) : "l"(ptr), "r"((int)p));
    return v;
}

// Forward substitution of one point: reference order w s se bnw bn bc be (_kernels.py:350-364), or
// (fast) FMA with the newest operands (own row, same-diagonal lane) last.
template <bool EXACT>
__device__ __forceinline__ double fwd_chain(double r, const double (&L)[7], double w1, double p1, double p0, double lw2,
                                            double lw1, double lp2, double lp1)
{
    double acc = r;
    if (EXACT) {
        acc = msub<true>(acc, L[0], w1);
        acc = msub<true>(acc, L[1], p1);
        acc = msub<true>(acc, L[2], p0);
        acc = msub<true>(acc, L[3], lw2);
        acc = msub<true>(acc, L[4], lw1);
        acc = msub<true>(acc, L[5], lp2);
        acc = msub<true>(acc, L[6], lp1);
    } else {
        acc = msub<false>(acc, L[1], p1);
        acc = msub<false>(acc, L[3], lw2);
        acc = msub<false>(acc, L[5], lp2);
        acc = msub<false>(acc, L[6], lp1);
        acc = msub<false>(acc, L[2], p0);
        acc = msub<false>(acc, L[4], lw1);
        acc = msub<false>(acc, L[0], w1);
    }
    return acc;
}
template <bool EXACT>
__device__ __forceinline__ double bwd_chain(double inv_d, double wf, const double (&Lq)[7], double wb1, double q1,
                                            double q0, double lw2, double lw1, double lq2, double lq1)
{
    double acc = EXACT ? dmul(inv_d, wf) : inv_d * wf;
    if (EXACT) {  // reference order (_kernels.py:416-428)
        acc = msub<true>(acc, Lq[0], wb1);
        acc = msub<true>(acc, Lq[1], q1);
        acc = msub<true>(acc, Lq[2], q0);
        acc = msub<true>(acc, Lq[3], lw2);
        acc = msub<true>(acc, Lq[4], lw1);
        acc = msub<true>(acc, Lq[5], lq2);
        acc = msub<true>(acc, Lq[6], lq1);
    } else {
        acc = msub<false>(acc, Lq[1], q1);
        acc = msub<false>(acc, Lq[3], lw2);
        acc = msub<false>(acc, Lq[5], lq2);
        acc = msub<false>(acc, Lq[6], lq1);
        acc = msub<false>(acc, Lq[2], q0);
        acc = msub<false>(acc, Lq[4], lw1);
        acc = msub<false>(acc, Lq[0], wb1);
    }
    return acc;
}

__device__ __forceinline__ void init_smem(Smem &S)
{
    for (int i = threadIdx.x; i < PW * HR * 32; i += blockDim.x) (&S.hring[0][0][0])[i] = sentv();
    if (threadIdx.x < PW * NG) mb_init(&S.mbar[0][0] + threadIdx.x, 1);
    mb_fence_init();
    __syncthreads();
}

// ------------------------------------------------------------------------------------------------
// Forward pass: residual r = f - A u, forward L substitution (unit lower), w_f = result.
//
// Iteration sg (= "sigma") computes the residual of step sg (staged lines of step sg) and the
// substitution of step tau = sg - 1, whose residual was computed one iteration earlier: the
// 15-term residual chain is off the substitution's critical path.  The inputs produced by other
// warps are taken speculatively (one volatile shared load / one prefetched global load issued at
// the top of the iteration) and validated once at the end; only a value that was still the
// sentinel sends the warp through the slow (polling) path.
// ------------------------------------------------------------------------------------------------
template <int K, bool EXACT, bool CONST_ROW>
__global__ void __launch_bounds__(PW * 32, 1) k_plane_fwd(const PlanDev P, const Args A, const __grid_constant__ Maps M)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    init_smem(S);
    const Geo g = A.g;
    const int n = P.n, ZP = g.ZP;
    uint32_t gcon = 0, giss = 0;  // TMA groups consumed / issued by this warp (all tasks)
    for (;;) {
        if (threadIdx.x == 0) S.task = atomicAdd(A.ticket, 1);
        __syncthreads();
        const int t = S.task;
        if (t >= A.ntasks) break;
        const int code = A.tasks[t];
        const int b = code >> 16, c = code & 0xffff;
        if (A.trace && threadIdx.x == 0) A.trace[TR * (int64_t)t] = gtimer();
        const int s0 = 2 + PW * b, z0 = 1 + 32 * c;
        const int s = s0 + warp, z = z0 + lane, y = s - z;
        const int xe = n - 1 - s, xe0 = n - 1 - s0;
        // from tau = z0-3: lane 0's first point (tau = z0+1) reads u(s, tau-1, z0-1), staged at step tau-3
        const int T0 = z0 - 3, T1 = z0 + 32 + xe0;
        const bool wlive = (s <= n - 2) && (z0 <= s - 1);
        const bool live = wlive && (z <= s - 1);
        double r2 = 0.0;
        double *hin = &S.hring[warp][0][0];
        double *hout = (warp + 1 < PW) ? &S.hring[warp + 1][0][0] : nullptr;
        auto hs = [](int tau) { return ((tau + HR) % HR) * 32; };
        if (!wlive) {
            // no rows here: pass zeros down the band (the neighbour values are boundary values)
            for (int tau = T0; tau <= T1; ++tau) {
                if (warp > 0 && tau <= T1 - 1) (void)take_s(hin + hs(tau + 1) + lane);
                if (hout && tau >= T0 + 1) put_s(hout + hs(tau) + lane, 0.0);
            }
        } else {
            // ---- per-row state -------------------------------------------------------------
            double d[7][K];
            int boff = 0;
            int64_t rbase = 0;
            if (live) {
                const int r = row_id(n, z, y);
                const double *sd = P.seedF + (int64_t)r * 7 * K;
#pragma unroll
                for (int m = 0; m < 7; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = sd[m * K + j];
                if (P.variant == 1) boff = P.bandoff[r];
                rbase = P.rowbase[r];
            } else {
#pragma unroll
                for (int m = 0; m < 7; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = 0.0;
            }
            // ---- TMA groups: group q stages steps sg = T0 + TG q .. + TG-1: one u box (planes s-1..s+1,
            // lines sg0+1 .. sg0+TG+2) and one f box (lines sg0 .. sg0+TG-1) --------------------------
            uint64_t *mb = S.mbar[warp];
            const int ngroups = (T1 - T0) / TG + 1;
            auto issue = [&](int q) {  // lane 0
                const int sl = giss % NG;
                const int sg0 = T0 + TG * q;
                double *tb = reinterpret_cast<double *>(S.tbuf[warp][sl]);
                mb_expect(&mb[sl], (3 * (TG + 2) + TG) * WIN * 8);
                tma3(tb, &M.u3, z0 - 1, sg0 + 1, s - 1, &mb[sl]);
                tma3(tb + FOFF, &M.f1, z0 - 1, sg0, s, &mb[sl]);
                ++giss;
            };
            if (lane == 0)
                for (int q = 0; q < ngroups && q < NG; ++q) issue(q);
            // ---- global handoff inputs, prefetched GS chain steps ahead ---------------------
            // warp 0: P(tau+1) = w_f(s-1, tau+1, z); lane 0: ga = w_f(s, tau-1, z0-1), gb = w_f(s-1, tau, z0-1)
            const double *pw0 = A.W + pidx(g, s - 1, 0, z);
            const double *pga = A.W + pidx(g, s, 0, z0 - 1);
            const double *pgb = A.W + pidx(g, s - 1, 0, z0 - 1);
            const bool gp_on = (warp == 0), gl_on = (lane == 0);
            double gp[GS], ga[GS], gb[GS];
#pragma unroll
            for (int j = 0; j < GS; ++j) {
                const int tau = T0 + j;
                gp[j] = (gp_on && tau + 1 >= 0) ? ldg_cg(pw0 + (int64_t)(tau + 1) * ZP) : 0.0;
                ga[j] = (gl_on && tau - 1 >= 0) ? ldg_cg(pga + (int64_t)(tau - 1) * ZP) : 0.0;
                gb[j] = (gl_on && tau >= 0) ? ldg_cg(pgb + (int64_t)tau * ZP) : 0.0;
            }
            // ---- sliding windows (residual of step sg) ----------------------------------------
            double al0 = 0, al1 = 0, al2 = 0, al3 = 0, al4 = 0;  // u(s, sg+2-j, z-1)
            double am0 = 0, am1 = 0, am2 = 0, am3 = 0;           // u(s, sg+2-j, z)
            double ah0 = 0, ah1 = 0;                             // u(s, sg+2-j, z+1)
            double bl0 = 0, bl1 = 0, bl2 = 0;                    // u(s-1, sg+1-j, z-1)
            double bm0 = 0, bm1 = 0;                             // u(s-1, sg+1-j, z)
            double cm0 = 0, cm1 = 0, cm2 = 0;                    // u(s+1, sg+1-j, z)
            double ch0 = 0, ch1 = 0;                             // u(s+1, sg+1-j, z+1)
            double rr_cur = 0.0;                                 // residual of the chain step
            double w1 = 0, w2 = 0;                               // own w_f at tau-1, tau-2
            double p1 = 0, p2 = 0;                               // w_f(s-1, tau, z), (s-1, tau-1, z)
            double ga_prev = 0, gb_prev = 0;
            long long cyc_slow = 0, cyc_wait = 0;
            const bool rearm_b = live && (warp == 0 || (lane == 0 && z0 > 32));
            const int i = lane + 1;
            auto step = [&](const int sg, const int j) {
                const int tau = sg - 1;
                const int jc = (j + GS - 1) % GS;  // prefetch slot of chain step tau
                const bool res_on = sg <= T1, chain_on = tau >= T0;
                const bool p_on = chain_on && tau <= T1 - 1;
                // (0) once per group: staged lines ready; the producer's next GS ring slots armed
                const long long cw0 = A.trace ? clock64() : 0;
                if (j == 0) {
                    if (res_on && (sg - T0) % TG == 0) mb_wait(&mb[gcon % NG], (gcon / NG) & 1);
                    if (hout) {
                        long long spins = 0;
                        for (;;) {
                            bool busy = false;
#pragma unroll
                            for (int k = 0; k < GS; ++k) {
                                const int tt = tau + k;
                                if (tt >= T0 + 1 && tt <= T1) busy |= !is_sent(lds_vol(hout + hs(tt) + lane));
                            }
                            if (!__any_sync(0xffffffffu, busy)) break;
                            if (++spins > (1ll << 28)) __trap();
                        }
                    }
                }
                if (A.trace) cyc_wait += clock64() - cw0;
                // (1) chain inputs, taken speculatively
                double p0 = 0.0;
                if (p_on) p0 = (warp == 0) ? gp[jc] : lds_vol(hin + hs(tau + 1) + lane);
                double ga_cur = ga[jc], gb_cur = gb[jc];
                double lw1 = __shfl_up_sync(0xffffffffu, w1, 1);
                double lw2 = __shfl_up_sync(0xffffffffu, w2, 1);
                double lp1 = __shfl_up_sync(0xffffffffu, p1, 1);
                double lp2 = __shfl_up_sync(0xffffffffu, p2, 1);
                if (lane == 0) {
                    lw1 = ga_cur; lw2 = ga_prev; lp1 = gb_cur; lp2 = gb_prev;
                }
                const int x = tau - z;
                const bool vpt = chain_on && live && x >= 1 && x <= xe;
                double L[7];
                {
                    const bool isb = (P.variant == 1) && vpt && band_pt(x, y, z, xe);
                    const double *st = P.store + 9 * (int64_t)(boff + band_off(x, y, z));
#pragma unroll
                    for (int m = 0; m < 7; ++m) L[m] = ld_if(isb, st + m, d[m][0]);
                }
                // (2) residual of step sg (independent of the chain)
                double rr_next = 0.0;
                if (res_on) {
                    const int k = (sg - T0) % TG;
                    const double *tb = reinterpret_cast<const double *>(S.tbuf[warp][gcon % NG]);
                    const double *la = tb + ((TG + 2) + k + 1) * WIN;      // u(s, sg+2)
                    const double *lb = tb + k * WIN;                       // u(s-1, sg+1)
                    const double *lc = tb + (2 * (TG + 2) + k) * WIN;      // u(s+1, sg+1)
                    const double *lf = tb + FOFF + k * WIN;                // f(s, sg)
                    al4 = al3; al3 = al2; al2 = al1; al1 = al0; al0 = la[i - 1];
                    am3 = am2; am2 = am1; am1 = am0; am0 = la[i];
                    ah1 = ah0; ah0 = la[i + 1];
                    bl2 = bl1; bl1 = bl0; bl0 = lb[i - 1];
                    bm1 = bm0; bm0 = lb[i];
                    cm2 = cm1; cm1 = cm0; cm0 = lc[i];
                    ch1 = ch0; ch0 = lc[i + 1];
                    const double fv = lf[i];
                    const int xs = sg - z;
                    if (live && xs >= 1 && xs <= xe) {
                        double a[15];
                        if (CONST_ROW) {
#pragma unroll
                            for (int q = 0; q < 15; ++q) a[q] = A.arow[q];
                        } else {
                            const double *ar = P.arows + 15 * (rbase + xs);
#pragma unroll
                            for (int q = 0; q < 15; ++q) a[q] = ar[q];
                        }
                        // stencil_apply order (_kernels.py:243-267): c, w s se bnw bn bc be, e n nw tse ts tc tw
                        double out = EXACT ? dmul(a[7], am2) : a[7] * am2;
                        out = madd<EXACT>(out, a[0], am3);
                        out = madd<EXACT>(out, a[1], bm1);
                        out = madd<EXACT>(out, a[2], bm0);
                        out = madd<EXACT>(out, a[3], al4);
                        out = madd<EXACT>(out, a[4], al3);
                        out = madd<EXACT>(out, a[5], bl2);
                        out = madd<EXACT>(out, a[6], bl1);
                        out = madd<EXACT>(out, a[8], am1);
                        out = madd<EXACT>(out, a[9], cm1);
                        out = madd<EXACT>(out, a[10], cm2);
                        out = madd<EXACT>(out, a[11], ah0);
                        out = madd<EXACT>(out, a[12], ah1);
                        out = madd<EXACT>(out, a[13], ch0);
                        out = madd<EXACT>(out, a[14], ch1);
                        rr_next = dsub(fv, out);
                        r2 = fma(rr_next, rr_next, r2);
                    }
                }
                // (3) substitution of step tau
                double acc = fwd_chain<EXACT>(rr_cur, L, w1, p1, p0, lw2, lw1, lp2, lp1);
                // (4) validate the speculative inputs
                const bool bad = p_on && (is_sent(p0) || (gl_on && (is_sent(ga_cur) || is_sent(gb_cur))));
                if (__any_sync(0xffffffffu, bad)) {
                    const long long cs0 = A.trace ? clock64() : 0;
                    long long spins = 0;
                    for (;;) {
                        if (p_on && is_sent(p0)) p0 = (warp == 0) ? ldg_cg(pw0 + (int64_t)(tau + 1) * ZP)
                                                                  : lds_vol(hin + hs(tau + 1) + lane);
                        if (gl_on && p_on) {
                            if (is_sent(ga_cur)) ga_cur = ldg_cg(pga + (int64_t)(tau - 1) * ZP);
                            if (is_sent(gb_cur)) gb_cur = ldg_cg(pgb + (int64_t)tau * ZP);
                        }
                        const bool still = p_on && (is_sent(p0) || (gl_on && (is_sent(ga_cur) || is_sent(gb_cur))));
                        if (!__any_sync(0xffffffffu, still)) break;
                        __nanosleep(32);
                        if (++spins > (1ll << 26)) __trap();
                    }
                    if (lane == 0) {
                        lw1 = ga_cur; lp1 = gb_cur;
                    }
                    acc = fwd_chain<EXACT>(rr_cur, L, w1, p1, p0, lw2, lw1, lp2, lp1);
                    if (A.trace) cyc_slow += clock64() - cs0;
                }
                const double wnew = vpt ? acc : 0.0;
                // (5) publish
                if (p_on && warp > 0) sts(hin + hs(tau + 1) + lane, sentv());   // re-arm the consumed slot
                if (hout && chain_on && tau >= T0 + 1) sts(hout + hs(tau) + lane, wnew);
                if (vpt) {
                    const int64_t pi = pidx(g, s, tau, z);
                    A.W[pi] = wnew;
                    if (rearm_b) A.B[pi] = sentv();
#pragma unroll
                    for (int m = 0; m < 7; ++m) march<K>(d[m]);
                }
                if (chain_on) {
                    ga_prev = ga_cur; gb_prev = gb_cur;
                    w2 = w1; w1 = wnew;
                    p2 = p1; p1 = p0;
                    // prefetch the global inputs of chain step tau + GS
                    const int tn = tau + GS;
                    if (gp_on) gp[jc] = ldg_cg(pw0 + (int64_t)(tn + 1) * ZP);
                    if (gl_on) {
                        ga[jc] = ldg_cg(pga + (int64_t)(tn - 1) * ZP);
                        gb[jc] = ldg_cg(pgb + (int64_t)tn * ZP);
                    }
                }
                rr_cur = rr_next;
                // (6) end of a staged group: release the slot, stage group + NG
                if (res_on && ((sg - T0) % TG == TG - 1 || sg == T1)) {
                    __syncwarp();
                    const int q = (sg - T0) / TG;
                    ++gcon;
                    if (lane == 0 && q + NG < ngroups) issue(q + NG);
                }
            };
            const long long ct0 = A.trace ? clock64() : 0;
            for (int sg0 = T0; sg0 <= T1 + 1; sg0 += GS) {
#pragma unroll
                for (int j = 0; j < GS; ++j)
                    if (sg0 + j <= T1 + 1) step(sg0 + j, j);
            }
            if (A.trace && lane == 0) {
                long long *tr = A.trace + TR * (int64_t)t + 4 + 3 * warp;
                tr[0] = clock64() - ct0;
                tr[1] = cyc_slow;
                tr[2] = cyc_wait;
            }
        }
        if (A.part) A.part[(int64_t)t * (PW * 32) + threadIdx.x] = r2;
        __syncthreads();
        if (A.trace && threadIdx.x == 0) {
            A.trace[TR * (int64_t)t + 1] = gtimer();
            A.trace[TR * (int64_t)t + 2] = smid();
            A.trace[TR * (int64_t)t + 3] = blockIdx.x;
        }
    }
}

// ------------------------------------------------------------------------------------------------
// Backward pass: D^{-1} scaling + L^T substitution (descending), fused u += w (multigrid.py:429).
// ------------------------------------------------------------------------------------------------
template <int K, bool EXACT>
__global__ void __launch_bounds__(PW * 32, 1) k_plane_bwd(const PlanDev P, const Args A, const __grid_constant__ Maps M)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    init_smem(S);
    const Geo g = A.g;
    const int n = P.n, ZP = g.ZP;
    uint32_t gcon = 0, giss = 0;
    for (;;) {
        if (threadIdx.x == 0) S.task = atomicAdd(A.ticket, 1);
        __syncthreads();
        const int t = S.task;
        if (t >= A.ntasks) break;
        const int code = A.tasks[A.ntasks - 1 - t];
        const int b = code >> 16, c = code & 0xffff;
        if (A.trace && threadIdx.x == 0) A.trace[TR * (int64_t)t] = gtimer();
        const int s0 = 2 + PW * b, z0 = 1 + 32 * c;
        const int s = s0 + PW - 1 - warp, z = z0 + lane, y = s - z;
        const int xe = n - 1 - s, xe0 = n - 1 - s0;
        const int T0 = z0 - 1, T1 = z0 + 32 + xe0;  // loop tau = T1 .. T0-1 (descending)
        const bool wlive = (s <= n - 2) && (z0 <= s - 1);
        const bool live = wlive && (z <= s - 1);
        double *hin = &S.hring[warp][0][0];
        double *hout = (warp + 1 < PW) ? &S.hring[warp + 1][0][0] : nullptr;
        auto hs = [](int tau) { return ((tau + HR) % HR) * 32; };
        if (!wlive) {
            for (int tau = T1; tau >= T0 - 1; --tau) {
                if (warp > 0 && tau >= T0) (void)take_s(hin + hs(tau - 1) + lane);
                if (hout && tau <= T1 - 1) put_s(hout + hs(tau) + lane, 0.0);
            }
        } else {
            double d[8][K];
            int bo_own = 0, bo_n = 0, bo_ts = 0, bo_tc = 0;
            if (live) {
                const int r = row_id(n, z, y);
                const double *sd = P.seedB + (int64_t)r * 8 * K;
#pragma unroll
                for (int m = 0; m < 8; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = sd[m * K + j];
                if (P.variant == 1) {
                    bo_own = P.bandoff[r];
                    if (s + 1 <= n - 2) {
                        bo_n = P.bandoff[row_id(n, z, y + 1)];
                        bo_tc = P.bandoff[row_id(n, z + 1, y)];
                    }
                    if (y >= 2) bo_ts = P.bandoff[row_id(n, z + 1, y - 1)];
                }
            } else {
#pragma unroll
                for (int m = 0; m < 8; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = 0.0;
            }
            uint64_t *mb = S.mbar[warp];
            // group q stages tau = T1 - TG q down to T1 - TG q - (TG-1): w_f and u boxes of TG lines
            const int ngroups = (T1 - (T0 - 1)) / TG + 1;
            auto issue = [&](int q) {
                const int sl = giss % NG;
                const int lo = T1 - TG * q - (TG - 1);
                double *tb = reinterpret_cast<double *>(S.tbuf[warp][sl]);
                mb_expect(&mb[sl], 2 * TG * WIN * 8);
                tma3(tb, &M.w1, z0 - 1, lo, s, &mb[sl]);
                tma3(tb + TG * WIN, &M.u1, z0 - 1, lo, s, &mb[sl]);
                ++giss;
            };
            if (lane == 0)
                for (int q = 0; q < ngroups && q < NG; ++q) issue(q);
            // warp 0: P'(tau-1) = w_b(s+1, tau-1, z); lane 31: ga = w_b(s, tau+1, z0+32), gb = w_b(s+1, tau, z0+32)
            const double *pw0 = A.B + pidx(g, s + 1, 0, z);
            const double *pga = A.B + pidx(g, s, 0, z0 + 32);
            const double *pgb = A.B + pidx(g, s + 1, 0, z0 + 32);
            const bool gp_on = (warp == 0), gl_on = (lane == 31);
            double gp[GS], ga[GS], gb[GS];
#pragma unroll
            for (int j = 0; j < GS; ++j) {
                const int tau = T1 - j;
                gp[j] = (gp_on && tau - 1 >= 0) ? ldg_cg(pw0 + (int64_t)(tau - 1) * ZP) : 0.0;
                ga[j] = gl_on ? ldg_cg(pga + (int64_t)(tau + 1) * ZP) : 0.0;
                gb[j] = gl_on ? ldg_cg(pgb + (int64_t)tau * ZP) : 0.0;
            }
            double wb1 = 0, wb2 = 0;  // own w_b at tau+1, tau+2
            double q1 = 0, q2 = 0;    // w_b(s+1, tau, z), (s+1, tau+1, z)
            double ga_prev = 0, gb_prev = 0;
            long long cyc_slow = 0, cyc_wait = 0;
            const bool b_out = live && (warp == PW - 1 || (lane == 0 && z0 > 32));
            const bool rearm_w = live && (warp == 0 || lane == 31);
            const int i = lane + 1;
            auto step = [&](const int tau, const int j) {
                const bool q_on = tau >= T0;
                const long long cw0 = A.trace ? clock64() : 0;
                if (j == 0) {
                    if ((T1 - tau) % TG == 0) mb_wait(&mb[gcon % NG], (gcon / NG) & 1);
                    if (hout) {
                        long long spins = 0;
                        for (;;) {
                            bool busy = false;
#pragma unroll
                            for (int k = 0; k < GS; ++k) {
                                const int tt = tau - k;
                                if (tt <= T1 - 1 && tt >= T0 - 1) busy |= !is_sent(lds_vol(hout + hs(tt) + lane));
                            }
                            if (!__any_sync(0xffffffffu, busy)) break;
                            if (++spins > (1ll << 28)) __trap();
                        }
                    }
                }
                if (A.trace) cyc_wait += clock64() - cw0;
                double q0 = 0.0;
                if (q_on) q0 = (warp == 0) ? gp[j] : lds_vol(hin + hs(tau - 1) + lane);
                double ga_cur = ga[j], gb_cur = gb[j];
                double lw1 = __shfl_down_sync(0xffffffffu, wb1, 1);
                double lw2 = __shfl_down_sync(0xffffffffu, wb2, 1);
                double lq1 = __shfl_down_sync(0xffffffffu, q1, 1);
                double lq2 = __shfl_down_sync(0xffffffffu, q2, 1);
                if (lane == 31) {
                    lw1 = ga_cur; lw2 = ga_prev; lq1 = gb_cur; lq2 = gb_prev;
                }
                const int x = tau - z;
                const bool vpt = live && x >= 1 && x <= xe;
                double wfv, uv;
                {
                    const int k = TG - 1 - (T1 - tau) % TG;  // line of tau in the group's boxes
                    const double *tb = reinterpret_cast<const double *>(S.tbuf[warp][gcon % NG]);
                    wfv = tb[k * WIN + i];
                    uv = tb[(TG + k) * WIN + i];
                }
                // L at the seven source points q_m = p - d_m (_lq, _kernels.py:434-441) and 1/D at p
                double Lq[7], inv_d;
                {
                    const bool v1 = P.variant == 1 && vpt;
                    const bool i0 = x + 1 <= xe, i1 = x <= xe - 1, i2 = x >= 2, i3 = y >= 2 && x + 1 <= xe,
                               i4 = y >= 2, i5 = x <= xe - 1, i6 = x >= 2;
                    const bool b0 = v1 && i0 && (x + 1 == xe || y == 1 || z == 1);
                    const bool b1 = v1 && i1 && (x == 1 || x == xe - 1 || z == 1);
                    const bool b2 = v1 && i2 && (x - 1 == 1 || x - 1 == xe - 1 || z == 1);
                    const bool b3 = v1 && i3 && (x + 1 == xe || y == 2);
                    const bool b4 = v1 && i4 && (x == 1 || x == xe || y == 2);
                    const bool b5 = v1 && i5 && (x == 1 || x == xe - 1 || y == 1);
                    const bool b6 = v1 && i6 && (x - 1 == 1 || x - 1 == xe - 1 || y == 1);
                    const bool bd = v1 && (x == 1 || x == xe || y == 1 || z == 1);
                    const double *st = P.store;
                    const int o0 = bo_own + ((z == 1 || y == 1) ? x : 1);
                    const int o1 = bo_n + ((z == 1) ? x - 1 : (x == 1 ? 0 : 1));
                    const int o2 = bo_n + ((z == 1) ? x - 2 : (x - 1 == 1 ? 0 : 1));
                    const int o3 = bo_ts + ((y == 2) ? x : 1);
                    const int o4 = bo_ts + ((y == 2) ? x - 1 : (x == 1 ? 0 : 1));
                    const int o5 = bo_tc + ((y == 1) ? x - 1 : (x == 1 ? 0 : 1));
                    const int o6 = bo_tc + ((y == 1) ? x - 2 : (x - 1 == 1 ? 0 : 1));
                    const int od = bo_own + band_off(x, y, z);
                    Lq[0] = i0 ? ld_if(b0, st + 9 * (int64_t)o0 + 0, d[0][0]) : 0.0;
                    Lq[1] = i1 ? ld_if(b1, st + 9 * (int64_t)o1 + 1, d[1][0]) : 0.0;
                    Lq[2] = i2 ? ld_if(b2, st + 9 * (int64_t)o2 + 2, d[2][0]) : 0.0;
                    Lq[3] = i3 ? ld_if(b3, st + 9 * (int64_t)o3 + 3, d[3][0]) : 0.0;
                    Lq[4] = i4 ? ld_if(b4, st + 9 * (int64_t)o4 + 4, d[4][0]) : 0.0;
                    Lq[5] = i5 ? ld_if(b5, st + 9 * (int64_t)o5 + 5, d[5][0]) : 0.0;
                    Lq[6] = i6 ? ld_if(b6, st + 9 * (int64_t)o6 + 6, d[6][0]) : 0.0;
                    inv_d = ld_if(bd, st + 9 * (int64_t)od + 8, d[7][0]);
                }
                double acc = bwd_chain<EXACT>(inv_d, wfv, Lq, wb1, q1, q0, lw2, lw1, lq2, lq1);
                const bool bad = (q_on && is_sent(q0)) || (gl_on && (is_sent(ga_cur) || is_sent(gb_cur)));
                if (__any_sync(0xffffffffu, bad)) {
                    const long long cs0 = A.trace ? clock64() : 0;
                    long long spins = 0;
                    for (;;) {
                        if (q_on && is_sent(q0)) q0 = (warp == 0) ? ldg_cg(pw0 + (int64_t)(tau - 1) * ZP)
                                                                  : lds_vol(hin + hs(tau - 1) + lane);
                        if (gl_on) {
                            if (is_sent(ga_cur)) ga_cur = ldg_cg(pga + (int64_t)(tau + 1) * ZP);
                            if (is_sent(gb_cur)) gb_cur = ldg_cg(pgb + (int64_t)tau * ZP);
                        }
                        const bool still = (q_on && is_sent(q0)) || (gl_on && (is_sent(ga_cur) || is_sent(gb_cur)));
                        if (!__any_sync(0xffffffffu, still)) break;
                        __nanosleep(32);
                        if (++spins > (1ll << 26)) __trap();
                    }
                    if (lane == 31) {
                        lw1 = ga_cur; lq1 = gb_cur;
                    }
                    acc = bwd_chain<EXACT>(inv_d, wfv, Lq, wb1, q1, q0, lw2, lw1, lq2, lq1);
                    if (A.trace) cyc_slow += clock64() - cs0;
                }
                const double wnew = vpt ? acc : 0.0;
                if (q_on && warp > 0) sts(hin + hs(tau - 1) + lane, sentv());
                if (hout && tau <= T1 - 1) sts(hout + hs(tau) + lane, wnew);
                if (vpt) {
                    const int64_t pi = pidx(g, s, tau, z);
                    A.u[pi] = dadd(uv, acc);
                    if (b_out) A.B[pi] = acc;
                    if (rearm_w) A.W[pi] = sentv();
#pragma unroll
                    for (int m = 0; m < 8; ++m) march<K>(d[m]);
                }
                ga_prev = ga_cur; gb_prev = gb_cur;
                wb2 = wb1; wb1 = wnew;
                q2 = q1; q1 = q0;
                const int tn = tau - GS;
                if (gp_on) gp[j] = (tn - 1 >= 0) ? ldg_cg(pw0 + (int64_t)(tn - 1) * ZP) : 0.0;
                if (gl_on) {
                    ga[j] = (tn + 1 >= 0) ? ldg_cg(pga + (int64_t)(tn + 1) * ZP) : 0.0;
                    gb[j] = (tn >= 0) ? ldg_cg(pgb + (int64_t)tn * ZP) : 0.0;
                }
                if ((T1 - tau) % TG == TG - 1 || tau == T0 - 1) {
                    __syncwarp();
                    const int q = (T1 - tau) / TG;
                    ++gcon;
                    if (lane == 0 && q + NG < ngroups) issue(q + NG);
                }
            };
            const long long ct0 = A.trace ? clock64() : 0;
            for (int t0 = T1; t0 >= T0 - 1; t0 -= GS) {
#pragma unroll
                for (int j = 0; j < GS; ++j)
                    if (t0 - j >= T0 - 1) step(t0 - j, j);
            }
            if (A.trace && lane == 0) {
                long long *tr = A.trace + TR * (int64_t)t + 4 + 3 * warp;
                tr[0] = clock64() - ct0;
                tr[1] = cyc_slow;
                tr[2] = cyc_wait;
            }
        }
        __syncthreads();
        if (A.trace && threadIdx.x == 0) {
            A.trace[TR * (int64_t)t + 1] = gtimer();
            A.trace[TR * (int64_t)t + 2] = smid();
            A.trace[TR * (int64_t)t + 3] = blockIdx.x;
        }
    }
}

// ------------------------------------------------------------------------------------------------
// Layout conversion, arming, norms.
// ------------------------------------------------------------------------------------------------
// One CTA per interior row (z, y); threads over x.
__global__ void k_plane_pack(const PlanDev P, Geo g, const double *__restrict__ src, double *__restrict__ dst)
{
    const RowInfo ri = P.rows[blockIdx.x];
    const int64_t base = P.rowbase[blockIdx.x];
    const int s = ri.y + ri.z;
    for (int x = 1 + threadIdx.x; x <= ri.xe; x += blockDim.x) dst[pidx(g, s, x + ri.z, ri.z)] = src[base + x];
}
__global__ void k_plane_unpack(const PlanDev P, Geo g, const double *__restrict__ src, double *__restrict__ dst)
{
    const RowInfo ri = P.rows[blockIdx.x];
    const int64_t base = P.rowbase[blockIdx.x];
    const int s = ri.y + ri.z;
    for (int x = 1 + threadIdx.x; x <= ri.xe; x += blockDim.x) dst[base + x] = src[pidx(g, s, x + ri.z, ri.z)];
}
// Arm the forward handoff positions of W: last diagonal of every band, rows z = 0 mod 32.
__global__ void k_plane_arm(const PlanDev P, Geo g, double *__restrict__ W)
{
    const RowInfo ri = P.rows[blockIdx.x];
    const int s = ri.y + ri.z;
    if (!((s - 2) % PW == PW - 1 || ri.z % 32 == 0)) return;
    for (int x = 1 + threadIdx.x; x <= ri.xe; x += blockDim.x) W[pidx(g, s, x + ri.z, ri.z)] = sentv();
}
// Deterministic fixed-order sum of the per-(task, lane) partials.
__global__ void __launch_bounds__(1024) k_plane_norm(const double *__restrict__ part, int count, double *__restrict__ out)
{
    __shared__ double red[1024];
    double sacc = 0.0;
    for (int i = threadIdx.x; i < count; i += 1024) sacc += part[i];
    red[threadIdx.x] = sacc;
    __syncthreads();
    for (int k = 512; k > 0; k >>= 1) {
        if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

// ------------------------------------------------------------------------------------------------
// Host side.
// ------------------------------------------------------------------------------------------------
struct Workspace {
    Geo g;
    double *u = nullptr, *f = nullptr, *W = nullptr, *B = nullptr, *part = nullptr;
    int *tasks = nullptr, *ticket = nullptr;
    int ntasks = 0;
    int ctas = 0;
    bool armed = false;
    cudaEvent_t done = nullptr;  // end of the last call that used this workspace
    long long *trace = nullptr;  // [2][ntasks][4] (TILU_PLANE_TRACE)
    Maps maps;
};

// TMA tensor map over one plane-layout vector: dims (ZP, TP, n+1), box (WIN, box_tau, box_s).
static bool encode_map(CUtensorMap *m, double *base, const Geo &g, int box_tau, int box_s)
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return false;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    const cuuint64_t dims[3] = {(cuuint64_t)g.ZP, (cuuint64_t)g.TP, (cuuint64_t)(g.n + 1)};
    const cuuint64_t strides[2] = {(cuuint64_t)g.ZP * 8, (cuuint64_t)g.TP * g.ZP * 8};
    const cuuint32_t box[3] = {(cuuint32_t)WIN, (cuuint32_t)box_tau, (cuuint32_t)box_s};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

// Band tasks in topological order: key 18 b + 32 c (a band starts ~18 steps after the one below it,
// a chunk 32 steps after the one below it); every dependency ((b-1, c), (b-1, c-1), (b, c-1)) has a
// strictly smaller key.
static std::vector<int> make_tasks(int n)
{
    std::vector<std::pair<long long, int>> v;
    for (int b = 0;; ++b) {
        const int s0 = 2 + PW * b;
        if (s0 > n - 2) break;
        const int smax = std::min(s0 + PW - 1, n - 2);
        const int nch = (smax - 1 + 31) / 32;
        for (int c = 0; c < nch; ++c) v.push_back({(18ll * b + 32ll * c) * 65536 + c, (b << 16) | c});
    }
    std::sort(v.begin(), v.end());
    std::vector<int> out;
    for (auto &e : v) out.push_back(e.second);
    return out;
}

template <int K, bool EXACT, bool CONST_ROW>
static cudaError_t set_attrs()
{
    cudaError_t e = cudaFuncSetAttribute(k_plane_fwd<K, EXACT, CONST_ROW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(Smem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_plane_bwd<K, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
}

template <int K, bool EXACT, bool CONST_ROW>
static bool launch_k(const PlanDev &P, const Args &A, const Maps &M, int ctas, bool fwd, cudaStream_t s)
{
    static bool attrs = (set_attrs<K, EXACT, CONST_ROW>() == cudaSuccess);
    if (!attrs) return false;
    if (fwd) k_plane_fwd<K, EXACT, CONST_ROW><<<ctas, PW * 32, sizeof(Smem), s>>>(P, A, M);
    else k_plane_bwd<K, EXACT><<<ctas, PW * 32, sizeof(Smem), s>>>(P, A, M);
    return true;
}
template <bool EXACT, bool CONST_ROW>
static bool launch_e(const PlanDev &P, const Args &A, const Maps &M, int ctas, bool fwd, cudaStream_t s)
{
    switch (P.kx1) {
    case 1: return launch_k<1, EXACT, CONST_ROW>(P, A, M, ctas, fwd, s);
    case 2: return launch_k<2, EXACT, CONST_ROW>(P, A, M, ctas, fwd, s);
    case 3: return launch_k<3, EXACT, CONST_ROW>(P, A, M, ctas, fwd, s);
    case 4: return launch_k<4, EXACT, CONST_ROW>(P, A, M, ctas, fwd, s);
    case 5: return launch_k<5, EXACT, CONST_ROW>(P, A, M, ctas, fwd, s);
    case 6: return launch_k<6, EXACT, CONST_ROW>(P, A, M, ctas, fwd, s);
    default: return false;
    }
}
static bool launch_pass(const PlanDev &P, const Args &A, const Maps &M, int ctas, bool exact, bool fwd, cudaStream_t s)
{
    const bool c = P.arow != nullptr;
    if (exact) return c ? launch_e<true, true>(P, A, M, ctas, fwd, s) : launch_e<true, false>(P, A, M, ctas, fwd, s);
    return c ? launch_e<false, true>(P, A, M, ctas, fwd, s) : launch_e<false, false>(P, A, M, ctas, fwd, s);
}

static int resident_ctas(const tilu_plan *p)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const char *e = std::getenv("TILU_PLANE_CTAS_PER_SM");
    int per = e ? std::atoi(e) : 2;
    if (per < 1) per = 1;
    if (per > 4) per = 4;
    (void)p;
    return sms * per;
}

static std::mutex g_ws_mu;

static int ws_create(tilu_plan *p, Workspace **out, cudaStream_t s)
{
    Workspace *w = new Workspace();
    w->g = make_geo(p->dev.n);
    const size_t pe = (size_t)plane_elems(w->g);
    std::vector<int> tasks = make_tasks(p->dev.n);
    w->ntasks = (int)tasks.size();
    w->ctas = std::min(w->ntasks, resident_ctas(p));
    void *m = nullptr;
    const size_t bytes = 4 * pe * sizeof(double) + (size_t)w->ntasks * PW * 32 * sizeof(double) +
                         (size_t)(w->ntasks + 8) * sizeof(int);
    if (cudaMalloc(&m, bytes) != cudaSuccess) {
        cudaGetLastError();
        delete w;
        return TILU_ENOMEM;
    }
    double *d = static_cast<double *>(m);
    w->u = d;
    w->f = d + pe;
    w->W = d + 2 * pe;
    w->B = d + 3 * pe;
    w->part = d + 4 * pe;
    w->ticket = reinterpret_cast<int *>(w->part + (size_t)w->ntasks * PW * 32);
    w->tasks = w->ticket + 8;
    cudaMemsetAsync(m, 0, bytes, s);
    cudaMemcpyAsync(w->tasks, tasks.data(), tasks.size() * sizeof(int), cudaMemcpyHostToDevice, s);
    if (!encode_map(&w->maps.u3, w->u, w->g, TG + 2, 3) || !encode_map(&w->maps.f1, w->f, w->g, TG, 1) ||
        !encode_map(&w->maps.w1, w->W, w->g, TG, 1) || !encode_map(&w->maps.u1, w->u, w->g, TG, 1)) {
        cudaFree(m);
        delete w;
        return TILU_ECUDA;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess || cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming) != cudaSuccess) {
        cudaFree(m);
        delete w;
        return TILU_ECUDA;
    }
    *out = w;
    return TILU_OK;
}

}  // namespace pl

bool plane_supported(const tilu_plan *p)
{
    if (p->flags & TILU_SCHED_SIMPLE) return false;
    static const char *e = std::getenv("TILU_PLANE");
    if (e && e[0] == '0') return false;
    return p->dev.kx1 <= 6 && p->dev.level >= 3 && p->dev.level <= 10 && p->dev.seedA == nullptr &&
           (p->dev.arow != nullptr || p->dev.arows != nullptr);
}

void plane_free(void *ws)
{
    if (!ws) return;
    pl::Workspace *w = static_cast<pl::Workspace *>(ws);
    cudaFree(w->u);
    if (w->trace) cudaFree(w->trace);
    if (w->done) cudaEventDestroy(w->done);
    delete w;
}

int64_t plane_interior_points(const tilu_plan *p) { return p->interior; }

// `sweeps` smoothing steps on one macro-tet in the reference layout: pack, sweeps, unpack.
int plane_sweep(const tilu_plan *cp, double *u, const double *f, int ntets, int sweeps, double *rnorm2,
                cudaStream_t s, int *launches)
{
    using namespace pl;
    tilu_plan *p = const_cast<tilu_plan *>(cp);
    if (ntets != 1) return TILU_EUNSUPPORTED;
    // One workspace per plan (planes of u, f, w_f, w_b; the zero boundary and the armed handoff
    // positions persist between calls).  Calls from several streams are serialised on it through
    // an event, so the plan stays usable from any stream.
    std::unique_lock<std::mutex> lk(g_ws_mu);
    if (!p->plane) {
        Workspace *nw = nullptr;
        const int rc = ws_create(p, &nw, s);
        if (rc) return rc;
        p->plane = nw;
    }
    Workspace *w = static_cast<Workspace *>(p->plane);
    cudaStreamWaitEvent(s, w->done, 0);
    const PlanDev &P = p->dev;
    int nl = 0;
    int rc = TILU_OK;
    Args A{};
    A.u = w->u;
    A.f = w->f;
    A.W = w->W;
    A.B = w->B;
    A.tasks = w->tasks;
    A.ntasks = w->ntasks;
    A.g = w->g;
    std::memcpy(A.arow, p->harow, sizeof(A.arow));
    const bool exact = !(p->flags & TILU_FAST);
    static const char *trace_path = std::getenv("TILU_PLANE_TRACE");  // file: per-task timeline of the last sweep
    if (trace_path && !w->trace) cudaMalloc(&w->trace, 2 * (size_t)w->ntasks * TR * sizeof(long long));
    prof_begin(s);
    k_plane_pack<<<P.nrows, 128, 0, s>>>(P, w->g, u, w->u);
    k_plane_pack<<<P.nrows, 128, 0, s>>>(P, w->g, f, w->f);
    if (!w->armed) {
        k_plane_arm<<<P.nrows, 128, 0, s>>>(P, w->g, w->W);
        ++nl;
        w->armed = true;
    }
    prof_end("plane_pack", s);
    nl += 2;
    for (int k = 0; k < sweeps && rc == TILU_OK; ++k) {
        cudaMemsetAsync(w->ticket, 0, 2 * sizeof(int), s);
        A.ticket = w->ticket;
        A.part = rnorm2 ? w->part : nullptr;
        A.trace = w->trace;
        prof_begin(s);
        bool ok = launch_pass(P, A, w->maps, w->ctas, exact, true, s);
        prof_end("plane_fwd", s);
        A.ticket = w->ticket + 1;
        A.part = nullptr;
        A.trace = w->trace ? w->trace + (size_t)w->ntasks * TR : nullptr;
        static const char *dbg = std::getenv("TILU_PLANE_DEBUG");  // "1": forward pass only, return w_f
        if (dbg && dbg[0] == '1') {
            k_plane_unpack<<<P.nrows, 128, 0, s>>>(P, w->g, w->W, u);
            w->armed = false;
            cudaEventRecord(w->done, s);
            return ok ? TILU_OK : TILU_EUNSUPPORTED;
        }
        prof_begin(s);
        ok = ok && launch_pass(P, A, w->maps, w->ctas, exact, false, s);
        prof_end("plane_bwd", s);
        nl += 2;
        if (!ok) rc = TILU_EUNSUPPORTED;
        if (rnorm2 && ok) {
            k_plane_norm<<<1, 1024, 0, s>>>(w->part, w->ntasks * PW * 32, rnorm2 + k);
            ++nl;
        }
    }
    if (trace_path && w->trace) {
        std::vector<long long> h(2 * (size_t)w->ntasks * TR);
        std::vector<int> tk(w->ntasks);
        cudaMemcpyAsync(h.data(), w->trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(tk.data(), w->tasks, tk.size() * sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (FILE *fp = std::fopen(trace_path, "w")) {
            std::fprintf(fp, "pass ticket b c start_ns end_ns sm cta [warp: cyc_total cyc_slow cyc_wait]\n");
            for (int pass = 0; pass < 2; ++pass)
                for (int t = 0; t < w->ntasks; ++t) {
                    const long long *r = &h[((size_t)pass * w->ntasks + t) * TR];
                    const int code = tk[pass == 0 ? t : w->ntasks - 1 - t];
                    std::fprintf(fp, "%d %d %d %d", pass, t, code >> 16, code & 0xffff);
                    for (int k = 0; k < TR; ++k) std::fprintf(fp, " %lld", r[k]);
                    std::fprintf(fp, "\n");
                }
            std::fclose(fp);
        }
    }
    prof_begin(s);
    k_plane_unpack<<<P.nrows, 128, 0, s>>>(P, w->g, w->u, u);
    prof_end("plane_unpack", s);
    ++nl;
    if (cudaGetLastError() != cudaSuccess) {
        rc = TILU_ECUDA;
        w->armed = false;
    }
    cudaEventRecord(w->done, s);
    if (launches) *launches += nl;
    return rc;
}

}  // namespace tilu
