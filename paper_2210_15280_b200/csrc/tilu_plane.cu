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
// Bands.  A CTA processes one band task: PW consecutive diagonals s0..s0+PW-1 of one 32-row chunk
// c.  Per diagonal k the CTA runs a *solver* warp (the substitution chain and the handoffs only)
// and helper warps that run ahead of it: forward, a march helper (the seven L values of every
// point: NDDF march, V1 band rows or stored factors) and a residual helper (f - A u from 3D TMA
// boxes of the u / f planes); backward, a march helper (the seven source-point L values and 1/D).
// Helpers hand a group of GS steps at a time to their solver through a shared-memory ring with
// mbarrier full / empty phases.  Solver k hands its values to solver k+1 through a shared-memory
// ring in which the data is the flag (a signalling-NaN sentinel marks an empty slot; the consumer
// re-arms the slot after reading it, the producer checks that its next slots are armed).  Across
// bands (the band's first diagonal needs the previous band's last one) and across chunks (lane 0
// needs row z0-1 of the chunk below) the values travel through global memory with the same
// sentinel protocol on the handoff positions only, prefetched PD steps ahead with cp.async:
//   forward : W (w_f, full plane, written by the forward pass).  Handoff positions are the last
//             diagonal of every band and the rows z = 0 mod 32.  The backward pass reads w_f and
//             re-arms those positions.
//   backward: B (w_b, handoff positions only: the first diagonal of every band and the rows
//             z = 1 mod 32, z > 32).  The forward pass re-arms them.
// Persistent CTAs (one per SM) take band tasks from one global ticket in a topological order
// (every task a band depends on has a smaller ticket), so a CTA only waits for tasks held by
// running CTAs: deadlock-free for any residency.
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
#include <type_traits>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "tilu_common.cuh"
#include "tilu_plan.cuh"
#include "tilu_sepk_dev.cuh"

namespace tilu {
void prof_begin(cudaStream_t s);
void prof_end(const char *name, cudaStream_t s);

namespace pl {

constexpr int PW = 4;    // diagonals per band (one solver warp + helper warps each)
constexpr int GS = 4;    // steps per group: helper ring and TMA unit, unroll factor, global prefetch distance
#ifndef TILU_PLANE_NS
#define TILU_PLANE_NS 2
#endif
constexpr int NS = TILU_PLANE_NS;  // helper -> solver ring depth (groups)
constexpr int NT = 3;    // TMA ring depth (groups)
#ifndef TILU_PLANE_HR
#define TILU_PLANE_HR 8
#endif
constexpr int HR = TILU_PLANE_HR;  // solver -> solver handoff ring depth (steps), power of two
#ifndef TILU_PLANE_PD
#define TILU_PLANE_PD 2
#endif
constexpr int PD = TILU_PLANE_PD;  // global handoff prefetch distance (steps), power of two
constexpr int WIN = 34;  // doubles per staged line: z0-1 .. z0+32
constexpr int RS = 10;   // doubles per lane and step in the helper -> solver ring (8 used; 80-byte stride)
// one staged group: forward u box [3 planes s-1..s+1][GS+4 lines][WIN] + f box [GS][WIN];
// backward w_f box [GS][WIN] + u box [GS][WIN]  (tensor copies need 128-byte aligned destinations)
constexpr int FOFF = (3 * (GS + 4) * WIN * 8 + 127) / 128 * 128 / 8;  // doubles: f box offset in a slot
constexpr int UOFF = (GS * WIN * 8 + 127) / 128 * 128 / 8;            // doubles: backward u box offset
constexpr int TSLOT = (FOFF * 8 + GS * WIN * 8 + 127) / 128 * 128;
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
// u3 = u, box (WIN, GS+4, 3); f1 = f, box (WIN, GS, 1); w1 = w_f, box (WIN, GS, 1); u1 = u, box (WIN, GS, 1).
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
    long long *steplog;    // TILU_PLANE_STEPLOG: [PW][2048] clock64 at every step of task 0 (or nullptr)
    long long *trace;      // TILU_PLANE_TRACE: [ntasks][4] = start ns, end ns, sm id, CTA (or nullptr)
    int prof_task;         // TILU_PLANE_PROF builds: ticket whose warps the steplog measures (TILU_PLANE_PROF_TASK)
    int64_t pe;            // doubles per plane vector (bounds checks of -DTILU_DEBUG_BOUNDS builds)
    Geo g;
    int stored;            // 1: L / 1/D from the stored ILU(0) factors (CellILU, ilu.py:210-227) instead of NDDF
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
// Handoff-ring accesses: volatile (re-read every time, never cached in registers) but without a
// compiler memory clobber, so independent loads and arithmetic still schedule around them.
__device__ __forceinline__ double lds_vol(const double *p) { return *reinterpret_cast<const volatile double *>(p); }
__device__ __forceinline__ void sts(double *p, double v) { *reinterpret_cast<volatile double *>(p) = v; }
// re-read of a global handoff value still at the sentinel: relaxed, GPU scope (tilu_common.cuh)
__device__ __forceinline__ double ldg_cg(const double *p) { return ld_rlx(p); }
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
    alignas(128) unsigned char tbuf[PW][NT][TSLOT];  // TMA ring (groups of GS steps)
    double ring[PW][NS][GS][32][RS];                // helpers -> solver: per step and lane 7 L values + residual
                                                    // (fwd) or 7 source-point L values + 1/D (bwd); RS = 10
                                                    // keeps the solver's four 16-byte loads conflict-free
    double hring[PW][HR][32];                       // solver k-1 -> solver k handoff ring
    double pre[PW][PD][3][32];                      // prefetched global handoff values (cp.async)
    uint64_t tfull[PW][NT];                         // TMA group landed
    uint64_t full[PW][NS];                          // helpers filled a ring group
    uint64_t empty[PW][NS];                         // solver drained a ring group
    int task;
};

// Asynchronous 8-byte global -> shared copies (LDGSTS), tracked by commit groups instead of register
// scoreboards, so a deep prefetch really stays in flight.
__device__ __forceinline__ void cpa8(uint32_t dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_pd() { asm volatile("cp.async.wait_group %0;" ::"n"(PD - 1) : "memory"); }

__device__ __forceinline__ void mb_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

// Predicated global load (no branch): v = p ? *ptr : other.
__device__ __forceinline__ double ld_if(bool p, const double *ptr, double other)
{
    double v = other;
    asm("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q ld.global.nc.f64 %0, [%1];\n}" : "+d"(v) : "l"(ptr), "r"((int)p));
    return v;
}

// The substitution split around the acquire of the step's handoff inputs (forward: p0 = (s-1, tau+1, z)
// and lane z-1's lw1, lp1, which lane 0 takes from the chunk below; backward, mirrored: q0 from diagonal
// s+1 and lane z+1's values): the terms of values already in registers are evaluated first.  Both
// passes have the same shape.  Exact mode keeps the reference order -- forward r - L_w w1 - L_s p1 - L_se p0
// - L_bnw lw2 - L_bn lw1 - L_bc lp2 - L_be lp1 (_kernels.py:350-364), backward r = inv_d w_f then the
// seven source points in the same slots (_kernels.py:416-428) -- the products are computed early but
// every subtraction happens in the same order, so the result is bitwise the reference's; fast mode
// subtracts the earlier inputs first and the step's inputs last with FMA.
template <bool EXACT>
struct ChainPart {
    double acc, t3, t5;
    __device__ __forceinline__ ChainPart(double r, const double (&L)[7], double w1, double p1, double lw2, double lp2)
    {
        if (EXACT) {
            acc = dsub(dsub(r, dmul(L[0], w1)), dmul(L[1], p1));
            t3 = dmul(L[3], lw2);
            t5 = dmul(L[5], lp2);
        } else {
            acc = fma(-L[0], w1, fma(-L[5], lp2, fma(-L[3], lw2, fma(-L[1], p1, r))));
            t3 = t5 = 0.0;
        }
    }
    __device__ __forceinline__ double finish(const double (&L)[7], double p0, double lw1, double lp1) const
    {
        if (EXACT) {
            double a = dsub(acc, dmul(L[2], p0));
            a = dsub(a, t3);
            a = dsub(a, dmul(L[4], lw1));
            a = dsub(a, t5);
            return dsub(a, dmul(L[6], lp1));
        }
        return fma(-L[4], lw1, fma(-L[2], p0, fma(-L[6], lp1, acc)));
    }
};

template <int HELPERS>
__device__ __forceinline__ void init_smem(Smem &S)
{
    for (int i = threadIdx.x; i < PW * HR * 32; i += blockDim.x) (&S.hring[0][0][0])[i] = sentv();
    if (threadIdx.x < PW * NT) mb_init(&S.tfull[0][0] + threadIdx.x, 1);
    if (threadIdx.x < PW * NS) {
        mb_init(&S.full[0][0] + threadIdx.x, 32 * HELPERS);
        mb_init(&S.empty[0][0] + threadIdx.x, 32);
    }
    mb_fence_init();
    __syncthreads();
}

__device__ __forceinline__ void trace_start(const Args &A, int t)
{
    if (A.trace && threadIdx.x == 0) A.trace[TR * (int64_t)t] = gtimer();
}
__device__ __forceinline__ void trace_end(const Args &A, int t)
{
    if (A.trace && threadIdx.x == 0) {
        A.trace[TR * (int64_t)t + 1] = gtimer();
        A.trace[TR * (int64_t)t + 2] = smid();
        A.trace[TR * (int64_t)t + 3] = blockIdx.x;
    }
}

// The solver's handoff with the neighbouring diagonals (both passes).  Producer back-pressure: before
// a group of GS steps, the GS ring slots it will write must be armed (consumed).
__device__ __forceinline__ void wait_armed(const double *hout, int t_first, int dir, int lo, int hi)
{
    // The consumer re-arms the slots in step order, so the slot of the group's last step being armed
    // implies all of them are.
    const int tl = dir > 0 ? min(t_first + GS - 1, hi) : max(t_first - (GS - 1), lo);
    if (tl < lo || tl > hi) return;
    const double *p = hout + (tl & (HR - 1)) * 32;
    long long spins = 0;
    while (__any_sync(0xffffffffu, !is_sent(lds_vol(p)))) {
        if (++spins > (1ll << 28)) __trap();
    }
}

// TILU_PLANE_STEPLOG instrumentation (task 0 only): per warp cycle counters
// (compiled in only with -DTILU_PLANE_PROF)
#ifdef TILU_PLANE_PROF
#define PLN_T0() const long long _pt0 = prof ? clock64() : 0
#define PLN_ADD(i) do { if (prof) pc[i] += clock64() - _pt0; } while (0)
#else
#define PLN_T0() (void)0
#define PLN_ADD(i) (void)0
#endif

// ------------------------------------------------------------------------------------------------
// Forward pass: residual r = f - A u, forward L substitution (unit lower), w_f = result.
//
// Per diagonal of the band three warps: the solver (role 0) runs only the substitution chain and
// the handoffs -- a short dependent sequence per step -- while the march helper (role 1: the seven
// L values of every point, NDDF march and V1 band rows) and the residual helper (role 2: the
// 15-point residual from TMA-staged planes) run ahead and pass their results through a
// shared-memory ring of GS-step groups (mbarrier full / empty).
// ------------------------------------------------------------------------------------------------
// AMODE: 0 = per-point rows (P.arows), 1 = constant row (A.arow), 2 = separable coefficient rows
// evaluated on the fly (P.sepk, config 3).
template <int K, bool EXACT, int AMODE>
__global__ void __launch_bounds__(3 * PW * 32, 1) k_plane_fwd(const PlanDev P, const Args A, const __grid_constant__ Maps M)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = wid % PW, role = wid / PW;
    init_smem<2>(S);
    const Geo g = A.g;
    const int n = P.n, ZP = g.ZP;
    uint32_t seq = 0, tseq = 0, tiss = 0;  // ring groups used; TMA groups consumed / issued (role 2)
    for (;;) {
        if (threadIdx.x == 0) S.task = atomicAdd(A.ticket, 1);
        __syncthreads();
        const int t = S.task;
        if (t >= A.ntasks) break;
        trace_start(A, t);
        const int code = A.tasks[t];
        const int b = code >> 16, c = code & 0xffff;
        const int s0 = 2 + PW * b, z0 = 1 + 32 * c;
        const int s = s0 + k, z = z0 + lane, y = s - z;
        const int xe = n - 1 - s, xe0 = n - 1 - s0;
        // steps from tau = z0-3 (uniform for the band): lane 0's first point is at tau = z0+1
        const int T0 = z0 - 3, T1 = z0 + 32 + xe0;
        const bool wlive = (s <= n - 2) && (z0 <= s - 1);
        const bool live = wlive && (z <= s - 1);
        const int lo = live ? z + 1 : 1 << 30, hi = live ? z + xe : -(1 << 30);  // steps with a point
        const int ngroups = (T1 - T0) / GS + 1;
        double r2 = 0.0;
#ifdef TILU_PLANE_PROF
        const bool prof = A.steplog && t == A.prof_task;
        long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const long long pstart = prof ? clock64() : 0;
#endif
        if (role == 0) {
            // ================================ solver ===========================================
            double *hin = &S.hring[k][0][lane];
            double *hout = (k + 1 < PW) ? &S.hring[k + 1][0][lane] : nullptr;
            if (!wlive) {
                // no rows here: pass zeros down the band (the neighbour values are boundary values)
                for (int tau = T0; tau <= T1; ++tau) {
                    if (k > 0 && tau <= T1 - 1) (void)take_s(hin + ((tau + 1) & (HR - 1)) * 32);
                    if (hout && tau >= T0 + 1) put_s(hout + (tau & (HR - 1)) * 32, 0.0);
                }
            } else {
                // Lean step: every solver reads its predecessor value p0 = (s-1, tau+1, z) from its input
                // ring hring[k] -- for k > 0 written by solver k-1, for k == 0 (no predecessor in the band)
                // filled by cp.async from the band below's w_f plane PD steps ahead (zeros for band 0) --
                // so the fast path is one shared-memory load and one vote for every warp; lane 0 also
                // takes ga = w_f(s, tau-1, z0-1), gb = w_f(s-1, tau, z0-1) of the chunk below (prefetched
                // into pre[k]).  No branches on the fast path; sentinels (producer not there yet) go to
                // the re-poll loop.
                const bool gl_on = (lane == 0);
                // the global inputs can only be nonzero when the band below (b > 0) / the chunk below (c > 0)
                // exists: otherwise they are boundary zeros and are neither fetched nor polled
                const bool gp_ld = (k == 0) && b > 0, gl_ld = gl_on && z0 > 1;
                const double *pw0 = A.W + pidx(g, s - 1, 1, z);        // P(tau+1) = pw0[tau * ZP]
                const double *pga = A.W + pidx(g, s, -1, z0 - 1);      // ga(tau) = pga[tau * ZP]
                const double *pgb = A.W + pidx(g, s - 1, 0, z0 - 1);   // gb(tau) = pgb[tau * ZP]
                double *pwo = A.W + pidx(g, s, 0, z);
                double *pbo = A.B + pidx(g, s, 0, z);
                if (k == 0) {  // band input ring: boundary zeros (band 0), else overwritten by the prefetch
#pragma unroll
                    for (int e = 0; e < HR; ++e) hin[e * 32] = 0.0;
                    __syncwarp();
                }
                const uint32_t hin_s = su32(hin), pre_s = su32(&S.pre[k][0][0][lane]);
                // global inputs of step tn, PD steps ahead (addresses of out-of-range steps stay inside the
                // allocation and read boundary zeros)
                auto prefetch = [&](const int tn) {
                    TILU_CHECK(!gp_ld || (pw0 + (int64_t)tn * ZP - A.W >= 0 && pw0 + (int64_t)tn * ZP - A.W < A.pe),
                               "plane fwd band input", tn, s);
                    TILU_CHECK(!gl_ld || (pga + (int64_t)tn * ZP - A.W >= 0 && pgb + (int64_t)tn * ZP - A.W < A.pe),
                               "plane fwd chunk input", tn, s);
                    if (gp_ld) cpa8(hin_s + (uint32_t)(((tn + 1) & (HR - 1)) * 32 * 8), pw0 + (int64_t)tn * ZP);
                    if (gl_ld) {
                        const uint32_t d = pre_s + (uint32_t)((tn & (PD - 1)) * 96 * 8);
                        cpa8(d + 32 * 8, pga + (int64_t)tn * ZP);
                        cpa8(d + 64 * 8, pgb + (int64_t)tn * ZP);
                    }
                    cpa_commit();
                };
#pragma unroll
                for (int i = 0; i < PD; ++i) prefetch(T0 + i);
                double w1 = 0, w2 = 0, p1 = 0, p2 = 0, ga_prev = 0, gb_prev = 0;
                const bool rearm_b = live && (k == 0 || (lane == 0 && z0 > 32));
                auto grp = [&](const int q) {
                    const int sl = seq % NS;
                    const int tq = T0 + GS * q;
                    {
                        PLN_T0();
                        if (hout) wait_armed(hout, tq, 1, T0 + 1, T1);
                        PLN_ADD(1);
                    }
                    {
                        PLN_T0();
                        mb_wait(&S.full[k][sl], (seq / NS) & 1);
                        PLN_ADD(2);
                    }
                    const double *rg = &S.ring[k][sl][0][lane][0];
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        const int tau = tq + j;
                        if (tau <= T1) {
#ifdef TILU_PLANE_PROF
                            const long long _s0 = prof ? clock64() : 0;
#endif
                            const bool p_on = tau <= T1 - 1;
                            // 1. everything that does not depend on this step's handoff inputs, ahead of
                            //    the acquire: the ring values, the lane z-1 shuffles of last step's values
                            //    and the leading part of the substitution
                            const double2 *r2 = reinterpret_cast<const double2 *>(rg + j * (32 * RS));
                            const double2 a0 = r2[0], a1 = r2[1], a2 = r2[2], a3 = r2[3];
                            const double L[7] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y, a3.x};
                            const double sw1 = __shfl_up_sync(0xffffffffu, w1, 1);
                            const double sw2 = __shfl_up_sync(0xffffffffu, w2, 1);
                            const double sp1 = __shfl_up_sync(0xffffffffu, p1, 1);
                            const double sp2 = __shfl_up_sync(0xffffffffu, p2, 1);
                            const double lw2 = gl_on ? ga_prev : sw2;
                            const double lp2 = gl_on ? gb_prev : sp2;
                            ChainPart<EXACT> part(a3.y, L, w1, p1, lw2, lp2);
                            // 2. acquire this step's inputs produced by other warps / CTAs
                            cpa_wait_pd();
                            double *hs = hin + ((tau + 1) & (HR - 1)) * 32;
                            const double *pv = &S.pre[k][tau & (PD - 1)][0][lane];
                            double p0 = p_on ? lds_vol(hs) : 0.0;
                            double ga_cur = gl_ld ? pv[32] : 0.0, gb_cur = gl_ld ? pv[64] : 0.0;
                            bool wt = p_on && (is_sent(p0) || is_sent(ga_cur) || is_sent(gb_cur));
                            if (__builtin_expect(__any_sync(0xffffffffu, wt), 0)) {
                                long long spins = 0;
                                do {
                                    if (is_sent(p0)) p0 = (k == 0) ? ldg_cg(pw0 + (int64_t)tau * ZP) : lds_vol(hs);
                                    if (is_sent(ga_cur)) ga_cur = ldg_cg(pga + (int64_t)tau * ZP);
                                    if (is_sent(gb_cur)) gb_cur = ldg_cg(pgb + (int64_t)tau * ZP);
                                    wt = is_sent(p0) || is_sent(ga_cur) || is_sent(gb_cur);
                                    if (++spins > (1ll << 26)) __trap();
                                } while (__any_sync(0xffffffffu, wt));
                            }
#ifdef TILU_PLANE_PROF
                            long long _s1 = 0;
                            if (prof) {
                                asm volatile("mov.u64 %0, %%clock64;" : "=l"(_s1) : "d"(p0), "d"(ga_cur), "d"(gb_cur));
                                pc[4] += _s1 - _s0;
                            }
#endif
                            // 3. the rest of the chain: the terms of this step's inputs
                            const double lw1 = gl_on ? ga_cur : sw1;
                            const double lp1 = gl_on ? gb_cur : sp1;
                            const double acc = part.finish(L, p0, lw1, lp1);
                            const bool vpt = tau >= lo && tau <= hi;
                            const double wnew = vpt ? acc : 0.0;
#ifdef TILU_PLANE_PROF
                            long long _s2 = 0;
                            if (prof) {
                                asm volatile("mov.u64 %0, %%clock64;" : "=l"(_s2) : "d"(wnew));
                                pc[5] += _s2 - _s1;
                            }
#endif
                            if (p_on && k > 0) sts(hs, sentv());                    // re-arm the input slot
                            if (hout && tau >= T0 + 1) sts(hout + (tau & (HR - 1)) * 32, wnew);
                            if (vpt) {
                                TILU_CHECK(pwo + (int64_t)tau * ZP - A.W >= 0 && pwo + (int64_t)tau * ZP - A.W < A.pe,
                                           "plane fwd w_f store", tau, s);
                                st_rlx(pwo + (int64_t)tau * ZP, wnew);             // polled by the next band / chunk
                                if (rearm_b) st_rlx(pbo + (int64_t)tau * ZP, sentv());
                            }
                            ga_prev = ga_cur; gb_prev = gb_cur;
                            w2 = w1; w1 = wnew;
                            p2 = p1; p1 = p0;
                            prefetch(tau + PD);
#ifdef TILU_PLANE_PROF
                            if (prof) pc[6] += clock64() - _s2;
#endif
                        }
                    }
                    mb_arrive(&S.empty[k][sl]);
                    ++seq;
                };
                for (int q = 0; q < ngroups; ++q) grp(q);
                asm volatile("cp.async.wait_all;" ::: "memory");
            }
        } else if (role == 1 && wlive) {
            // ============================ march helper ==========================================
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
            const bool v1 = P.variant == 1, stored = A.stored != 0;
            const bool rowband = z == 1 || y == 1;
            // Loaded GS steps ahead: bl[j] = V1 band row of step tq + j (when a band point), or with
            // stored factors the factor row of every point (_kernels.py:150-166 reads factors[p, m])
            auto band_ld = [&](int tau, double(&v)[7]) {
                const bool vp = tau >= lo && tau <= hi;
                const int x = tau - z;
                const bool isb = stored ? vp : (v1 && vp && (rowband || tau == lo || tau == hi));
                const double *st = stored ? P.factors + 9 * (rbase + x)
                                          : P.store + 9 * (int64_t)(boff + (rowband ? x - 1 : (tau == lo ? 0 : 1)));
                TILU_CHECK(!isb || (stored ? (rbase + x >= 0 && rbase + x < P.grid)
                                           : (boff + (rowband ? x - 1 : (tau == lo ? 0 : 1)) < P.nband_dbg)),
                           "plane fwd band / factor row", tau, z);
                if (__any_sync(0xffffffffu, isb)) {
#pragma unroll
                    for (int m = 0; m < 7; ++m) v[m] = ld_if(isb, st + m, 0.0);
                }
            };
            double bl[GS][7];
#pragma unroll
            for (int j = 0; j < GS; ++j) band_ld(T0 + j, bl[j]);
            for (int q = 0; q < ngroups; ++q, ++seq) {
                const int sl = seq % NS;
                const int tq = T0 + GS * q;
                {
                    PLN_T0();
                    mb_wait(&S.empty[k][sl], ((seq / NS) & 1) ^ 1);
                    PLN_ADD(2);
                }
                double *rg = &S.ring[k][sl][0][lane][0];
#pragma unroll
                for (int j = 0; j < GS; ++j) {
                    const int tau = tq + j;
                    const bool vpt = tau >= lo && tau <= hi;
                    const bool isb = stored || (v1 && vpt && (rowband || tau == lo || tau == hi));
#pragma unroll
                    for (int m = 0; m < 7; ++m) rg[j * (32 * RS) + m] = isb ? bl[j][m] : d[m][0];
                    if (vpt && !stored) {
#pragma unroll
#ifndef TILU_PLANE_NOHELP
                        for (int m = 0; m < 7; ++m) march<K>(d[m]);
#endif
                    }
                    band_ld(tau + GS, bl[j]);
                }
                mb_arrive(&S.full[k][sl]);
            }
        } else if (role == 2 && wlive) {
            // =========================== residual helper ========================================
            int64_t rbase = 0;
            if (live) rbase = P.rowbase[row_id(n, z, y)];
            // separable coefficient: the y / z table windows are constant along the row
            double gyw[7], gzw[7];
            if (AMODE == 2) {
                const int T4 = 4 * n + 1;
                sepk_window(P.sepk + T4, live ? 4 * y : 4, gyw);
                sepk_window(P.sepk + 2 * T4, live ? 4 * z : 4, gzw);
            }
            // operator surrogate (AMODE 3, a_mode='surrogate'): the 15 weights of a point are the heads of 15
            // forward-difference tables seeded per row (P.seedA, runtime extent akx1 <= AKMAX, zero-padded: the
            // padding entries add 0.0 and never reach an entry that is read) and marched after every point
            // (_kernels.py:444-483 surrogate_apply_residual)
            constexpr int AKMAX = 4;
            double da[AMODE == 3 ? 15 : 1][AMODE == 3 ? AKMAX : 1];
            if (AMODE == 3) {
                const int ak = P.akx1;
                const double *sd = P.seedA + (int64_t)(live ? row_id(n, z, y) : 0) * 15 * ak;
#pragma unroll
                for (int m = 0; m < 15; ++m)
#pragma unroll
                    for (int j = 0; j < AKMAX; ++j) da[m][j] = (live && j < ak) ? sd[m * ak + j] : 0.0;
            }
            auto issue = [&](int q) {  // lane 0: u box (planes s-1..s+1, lines tq-2 .. tq+GS+1) + f box
                const int sl = tiss % NT;
                const int tq = T0 + GS * q;
                double *tb = reinterpret_cast<double *>(S.tbuf[k][sl]);
                mb_expect(&S.tfull[k][sl], (3 * (GS + 4) + GS) * WIN * 8);
                tma3(tb, &M.u3, z0 - 1, tq - 2, s - 1, &S.tfull[k][sl]);
                tma3(tb + FOFF, &M.f1, z0 - 1, tq, s, &S.tfull[k][sl]);
                ++tiss;
            };
            if (lane == 0)
                for (int q = 0; q < ngroups && q < NT; ++q) issue(q);
            for (int q = 0; q < ngroups; ++q, ++seq, ++tseq) {
                const int sl = seq % NS, tsl = tseq % NT;
                const int tq = T0 + GS * q;
                {
                    PLN_T0();
                    mb_wait(&S.tfull[k][tsl], (tseq / NT) & 1);
                    PLN_ADD(3);
                }
                {
                    PLN_T0();
                    mb_wait(&S.empty[k][sl], ((seq / NS) & 1) ^ 1);
                    PLN_ADD(2);
                }
                double *rg = &S.ring[k][sl][0][lane][0];
#pragma unroll
                for (int j = 0; j < GS; ++j) {
                    const int sg = tq + j;
                    const double *tb = reinterpret_cast<const double *>(S.tbuf[k][tsl]) + j * WIN + lane + 1;
                    const double *u1 = tb + (GS + 4) * WIN;      // plane s,   line sg-2 at offset 0
                    const double *u0 = tb;                       // plane s-1
                    const double *u2 = tb + 2 * (GS + 4) * WIN;  // plane s+1
                    constexpr int Wn = WIN;
                    double res = 0.0;
#ifndef TILU_PLANE_NOHELP
                    if (sg >= lo && sg <= hi) {
#else
                    if (false) {  // experiment: residual helper without arithmetic (results invalid)
#endif
                        double a[15];
                        if (AMODE == 3) {
#pragma unroll
                            for (int qq = 0; qq < 15; ++qq) a[qq] = da[qq][0];
                        } else if (AMODE == 2) {
                            double hxw[7];
                            sepk_window(P.sepk, 4 * (sg - z), hxw);
                            sepk_row(hxw, gyw, gzw, P.sepk_c0, P.sepk_w, a);
                        } else if (AMODE == 1) {
#pragma unroll
                            for (int qq = 0; qq < 15; ++qq) a[qq] = A.arow[qq];
                        } else {
                            TILU_CHECK(rbase + (sg - z) >= 0 && rbase + (sg - z) < P.grid, "plane residual row", sg, z);
                            const double *ar = P.arows + 15 * (rbase + (sg - z));
#pragma unroll
                            for (int qq = 0; qq < 15; ++qq) a[qq] = ar[qq];
                        }
                        if (AMODE == 3) {
                            // surrogate_apply_residual order (_kernels.py:470-480): every product subtracted
                            // from the running value f - c u - w .. - tw
                            double rr = msub<EXACT>(tb[FOFF], a[7], u1[2 * Wn]);
                            rr = msub<EXACT>(rr, a[0], u1[1 * Wn]);
                            rr = msub<EXACT>(rr, a[1], u0[2 * Wn]);
                            rr = msub<EXACT>(rr, a[2], u0[3 * Wn]);
                            rr = msub<EXACT>(rr, a[3], u1[0 * Wn - 1]);
                            rr = msub<EXACT>(rr, a[4], u1[1 * Wn - 1]);
                            rr = msub<EXACT>(rr, a[5], u0[1 * Wn - 1]);
                            rr = msub<EXACT>(rr, a[6], u0[2 * Wn - 1]);
                            rr = msub<EXACT>(rr, a[8], u1[3 * Wn]);
                            rr = msub<EXACT>(rr, a[9], u2[2 * Wn]);
                            rr = msub<EXACT>(rr, a[10], u2[1 * Wn]);
                            rr = msub<EXACT>(rr, a[11], u1[4 * Wn + 1]);
                            rr = msub<EXACT>(rr, a[12], u1[3 * Wn + 1]);
                            rr = msub<EXACT>(rr, a[13], u2[3 * Wn + 1]);
                            rr = msub<EXACT>(rr, a[14], u2[2 * Wn + 1]);
                            res = rr;
                            r2 = fma(res, res, r2);
#pragma unroll
                            for (int qq = 0; qq < 15; ++qq) march<AKMAX>(da[qq]);
                        } else {
                        // stencil_apply order (_kernels.py:243-267): c, w s se bnw bn bc be, e n nw tse ts tc tw
                        double out = EXACT ? dmul(a[7], u1[2 * Wn]) : a[7] * u1[2 * Wn];
                        out = madd<EXACT>(out, a[0], u1[1 * Wn]);        // w   (s,   sg-1, z)
                        out = madd<EXACT>(out, a[1], u0[2 * Wn]);        // s   (s-1, sg,   z)
                        out = madd<EXACT>(out, a[2], u0[3 * Wn]);        // se  (s-1, sg+1, z)
                        out = madd<EXACT>(out, a[3], u1[0 * Wn - 1]);    // bnw (s,   sg-2, z-1)
                        out = madd<EXACT>(out, a[4], u1[1 * Wn - 1]);    // bn  (s,   sg-1, z-1)
                        out = madd<EXACT>(out, a[5], u0[1 * Wn - 1]);    // bc  (s-1, sg-1, z-1)
                        out = madd<EXACT>(out, a[6], u0[2 * Wn - 1]);    // be  (s-1, sg,   z-1)
                        out = madd<EXACT>(out, a[8], u1[3 * Wn]);        // e   (s,   sg+1, z)
                        out = madd<EXACT>(out, a[9], u2[2 * Wn]);        // n   (s+1, sg,   z)
                        out = madd<EXACT>(out, a[10], u2[1 * Wn]);       // nw  (s+1, sg-1, z)
                        out = madd<EXACT>(out, a[11], u1[4 * Wn + 1]);   // tse (s,   sg+2, z+1)
                        out = madd<EXACT>(out, a[12], u1[3 * Wn + 1]);   // ts  (s,   sg+1, z+1)
                        out = madd<EXACT>(out, a[13], u2[3 * Wn + 1]);   // tc  (s+1, sg+1, z+1)
                        out = madd<EXACT>(out, a[14], u2[2 * Wn + 1]);   // tw  (s+1, sg,   z+1)
                        res = dsub(tb[FOFF], out);
                        r2 = fma(res, res, r2);
                        }
                    }
                    rg[j * (32 * RS) + 7] = res;
                }
                __syncwarp();
                if (lane == 0 && q + NT < ngroups) issue(q + NT);
                mb_arrive(&S.full[k][sl]);
            }
        }
        if (A.part && role == 2) A.part[(int64_t)t * (PW * 32) + k * 32 + lane] = r2;
#ifdef TILU_PLANE_PROF
        if (prof && lane == 0) {
            long long *sl = A.steplog + wid * 8;
            sl[0] += clock64() - pstart;
            for (int i = 1; i < 5; ++i) sl[i] += pc[i];
            sl[5] += ngroups;
            sl[6] += pc[5];
            sl[7] += pc[6];
        }
#endif
        __syncthreads();
        trace_end(A, t);
    }
}

// ------------------------------------------------------------------------------------------------
// Backward pass: D^{-1} scaling + L^T substitution (descending), fused u += w (multigrid.py:429).
// Per diagonal two warps: the solver (role 0: substitution, handoffs, TMA of w_f and u) and the
// march helper (role 1: the seven source-point L values and 1/D of every point, V1 band rows).
// ------------------------------------------------------------------------------------------------
template <int K, bool EXACT>
__global__ void __launch_bounds__(2 * PW * 32, 1) k_plane_bwd(const PlanDev P, const Args A, const __grid_constant__ Maps M)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = wid % PW, role = wid / PW;
    init_smem<1>(S);
    const Geo g = A.g;
    const int n = P.n, ZP = g.ZP;
    uint32_t seq = 0, tseq = 0, tiss = 0;
    for (;;) {
        if (threadIdx.x == 0) S.task = atomicAdd(A.ticket, 1);
        __syncthreads();
        const int t = S.task;
        if (t >= A.ntasks) break;
        trace_start(A, t);
        const int code = A.tasks[A.ntasks - 1 - t];
        const int b = code >> 16, c = code & 0xffff;
        const int s0 = 2 + PW * b, z0 = 1 + 32 * c;
        const int s = s0 + PW - 1 - k, z = z0 + lane, y = s - z;
        const int xe = n - 1 - s, xe0 = n - 1 - s0;
        const int T0 = z0 - 1, T1 = z0 + 32 + xe0;  // steps tau = T1 .. T0-1 (descending)
        const bool wlive = (s <= n - 2) && (z0 <= s - 1);
        const bool live = wlive && (z <= s - 1);
        const int lo = live ? z + 1 : 1 << 30, hi = live ? z + xe : -(1 << 30);
        const int ngroups = (T1 - (T0 - 1)) / GS + 1;
        if (role == 0) {
            double *hin = &S.hring[k][0][lane];
            double *hout = (k + 1 < PW) ? &S.hring[k + 1][0][lane] : nullptr;
            if (!wlive) {
                for (int tau = T1; tau >= T0 - 1; --tau) {
                    if (k > 0 && tau >= T0) (void)take_s(hin + ((tau - 1) & (HR - 1)) * 32);
                    if (hout && tau <= T1 - 1) put_s(hout + (tau & (HR - 1)) * 32, 0.0);
                }
            } else {
                // group q stages tau = T1 - GS q .. T1 - GS q - (GS-1): w_f and u boxes of GS lines
                auto issue = [&](int q) {
                    const int sl = tiss % NT;
                    const int lo_t = T1 - GS * q - (GS - 1);
                    double *tb = reinterpret_cast<double *>(S.tbuf[k][sl]);
                    mb_expect(&S.tfull[k][sl], 2 * GS * WIN * 8);
                    tma3(tb, &M.w1, z0 - 1, lo_t, s, &S.tfull[k][sl]);
                    tma3(tb + UOFF, &M.u1, z0 - 1, lo_t, s, &S.tfull[k][sl]);
                    ++tiss;
                };
                if (lane == 0)
                    for (int q = 0; q < ngroups && q < NT; ++q) issue(q);
                // warp 0: P'(tau-1) = w_b(s+1, tau-1, z); lane 31: ga = w_b(s, tau+1, z0+32), gb = w_b(s+1, tau, z0+32)
                const double *pw0 = A.B + pidx(g, s + 1, -1, z);
                const double *pga = A.B + pidx(g, s, 1, z0 + 32);
                const double *pgb = A.B + pidx(g, s + 1, 0, z0 + 32);
                double *puo = A.u + pidx(g, s, 0, z);
                double *pbo = A.B + pidx(g, s, 0, z);
                double *pwo = A.W + pidx(g, s, 0, z);
                const bool gp_on = (k == 0), gl_on = (lane == 31);
                // nonzero only when the band above exists / row z0+32 exists on diagonal s or s+1
                const bool gp_ld = gp_on && s0 + PW <= n - 2, gl_ld = gl_on && z0 + 32 <= s;
                double *pre = &S.pre[k][0][0][lane];
                const uint32_t pre_s = su32(pre);
                const double *nw0 = pw0 + T1 * ZP, *nga = pga + T1 * ZP, *ngb = pgb + T1 * ZP;
                int tn = T1;
                auto prefetch = [&]() {
                    const uint32_t d = pre_s + (uint32_t)((tn & (PD - 1)) * 96 * 8);
                    if (gp_ld) cpa8(d, nw0);
                    if (gl_ld) {
                        cpa8(d + 32 * 8, nga);
                        cpa8(d + 64 * 8, ngb);
                    }
                    cpa_commit();
                    nw0 -= ZP; nga -= ZP; ngb -= ZP; --tn;
                };
                for (int i = 0; i < PD; ++i) prefetch();
                double *uo = puo + T1 * ZP, *bo = pbo + T1 * ZP, *wo = pwo + T1 * ZP;
                double wb1 = 0, wb2 = 0, q1 = 0, q2 = 0, ga_prev = 0, gb_prev = 0;
                const bool b_out = live && (k == PW - 1 || (lane == 0 && z0 > 32));
                const bool rearm_w = live && (k == 0 || lane == 31);
                auto grp = [&](const int q) {
                    const int sl = seq % NS, tsl = tseq % NT;
                    const int tq = T1 - GS * q;
                    if (hout) wait_armed(hout, tq, -1, T0 - 1, T1 - 1);
                    mb_wait(&S.tfull[k][tsl], (tseq / NT) & 1);
                    mb_wait(&S.full[k][sl], (seq / NS) & 1);
                    const double *rg = &S.ring[k][sl][0][lane][0];
                    const double *tb = reinterpret_cast<const double *>(S.tbuf[k][tsl]) + lane + 1;
#pragma unroll
                    for (int j = 0; j < GS; ++j) {
                        const int tau = tq - j;
                        if (tau >= T0 - 1) {
                            const bool q_on = tau >= T0;
                            // 1. ahead of the acquire: ring values (seven source-point L and 1/D), the staged
                            //    w_f and u of this step, lane z+1's last values, the leading part of the chain
                            const double2 *r2 = reinterpret_cast<const double2 *>(rg + j * (32 * RS));
                            const double2 a0 = r2[0], a1 = r2[1], a2 = r2[2], a3 = r2[3];
                            const double Lq[7] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y, a3.x};
                            const double wfv = tb[(GS - 1 - j) * WIN];          // line of tau in the boxes
                            const double uv = tb[UOFF + (GS - 1 - j) * WIN];
                            const double sw1 = __shfl_down_sync(0xffffffffu, wb1, 1);
                            const double sw2 = __shfl_down_sync(0xffffffffu, wb2, 1);
                            const double sq1 = __shfl_down_sync(0xffffffffu, q1, 1);
                            const double sq2 = __shfl_down_sync(0xffffffffu, q2, 1);
                            const double lw2 = gl_on ? ga_prev : sw2;
                            const double lq2 = gl_on ? gb_prev : sq2;
                            // reference order (_kernels.py:416-428): inv_d w, then w s se bnw bn bc be sources
                            ChainPart<EXACT> part(EXACT ? dmul(a3.y, wfv) : a3.y * wfv, Lq, wb1, q1, lw2, lq2);
                            // 2. acquire this step's inputs produced by other warps / CTAs
                            double q0 = 0.0;
                            cpa_wait_pd();
                            const double *pv = pre + (tau & (PD - 1)) * 96;
                            if (q_on) q0 = gp_on ? (gp_ld ? pv[0] : 0.0) : lds_vol(hin + ((tau - 1) & (HR - 1)) * 32);
                            double ga_cur = gl_ld ? pv[32] : 0.0, gb_cur = gl_ld ? pv[64] : 0.0;
                            if (__any_sync(0xffffffffu,
                                           (q_on && is_sent(q0)) || (gl_ld && (is_sent(ga_cur) || is_sent(gb_cur))))) {
                                long long spins = 0;
                                for (;;) {
                                    if (q_on && is_sent(q0)) q0 = gp_on ? ldg_cg(pw0 + tau * ZP)
                                                                        : lds_vol(hin + ((tau - 1) & (HR - 1)) * 32);
                                    if (gl_ld) {
                                        if (is_sent(ga_cur)) ga_cur = ldg_cg(pga + tau * ZP);
                                        if (is_sent(gb_cur)) gb_cur = ldg_cg(pgb + tau * ZP);
                                    }
                                    const bool still =
                                        (q_on && is_sent(q0)) || (gl_ld && (is_sent(ga_cur) || is_sent(gb_cur)));
                                    if (!__any_sync(0xffffffffu, still)) break;
                                    if (++spins > (1ll << 26)) __trap();
                                }
                            }
                            // 3. the terms of this step's inputs
                            const double lw1 = gl_on ? ga_cur : sw1;
                            const double lq1 = gl_on ? gb_cur : sq1;
                            const double acc = part.finish(Lq, q0, lw1, lq1);
                            const bool vpt = tau >= lo && tau <= hi;
                            const double wnew = vpt ? acc : 0.0;
                            if (q_on && k > 0) sts(hin + ((tau - 1) & (HR - 1)) * 32, sentv());
                            if (hout && tau <= T1 - 1) sts(hout + (tau & (HR - 1)) * 32, wnew);
                            if (vpt) {
                                TILU_CHECK(uo - A.u >= 0 && uo - A.u < A.pe, "plane bwd u store", tau, s);
                                *uo = dadd(uv, acc);
                                if (b_out) st_rlx(bo, acc);       // polled by the band / chunk below
                                if (rearm_w) st_rlx(wo, sentv());
                            }
                            uo -= ZP; bo -= ZP; wo -= ZP;
                            ga_prev = ga_cur; gb_prev = gb_cur;
                            wb2 = wb1; wb1 = wnew;
                            q2 = q1; q1 = q0;
                            prefetch();
                        }
                    }
                    __syncwarp();
                    if (lane == 0 && q + NT < ngroups) issue(q + NT);
                    mb_arrive(&S.empty[k][sl]);
                    ++seq;
                    ++tseq;
                };
                for (int q = 0; q < ngroups; ++q) grp(q);
                asm volatile("cp.async.wait_all;" ::: "memory");
            }
        } else if (wlive) {
            // ============================ march helper ==========================================
            double d[8][K];
            int bo_own = 0, bo_n = 0, bo_ts = 0, bo_tc = 0;
            int64_t rb_own = 0, rb_n = 0, rb_ts = 0, rb_tc = 0;  // row bases (stored factors)
            if (live) {
                const int r = row_id(n, z, y);
                const double *sd = P.seedB + (int64_t)r * 8 * K;
#pragma unroll
                for (int m = 0; m < 8; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = sd[m * K + j];
                rb_own = P.rowbase[r];
                if (s + 1 <= n - 2) {
                    rb_n = P.rowbase[row_id(n, z, y + 1)];
                    rb_tc = P.rowbase[row_id(n, z + 1, y)];
                }
                if (y >= 2) rb_ts = P.rowbase[row_id(n, z + 1, y - 1)];
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
            const bool v1 = P.variant == 1, stored = A.stored != 0;
            const bool zr1 = z == 1, yr1 = y == 1, yr2 = y == 2, yge2 = y >= 2;
            // band / interior tests of the seven source points q_m = p - d_m (_lq, _kernels.py:434-441)
            // and of p (1/D).  Masks: bit m = q_m interior (m < 7); band bits in bmask (bit 7 = p).
            auto tests = [&](int tau, unsigned &imask, unsigned &bmask) {
                const int x = tau - z;
                const bool vpt = tau >= lo && tau <= hi;
                const bool x1 = x == 1, x2 = x == 2, xm1 = x == xe - 1, xm0 = x == xe;
                const bool i0 = x + 1 <= xe, i1 = x <= xe - 1, i2 = x >= 2, i3 = yge2 && x + 1 <= xe;
                imask = (unsigned)i0 | (unsigned)i1 << 1 | (unsigned)i2 << 2 | (unsigned)i3 << 3 |
                        (unsigned)yge2 << 4 | (unsigned)i1 << 5 | (unsigned)i2 << 6;
                bmask = 0;
                if (v1 && vpt) {
                    bmask = (unsigned)(i0 && (xm1 || yr1 || zr1)) | (unsigned)(i1 && (x1 || xm1 || zr1)) << 1 |
                            (unsigned)(i2 && (x2 || xm0 || zr1)) << 2 | (unsigned)(i3 && (xm1 || yr2)) << 3 |
                            (unsigned)(yge2 && (x1 || xm0 || yr2)) << 4 | (unsigned)(i1 && (x1 || xm1 || yr1)) << 5 |
                            (unsigned)(i2 && (x2 || xm0 || yr1)) << 6 | (unsigned)(x1 || xm0 || yr1 || zr1) << 7;
                }
            };
            // store rows of the band source points (only evaluated when some lane has a band point)
            auto offsets = [&](int tau, int (&o)[8]) {
                const int x = tau - z;
                const bool x1 = x == 1, x2 = x == 2;
                o[0] = bo_own + ((zr1 || yr1) ? x : 1);
                o[1] = bo_n + (zr1 ? x - 1 : (x1 ? 0 : 1));
                o[2] = bo_n + (zr1 ? x - 2 : (x2 ? 0 : 1));
                o[3] = bo_ts + (yr2 ? x : 1);
                o[4] = bo_ts + (yr2 ? x - 1 : (x1 ? 0 : 1));
                o[5] = bo_tc + (yr1 ? x - 1 : (x1 ? 0 : 1));
                o[6] = bo_tc + (yr1 ? x - 2 : (x2 ? 0 : 1));
                o[7] = bo_own + ((zr1 || yr1) ? x - 1 : (x1 ? 0 : 1));
            };
            // masks and band / factor values of step tau, computed GS steps ahead (one tests() per step)
            auto band_ld = [&](int tau, double(&v)[8], unsigned &im, unsigned &bm) {
                tests(tau, im, bm);
                if (stored) {  // factors of the source points q_m (transposed entries) and 1/D at p (_kernels.py:169-192)
                    const int x = tau - z;
                    const bool vp = tau >= lo && tau <= hi;
                    bm = vp ? 0xFFu : 0u;
                    const int64_t rk[8] = {rb_own + x + 1, rb_n + x, rb_n + x - 1, rb_ts + x + 1,
                                           rb_ts + x,      rb_tc + x, rb_tc + x - 1, rb_own + x};
#pragma unroll
                    for (int m = 0; m < 8; ++m)
                        v[m] = ld_if(vp && (m == 7 || ((im >> m) & 1u)), P.factors + 9 * rk[m] + (m < 7 ? m : 8), 0.0);
                    return;
                }
                if (__any_sync(0xffffffffu, bm != 0u)) {
                    int o[8];
                    offsets(tau, o);
#pragma unroll
                    for (int m = 0; m < 8; ++m)
                        v[m] = ld_if((bm >> m) & 1u, P.store + 9 * (int64_t)o[m] + (m < 7 ? m : 8), 0.0);
                }
            };
            double bl[GS][8];
            unsigned bim[GS], bbm[GS];
#pragma unroll
            for (int j = 0; j < GS; ++j) band_ld(T1 - j, bl[j], bim[j], bbm[j]);
            for (int q = 0; q < ngroups; ++q, ++seq) {
                const int sl = seq % NS;
                const int tq = T1 - GS * q;
                mb_wait(&S.empty[k][sl], ((seq / NS) & 1) ^ 1);
                double *rg = &S.ring[k][sl][0][lane][0];
#pragma unroll
                for (int j = 0; j < GS; ++j) {
                    const int tau = tq - j;
                    const unsigned im = bim[j], bm = bbm[j];
#pragma unroll
                    for (int m = 0; m < 7; ++m)
                        rg[j * (32 * RS) + m] = ((im >> m) & 1u) ? (((bm >> m) & 1u) ? bl[j][m] : d[m][0]) : 0.0;
                    rg[j * (32 * RS) + 7] = ((bm >> 7) & 1u) ? bl[j][7] : d[7][0];
                    if (tau >= lo && tau <= hi && !stored) {
#pragma unroll
                        for (int m = 0; m < 8; ++m) march<K>(d[m]);
                    }
                    band_ld(tau - GS, bl[j], bim[j], bbm[j]);
                }
                mb_arrive(&S.full[k][sl]);
            }
        }
        __syncthreads();
        trace_end(A, t);
    }
}

// Experimental one-warp-per-diagonal variant (no helper warps).  Bitwise equal, but measured slower at
// every level (L9 forward 1.82 ms vs 1.02 ms: one warp per scheduler partition hides no latency), so it
// is only compiled with -DTILU_PLANE_FUSED_BUILD and selected with TILU_PLANE_FUSED=1.
#ifdef TILU_PLANE_FUSED_BUILD
#include "tilu_plane_fused.cuh"
#endif

// ------------------------------------------------------------------------------------------------
// Layout conversion, arming, norms.
// ------------------------------------------------------------------------------------------------
// Layout conversion by 32 x 32 tiles of one diagonal plane s: (tau block, z block).  A warp reads
// whole segments of 32 consecutive x of one reference row (coalesced), the tile is transposed in
// shared memory, and every plane line (fixed tau, 32 consecutive z) is written as one segment.
// grid = (tau blocks, z blocks, diagonals 2 .. n-2); UNPACK reverses the direction.
template <bool UNPACK>
__global__ void __launch_bounds__(256) k_plane_xpose(const PlanDev P, Geo g, const double *__restrict__ src,
                                                     double *__restrict__ dst)
{
    __shared__ double tile[32][33];
    const int n = P.n;
    const int s = 2 + blockIdx.z, tau0 = 2 + 32 * blockIdx.x, z0 = 1 + 32 * blockIdx.y;
    const int xe = n - 1 - s;
    if (z0 > s - 1 || tau0 > z0 + 31 + xe || tau0 + 31 < z0 + 1) return;  // no interior point in the tile
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
    if (!UNPACK) {
        // reference rows z = z0 + r: x = tau - z for tau = tau0 + lane
        for (int r = wy; r < 32; r += 8) {
            const int z = z0 + r, x = tau0 + lane - z;
            double v = 0.0;
            if (z <= s - 1 && x >= 1 && x <= xe) v = src[row_offset(n, z, s - z) + x];
            tile[r][lane] = v;
        }
        __syncthreads();
        for (int c = wy; c < 32; c += 8) {  // plane line tau = tau0 + c, z = z0 + lane
            const int z = z0 + lane, x = tau0 + c - z;
            if (z <= s - 1 && x >= 1 && x <= xe) dst[pidx(g, s, tau0 + c, z)] = tile[lane][c];
        }
    } else {
        for (int c = wy; c < 32; c += 8) {
            const int z = z0 + lane, x = tau0 + c - z;
            tile[lane][c] = (z <= s - 1 && x >= 1 && x <= xe) ? src[pidx(g, s, tau0 + c, z)] : 0.0;
        }
        __syncthreads();
        for (int r = wy; r < 32; r += 8) {
            const int z = z0 + r, x = tau0 + lane - z;
            if (z <= s - 1 && x >= 1 && x <= xe) dst[row_offset(n, z, s - z) + x] = tile[r][lane];
        }
    }
}
// Boundary values of u (x = 0, y = 0, z = 0 or x + y + z = n) into the plane layout: the residual reads them
// as given (the all-Dirichlet case has zeros there; the cell stage of a hybrid mesh carries the shared
// interface values, multigrid.py:414-429).  The kernels never write these positions; copied on every call
// because the planes persist between calls.  grid = (y, z) over the closed lattice, threads over x.
__global__ void __launch_bounds__(128) k_plane_pack_boundary(int n, Geo g, const double *__restrict__ src,
                                                             double *__restrict__ dst)
{
    const int y = blockIdx.x, z = blockIdx.y;
    if (y + z > n) return;
    const int xm = n - y - z;
    const int64_t base = row_offset(n, z, y);
    if (y == 0 || z == 0) {
        for (int x = threadIdx.x; x <= xm; x += blockDim.x) dst[pidx(g, y + z, x + z, z)] = src[base + x];
    } else if (threadIdx.x < 2) {
        const int x = threadIdx.x ? xm : 0;
        dst[pidx(g, y + z, x + z, z)] = src[base + x];
    }
}

static void launch_xpose(const PlanDev &P, const Geo &g, const double *src, double *dst, bool unpack, cudaStream_t s)
{
    const int n = P.n;
    const dim3 grid((n - 3 + 31) / 32, (n - 3 + 31) / 32, n - 3);
    if (unpack) k_plane_xpose<true><<<grid, 256, 0, s>>>(P, g, src, dst);
    else k_plane_xpose<false><<<grid, 256, 0, s>>>(P, g, src, dst);
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
    long long *steplog = nullptr;
    Maps maps;
#ifdef TILU_PLANE_FUSED_BUILD
    MapsF mapsf;
#endif
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

// Band tasks in topological order: key kb b + kc c; every dependency ((b-1, c), (b-1, c-1), (b, c-1))
// has a strictly smaller key.
static std::vector<int> make_tasks(int n)
{
    // start-time model: a band starts ~7 steps after the band below (4 diagonals x 2-step lag + the
    // global hop), a chunk ~36 steps after the chunk below (32-lane skew + hop); TILU_PLANE_KEY=kb,kc
    // overrides (measurement only).  Any positive weights keep the order topological.
    long long kb = 7, kc = 36;
    if (const char *e = std::getenv("TILU_PLANE_KEY")) {
        long long a = 0, c = 0;
        if (std::sscanf(e, "%lld,%lld", &a, &c) == 2 && a > 0 && c > 0) {
            kb = a;
            kc = c;
        }
    }
    std::vector<std::pair<long long, int>> v;
    for (int b = 0;; ++b) {
        const int s0 = 2 + PW * b;
        if (s0 > n - 2) break;
        const int smax = std::min(s0 + PW - 1, n - 2);
        const int nch = (smax - 1 + 31) / 32;
        for (int c = 0; c < nch; ++c) v.push_back({(kb * b + kc * c) * 65536 + c, (b << 16) | c});
    }
    std::sort(v.begin(), v.end());
    std::vector<int> out;
    for (auto &e : v) out.push_back(e.second);
    return out;
}

template <int K, bool EXACT, int AMODE>
static cudaError_t set_attrs()
{
    cudaError_t e = cudaFuncSetAttribute(k_plane_fwd<K, EXACT, AMODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(Smem));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_plane_bwd<K, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
}

template <int K, bool EXACT, int AMODE>
static bool launch_k(const PlanDev &P, const Args &A, const Maps &M, int ctas, bool fwd, cudaStream_t s)
{
    // the dynamic shared-memory attribute belongs to a device context: set once per device ordinal
    static signed char attrs[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!attrs[dev]) attrs[dev] = (set_attrs<K, EXACT, AMODE>() == cudaSuccess) ? 1 : -1;
    if (attrs[dev] < 0) return false;
    if (fwd) k_plane_fwd<K, EXACT, AMODE><<<ctas, 3 * PW * 32, sizeof(Smem), s>>>(P, A, M);
    else k_plane_bwd<K, EXACT><<<ctas, 2 * PW * 32, sizeof(Smem), s>>>(P, A, M);
    return true;
}
template <bool EXACT, int AMODE>
static bool launch_e(const PlanDev &P, const Args &A, const Maps &M, int ctas, bool fwd, cudaStream_t s)
{
    switch (P.kx1) {
    case 1: return launch_k<1, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 2: return launch_k<2, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 3: return launch_k<3, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 4: return launch_k<4, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 5: return launch_k<5, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 6: return launch_k<6, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    default: return false;
    }
}
static bool launch_pass(const PlanDev &P, const Args &A, const Maps &M, int ctas, bool exact, bool fwd, cudaStream_t s)
{
    const int am = P.seedA ? 3 : P.sepk ? 2 : P.arow ? 1 : 0;
    if (am == 3) return exact ? launch_e<true, 3>(P, A, M, ctas, fwd, s) : launch_e<false, 3>(P, A, M, ctas, fwd, s);
    if (exact) return am == 2 ? launch_e<true, 2>(P, A, M, ctas, fwd, s)
                    : am == 1 ? launch_e<true, 1>(P, A, M, ctas, fwd, s) : launch_e<true, 0>(P, A, M, ctas, fwd, s);
    return am == 2 ? launch_e<false, 2>(P, A, M, ctas, fwd, s)
         : am == 1 ? launch_e<false, 1>(P, A, M, ctas, fwd, s) : launch_e<false, 0>(P, A, M, ctas, fwd, s);
}

#ifdef TILU_PLANE_FUSED_BUILD
// Fused kernels (tilu_plane_fused.cuh): constant row or separable-coefficient rows, no stored factors.
template <int K, bool EXACT, int AMODE>
static bool launchf_k(const PlanDev &P, const Args &A, const MapsF &M, int ctas, bool fwd, cudaStream_t s)
{
    static signed char attrs[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!attrs[dev]) {
        cudaError_t e = cudaFuncSetAttribute(k_planef_fwd<K, EXACT, AMODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(SmemF));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_planef_bwd<K, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemF));
        attrs[dev] = (e == cudaSuccess) ? 1 : -1;
    }
    if (attrs[dev] < 0) return false;
    if (fwd) k_planef_fwd<K, EXACT, AMODE><<<ctas, PW * 32, sizeof(SmemF), s>>>(P, A, M);
    else k_planef_bwd<K, EXACT><<<ctas, PW * 32, sizeof(SmemF), s>>>(P, A, M);
    return true;
}
template <bool EXACT, int AMODE>
static bool launchf_e(const PlanDev &P, const Args &A, const MapsF &M, int ctas, bool fwd, cudaStream_t s)
{
    switch (P.kx1) {
    case 1: return launchf_k<1, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 2: return launchf_k<2, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 3: return launchf_k<3, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 4: return launchf_k<4, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 5: return launchf_k<5, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    case 6: return launchf_k<6, EXACT, AMODE>(P, A, M, ctas, fwd, s);
    default: return false;
    }
}
static bool fused_ok(const PlanDev &P, bool stored)
{
    static const char *e = std::getenv("TILU_PLANE_FUSED");
    if (!e || e[0] != '1') return false;
    return !stored && (P.sepk || P.arow);
}
static bool launchf_pass(const PlanDev &P, const Args &A, const MapsF &M, int ctas, bool exact, bool fwd, cudaStream_t s)
{
    if (P.sepk) return exact ? launchf_e<true, 2>(P, A, M, ctas, fwd, s) : launchf_e<false, 2>(P, A, M, ctas, fwd, s);
    return exact ? launchf_e<true, 1>(P, A, M, ctas, fwd, s) : launchf_e<false, 1>(P, A, M, ctas, fwd, s);
}
#endif

static int resident_ctas(const tilu_plan *p)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static const char *e = std::getenv("TILU_PLANE_CTAS_PER_SM");
    int per = e ? std::atoi(e) : 1;  // one CTA per SM (shared memory: ~166 KB per CTA)
    if (per < 1) per = 1;
    if (per > 1) per = 1;
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
    static const char *nt = std::getenv("TILU_PLANE_NTASKS");  // debug: only the first N tasks (results invalid)
    if (nt && std::atoi(nt) > 0 && (size_t)std::atoi(nt) < tasks.size()) tasks.resize(std::atoi(nt));
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
    if (!encode_map(&w->maps.u3, w->u, w->g, GS + 4, 3) || !encode_map(&w->maps.f1, w->f, w->g, GS, 1) ||
        !encode_map(&w->maps.w1, w->W, w->g, GS, 1) || !encode_map(&w->maps.u1, w->u, w->g, GS, 1)) {
        cudaFree(m);
        delete w;
        return TILU_ECUDA;
    }
#ifdef TILU_PLANE_FUSED_BUILD
    if (!encode_map(&w->mapsf.u3g, w->u, w->g, GS, 3)) {
        cudaFree(m);
        delete w;
        return TILU_ECUDA;
    }
    w->mapsf.f1 = w->maps.f1;
    w->mapsf.w1 = w->maps.w1;
    w->mapsf.u1 = w->maps.u1;
#endif
    if (cudaStreamSynchronize(s) != cudaSuccess || cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming) != cudaSuccess) {
        cudaFree(m);
        delete w;
        return TILU_ECUDA;
    }
    *out = w;
    return TILU_OK;
}

}  // namespace pl

extern "C" int tilu_plane_tasks(int level, int *out, int cap)
{
    if (level < 2 || level > 12) return -1;
    const std::vector<int> t = pl::make_tasks(1 << level);
    for (int i = 0; i < (int)t.size() && i < cap && out; ++i) out[i] = t[i];
    return (int)t.size();
}

bool plane_supported(const tilu_plan *p)
{
    if (p->flags & TILU_SCHED_SIMPLE) return false;
    static const char *e = std::getenv("TILU_PLANE");
    if (e && e[0] == '0') return false;
    // operator surrogate (seedA): x extent up to 4 (a_degrees <= 3) in the residual helper's registers
    if (p->dev.seedA != nullptr) return p->dev.kx1 <= 6 && p->dev.level >= 3 && p->dev.level <= 10 && p->dev.akx1 <= 4;
    return p->dev.kx1 <= 6 && p->dev.level >= 3 && p->dev.level <= 10 &&
           (p->dev.arow != nullptr || p->dev.arows != nullptr || p->dev.sepk != nullptr);
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

// The workspace's "last call finished" event, usable inside a stream capture (CUDA graph of a multigrid
// cycle): there the wait / record become external event nodes; outside a capture the plain calls.
static bool capturing(cudaStream_t s)
{
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive;
}
static void ws_wait(cudaEvent_t e, cudaStream_t s) { cudaStreamWaitEvent(s, e, capturing(s) ? cudaEventWaitExternal : 0); }
static void ws_record(cudaEvent_t e, cudaStream_t s)
{
    cudaEventRecordWithFlags(e, s, capturing(s) ? cudaEventRecordExternal : 0);
}

// `sweeps` smoothing steps on one macro-tet in the reference layout: pack, sweeps, unpack.
int plane_sweep(const tilu_plan *cp, double *u, const double *f, int ntets, int sweeps, double *rnorm2,
                cudaStream_t s, int *launches, bool stored)
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
    ws_wait(w->done, s);
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
    A.pe = plane_elems(w->g);
    std::memcpy(A.arow, p->harow, sizeof(A.arow));
    A.stored = stored ? 1 : 0;
    if (stored && !p->dev.factors) return TILU_EINVAL;
    const bool exact = !(p->flags & TILU_FAST);
    static const char *trace_path = std::getenv("TILU_PLANE_TRACE");  // file: per-task timeline of the last sweep
    if (trace_path && !w->trace) cudaMalloc(&w->trace, 2 * (size_t)w->ntasks * TR * sizeof(long long));
    static const char *steplog_path = std::getenv("TILU_PLANE_STEPLOG");
    if (steplog_path && !w->steplog) {
        cudaMalloc(&w->steplog, 2 * 3 * PW * 8 * sizeof(long long));
        cudaMemset(w->steplog, 0, 2 * 3 * PW * 8 * sizeof(long long));
    }
    prof_begin(s);
    launch_xpose(P, w->g, u, w->u, false, s);
    k_plane_pack_boundary<<<dim3(P.n + 1, P.n + 1), 128, 0, s>>>(P.n, w->g, u, w->u);
    ++nl;
    launch_xpose(P, w->g, f, w->f, false, s);
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
        A.steplog = w->steplog;
        {
            static const char *pt = std::getenv("TILU_PLANE_PROF_TASK");
            A.prof_task = pt ? std::atoi(pt) : 0;
        }
        prof_begin(s);
#ifdef TILU_PLANE_FUSED_BUILD
        const bool fused = fused_ok(P, stored);
        bool ok = fused ? launchf_pass(P, A, w->mapsf, w->ctas, exact, true, s)
                        : launch_pass(P, A, w->maps, w->ctas, exact, true, s);
#else
        bool ok = launch_pass(P, A, w->maps, w->ctas, exact, true, s);
#endif
        prof_end("plane_fwd", s);
        A.ticket = w->ticket + 1;
        A.part = nullptr;
        A.trace = w->trace ? w->trace + (size_t)w->ntasks * TR : nullptr;
        A.steplog = w->steplog ? w->steplog + 3 * PW * 8 : nullptr;
        static const char *dbg = std::getenv("TILU_PLANE_DEBUG");  // "1": forward pass only, return w_f
        if (dbg && dbg[0] == '1') {
            launch_xpose(P, w->g, w->W, u, true, s);
            w->armed = false;
            ws_record(w->done, s);
            return ok ? TILU_OK : TILU_EUNSUPPORTED;
        }
        prof_begin(s);
#ifdef TILU_PLANE_FUSED_BUILD
        ok = ok && (fused ? launchf_pass(P, A, w->mapsf, w->ctas, exact, false, s)
                          : launch_pass(P, A, w->maps, w->ctas, exact, false, s));
#else
        ok = ok && launch_pass(P, A, w->maps, w->ctas, exact, false, s);
#endif
        prof_end("plane_bwd", s);
        nl += 2;
        if (!ok) rc = TILU_EUNSUPPORTED;
        if (rnorm2 && ok) {
            k_plane_norm<<<1, 1024, 0, s>>>(w->part, w->ntasks * PW * 32, rnorm2 + k);
            ++nl;
        }
    }
    if (steplog_path && w->steplog) {
        std::vector<long long> h(2 * 3 * PW * 8);
        cudaMemcpy(h.data(), w->steplog, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        if (FILE *fp = std::fopen(steplog_path, "w")) {
            std::fprintf(fp, "warp total armed ringwait tmawait acquire groups chain tail  (fused: total armed tma cpwait acquire plain - groups; rows 12.. = backward)\n");
            for (int wv = 0; wv < 2 * 3 * PW; ++wv) {
                std::fprintf(fp, "%d", wv);
                for (int i = 0; i < 8; ++i) std::fprintf(fp, " %lld", h[wv * 8 + i]);
                std::fprintf(fp, "\n");
            }
            std::fclose(fp);
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
    launch_xpose(P, w->g, w->u, u, true, s);
    prof_end("plane_unpack", s);
    ++nl;
    if (cudaGetLastError() != cudaSuccess) {
        rc = TILU_ECUDA;
        w->armed = false;
    }
    ws_record(w->done, s);
    if (launches) *launches += nl;
    return rc;
}

}  // namespace tilu
