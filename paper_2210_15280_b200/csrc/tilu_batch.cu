// Batched fast path: many macro-tets that share one surrogate (identical operator, e.g. the
// 384 Kuhn tets of config 4) swept together in an interleaved layout.
//
// Layout ("packed"): tets are grouped by 32; group g stores fp64 [grid][32], i.e. the 32 tets'
// values of one lattice point are one 256-byte segment.  A warp processes one lattice row for
// the 32 tets of its group (lane = tet), so every load and store of u, f, w is a fully
// coalesced 256 B access, no lane is ever idle, and each lane executes exactly the reference's
// serial operation sequence for its own tet (bitwise parity in exact mode).
//
// Execution: dataflow, no barriers on the compute path.  One CTA per (group, z-layer); CTAs take
// tickets in dependency order (ascending z forward, descending backward), so a CTA only ever
// waits for CTAs that already run: deadlock-free for any residency.  Inside a CTA, BW compute
// warps claim the layer's rows one at a time from a shared counter (in y order forward, reverse
// order backward) and each publishes its row's progress (points done) in shared memory with
// st.release.cta after every point.  Before touching point x (and the point it prefetches) a warp
// checks exactly the rows it reads: the previous row of its own layer (shared memory,
// ld.acquire.cta = plain LDS) and the two rows of the neighbouring layer (global progress array,
// relaxed gpu-scope loads, cached in registers and re-polled only when insufficient).  One sync
// warp per CTA mirrors the shared progress array to global memory behind one st.release.gpu
// (MEMBAR.GPU, cumulative over what it observed) per round, off the compute path.
// Polling uses relaxed loads: ld.acquire.gpu / __threadfence emit CCTL.IVALL on sm_100a (whole-L1
// invalidation) and would wipe the u reuse in L1; a consumer never touches a w line before its
// producer wrote it, and cross-layer data is read with ld.global.cg after the progress value has
// returned, so no stale copy can be observed.
//
// Forward kernel  = residual f - A u (15-point stencil) + forward L substitution, writes w.
// Backward kernel = D^{-1} scaling + L^T substitution + u += w, writes w (in place) and u.
// Every load of point x+1 is issued while point x computes (one-point software prefetch).
#include <algorithm>
#include <cstdio>

#include "tilu_batch.cuh"
#include "tilu_common.cuh"
#include "tilu_plan.cuh"

namespace tilu {

__device__ __forceinline__ int ld_relaxed(const int *p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(int *p, int v)
{
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cta(const int *p)
{
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta(int *p, int v)
{
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

// Warp-wide wait until *flag >= need (flag in shared or global memory).  Only lane 0 polls; the
// warp then reconverges through __syncwarp(), which also orders lane 0's acquire before every
// lane's subsequent loads.  (Letting all lanes poll is unsafe under independent thread scheduling:
// lanes can leave the loop at different times while the compiler keeps the warp-uniform row
// index in a uniform register -- observed as an out-of-range shared access.)  A dependency bug
// must fail loudly, not hang the device: after ~10 s of polling the kernel traps.
__device__ __forceinline__ int wait_shared(const int *flag, int need, int lane)
{
    int v = 0;
    if (lane == 0) {
        long long polls = 0;
        while ((v = ld_acquire_cta(flag)) < need) {
            __nanosleep(32);
            if (++polls > (1ll << 28)) __trap();
        }
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, v, 0);
}
__device__ __forceinline__ int wait_global(const int *flag, int need, int lane)
{
    int v = 0;
    if (lane == 0) {
        long long polls = 0;
        while ((v = ld_relaxed(flag)) < need) {
            __nanosleep(64);
            if (++polls > (1ll << 27)) __trap();
        }
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, v, 0);
}

__device__ __forceinline__ bool in_band_b(int x, int y, int z, int xe) { return z == 1 || y == 1 || x == 1 || x == xe; }

// Debug build (-DTILU_DEBUG_BOUNDS): every packed / table access is range-checked.
#ifdef TILU_DEBUG_BOUNDS
#define TILU_CHECK(cond, what, a, b)                                                                  \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("tilu bounds: %s (%lld, %lld) block %d thread %d\n", what, (long long)(a), (long long)(b), \
                   blockIdx.x, threadIdx.x);                                                          \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define TILU_CHECK(cond, what, a, b) ((void)0)
#endif

// Sync warp: mirror this layer's per-row progress (shared) to the global array the neighbouring
// layer polls.  Each round: read all rows, one st.release.gpu (MEMBAR.GPU, cumulative over the
// observed progress and thus over the w stores it covers), then relaxed stores of the values.
__device__ __forceinline__ void progress_mirror(const int *s_prog, const int *s_done, int *gp, int R, int lane)
{
    constexpr int PER = (MAXR + 31) / 32;
    for (;;) {
        const int done = ld_acquire_cta(s_done);
        int v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int y = lane + 1 + 32 * k;
            v[k] = y <= R ? ld_acquire_cta(&s_prog[y]) : 0;
        }
        __syncwarp();
        if (lane == 0) st_release(&gp[MAXR + 2], done);  // the MEMBAR.GPU of this round
        __syncwarp();
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int y = lane + 1 + 32 * k;
            if (y <= R) st_relaxed(&gp[y], v[k]);
        }
        if (done >= R) return;  // `done` was read before the values: they are final
        __nanosleep(256);
    }
}

// ----------------------------------------------------------------------------------------------
// Shared NDDF tables: every lane of a warp works on a different tet of the SAME lattice row and
// all tets share the surrogate, so the forward-difference tables are identical across lanes.
// They live once per warp in shared memory and one forward-difference step is done lane-parallel:
// lane e updates entry e (d[m][j] += d[m][j+1]), reading all old values before any write --
// the same unfused additions as the reference's serial march (_kernels.py:313-316), 28-32 lanes
// busy instead of 28-32 dependent-free adds in every lane.
// ----------------------------------------------------------------------------------------------
template <int M, int K>
__device__ __forceinline__ void smem_load_table(double *tab, const double *__restrict__ src, int lane)
{
    for (int e = lane; e < M * K; e += 32) tab[e] = src[e];
    __syncwarp();
}

template <int M, int K>
__device__ __forceinline__ void smem_march(double *tab, int lane)
{
    constexpr int NE = M * (K - 1);
    if (NE == 0) return;
    constexpr int IT = NE > 0 ? (NE + 31) / 32 : 1;
    double nv[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const int e = lane + 32 * i;
        if (e < NE) {
            const int m = e / (K - 1), j = e - m * (K - 1);
            nv[i] = dadd(tab[m * K + j], tab[m * K + j + 1]);
        }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const int e = lane + 32 * i;
        if (e < NE) {
            const int m = e / (K - 1), j = e - m * (K - 1);
            tab[m * K + j] = nv[i];
        }
    }
    __syncwarp();
}

// ----------------------------------------------------------------------------------------------
// forward: residual + L solve
// ----------------------------------------------------------------------------------------------
struct FwdSlot {
    double ue, us, un, ubn, ubc, uts, utc, f, ws, wbn, wbc;
};

struct FwdRow {
    int y, m, rid, boff;
    uint32_t oc, os, on, obn, obc, ots, otc;
};

__device__ __forceinline__ void fwd_load(FwdSlot &S, const double *__restrict__ u, const double *__restrict__ f,
                                         const double *__restrict__ w, const FwdRow &R, int p)
{
    const uint32_t X = (uint32_t)p * 32u;
    TILU_CHECK(p >= 1 && p <= R.m, "fwd_load p", p, R.m);
    S.ue = u[R.oc + X + 32];
    S.us = u[R.os + X + 32];
    S.un = u[R.on + X];
    S.ubn = u[R.obn + X];
    S.ubc = u[R.obc + X + 32];
    S.uts = u[R.ots + X + 32];
    S.utc = u[R.otc + X];
    S.f = f[R.oc + X];
    S.ws = w[R.os + X + 32];          // same layer: written by a warp of this CTA
    S.wbn = ldcg(w + R.obn + X);      // layer below: written by another CTA
    S.wbc = ldcg(w + R.obc + X + 32);
}

// Lane m < 7 fetches the V1 band-store entry L_m of point p (uniform over the warp's tets).
__device__ __forceinline__ void fwd_band_load(double &dst, const PlanDev &P, const FwdRow &R, int z, int p, int lane)
{
    if (P.variant == 1 && lane < 7 && in_band_b(p, R.y, z, R.m)) {
        TILU_CHECK(R.boff + ((z == 1 || R.y == 1) ? p - 1 : (p == 1 ? 0 : 1)) < P.nband_dbg, "fwd band", R.boff, p);
        dst = P.store[9 * (int64_t)(R.boff + ((z == 1 || R.y == 1) ? p - 1 : (p == 1 ? 0 : 1))) + lane];
    }
}

template <int K, bool EXACT, bool CONST_ROW>
__global__ void __launch_bounds__(NT, 2) k_batch_fwd(PlanDev P, BatchArgs A)
{
    __shared__ int s_ticket, s_next, s_done;
    __shared__ int s_prog[MAXR + 2];
    __shared__ double s_red[BW][32];
    __shared__ double s_tab[BW][7 * K];
    __shared__ double s_L[BW][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_ticket = atomicAdd(A.ticket, 1);
        s_next = 0;
        s_done = 0;
    }
    for (int i = threadIdx.x; i < MAXR + 2; i += NT) s_prog[i] = i == 0 ? (1 << 30) : 0;  // row 0: boundary
    __syncthreads();
    if (A.max_ticket >= 0 && s_ticket > A.max_ticket) return;
    const int nl = P.n - 3, n = P.n;
    TILU_CHECK(s_ticket < A.G * nl, "fwd ticket", s_ticket, A.G);
    const int zi = s_ticket / A.G, g = s_ticket - (s_ticket / A.G) * A.G;
    const int z = zi + 1, Rn = n - 2 - z;
    int *gp = A.gprog + ((size_t)g * nl + zi) * GSTRIDE;
    const int *gb = z > 1 ? gp - GSTRIDE : nullptr;  // layer below
    double ss = 0.0;
    if (warp == BW) {
        progress_mirror(s_prog, &s_done, gp, Rn, lane);
    } else {
        const size_t gbase = (size_t)g * P.grid * 32 + lane;
        const double *__restrict__ u = A.u + gbase;
        const double *__restrict__ f = A.f + gbase;
        double *__restrict__ w = A.w + gbase;
        double *tab = s_tab[warp];
        double *sL = s_L[warp];
        for (;;) {
            int y = 0;
            if (lane == 0) y = atomicAdd(&s_next, 1) + 1;
            y = __shfl_sync(0xffffffffu, y, 0);
            if (y > Rn) break;
            TILU_CHECK(y >= 1 && y <= Rn && z >= 1 && z <= nl, "fwd row", y, z);
            FwdRow R;
            R.y = y;
            R.m = n - 1 - z - y;
            R.rid = row_id(n, z, y);
            R.oc = (uint32_t)row_offset(n, z, y) * 32u;
            R.os = (uint32_t)row_offset(n, z, y - 1) * 32u;
            R.on = (uint32_t)row_offset(n, z, y + 1) * 32u;
            R.obn = (uint32_t)row_offset(n, z - 1, y + 1) * 32u;
            R.obc = (uint32_t)row_offset(n, z - 1, y) * 32u;
            R.ots = (uint32_t)row_offset(n, z + 1, y - 1) * 32u;
            R.otc = (uint32_t)row_offset(n, z + 1, y) * 32u;
            R.boff = P.variant == 1 ? P.bandoff[R.rid] : 0;
            const int m = R.m;
            smem_load_table<7, K>(tab, P.seedF + (int64_t)R.rid * 7 * K, lane);
            // dependencies of point p: row y-1 of this layer (length m+1) up to p+1; the layer
            // below: row y (length m+1) up to p+1 and row y+1 (length m) up to p
            int cs = 0, cby = 0, cbn = 0;
            auto ensure = [&](int p) {
                if (cs < p + 1) cs = wait_shared(&s_prog[y - 1], p + 1, lane);
                if (gb) {
                    if (cby < p + 1) cby = wait_global(&gb[y], p + 1, lane);
                    if (cbn < p) cbn = wait_global(&gb[y + 1], p, lane);
                }
            };
            ensure(1);
            // sliding windows (values of point x-1 / x that point x+1 reuses) and point 1
            double u_wm = u[R.oc], u_c = u[R.oc + 32], us0 = u[R.os + 32], un_m = u[R.on], ubn_m = u[R.obn];
            double ubc0 = u[R.obc + 32], uts0 = u[R.ots + 32], utc_m = u[R.otc];
            double ws0 = w[R.os + 32], wbn_m = ldcg(w + R.obn), wbc0 = ldcg(w + R.obc + 32), wprev = 0.0;
            FwdSlot C, N;
            fwd_load(C, u, f, w, R, 1);
            double cband = 0.0, nband = 0.0;
            fwd_band_load(cband, P, R, z, 1, lane);
            for (int x = 1; x <= m; ++x) {
                const int pn = min(x + 1, m);  // prefetch (at the row end: re-read point m, unused)
                ensure(pn);
                fwd_load(N, u, f, w, R, pn);
                fwd_band_load(nband, P, R, z, pn, lane);
                double ap[15];
                const double *a = A.arow;
                if (!CONST_ROW) {
                    const double *ar = P.arows + 15 * (int64_t)(R.oc / 32u + x);
#pragma unroll
                    for (int i = 0; i < 15; ++i) ap[i] = ar[i];
                    a = ap;
                }
                // residual in stencil_apply order (_kernels.py:255-266), then f - A u
                double acc = EXACT ? dmul(a[7], u_c) : a[7] * u_c;
                acc = madd<EXACT>(acc, a[0], u_wm);
                acc = madd<EXACT>(acc, a[1], us0);
                acc = madd<EXACT>(acc, a[2], C.us);
                acc = madd<EXACT>(acc, a[3], ubn_m);
                acc = madd<EXACT>(acc, a[4], C.ubn);
                acc = madd<EXACT>(acc, a[5], ubc0);
                acc = madd<EXACT>(acc, a[6], C.ubc);
                acc = madd<EXACT>(acc, a[8], C.ue);
                acc = madd<EXACT>(acc, a[9], C.un);
                acc = madd<EXACT>(acc, a[10], un_m);
                acc = madd<EXACT>(acc, a[11], C.uts);
                acc = madd<EXACT>(acc, a[12], uts0);
                acc = madd<EXACT>(acc, a[13], C.utc);
                acc = madd<EXACT>(acc, a[14], utc_m);
                const double r = dsub(C.f, acc);
                ss = fma(r, r, ss);
                // L entries: lane m publishes L_m (band store or the shared NDDF table)
                if (lane < 7) sL[lane] = (P.variant == 1 && in_band_b(x, y, z, m)) ? cband : tab[lane * K];
                __syncwarp();
                double v;
                if (EXACT) {  // reference order: own-row term first (_kernels.py:349-364)
                    v = msub<true>(r, sL[0], wprev);
                    v = msub<true>(v, sL[1], ws0);
                    v = msub<true>(v, sL[2], C.ws);
                    v = msub<true>(v, sL[3], wbn_m);
                    v = msub<true>(v, sL[4], C.wbn);
                    v = msub<true>(v, sL[5], wbc0);
                    v = msub<true>(v, sL[6], C.wbc);
                } else {  // own-row term last: one FMA on the row's dependency chain
                    v = msub<false>(r, sL[1], ws0);
                    v = msub<false>(v, sL[2], C.ws);
                    v = msub<false>(v, sL[3], wbn_m);
                    v = msub<false>(v, sL[4], C.wbn);
                    v = msub<false>(v, sL[5], wbc0);
                    v = msub<false>(v, sL[6], C.wbc);
                    v = msub<false>(v, sL[0], wprev);
                }
                w[R.oc + (uint32_t)x * 32u] = v;
                smem_march<7, K>(tab, lane);  // ends with __syncwarp: orders this point's stores
                if (lane == 0) st_release_cta(&s_prog[y], x);
                u_wm = u_c;
                u_c = C.ue;
                us0 = C.us;
                un_m = C.un;
                ubn_m = C.ubn;
                ubc0 = C.ubc;
                uts0 = C.uts;
                utc_m = C.utc;
                ws0 = C.ws;
                wbn_m = C.wbn;
                wbc0 = C.wbc;
                wprev = v;
                C = N;
                cband = nband;
            }
            if (lane == 0) atomicAdd(&s_done, 1);
        }
    }
    if (A.part) {
        if (warp < BW) s_red[warp][lane] = ss;
        __syncthreads();
        if (warp == 0) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < BW; ++k) t += s_red[k][lane];
            A.part[((int64_t)g * nl + zi) * 32 + lane] = t;
        }
    }
}

// ----------------------------------------------------------------------------------------------
// backward: D^{-1} + L^T solve + update (rows in descending y, points in descending x)
// ----------------------------------------------------------------------------------------------
struct BwdSlot {
    double wn, wts, wtc, wf, u;
};

struct BwdRow {
    int y, m, rid;
    int qboff, qrow_band, qxe;  // lane m < 7: band offset / band-row flag / length of the row of
                                // q_m = p - d_m; lane 7: the own row (1/D)
    uint32_t oc, on, ots, otc;
};

__device__ __forceinline__ void bwd_load(BwdSlot &S, const double *__restrict__ u, const double *__restrict__ w,
                                         const BwdRow &R, int x)
{
    const uint32_t X = (uint32_t)x * 32u;
    TILU_CHECK(x >= 1 && x <= R.m, "bwd_load x", x, R.m);
    S.wn = w[R.on + X - 32];         // same layer (row y+1): written by a warp of this CTA
    S.wts = ldcg(w + R.ots + X);     // layer above: written by another CTA
    S.wtc = ldcg(w + R.otc + X - 32);
    S.wf = w[R.oc + X];
    S.u = u[R.oc + X];
}

// Lane m < 7 classifies q_m = p - d_m of point (x, y, z) and fetches its band-store entry L_m
// (_kernels.py:434-441 _lq); lane 7 does the same for 1/D at p.  Returns the source code:
// 0 = q outside the interior, 1 = band store (value in dst), 2 = NDDF table.
__device__ __forceinline__ int bwd_band_load(double &dst, const BwdRow &R, const PlanDev &P, int n, int z, int x,
                                             int lane)
{
    if (lane >= 8) return 2;
    if (lane < 7) {
        const int qx = x - kDX[lane], qy = R.y - kDY[lane], qz = z - kDZ[lane];
        if (!interior(qx, qy, qz, n)) return 0;
        if (P.variant == 1 && (R.qrow_band || qx == 1 || qx == R.qxe)) {
            TILU_CHECK(R.qboff + (R.qrow_band ? qx - 1 : (qx == 1 ? 0 : 1)) < P.nband_dbg, "bwd band q", R.qboff, qx);
            dst = P.store[9 * (int64_t)(R.qboff + (R.qrow_band ? qx - 1 : (qx == 1 ? 0 : 1))) + lane];
            return 1;
        }
        return 2;
    }
    if (P.variant == 1 && in_band_b(x, R.y, z, R.m)) {
        TILU_CHECK(R.qboff + ((z == 1 || R.y == 1) ? x - 1 : (x == 1 ? 0 : 1)) < P.nband_dbg, "bwd band p", R.qboff, x);
        dst = P.store[9 * (int64_t)(R.qboff + ((z == 1 || R.y == 1) ? x - 1 : (x == 1 ? 0 : 1))) + 8];
        return 1;
    }
    return 2;
}

template <int K, bool EXACT>
__global__ void __launch_bounds__(NT, 2) k_batch_bwd(PlanDev P, BatchArgs A)
{
    __shared__ int s_ticket, s_next, s_done;
    __shared__ int s_prog[MAXR + 2];
    __shared__ double s_tab[BW][8 * K];
    __shared__ double s_L[BW][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_ticket = atomicAdd(A.ticket, 1);
        s_next = 0;
        s_done = 0;
    }
    for (int i = threadIdx.x; i < MAXR + 2; i += NT) s_prog[i] = 0;
    __syncthreads();
    if (A.max_ticket >= 0 && s_ticket > A.max_ticket) return;
    const int nl = P.n - 3, n = P.n;
    TILU_CHECK(s_ticket < A.G * nl, "bwd ticket", s_ticket, A.G);
    const int li = s_ticket / A.G, g = s_ticket - li * A.G;
    const int zi = nl - 1 - li;
    const int z = zi + 1, Rn = n - 2 - z;
    if (threadIdx.x == 0) s_prog[Rn + 1] = 1 << 30;  // row R+1 of this layer: boundary
    __syncthreads();
    int *gp = A.gprog + ((size_t)g * nl + zi) * GSTRIDE;
    const int *ga = z < nl ? gp + GSTRIDE : nullptr;  // layer above
    if (warp == BW) {
        progress_mirror(s_prog, &s_done, gp, Rn, lane);
        return;
    }
    const size_t gbase = (size_t)g * P.grid * 32 + lane;
    double *__restrict__ u = A.u + gbase;
    double *__restrict__ w = A.w + gbase;
    double *tab = s_tab[warp];
    double *sL = s_L[warp];
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&s_next, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        const int y = Rn - t;
        if (y < 1) break;
        TILU_CHECK(y <= Rn && z >= 1 && z <= nl, "bwd row", y, z);
        BwdRow R;
        R.y = y;
        R.m = n - 1 - z - y;
        R.rid = row_id(n, z, y);
        R.oc = (uint32_t)row_offset(n, z, y) * 32u;
        R.on = (uint32_t)row_offset(n, z, y + 1) * 32u;
        R.ots = (uint32_t)row_offset(n, z + 1, y - 1) * 32u;
        R.otc = (uint32_t)row_offset(n, z + 1, y) * 32u;
        const int m = R.m;
        if (lane < 8) {  // the row of q_m (lane m) or the own row (lane 7)
            const int qy = lane < 7 ? y - kDY[lane] : y, qz = lane < 7 ? z - kDZ[lane] : z;
            const bool valid = qy >= 1 && qz >= 1 && qy + qz <= n - 2;
            R.qxe = n - 1 - qz - qy;
            R.qrow_band = (qz == 1 || qy == 1);
            R.qboff = (P.variant == 1 && valid) ? P.bandoff[row_id(n, qz, qy)] : 0;
        }
        smem_load_table<8, K>(tab, P.seedB + (int64_t)R.rid * 8 * K, lane);
        // dependencies of the k-th point (x = m - k + 1): row y+1 of this layer (length m-1) and
        // row y of the layer above (length m-1) up to min(k, m-1) points, row y-1 of the layer above
        // (length m) up to k points
        int cn = 0, cts = 0, ctc = 0;
        auto ensure = [&](int k) {
            const int k1 = min(k, m - 1);
            if (cn < k1) cn = wait_shared(&s_prog[y + 1], k1, lane);
            if (ga) {
                if (y >= 2 && cts < k) cts = wait_global(&ga[y - 1], k, lane);
                if (y <= Rn - 1 && ctc < k1) ctc = wait_global(&ga[y], k1, lane);
            }
        };
        ensure(1);
        const uint32_t M = (uint32_t)m * 32u;
        double wn_hi = w[R.on + M], wts_hi = ldcg(w + R.ots + M + 32), wtc_hi = ldcg(w + R.otc + M), wprev = 0.0;
        BwdSlot C, N;
        bwd_load(C, u, w, R, m);
        double cband = 0.0, nband = 0.0;
        int csrc = bwd_band_load(cband, R, P, n, z, m, lane), nsrc = 2;
        for (int k = 1; k <= m; ++k) {
            const int x = m - k + 1;
            const int kn = min(k + 1, m);  // prefetch the next point (at the row end: re-read x = 1)
            ensure(kn);
            const int xn = m - kn + 1;
            bwd_load(N, u, w, R, xn);
            nsrc = bwd_band_load(nband, R, P, n, z, xn, lane);
            if (lane < 8) sL[lane] = csrc == 0 ? 0.0 : (csrc == 1 ? cband : tab[lane * K]);
            __syncwarp();
            const double inv_d = sL[7];
            double v = EXACT ? dmul(inv_d, C.wf) : inv_d * C.wf;
            if (EXACT) {  // reference order (_kernels.py:404-425)
                v = msub<true>(v, sL[0], wprev);
                v = msub<true>(v, sL[1], wn_hi);
                v = msub<true>(v, sL[2], C.wn);
                v = msub<true>(v, sL[3], wts_hi);
                v = msub<true>(v, sL[4], C.wts);
                v = msub<true>(v, sL[5], wtc_hi);
                v = msub<true>(v, sL[6], C.wtc);
            } else {
                v = msub<false>(v, sL[1], wn_hi);
                v = msub<false>(v, sL[2], C.wn);
                v = msub<false>(v, sL[3], wts_hi);
                v = msub<false>(v, sL[4], C.wts);
                v = msub<false>(v, sL[5], wtc_hi);
                v = msub<false>(v, sL[6], C.wtc);
                v = msub<false>(v, sL[0], wprev);
            }
            const uint32_t X = (uint32_t)x * 32u;
            w[R.oc + X] = v;
            u[R.oc + X] = dadd(C.u, v);
            smem_march<8, K>(tab, lane);  // ends with __syncwarp: orders this point's stores
            if (lane == 0) st_release_cta(&s_prog[y], k);
            wn_hi = C.wn;
            wts_hi = C.wts;
            wtc_hi = C.wtc;
            wprev = v;
            C = N;
            cband = nband;
            csrc = nsrc;
        }
        if (lane == 0) atomicAdd(&s_done, 1);
    }
}

// ----------------------------------------------------------------------------------------------
// layout conversion and norms
// ----------------------------------------------------------------------------------------------
// dst[g][r][l] = src[g*32+l][r] (zero for padded tets): 32x32 tiles through shared memory.
__global__ void __launch_bounds__(256) k_pack(const double *__restrict__ src, double *__restrict__ dst, int64_t grid,
                                              int ntets)
{
    __shared__ double tile[32][33];
    const int g = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int k = ty; k < 32; k += 8) {
        const int t = g * 32 + k;
        const int64_t r = r0 + tx;
        tile[k][tx] = (t < ntets && r < grid) ? src[(int64_t)t * grid + r] : 0.0;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int64_t r = r0 + k;
        if (r < grid) dst[((int64_t)g * grid + r) * 32 + tx] = tile[tx][k];
    }
}

__global__ void __launch_bounds__(256) k_unpack(const double *__restrict__ src, double *__restrict__ dst, int64_t grid,
                                                int ntets)
{
    __shared__ double tile[32][33];
    const int g = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int k = ty; k < 32; k += 8) {
        const int64_t r = r0 + k;
        tile[k][tx] = (r < grid) ? src[((int64_t)g * grid + r) * 32 + tx] : 0.0;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int t = g * 32 + k;
        const int64_t r = r0 + tx;
        if (t < ntets && r < grid) dst[(int64_t)t * grid + r] = tile[tx][k];
    }
}

// rnorm2[t] = sum over layers of the forward kernel's per-(layer, lane) partials, fixed order.
__global__ void k_batch_norms(const double *__restrict__ part, int nl, int ntets, double *__restrict__ out)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntets) return;
    const int g = t / 32, l = t % 32;
    double s = 0.0;
    for (int zi = 0; zi < nl; ++zi) s += part[((int64_t)g * nl + zi) * 32 + l];
    out[t] = s;
}

// ----------------------------------------------------------------------------------------------
// host launchers
// ----------------------------------------------------------------------------------------------
void launch_pack(const double *src, double *dst, int64_t grid, int ntets, cudaStream_t s)
{
    dim3 gr((unsigned)((grid + 31) / 32), (unsigned)((ntets + 31) / 32));
    k_pack<<<gr, 256, 0, s>>>(src, dst, grid, ntets);
}

void launch_unpack(const double *src, double *dst, int64_t grid, int ntets, cudaStream_t s)
{
    dim3 gr((unsigned)((grid + 31) / 32), (unsigned)((ntets + 31) / 32));
    k_unpack<<<gr, 256, 0, s>>>(src, dst, grid, ntets);
}

void launch_batch_norms(const double *part, int nl, int ntets, double *out, cudaStream_t s)
{
    k_batch_norms<<<(ntets + 127) / 128, 128, 0, s>>>(part, nl, ntets, out);
}

template <int K>
static void launch_fwd_k(const PlanDev &P, const BatchArgs &A, bool exact, cudaStream_t s)
{
    const unsigned grid = (unsigned)(A.G * (P.n - 3));
    const bool c = P.arow != nullptr;
    if (exact) {
        if (c) k_batch_fwd<K, true, true><<<grid, NT, 0, s>>>(P, A);
        else k_batch_fwd<K, true, false><<<grid, NT, 0, s>>>(P, A);
    } else {
        if (c) k_batch_fwd<K, false, true><<<grid, NT, 0, s>>>(P, A);
        else k_batch_fwd<K, false, false><<<grid, NT, 0, s>>>(P, A);
    }
}

template <int K>
static void launch_bwd_k(const PlanDev &P, const BatchArgs &A, bool exact, cudaStream_t s)
{
    const unsigned grid = (unsigned)(A.G * (P.n - 3));
    if (exact) k_batch_bwd<K, true><<<grid, NT, 0, s>>>(P, A);
    else k_batch_bwd<K, false><<<grid, NT, 0, s>>>(P, A);
}

bool launch_batch_pass(const PlanDev &P, const BatchArgs &A, bool exact, bool fwd, cudaStream_t s)
{
#define TILU_CASE(KK) \
    case KK: fwd ? launch_fwd_k<KK>(P, A, exact, s) : launch_bwd_k<KK>(P, A, exact, s); return true;
    switch (P.kx1) {
        TILU_CASE(1) TILU_CASE(2) TILU_CASE(3) TILU_CASE(4) TILU_CASE(5) TILU_CASE(6) TILU_CASE(7) TILU_CASE(8)
        TILU_CASE(9)
    default: return false;
    }
#undef TILU_CASE
}

}  // namespace tilu
