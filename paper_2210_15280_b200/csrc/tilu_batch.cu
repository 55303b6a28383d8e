// Batched fast path: many macro-tets that share one surrogate (identical operator, e.g. the
// 384 Kuhn tets of config 4) swept together in an interleaved layout.
//
// Layout ("packed"): tets are grouped by 32; group g stores fp64 [grid][32], i.e. the 32 tets'
// values of one lattice point are one 256-byte segment.  A warp processes one lattice row for
// the 32 tets of its group (lane = tet), so every load and store of u, f, w is a fully
// coalesced 256 B access, no lane is ever idle, and each lane executes exactly the reference's
// serial operation sequence for its own tet (bitwise parity in exact mode).
//
// Schedule: one CTA per (group, z-layer), BW warps per CTA, each warp owns one row of the layer
// at a time.  A host-side greedy list schedule (batch_schedule below) gives every row (y, z) a
// start step S: point (x, y, z) runs at forward step S + x - 1, rows start in y order as soon as
//   * a warp of the CTA is free,
//   * S(y) >= S(y-1) + AMIN: row y reads row y-1 (same layer, another warp) only from
//     synchronisation windows already closed by a CTA barrier, even one point ahead (prefetch);
//     the CTA therefore synchronises once per BWIN steps, not per step;
//   * S_z(y) >= S_{z-1}(y+1) + 1 + D and >= S_{z-1}(y) + 2 + D: everything read from the layer
//     below (another CTA, usually another SM) was produced >= D + 1 steps earlier.  Layers hand
//     over through release/acquire progress counters published at every window end; D is slack
//     so the consumer rarely waits.
// The backward pass runs the exact time reversal of this schedule (T_b = Tmax - T), which
// satisfies the transposed dependencies.  CTAs take (group, layer) tickets in layer order
// (ascending z forward, descending backward), so a CTA only ever waits for CTAs that already
// hold earlier tickets: no deadlock whatever the residency.  tests/test_schedule.py verifies
// dependencies, warp exclusivity and handoff completion on the host.
//
// Forward kernel  = residual f - A u (15-point stencil) + forward L substitution, writes w.
// Backward kernel = D^{-1} scaling + L^T substitution + u += w, writes w (in place) and u.
// Every load of point x+1 is issued while point x computes (one-point software prefetch).
#include <algorithm>

#include "tilu_batch.cuh"
#include "tilu_common.cuh"
#include "tilu_plan.cuh"

namespace tilu {

// Progress counters are polled with relaxed gpu-scope loads: ld.acquire.gpu would emit
// CCTL.IVALL (invalidate the SM's whole L1) on every poll and wipe the u-reuse the compute warps
// rely on.  No acquire is needed for correctness here: a consumer never touches a w line before
// its producer wrote it (dependency order), so L1 cannot hold a stale copy, and the consumer's
// data loads are issued only after the flag value has returned (control dependency + bar.sync).
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
__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

// Thread 0 waits until the neighbouring layer's progress counter reaches `need`.  A schedule bug
// must fail loudly, not hang the device: after ~10 s of polling the kernel traps.
__device__ __forceinline__ void wait_progress(const int *flag, int need)
{
    long long polls = 0;
    while (ld_relaxed(flag) < need) {
        __nanosleep(64);
        if (++polls > (1ll << 27)) __trap();
    }
}

// The sync warp (warp BW) of a CTA: window by window it publishes the CTA's progress (fence +
// release, after the barrier that closes the window) and makes sure the data the NEXT window
// reads from the neighbouring layer is published before it arrives at the barrier that opens it.
// Compute warps only ever meet it at that one barrier per window.
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// trace layout per CTA (8 x u64): start ns, first-window-open ns, end ns, sync-warp dependency-wait
// cycles, sync-warp release (MEMBAR) cycles, warp-0 barrier-wait cycles, warp-0 step cycles, windows
constexpr int TRACE_W = 8;

__device__ __forceinline__ void sync_warp_loop(int *myflag, const int *dep, int depEnd, int D, int t0, int t1,
                                               unsigned long long *trace)
{
    // everything a window starting at tau0 reads from the neighbouring layer (including the PF-ahead
    // prefetches) has step <= tau0 + BWIN + PF - 2 - D; the neighbour never publishes past depEnd
    const bool leader = (threadIdx.x & 31) == 0;
    unsigned long long waited = 0, released = 0, nwin = 0;
    if (trace && leader) trace[0] = gtimer();
    if (leader && dep) wait_progress(dep, min(t0 + BWIN + PF - 2 - D, depEnd));
    if (trace && leader) trace[1] = gtimer();
    __syncthreads();  // opens the first window
    for (int tau0 = t0; tau0 <= t1; tau0 += BWIN) {
        const int tau1 = tau0 + BWIN;
        if (leader && dep && tau1 <= t1) {
            const long long a = trace ? clock64() : 0;
            wait_progress(dep, min(tau1 + BWIN + PF - 2 - D, depEnd));
            if (trace) waited += clock64() - a;
        }
        __syncthreads();  // closes this window / opens the next
        if (leader) {
            const long long a = trace ? clock64() : 0;
            st_release(myflag, min(tau1, t1 + 1) - 1);  // MEMBAR.GPU + store, cumulative over the barrier
            if (trace) released += clock64() - a;
        }
        ++nwin;
    }
    if (trace && leader) {
        trace[2] = gtimer();
        trace[3] = waited;
        trace[4] = released;
        trace[7] = nwin;
    }
}

__device__ __forceinline__ bool in_band_b(int x, int y, int z, int xe) { return z == 1 || y == 1 || x == 1 || x == xe; }
__device__ __forceinline__ int band_idx_b(const PlanDev &P, int row, int x, int y, int z)
{
    return P.bandoff[row] + ((z == 1 || y == 1) ? x - 1 : (x == 1 ? 0 : 1));
}

__device__ __forceinline__ double lq_b(const PlanDev &P, int m, int qx, int qy, int qz, double dval)
{
    const int n = P.n;
    if (!interior(qx, qy, qz, n)) return 0.0;
    if (P.variant == 1) {
        const int xe = n - 1 - qz - qy;
        if (in_band_b(qx, qy, qz, xe)) return P.store[9 * (int64_t)band_idx_b(P, row_id(n, qz, qy), qx, qy, qz) + m];
    }
    return dval;
}

// ----------------------------------------------------------------------------------------------
// host: greedy list schedule
// ----------------------------------------------------------------------------------------------
void batch_schedule(int n, int bwin, int pf, std::vector<LayerSched> &layers, std::vector<RowSched> &rows, int &Tmax,
                    int &D)
{
    const int nl = n - 3;
    const int amin = bwin + 1 + pf;
    D = 2 * bwin + 1 + pf;
    layers.assign(nl, LayerSched{});
    rows.assign((size_t)(n - 3) * (n - 2) / 2 + 1, RowSched{0, 0, 0});
    Tmax = 0;
    for (int z = 1; z <= nl; ++z) {
        const int R = n - 2 - z;
        LayerSched &L = layers[z - 1];
        int free_at[BW], lastrow[BW];
        for (int w = 0; w < BW; ++w) {
            free_at[w] = 0;
            lastrow[w] = 0;
            L.first[w] = L.last[w] = 0;
        }
        int prev_start = -(1 << 29);
        L.T0 = 1 << 30;
        L.T1 = 0;
        for (int y = 1; y <= R; ++y) {
            const int m = n - 1 - z - y;
            int t = std::max(0, prev_start + amin);
            if (z > 1) {
                t = std::max(t, rows[row_id(n, z - 1, y + 1)].start + 1 + D);
                t = std::max(t, rows[row_id(n, z - 1, y)].start + 2 + D);
            }
            int wbest = 0;
            for (int w = 1; w < BW; ++w)
                if (free_at[w] < free_at[wbest]) wbest = w;
            t = std::max(t, free_at[wbest]);
            RowSched &rs = rows[row_id(n, z, y)];
            rs.start = t;
            rs.next = 0;
            rs.prev = lastrow[wbest];
            if (lastrow[wbest]) rows[row_id(n, z, lastrow[wbest])].next = y;
            else L.first[wbest] = y;
            lastrow[wbest] = y;
            L.last[wbest] = y;
            free_at[wbest] = t + m;
            prev_start = t;
            L.T0 = std::min(L.T0, t);
            L.T1 = std::max(L.T1, t + m - 1);
        }
        Tmax = std::max(Tmax, L.T1);
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
#ifdef TILU_ABLATE_NOMARCH
    return;
#endif
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
//
// Per compute warp: one row at a time.  Loads run PF points ahead through a RING-slot register
// ring; the window loop is unrolled RING (= BWIN) times so every ring index is a compile-time
// constant: the point processed at step tau uses slot (tau - T0) % RING, the prefetch issued at
// tau fills slot (tau + PF - T0) % RING.
// ----------------------------------------------------------------------------------------------
struct FwdSlot {
    double ue, us, un, ubn, ubc, uts, utc, f, ws, wbn, wbc;
};

struct FwdRow {
    int y, m, rid, start;
    int boff;           // first band-store entry of the row (V1)
    uint32_t oc, os, on, obn, obc, ots, otc;
    double lring[RING];  // lane m < 7: prefetched band-store entry L_m of the slot's point (V1)
    // sliding windows: the values of point x-1 / x that point x+1 reuses
    double u_wm, u_c, us0, un_m, ubn_m, ubc0, uts0, utc_m, ws0, wbn_m, wbc0, wprev;
    FwdSlot ring[RING];
    double ss;
};

__device__ __forceinline__ void fwd_load(FwdSlot &S, const double *__restrict__ u, const double *__restrict__ f,
                                         const double *__restrict__ w, const FwdRow &R, int p)
{
    const uint32_t X = (uint32_t)p * 32u;
#ifdef TILU_ABLATE_NOLOAD
    S.ue = X * 1e-9; S.us = S.ue + 1; S.un = S.ue + 2; S.ubn = S.ue + 3; S.ubc = S.ue + 4; S.uts = S.ue + 5;
    S.utc = S.ue + 6; S.f = S.ue + 7; S.ws = S.ue + 8; S.wbn = S.ue + 9; S.wbc = S.ue + 10;
    return;
#endif
    S.ue = u[R.oc + X + 32];
    S.us = u[R.os + X + 32];
    S.un = u[R.on + X];
    S.ubn = u[R.obn + X];
    S.ubc = u[R.obc + X + 32];
    S.uts = u[R.ots + X + 32];
    S.utc = u[R.otc + X];
    S.f = f[R.oc + X];
    S.ws = ldcg(w + R.os + X + 32);
    S.wbn = ldcg(w + R.obn + X);
    S.wbc = ldcg(w + R.obc + X + 32);
}

// Lane m < 7 fetches the V1 band-store entry L_m of point p (uniform over the warp's tets) ahead.
__device__ __forceinline__ void fwd_band_load(double &dst, const PlanDev &P, const FwdRow &R, int z, int p, int lane)
{
    if (P.variant == 1 && lane < 7 && in_band_b(p, R.y, z, R.m))
        dst = P.store[9 * (int64_t)(R.boff + ((z == 1 || R.y == 1) ? p - 1 : (p == 1 ? 0 : 1))) + lane];
}

template <int K, bool EXACT, bool CONST_ROW>
__global__ void __launch_bounds__(NT, 2) k_batch_fwd(PlanDev P, BatchArgs A)
{
    // Rolled step loop with a current / next load buffer (one point of prefetch): smaller code and
    // register footprint than the unrolled ring, which lets two CTAs (18 warps) share an SM.
    __shared__ int s_ticket;
    __shared__ double s_red[BW][32];
    __shared__ double s_tab[BW][7 * K];
    __shared__ double s_L[BW][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_ticket = atomicAdd(A.ticket, 1) + 1;  // counter starts at -1
    __syncthreads();
    if (A.max_ticket >= 0 && s_ticket > A.max_ticket) return;
    const int nl = P.n - 3;
    const int zi = s_ticket / A.G, g = s_ticket - (s_ticket / A.G) * A.G;
    const int n = P.n, z = zi + 1;
    const int T0 = A.sched[zi].T0, T1 = A.sched[zi].T1;
    int *myflag = A.flags + g * nl + zi;
    if (warp == BW) {
        sync_warp_loop(myflag, z > 1 ? myflag - 1 : nullptr, z > 1 ? A.sched[zi - 1].T1 : 0, A.D, T0, T1,
                       A.trace ? A.trace + TRACE_W * (size_t)s_ticket : nullptr);
    } else {
        const size_t gb = (size_t)g * P.grid * 32 + lane;
        const double *__restrict__ u = A.u + gb;
        const double *__restrict__ f = A.f + gb;
        double *__restrict__ w = A.w + gb;
        double *tab = s_tab[warp];
        double *sL = s_L[warp];
        FwdRow R;
        R.y = A.sched[zi].first[warp];
        R.start = R.y ? A.rows[row_id(n, z, R.y)].start : 0;
        R.ss = 0.0;
        FwdSlot C{}, N{};
        double cband = 0.0, nband = 0.0;
        __syncthreads();  // first window opened by the sync warp
        for (int tau0 = T0; tau0 <= T1; tau0 += BWIN) {
            for (int tau = tau0; tau < tau0 + BWIN; ++tau) {
                if (!R.y) break;
                const int x = tau - R.start + 1;
                if (x < 1) continue;
                if (x == 1) {  // row start: offsets, seed table, windows, point-1 values
                    const int y = R.y;
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
                    smem_load_table<7, K>(tab, P.seedF + (int64_t)R.rid * 7 * K, lane);
                    R.u_wm = u[R.oc];
                    R.u_c = u[R.oc + 32];
                    R.us0 = u[R.os + 32];
                    R.un_m = u[R.on];
                    R.ubn_m = u[R.obn];
                    R.ubc0 = u[R.obc + 32];
                    R.uts0 = u[R.ots + 32];
                    R.utc_m = u[R.otc];
                    R.ws0 = ldcg(w + R.os + 32);
                    R.wbn_m = ldcg(w + R.obn);
                    R.wbc0 = ldcg(w + R.obc + 32);
                    R.wprev = 0.0;
                    fwd_load(C, u, f, w, R, 1);
                    fwd_band_load(cband, P, R, z, 1, lane);
                }
                // prefetch point x+1 (branch-free: at the row end it re-reads point m, unused)
                const int pp = min(x + 1, R.m);
                fwd_load(N, u, f, w, R, pp);
                fwd_band_load(nband, P, R, z, pp, lane);
                double ap[15];
                const double *a = A.arow;
                if (!CONST_ROW) {
                    const double *ar = P.arows + 15 * (int64_t)(R.oc / 32u + x);
#pragma unroll
                    for (int i = 0; i < 15; ++i) ap[i] = ar[i];
                    a = ap;
                }
                // residual in stencil_apply order (_kernels.py:255-266), then f - A u
                double acc = EXACT ? dmul(a[7], R.u_c) : a[7] * R.u_c;
                acc = madd<EXACT>(acc, a[0], R.u_wm);
                acc = madd<EXACT>(acc, a[1], R.us0);
                acc = madd<EXACT>(acc, a[2], C.us);
                acc = madd<EXACT>(acc, a[3], R.ubn_m);
                acc = madd<EXACT>(acc, a[4], C.ubn);
                acc = madd<EXACT>(acc, a[5], R.ubc0);
                acc = madd<EXACT>(acc, a[6], C.ubc);
                acc = madd<EXACT>(acc, a[8], C.ue);
                acc = madd<EXACT>(acc, a[9], C.un);
                acc = madd<EXACT>(acc, a[10], R.un_m);
                acc = madd<EXACT>(acc, a[11], C.uts);
                acc = madd<EXACT>(acc, a[12], R.uts0);
                acc = madd<EXACT>(acc, a[13], C.utc);
                acc = madd<EXACT>(acc, a[14], R.utc_m);
                const double r = dsub(C.f, acc);
                R.ss = fma(r, r, R.ss);
                // L entries: lane m publishes L_m (band store or the shared NDDF table)
                if (lane < 7) sL[lane] = (P.variant == 1 && in_band_b(x, R.y, z, R.m)) ? cband : tab[lane * K];
                __syncwarp();
                double v;
                if (EXACT) {  // reference order: own-row term first (_kernels.py:349-364)
                    v = msub<true>(r, sL[0], R.wprev);
                    v = msub<true>(v, sL[1], R.ws0);
                    v = msub<true>(v, sL[2], C.ws);
                    v = msub<true>(v, sL[3], R.wbn_m);
                    v = msub<true>(v, sL[4], C.wbn);
                    v = msub<true>(v, sL[5], R.wbc0);
                    v = msub<true>(v, sL[6], C.wbc);
                } else {  // own-row term last: one FMA on the row's dependency chain
                    v = msub<false>(r, sL[1], R.ws0);
                    v = msub<false>(v, sL[2], C.ws);
                    v = msub<false>(v, sL[3], R.wbn_m);
                    v = msub<false>(v, sL[4], C.wbn);
                    v = msub<false>(v, sL[5], R.wbc0);
                    v = msub<false>(v, sL[6], C.wbc);
                    v = msub<false>(v, sL[0], R.wprev);
                }
                w[R.oc + (uint32_t)x * 32u] = v;
                smem_march<7, K>(tab, lane);
                R.u_wm = R.u_c;
                R.u_c = C.ue;
                R.us0 = C.us;
                R.un_m = C.un;
                R.ubn_m = C.ubn;
                R.ubc0 = C.ubc;
                R.uts0 = C.uts;
                R.utc_m = C.utc;
                R.ws0 = C.ws;
                R.wbn_m = C.wbn;
                R.wbc0 = C.wbc;
                R.wprev = v;
                C = N;
                cband = nband;
                if (x == R.m) {
                    R.y = A.rows[R.rid].next;
                    if (R.y) R.start = A.rows[row_id(n, z, R.y)].start;
                }
            }
            __syncthreads();
        }
        s_red[warp][lane] = R.ss;
    }
    if (A.part) {
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
// backward: D^{-1} + L^T solve + update, exact time reversal of the forward schedule
// ----------------------------------------------------------------------------------------------
struct BwdSlot {
    double wn, wts, wtc, wf, u;
};

struct BwdRow {
    int y, m, rid, bstart;  // bstart: backward step of the row's first point (x = m)
    int qboff, qrow_band, qxe;  // lane m < 7: band offset / band-row flag / length of the row of q_m = p - d_m;
                                // lane 7: the own row (1/D)
    uint32_t oc, on, ots, otc;
    double lring[RING];   // lane m: prefetched value of L_m at q_m (lane 7: 1/D at p)
    unsigned lsrc;        // 2 bits per slot: 0 = q outside the interior, 1 = band store, 2 = NDDF
    double wn_hi, wts_hi, wtc_hi, wprev;
    BwdSlot ring[RING];
};

__device__ __forceinline__ void bwd_load(BwdSlot &S, const double *__restrict__ u, const double *__restrict__ w,
                                         const BwdRow &R, int x)
{
    const uint32_t X = (uint32_t)x * 32u;
    S.wn = ldcg(w + R.on + X - 32);
    S.wts = ldcg(w + R.ots + X);
    S.wtc = ldcg(w + R.otc + X - 32);
    S.wf = w[R.oc + X];
    S.u = u[R.oc + X];
}

// Lane m < 7 classifies q_m = p - d_m of point (x, y, z) and fetches its band-store entry L_m ahead
// (_kernels.py:434-441 _lq); lane 7 does the same for 1/D at p.  Result: source code in R.lsrc.
__device__ __forceinline__ void bwd_band_load(BwdRow &R, const PlanDev &P, int n, int z, int x, int lane, int SLOT)
{
    if (lane >= 8) return;
    unsigned code = 2;
    if (lane < 7) {
        const int qx = x - kDX[lane], qy = R.y - kDY[lane], qz = z - kDZ[lane];
        if (!interior(qx, qy, qz, n)) code = 0;
        else if (P.variant == 1 && (R.qrow_band || qx == 1 || qx == R.qxe)) {
            code = 1;
            R.lring[SLOT] = P.store[9 * (int64_t)(R.qboff + (R.qrow_band ? qx - 1 : (qx == 1 ? 0 : 1))) + lane];
        }
    } else if (P.variant == 1 && in_band_b(x, R.y, z, R.m)) {
        code = 1;
        R.lring[SLOT] = P.store[9 * (int64_t)(R.qboff + ((z == 1 || R.y == 1) ? x - 1 : (x == 1 ? 0 : 1))) + 8];
    }
    R.lsrc = (R.lsrc & ~(3u << (2 * SLOT))) | (code << (2 * SLOT));
}

template <int K, bool EXACT, int SLOT>
__device__ __forceinline__ void bwd_step(BwdRow &R, const PlanDev &P, const BatchArgs &A, int n, int z, int tau,
                                         double *__restrict__ u, double *__restrict__ w, double *tab, double *sL,
                                         int lane)
{
    if (!R.y) return;
    const int k = tau - R.bstart;  // 0-based position along the descending row
    if (k < 0) return;
    const int y = R.y;
    if (k == 0) {
        R.m = n - 1 - z - y;
        R.rid = row_id(n, z, y);
        R.oc = (uint32_t)row_offset(n, z, y) * 32u;
        R.on = (uint32_t)row_offset(n, z, y + 1) * 32u;
        R.ots = (uint32_t)row_offset(n, z + 1, y - 1) * 32u;
        R.otc = (uint32_t)row_offset(n, z + 1, y) * 32u;
        if (lane < 8) {  // the row of q_m (lane m) or the own row (lane 7)
            const int qy = lane < 7 ? y - kDY[lane] : y, qz = lane < 7 ? z - kDZ[lane] : z;
            const bool valid = qy >= 1 && qz >= 1 && qy + qz <= n - 2;
            R.qxe = n - 1 - qz - qy;
            R.qrow_band = (qz == 1 || qy == 1);
            R.qboff = (P.variant == 1 && valid) ? P.bandoff[row_id(n, qz, qy)] : 0;
        }
        smem_load_table<8, K>(tab, P.seedB + (int64_t)R.rid * 8 * K, lane);
        const uint32_t M = (uint32_t)R.m * 32u;
        R.wn_hi = ldcg(w + R.on + M);
        R.wts_hi = ldcg(w + R.ots + M + 32);
        R.wtc_hi = ldcg(w + R.otc + M);
        R.wprev = 0.0;
#pragma unroll
        for (int q = 0; q < PF; ++q)
            if (R.m - q >= 1) {
                bwd_load(R.ring[(SLOT + q) % RING], u, w, R, R.m - q);
                bwd_band_load(R, P, n, z, R.m - q, lane, (SLOT + q) % RING);
            }
    }
    const int x = R.m - k;
    const BwdSlot C = R.ring[SLOT];
    if (lane < 8) {
        const unsigned code = (R.lsrc >> (2 * SLOT)) & 3u;
        sL[lane] = code == 0 ? 0.0 : (code == 1 ? R.lring[SLOT] : tab[lane * K]);
    }
    __syncwarp();
    double Lq[7];
#pragma unroll
    for (int mm = 0; mm < 7; ++mm) Lq[mm] = sL[mm];
    const double inv_d = sL[7];
    double v = EXACT ? dmul(inv_d, C.wf) : inv_d * C.wf;
    if (EXACT) {  // reference order (_kernels.py:404-425)
        v = msub<true>(v, Lq[0], R.wprev);
        v = msub<true>(v, Lq[1], R.wn_hi);
        v = msub<true>(v, Lq[2], C.wn);
        v = msub<true>(v, Lq[3], R.wts_hi);
        v = msub<true>(v, Lq[4], C.wts);
        v = msub<true>(v, Lq[5], R.wtc_hi);
        v = msub<true>(v, Lq[6], C.wtc);
    } else {
        v = msub<false>(v, Lq[1], R.wn_hi);
        v = msub<false>(v, Lq[2], C.wn);
        v = msub<false>(v, Lq[3], R.wts_hi);
        v = msub<false>(v, Lq[4], C.wts);
        v = msub<false>(v, Lq[5], R.wtc_hi);
        v = msub<false>(v, Lq[6], C.wtc);
        v = msub<false>(v, Lq[0], R.wprev);
    }
    const uint32_t X = (uint32_t)x * 32u;
    w[R.oc + X] = v;
    u[R.oc + X] = dadd(C.u, v);
    {   // prefetch point x-PF (branch-free: below x = 1 the loads re-read point 1, unused)
        const int pp = max(x - PF, 1);
        bwd_load(R.ring[(SLOT + PF) % RING], u, w, R, pp);
        bwd_band_load(R, P, n, z, pp, lane, (SLOT + PF) % RING);
    }
    smem_march<8, K>(tab, lane);
    R.wn_hi = C.wn;
    R.wts_hi = C.wts;
    R.wtc_hi = C.wtc;
    R.wprev = v;
    if (x == 1) {
        R.y = A.rows[R.rid].prev;
        if (R.y) R.bstart = A.Tmax - (A.rows[row_id(n, z, R.y)].start + (n - 1 - z - R.y) - 1);
    }
}

template <int K, bool EXACT>
__global__ void __launch_bounds__(NT, 2) k_batch_bwd(PlanDev P, BatchArgs A)
{
    __shared__ int s_ticket;
    __shared__ double s_tab[BW][8 * K];
    __shared__ double s_L[BW][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_ticket = atomicAdd(A.ticket, 1) + 1;
    __syncthreads();
    const int nl = P.n - 3;
    const int li = s_ticket / A.G, g = s_ticket - li * A.G;
    const int zi = nl - 1 - li;
    const int n = P.n, z = zi + 1;
    int *myflag = A.flags + g * nl + zi;
    const int tb0 = A.Tmax - A.sched[zi].T1, tb1 = A.Tmax - A.sched[zi].T0;
    if (warp == BW) {
        sync_warp_loop(myflag, z < nl ? myflag + 1 : nullptr, z < nl ? A.Tmax - A.sched[zi + 1].T0 : 0, A.D, tb0,
                       tb1, A.trace ? A.trace + TRACE_W * (size_t)s_ticket : nullptr);
        return;
    }
    const size_t gb = (size_t)g * P.grid * 32 + lane;
    double *__restrict__ u = A.u + gb;
    double *__restrict__ w = A.w + gb;
    double *tab = s_tab[warp];
    BwdRow R;
    R.lsrc = 0;
    R.y = A.sched[zi].last[warp];
    R.bstart = R.y ? A.Tmax - (A.rows[row_id(n, z, R.y)].start + (n - 1 - z - R.y) - 1) : 0;
    __syncthreads();  // first window opened by the sync warp
    for (int tau0 = tb0; tau0 <= tb1; tau0 += BWIN) {
        bwd_step<K, EXACT, 0>(R, P, A, n, z, tau0 + 0, u, w, tab, s_L[warp], lane);
        bwd_step<K, EXACT, 1>(R, P, A, n, z, tau0 + 1, u, w, tab, s_L[warp], lane);
        bwd_step<K, EXACT, 2>(R, P, A, n, z, tau0 + 2, u, w, tab, s_L[warp], lane);
        bwd_step<K, EXACT, 3>(R, P, A, n, z, tau0 + 3, u, w, tab, s_L[warp], lane);
        __syncthreads();
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
