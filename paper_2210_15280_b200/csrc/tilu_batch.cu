// Batched fast path: many macro-tets that share one surrogate (identical operator, e.g. the
// 384 Kuhn tets of config 4) swept together in an interleaved layout.
//
// Layout ("packed"): tets are grouped by 32; group g stores fp64 [grid][32], i.e. the 32 tets'
// values of one lattice point are one 256-byte segment.  A warp processes one lattice row for
// the 32 tets of its group (lane = tet), so every load and store of u, f, w is a fully
// coalesced 256 B access, no lane is ever idle, and each lane executes exactly the reference's
// serial operation sequence for its own tet (bitwise parity in exact mode).
//
// Schedule: one CTA per (group, z-layer), BW warps per CTA, row y of layer z handled by warp
// (y-1) % BW.  Point (x, y, z) runs at global step T = O_z + A_z (y-1) + (x-1):
//   * A_z >= 2 row skew inside a layer, A_z * BW >= longest row so a warp owns one row at a
//     time; row y needs row y-1's values from >= A_z - 1 steps earlier, so the CTA
//     synchronises only every B_z = A_z - 1 steps (one bar.sync per window, not per step);
//   * O_z - O_{z-1} = A_{z-1} R_z - A_z (R_z - 1) + 1 + D: every value a layer needs from the
//     layer below was produced >= D + 1 steps earlier.  Layers run in different CTAs (often on
//     different SMs) and hand over through release/acquire progress counters; D is slack so the
//     consumer rarely waits.
// The backward pass runs the exact time reversal of this schedule (T_b = Tmax - T), which
// satisfies the transposed dependencies.  CTAs take (group, layer) tickets in layer order
// (ascending z forward, descending backward), so a CTA only ever waits for CTAs that already
// hold earlier tickets: no deadlock whatever the residency.
//
// Forward kernel  = residual f - A u (15-point stencil) + forward L substitution, writes w.
// Backward kernel = D^{-1} scaling + L^T substitution + u += w, writes w (in place) and u.
#include "tilu_batch.cuh"
#include "tilu_common.cuh"
#include "tilu_plan.cuh"

namespace tilu {

__device__ __forceinline__ int ld_acquire(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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
    while (ld_acquire(flag) < need) {
        __nanosleep(64);
        if (++polls > (1ll << 27)) __trap();
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
// forward: residual + L solve
// ----------------------------------------------------------------------------------------------
template <int K, bool EXACT, bool CONST_ROW>
__global__ void __launch_bounds__(BW * 32, 2) k_batch_fwd(PlanDev P, BatchArgs A)
{
    __shared__ int s_ticket;
    __shared__ double s_red[BW][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_ticket = atomicAdd(A.ticket, 1) + 1;  // counter starts at -1
    __syncthreads();
    const int nl = P.n - 3;
    const int zi = s_ticket / A.G, g = s_ticket - (s_ticket / A.G) * A.G;
    const int n = P.n, z = zi + 1, R = n - 2 - z;
    const LayerSched S = A.sched[zi];
    const size_t gb = (size_t)g * P.grid * 32 + lane;
    const double *__restrict__ u = A.u + gb;
    const double *__restrict__ f = A.f + gb;
    double *__restrict__ w = A.w + gb;
    int *myflag = A.flags + g * nl + zi;
    const int *below = z > 1 ? myflag - 1 : nullptr;

    double a[15];
    if (CONST_ROW) {
#pragma unroll
        for (int i = 0; i < 15; ++i) a[i] = P.arow[i];
    }

    int y = warp + 1;
    int m = 0, rid = 0;
    uint32_t oc = 0, os = 0, on = 0, obn = 0, obc = 0, ots = 0, otc = 0;
    double d[7][K];
    double u_wm = 0, u_c = 0, us0 = 0, un_m = 0, ubn_m = 0, ubc0 = 0, uts0 = 0, utc_m = 0;
    double ws0 = 0, wbn_m = 0, wbc0 = 0, wprev = 0;
    double ss = 0.0;

    for (int tau0 = S.T0; tau0 <= S.T1; tau0 += S.B) {
        if (threadIdx.x == 0 && below) {
            // everything this window reads from layer z-1 has T <= tau0 + B - 2 - D; the layer below
            // never publishes beyond its own last step
            const int need = min(tau0 + S.B - 2 - A.D, A.sched[zi - 1].T1);
            wait_progress(below, need);
        }
        __syncthreads();
        const int tau1 = min(tau0 + S.B, S.T1 + 1);
        for (int tau = tau0; tau < tau1; ++tau) {
            if (y > R) break;
            const int x = tau - (S.O + S.A * (y - 1)) + 1;
            if (x < 1) continue;
            if (x == 1) {  // row start: offsets, seed table, stencil windows
                m = n - 1 - z - y;
                rid = row_id(n, z, y);
                oc = (uint32_t)row_offset(n, z, y) * 32u;
                os = (uint32_t)row_offset(n, z, y - 1) * 32u;
                on = (uint32_t)row_offset(n, z, y + 1) * 32u;
                obn = (uint32_t)row_offset(n, z - 1, y + 1) * 32u;
                obc = (uint32_t)row_offset(n, z - 1, y) * 32u;
                ots = (uint32_t)row_offset(n, z + 1, y - 1) * 32u;
                otc = (uint32_t)row_offset(n, z + 1, y) * 32u;
                const double *sd = P.seedF + (int64_t)rid * 7 * K;
#pragma unroll
                for (int mm = 0; mm < 7; ++mm)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[mm][j] = sd[mm * K + j];
                u_wm = u[oc];
                u_c = u[oc + 32];
                us0 = u[os + 32];
                un_m = u[on];
                ubn_m = u[obn];
                ubc0 = u[obc + 32];
                uts0 = u[ots + 32];
                utc_m = u[otc];
                ws0 = ldcg(w + os + 32);
                wbn_m = ldcg(w + obn);
                wbc0 = ldcg(w + obc + 32);
                wprev = 0.0;
            }
            const uint32_t X = (uint32_t)x * 32u;
            // newest window entries
            const double u_e = u[oc + X + 32], us1 = u[os + X + 32], un0 = u[on + X];
            const double ubn0 = u[obn + X], ubc1 = u[obc + X + 32], uts1 = u[ots + X + 32], utc0 = u[otc + X];
            const double fx = f[oc + X];
            const double ws1 = ldcg(w + os + X + 32), wbn0 = ldcg(w + obn + X), wbc1 = ldcg(w + obc + X + 32);
            if (!CONST_ROW) {
                const double *ar = P.arows + 15 * (int64_t)(oc / 32u + x);
#pragma unroll
                for (int i = 0; i < 15; ++i) a[i] = ar[i];
            }
            // residual in stencil_apply order (_kernels.py:255-266), then f - A u
            double acc = EXACT ? dmul(a[7], u_c) : a[7] * u_c;
            acc = madd<EXACT>(acc, a[0], u_wm);
            acc = madd<EXACT>(acc, a[1], us0);
            acc = madd<EXACT>(acc, a[2], us1);
            acc = madd<EXACT>(acc, a[3], ubn_m);
            acc = madd<EXACT>(acc, a[4], ubn0);
            acc = madd<EXACT>(acc, a[5], ubc0);
            acc = madd<EXACT>(acc, a[6], ubc1);
            acc = madd<EXACT>(acc, a[8], u_e);
            acc = madd<EXACT>(acc, a[9], un0);
            acc = madd<EXACT>(acc, a[10], un_m);
            acc = madd<EXACT>(acc, a[11], uts1);
            acc = madd<EXACT>(acc, a[12], uts0);
            acc = madd<EXACT>(acc, a[13], utc0);
            acc = madd<EXACT>(acc, a[14], utc_m);
            const double r = dsub(fx, acc);
            ss = fma(r, r, ss);
            // L entries: NDDF marchers or the V1 band store
            double L[7];
            if (P.variant == 1 && in_band_b(x, y, z, m)) {
                const double *st = P.store + 9 * (int64_t)band_idx_b(P, rid, x, y, z);
#pragma unroll
                for (int mm = 0; mm < 7; ++mm) L[mm] = st[mm];
            } else {
#pragma unroll
                for (int mm = 0; mm < 7; ++mm) L[mm] = d[mm][0];
            }
            double v;
            if (EXACT) {  // reference order: own-row term first (_kernels.py:349-364)
                v = msub<true>(r, L[0], wprev);
                v = msub<true>(v, L[1], ws0);
                v = msub<true>(v, L[2], ws1);
                v = msub<true>(v, L[3], wbn_m);
                v = msub<true>(v, L[4], wbn0);
                v = msub<true>(v, L[5], wbc0);
                v = msub<true>(v, L[6], wbc1);
            } else {      // own-row term last: one FMA on the row's dependency chain
                v = msub<false>(r, L[1], ws0);
                v = msub<false>(v, L[2], ws1);
                v = msub<false>(v, L[3], wbn_m);
                v = msub<false>(v, L[4], wbn0);
                v = msub<false>(v, L[5], wbc0);
                v = msub<false>(v, L[6], wbc1);
                v = msub<false>(v, L[0], wprev);
            }
            w[oc + X] = v;
#pragma unroll
            for (int mm = 0; mm < 7; ++mm) march<K>(d[mm]);
            // slide the windows
            u_wm = u_c;
            u_c = u_e;
            us0 = us1;
            un_m = un0;
            ubn_m = ubn0;
            ubc0 = ubc1;
            uts0 = uts1;
            utc_m = utc0;
            ws0 = ws1;
            wbn_m = wbn0;
            wbc0 = wbc1;
            wprev = v;
            if (x == m) y += BW;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_release(myflag, tau1 - 1);
        }
    }
    if (A.part) {
        s_red[warp][lane] = ss;
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
template <int K, bool EXACT>
__global__ void __launch_bounds__(BW * 32, 2) k_batch_bwd(PlanDev P, BatchArgs A)
{
    __shared__ int s_ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_ticket = atomicAdd(A.ticket, 1) + 1;  // counter starts at -1
    __syncthreads();
    const int nl = P.n - 3;
    const int li = s_ticket / A.G, g = s_ticket - li * A.G;
    const int zi = nl - 1 - li;
    const int n = P.n, z = zi + 1, R = n - 2 - z;
    const LayerSched S = A.sched[zi];
    const size_t gb = (size_t)g * P.grid * 32 + lane;
    double *__restrict__ u = A.u + gb;
    double *__restrict__ w = A.w + gb;
    int *myflag = A.flags + g * nl + zi;
    const int *above = z < nl ? myflag + 1 : nullptr;

    // the warp's rows in descending order
    int y = warp < R ? warp + 1 + ((R - 1 - warp) / BW) * BW : 0;  // largest y <= R with (y-1) % BW == warp
    int m = 0, rid = 0;
    uint32_t oc = 0, on = 0, ots = 0, otc = 0;
    double d[8][K];
    double wn_hi = 0, wts_hi = 0, wtc_hi = 0, wprev = 0;
    const int tb0 = A.Tmax - S.T1, tb1 = A.Tmax - S.T0;

    for (int tau0 = tb0; tau0 <= tb1; tau0 += S.B) {
        if (threadIdx.x == 0 && above) {
            const int need = min(tau0 + S.B - 2 - A.D, A.Tmax - A.sched[zi + 1].T0);
            wait_progress(above, need);
        }
        __syncthreads();
        const int tau1 = min(tau0 + S.B, tb1 + 1);
        for (int tau = tau0; tau < tau1; ++tau) {
            if (y < 1) break;
            const int mrow = n - 1 - z - y;
            const int x = A.Tmax - tau - (S.O + S.A * (y - 1)) + 1;
            if (x > mrow) continue;
            if (x == mrow) {  // row start (x descending)
                m = mrow;
                rid = row_id(n, z, y);
                oc = (uint32_t)row_offset(n, z, y) * 32u;
                on = (uint32_t)row_offset(n, z, y + 1) * 32u;
                ots = (uint32_t)row_offset(n, z + 1, y - 1) * 32u;
                otc = (uint32_t)row_offset(n, z + 1, y) * 32u;
                const double *sd = P.seedB + (int64_t)rid * 8 * K;
#pragma unroll
                for (int mm = 0; mm < 8; ++mm)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[mm][j] = sd[mm * K + j];
                const uint32_t M = (uint32_t)m * 32u;
                wn_hi = ldcg(w + on + M);
                wts_hi = ldcg(w + ots + M + 32);
                wtc_hi = ldcg(w + otc + M);
                wprev = 0.0;
            }
            const uint32_t X = (uint32_t)x * 32u;
            const double wn_lo = ldcg(w + on + X - 32), wts_lo = ldcg(w + ots + X), wtc_lo = ldcg(w + otc + X - 32);
            const double wf = w[oc + X];
            const double uo = u[oc + X];
            const bool band = P.variant == 1 && in_band_b(x, y, z, m);
            const double inv_d = band ? P.store[9 * (int64_t)band_idx_b(P, rid, x, y, z) + 8] : d[7][0];
            double Lq[7];
            Lq[0] = lq_b(P, 0, x + 1, y, z, d[0][0]);
            Lq[1] = lq_b(P, 1, x, y + 1, z, d[1][0]);
            Lq[2] = lq_b(P, 2, x - 1, y + 1, z, d[2][0]);
            Lq[3] = lq_b(P, 3, x + 1, y - 1, z + 1, d[3][0]);
            Lq[4] = lq_b(P, 4, x, y - 1, z + 1, d[4][0]);
            Lq[5] = lq_b(P, 5, x, y, z + 1, d[5][0]);
            Lq[6] = lq_b(P, 6, x - 1, y, z + 1, d[6][0]);
            double v = EXACT ? dmul(inv_d, wf) : inv_d * wf;
            if (EXACT) {  // reference order (_kernels.py:404-425)
                v = msub<true>(v, Lq[0], wprev);
                v = msub<true>(v, Lq[1], wn_hi);
                v = msub<true>(v, Lq[2], wn_lo);
                v = msub<true>(v, Lq[3], wts_hi);
                v = msub<true>(v, Lq[4], wts_lo);
                v = msub<true>(v, Lq[5], wtc_hi);
                v = msub<true>(v, Lq[6], wtc_lo);
            } else {
                v = msub<false>(v, Lq[1], wn_hi);
                v = msub<false>(v, Lq[2], wn_lo);
                v = msub<false>(v, Lq[3], wts_hi);
                v = msub<false>(v, Lq[4], wts_lo);
                v = msub<false>(v, Lq[5], wtc_hi);
                v = msub<false>(v, Lq[6], wtc_lo);
                v = msub<false>(v, Lq[0], wprev);
            }
            w[oc + X] = v;
            u[oc + X] = dadd(uo, v);
#pragma unroll
            for (int mm = 0; mm < 8; ++mm) march<K>(d[mm]);
            wn_hi = wn_lo;
            wts_hi = wts_lo;
            wtc_hi = wtc_lo;
            wprev = v;
            if (x == 1) y -= BW;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            st_release(myflag, tau1 - 1);
        }
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
        if (c) k_batch_fwd<K, true, true><<<grid, BW * 32, 0, s>>>(P, A);
        else k_batch_fwd<K, true, false><<<grid, BW * 32, 0, s>>>(P, A);
    } else {
        if (c) k_batch_fwd<K, false, true><<<grid, BW * 32, 0, s>>>(P, A);
        else k_batch_fwd<K, false, false><<<grid, BW * 32, 0, s>>>(P, A);
    }
}

template <int K>
static void launch_bwd_k(const PlanDev &P, const BatchArgs &A, bool exact, cudaStream_t s)
{
    const unsigned grid = (unsigned)(A.G * (P.n - 3));
    if (exact) k_batch_bwd<K, true><<<grid, BW * 32, 0, s>>>(P, A);
    else k_batch_bwd<K, false><<<grid, BW * 32, 0, s>>>(P, A);
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
