// Fused band kernels of the plane-layout path (included inside namespace tilu::pl of tilu_plane.cu).
//
// Same geometry, band tasks, ticket order and handoff protocol as the warp-specialised kernels of
// tilu_plane.cu, but ONE warp per diagonal does everything for its 32 rows: the NDDF march of the
// L values (registers), the residual from TMA-staged lines (forward) and the substitution chain.
// No helper -> solver rings, no full / empty barriers: per step the only loop-carried dependency is
// the chain itself, everything else (march, residual, staging, prefetch) is independent work the
// scheduler interleaves across the GS unrolled steps of a group.  Per SM one CTA of PW warps (one
// per scheduler partition).
//
// Staging (TMA, one elected lane, ring of FNG groups): forward, one 3D box (WIN z, GS lines, planes
// s-1..s+1) of u and one box of f per group -- every u line is fetched once (a step's neighbours
// at tau-2..tau+2 are in the current or the next group's box); backward, one box of w_f and one of
// u per group.
//
// Step variants: "plain" groups (every lane has an interior point at every step of the group, no
// lane on a V1 band row) run straight-line code without validity predicates; the other groups (the
// skewed start / end of a task, chunks with rows z = 1 or y <= 2, partly dead warps) run the general
// step.  Both are the reference's operation sequence per lane: exact mode is bitwise.
//
// Coverage: constant stencil row (AMODE 1) and on-the-fly separable-coefficient rows (AMODE 2,
// config 3), V1 / V2, exact / fast.  Per-point rows and stored factors stay on the warp-specialised
// kernels.

constexpr int FNG = 8;                                          // TMA ring depth (groups)
constexpr int FUB = (3 * GS * WIN * 8 + 127) / 128 * 128 / 8;   // doubles: u box [3][GS][WIN]
constexpr int FLB = (GS * WIN * 8 + 127) / 128 * 128 / 8;       // doubles: one [GS][WIN] box
constexpr int FSLOT = FUB + FLB;                                // forward slot: u box + f box
constexpr int BSLOT = 2 * FLB;                                  // backward slot: w_f box + u box

struct MapsF {
    CUtensorMap u3g, f1, w1, u1;  // u box (WIN, GS, 3); f, w_f, u boxes (WIN, GS, 1)
};

struct SmemF {
    alignas(128) double tb[PW][FNG][FSLOT];  // TMA ring (the backward pass uses BSLOT doubles per slot)
    double hring[PW][HR][32];                // warp k-1 -> warp k handoff ring (data is the flag)
    double pre[PW][PD][3][32];               // prefetched global handoff values (cp.async)
    uint64_t tfull[PW][FNG];                 // TMA group landed
    int task;
};

// cp.async wait without a compiler memory barrier: every access to the copied-to shared memory is a
// volatile access, which the compiler keeps in program order with this volatile asm.
__device__ __forceinline__ void cpa_wait_pd_nb() { asm volatile("cp.async.wait_group %0;" ::"n"(PD - 1)); }

__device__ __forceinline__ void initf(SmemF &S)
{
    for (int i = threadIdx.x; i < PW * HR * 32; i += blockDim.x) (&S.hring[0][0][0])[i] = sentv();
    if (threadIdx.x < PW * FNG) mb_init(&S.tfull[0][0] + threadIdx.x, 1);
    mb_fence_init();
    __syncthreads();
}

#ifdef TILU_PLANE_PROF
#define PF_DECL long long pfc[6] = {0, 0, 0, 0, 0, 0}; const bool pfon = A.steplog && t == A.prof_task; const long long pf_start = clock64()
#define PF_T0(v) const long long v = pfon ? clock64() : 0
#define PF_ADD(i, v) do { if (pfon) pfc[i] += clock64() - v; } while (0)
#define PF_OUT(nsteps) do { if (pfon && lane == 0) { long long *sl = A.steplog + k * 8; sl[0] += clock64() - pf_start; \
    for (int i = 0; i < 6; ++i) sl[1 + i] += pfc[i]; sl[7] += (nsteps); } } while (0)
#else
#define PF_DECL (void)0
#define PF_T0(v) (void)0
#define PF_ADD(i, v) (void)0
#define PF_OUT(nsteps) (void)0
#endif

// ------------------------------------------------------------------------------------------------
// Forward: r = f - A u, w_f = L^{-1} r.
// ------------------------------------------------------------------------------------------------
template <int K, bool EXACT, int AMODE>
__global__ void __launch_bounds__(PW * 32, 1) k_planef_fwd(const PlanDev P, const Args A, const __grid_constant__ MapsF M)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SmemF &S = *reinterpret_cast<SmemF *>(smem_raw);
    const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
    initf(S);
    const Geo g = A.g;
    const int n = P.n, ZP = g.ZP;
    uint32_t tseq = 0;  // TMA groups consumed by this warp so far
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
        const int T0 = z0 - 3, T1 = z0 + 32 + xe0;
        const bool wlive = (s <= n - 2) && (z0 <= s - 1);
        const bool live = wlive && (z <= s - 1);
        const int lo = live ? z + 1 : 1 << 30, hi = live ? z + xe : -(1 << 30);
        const int ngroups = (T1 - T0) / GS + 1;
        double r2 = 0.0;
        PF_DECL;
        double *hin = &S.hring[k][0][lane];
        double *hout = (k + 1 < PW) ? &S.hring[k + 1][0][lane] : nullptr;
        if (!wlive) {
            for (int tau = T0; tau <= T1; ++tau) {
                if (k > 0 && tau <= T1 - 1) (void)take_s(hin + ((tau + 1) & (HR - 1)) * 32);
                if (hout && tau >= T0 + 1) put_s(hout + (tau & (HR - 1)) * 32, 0.0);
            }
        } else {
            const bool gl_on = (lane == 0);
            const bool gp_ld = (k == 0) && b > 0, gl_ld = gl_on && z0 > 1;
            const double *pw0 = A.W + pidx(g, s - 1, 1, z);        // P(tau+1) = pw0[tau * ZP]
            const double *pga = A.W + pidx(g, s, -1, z0 - 1);      // ga(tau) = pga[tau * ZP]
            const double *pgb = A.W + pidx(g, s - 1, 0, z0 - 1);   // gb(tau) = pgb[tau * ZP]
            double *pwo = A.W + pidx(g, s, 0, z);
            double *pbo = A.B + pidx(g, s, 0, z);
            if (k == 0) {
#pragma unroll
                for (int e = 0; e < HR; ++e) hin[e * 32] = 0.0;
                __syncwarp();
            }
            const uint32_t hin_s = su32(hin), pre_s = su32(&S.pre[k][0][0][lane]);
            auto prefetch = [&](const int tn) {
                if (gp_ld) cpa8(hin_s + (uint32_t)(((tn + 1) & (HR - 1)) * 32 * 8), pw0 + (int64_t)tn * ZP);
                if (gl_ld) {
                    const uint32_t dd = pre_s + (uint32_t)((tn & (PD - 1)) * 96 * 8);
                    cpa8(dd + 32 * 8, pga + (int64_t)tn * ZP);
                    cpa8(dd + 64 * 8, pgb + (int64_t)tn * ZP);
                }
                cpa_commit();
            };
#pragma unroll
            for (int i = 0; i < PD; ++i) prefetch(T0 + i);
            // ---- march state: seven forward-difference tables, V1 band rows GS steps ahead ----
            double d[7][K];
            int boff = 0;
            if (live) {
                const int r = row_id(n, z, y);
                const double *sd = P.seedF + (int64_t)r * 7 * K;
#pragma unroll
                for (int m = 0; m < 7; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = sd[m * K + j];
                if (P.variant == 1) boff = P.bandoff[r];
            } else {
#pragma unroll
                for (int m = 0; m < 7; ++m)
#pragma unroll
                    for (int j = 0; j < K; ++j) d[m][j] = 0.0;
            }
            const bool v1 = P.variant == 1;
            const bool rowband = z == 1 || y == 1;
            auto band_ld = [&](int tau, double(&v)[7]) {
                const bool vp = tau >= lo && tau <= hi;
                const bool isb = v1 && vp && (rowband || tau == lo || tau == hi);
                if (__any_sync(0xffffffffu, isb)) {
                    const double *st = P.store + 9 * (int64_t)(boff + (rowband ? tau - z - 1 : (tau == lo ? 0 : 1)));
                    TILU_CHECK(!isb || (boff + (rowband ? tau - z - 1 : (tau == lo ? 0 : 1)) < P.nband_dbg),
                               "planef fwd band row", tau, z);
#pragma unroll
                    for (int m = 0; m < 7; ++m) v[m] = ld_if(isb, st + m, 0.0);
                }
            };
            double bl[GS][7];
#pragma unroll
            for (int j = 0; j < GS; ++j) band_ld(T0 + j, bl[j]);
            // ---- residual state ----
            double gyw[7], gzw[7];
            if (AMODE == 2) {
                const int T4 = 4 * n + 1;
                sepk_window(P.sepk + T4, live ? 4 * y : 4, gyw);
                sepk_window(P.sepk + 2 * T4, live ? 4 * z : 4, gzw);
            }
            // ---- TMA staging: group q = u lines [T0-2+GS q, +GS) of planes s-1..s+1, f lines [T0+GS q, +GS) ----
            const uint32_t tq0 = tseq;
            auto issue = [&](int q) {
                const uint32_t sq = tq0 + (uint32_t)q;
                const int sl = sq % FNG;
                double *tb = S.tb[k][sl];
                mb_expect(&S.tfull[k][sl], (3 * GS + GS) * WIN * 8);
                tma3(tb, &M.u3g, z0 - 1, T0 - 2 + GS * q, s - 1, &S.tfull[k][sl]);
                tma3(tb + FUB, &M.f1, z0 - 1, T0 + GS * q, s, &S.tfull[k][sl]);
            };
            if (lane == 0)
                for (int q = 0; q <= ngroups && q < FNG; ++q) issue(q);
            // plain groups: all 32 lanes live, no lane on a band row, every lane inside its row
            const bool wplain = (z0 + 31 <= s - 1) && (z0 > 1) && (s - (z0 + 31) >= 2);
            const int plo = z0 + 33, phi = z0 + xe - 1;  // every lane: lo < plo, hi > phi (x = 1 / x = xe are band points)

            double w1 = 0, p1 = 0, lw1p = 0, lp1p = 0;  // own last value, P(tau), lane z-1's last w / P
            const bool rearm_b = live && (k == 0 || (lane == 0 && z0 > 32));

            auto step = [&](auto plain_c, const int tau, const int j, const double *uc, const double *un,
                            const double *fb) {
                constexpr bool PLAIN = decltype(plain_c)::value;
                const bool vpt = PLAIN ? true : (tau >= lo && tau <= hi);
                const bool p_on = PLAIN ? true : (tau <= T1 - 1);
                // (a) the seven L values of this point, then advance the tables
                double L[7];
                if (PLAIN) {
#pragma unroll
                    for (int m = 0; m < 7; ++m) L[m] = d[m][0];
#pragma unroll
                    for (int m = 0; m < 7; ++m) march<K>(d[m]);
                } else {
                    const bool isb = v1 && vpt && (rowband || tau == lo || tau == hi);
#pragma unroll
                    for (int m = 0; m < 7; ++m) L[m] = isb ? bl[j][m] : d[m][0];
                    if (vpt) {
#pragma unroll
                        for (int m = 0; m < 7; ++m) march<K>(d[m]);
                    }
                    band_ld(tau + GS, bl[j]);
                }
                // (b) residual of this point (stencil_apply order, _kernels.py:243-267)
                double res;
                {
                    auto U = [&](int ds, int dt, int dz) -> double {
                        const int l = j + dt + 2;
                        return (l < GS ? uc : un)[((ds + 1) * GS + (l % GS)) * WIN + dz];
                    };
                    double a[15];
                    if (AMODE == 2) {
                        double hxw[7];
                        const int x = PLAIN ? tau - z : (vpt ? tau - z : 1);
                        sepk_window(P.sepk, 4 * x, hxw);
                        sepk_row(hxw, gyw, gzw, P.sepk_c0, P.sepk_w, a);
                    } else {
#pragma unroll
                        for (int qq = 0; qq < 15; ++qq) a[qq] = A.arow[qq];
                    }
                    double out = EXACT ? dmul(a[7], U(0, 0, 0)) : a[7] * U(0, 0, 0);
                    out = madd<EXACT>(out, a[0], U(0, -1, 0));    // w   (s,   tau-1, z)
                    out = madd<EXACT>(out, a[1], U(-1, 0, 0));    // s   (s-1, tau,   z)
                    out = madd<EXACT>(out, a[2], U(-1, 1, 0));    // se  (s-1, tau+1, z)
                    out = madd<EXACT>(out, a[3], U(0, -2, -1));   // bnw (s,   tau-2, z-1)
                    out = madd<EXACT>(out, a[4], U(0, -1, -1));   // bn  (s,   tau-1, z-1)
                    out = madd<EXACT>(out, a[5], U(-1, -1, -1));  // bc  (s-1, tau-1, z-1)
                    out = madd<EXACT>(out, a[6], U(-1, 0, -1));   // be  (s-1, tau,   z-1)
                    out = madd<EXACT>(out, a[8], U(0, 1, 0));     // e   (s,   tau+1, z)
                    out = madd<EXACT>(out, a[9], U(1, 0, 0));     // n   (s+1, tau,   z)
                    out = madd<EXACT>(out, a[10], U(1, -1, 0));   // nw  (s+1, tau-1, z)
                    out = madd<EXACT>(out, a[11], U(0, 2, 1));    // tse (s,   tau+2, z+1)
                    out = madd<EXACT>(out, a[12], U(0, 1, 1));    // ts  (s,   tau+1, z+1)
                    out = madd<EXACT>(out, a[13], U(1, 1, 1));    // tc  (s+1, tau+1, z+1)
                    out = madd<EXACT>(out, a[14], U(1, 0, 1));    // tw  (s+1, tau,   z+1)
                    res = dsub(fb[j * WIN], out);
                    if (!PLAIN) res = vpt ? res : 0.0;
                    r2 = fma(res, res, r2);
                }
                // (c) substitution: the terms of register-resident inputs first (same subtraction order)
                const double lw2 = lw1p, lp2 = lp1p;
                const double sw1 = __shfl_up_sync(0xffffffffu, w1, 1);
                const double sp1 = __shfl_up_sync(0xffffffffu, p1, 1);
                ChainPart<EXACT> part(res, L, w1, p1, lw2, lp2);
                PF_T0(pa0);
                cpa_wait_pd_nb();
                PF_ADD(2, pa0);
                PF_T0(pa1);
                double *hs = hin + ((tau + 1) & (HR - 1)) * 32;
                const volatile double *pv = &S.pre[k][tau & (PD - 1)][0][lane];
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
                PF_ADD(3, pa1);
                const double lw1 = gl_on ? ga_cur : sw1;
                const double lp1 = gl_on ? gb_cur : sp1;
                const double acc = part.finish(L, p0, lw1, lp1);
                const double wnew = vpt ? acc : 0.0;
                if (p_on && k > 0) sts(hs, sentv());
                if (hout && (PLAIN || tau >= T0 + 1)) sts(hout + (tau & (HR - 1)) * 32, wnew);
                if (vpt) {
                    TILU_CHECK(pwo + (int64_t)tau * ZP - A.W >= 0 && pwo + (int64_t)tau * ZP - A.W < A.pe,
                               "planef fwd w_f store", tau, s);
                    st_rlx(pwo + (int64_t)tau * ZP, wnew);
                    if (rearm_b) st_rlx(pbo + (int64_t)tau * ZP, sentv());
                }
                lw1p = lw1; lp1p = lp1;
                w1 = wnew; p1 = p0;
                prefetch(tau + PD);
            };

            bool bl_ok = true;
            for (int q = 0; q < ngroups; ++q) {
                const uint32_t sq = tq0 + (uint32_t)q;
                const int sl = sq % FNG, sn = (sq + 1) % FNG;
                const int tq = T0 + GS * q;
                PF_T0(pg0);
                if (hout) wait_armed(hout, tq, 1, T0 + 1, T1);
                PF_ADD(0, pg0);
                PF_T0(pg1);
                mb_wait(&S.tfull[k][sl], (sq / FNG) & 1);
                mb_wait(&S.tfull[k][sn], ((sq + 1) / FNG) & 1);
                PF_ADD(1, pg1);
#ifdef TILU_PLANE_PROF
                if (pfon && wplain && tq >= plo && tq + GS - 1 <= phi) pfc[4] += 1;
#endif
                const double *uc = S.tb[k][sl] + lane + 1;
                const double *un = S.tb[k][sn] + lane + 1;
                const double *fb = uc + FUB;
                if (wplain && tq >= plo && tq + GS - 1 <= phi) {
#pragma unroll
                    for (int j = 0; j < GS; ++j) step(std::true_type{}, tq + j, j, uc, un, fb);
                    bl_ok = false;  // plain steps do not look ahead for band rows
                } else {
                    if (!bl_ok) {
#pragma unroll
                        for (int j = 0; j < GS; ++j) band_ld(tq + j, bl[j]);
                        bl_ok = true;
                    }
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (tq + j <= T1) step(std::false_type{}, tq + j, j, uc, un, fb);
                }
                __syncwarp();
                if (lane == 0 && q + FNG <= ngroups) issue(q + FNG);
            }
            tseq = tq0 + (uint32_t)ngroups + 1u;
            PF_OUT(ngroups);
            // the extra group (index ngroups) was waited for as "next" of the last group
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        if (A.part) A.part[(int64_t)t * (PW * 32) + k * 32 + lane] = r2;
        __syncthreads();
        trace_end(A, t);
    }
}

// ------------------------------------------------------------------------------------------------
// Backward: w = D^{-1} w_f, L^T substitution (descending), u += w.
// ------------------------------------------------------------------------------------------------
template <int K, bool EXACT>
__global__ void __launch_bounds__(PW * 32, 1) k_planef_bwd(const PlanDev P, const Args A, const __grid_constant__ MapsF M)
{
    extern __shared__ __align__(128) unsigned char smem_raw[];
    SmemF &S = *reinterpret_cast<SmemF *>(smem_raw);
    const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
    initf(S);
    const Geo g = A.g;
    const int n = P.n, ZP = g.ZP;
    uint32_t tseq = 0;
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
        PF_DECL;
        double *hin = &S.hring[k][0][lane];
        double *hout = (k + 1 < PW) ? &S.hring[k + 1][0][lane] : nullptr;
        if (!wlive) {
            for (int tau = T1; tau >= T0 - 1; --tau) {
                if (k > 0 && tau >= T0) (void)take_s(hin + ((tau - 1) & (HR - 1)) * 32);
                if (hout && tau <= T1 - 1) put_s(hout + (tau & (HR - 1)) * 32, 0.0);
            }
        } else {
            const uint32_t tq0 = tseq;
            auto issue = [&](int q) {
                const uint32_t sq = tq0 + (uint32_t)q;
                const int sl = sq % FNG;
                const int lo_t = T1 - GS * q - (GS - 1);
                double *tb = S.tb[k][sl];
                mb_expect(&S.tfull[k][sl], 2 * GS * WIN * 8);
                tma3(tb, &M.w1, z0 - 1, lo_t, s, &S.tfull[k][sl]);
                tma3(tb + FLB, &M.u1, z0 - 1, lo_t, s, &S.tfull[k][sl]);
            };
            if (lane == 0)
                for (int q = 0; q < ngroups && q < FNG; ++q) issue(q);
            const double *pw0 = A.B + pidx(g, s + 1, -1, z);
            const double *pga = A.B + pidx(g, s, 1, z0 + 32);
            const double *pgb = A.B + pidx(g, s + 1, 0, z0 + 32);
            double *puo = A.u + pidx(g, s, 0, z);
            double *pbo = A.B + pidx(g, s, 0, z);
            double *pwo = A.W + pidx(g, s, 0, z);
            const bool gp_on = (k == 0), gl_on = (lane == 31);
            const bool gp_ld = gp_on && s0 + PW <= n - 2, gl_ld = gl_on && z0 + 32 <= s;
            volatile double *pre = &S.pre[k][0][0][lane];
            const uint32_t pre_s = su32(&S.pre[k][0][0][lane]);
            auto prefetch = [&](const int tn) {
                const uint32_t dd = pre_s + (uint32_t)((tn & (PD - 1)) * 96 * 8);
                if (gp_ld) cpa8(dd, pw0 + (int64_t)tn * ZP);
                if (gl_ld) {
                    cpa8(dd + 32 * 8, pga + (int64_t)tn * ZP);
                    cpa8(dd + 64 * 8, pgb + (int64_t)tn * ZP);
                }
                cpa_commit();
            };
#pragma unroll
            for (int i = 0; i < PD; ++i) prefetch(T1 - i);
            // ---- march state: seven shifted L tables + 1/D, band rows of the source points ----
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
            const bool v1 = P.variant == 1;
            const bool zr1 = z == 1, yr1 = y == 1, yr2 = y == 2, yge2 = y >= 2;
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
            auto band_ld = [&](int tau, double(&v)[8], unsigned &im, unsigned &bm) {
                tests(tau, im, bm);
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
            // plain groups: all lanes live, y >= 3 and z >= 2 everywhere, every lane at least two points
            // inside both ends of its row (every source point interior, none on the band)
            const bool wplain = (z0 + 31 <= s - 1) && (z0 > 1) && (s - (z0 + 31) >= 3);
            const int plo = z0 + 32 + 2, phi = z0 + xe - 2;

            double wb1 = 0, q1 = 0, lw1p = 0, lq1p = 0;
            const bool b_out = live && (k == PW - 1 || (lane == 0 && z0 > 32));
            const bool rearm_w = live && (k == 0 || lane == 31);

            auto step = [&](auto plain_c, const int tau, const int j, const double *tb) {
                constexpr bool PLAIN = decltype(plain_c)::value;
                const bool vpt = PLAIN ? true : (tau >= lo && tau <= hi);
                const bool q_on = PLAIN ? true : (tau >= T0);
                // (a) the seven source-point L values and 1/D, then advance the tables
                double Lq[7], invd;
                if (PLAIN) {
#pragma unroll
                    for (int m = 0; m < 7; ++m) Lq[m] = d[m][0];
                    invd = d[7][0];
#pragma unroll
                    for (int m = 0; m < 8; ++m) march<K>(d[m]);
                } else {
                    const unsigned im = bim[j], bm = bbm[j];
#pragma unroll
                    for (int m = 0; m < 7; ++m)
                        Lq[m] = ((im >> m) & 1u) ? (((bm >> m) & 1u) ? bl[j][m] : d[m][0]) : 0.0;
                    invd = ((bm >> 7) & 1u) ? bl[j][7] : d[7][0];
                    if (vpt) {
#pragma unroll
                        for (int m = 0; m < 8; ++m) march<K>(d[m]);
                    }
                    band_ld(tau - GS, bl[j], bim[j], bbm[j]);
                }
                const double wfv = tb[(GS - 1 - j) * WIN];
                const double uv = tb[FLB + (GS - 1 - j) * WIN];
                const double lw2 = lw1p, lq2 = lq1p;
                const double sw1 = __shfl_down_sync(0xffffffffu, wb1, 1);
                const double sq1 = __shfl_down_sync(0xffffffffu, q1, 1);
                // reference order (_kernels.py:416-428): inv_d w, then the w s se bnw bn bc be sources
                ChainPart<EXACT> part(EXACT ? dmul(invd, wfv) : invd * wfv, Lq, wb1, q1, lw2, lq2);
                PF_T0(pa0);
                cpa_wait_pd_nb();
                PF_ADD(2, pa0);
                PF_T0(pa1);
                volatile double *pv = pre + (tau & (PD - 1)) * 96;
                double *hs = hin + ((tau - 1) & (HR - 1)) * 32;
                double q0 = 0.0;
                if (q_on) q0 = gp_on ? (gp_ld ? pv[0] : 0.0) : lds_vol(hs);
                double ga_cur = gl_ld ? pv[32] : 0.0, gb_cur = gl_ld ? pv[64] : 0.0;
                if (__builtin_expect(__any_sync(0xffffffffu, (q_on && is_sent(q0)) ||
                                                                 (gl_ld && (is_sent(ga_cur) || is_sent(gb_cur)))), 0)) {
                    long long spins = 0;
                    for (;;) {
                        if (q_on && is_sent(q0)) q0 = gp_on ? ldg_cg(pw0 + (int64_t)tau * ZP) : lds_vol(hs);
                        if (gl_ld) {
                            if (is_sent(ga_cur)) ga_cur = ldg_cg(pga + (int64_t)tau * ZP);
                            if (is_sent(gb_cur)) gb_cur = ldg_cg(pgb + (int64_t)tau * ZP);
                        }
                        const bool still = (q_on && is_sent(q0)) || (gl_ld && (is_sent(ga_cur) || is_sent(gb_cur)));
                        if (!__any_sync(0xffffffffu, still)) break;
                        if (++spins > (1ll << 26)) __trap();
                    }
                }
                PF_ADD(3, pa1);
                const double lw1 = gl_on ? ga_cur : sw1;
                const double lq1 = gl_on ? gb_cur : sq1;
                const double acc = part.finish(Lq, q0, lw1, lq1);
                const double wnew = vpt ? acc : 0.0;
                if (q_on && k > 0) sts(hs, sentv());
                if (hout && (PLAIN || tau <= T1 - 1)) sts(hout + (tau & (HR - 1)) * 32, wnew);
                if (vpt) {
                    TILU_CHECK(puo + (int64_t)tau * ZP - A.u >= 0 && puo + (int64_t)tau * ZP - A.u < A.pe,
                               "planef bwd u store", tau, s);
                    puo[(int64_t)tau * ZP] = dadd(uv, acc);
                    if (b_out) st_rlx(pbo + (int64_t)tau * ZP, acc);
                    if (rearm_w) st_rlx(pwo + (int64_t)tau * ZP, sentv());
                }
                lw1p = lw1; lq1p = lq1;
                wb1 = wnew; q1 = q0;
                prefetch(tau - PD);
            };

            bool bl_ok = true;
            for (int q = 0; q < ngroups; ++q) {
                const uint32_t sq = tq0 + (uint32_t)q;
                const int sl = sq % FNG;
                const int tq = T1 - GS * q;
                PF_T0(pg0);
                if (hout) wait_armed(hout, tq, -1, T0 - 1, T1 - 1);
                PF_ADD(0, pg0);
                PF_T0(pg1);
                mb_wait(&S.tfull[k][sl], (sq / FNG) & 1);
                PF_ADD(1, pg1);
#ifdef TILU_PLANE_PROF
                if (pfon && wplain && tq <= phi && tq - (GS - 1) >= plo) pfc[4] += 1;
#endif
                const double *tb = S.tb[k][sl] + lane + 1;
                if (wplain && tq <= phi && tq - (GS - 1) >= plo) {
#pragma unroll
                    for (int j = 0; j < GS; ++j) step(std::true_type{}, tq - j, j, tb);
                    bl_ok = false;
                } else {
                    if (!bl_ok) {
#pragma unroll
                        for (int j = 0; j < GS; ++j) band_ld(tq - j, bl[j], bim[j], bbm[j]);
                        bl_ok = true;
                    }
#pragma unroll
                    for (int j = 0; j < GS; ++j)
                        if (tq - j >= T0 - 1) step(std::false_type{}, tq - j, j, tb);
                }
                __syncwarp();
                if (lane == 0 && q + FNG < ngroups) issue(q + FNG);
            }
            tseq = tq0 + (uint32_t)ngroups;
            PF_OUT(ngroups);
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        __syncthreads();
        trace_end(A, t);
    }
}
