// C ABI of libtilu (include/tilu.h): plan construction and the stream-ordered drivers that
// chain the kernels of one smoothing step.  No exceptions cross the boundary; every entry
// point returns a status code and records a thread-local message.
#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "tilu.h"
#include "tilu_batch.cuh"
#include "tilu_common.cuh"
#include "tilu_plan.cuh"

namespace tilu {
void launch_seed(const PlanDev &P, const double *lcoefs, const double *dcoefs, double *seedF, double *seedB,
                 cudaStream_t s);
void launch_seed_op(const PlanDev &P, const double *acoefs, int ky1, int kz1, double *seedA, cudaStream_t s);
void launch_residual(const PlanDev &P, bool exact, const double *u, const double *f, double *w, double *part,
                     int ntets, bool apply_only, cudaStream_t s);
bool launch_residual_sop(const PlanDev &P, const double *u, const double *f, double *w, double *part, int ntets,
                         cudaStream_t s);
void launch_reduce_rows(const double *part, int nrows, double *out, int ntets, cudaStream_t s);
bool launch_simple_solve(const PlanDev &P, bool exact, bool stored, double *w, double *state, double *u, int ntets,
                         int which, cudaStream_t s);
void launch_pack(const double *src, double *dst, int64_t grid, int ntets, int tpl, cudaStream_t s);
void launch_unpack(const double *src, double *dst, int64_t grid, int ntets, int tpl, cudaStream_t s);
void launch_batch_norms(double *part, int nrows, int ntets, int tpl, double *out, cudaStream_t s);
size_t norm_scratch_doubles(int G, int tpl);
bool launch_batch_pass(const PlanDev &P, const BatchArgs &A, bool exact, bool fwd, cudaStream_t s);
bool launch_coef_tables(const PlanDev &P, double *cf, double *cb, cudaStream_t s);
void launch_arm(const PlanDev &P, double *wa, const unsigned long long *hdr, unsigned long long key, int G, int tpl,
                cudaStream_t s);
// plane-layout fast path (tilu_plane.cu)
void prof_begin(cudaStream_t s);
void prof_end(const char *name, cudaStream_t s);
bool plane_supported(const tilu_plan *plan);
void plane_free(void *ws);
int plane_sweep(const tilu_plan *plan, double *u, const double *f, int ntets, int sweeps, double *rnorm2,
                cudaStream_t s, int *launches, bool stored);
}  // namespace tilu

using namespace tilu;

// ---- per-kernel event timing (tilu_profile_*) ------------------------------------------------
namespace {
struct ProfRec {
    const char *name;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof_pending;
std::map<std::string, std::pair<int, double>> g_prof_acc;
thread_local cudaEvent_t g_prof_open = nullptr;
}  // namespace

namespace tilu {
void prof_begin(cudaStream_t s)
{
    if (!g_prof_on) return;
    cudaEventCreate(&g_prof_open);
    cudaEventRecord(g_prof_open, s);
}
void prof_end(const char *name, cudaStream_t s)
{
    if (!g_prof_on || !g_prof_open) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_pending.push_back({name, g_prof_open, b});
    g_prof_open = nullptr;
}
}  // namespace tilu

namespace {
thread_local char g_err[512] = "";
thread_local int g_launches = 0;

int fail(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

}  // namespace

// error / launch accounting for the other translation units of the ABI (tilu_factor.cu, tilu_mg.cu)
namespace tilu {
int abi_fail(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}
void abi_count_launches(int k) { g_launches = k; }
}  // namespace tilu

namespace {
int check_cuda(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(TILU_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return TILU_OK;
}

template <class T>
int dev_upload(tilu_plan *p, T **dst, const T *src, size_t count)
{
    *dst = nullptr;
    if (count == 0) return TILU_OK;
    if (p->nallocs >= (int)(sizeof(p->allocs) / sizeof(p->allocs[0]))) return fail(TILU_ENOMEM, "too many plan buffers");
    void *d = nullptr;
    if (cudaMalloc(&d, count * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        return fail(TILU_ENOMEM, "cudaMalloc(%zu bytes) failed", count * sizeof(T));
    }
    p->allocs[p->nallocs++] = d;
    if (src && cudaMemcpy(d, src, count * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(TILU_ECUDA, "upload failed: %s", cudaGetErrorString(cudaGetLastError()));
    *dst = static_cast<T *>(d);
    return TILU_OK;
}

struct Scratch {
    cudaStream_t s;
    std::vector<void *> bufs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    ~Scratch()
    {
        for (void *b : bufs) cudaFreeAsync(b, s);
    }
    double *get(size_t count)
    {
        void *d = nullptr;
        if (cudaMallocAsync(&d, count * sizeof(double), s) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        bufs.push_back(d);
        return static_cast<double *>(d);
    }
};

bool valid_plan(const tilu_plan_t *p) { return p != nullptr && p->dev.n > 0; }
}  // namespace

// Smallest level routed to the plane kernels (TILU_PLANE_MIN_LEVEL overrides, tests use 3).
static int plane_min_level()
{
    static const char *e = std::getenv("TILU_PLANE_MIN_LEVEL");
    return e ? std::atoi(e) : 5;
}

bool batch_ok(const tilu_plan_t *p)
{
    // packed element offsets are 32-bit: grid * 64 < 2^32 (level <= 9)
    // the batched kernels take the residual from the constant row, per-point rows or the operator
    // surrogate (seedA); the separable on-the-fly rows (sepk) are plane / reference-layout only
    return !(p->flags & TILU_SCHED_SIMPLE) && p->dev.level <= 9 && p->dev.n >= 4 && p->bsched != nullptr &&
           (p->dev.arow != nullptr || p->dev.arows != nullptr || p->dev.seedA != nullptr);
}

// Tets per lane of the packed layout (groups of 32 * tpl tets).  More tets per lane amortise the
// per-point bookkeeping and, above all, every producer -> consumer handoff between rows over more
// DoF, once there are enough tets to keep the groups filled (T = 4 measured slower: register
// spills, fewer warps).  TILU_TPL=1|2 overrides (measurement only).
int batch_tpl(int ntets)
{
    static const char *e = std::getenv("TILU_TPL");
    if (e && (e[0] == '1' || e[0] == '2')) return e[0] - '0';
    // 65..96 tets: three full 32-lane groups beat one full + one half-empty 64-lane group (tools/tets_scan.py:
    // 1.46 vs 1.57 ms per sweep at level 7)
    if (ntets > 64 && ntets <= 96) return 1;
    return ntets > 32 ? 2 : 1;
}

// Per-point coefficient tables (2 x [grid][8] doubles, shared by all tets of a batch) can replace the
// per-warp NDDF march for large batches: 46 MB at level 7 (L2-resident), 360 MB at level 8.  Off by
// default -- the north star evaluates the L/U weights on the fly, and on config 4 the tables gain
// only ~2% (r02a bench: 3.13 vs 3.19 ms/sweep).  TILU_TAB=1 turns them on (measurement only).
static std::mutex g_coef_mu;
static bool want_tables(const tilu_plan_t *p, int ntets)
{
    static const char *e = std::getenv("TILU_TAB");
    return e && e[0] == '1' && batch_tpl(ntets) == 2 && p->dev.level <= 8;
}
static int ensure_tables(const tilu_plan_t *cp, cudaStream_t s)
{
    std::lock_guard<std::mutex> lk(g_coef_mu);
    tilu_plan_t *p = const_cast<tilu_plan_t *>(cp);
    if (p->coef) return TILU_OK;
    const size_t nd = (size_t)p->dev.grid * 8;
    void *d = nullptr;
    if (cudaMalloc(&d, 2 * nd * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return fail(TILU_ENOMEM, "coefficient tables: out of device memory");
    }
    double *cf = static_cast<double *>(d), *cb = cf + nd;
    cudaMemsetAsync(d, 0, 2 * nd * sizeof(double), s);
    if (!launch_coef_tables(p->dev, cf, cb, s)) {
        cudaFree(d);
        return fail(TILU_EUNSUPPORTED, "kx+1 = %d not compiled", p->dev.kx1);
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) {
        cudaFree(d);
        return check_cuda("coefficient tables");
    }
    p->coef = d;
    p->dev.coefF = cf;
    p->dev.coefB = cb;
    return TILU_OK;
}

size_t packed_doubles(const tilu_plan_t *p, int ntets)
{
    const int gw = 32 * batch_tpl(ntets);
    return (size_t)((ntets + gw - 1) / gw) * p->dev.grid * gw;
}

// Scratch of the packed path: [header: 8 doubles][w_f: packed][w_b: packed].  The header holds a
// key (layout of this plan and batch) when w_f is armed (sentinel on the interior): the backward
// pass re-arms w_f as it goes and its last warp writes the key, so only the first call on a fresh
// (zeroed) scratch, or one after a failed call, pays the arming pass.
constexpr size_t kScratchHdr = 8;
size_t packed_scratch_doubles(const tilu_plan_t *p, int ntets) { return kScratchHdr + 2 * packed_doubles(p, ntets); }

static unsigned long long scratch_key(const tilu_plan_t *p, int ntets)
{
    return 0x74696C7500000000ull ^ ((unsigned long long)(uint32_t)ntets << 12) ^
           ((unsigned long long)batch_tpl(ntets) << 8) ^ (unsigned long long)p->dev.level;
}

// `sweeps` fused sweeps on packed vectors (u, f [G][grid][32 * tpl]; ws = packed scratch).
int packed_sweeps(const tilu_plan_t *p, double *up, const double *fp, double *ws, int ntets, int sweeps,
                  double *rnorm2, cudaStream_t s)
{
    const PlanDev &P = p->dev;
    const int tpl = batch_tpl(ntets), gw = 32 * tpl;
    const int G = (ntets + gw - 1) / gw;
    if (want_tables(p, ntets) && !p->coef) {
        const int rc = ensure_tables(p, s);
        if (rc) return rc;
    }
    PlanDev PK = P;  // kernels see the tables only when this batch wants them
    if (!want_tables(p, ntets)) PK.coefF = PK.coefB = nullptr;
    Scratch sc(s);
    int *sync = reinterpret_cast<int *>(sc.get(2));  // fwd ticket, bwd ticket, bwd done
    double *part = rnorm2 ? sc.get((size_t)G * P.nrows * gw + norm_scratch_doubles(G, tpl)) : nullptr;
    if (!sync || (rnorm2 && !part)) return fail(TILU_ENOMEM, "scratch allocation failed");
    const bool exact = !(p->flags & TILU_FAST);
    BatchArgs A{};
    static const char *mt = std::getenv("TILU_DEBUG_MAX_TICKET");
    A.max_ticket = mt ? std::atoi(mt) : -1;
    A.u = up;
    A.f = fp;
    A.hdr = reinterpret_cast<unsigned long long *>(ws);
    A.wa = ws + kScratchHdr;
    A.wb = A.wa + packed_doubles(p, ntets);
    A.key = scratch_key(p, ntets);
    A.G = G;
    A.ntets = ntets;
    A.tpl = tpl;
    std::memcpy(A.arow, p->harow, sizeof(A.arow));
    prof_begin(s);
    launch_arm(P, A.wa, A.hdr, A.key, G, tpl, s);  // no-op when the scratch is armed
    prof_end("arm", s);
    ++g_launches;
    for (int k = 0; k < sweeps; ++k) {
        cudaMemsetAsync(sync, 0, 4 * sizeof(int), s);
        A.ticket = sync;
        A.part = part;
        prof_begin(s);
        bool ok = launch_batch_pass(PK, A, exact, true, s);
        prof_end("batch_fwd", s);
        A.ticket = sync + 1;
        A.done = sync + 2;
        A.part = nullptr;
        prof_begin(s);
        ok = ok && launch_batch_pass(PK, A, exact, false, s);
        prof_end("batch_bwd", s);
        if (!ok) return fail(TILU_EUNSUPPORTED, "kx+1 = %d not compiled", P.kx1);
        g_launches += 2;
        if (rnorm2) {
            prof_begin(s);
            launch_batch_norms(part, P.nrows, ntets, tpl, rnorm2 + (int64_t)k * ntets, s);
            prof_end("batch_norms", s);
            g_launches += 2;
        }
    }
    return TILU_OK;
}

extern "C" {

void tilu_profile_enable(int on) { g_prof_on = on != 0; }

void tilu_profile_reset(void)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof_pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof_pending.clear();
    g_prof_acc.clear();
}

int tilu_profile_read(char *names, int *counts, double *ms, int cap)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto &r : g_prof_pending) {
        float t = 0.f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&t, r.a, r.b);
        auto &e = g_prof_acc[r.name];
        e.first += 1;
        e.second += t;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof_pending.clear();
    int i = 0;
    for (auto &kv : g_prof_acc) {
        if (i >= cap) break;
        std::snprintf(names + 64 * i, 64, "%s", kv.first.c_str());
        counts[i] = kv.second.first;
        ms[i] = kv.second.second;
        ++i;
    }
    return (int)g_prof_acc.size();
}

const char *tilu_last_error(void) { return g_err; }
int tilu_version(void) { return 100; }
int tilu_last_launch_count(void) { return g_launches; }
int64_t tilu_plan_grid_size(const tilu_plan_t *p) { return p ? p->dev.grid : -1; }
int64_t tilu_plan_interior_size(const tilu_plan_t *p) { return p ? p->interior : -1; }

void tilu_plan_destroy(tilu_plan_t *p)
{
    if (!p) return;
    for (int i = 0; i < p->nallocs; ++i) cudaFree(p->allocs[i]);
    if (p->coef) cudaFree(p->coef);
    plane_free(p->plane);
    delete p;
}

int tilu_plan_create(const tilu_desc_t *d, tilu_plan_t **out)
{
    g_launches = 0;
    if (!d || !out) return fail(TILU_EINVAL, "null descriptor / output");
    *out = nullptr;
    if (d->level < 2 || d->level > 10) return fail(TILU_EINVAL, "level %d outside 2..10", d->level);
    if (d->kx1 < 1 || d->ky1 < 1 || d->kz1 < 1) return fail(TILU_EINVAL, "coefficient extents must be >= 1");
    if (d->kx1 > 9 || d->ky1 > 16 || d->kz1 > 16) return fail(TILU_EUNSUPPORTED, "kx+1 <= 9 (and ky+1, kz+1 <= 16) supported");
    if (d->variant != TILU_VARIANT_V1 && d->variant != TILU_VARIANT_V2) return fail(TILU_EINVAL, "variant must be V1 or V2");
    if (!d->lcoefs || !d->dcoefs) return fail(TILU_EINVAL, "lcoefs / dcoefs required");
    if (d->acoefs && (d->akx1 < 1 || d->akx1 > 9 || d->aky1 < 1 || d->akz1 < 1 || d->aky1 > 16 || d->akz1 > 16))
        return fail(TILU_EUNSUPPORTED, "operator surrogate extents unsupported");
    const int n = 1 << d->level;
    if (n < 4) return fail(TILU_EINVAL, "level too small");

    {   // keep stream-ordered scratch cached between calls instead of returning it to the driver
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
    }
    tilu_plan *p = new (std::nothrow) tilu_plan();
    if (!p) return fail(TILU_ENOMEM, "host allocation failed");
    std::memset(p, 0, sizeof(*p));
    p->flags = d->flags;
    PlanDev &P = p->dev;
    P.level = d->level;
    P.n = n;
    P.grid = num_points(n);
    P.kx1 = d->kx1;
    P.ky1 = d->ky1;
    P.kz1 = d->kz1;
    P.variant = d->variant;
    P.h = 1.0 / n;
    P.tmin = 6;
    P.tmax = 3 * n - 6;
    p->interior = num_points(n - 4);

    // rows in (z, y) order
    std::vector<RowInfo> rows;
    std::vector<int64_t> rowbase;
    for (int z = 1; z <= n - 3; ++z)
        for (int y = 1; y <= n - 2 - z; ++y) {
            rows.push_back({z, y, n - 1 - z - y, 1 + 2 * y + 3 * z});
            rowbase.push_back(row_offset(n, z, y));
        }
    P.nrows = (int)rows.size();
    p->nband = 0;

    int rc = TILU_OK;
    std::vector<int> bandoff;
    if (d->variant == TILU_VARIANT_V1) {
        if (!d->band_ranks || !d->store_rows || d->nband <= 0) {
            tilu_plan_destroy(p);
            return fail(TILU_EINVAL, "V1 needs band_ranks and store_rows");
        }
        // The reference looks rows up by binary search in the sorted band ranks (_kernels.py:27-36);
        // accept exactly the canonical band set (surrogate.py:223-229) so per-row offsets are equivalent.
        int64_t k = 0;
        bool ok = true;
        for (size_t r = 0; r < rows.size() && ok; ++r) {
            const RowInfo &ri = rows[r];
            bandoff.push_back((int)k);
            for (int x = 1; x <= ri.xe; ++x) {
                const bool band = ri.z == 1 || ri.y == 1 || x == 1 || x == ri.xe;
                if (!band) continue;
                if (k >= d->nband || d->band_ranks[k] != rowbase[r] + x) { ok = false; break; }
                ++k;
            }
        }
        if (!ok || k != d->nband) {
            tilu_plan_destroy(p);
            return fail(TILU_EINVAL, "band_ranks is not the canonical boundary band of level %d", d->level);
        }
        p->nband = d->nband;
        P.nband_dbg = d->nband;
    }

    RowInfo *drows = nullptr;
    int64_t *drowbase = nullptr;
    int *dbandoff = nullptr;
    double *dstore = nullptr, *dl = nullptr, *dd = nullptr, *dseedF = nullptr, *dseedB = nullptr, *darow = nullptr;
    double *dacoefs = nullptr, *dseedA = nullptr, *dfactors = nullptr;
    const int K = d->kx1;
    if ((rc = dev_upload(p, &drows, rows.data(), rows.size())) ||
        (rc = dev_upload(p, &drowbase, rowbase.data(), rowbase.size())) ||
        (rc = dev_upload(p, &dl, d->lcoefs, (size_t)7 * K * d->ky1 * d->kz1)) ||
        (rc = dev_upload(p, &dd, d->dcoefs, (size_t)K * d->ky1 * d->kz1)) ||
        (rc = dev_upload(p, &dseedF, (const double *)nullptr, (size_t)P.nrows * 7 * K)) ||
        (rc = dev_upload(p, &dseedB, (const double *)nullptr, (size_t)P.nrows * 8 * K))) {
        tilu_plan_destroy(p);
        return rc;
    }
    if (d->variant == TILU_VARIANT_V1 &&
        ((rc = dev_upload(p, &dbandoff, bandoff.data(), bandoff.size())) ||
         (rc = dev_upload(p, &dstore, d->store_rows, (size_t)d->nband * 9)))) {
        tilu_plan_destroy(p);
        return rc;
    }
    if (d->arow) std::memcpy(p->harow, d->arow, sizeof(p->harow));
    if (d->arow && (rc = dev_upload(p, &darow, d->arow, 15))) {
        tilu_plan_destroy(p);
        return rc;
    }
    if (d->factors && (rc = dev_upload(p, &dfactors, d->factors, (size_t)P.grid * 9))) {
        tilu_plan_destroy(p);
        return rc;
    }
    double *dsepk = nullptr;
    if (d->sepk_tables) {
        if (!(d->sepk_w > 0.0)) {
            tilu_plan_destroy(p);
            return fail(TILU_EINVAL, "separable coefficient: W must be positive");
        }
        if ((rc = dev_upload(p, &dsepk, d->sepk_tables, (size_t)3 * (4 * n + 1)))) {
            tilu_plan_destroy(p);
            return rc;
        }
        P.sepk = dsepk;
        P.sepk_c0 = d->sepk_c0;
        P.sepk_w = d->sepk_w;
    }
    P.rows = drows;
    P.rowbase = drowbase;
    P.bandoff = dbandoff;
    P.store = dstore;
    P.seedF = dseedF;
    P.seedB = dseedB;
    // one operator form: on-the-fly separable rows, else the constant row, else per-point rows
    P.arow = dsepk ? nullptr : darow;
    P.arows = (dsepk || d->arow) ? nullptr : d->arows_dev;
    P.factors = dfactors ? dfactors : d->factors_dev;
    {
        const double zeros[15] = {};
        double *dz = nullptr;
        if ((rc = dev_upload(p, &dz, zeros, 15))) {
            tilu_plan_destroy(p);
            return rc;
        }
        p->zrow = dz;
    }
    if (d->acoefs) {
        P.akx1 = d->akx1;
        p->ky1a = d->aky1;
        p->kz1a = d->akz1;
        if ((rc = dev_upload(p, &dacoefs, d->acoefs, (size_t)15 * d->akx1 * d->aky1 * d->akz1)) ||
            (rc = dev_upload(p, &dseedA, (const double *)nullptr, (size_t)P.nrows * 15 * d->akx1))) {
            tilu_plan_destroy(p);
            return rc;
        }
        P.seedA = dseedA;
    }
    p->bsched = (n - 3 <= MAXR) ? reinterpret_cast<const void *>(1) : nullptr;  // batched path supports this level
    {
        std::vector<std::pair<std::pair<int, int>, int>> keyed;  // ((2y + 3z, z), (z << 10) | y)
        for (int z = 1; z <= n - 3; ++z)
            for (int y = 1; y <= n - 2 - z; ++y) keyed.push_back({{2 * y + 3 * z, z}, (z << 10) | y});
        std::sort(keyed.begin(), keyed.end());
        std::vector<int> order;
        for (auto &k : keyed) order.push_back(k.second);
        int *dorder = nullptr;
        if ((rc = dev_upload(p, &dorder, order.data(), order.size()))) {
            tilu_plan_destroy(p);
            return rc;
        }
        P.order = dorder;
    }
    launch_seed(P, dl, dd, dseedF, dseedB, 0);
    if (d->acoefs) launch_seed_op(P, dacoefs, d->aky1, d->akz1, dseedA, 0);
    if (cudaDeviceSynchronize() != cudaSuccess || (rc = check_cuda("seed tables"))) {
        rc = fail(TILU_ECUDA, "seed kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
        tilu_plan_destroy(p);
        return rc;
    }
    *out = p;
    return TILU_OK;
}

static int sweep_common(const tilu_plan_t *p, double *u, const double *f, int ntets, int sweeps, double *rnorm2,
                        bool stored, void *stream);

// solve_into on the fast kernels: w <- (L D L^T)^{-1} w is one smoothing step from u = 0 with right-hand side
// w and a ZERO operator row -- the residual f - 0 u is f bit for bit, and u = 0 + w' is w' -- so the plane /
// batched sweep kernels serve the drop-in method at their speed (the one-CTA-per-tet reference-layout kernels
// are ~10x slower from level 6 up).  The plan copy only swaps the operator; lazily built members (plane
// workspace, coefficient tables) created during the call are handed back to the plan.
static int solve_via_sweep(const tilu_plan_t *p, double *w, int ntets, bool stored, cudaStream_t s)
{
    static std::mutex mu;  // two first calls on one plan must not both create its workspace
    std::unique_lock<std::mutex> lk(mu, std::defer_lock);
    if ((ntets == 1 && !p->plane) || (ntets > 1 && !p->coef)) lk.lock();
    tilu_plan q = *p;
    q.dev.arow = p->zrow;
    q.dev.arows = nullptr;
    q.dev.sepk = nullptr;
    q.dev.seedA = nullptr;
    std::memset(q.harow, 0, sizeof(q.harow));
    Scratch sc(s);
    const size_t nd = (size_t)ntets * p->dev.grid;
    double *u0 = sc.get(nd);
    if (!u0) return fail(TILU_ENOMEM, "scratch allocation failed");
    cudaMemsetAsync(u0, 0, nd * sizeof(double), s);
    const int rc = sweep_common(&q, u0, w, ntets, 1, nullptr, stored, s);
    tilu_plan *mp = const_cast<tilu_plan *>(p);
    if (!mp->plane && q.plane) mp->plane = q.plane;
    if (!mp->coef && q.coef) mp->coef = q.coef;
    if (rc) return rc;
    const int nl = g_launches;
    cudaMemcpyAsync(w, u0, nd * sizeof(double), cudaMemcpyDeviceToDevice, s);
    g_launches = nl;
    return check_cuda("solve (sweep route)");
}

static bool sweep_route_fast(const tilu_plan_t *p, int ntets, bool stored)
{
    if (p->flags & TILU_SCHED_SIMPLE) return false;
    tilu_plan q = *p;
    q.dev.arow = p->zrow;
    q.dev.seedA = nullptr;
    const bool plane = ntets == 1 && plane_supported(&q) && !(p->flags & TILU_SCHED_BATCH) &&
                       ((p->flags & TILU_SCHED_PLANE) || p->dev.level >= plane_min_level());
    const bool batch = !stored && batch_ok(&q) && (ntets >= 2 || p->dev.level >= 6);
    return plane || batch;
}

static int solve_common(const tilu_plan_t *p, double *w, int ntets, int which, bool stored, void *stream)
{
    g_launches = 0;
    if (!valid_plan(p) || !w || ntets < 1) return fail(TILU_EINVAL, "invalid plan / vector / ntets");
    if (stored && !p->dev.factors) return fail(TILU_EINVAL, "plan has no stored factors");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (which == 3 && p->zrow && sweep_route_fast(p, ntets, stored)) return solve_via_sweep(p, w, ntets, stored, s);
    Scratch sc(s);
    double *state = nullptr;
    if (!stored && !(state = sc.get((size_t)ntets * p->dev.nrows * 8 * p->dev.kx1)))
        return fail(TILU_ENOMEM, "scratch allocation failed");
    prof_begin(s);
    const bool ok = launch_simple_solve(p->dev, !(p->flags & TILU_FAST), stored, w, state, nullptr, ntets, which, s);
    prof_end(stored ? "stored_solve" : "simple_solve", s);
    if (!ok) return fail(TILU_EUNSUPPORTED, "kx+1 = %d not compiled", p->dev.kx1);
    g_launches = (which == 3) ? 2 : 1;
    return check_cuda("solve");
}

int tilu_solve_into(const tilu_plan_t *p, double *w, int ntets, void *stream) { return solve_common(p, w, ntets, 3, false, stream); }
int tilu_surrogate_forward(const tilu_plan_t *p, double *w, int ntets, void *stream) { return solve_common(p, w, ntets, 1, false, stream); }
int tilu_surrogate_backward(const tilu_plan_t *p, double *w, int ntets, void *stream) { return solve_common(p, w, ntets, 2, false, stream); }
int tilu_stored_solve_into(const tilu_plan_t *p, double *w, int ntets, void *stream) { return solve_common(p, w, ntets, 3, true, stream); }

static int residual_into(const tilu_plan_t *p, const double *u, const double *f, double *w, int ntets, double *rnorm2,
                         double *part, cudaStream_t s)
{
    const PlanDev &P = p->dev;
    if (P.seedA) {
        prof_begin(s);
        const bool ok = launch_residual_sop(P, u, f, w, part, ntets, s);
        prof_end("residual_sop", s);
        if (!ok) return fail(TILU_EUNSUPPORTED, "operator surrogate degree");
    } else if (P.arow || P.arows || P.sepk) {
        prof_begin(s);
        launch_residual(P, !(p->flags & TILU_FAST), u, f, w, part, ntets, false, s);
        prof_end("residual", s);
    } else {
        return fail(TILU_EINVAL, "plan has no operator (arow / arows_dev / acoefs / sepk_tables)");
    }
    ++g_launches;
    if (rnorm2) {
        prof_begin(s);
        launch_reduce_rows(part, P.nrows, rnorm2, ntets, s);
        prof_end("reduce_rows", s);
        ++g_launches;
    }
    return TILU_OK;
}

int tilu_residual(const tilu_plan_t *p, const double *u, const double *f, double *w, int ntets, double *rnorm2,
                  void *stream)
{
    g_launches = 0;
    if (!valid_plan(p) || !u || !f || !w || ntets < 1) return fail(TILU_EINVAL, "invalid arguments");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Scratch sc(s);
    double *part = rnorm2 ? sc.get((size_t)ntets * p->dev.nrows) : nullptr;
    if (rnorm2 && !part) return fail(TILU_ENOMEM, "scratch allocation failed");
    int rc = residual_into(p, u, f, w, ntets, rnorm2, part, s);
    return rc ? rc : check_cuda("residual");
}

int tilu_stencil_apply(const tilu_plan_t *p, const double *u, double *out, int ntets, void *stream)
{
    g_launches = 0;
    if (!valid_plan(p) || !u || !out || ntets < 1) return fail(TILU_EINVAL, "invalid arguments");
    if (!p->dev.arow && !p->dev.arows && !p->dev.sepk) return fail(TILU_EINVAL, "plan has no stencil rows");
    launch_residual(p->dev, true, u, nullptr, out, nullptr, ntets, true, static_cast<cudaStream_t>(stream));
    g_launches = 1;
    return check_cuda("stencil_apply");
}

static int sweep_common(const tilu_plan_t *p, double *u, const double *f, int ntets, int sweeps, double *rnorm2,
                        bool stored, void *stream)
{
    g_launches = 0;
    if (!valid_plan(p) || !u || !f || ntets < 1 || sweeps < 0) return fail(TILU_EINVAL, "invalid arguments");
    if (stored && !p->dev.factors) return fail(TILU_EINVAL, "plan has no stored factors");
    if (sweeps == 0) return TILU_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const PlanDev &P = p->dev;
    // One macro-tet: the plane-layout band kernels (tilu_plane.cu) parallelise the sweep inside the tet.
    if (ntets == 1 && plane_supported(p) && !(p->flags & TILU_SCHED_BATCH) &&
        ((p->flags & TILU_SCHED_PLANE) || P.level >= plane_min_level())) {
        int nl = 0;
        const int rc = plane_sweep(p, u, f, ntets, sweeps, rnorm2, s, &nl, stored);
        g_launches += nl;
        if (rc) return fail(rc, "plane sweep failed (%d): %s", rc, cudaGetErrorString(cudaGetLastError()));
        return check_cuda("plane sweep");
    }
    // Batched dataflow kernels for several tets, and for one large tet (1 tet in a 32-lane group still
    // beats the one-CTA-per-tet reference-layout kernels by ~10x from level 6 up: tools/single_tet.py).
    if (!stored && batch_ok(p) && (ntets >= 2 || P.level >= 6)) {
        // reference layout in, packed sweeps, reference layout out
        Scratch sc(s);
        const size_t pk = packed_doubles(p, ntets);
        double *up = sc.get(pk), *fp = sc.get(pk), *wp = sc.get(packed_scratch_doubles(p, ntets));
        if (!up || !fp || !wp) return fail(TILU_ENOMEM, "scratch allocation failed");
        cudaMemsetAsync(wp, 0, kScratchHdr * sizeof(double), s);  // header 0: arm on first use
        prof_begin(s);
        launch_pack(u, up, P.grid, ntets, batch_tpl(ntets), s);
        launch_pack(f, fp, P.grid, ntets, batch_tpl(ntets), s);
        prof_end("pack", s);
        int rc = packed_sweeps(p, up, fp, wp, ntets, sweeps, rnorm2, s);
        if (rc) return rc;
        prof_begin(s);
        launch_unpack(up, u, P.grid, ntets, batch_tpl(ntets), s);
        prof_end("unpack", s);
        g_launches += 3;  // + the sweeps' own launches counted by packed_sweeps
        return check_cuda("batched sweep");
    }
    Scratch sc(s);
    double *w = sc.get((size_t)ntets * P.grid);
    double *state = stored ? nullptr : sc.get((size_t)ntets * P.nrows * 8 * P.kx1);
    double *part = sc.get((size_t)ntets * P.nrows);
    if (!w || (!stored && !state) || !part) return fail(TILU_ENOMEM, "scratch allocation failed");
    cudaMemsetAsync(w, 0, sizeof(double) * ntets * P.grid, s);
    const bool exact = !(p->flags & TILU_FAST);
    for (int k = 0; k < sweeps; ++k) {
        int rc = residual_into(p, u, f, w, ntets, rnorm2 ? rnorm2 + (int64_t)k * ntets : nullptr, part, s);
        if (rc) return rc;
        prof_begin(s);
        bool ok = launch_simple_solve(P, exact, stored, w, state, u, ntets, 1, s);
        prof_end(stored ? "stored_fwd" : "simple_fwd", s);
        prof_begin(s);
        ok = ok && launch_simple_solve(P, exact, stored, w, state, u, ntets, 2, s);
        prof_end(stored ? "stored_bwd" : "simple_bwd", s);
        if (!ok) return fail(TILU_EUNSUPPORTED, "kx+1 = %d not compiled", P.kx1);
        g_launches += 2;
    }
    return check_cuda("sweep");
}

int64_t tilu_packed_size(const tilu_plan_t *p, int ntets)
{
    return (p && ntets > 0) ? (int64_t)packed_doubles(p, ntets) : -1;
}
int64_t tilu_packed_scratch_size(const tilu_plan_t *p, int ntets)
{
    return (p && ntets > 0) ? (int64_t)packed_scratch_doubles(p, ntets) : -1;
}

int tilu_pack(const tilu_plan_t *p, const double *src, double *dst, int ntets, void *stream)
{
    g_launches = 0;
    if (!valid_plan(p) || !src || !dst || ntets < 1) return fail(TILU_EINVAL, "invalid arguments");
    launch_pack(src, dst, p->dev.grid, ntets, batch_tpl(ntets), static_cast<cudaStream_t>(stream));
    g_launches = 1;
    return check_cuda("pack");
}

int tilu_unpack(const tilu_plan_t *p, const double *src, double *dst, int ntets, void *stream)
{
    g_launches = 0;
    if (!valid_plan(p) || !src || !dst || ntets < 1) return fail(TILU_EINVAL, "invalid arguments");
    launch_unpack(src, dst, p->dev.grid, ntets, batch_tpl(ntets), static_cast<cudaStream_t>(stream));
    g_launches = 1;
    return check_cuda("unpack");
}

int tilu_sweep_packed(const tilu_plan_t *p, double *u_p, const double *f_p, double *w_p, int ntets, int sweeps,
                      double *rnorm2, void *stream)
{
    g_launches = 0;
    if (!valid_plan(p) || !u_p || !f_p || !w_p || ntets < 1 || sweeps < 0) return fail(TILU_EINVAL, "invalid arguments");
    if (!batch_ok(p)) return fail(TILU_EUNSUPPORTED, "packed sweeps need level <= 9 and the batched schedule");
    int rc = packed_sweeps(p, u_p, f_p, w_p, ntets, sweeps, rnorm2, static_cast<cudaStream_t>(stream));
    return rc ? rc : check_cuda("packed sweep");
}

int tilu_sweep(const tilu_plan_t *p, double *u, const double *f, int ntets, int sweeps, double *rnorm2, void *stream)
{
    return sweep_common(p, u, f, ntets, sweeps, rnorm2, false, stream);
}

int tilu_stored_sweep(const tilu_plan_t *p, double *u, const double *f, int ntets, int sweeps, double *rnorm2,
                      void *stream)
{
    return sweep_common(p, u, f, ntets, sweeps, rnorm2, true, stream);
}

}  // extern "C"
