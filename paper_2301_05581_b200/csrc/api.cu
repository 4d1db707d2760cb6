// api.cu -- the C-ABI of libnufi_b200.so (declared in include/nufi.h).
//
// Owns the device-resident potential history (PotentialHistory,
// spline.py:108-155, preallocated to n_max + 1 slabs instead of doubling),
// the per-step scratch, and the launch sequence of one NuFI step:
//   trace_rho (trace + f0 + per-tile v-sums)  -> reduce_blocks (fixed-order
//   v-block sums) -> [caller's allreduce for multi-rank] -> field_update
//   (combine, neutralise, Poisson, spline fit, append, W, E).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <string>
#include <algorithm>
#include <map>
#include <vector>

#include "field_common.cuh"

namespace nufi {
size_t trace_rho_smem_bytes(const TraceRhoParams &p, int threads);
cudaError_t launch_trace_rho(int d, int ppt, bool pow2, const TraceRhoParams &p, double K, int ctas, int threads,
                             cudaStream_t st);
cudaError_t launch_sweep_moments(int d, int ppt, bool pow2, const TraceRhoParams &p, double K, int ctas, int threads,
                                 cudaStream_t st);
cudaError_t launch_reduce_moments(const double *part, int rows, int d, double measure, double *out, cudaStream_t st);
int launch_reduce_exchange(const double *partial, const double *fminmax, int nodes, int node_tiles, int vt_per_block,
                           int b_lo, int b_hi, int B, const MgExchange &x, cudaStream_t st);
cudaError_t launch_reduce_blocks(const double *partial, const double *fminmax, double *out, int nodes,
                                 int node_tiles, int vt_per_block, int b_lo, int b_hi, int B, cudaStream_t st);
cudaError_t launch_trace_points_ring(int d, bool pow2, const double *ev_hist, int ev_slab_elems, int N, double L,
                                     int n, double tau, double K, double *X, double *V, int64_t M, int half_kick,
                                     cudaStream_t st);
cudaError_t launch_bspline_weights(const double *t, int64_t M, double *w, double *dw, cudaStream_t st);
cudaError_t launch_trace_points_generic(int d, const double *hist, int nodes, const double *ovr,
                                        const double *ovr_slabs, int N, double L, int n, double tau, double *X,
                                        double *V, int64_t M, int half_kick, cudaStream_t st);
cudaError_t launch_trace_points(int d, int mode, bool pow2, const double *hist, const double *ev_hist,
                                int ev_slab_elems, int N, int nodes, double L, int n, double tau, double K, double *X,
                                double *V, int64_t M, int half_kick, cudaStream_t st);
cudaError_t launch_eval_field(int d, const double *c, int N, double L, const double *X, int64_t M, double *phi,
                              double *E, cudaStream_t st);
cudaError_t launch_poisson_fit(const FieldParams &p, int mode, const double *in, double *out, double *spec_re,
                               double *spec_im, double *W, int *status, cudaStream_t st);
cudaError_t launch_eval_f0(int d, const F0Params &f0, const double *X, const double *V, int64_t M, double *F,
                           cudaStream_t st);
cudaError_t launch_trace_rho_1d(const TraceRhoParams &p, const FieldParams &fp, int fuse, unsigned *ticket, int ctas,
                                int threads, cudaStream_t st);
int trace_rho_1d_sps(int N, bool wide);
cudaError_t launch_trace_rho_global(int d, bool mom, bool pow2, const TraceRhoParams &p, double K, int ctas,
                                    int threads, cudaStream_t st);
cudaError_t launch_field_large(const FieldParams &f, double *scratch, cudaStream_t st);
size_t field_large_scratch_doubles(int nodes);
cudaError_t launch_halo_table(int d, int N, int *halo, cudaStream_t st);
cudaError_t launch_field_tables(double *tw, double *fac, double *k2, int d, int N, int nodes, double k_scale,
                                cudaStream_t st);
cudaError_t launch_run_1d(const Run1DParams &P, int threads, int device, cudaStream_t st, int *grid_out);
cudaError_t launch_build_ev_slabs(double *hist, double *ev_hist, int d, int N, int nodes, int ev_slab_elems,
                                  double K, int64_t r0, int64_t r1, int f32, cudaStream_t st);
}  // namespace nufi

namespace nufi {
cudaError_t launch_field_update(const FieldParams &p, cudaStream_t st, int threads);
cudaError_t launch_rho_bar(const RhoBarParams &p, cudaStream_t st);
}  // namespace nufi

using namespace nufi;

// ----------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------

static thread_local std::string g_last_error;

static int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

#define CU(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t _e = (expr);                                                                  \
        if (_e != cudaSuccess)                                                                    \
            return fail(NUFI_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));     \
    } while (0)

// Stream-ordered temporary device buffers of one call, released on every exit path
// (including the early returns of CU).
struct AsyncTemps {
    cudaStream_t st;
    void *p[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    int n = 0;
    explicit AsyncTemps(cudaStream_t s) : st(s) {}
    template <class T>
    cudaError_t alloc(T **out, size_t bytes) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(out), bytes, st);
        if (e == cudaSuccess) p[n++] = *out;
        return e;
    }
    ~AsyncTemps() {
        for (int i = 0; i < n; ++i) cudaFreeAsync(p[i], st);
    }
};

#define CHECK_HANDLE(h)                                                                           \
    do {                                                                                          \
        if (!(h)) return fail(NUFI_ERR_USAGE, "null handle");                                     \
        CU(cudaSetDevice((h)->device));                                                           \
    } while (0)

// ----------------------------------------------------------------------------
// handle
// ----------------------------------------------------------------------------

struct nufi_handle {
    nufi_config cfg{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;

    int d = 1, N = 0, Nv = 0, nodes = 0;
    int64_t V = 0;  // Nv^d
    int64_t cap = 0;
    bool pow2 = false;
    double hx = 0, inv_h = 0, hv = 0, hv_d = 0, L_d = 0, K = 0, rho_bar = 0;
    F0Params f0{};

    // v-blocks and CTA tiling
    int B = 1, b_lo = 0, b_hi = 1;
    int threads = 128, ppt = 1, passes = 1, vt_rows = 4, vt_total = 1, vt_per_block = 1, node_tiles = 1;
    int sps = 1, stages = 2, ev_elems = 0;

    // device buffers
    double *hist = nullptr, *ev_hist = nullptr;
    double *partial = nullptr, *fminmax = nullptr, *blocks = nullptr;
    double *d_rho = nullptr, *d_E = nullptr, *d_W = nullptr, *d_stats = nullptr, *d_rho_bar = nullptr;
    double *row_last = nullptr;  // split d = 1 runs: the helpers' last rows (+ (min, max) pairs), lazily
    double *tables = nullptr;  // field_common.cuh constant tables: 4N + 3 Nx^d doubles
    unsigned *ticket = nullptr;  // last-CTA-done counter of the fused d = 1 step
    unsigned *tile_cnt = nullptr;  // d >= 2 fused block reduce: node_tiles + 1 arrival counters
    double *block_mm = nullptr;    // d >= 2 fused block reduce: (min, max) per (block, node tile)
    unsigned *barrier = nullptr;  // grid-barrier counter of the persistent d = 1 run kernel
    int *d_status = nullptr;
    int64_t *d_len = nullptr;
    // run outputs (device) and their pinned host staging
    double *run_dev = nullptr, *run_host = nullptr;
    size_t run_elems = 0;
    // observable sweep: per-CTA moment rows + the reduced vector (lazily allocated)
    double *mom_part = nullptr, *d_mom = nullptr;
    // multi-rank run with the exchange fused into the persistent d = 1 kernel
    int mg_world = 1, mg_rank = 0, mg_emulated = 0;
    unsigned mg_steps = 0;            // arrival-flag base (steps run so far in mg mode)
    void *mg_own = nullptr;           // cudaMalloc'd: exchange table (2 x stride) + G flags
    void *mg_peer[NUFI_MG_MAX] = {};  // every rank's buffer (own / IPC-opened / emulated)
    bool mg_opened[NUFI_MG_MAX] = {};
    double *mg_part[NUFI_MG_MAX] = {}, *mg_fmm[NUFI_MG_MAX] = {};  // emulated ranks' partials
    unsigned *mg_bar[NUFI_MG_MAX] = {};
    int *mg_error = nullptr;
    // installed non-spline fields (FlowContext.install_field, flow.py:44-47): per step
    // [flag, E0_x, E0_y, E0_z]; honoured by the point-level trace (the reference's generic path)
    std::vector<double> ovr;                        // per slot: kind (0 stored, 1 uniform, 2 spline) + 3 values
    std::map<int64_t, std::vector<double>> ovr_spline;  // installed SplineField slabs by slot
    int64_t n_ovr = 0;

    // stream-ordered drop-in calls (nufi_rho_async / nufi_field_update_async): a ring of
    // pinned host entries [rho | stats 3 | W 1 | pad | E nodes*d | coeffs nodes], one event each
    std::vector<double *> aring;     // per-slot pointers into aring_block
    double *aring_block = nullptr;   // one contiguous pinned block of all slots
    size_t aring_block_elems = 0;
    std::vector<cudaEvent_t> aev;
    size_t aslot_elems = 0;
    bool d_rho_async = false;  // d_rho holds the density of the last nufi_rho_async
    int64_t spec = -1;         // slot n holds a speculative (uncommitted) tail of nufi_rho_async(n)

    int64_t len = 0;  // host mirror of the history length
    bool large = false;   // Nx^d > MAX_FIELD_NODES: multi-CTA tail (field_large.cu)
    bool gl = false;      // slabs too large for a shared-memory ring: traced in place (GL kernels)
    double *large_scratch = nullptr;
    int *halo = nullptr;  // d >= 2 evaluation-slab source indices
    int f32 = 0;      // NUFI_FLAG_F32_HISTORY

    // optional per-launch event timing (nufi_profile)
    bool profiling = false;
    struct Pending {
        cudaEvent_t a, b;
        int kind;  // 0 trace, 1 reduce, 2 field
        double point_steps;
    };
    std::vector<Pending> pending;
    double prof[8] = {0};
};

// Record events around one launch when profiling (resolved lazily by nufi_profile_read).
struct ProfScope {
    nufi_handle *h;
    int kind;
    double ps;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(nufi_handle *h_, int kind_, double ps_ = 0) : h(h_), kind(kind_), ps(ps_) {
        if (h->profiling) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, h->stream);
        }
    }
    ~ProfScope() {
        if (h->profiling) {
            cudaEventRecord(b, h->stream);
            h->pending.push_back({a, b, kind, ps});
        }
    }
};

static bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---- memory: stream-ordered device allocations from the device's default pool
// (retained across handles: release threshold = max), pinned host staging from a
// process-wide cache.  Creating and destroying a handle per run (the public
// Simulation(...).run() call) then costs no cudaMalloc / cudaFree / page pinning,
// each of which synchronises the device or the OS (measured 25-275 ms per destroy).
static cudaError_t pool_init(int device) {
    static bool done[64] = {false};
    if (device < 0 || device >= 64 || done[device]) return cudaSuccess;
    cudaMemPool_t pool;
    cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
    if (e != cudaSuccess) return e;
    uint64_t thr = UINT64_MAX;
    e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    if (e == cudaSuccess) done[device] = true;
    return e;
}

template <typename T>
static cudaError_t dalloc(T **p, size_t bytes, cudaStream_t st) {
    return cudaMallocAsync(reinterpret_cast<void **>(p), bytes ? bytes : 8, st);
}

struct PinnedCache {
    std::mutex mu;
    std::vector<std::pair<size_t, double *>> free_blocks;
};
static PinnedCache &pinned_cache() {
    static PinnedCache *c = new PinnedCache();  // never destroyed: no teardown-order issues
    return *c;
}
static cudaError_t pinned_get(double **p, size_t elems) {
    {
        std::lock_guard<std::mutex> lk(pinned_cache().mu);
        auto &v = pinned_cache().free_blocks;
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i].first >= elems) {
                *p = v[i].second;
                v.erase(v.begin() + i);
                return cudaSuccess;
            }
    }
    return cudaMallocHost(reinterpret_cast<void **>(p), elems * sizeof(double));
}
static void pinned_put(double *p, size_t elems) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(pinned_cache().mu);
    pinned_cache().free_blocks.push_back({elems, p});
}

// Library-owned streams are recycled across handles (creating + destroying a stream costs
// ~90 us of host time, a third of a small run's end-to-end overhead); a stream returns to
// the pool idle (nufi_destroy synchronises it first).  Bounded per device.
struct StreamPool {
    std::mutex mu;
    std::map<int, std::vector<cudaStream_t>> free_streams;
};
static StreamPool &stream_pool() {
    static StreamPool *p = new StreamPool();  // never destroyed: no teardown-order issues
    return *p;
}
static cudaError_t stream_get(int device, cudaStream_t *st) {
    {
        std::lock_guard<std::mutex> lk(stream_pool().mu);
        auto &v = stream_pool().free_streams[device];
        if (!v.empty()) {
            *st = v.back();
            v.pop_back();
            return cudaSuccess;
        }
    }
    return cudaStreamCreateWithFlags(st, cudaStreamNonBlocking);
}
static void stream_put(int device, cudaStream_t st) {
    {
        std::lock_guard<std::mutex> lk(stream_pool().mu);
        auto &v = stream_pool().free_streams[device];
        if (v.size() < 16) {
            v.push_back(st);
            return;
        }
    }
    cudaStreamDestroy(st);
}

static int ipow(int b, int e) {
    int r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
}

// Reference validation rules.
static int validate(const nufi_config &c) {
    char buf[256];
    if (c.d < 1 || c.d > 3) {
        snprintf(buf, sizeof buf, "dimension must be 1, 2 or 3, got %d", c.d);  // grids.py:28-29
        return fail(NUFI_ERR_USAGE, buf);
    }
    if (c.Nx < 2 || c.Nv < 2) {
        snprintf(buf, sizeof buf, "need Nx >= 2 and Nv >= 2, got Nx=%d, Nv=%d", c.Nx, c.Nv);  // grids.py:30-31
        return fail(NUFI_ERR_USAGE, buf);
    }
    if (!(c.L > 0 && c.vmax > 0)) {
        snprintf(buf, sizeof buf, "need L > 0 and vmax > 0, got L=%g, vmax=%g", c.L, c.vmax);  // grids.py:32-33
        return fail(NUFI_ERR_USAGE, buf);
    }
    if (c.Nx < 4) {
        snprintf(buf, sizeof buf, "spline fitting needs Nx >= 4, got %d", c.Nx);  // spline.py:73-74
        return fail(NUFI_ERR_USAGE, buf);
    }
    if (!(c.tau > 0)) {
        snprintf(buf, sizeof buf, "time step must be positive, got %g", c.tau);  // spline.py:119-120
        return fail(NUFI_ERR_USAGE, buf);
    }
    if (c.n_max < 0) return fail(NUFI_ERR_USAGE, "n_max must be >= 0");
    if (c.flags & ~NUFI_FLAG_F32_HISTORY) return fail(NUFI_ERR_USAGE, "unknown nufi_config flags");
    for (int a = 0; a < c.d; ++a) {
        const nufi_profile &p = c.profiles[a];
        if (p.n_centers < 1 || p.n_centers > NUFI_MAX_CENTERS)
            return fail(NUFI_ERR_USAGE, "centers and weights must be non-empty and equal-length");  // initial.py:33-34
        if (p.power != 0 && p.power != 2) {
            snprintf(buf, sizeof buf, "velocity power must be 0 or 2, got %d", p.power);  // initial.py:35-36
            return fail(NUFI_ERR_USAGE, buf);
        }
        for (int m = 0; m < p.n_centers; ++m)
            if (!(p.weights[m] > 0)) return fail(NUFI_ERR_USAGE, "mixture weights must be positive");  // initial.py:37-38
    }
    if (c.alpha < 0) {
        snprintf(buf, sizeof buf, "perturbation amplitude must be >= 0, got %g", c.alpha);  // initial.py:91-92
        return fail(NUFI_ERR_USAGE, buf);
    }
    if (c.alpha * c.d > 1.0 + 1e-12) {
        snprintf(buf, sizeof buf, "alpha*d = %g > 1 makes f0 negative", c.alpha * c.d);  // initial.py:93-94
        return fail(NUFI_ERR_USAGE, buf);
    }
    const double cycles = c.k * c.L / (2.0 * M_PI);
    if (std::fabs(cycles - std::round(cycles)) > 1e-9) {
        snprintf(buf, sizeof buf, "k*L = %g is not a multiple of 2*pi; f0 would not be x-periodic", c.k * c.L);
        return fail(NUFI_ERR_USAGE, buf);  // initial.py:95-99
    }
    const long long nodes = (long long)std::pow((double)c.Nx, c.d);
    if (nodes > MAX_GRID_NODES) {
        snprintf(buf, sizeof buf, "Nx^d = %lld exceeds the supported grid size %d", nodes, MAX_GRID_NODES);
        return fail(NUFI_ERR_CONFIG, buf);
    }
    const double V = std::pow((double)c.Nv, c.d);
    if (V * (double)nodes > 9.0e15) return fail(NUFI_ERR_CONFIG, "too many quadrature points");
    return NUFI_OK;
}

// CTA tiling: v-rows per CTA tile = warps * ppt * passes must divide V / B.
static void choose_tiling(nufi_handle *h) {
    const int64_t per_block = h->V / h->B;
    int warps, ppt, passes;
    if (h->d == 1) {
        warps = 8, ppt = 1, passes = 1;  // trace_rho_1d: one point per thread
        if (h->N == 256) {
            // throughput regime (many tiles per SM): one 16-warp CTA per SM sharing one deep
            // ring (2 x 16 slabs) beats two 8-warp CTAs with 2 x 8 each (sl1 218.7 -> 203 ms)
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
            // rows of the FULL grid, not this rank's share: the tile height fixes how a block's
            // rows are grouped when summed, so every rank count must pick the same one
            const int64_t rows = per_block * h->B, nt = (h->nodes + 31) / 32;
            if ((rows / 16) * nt >= 2 * (int64_t)sms) warps = 16;
            // the 16-warp (WIDE) run kernel exists for N = 256 only
            if (const char *e = getenv("NUFI_D1_WARPS")) warps = atoi(e) >= 16 ? 16 : 8;
        }
    } else if (h->d == 2) {
        warps = 8, ppt = 2, passes = 1;  // 2 interleaved points per thread, 2 CTAs / SM
    } else {
        warps = 8, ppt = 2, passes = 4;
    }
    if (h->d >= 2) {
        if (const char *e = getenv("NUFI_PPT")) ppt = std::max(1, std::min(2, atoi(e)));
        if (const char *e = getenv("NUFI_PASSES")) passes = std::max(1, atoi(e));
    }
    while (warps > 1 && (per_block % (warps * ppt) != 0)) warps >>= 1;
    if (h->d == 1) {
        // latency-bound small grids: fewer rows per tile so the tiles spread over all SMs
        // (wl1: 64 tiles of 8 rows -> 128 tiles of 4); the CTA stays 9 warps wide
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
        const int64_t nt = (h->nodes + 31) / 32;
        // rows of the full grid (see above): a sharded rank tiles exactly like one GPU, so its
        // block sums -- and the history -- are bit-identical for every rank count
        const int64_t rows = per_block * h->B;
        while (warps > 1 && (rows / (warps / 2)) * nt <= sms && per_block % (warps / 2) == 0) warps >>= 1;
    }
    while (ppt > 1 && (per_block % (warps * ppt) != 0)) ppt >>= 1;
    while (passes > 1 && (per_block % ((int64_t)warps * ppt * passes) != 0)) passes >>= 1;
    if (per_block % ((int64_t)warps * ppt * passes) != 0) warps = ppt = passes = 1;
    h->threads = h->d == 1 ? (warps > 8 ? 512 : 256) : warps * 32;  // d = 1: warp slots (+ producer)
    h->ppt = ppt;
    h->passes = passes;
    h->vt_rows = warps * ppt * passes;
    h->vt_total = (int)(h->V / h->vt_rows);
    h->vt_per_block = (int)(per_block / h->vt_rows);
    h->node_tiles = (h->nodes + 31) / 32;
    // TMA ring: slabs per stage and stage count
    const int slab_bytes = h->ev_elems * 8;
    if (h->d == 1) {
        h->sps = trace_rho_1d_sps(h->N, h->threads > 256);  // must match the kernel's template instantiation
        // N = 256: 4 stages so 2 CTAs / SM still fit (the tail workspace aliases the ring);
        // small grids run one CTA per SM and take a deeper ring (ts1 barrier wait -5 %)
        // deep stages, few hand-offs: 2 x 64 slabs (N = 64, one CTA / SM), 2 x 8 (N = 256, two CTAs / SM)
        h->stages = (h->N == 64 && h->sps >= 32) || (h->N == 256 && h->sps >= 8) ? 2 : (h->N <= 64 ? 6 : 4);
        if (const char *e = getenv("NUFI_D1_STAGES")) h->stages = std::max(2, atoi(e));
    } else if (h->d == 2) {
        // 2-deep ring with stages as large as two CTAs per SM allow (~100 KB of ring per CTA):
        // fewer, larger refills (wl2: 5 slabs per stage, +2 % over 4)
        h->sps = std::max(1, (100 * 1024) / (2 * slab_bytes));
        h->stages = 2;
    } else {
        h->sps = std::max(1, 32768 / slab_bytes);
        h->stages = 2;
    }
    if (h->d >= 2) {
        if (const char *e = getenv("NUFI_SPS")) h->sps = std::max(1, atoi(e));
        if (const char *e = getenv("NUFI_STAGES")) h->stages = std::max(2, atoi(e));
        // keep the ring within the 227 KB per-CTA shared-memory limit
        while (h->sps > 1 && (size_t)h->stages * h->sps * slab_bytes > 200 * 1024) --h->sps;
        while (h->stages > 2 && (size_t)h->stages * h->sps * slab_bytes > 200 * 1024) --h->stages;
        h->gl = (size_t)h->stages * h->sps * slab_bytes > 200 * 1024;  // even 2 x 1 slab does not fit
    }
}

// f0 descriptor + background density (initial.py:165-180, 187-208)
static int install_ic(nufi_handle *h, const nufi_config &c) {
    h->cfg.alpha = c.alpha;
    h->cfg.k = c.k;
    h->cfg.rho_bar = c.rho_bar;
    for (int a = 0; a < 3; ++a) h->cfg.profiles[a] = c.profiles[a];
    h->f0 = F0Params{};
    h->f0.d = c.d;
    h->f0.alpha = c.alpha;
    h->f0.k = c.k;
    for (int a = 0; a < c.d; ++a) {
        h->f0.n_centers[a] = c.profiles[a].n_centers;
        h->f0.power[a] = c.profiles[a].power;
        for (int m = 0; m < NUFI_MAX_CENTERS; ++m) {
            h->f0.centers[a][m] = c.profiles[a].centers[m];
            h->f0.weights[a][m] = c.profiles[a].weights[m];
        }
    }
    if (std::isnan(c.rho_bar)) {
        RhoBarParams rp{};
        rp.d = c.d;
        rp.N = c.Nx;
        rp.Nv = c.Nv;
        rp.hx = h->hx;
        rp.hv = h->hv;
        rp.vmax = c.vmax;
        rp.hx_d = std::pow(h->hx, (double)c.d);
        rp.hv_d = h->hv_d;
        rp.L_d = h->L_d;
        rp.f0 = h->f0;
        rp.out = h->d_rho_bar;
        CU(launch_rho_bar(rp, h->stream));
        CU(cudaMemcpyAsync(&h->rho_bar, h->d_rho_bar, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CU(cudaStreamSynchronize(h->stream));
    } else {
        h->rho_bar = c.rho_bar;
    }
    return NUFI_OK;
}

static int grow(nufi_handle *h, int64_t cap) {
    if (cap <= h->cap) return NUFI_OK;
    double *nh = nullptr, *ne = nullptr;
    CU(dalloc(&nh, cap * (size_t)h->nodes * sizeof(double), h->stream));
    CU(dalloc(&ne, cap * (size_t)h->ev_elems * sizeof(double), h->stream));
    if (h->len > 0) {
        CU(cudaMemcpyAsync(nh, h->hist, h->len * (size_t)h->nodes * sizeof(double), cudaMemcpyDeviceToDevice,
                           h->stream));
        CU(cudaMemcpyAsync(ne, h->ev_hist, h->len * (size_t)h->ev_elems * sizeof(double), cudaMemcpyDeviceToDevice,
                           h->stream));
    }
    CU(cudaStreamSynchronize(h->stream));
    cudaFreeAsync(h->hist, h->stream);
    cudaFreeAsync(h->ev_hist, h->stream);
    h->hist = nh;
    h->ev_hist = ne;
    h->cap = cap;
    h->cfg.n_max = (int32_t)(cap - 1);
    return NUFI_OK;
}

extern "C" {

int nufi_set_initial_condition(nufi_handle *h, const nufi_config *cfg) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    if (!cfg) return fail(NUFI_ERR_USAGE, "null config");
    if (cfg->d != h->cfg.d || cfg->Nx != h->cfg.Nx || cfg->Nv != h->cfg.Nv || cfg->L != h->cfg.L ||
        cfg->vmax != h->cfg.vmax)
        return fail(NUFI_ERR_USAGE, "initial condition grid does not match the history grid");
    nufi_config c = h->cfg;
    c.alpha = cfg->alpha;
    c.k = cfg->k;
    c.rho_bar = cfg->rho_bar;
    for (int a = 0; a < 3; ++a) c.profiles[a] = cfg->profiles[a];
    int rc = validate(c);
    if (rc) return rc;
    return install_ic(h, c);
}

int nufi_reserve(nufi_handle *h, int64_t slabs) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    if (slabs > (int64_t)1 << 30) return fail(NUFI_ERR_USAGE, "capacity too large");
    return grow(h, slabs);
}

int64_t nufi_capacity(nufi_handle *h) { return h ? h->cap : 0; }

const char *nufi_last_error(void) { return g_last_error.c_str(); }
int nufi_abi_version(void) { return NUFI_ABI_VERSION; }

int nufi_create(const nufi_config *cfg, int device, void *stream, nufi_handle **out) {
    if (!cfg || !out) return fail(NUFI_ERR_USAGE, "null argument");
    *out = nullptr;
    int rc = validate(*cfg);
    if (rc) return rc;
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(NUFI_ERR_USAGE, "invalid device index");
    CU(cudaSetDevice(device));

    nufi_handle *h = new nufi_handle();
    h->cfg = *cfg;
    h->device = device;
    if (stream) {
        h->stream = (cudaStream_t)stream;
    } else {
        CU(stream_get(device, &h->stream));
        h->own_stream = true;
    }
    const nufi_config &c = *cfg;
    h->d = c.d;
    h->N = c.Nx;
    h->Nv = c.Nv;
    h->nodes = ipow(c.Nx, c.d);
    h->V = 1;
    for (int a = 0; a < c.d; ++a) h->V *= c.Nv;
    h->cap = (int64_t)c.n_max + 1;
    h->pow2 = (c.Nx & (c.Nx - 1)) == 0;
    h->hx = c.L / c.Nx;                       // grids.py:37-38
    h->hv = 2.0 * c.vmax / c.Nv;              // grids.py:41-42
    h->inv_h = (double)c.Nx / c.L;            // kernels.py:187
    h->hv_d = std::pow(h->hv, (double)c.d);   // density.py:75
    h->L_d = std::pow(c.L, (double)c.d);      // poisson.py:120
    h->K = -(c.tau * c.tau) * (h->inv_h * h->inv_h);
    // v-blocks (fixed combine order, independent of the rank count)
    int B = c.v_blocks > 0 ? c.v_blocks : 8;
    if (B > 8) {
        if (h->own_stream) stream_put(device, h->stream);
        delete h;
        return fail(NUFI_ERR_USAGE, "v_blocks must be <= 8");
    }
    while (B > 1 && (h->V % B != 0)) --B;
    if (c.v_blocks > 0 && B != c.v_blocks) {
        if (h->own_stream) stream_put(device, h->stream);
        delete h;
        return fail(NUFI_ERR_USAGE, "v_blocks must divide Nv^d");
    }
    h->B = B;
    h->b_lo = c.block_hi > c.block_lo ? c.block_lo : 0;
    h->b_hi = c.block_hi > c.block_lo ? c.block_hi : B;
    if (h->b_lo < 0 || h->b_hi > B) {
        if (h->own_stream) stream_put(device, h->stream);
        delete h;
        return fail(NUFI_ERR_USAGE, "block range outside [0, v_blocks)");
    }
    h->ev_elems = ev_slab_elems(c.d, c.Nx);
    h->f32 = (c.flags & NUFI_FLAG_F32_HISTORY) ? 1 : 0;
    // beyond one CTA: too many nodes, or (d = 1, 14-16 work rows of N doubles) a single-CTA
    // tail that would not fit the 227 KB of shared memory a CTA can have
    h->large = h->nodes > MAX_FIELD_NODES || field_smem_doubles(h->nodes, c.Nx, c.d == 1) * sizeof(double) > 227 * 1024;
    choose_tiling(h);
    if (h->large && h->d == 1) h->gl = true;  // d = 1 beyond one CTA: generic in-place trace

    const size_t nodes = h->nodes;
    CU(pool_init(device));
    CU(dalloc(&h->hist, h->cap * nodes * sizeof(double), h->stream));
    CU(dalloc(&h->ev_hist, h->cap * (size_t)h->ev_elems * sizeof(double), h->stream));
    // x2: the persistent d = 1 run kernel double-buffers the tile partials by step parity
    CU(dalloc(&h->partial, 2 * (size_t)h->vt_total * h->node_tiles * 32 * sizeof(double), h->stream));
    CU(dalloc(&h->fminmax, 2 * (size_t)h->vt_total * h->node_tiles * 2 * sizeof(double), h->stream));
    CU(dalloc(&h->blocks, ((size_t)h->B * nodes + 2 * h->B) * sizeof(double), h->stream));
    CU(dalloc(&h->d_rho, nodes * sizeof(double), h->stream));
    CU(dalloc(&h->d_E, nodes * c.d * sizeof(double), h->stream));
    CU(dalloc(&h->d_W, 8 * sizeof(double), h->stream));
    CU(dalloc(&h->d_stats, 8 * sizeof(double), h->stream));
    CU(dalloc(&h->d_rho_bar, sizeof(double), h->stream));
    CU(dalloc(&h->d_status, sizeof(int), h->stream));
    CU(dalloc(&h->d_len, sizeof(int64_t), h->stream));
    if (h->large) CU(dalloc(&h->large_scratch, field_large_scratch_doubles(h->nodes) * sizeof(double), h->stream));
    if (c.d >= 2) {
        CU(dalloc(&h->halo, (size_t)ev_slab_raw_elems(c.d, c.Nx) * sizeof(int), h->stream));
        CU(launch_halo_table(c.d, c.Nx, h->halo, h->stream));
        CU(dalloc(&h->tile_cnt, ((size_t)h->node_tiles + 1) * sizeof(unsigned), h->stream));
        CU(cudaMemsetAsync(h->tile_cnt, 0, ((size_t)h->node_tiles + 1) * sizeof(unsigned), h->stream));
        CU(dalloc(&h->block_mm, (size_t)h->B * h->node_tiles * 2 * sizeof(double), h->stream));
    }
    CU(dalloc(&h->tables, (4 * (size_t)h->N + 3 * nodes) * sizeof(double), h->stream));
    CU(dalloc(&h->ticket, sizeof(unsigned), h->stream));
    CU(dalloc(&h->barrier, sizeof(unsigned), h->stream));
    CU(cudaMemsetAsync(h->ticket, 0, sizeof(unsigned), h->stream));
    CU(launch_field_tables(h->tables, h->tables + 2 * h->N, h->tables + 2 * h->N + 2 * nodes, c.d, c.Nx, h->nodes,
                           2.0 * M_PI / c.L, h->stream));
    CU(cudaMemsetAsync(h->d_status, 0, sizeof(int), h->stream));
    CU(cudaMemsetAsync(h->d_len, 0, sizeof(int64_t), h->stream));

    rc = install_ic(h, c);
    if (rc) {
        nufi_destroy(h);
        return rc;
    }
    *out = h;
    return NUFI_OK;
}

// Frees every multi-rank resource and returns the handle to single-rank mode.
static void mg_release(nufi_handle *h) {
    cudaStreamSynchronize(h->stream);
    for (int q = 0; q < NUFI_MG_MAX; ++q) {
        if (h->mg_opened[q]) cudaIpcCloseMemHandle(h->mg_peer[q]);
        else if (h->mg_peer[q] && h->mg_peer[q] != h->mg_own) cudaFree(h->mg_peer[q]);
        if (q > 0 && h->mg_part[q]) cudaFree(h->mg_part[q]);
        if (q > 0 && h->mg_fmm[q]) cudaFree(h->mg_fmm[q]);
        if (h->mg_bar[q] && h->mg_bar[q] != h->barrier) cudaFree(h->mg_bar[q]);
        h->mg_opened[q] = false;
        h->mg_peer[q] = nullptr;
        if (q > 0) h->mg_part[q] = nullptr, h->mg_fmm[q] = nullptr;
        h->mg_bar[q] = nullptr;
    }
    if (h->mg_own) cudaFree(h->mg_own);
    if (h->mg_error) cudaFree(h->mg_error);
    h->mg_own = nullptr;
    h->mg_error = nullptr;
    h->mg_world = 1;
    h->mg_rank = 0;
    h->mg_emulated = 0;
    h->mg_steps = 0;
}

int nufi_mg_teardown(nufi_handle *h) {
    CHECK_HANDLE(h);
    mg_release(h);
    CU(cudaGetLastError());
    return NUFI_OK;
}

int nufi_destroy(nufi_handle *h) {
    if (!h) return NUFI_OK;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    for (void *p : {(void *)h->hist, (void *)h->ev_hist, (void *)h->partial, (void *)h->fminmax, (void *)h->blocks,
                    (void *)h->row_last,
                    (void *)h->d_rho, (void *)h->d_E, (void *)h->d_W, (void *)h->d_stats, (void *)h->d_rho_bar,
                    (void *)h->d_status, (void *)h->d_len, (void *)h->run_dev, (void *)h->tables,
                    (void *)h->ticket, (void *)h->barrier, (void *)h->mom_part, (void *)h->d_mom,
                    (void *)h->large_scratch, (void *)h->halo, (void *)h->tile_cnt, (void *)h->block_mm})
        if (p) cudaFreeAsync(p, h->stream);
    mg_release(h);
    for (size_t q = 0; q < h->aev.size(); ++q) cudaEventDestroy(h->aev[q]);
    pinned_put(h->aring_block, h->aring_block_elems);
    cudaStreamSynchronize(h->stream);  // frees complete -> the pool can hand the memory to the next handle
    pinned_put(h->run_host, h->run_elems);
    if (h->own_stream) stream_put(h->device, h->stream);  // idle: synchronised above
    delete h;
    return NUFI_OK;
}

int nufi_sync(nufi_handle *h) {
    CHECK_HANDLE(h);
    CU(cudaStreamSynchronize(h->stream));
    return NUFI_OK;
}

int nufi_rho_bar(nufi_handle *h, double *out) {
    if (!h || !out) return fail(NUFI_ERR_USAGE, "null argument");
    *out = h->rho_bar;
    return NUFI_OK;
}

int64_t nufi_partials_len(nufi_handle *h) { return h ? (int64_t)h->B * h->nodes + 2 * h->B : 0; }

// ---- history --------------------------------------------------------------

int nufi_history_len(nufi_handle *h, int64_t *len) {
    if (!h || !len) return fail(NUFI_ERR_USAGE, "null argument");
    *len = h->len;
    return NUFI_OK;
}

int nufi_load_history(nufi_handle *h, const double *coeffs, int64_t count) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    if (count < 0 || count > h->cap) return fail(NUFI_ERR_USAGE, "history count exceeds the capacity n_max + 1");
    if (count > 0 && !coeffs) return fail(NUFI_ERR_USAGE, "null coefficients");
    if (count > 0) {
        CU(cudaMemcpyAsync(h->hist, coeffs, (size_t)count * h->nodes * sizeof(double), cudaMemcpyDefault, h->stream));
        CU(launch_build_ev_slabs(h->hist, h->ev_hist, h->d, h->N, h->nodes, h->ev_elems, h->K, 0, count, h->f32,
                                 h->stream));
    }
    h->len = count;
    CU(cudaMemcpyAsync(h->d_len, &h->len, sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return NUFI_OK;
}

int nufi_get_history(nufi_handle *h, double *coeffs, int64_t first, int64_t count) {
    CHECK_HANDLE(h);
    if (first < 0 || count < 0 || first + count > h->len)
        return fail(NUFI_ERR_USAGE, "requested rows outside the stored history");
    if (count == 0) return NUFI_OK;
    CU(cudaMemcpyAsync(coeffs, h->hist + (size_t)first * h->nodes, (size_t)count * h->nodes * sizeof(double),
                       cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return NUFI_OK;
}

int nufi_append_coeffs(nufi_handle *h, const double *coeffs) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    if (!coeffs) return fail(NUFI_ERR_USAGE, "null coefficients");
    if (h->len >= h->cap) return fail(NUFI_ERR_USAGE, "history is full (capacity n_max + 1)");
    CU(cudaMemcpyAsync(h->hist + (size_t)h->len * h->nodes, coeffs, (size_t)h->nodes * sizeof(double),
                       cudaMemcpyDefault, h->stream));
    CU(launch_build_ev_slabs(h->hist, h->ev_hist, h->d, h->N, h->nodes, h->ev_elems, h->K, h->len, h->len + 1,
                             h->f32, h->stream));
    h->len += 1;
    CU(cudaStreamSynchronize(h->stream));
    return NUFI_OK;
}

int nufi_truncate_history(nufi_handle *h, int64_t count) {
    if (h) h->spec = -1;
    if (!h) return fail(NUFI_ERR_USAGE, "null handle");
    if (count < 0 || count > h->len) return fail(NUFI_ERR_USAGE, "truncate beyond the stored history");
    h->len = count;
    return NUFI_OK;
}

}  // extern "C"

// ---- internal step pieces -------------------------------------------------

static TraceRhoParams trace_params(nufi_handle *h, int64_t n, int b_lo) {
    TraceRhoParams p{};
    p.N = h->N;
    p.nodes = h->nodes;
    p.Nv = h->Nv;
    p.V = h->V;
    p.node_tiles = h->node_tiles;
    p.vt_rows = h->vt_rows;
    p.passes = h->passes;
    p.vt_lo = b_lo * h->vt_per_block;
    p.B = h->B;
    p.vt_per_block = h->vt_per_block;
    p.n = (int)n;
    p.hx = h->hx;
    p.inv_h = h->inv_h;
    p.vmax = h->cfg.vmax;
    p.hv = h->hv;
    p.vel_to_scaled = h->cfg.tau * h->inv_h;
    p.scaled_to_vel = 1.0 / p.vel_to_scaled;
    p.ev_hist = h->ev_hist;
    p.ev_slab_elems = h->ev_elems;
    p.slabs_per_stage = h->sps;
    p.stages = h->stages;
    p.f0 = h->f0;
    p.partial = h->partial;
    p.fminmax = h->fminmax;
    return p;
}

// CTA width of every d = 1 tail (see launch_field_update); 0 = by size for d >= 2
static int field_threads(const nufi_handle *h) { return h->d == 1 ? h->threads + 32 : 0; }

static FieldParams field_params(nufi_handle *h);

// the step tail: one CTA (field_update_body) or, beyond MAX_FIELD_NODES, the multi-CTA
// sequence of field_large.cu
static cudaError_t enqueue_field(nufi_handle *h, const FieldParams &f_in) {
    if (h->large) return launch_field_large(f_in, h->large_scratch, h->stream);
    static const char *dbg = getenv("NUFI_FIELD_STAMPS");  // debug: phase timestamps of the tail
    if (!dbg) return launch_field_update(f_in, h->stream, field_threads(h));
    FieldParams f = f_in;
    unsigned long long *ts = nullptr, host[10] = {0};
    cudaMalloc(&ts, sizeof host);
    cudaMemsetAsync(ts, 0, sizeof host, h->stream);
    f.tstamps = ts;
    cudaError_t e = launch_field_update(f, h->stream, field_threads(h));
    cudaMemcpyAsync(host, ts, sizeof host, cudaMemcpyDeviceToHost, h->stream);
    cudaStreamSynchronize(h->stream);
    cudaFree(ts);
    if (FILE *fp = fopen(dbg, "a")) {
        for (int k = 1; k < 10; ++k)
            if (host[k]) fprintf(fp, " %d:%.2f", k, (double)(host[k] - host[0]) * 1e-3);
        fprintf(fp, "\n");
        fclose(fp);
    }
    return e;
}

static FieldParams field_params(nufi_handle *h) {
    FieldParams f{};
    f.d = h->d;
    f.N = h->N;
    f.nodes = h->nodes;
    f.B = h->B;
    f.L = h->cfg.L;
    f.inv_h = h->inv_h;
    f.hv_d = h->hv_d;
    f.rho_bar = h->rho_bar;
    f.L_d = h->L_d;
    f.K = h->K;
    f.twc = h->tables;
    f.tws = h->tables + h->N;
    f.fac = h->tables + 2 * h->N;
    f.k2 = h->tables + 2 * h->N + 2 * h->nodes;
    if (h->d == 1) {
        f.gc = f.k2 + h->nodes;
        f.gp = f.gc + h->N;
    }
    f.halo = h->halo;
    f.hist = h->hist;
    f.ev_hist = h->ev_hist;
    f.ev_slab_elems = h->ev_elems;
    f.status = h->d_status;
    f.hist_len = h->d_len;
    f.f32_hist = h->f32;
    return f;
}

static double point_steps(nufi_handle *h, int64_t n, int nblocks) {
    return (double)h->nodes * (double)(h->V / h->B) * nblocks * (double)n;
}

// trace + f0 + per-tile v-sums for blocks [b_lo, b_hi) (no tail)
static int enqueue_trace(nufi_handle *h, int64_t n, int b_lo, int b_hi) {
    const TraceRhoParams p = trace_params(h, n, b_lo);
    const int ctas = (b_hi - b_lo) * h->vt_per_block * h->node_tiles;
    ProfScope ps(h, 0, point_steps(h, n, b_hi - b_lo));
    if (h->gl) {
        TraceRhoParams q = p;
        if (h->d >= 2) q.passes = h->passes * h->ppt;  // one point per thread, same rows
        CU(launch_trace_rho_global(h->d, false, h->pow2, q, h->K, ctas, h->d == 1 ? 32 * h->vt_rows : h->threads,
                                   h->stream));
    } else if (h->d == 1) {
        FieldParams none{};
        CU(launch_trace_rho_1d(p, none, 0, h->ticket, ctas, h->threads + 32, h->stream));
    } else {
        CU(launch_trace_rho(h->d, h->ppt, h->pow2, p, h->K, ctas, h->threads, h->stream));
    }
    return NUFI_OK;
}

// per-tile sums -> block table rows [b_lo, b_hi) of out (B*nodes sums, then B (min, max))
static int enqueue_reduce(nufi_handle *h, int b_lo, int b_hi, double *out) {
    ProfScope ps(h, 1);
    CU(launch_reduce_blocks(h->partial, h->fminmax, out, h->nodes, h->node_tiles, h->vt_per_block, b_lo, b_hi, h->B,
                            h->stream));
    return NUFI_OK;
}

// trace of blocks [b_lo, b_hi) -> block table `out`: d >= 2 in ONE launch (the block reduce
// fused into the trace kernel, same order as reduce_blocks_kernel), d = 1 trace + reduce
static int enqueue_trace_blocks(nufi_handle *h, int64_t n, int b_lo, int b_hi, double *out) {
    static const bool nofuse = getenv("NUFI_NOFUSE_REDUCE") != nullptr;
    if (h->d == 1 || nofuse || !h->tile_cnt) {
        int rc = enqueue_trace(h, n, b_lo, b_hi);
        if (!rc) rc = enqueue_reduce(h, b_lo, b_hi, out);
        return rc;
    }
    TraceRhoParams p = trace_params(h, n, b_lo);
    p.block_out = out;
    p.block_mm = h->block_mm;
    p.tile_cnt = h->tile_cnt;
    p.b_lo = b_lo;
    p.b_hi = b_hi;
    const int ctas = (b_hi - b_lo) * h->vt_per_block * h->node_tiles;
    ProfScope ps(h, 0, point_steps(h, n, b_hi - b_lo));
    if (h->gl) {
        TraceRhoParams q = p;
        q.passes = h->passes * h->ppt;  // one point per thread, same rows
        CU(launch_trace_rho_global(h->d, false, h->pow2, q, h->K, ctas, h->threads, h->stream));
    } else {
        CU(launch_trace_rho(h->d, h->ppt, h->pow2, p, h->K, ctas, h->threads, h->stream));
    }
    return NUFI_OK;
}

// outputs of one step (device pointers, any may be null)
struct StepOut {
    double *rho = nullptr, *E = nullptr, *W = nullptr, *stats = nullptr, *coeffs = nullptr;
    int *status_mirror = nullptr;
};

// A whole single-rank step n: compute_rho (+ the field update tail when full).
// d = 1: one fused launch (the last CTA runs the tail); d = 2, 3: trace ->
// block reduce -> field_update.
static int enqueue_step(nufi_handle *h, int64_t n, bool full, const StepOut &o) {
    h->d_rho_async = false;
    FieldParams f = field_params(h);
    f.slot = n;
    f.rho_out = o.rho;
    f.stats_out = o.stats;
    f.W_out = o.W;
    f.E_out = o.E;
    f.coeffs_out = o.coeffs;
    f.status_mirror = o.status_mirror;
    f.finish_only = full ? 0 : 1;
    static const bool nofuse = getenv("NUFI_NOFUSE") != nullptr;
    if (h->d == 1 && !nofuse && !h->large) {
        f.sums = h->partial;
        f.rows_per_block = h->vt_per_block;
        f.minmax = h->fminmax;
        f.mm_per_block = h->vt_per_block * h->node_tiles;
        const TraceRhoParams p = trace_params(h, n, 0);
        const int ctas = h->B * h->vt_per_block * h->node_tiles;
        ProfScope ps(h, 0, point_steps(h, n, h->B));
        CU(launch_trace_rho_1d(p, f, 1, h->ticket, ctas, h->threads + 32, h->stream));
        return NUFI_OK;
    }
    int rc = enqueue_trace_blocks(h, n, 0, h->B, h->blocks);
    if (rc) return rc;
    f.sums = h->blocks;
    f.rows_per_block = 1;
    f.minmax = h->blocks + (size_t)h->B * h->nodes;
    f.mm_per_block = 1;
    ProfScope ps(h, 2);
    CU(enqueue_field(h, f));
    return NUFI_OK;
}

static int copy_out(nufi_handle *h, void *dst, const void *src, size_t bytes) {
    if (dst) CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->stream));
    return NUFI_OK;
}

static int check_status(nufi_handle *h, const char *what) {
    int st = 0;
    CU(cudaMemcpyAsync(&st, h->d_status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (st == NUFI_ERR_NUMERICAL) {
        CU(cudaMemsetAsync(h->d_status, 0, sizeof(int), h->stream));
        return fail(NUFI_ERR_NUMERICAL, std::string(what) +
                                            ": density is not neutral: nodal mean exceeds 1e-8 max|rho|; "
                                            "subtract the mean before solving");
    }
    return NUFI_OK;
}

static int usage_history(nufi_handle *h, int64_t n) {
    char buf[160];
    snprintf(buf, sizeof buf, "psi_tilde at step %lld needs fields 0..%lld; history holds %lld", (long long)n,
             (long long)(n - 1), (long long)h->len);  // flow.py:55-62
    return fail(NUFI_ERR_USAGE, buf);
}

static int copy_step_outputs(nufi_handle *h, double *rho_out, double *E_out, double *W_out, double *stats3) {
    int rc = copy_out(h, rho_out, h->d_rho, h->nodes * sizeof(double));
    if (!rc) rc = copy_out(h, E_out, h->d_E, (size_t)h->nodes * h->d * sizeof(double));
    if (!rc) rc = copy_out(h, W_out, h->d_W, sizeof(double));
    if (!rc) rc = copy_out(h, stats3, h->d_stats, 3 * sizeof(double));
    if (rc) return rc;
    CU(cudaStreamSynchronize(h->stream));
    return NUFI_OK;
}

extern "C" {

// installed fields are a test hook of the point-level flow (flow.py:44-82); the fused
// density / run kernels trace stored splines only
static int refuse_installed(nufi_handle *h) {
    if (h->n_ovr > 0)
        return fail(NUFI_ERR_USAGE, "installed (non-spline) fields are honoured by the point-level trace only; "
                                    "clear them before compute_rho / run / step");
    return NUFI_OK;
}

// the dense override table (4 doubles per step) covers `step`; a step far beyond anything the
// history can hold is a usage error, not a host allocation that would throw through the C-ABI
static int ovr_cover(nufi_handle *h, int64_t step) {
    if (step < 0) return fail(NUFI_ERR_USAGE, "step index must be >= 0");
    if (step >= std::max<int64_t>(h->cap, (int64_t)1 << 20))
        return fail(NUFI_ERR_USAGE, "step index beyond the history's reach (max(capacity, 2^20))");
    if ((size_t)(4 * (step + 1)) > h->ovr.size()) h->ovr.resize(4 * (size_t)(step + 1), 0.0);
    return NUFI_OK;
}

int nufi_set_uniform_field(nufi_handle *h, int64_t step, const double *E0) {
    CHECK_HANDLE(h);
    if (int rc = ovr_cover(h, step)) return rc;
    const bool was = h->ovr[4 * step] != 0.0;
    h->ovr_spline.erase(step);
    if (E0) {
        h->ovr[4 * step] = 1.0;
        for (int a = 0; a < 3; ++a) h->ovr[4 * step + 1 + a] = a < h->d ? E0[a] : 0.0;
    } else {
        for (int a = 0; a < 4; ++a) h->ovr[4 * step + a] = 0.0;
    }
    h->n_ovr += (E0 ? 1 : 0) - (was ? 1 : 0);
    return NUFI_OK;
}

int nufi_set_spline_field(nufi_handle *h, int64_t step, const double *coeffs) {
    CHECK_HANDLE(h);
    if (int rc = ovr_cover(h, step)) return rc;
    const bool was = h->ovr[4 * step] != 0.0;
    for (int a = 0; a < 4; ++a) h->ovr[4 * step + a] = 0.0;
    h->ovr_spline.erase(step);
    if (coeffs) {
        std::vector<double> c((size_t)h->nodes);
        if (is_device_ptr(coeffs)) {
            CU(cudaMemcpyAsync(c.data(), coeffs, c.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
            CU(cudaStreamSynchronize(h->stream));
        } else {
            std::copy(coeffs, coeffs + c.size(), c.begin());
        }
        h->ovr_spline[step] = std::move(c);
        h->ovr[4 * step] = 2.0;
    }
    h->n_ovr += (coeffs ? 1 : 0) - (was ? 1 : 0);
    return NUFI_OK;
}

int nufi_clear_fields(nufi_handle *h) {
    CHECK_HANDLE(h);
    h->ovr.clear();
    h->ovr_spline.clear();
    h->n_ovr = 0;
    return NUFI_OK;
}

int nufi_rho_partials(nufi_handle *h, int64_t n, double *partials, int64_t *evals) {
    CHECK_HANDLE(h);
    if (int rc = refuse_installed(h)) return rc;
    if (n < 0) return fail(NUFI_ERR_USAGE, "step index must be >= 0");
    if (n > 0 && h->len < n) return usage_history(h, n);
    if (!is_device_ptr(partials)) return fail(NUFI_ERR_USAGE, "partials must be a device buffer");
    CU(cudaMemsetAsync(partials, 0, nufi_partials_len(h) * sizeof(double), h->stream));
    int rc = enqueue_trace_blocks(h, n, h->b_lo, h->b_hi, partials);
    if (rc) return rc;
    if (evals) *evals += (int64_t)point_steps(h, n, h->b_hi - h->b_lo);
    return NUFI_OK;
}

int nufi_rho_finish(nufi_handle *h, const double *partials, double *rho_out, double *stats3) {
    CHECK_HANDLE(h);
    h->d_rho_async = false;
    if (!is_device_ptr(partials)) return fail(NUFI_ERR_USAGE, "partials must be a device buffer");
    FieldParams f = field_params(h);
    f.sums = partials;
    f.rows_per_block = 1;
    f.minmax = partials + (size_t)h->B * h->nodes;
    f.mm_per_block = 1;
    f.rho_out = h->d_rho;
    f.stats_out = h->d_stats;
    f.finish_only = 1;
    {
        ProfScope ps(h, 2);
        CU(enqueue_field(h, f));
    }
    return copy_step_outputs(h, rho_out, nullptr, nullptr, stats3);
}

int nufi_rho(nufi_handle *h, int64_t n, double *rho_out, double *stats3, int64_t *evals) {
    CHECK_HANDLE(h);
    if (int rc = refuse_installed(h)) return rc;
    if (n < 0) return fail(NUFI_ERR_USAGE, "step index must be >= 0");
    if (n > 0 && h->len < n) return usage_history(h, n);
    StepOut o;
    o.rho = h->d_rho;
    o.stats = h->d_stats;
    int rc = enqueue_step(h, n, false, o);
    if (rc) return rc;
    if (evals) *evals += (int64_t)point_steps(h, n, h->B);
    return copy_step_outputs(h, rho_out, nullptr, nullptr, stats3);
}

int nufi_field_update(nufi_handle *h, const double *rho, double *W_out, double *E_out, double *coeffs_out) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    h->d_rho_async = false;
    if (!rho) return fail(NUFI_ERR_USAGE, "null rho");
    if (h->len >= h->cap) return fail(NUFI_ERR_USAGE, "history is full (capacity n_max + 1)");
    CU(cudaMemcpyAsync(h->d_rho, rho, h->nodes * sizeof(double), cudaMemcpyDefault, h->stream));
    FieldParams f = field_params(h);
    f.rho_in = h->d_rho;
    f.slot = h->len;
    f.W_out = h->d_W;
    f.E_out = h->d_E;
    {
        ProfScope ps(h, 2);
        CU(enqueue_field(h, f));
    }
    int rc = check_status(h, "solve_poisson");
    if (rc) return rc;
    h->len += 1;
    rc = copy_out(h, coeffs_out, h->hist + (size_t)(h->len - 1) * h->nodes, h->nodes * sizeof(double));
    if (rc) return rc;
    return copy_step_outputs(h, nullptr, E_out, W_out, nullptr);
}

// ---- stream-ordered drop-in calls: outputs land in a pinned ring entry, no host sync ----

// entry layout: [rho nodes | stats 3 | W 1 | status (int) 1 | pad 1 | E nodes*d | coeffs nodes]
static size_t aslot_off_stats(const nufi_handle *h) { return (size_t)h->nodes; }
static size_t aslot_off_W(const nufi_handle *h) { return (size_t)h->nodes + 3; }
static size_t aslot_off_status(const nufi_handle *h) { return (size_t)h->nodes + 4; }
static size_t aslot_off_E(const nufi_handle *h) { return (size_t)h->nodes + 6; }
static size_t aslot_off_C(const nufi_handle *h) { return (size_t)h->nodes * (1 + h->d) + 6; }

int nufi_async_slots(nufi_handle *h, int slots) {
    CHECK_HANDLE(h);
    if (slots < 1 || slots > 4096) return fail(NUFI_ERR_USAGE, "slots must be 1..4096");
    CU(cudaStreamSynchronize(h->stream));
    for (size_t q = 0; q < h->aev.size(); ++q) cudaEventDestroy(h->aev[q]);
    pinned_put(h->aring_block, h->aring_block_elems);
    h->aring_block = nullptr;
    h->aring.assign(slots, nullptr);
    h->aev.assign(slots, nullptr);
    h->aslot_elems = (size_t)h->nodes * (2 + h->d) + 6;
    h->aring_block_elems = (size_t)slots * h->aslot_elems;
    CU(pinned_get(&h->aring_block, h->aring_block_elems));
    for (int q = 0; q < slots; ++q) {
        h->aring[q] = h->aring_block + (size_t)q * h->aslot_elems;
        CU(cudaEventCreateWithFlags(&h->aev[q], cudaEventDisableTiming));
    }
    return NUFI_OK;
}

int nufi_async_ring(nufi_handle *h, double **base, int64_t *slot_elems) {
    CHECK_HANDLE(h);
    if (!base || !slot_elems) return fail(NUFI_ERR_USAGE, "null argument");
    *base = h->aring_block;
    *slot_elems = (int64_t)h->aslot_elems;
    return NUFI_OK;
}

static int aslot_check(nufi_handle *h, int slot) {
    if (slot < 0 || slot >= (int)h->aring.size()) return fail(NUFI_ERR_USAGE, "async slot out of range");
    return NUFI_OK;
}

int nufi_rho_async(nufi_handle *h, int64_t n, int slot, int64_t *evals, int *speculative) {
    CHECK_HANDLE(h);
    if (int rc = refuse_installed(h)) return rc;
    if (int rc = aslot_check(h, slot)) return rc;
    if (n < 0) return fail(NUFI_ERR_USAGE, "step index must be >= 0");
    if (n > 0 && h->len < n) return usage_history(h, n);
    double *e = h->aring[slot];
    int *st_mirror = reinterpret_cast<int *>(e + aslot_off_status(h));
    const bool spec = n == h->len && n < h->cap && !h->large;
    StepOut o;
    if (spec) {
        // the loop's next step: run the whole step (compute_rho + the tail into slot n, NOT
        // yet committed to the history length) in one launch, every output written straight
        // into the pinned entry; advance() of this density then only commits
        o.rho = e;
        o.stats = e + aslot_off_stats(h);
        o.W = e + aslot_off_W(h);
        o.E = e + aslot_off_E(h);
        o.coeffs = e + aslot_off_C(h);
        o.status_mirror = st_mirror;
        int rc = enqueue_step(h, n, true, o);
        if (rc) return rc;
        if (h->large) CU(cudaMemcpyAsync(st_mirror, h->d_status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        h->spec = n;
    } else {
        o.rho = h->d_rho;
        o.stats = h->d_stats;
        int rc = enqueue_step(h, n, false, o);
        if (rc) return rc;
        CU(cudaMemcpyAsync(e, h->d_rho, h->nodes * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CU(cudaMemcpyAsync(e + aslot_off_stats(h), h->d_stats, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream));
        CU(cudaMemcpyAsync(st_mirror, h->d_status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        h->d_rho_async = true;
    }
    CU(cudaEventRecord(h->aev[slot], h->stream));
    if (evals) *evals += (int64_t)point_steps(h, n, h->B);
    if (speculative) *speculative = spec ? 1 : 0;
    return NUFI_OK;
}

int nufi_commit_async(nufi_handle *h, int64_t n) {
    CHECK_HANDLE(h);
    if (h->spec != n || h->len != n) return fail(NUFI_ERR_USAGE, "no speculative tail of this step to commit");
    h->spec = -1;
    h->len += 1;  // provisional like nufi_field_update_async
    return NUFI_OK;
}

int nufi_field_update_async(nufi_handle *h, const double *rho, int slot) {
    CHECK_HANDLE(h);
    if (int rc = aslot_check(h, slot)) return rc;
    if (h->len >= h->cap) return fail(NUFI_ERR_USAGE, "history is full (capacity n_max + 1)");
    if (!rho && !h->d_rho_async)
        return fail(NUFI_ERR_USAGE, "no device density: the last call that wrote one was not nufi_rho_async");
    h->spec = -1;
    if (rho) CU(cudaMemcpyAsync(h->d_rho, rho, h->nodes * sizeof(double), cudaMemcpyDefault, h->stream));
    h->d_rho_async = false;
    double *e = h->aring[slot];
    FieldParams f = field_params(h);
    f.rho_in = h->d_rho;  // NULL rho: the density the last nufi_rho_async left on the device
    f.slot = h->len;
    f.W_out = e + aslot_off_W(h);  // written straight into the pinned entry
    f.E_out = e + aslot_off_E(h);
    f.coeffs_out = e + aslot_off_C(h);
    f.status_mirror = reinterpret_cast<int *>(e + aslot_off_status(h));
    {
        ProfScope ps(h, 2);
        CU(enqueue_field(h, f));
    }
    if (h->large) CU(cudaMemcpyAsync(f.status_mirror, h->d_status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaEventRecord(h->aev[slot], h->stream));
    h->len += 1;  // provisional; nufi_async_wait / nufi_check_status reconcile a failed step
    return NUFI_OK;
}

int nufi_async_wait(nufi_handle *h, int slot, double **entry) {
    CHECK_HANDLE(h);
    if (int rc = aslot_check(h, slot)) return rc;
    CU(cudaEventSynchronize(h->aev[slot]));
    int st = 0;
    memcpy(&st, h->aring[slot] + aslot_off_status(h), sizeof(int));  // the status as of this entry
    if (st != 0) {
        int rc = nufi_check_status(h);  // reconciles len, clears the flag, sets the message
        if (rc) return rc;
        // the failure was reported through an earlier entry: this entry's work was skipped
        return fail(st, "step skipped: an earlier enqueued step failed (density not neutral)");
    }
    if (entry) *entry = h->aring[slot];
    return NUFI_OK;
}

int nufi_step(nufi_handle *h, int64_t n, double *rho_out, double *E_out, double *W_out, double *stats3,
              int64_t *evals) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    if (int rc = refuse_installed(h)) return rc;
    if (n != h->len) {
        char buf[160];
        snprintf(buf, sizeof buf, "step %lld requires a history of exactly %lld fields, have %lld", (long long)n,
                 (long long)n, (long long)h->len);
        return fail(NUFI_ERR_USAGE, buf);
    }
    if (n >= h->cap) return fail(NUFI_ERR_USAGE, "history is full (capacity n_max + 1)");
    StepOut o;
    o.rho = h->d_rho;
    o.E = h->d_E;
    o.W = h->d_W;
    o.stats = h->d_stats;
    int rc = enqueue_step(h, n, true, o);
    if (!rc) rc = check_status(h, "solve_poisson");
    if (rc) return rc;
    h->len += 1;
    if (evals) *evals += (int64_t)point_steps(h, n, h->B);
    return copy_step_outputs(h, rho_out, E_out, W_out, stats3);
}

int nufi_step_finish(nufi_handle *h, int64_t n, const double *partials, double *rho_out, double *E_out,
                     double *W_out, double *stats3) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    h->d_rho_async = false;
    if (n != h->len) return fail(NUFI_ERR_USAGE, "step_finish requires len == n");
    if (n >= h->cap) return fail(NUFI_ERR_USAGE, "history is full (capacity n_max + 1)");
    if (!is_device_ptr(partials)) return fail(NUFI_ERR_USAGE, "partials must be a device buffer");
    FieldParams f = field_params(h);
    f.sums = partials;
    f.rows_per_block = 1;
    f.minmax = partials + (size_t)h->B * h->nodes;
    f.mm_per_block = 1;
    f.slot = n;
    f.rho_out = h->d_rho;
    f.stats_out = h->d_stats;
    f.W_out = h->d_W;
    f.E_out = h->d_E;
    {
        ProfScope ps(h, 2);
        CU(enqueue_field(h, f));
    }
    int rc = check_status(h, "solve_poisson");
    if (rc) return rc;
    h->len += 1;
    return copy_step_outputs(h, rho_out, E_out, W_out, stats3);
}

int nufi_step_finish_async(nufi_handle *h, int64_t n, const double *partials, double *rho_out, double *E_out,
                           double *W_out, double *stats3) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    h->d_rho_async = false;
    if (n != h->len) return fail(NUFI_ERR_USAGE, "step_finish requires len == n");
    if (n >= h->cap) return fail(NUFI_ERR_USAGE, "history is full (capacity n_max + 1)");
    for (const void *q : {(const void *)partials, (const void *)rho_out, (const void *)E_out, (const void *)W_out,
                          (const void *)stats3})
        if (q && !is_device_ptr(q)) return fail(NUFI_ERR_USAGE, "async step outputs must be device buffers");
    if (!partials) return fail(NUFI_ERR_USAGE, "null partials");
    FieldParams f = field_params(h);
    f.sums = partials;
    f.rows_per_block = 1;
    f.minmax = partials + (size_t)h->B * h->nodes;
    f.mm_per_block = 1;
    f.slot = n;
    f.rho_out = rho_out;
    f.stats_out = stats3;
    f.W_out = W_out;
    f.E_out = E_out;
    {
        ProfScope ps(h, 2);
        CU(enqueue_field(h, f));
    }
    h->len += 1;  // provisional; nufi_check_status() reconciles with the device length
    return NUFI_OK;
}

int nufi_check_status(nufi_handle *h) {
    CHECK_HANDLE(h);
    int st = 0;
    int64_t dlen = 0;
    CU(cudaMemcpyAsync(&st, h->d_status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaMemcpyAsync(&dlen, h->d_len, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (st == NUFI_ERR_NUMERICAL) {
        h->len = dlen;  // the fields actually appended before the failing step
        CU(cudaMemsetAsync(h->d_status, 0, sizeof(int), h->stream));
        return fail(NUFI_ERR_NUMERICAL, "solve_poisson: density is not neutral: nodal mean exceeds 1e-8 max|rho|");
    }
    if (st == NUFI_ERR_COMM) {
        h->len = dlen;
        CU(cudaMemsetAsync(h->d_status, 0, sizeof(int), h->stream));
        return fail(NUFI_ERR_COMM, "multi-rank step: a peer rank did not arrive within 4 s (watchdog)");
    }
    return NUFI_OK;
}

// ---- multi-rank d = 1 runs with the exchange fused into the persistent kernel ----

static size_t mg_xstride(const nufi_handle *h) { return (size_t)h->B * h->nodes + 2 * (size_t)h->B; }
static size_t mg_bytes(const nufi_handle *h) {
    return 2 * mg_xstride(h) * sizeof(double) + 256 + NUFI_MG_MAX * sizeof(unsigned);
}
static double *mg_table(void *buf) { return reinterpret_cast<double *>(buf); }
static unsigned *mg_flags(const nufi_handle *h, void *buf) {
    return reinterpret_cast<unsigned *>(reinterpret_cast<char *>(buf) + 2 * mg_xstride(h) * sizeof(double) + 128);
}

int nufi_mg_setup(nufi_handle *h, int world, int rank, int emulate, void *ipc_handle_out) {
    CHECK_HANDLE(h);
    if (h->large)
        return fail(NUFI_ERR_USAGE, "the fused multi-rank exchange needs the single-CTA step tail (Nx^d <= 4096)");
    if (world < 2 || world > NUFI_MG_MAX || rank < 0 || rank >= world)
        return fail(NUFI_ERR_USAGE, "world must be 2..8 and 0 <= rank < world");
    if (h->B % world) return fail(NUFI_ERR_USAGE, "v_blocks must be a multiple of the rank count");
    if (h->mg_own) return fail(NUFI_ERR_USAGE, "multi-rank mode already set up");
    if (emulate) {
        if (h->b_lo != 0 || h->b_hi != h->B)
            return fail(NUFI_ERR_USAGE, "an emulated run covers all velocity blocks");
    } else if (h->b_lo != rank * (h->B / world) || h->b_hi != (rank + 1) * (h->B / world)) {
        return fail(NUFI_ERR_USAGE, "handle block range does not match this rank's share");
    }
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaMalloc(&h->mg_own, mg_bytes(h)));  // plain cudaMalloc: IPC-exportable
    CU(cudaMemset(h->mg_own, 0, mg_bytes(h)));
    CU(cudaMalloc(&h->mg_error, sizeof(int)));
    CU(cudaMemset(h->mg_error, 0, sizeof(int)));
    h->mg_world = world;
    h->mg_rank = emulate ? 0 : rank;
    h->mg_emulated = emulate ? 1 : 0;
    h->mg_steps = 0;
    h->mg_peer[h->mg_rank] = h->mg_own;
    if (emulate) {
        const size_t pbytes = 2 * (size_t)h->vt_total * h->node_tiles * 32 * sizeof(double);
        const size_t fbytes = 2 * (size_t)h->vt_total * h->node_tiles * 2 * sizeof(double);
        h->mg_part[0] = h->partial;
        h->mg_fmm[0] = h->fminmax;
        for (int q = 0; q < world; ++q) {
            if (q > 0) {
                CU(cudaMalloc(&h->mg_peer[q], mg_bytes(h)));
                CU(cudaMemset(h->mg_peer[q], 0, mg_bytes(h)));
                CU(cudaMalloc(&h->mg_part[q], pbytes));
                CU(cudaMalloc(&h->mg_fmm[q], fbytes));
            }
            CU(cudaMalloc(&h->mg_bar[q], sizeof(unsigned)));
        }
    } else if (ipc_handle_out) {
        cudaIpcMemHandle_t ipc;
        CU(cudaIpcGetMemHandle(&ipc, h->mg_own));
        memcpy(ipc_handle_out, &ipc, sizeof ipc);
    }
    return NUFI_OK;
}

int nufi_mg_connect(nufi_handle *h, const void *ipc_handles) {
    CHECK_HANDLE(h);
    if (!h->mg_own || h->mg_emulated) return fail(NUFI_ERR_USAGE, "call nufi_mg_setup (real mode) first");
    if (!ipc_handles) return fail(NUFI_ERR_USAGE, "null handles");
    for (int q = 0; q < h->mg_world; ++q) {
        if (q == h->mg_rank) continue;
        cudaIpcMemHandle_t ipc;
        memcpy(&ipc, reinterpret_cast<const char *>(ipc_handles) + q * sizeof(cudaIpcMemHandle_t), sizeof ipc);
        cudaError_t e = cudaIpcOpenMemHandle(&h->mg_peer[q], ipc, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(NUFI_ERR_COMM, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
        h->mg_opened[q] = true;
    }
    return NUFI_OK;
}

int nufi_mg_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

// d >= 2 multi-rank step with the exchange fused into the block reduce (no NCCL):
// trace this rank's blocks -> reduce_exchange (block sums stored into every rank's table
// over peer memory + arrival counters) -> field update waiting on the counters.  Emulated
// mode (one GPU): all blocks traced, then one reduce_exchange per virtual rank (each
// writing every virtual rank's table), then rank 0's field update -- the same kernels and
// the same table contents as a real run.  Stream-ordered, device outputs, no host sync;
// nufi_check_status reports a peer that never arrived (NUFI_ERR_COMM).
int nufi_mg_step_async(nufi_handle *h, int64_t n, double *rho_out, double *E_out, double *W_out, double *stats3) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    h->d_rho_async = false;
    if (!h->mg_own || h->d == 1) return fail(NUFI_ERR_USAGE, "call nufi_mg_setup on a d >= 2 handle first");
    if (!h->mg_emulated) {
        for (int q = 0; q < h->mg_world; ++q)
            if (!h->mg_peer[q]) return fail(NUFI_ERR_USAGE, "call nufi_mg_connect first");
    }
    if (int rc = refuse_installed(h)) return rc;
    if (n != h->len) return fail(NUFI_ERR_USAGE, "mg_step requires len == n");
    if (n >= h->cap) return fail(NUFI_ERR_USAGE, "history is full (capacity n_max + 1)");
    for (const void *q : {(const void *)rho_out, (const void *)E_out, (const void *)W_out, (const void *)stats3})
        if (q && !is_device_ptr(q)) return fail(NUFI_ERR_USAGE, "async step outputs must be device buffers");
    const int G = h->mg_world, nb = h->B / G;
    const size_t xoff = (size_t)(h->mg_steps & 1u) * mg_xstride(h);
    MgExchange x{};
    x.G = G;
    for (int q = 0; q < G; ++q) {
        x.tab[q] = mg_table(h->mg_peer[q]) + xoff;
        x.flags[q] = mg_flags(h, h->mg_peer[q]);
    }
    int rc = enqueue_trace(h, n, h->b_lo, h->b_hi);
    if (rc) return rc;
    int ctas = -1;
    {
        ProfScope ps(h, 1);
        for (int r = 0; r < G; ++r) {
            if (!h->mg_emulated && r != h->mg_rank) continue;
            x.src = r;
            ctas = launch_reduce_exchange(h->partial, h->fminmax, h->nodes, h->node_tiles, h->vt_per_block, r * nb,
                                          (r + 1) * nb, h->B, x, h->stream);
            if (ctas < 0) return fail(NUFI_ERR_CUDA, "reduce_exchange launch failed");
        }
    }
    FieldParams f = field_params(h);
    f.sums = x.tab[h->mg_rank];
    f.rows_per_block = 1;
    f.minmax = f.sums + (size_t)h->B * h->nodes;
    f.mm_per_block = 1;
    f.slot = n;
    f.rho_out = rho_out;
    f.stats_out = stats3;
    f.W_out = W_out;
    f.E_out = E_out;
    f.wait_flags = x.flags[h->mg_rank];
    f.wait_G = G;
    f.wait_target = (h->mg_steps + 1u) * (unsigned)ctas;  // every rank launches the same CTA count
    f.wait_error = h->mg_error;
    {
        ProfScope ps(h, 2);
        CU(enqueue_field(h, f));
    }
    h->mg_steps += 1;
    h->len += 1;  // provisional; nufi_check_status() reconciles with the device length
    return NUFI_OK;
}

int nufi_run(nufi_handle *h, int64_t n_last, double *rho_hist, double *E_hist, double *W_hist, double *stats_hist,
             int64_t *evals) {
    if (h) h->spec = -1;
    CHECK_HANDLE(h);
    h->d_rho_async = false;
    if (int rc = refuse_installed(h)) return rc;
    const int64_t first = h->len;
    if (n_last < first) return NUFI_OK;
    if (n_last >= h->cap) return fail(NUFI_ERR_USAGE, "n_last exceeds n_max");
    const int64_t steps = n_last - first + 1;
    const size_t nodes = h->nodes, d = h->d;
    const size_t per_step = nodes + nodes * d + 1 + 3;  // rho, E, W, stats
    // device output rows: caller's device buffers directly, else internal + pinned staging
    const bool dev[4] = {is_device_ptr(rho_hist), is_device_ptr(E_hist), is_device_ptr(W_hist),
                         is_device_ptr(stats_hist)};
    const size_t need = (size_t)steps * per_step;
    if (need > h->run_elems) {
        if (h->run_dev) cudaFreeAsync(h->run_dev, h->stream);
        pinned_put(h->run_host, h->run_elems);
        h->run_dev = nullptr;
        h->run_host = nullptr;
        CU(dalloc(&h->run_dev, need * sizeof(double), h->stream));
        CU(pinned_get(&h->run_host, need));
        h->run_elems = need;
    }
    double *base_dev[4] = {h->run_dev, h->run_dev + steps * nodes, h->run_dev + steps * (nodes + nodes * d),
                           h->run_dev + steps * (nodes + nodes * d + 1)};
    double *base_host[4] = {h->run_host, h->run_host + steps * nodes, h->run_host + steps * (nodes + nodes * d),
                            h->run_host + steps * (nodes + nodes * d + 1)};
    double *user[4] = {rho_hist, E_hist, W_hist, stats_hist};
    const size_t width[4] = {nodes, nodes * d, 1, 3};
    for (int q = 0; q < 4; ++q)
        if (dev[q]) base_dev[q] = user[q];

    static const bool nopersist = getenv("NUFI_NOPERSIST") != nullptr;
    bool persist = h->d == 1 && !nopersist && !h->large;
    if (h->mg_world > 1 && !persist)
        return fail(NUFI_ERR_USAGE, "a connected multi-rank handle runs only the persistent d = 1 kernel");
    if (persist) {
        // whole run in one cooperative launch (run_1d.cu)
        Run1DParams P{};
        P.tp = trace_params(h, 0, 0);
        P.fp = field_params(h);
        P.fp.sums = h->partial;
        P.fp.rows_per_block = h->vt_per_block;
        P.fp.minmax = h->fminmax;
        P.fp.mm_per_block = h->vt_per_block * h->node_tiles;
        P.n_first = (int)first;
        P.n_last = (int)n_last;
        P.rho_hist = base_dev[0];
        P.E_hist = base_dev[1];
        P.W_hist = base_dev[2];
        P.stats_hist = base_dev[3];
        P.barrier = h->barrier;
        P.tiles = h->B * h->vt_per_block * h->node_tiles;
        P.blocks = h->blocks;
        // two-level combine when every CTA re-reading all tile partials would dominate the tail
        P.two_level = (int64_t)h->vt_total * h->nodes > 16384 ? 1 : 0;
        if (const char *e = getenv("NUFI_TWO_LEVEL")) P.two_level = atoi(e);
        // next-step ring prefetch: every ring stage must hold the tail workspace
        P.prefetch = h->stages >= 2 &&
                     (int64_t)h->sps * h->ev_elems >= (int64_t)field_smem_doubles(h->nodes, h->N, true) &&
                     !getenv("NUFI_NOPREFETCH");
        // split: with one tile per CTA and SMs to spare, helper CTAs trace every tile's last row
        // so no SM holds more than vt_rows - 1 tracing warps (shared-memory contention of the
        // gathers; profiles/r02_d1_chain_floor.txt).  Bit-identical (the tail completes each
        // tile's sequential sum).  Single rank only; NUFI_D1_SPLIT=0 turns it off.
        P.split_helpers = 0;
        if (h->mg_world <= 1 && h->vt_rows >= 4 && !P.two_level && !(getenv("NUFI_D1_SPLIT") && atoi(getenv("NUFI_D1_SPLIT")) == 0)) {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
            const int helpers = (P.tiles + h->vt_rows - 2) / (h->vt_rows - 1);
            if (P.tiles + helpers <= sms) {
                if (!h->row_last) CU(dalloc(&h->row_last, 2 * (size_t)P.tiles * 34 * sizeof(double), h->stream));
                P.split_helpers = helpers;
                P.row_last = h->row_last;
                P.row_last_mm = h->row_last + 2 * (size_t)P.tiles * 32;
            }
        }
        if (h->mg_world > 1) {
            if (!h->mg_emulated)
                for (int q = 0; q < h->mg_world; ++q)
                    if (!h->mg_peer[q]) return fail(NUFI_ERR_USAGE, "multi-rank run: call nufi_mg_connect first");
            P.two_level = 0;
            P.mg_ranks = h->mg_world;
            P.mg_emulated = h->mg_emulated;
            P.mg_rank = h->mg_rank;
            P.mg_base = h->mg_steps;
            P.mg_error = h->mg_error;
            for (int q = 0; q < h->mg_world; ++q) {
                P.mg_xtab[q] = mg_table(h->mg_peer[q]);
                P.mg_flags[q] = mg_flags(h, h->mg_peer[q]);
                P.mg_partial[q] = h->mg_part[q];
                P.mg_fminmax[q] = h->mg_fmm[q];
                P.mg_barrier[q] = h->mg_bar[q];
                if (h->mg_emulated && h->mg_bar[q]) CU(cudaMemsetAsync(h->mg_bar[q], 0, sizeof(unsigned), h->stream));
            }
        }
        static const char *stamp_path = getenv("NUFI_STAMPS");  // debug: per-step phase timestamps
        unsigned long long *stamps = nullptr;
        if (stamp_path) CU(cudaMalloc(&stamps, (3 * steps + 10 + 6 * 1024) * sizeof(unsigned long long)));
        if (stamps) CU(cudaMemsetAsync(stamps, 0, (3 * steps + 10 + 6 * 1024) * sizeof(unsigned long long), h->stream));
        P.stamps = stamps;
        CU(cudaMemsetAsync(h->barrier, 0, sizeof(unsigned), h->stream));
        {
            const double ps = (double)h->nodes * h->V * (double)((n_last * (n_last + 1) - (first - 1) * first) / 2);
            ProfScope prof(h, 0, ps);
            int grid = 0;
            const cudaError_t le = launch_run_1d(P, h->threads + 32, h->device, h->stream, &grid);
            if (le == cudaErrorCooperativeLaunchTooLarge && h->mg_world == 1) {
                // the device cannot host the whole grid at once (e.g. shared with other
                // work): fall back to one launch per step, same results
                cudaGetLastError();
                persist = false;
            } else {
                CU(le);
            }
        }
        if (stamps) {
            std::vector<unsigned long long> st(3 * steps + 10 + 6 * 1024);
            CU(cudaMemcpyAsync(st.data(), stamps, st.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               h->stream));
            CU(cudaStreamSynchronize(h->stream));
            cudaFree(stamps);
            if (FILE *f = fopen(stamp_path, "w")) {
                for (int64_t i = 0; i < steps; ++i)
                    fprintf(f, "%lld %llu %llu %llu\n", (long long)(first + i), st[3 * i], st[3 * i + 1], st[3 * i + 2]);
                fprintf(f, "# tail phases (last step):");
                for (int k = 0; k < 9; ++k) fprintf(f, " %llu", st[3 * steps + k]);
                fprintf(f, "\n");
                fprintf(f, "# wait/total cycles per cta (last step):");
                for (int c = 0; c < 1024; ++c)
                    if (st[3 * steps + 10 + 4 * 1024 + 2 * c + 1])
                        fprintf(f, " %llu/%llu", st[3 * steps + 10 + 4 * 1024 + 2 * c], st[3 * steps + 10 + 4 * 1024 + 2 * c + 1]);
                fprintf(f, "\n");
                for (int q = 0; q < 4; ++q) {
                    fprintf(f, "# cta trace end, step %d:", 400 * (q + 1));
                    for (int c = 0; c < 1024; ++c)
                        if (st[3 * steps + 10 + q * 1024 + c]) fprintf(f, " %llu", st[3 * steps + 10 + q * 1024 + c]);
                    fprintf(f, "\n");
                }
                fclose(f);
            }
        }
        for (int q = 0; q < 4; ++q)
            if (persist && user[q] && !dev[q])
                CU(cudaMemcpyAsync(base_host[q], base_dev[q], steps * width[q] * sizeof(double),
                                   cudaMemcpyDeviceToHost, h->stream));
    }
    if (!persist) {
    for (int64_t n = first; n <= n_last; ++n) {
        const int64_t row = n - first;
        StepOut o;
        o.rho = base_dev[0] + row * width[0];
        o.E = base_dev[1] + row * width[1];
        o.W = base_dev[2] + row * width[2];
        o.stats = base_dev[3] + row * width[3];
        int rc = enqueue_step(h, n, true, o);
        if (rc) return rc;
        // per-step device -> pinned host copies of host-bound outputs (async)
        for (int q = 0; q < 4; ++q)
            if (user[q] && !dev[q])
                CU(cudaMemcpyAsync(base_host[q] + row * width[q], base_dev[q] + row * width[q],
                                   width[q] * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    }
    }
    int rc = check_status(h, "solve_poisson");  // synchronises
    if (rc) return rc;
    if (h->mg_world > 1 && persist) {
        int err = 0;
        CU(cudaMemcpy(&err, h->mg_error, sizeof(int), cudaMemcpyDeviceToHost));
        if (err) return fail(NUFI_ERR_COMM, "multi-rank run: a peer rank did not arrive within 4 s (watchdog)");
        h->mg_steps += (unsigned)steps;  // every rank runs the same sequence: identical bases
    }
    h->len = n_last + 1;
    for (int q = 0; q < 4; ++q)
        if (user[q] && !dev[q]) memcpy(user[q], base_host[q], steps * width[q] * sizeof(double));
    if (evals) *evals += (int64_t)h->nodes * h->V * ((n_last * (n_last + 1) - (first - 1) * first) / 2);
    return NUFI_OK;
}

int nufi_profiling(nufi_handle *h, int enable) {
    CHECK_HANDLE(h);
    CU(cudaStreamSynchronize(h->stream));
    for (auto &p : h->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    h->pending.clear();
    for (double &v : h->prof) v = 0;
    h->profiling = enable != 0;
    return NUFI_OK;
}

int nufi_profiling_read(nufi_handle *h, double *out8) {
    CHECK_HANDLE(h);
    CU(cudaStreamSynchronize(h->stream));
    for (auto &p : h->pending) {
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, p.a, p.b));
        h->prof[2 * p.kind] += ms;
        h->prof[2 * p.kind + 1] += 1;
        if (p.kind == 0) h->prof[6] += p.point_steps;
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    h->pending.clear();
    for (int i = 0; i < 8; ++i) out8[i] = h->prof[i];
    return NUFI_OK;
}

int nufi_trace(nufi_handle *h, int64_t n, double *X, double *V, int64_t M, int half_kick, int mode, int64_t *evals) {
    CHECK_HANDLE(h);
    if (M < 0) return fail(NUFI_ERR_USAGE, "point count must be >= 0");
    if (n < 0) return fail(NUFI_ERR_USAGE, "step index must be >= 0");
    if (mode != NUFI_TRACE_FAST && mode != NUFI_TRACE_PARITY) return fail(NUFI_ERR_USAGE, "unknown trace mode");
    if (n == 0) return NUFI_OK;  // kernels.py:397-398
    const int64_t need = half_kick ? n + 1 : n;
    if (h->n_ovr > 0) {
        // flow.py:55-62 with installed fields: have = max(len, 1 + max installed step); a
        // slot that is neither stored nor installed cannot be evaluated (history.entry)
        int64_t top = -1;
        for (int64_t k = 0; 4 * k < (int64_t)h->ovr.size(); ++k)
            if (h->ovr[4 * k] != 0.0) top = k;
        const int64_t have = std::max<int64_t>(h->len, top + 1);
        bool missing = have < need;
        for (int64_t k = h->len; k < need && !missing; ++k)
            missing = 4 * k >= (int64_t)h->ovr.size() || h->ovr[4 * k] == 0.0;
        if (missing) {
            char buf[160];
            snprintf(buf, sizeof buf, "trace at step %lld needs fields 0..%lld; history holds %lld", (long long)n,
                     (long long)(need - 1), (long long)have);
            return fail(NUFI_ERR_USAGE, buf);
        }
    } else if (h->len < need) {
        char buf[160];
        snprintf(buf, sizeof buf, "need %lld stored fields for step %lld, have %lld", (long long)need, (long long)n,
                 (long long)h->len);  // kernels.py:399-402
        return fail(NUFI_ERR_USAGE, buf);
    }
    if (M == 0) return NUFI_OK;  // kernels.py:403-404
    if (!X || !V) return fail(NUFI_ERR_USAGE, "null points");
    const size_t bytes = (size_t)M * h->d * sizeof(double);
    double *dX = X, *dV = V, *dovr = nullptr;
    const bool dx = is_device_ptr(X), dv = is_device_ptr(V);
    AsyncTemps tmp(h->stream);
    if (!dx) CU(tmp.alloc(&dX, bytes));
    if (!dv) CU(tmp.alloc(&dV, bytes));
    if (!dx) CU(cudaMemcpyAsync(dX, X, bytes, cudaMemcpyHostToDevice, h->stream));
    if (!dv) CU(cudaMemcpyAsync(dV, V, bytes, cudaMemcpyHostToDevice, h->stream));
    if (h->n_ovr > 0) {
        // the reference's generic path (flow.py:65-82): every slot through its field object
        std::vector<double> tab(4 * (size_t)(n + 1), 0.0);
        std::copy(h->ovr.begin(), h->ovr.begin() + std::min(h->ovr.size(), tab.size()), tab.begin());
        // installed SplineField slabs of slots 0..n, packed in slot order
        std::vector<double> slabs;
        for (const auto &kv : h->ovr_spline) {
            if (kv.first > n) break;
            tab[4 * (size_t)kv.first + 1] = (double)(slabs.size() / h->nodes);
            slabs.insert(slabs.end(), kv.second.begin(), kv.second.end());
        }
        double *dslabs = nullptr;
        CU(tmp.alloc(&dovr, tab.size() * sizeof(double)));
        CU(cudaMemcpyAsync(dovr, tab.data(), tab.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        if (!slabs.empty()) {
            CU(tmp.alloc(&dslabs, slabs.size() * sizeof(double)));
            CU(cudaMemcpyAsync(dslabs, slabs.data(), slabs.size() * sizeof(double), cudaMemcpyHostToDevice,
                               h->stream));
        }
        CU(launch_trace_points_generic(h->d, h->hist, h->nodes, dovr, dslabs, h->N, h->cfg.L, (int)n, h->cfg.tau, dX,
                                       dV, M, half_kick ? 1 : 0, h->stream));
    } else {
        cudaError_t e = cudaErrorNotSupported;
        // d >= 2: slabs staged in a shared-memory ring (NUFI_TP_NORING=1: the in-place kernel, for tests)
        if (mode == NUFI_TRACE_FAST && !h->gl && !getenv("NUFI_TP_NORING"))
            e = launch_trace_points_ring(h->d, h->pow2, h->ev_hist, h->ev_elems, h->N, h->cfg.L, (int)n, h->cfg.tau,
                                         h->K, dX, dV, M, half_kick ? 1 : 0, h->stream);
        if (e == cudaErrorNotSupported)
            e = launch_trace_points(h->d, mode, h->pow2, h->hist, h->ev_hist, h->ev_elems, h->N, h->nodes, h->cfg.L,
                                    (int)n, h->cfg.tau, h->K, dX, dV, M, half_kick ? 1 : 0, h->stream);
        CU(e);
    }
    if (!dx) CU(cudaMemcpyAsync(X, dX, bytes, cudaMemcpyDeviceToHost, h->stream));
    if (!dv) CU(cudaMemcpyAsync(V, dV, bytes, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (evals) *evals += M * need;
    return NUFI_OK;
}

int nufi_moments(nufi_handle *h, int64_t n, double *out, int64_t *evals) {
    CHECK_HANDLE(h);
    if (int rc = refuse_installed(h)) return rc;
    if (n < 0) return fail(NUFI_ERR_USAGE, "step index must be >= 0");
    if (!out) return fail(NUFI_ERR_USAGE, "null output");
    if (n > 0 && h->len < n + 1) {
        char buf[160];
        snprintf(buf, sizeof buf, "psi at step %lld needs fields 0..%lld; history holds %lld", (long long)n,
                 (long long)n, (long long)h->len);  // flow.py:55-62, 106-112
        return fail(NUFI_ERR_USAGE, buf);
    }
    const int nm = mom_sums(h->d) + 2;
    const int ctas = (h->b_hi - h->b_lo) * h->vt_per_block * h->node_tiles;
    if (!h->mom_part) {
        const size_t rows = h->d == 1 ? (size_t)h->V : (size_t)h->vt_total;  // d = 1 sweep tiles may be finer
        CU(dalloc(&h->mom_part, rows * h->node_tiles * nm * sizeof(double), h->stream));
        CU(dalloc(&h->d_mom, 16 * sizeof(double), h->stream));
    }
    TraceRhoParams p = trace_params(h, n, h->b_lo);
    p.partial = h->mom_part;
    // one point per thread for the sweep (the extra moment accumulators would
    // spill the 2-point d = 3 variant); the same rows in twice the passes
    const int ppt = 1;
    p.passes = h->passes * h->ppt;
    int threads = h->threads, ctas_s = ctas;
    if (h->d == 1) {
        // its own tiles: w rows strided across each residue-class block (d1_row), so a
        // rank's share of blocks is exactly its share of rows
        const int rpb = (int)(h->V / h->B);
        int w = 8;
        while (w > 1 && rpb % w) w >>= 1;
        p.vt_rows = w;
        p.passes = 1;
        p.vt_per_block = rpb / w;
        p.vt_lo = h->b_lo * p.vt_per_block;
        threads = 32 * w;
        ctas_s = (h->b_hi - h->b_lo) * p.vt_per_block * h->node_tiles;
    }
    const double measure = std::pow(h->hx, (double)h->d) * h->hv_d;  // density.py:107
    {
        ProfScope ps(h, 0, point_steps(h, n > 0 ? n + 1 : 0, h->b_hi - h->b_lo));
        if (h->gl)
            CU(launch_trace_rho_global(h->d, true, h->pow2, p, h->K, ctas_s, threads, h->stream));
        else
            CU(launch_sweep_moments(h->d, ppt, h->pow2, p, h->K, ctas_s, threads, h->stream));
    }
    CU(launch_reduce_moments(h->mom_part, ctas_s, h->d, measure, h->d_mom, h->stream));
    CU(cudaMemcpyAsync(out, h->d_mom, nm * sizeof(double), cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (evals && n > 0) *evals += (int64_t)point_steps(h, n + 1, h->b_hi - h->b_lo);
    return NUFI_OK;
}

int nufi_eval_field(nufi_handle *h, int64_t slot, const double *X, int64_t M, double *phi_out, double *E_out) {
    CHECK_HANDLE(h);
    if (M < 0) return fail(NUFI_ERR_USAGE, "point count must be >= 0");
    if (slot < 0 || slot >= h->len) return fail(NUFI_ERR_USAGE, "history has no entry at that index");  // spline.py:144-146
    if (M == 0) return NUFI_OK;
    if (!X) return fail(NUFI_ERR_USAGE, "null points");
    const size_t bytes = (size_t)M * h->d * sizeof(double);
    const double *dX = X;
    double *tX = nullptr, *dphi = phi_out, *dE = E_out, *tphi = nullptr, *tE = nullptr;
    AsyncTemps tmp(h->stream);
    if (!is_device_ptr(X)) {
        CU(tmp.alloc(&tX, bytes));
        CU(cudaMemcpyAsync(tX, X, bytes, cudaMemcpyHostToDevice, h->stream));
        dX = tX;
    }
    if (phi_out && !is_device_ptr(phi_out)) {
        CU(tmp.alloc(&tphi, (size_t)M * sizeof(double)));
        dphi = tphi;
    }
    if (E_out && !is_device_ptr(E_out)) {
        CU(tmp.alloc(&tE, bytes));
        dE = tE;
    }
    CU(launch_eval_field(h->d, h->hist + (size_t)slot * h->nodes, h->N, h->cfg.L, dX, M, dphi, dE, h->stream));
    if (tphi) CU(cudaMemcpyAsync(phi_out, tphi, (size_t)M * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    if (tE) CU(cudaMemcpyAsync(E_out, tE, bytes, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return NUFI_OK;
}

// solve_poisson / fit_spline one by one (host or device buffers of Nx^d doubles)
static int poisson_fit(nufi_handle *h, int mode, const double *in, double *out, double *spec_re, double *spec_im,
                       double *W_out) {
    CHECK_HANDLE(h);
    if (!in || (!out && mode != 2) || (mode >= 2 && (!spec_im || (mode == 2 && !spec_re))))
        return fail(NUFI_ERR_USAGE, "null argument");
    const size_t bytes = (size_t)h->nodes * sizeof(double);
    // device staging: in, out, spec re / im, W (one allocation)
    double *buf = nullptr;
    AsyncTemps tmp(h->stream);
    CU(tmp.alloc(&buf, 4 * bytes + 64));
    double *din = buf, *dout = buf + h->nodes, *dre = buf + 2 * h->nodes, *dim = buf + 3 * h->nodes,
           *dW = buf + 4 * h->nodes;
    CU(cudaMemcpyAsync(din, in, bytes, cudaMemcpyDefault, h->stream));
    if (mode == 3) CU(cudaMemcpyAsync(dim, spec_im, bytes, cudaMemcpyDefault, h->stream));  // input
    CU(cudaMemsetAsync(h->d_status, 0, sizeof(int), h->stream));
    FieldParams f = field_params(h);
    CU(launch_poisson_fit(f, mode, din, dout, dre, dim, dW, h->d_status, h->stream));
    int st = 0;
    CU(cudaMemcpyAsync(&st, h->d_status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    if (out) CU(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDefault, h->stream));
    if (mode != 3) {
        if (spec_re) CU(cudaMemcpyAsync(spec_re, dre, bytes, cudaMemcpyDefault, h->stream));
        if (spec_im) CU(cudaMemcpyAsync(spec_im, dim, bytes, cudaMemcpyDefault, h->stream));
    }
    if (W_out) CU(cudaMemcpyAsync(W_out, dW, sizeof(double), cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (st == NUFI_ERR_NUMERICAL) {
        CU(cudaMemsetAsync(h->d_status, 0, sizeof(int), h->stream));
        return fail(NUFI_ERR_NUMERICAL, "density is not neutral: nodal mean exceeds 1e-8 max|rho|; "
                                        "subtract the mean before solving");  // poisson.py:98-104
    }
    return NUFI_OK;
}

int nufi_solve_poisson(nufi_handle *h, const double *rho, double *phi_out, double *spec_re, double *spec_im,
                       double *W_out) {
    return poisson_fit(h, 0, rho, phi_out, spec_re, spec_im, W_out);
}

int nufi_fit_spline(nufi_handle *h, const double *phi, double *coeffs_out) {
    return poisson_fit(h, 1, phi, coeffs_out, nullptr, nullptr, nullptr);
}

int nufi_transform_values(nufi_handle *h, const double *values, double *spec_re, double *spec_im) {
    return poisson_fit(h, 2, values, nullptr, spec_re, spec_im, nullptr);
}

int nufi_inverse_transform(nufi_handle *h, const double *spec_re, const double *spec_im, double *values_out) {
    return poisson_fit(h, 3, spec_re, values_out, nullptr, const_cast<double *>(spec_im), nullptr);
}

int nufi_bspline_weights(nufi_handle *h, const double *t, int64_t M, double *w_out, double *dw_out) {
    CHECK_HANDLE(h);
    if (M < 0) return fail(NUFI_ERR_USAGE, "point count must be >= 0");
    if (M == 0) return NUFI_OK;
    if (!t || (!w_out && !dw_out)) return fail(NUFI_ERR_USAGE, "null argument");
    const size_t bytes = (size_t)M * sizeof(double);
    AsyncTemps tmp(h->stream);
    const double *dt = t;
    double *dw = w_out, *ddw = dw_out;
    if (!is_device_ptr(t)) {
        double *p = nullptr;
        CU(tmp.alloc(&p, bytes));
        CU(cudaMemcpyAsync(p, t, bytes, cudaMemcpyHostToDevice, h->stream));
        dt = p;
    }
    const bool hw = w_out && !is_device_ptr(w_out), hdw = dw_out && !is_device_ptr(dw_out);
    if (hw) CU(tmp.alloc(&dw, 4 * bytes));
    if (hdw) CU(tmp.alloc(&ddw, 4 * bytes));
    CU(launch_bspline_weights(dt, M, dw, ddw, h->stream));
    if (hw) CU(cudaMemcpyAsync(w_out, dw, 4 * bytes, cudaMemcpyDeviceToHost, h->stream));
    if (hdw) CU(cudaMemcpyAsync(dw_out, ddw, 4 * bytes, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return NUFI_OK;
}

int nufi_eval_f0(nufi_handle *h, const double *X, const double *V, int64_t M, double *F) {
    CHECK_HANDLE(h);
    if (M < 0) return fail(NUFI_ERR_USAGE, "point count must be >= 0");
    if (M == 0) return NUFI_OK;
    if (!X || !V || !F) return fail(NUFI_ERR_USAGE, "null argument");
    const size_t bytes = (size_t)M * h->d * sizeof(double);
    const double *dX = X, *dV = V;
    double *dF = F;
    double *tX = nullptr, *tV = nullptr, *tF = nullptr;
    AsyncTemps tmp(h->stream);
    if (!is_device_ptr(X)) {
        CU(tmp.alloc(&tX, bytes));
        CU(cudaMemcpyAsync(tX, X, bytes, cudaMemcpyHostToDevice, h->stream));
        dX = tX;
    }
    if (!is_device_ptr(V)) {
        CU(tmp.alloc(&tV, bytes));
        CU(cudaMemcpyAsync(tV, V, bytes, cudaMemcpyHostToDevice, h->stream));
        dV = tV;
    }
    const bool df = is_device_ptr(F);
    if (!df) {
        CU(tmp.alloc(&tF, M * sizeof(double)));
        dF = tF;
    }
    CU(launch_eval_f0(h->d, h->f0, dX, dV, M, dF, h->stream));
    if (!df) CU(cudaMemcpyAsync(F, dF, M * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return NUFI_OK;
}

}  // extern "C"
