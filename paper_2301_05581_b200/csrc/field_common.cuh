// field_common.cuh -- the per-step tail of the NuFI loop as a CTA-wide device routine.
//
// Replaces, per step:
//   density.compute_rho's combine + neutralisation   density.py:80-85
//   poisson.solve_poisson                             poisson.py:90-112
//   spline.fit_spline                                 spline.py:71-86
//   PotentialHistory.append                           spline.py:132-142
//   poisson.electric_energy                           poisson.py:115-120
//   E at the nodes (SplineField.eval_E_many)          spline.py:50-52, kernels.py:102-123
//
// Spectral steps are separable shared-memory DFTs (Nx^d <= 4096) with exact
// integer twiddle indices; every output's sum is split over G lanes and
// combined with warp shuffles, so one CTA finishes a 64-point problem in ~1 us.
// fit_spline's forward FFT of phi is fused away: for real rho the spectrum of
// phi is phi_hat * N^d, so the coefficient slab is Re IDFT(phi_hat / prod sym)
// (poisson.py:85-87 then spline.py:78-84, one transform pair instead of two).
// The constant per-mode factors 1 / (N^d k^2 prod_a sym(alpha_a)) and k^2 are
// tabulated once per handle (field_tables_kernel).
//
// Called by field_update_kernel (one CTA) and, for d = 1, by the last CTA of
// the fused trace kernel (trace_rho_1d.cu) so a whole step is one launch.
#pragma once

#include <cfloat>

#include "trace_common.cuh"

namespace nufi {

struct FieldParams {
    int d, N, nodes, B;
    double L, inv_h, hv_d, rho_bar, L_d;
    double K;  // kick scale of the evaluation slabs (trace_common.cuh)
    // constant tables (device, field_tables_kernel): twiddles cos/sin(2 pi m / N);
    // fac[0:nodes] = 1 / (N^d k^2 prod_a sym(alpha_a)) (0 at the zero / Nyquist modes),
    // fac[nodes:2 nodes] = prod_a sym(alpha_a); k2 = |2 pi alpha / L|^2
    const double *twc, *tws, *fac, *k2;
    // d = 1 only: circulant kernels of the (linear, translation-invariant) field
    // map, c = gc (*) rho and phi = gp (*) rho (field_conv_kernels_kernel)
    const double *gc, *gp;
    // d >= 2: source index of every evaluation-slab element (ev_halo_source, tabulated)
    const int *halo;
    // v-sums: B blocks of rows_per_block rows of Nx^d sums, combined in fixed order;
    // min / max: B blocks of mm_per_block (min, max) pairs
    const double *sums;
    int rows_per_block;
    const double *minmax;
    int mm_per_block;
    // d = 1 split run (run_1d.cu): the last row of every tile is traced by helper CTAs; a tile
    // row partial is then sums + sums_last (the tile's sequential sum's last add), and the
    // (min, max) pairs of minmax_last join those of minmax.  Nullable.
    const double *sums_last;
    const double *minmax_last;
    const double *rho_in;  // alternative input: a neutral rho (nufi_field_update)
    // step slot
    int64_t slot;
    double *hist;     // (cap, nodes) raw coefficient history
    double *ev_hist;  // (cap, ev_slab_elems) evaluation slabs
    int ev_slab_elems;
    // outputs (nullable)
    double *rho_out, *stats_out, *W_out, *E_out, *coeffs_out;
    double *ev_local;   // optional second destination of the evaluation slab (persistent kernel smem)
    int *status;        // NUFI_ERR_NUMERICAL when rho is not neutral
    int *status_mirror; // optional (e.g. pinned host): *status copied here when the tail ends
    int64_t *hist_len;  // device-side history length: slot + 1 after the append, slot after a failed
                        // neutrality check (what nufi_check_status reconciles the host length to)
    int finish_only;    // compute_rho only: stop after rho / stats
    int f32_hist;       // FP32 history (spline.py:118-125): stored slabs rounded to float
    unsigned long long *tstamps;  // debug: phase timestamps (thread 0), 10 slots
    // d = 1: shared-memory doubles available beyond field_smem_doubles(N, N, true) for staging
    // the tile-row partials with cp.async (0: read them with register loads)
    int64_t stage_cap;
    // multi-rank d >= 2 step (nufi_mg_step_async): before reading `sums`, wait until
    // wait_flags[q] >= wait_target for every source rank q < wait_G (system-scope acquire;
    // 4 s watchdog -> *wait_error = 1 and NUFI_ERR_COMM in *status, history untouched)
    const unsigned *wait_flags;
    int wait_G;
    unsigned wait_target;
    int *wait_error;
};

// end of a tail launch: publish the (sticky) device status to p.status_mirror
__device__ __forceinline__ void mirror_status(const FieldParams &p) {
    if (!p.status_mirror) return;
    __syncthreads();
    if (threadIdx.x == 0) *(volatile int *)p.status_mirror = p.status ? *(volatile int *)p.status : 0;
}

#ifndef NUFI_MG_MAX
#define NUFI_MG_MAX 8
#endif

// d = 1 whole-run persistent kernel (run_1d.cu)
struct Run1DParams {
    TraceRhoParams tp;  // geometry / arithmetic (tp.n unused)
    FieldParams fp;     // tail template (slot and outputs set per step)
    int n_first, n_last;
    double *rho_hist, *E_hist, *W_hist, *stats_hist;  // device rows (n - n_first), nullable
    unsigned *barrier;                                // zero at launch
    int tiles;                                        // node_tiles * v-tiles
    unsigned long long *stamps;                       // optional: CTA 0 globaltimer per step x 3
    double *blocks;   // two-level combine: B * nodes block sums + B (min, max)
    int two_level;    // combine tile partials across the grid first (second grid barrier)
    int prefetch;     // issue the next step's first ring group before this step's tail (the
                      // tail then works in another ring stage); needs stage >= tail workspace
    // ---- multi-rank run with the exchange fused into the kernel (run_1d.cu) ----
    int mg_ranks;          // G ranks (1: single GPU)
    int mg_emulated;       // 1: the G ranks are CTA groups of this one cooperative launch
    int mg_rank;           // real mode: this launch's rank
    int mg_ctas;           // CTAs per rank
    unsigned mg_base;      // arrival-flag value before this run's first step (monotonic)
    int *mg_error;         // watchdog: set when a peer never arrives (device flag)
    double *mg_xtab[NUFI_MG_MAX];     // per rank: exchange table, 2 x (B Nx + 2B) doubles (step parity)
    unsigned *mg_flags[NUFI_MG_MAX];  // per rank: G arrival flags, slot q written by rank q
    // per-rank local buffers in emulated mode (real mode: tp.partial / tp.fminmax / barrier)
    double *mg_partial[NUFI_MG_MAX], *mg_fminmax[NUFI_MG_MAX];
    unsigned *mg_barrier[NUFI_MG_MAX];
    // ---- split: helper CTAs trace every tile's last row (single rank, one tile per CTA) ----
    int split_helpers;     // helper CTAs after the tiles' CTAs (0: no split)
    double *row_last;      // 2 x (v-tiles x nodes): the last rows, by step parity
    double *row_last_mm;   // 2 x (tiles x 2): their (min, max) pairs
};

#define NUFI_STAMP(p, k)                                                              \
    do {                                                                              \
        if ((p).tstamps && threadIdx.x == 0) {                                        \
            unsigned long long _t;                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                   \
            (p).tstamps[k] = _t;                                                      \
        }                                                                             \
    } while (0)

// shared-memory doubles the routine needs: 4 work arrays, twiddles, the
// per-block sums (B <= 8 blocks staged when rows_per_block > 1), scratch
__host__ __device__ constexpr int field_smem_doubles(int nodes, int N, bool staged) {
    // staged (d = 1): + 8 block-sum rows and a 2N complex work buffer (circulant_fft4)
    return 4 * nodes + 2 * N + (staged ? 8 * nodes + 2 * N : 0) + 128;  // scratch: 3 x 32 warp slots
}

// FP32 history mode: a stored coefficient is the float32 rounding of the fit
// (PotentialHistory(dtype=float32) casts on append, spline.py:140), read back as double.
__device__ __forceinline__ double hist_round(double c, int f32) { return f32 ? (double)__double2float_rn(c) : c; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// CTA-wide sum in a fixed order (deterministic for a fixed blockDim): warp xor-trees, then
// warp 0 combines the per-warp values with one more xor-tree (one thread per warp value
// instead of every thread looping over all warps).
__device__ __forceinline__ double cta_sum(double v, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const double s = warp_sum(lane < nw ? scratch[lane] : 0.0);
        if (lane == 0) scratch[96] = s;
    }
    __syncthreads();
    const double s = scratch[96];
    __syncthreads();
    return s;
}

__device__ __forceinline__ double cta_max(double v, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double s = lane < nw ? scratch[lane] : -DBL_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
        if (lane == 0) scratch[96] = s;
    }
    __syncthreads();
    const double s = scratch[96];
    __syncthreads();
    return s;
}

// sum, min and max over the CTA with one shared-memory round trip (the sum in the order of
// cta_sum); every thread gets the results
__device__ __forceinline__ void cta_sum_min_max(double s, double mn, double mx, double *scratch, double &S,
                                                double &MN, double &MX) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    __syncthreads();
    if (lane == 0) {
        scratch[warp] = s;
        scratch[32 + warp] = mn;
        scratch[64 + warp] = mx;
    }
    __syncthreads();
    if (warp == 0) {
        double a = lane < nw ? scratch[lane] : 0.0;
        double b = lane < nw ? scratch[32 + lane] : DBL_MAX;
        double c = lane < nw ? scratch[64 + lane] : -DBL_MAX;
        a = warp_sum(a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            b = fmin(b, __shfl_xor_sync(0xffffffffu, b, o));
            c = fmax(c, __shfl_xor_sync(0xffffffffu, c, o));
        }
        if (lane == 0) {
            scratch[96] = a;
            scratch[97] = b;
            scratch[98] = c;
        }
    }
    __syncthreads();
    S = scratch[96];
    MN = scratch[97];
    MX = scratch[98];
    __syncthreads();
}

// One separable DFT pass along the axis of stride st:
//   out[e] = sum_x in[e with x on the axis] * exp(sign * 2 pi i alpha x / N)
// Each output is summed by G consecutive lanes (G | 32), combined by shuffles.
__device__ __forceinline__ void dft_pass(const double *__restrict__ ire, const double *__restrict__ iim,
                                         double *__restrict__ ore, double *__restrict__ oim,
                                         const double *__restrict__ twc, const double *__restrict__ tws, int N,
                                         int nodes, int st, double sign, int G, bool pow2) {
    const int T = blockDim.x;
    const int part = threadIdx.x % G;
    for (int e = threadIdx.x / G; e < nodes; e += T / G) {
        const int inner = e % st;
        const int alpha = (e / st) % N;
        const int base = (e / (st * N)) * st * N + inner;
        double re = 0.0, im = 0.0;
        for (int x = part; x < N; x += G) {
            int m = alpha * x;
            m = pow2 ? (m & (N - 1)) : (m % N);
            const double c = twc[m], s = sign * tws[m];
            const double xr = ire[base + x * st], xi = iim[base + x * st];
            re = fma(xr, c, fma(-xi, s, re));
            im = fma(xr, s, fma(xi, c, im));
        }
        if (G > 1) {
            const unsigned mask = __activemask();
            for (int o = G >> 1; o > 0; o >>= 1) {
                re += __shfl_xor_sync(mask, re, o, G);
                im += __shfl_xor_sync(mask, im, o, G);
            }
        }
        if (part == 0) {
            ore[e] = re;
            oim[e] = im;
        }
    }
    __syncthreads();
}

// One separable FFT along the axis of stride st = 2^logst (N = 2^logN), Stockham autosort
// (no bit-reversal pass): one radix-2 stage when logN is odd, then radix-4 stages, each a
// shared-memory ping-pong between (ar, ai) and (br, bi) with one CTA barrier -- log4 N + 1
// passes over the data instead of the log2 N + 1 of a radix-2 pass sequence with a
// bit-reversal copy.  The transform: out[.. alpha ..] = sum_x in[.. x ..] e^{sign 2 pi i alpha x / N}.  On return (ar, ai)
// hold the result (the pointers are swapped once per stage).
__device__ __forceinline__ void fft_axis_stockham(double *&ar, double *&ai, double *&br, double *&bi,
                                                  const double *__restrict__ twc, const double *__restrict__ tws,
                                                  int logN, int nodes, int logst, double sign) {
    const int T = blockDim.x, N = 1 << logN;
    int lognc = logN, logs = 0;  // current sub-transform length 2^lognc, stride 2^logs
    while (lognc > 0) {
        const int logr = (lognc & 1) ? 1 : 2;  // radix 2 first when log2 N is odd, then radix 4
        const int logm = lognc - logr;
        const int nb = nodes >> logr;  // butterflies of this stage
        const int tshift = logN - lognc;  // twiddle index = p * N / ncur
        for (int b = threadIdx.x; b < nb; b += T) {
            int inner = 0, rest = b;
            if (logst) {
                inner = b & ((1 << logst) - 1);
                rest = b >> logst;
            }
            const int q = rest & ((1 << logs) - 1);
            const int pp = (rest >> logs) & ((1 << logm) - 1);
            const int outer = rest >> (logs + logm);
            const int base = (outer << (logst + logN)) + inner;
            const int ix = base + ((q + (pp << logs)) << logst);    // x = q + s p
            const int ox = base + ((q + (pp << (logs + logr))) << logst);  // y = q + s r p
            const int mst = 1 << (logm + logs + logst);   // input step  s m  (in elements)
            const int sst = 1 << (logs + logst);          // output step s
            const int tw = pp << tshift;
            if (logr == 1) {
                const double a_r = ar[ix], a_i = ai[ix], b_r = ar[ix + mst], b_i = ai[ix + mst];
                const double wr = twc[tw], wi = sign * tws[tw];
                const double dr = a_r - b_r, di = a_i - b_i;
                br[ox] = a_r + b_r;
                bi[ox] = a_i + b_i;
                br[ox + sst] = fma(dr, wr, -di * wi);
                bi[ox + sst] = fma(dr, wi, di * wr);
            } else {
                const double a_r = ar[ix], a_i = ai[ix];
                const double b_r = ar[ix + mst], b_i = ai[ix + mst];
                const double c_r = ar[ix + 2 * mst], c_i = ai[ix + 2 * mst];
                const double d_r = ar[ix + 3 * mst], d_i = ai[ix + 3 * mst];
                const double w1r = twc[tw], w1i = sign * tws[tw];
                const double w2r = twc[2 * tw], w2i = sign * tws[2 * tw];
                const double w3r = twc[3 * tw], w3i = sign * tws[3 * tw];
                const double apc_r = a_r + c_r, apc_i = a_i + c_i, amc_r = a_r - c_r, amc_i = a_i - c_i;
                const double bpd_r = b_r + d_r, bpd_i = b_i + d_i;
                // j (b - d) with j = sign * i
                const double jb_r = -sign * (b_i - d_i), jb_i = sign * (b_r - d_r);
                br[ox] = apc_r + bpd_r;
                bi[ox] = apc_i + bpd_i;
                const double x1r = amc_r + jb_r, x1i = amc_i + jb_i;
                const double x2r = apc_r - bpd_r, x2i = apc_i - bpd_i;
                const double x3r = amc_r - jb_r, x3i = amc_i - jb_i;
                br[ox + sst] = fma(x1r, w1r, -x1i * w1i);
                bi[ox + sst] = fma(x1r, w1i, x1i * w1r);
                br[ox + 2 * sst] = fma(x2r, w2r, -x2i * w2i);
                bi[ox + 2 * sst] = fma(x2r, w2i, x2i * w2r);
                br[ox + 3 * sst] = fma(x3r, w3r, -x3i * w3i);
                bi[ox + 3 * sst] = fma(x3r, w3i, x3i * w3r);
            }
        }
        __syncthreads();
        double *tr = ar, *ti = ai;
        ar = br, ai = bi, br = tr, bi = ti;
        lognc = logm;
        logs += logr;
    }
    (void)N;
}

// In-place radix-2 complex FFT of length N = 2^logN on shared arrays (re, im) whose
// input is already in bit-reversed order; sign -1: forward e^{-2 pi i jk/N}, +1:
// unscaled inverse.  twc / tws: cos / sin(2 pi m / N), m < N.  One butterfly per
// thread per stage, a CTA barrier between stages.
static __device__ __forceinline__ void fft_radix2(double *re, double *im, const double *twc, const double *tws, int N,
                                                  double sign) {
    for (int half = 1; half < N; half <<= 1) {
        const int stride = N / (2 * half);
        for (int b = threadIdx.x; b < N / 2; b += blockDim.x) {
            const int pos = b & (half - 1);
            const int i0 = ((b - pos) << 1) + pos, i1 = i0 + half;
            const double wr = twc[pos * stride], wi = sign * tws[pos * stride];
            const double ur = re[i1], ui = im[i1];
            const double xr = fma(ur, wr, -ui * wi), xi = fma(ur, wi, ui * wr);
            const double ar = re[i0], ai = im[i0];
            re[i1] = ar - xr;
            im[i1] = ai - xi;
            re[i0] = ar + xr;
            im[i0] = ai + xi;
        }
        __syncthreads();
    }
}

// Skewed shared-memory layouts of the d = 1 convolution operands (N <= 64), so the
// blocked loads of circulant_blocked hit distinct banks: r at i + i/8, kernels at m + m/4.
__device__ __forceinline__ int rsk(int i) { return i + (i >> 3); }
__device__ __forceinline__ int gsk(int m) { return m + (m >> 2); }

// c = gc (*) r and phi = gp (*) r for 4 <= N <= 64 (power of two), operands skewed
// (rsk / gsk), outputs plain.  Each lane computes 4 consecutive outputs over TP =
// min(8, N) consecutive taps, sliding a 4-value window along the kernel: one kernel
// load and one r load per 4 FMAs (the one-output-per-lane-group form was bound by its
// 2 loads per FMA).  The P = N / TP tap parts of an output group sit in lanes Q = 32 / P
// apart and are combined by an xor tree.  The order depends on N only.
template <int TP>
__device__ __forceinline__ void circulant_blocked_taps(const double *g, const double *r, int j0, int i0, int M,
                                                       double &a0, double &a1, double &a2, double &a3) {
    // every load issued up front (compile-time tap count): r[i0 .. i0+TP) and the TP + 3
    // kernel values g[j0 + 3 - i0 - t'] the sliding window visits
    double rv[TP], gv[TP + 3];
#pragma unroll
    for (int t = 0; t < TP; ++t) rv[t] = r[rsk(i0 + t)];
#pragma unroll
    for (int u = 0; u < TP + 3; ++u) gv[u] = g[gsk((j0 + 3 - i0 - u) & M)];
    // tap t, output k: g[j0 + k - i0 - t] = gv[3 - k + t]
#pragma unroll
    for (int t = 0; t < TP; ++t) {
        a0 = fma(gv[3 + t], rv[t], a0);
        a1 = fma(gv[2 + t], rv[t], a1);
        a2 = fma(gv[1 + t], rv[t], a2);
        a3 = fma(gv[t], rv[t], a3);
    }
}

static __device__ __forceinline__ void circulant_blocked(const double *gc, const double *gp, const double *r,
                                                         double *c, double *phi, int N) {
    // powers of two throughout: shifts and masks only (an integer division costs ~100s of cycles)
    const int logN = 31 - __clz(N), logTP = logN < 3 ? logN : 3, logP = logN - logTP, logQ = 5 - logP;
    const int TP = 1 << logTP, P = 1 << logP, Q = 1 << logQ, G = N >> 1;  // G groups of 4 outputs
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, ln = threadIdx.x & 31;
    const int part = ln >> logQ, gl = ln & (Q - 1), M = N - 1;
    for (int wb = 0; wb * Q < G; wb += nw) {  // warp-uniform trip count
        if ((wb + warp) * Q >= G) break;         // whole warp idle (warp-uniform)
        const int grp = (wb + warp) * Q + gl;
        const bool active = grp < G;
        const int o0 = active ? 4 * grp : 0;
        const bool isc = o0 < N;
        const double *g = isc ? gc : gp;
        const int j0 = isc ? o0 : o0 - N, i0 = part * TP;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (TP == 8)
            circulant_blocked_taps<8>(g, r, j0, i0, M, a0, a1, a2, a3);
        else  // N = 4
            circulant_blocked_taps<4>(g, r, j0, i0, M, a0, a1, a2, a3);
        for (int q = P >> 1; q > 0; q >>= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, q * Q);
            a1 += __shfl_xor_sync(0xffffffffu, a1, q * Q);
            a2 += __shfl_xor_sync(0xffffffffu, a2, q * Q);
            a3 += __shfl_xor_sync(0xffffffffu, a3, q * Q);
        }
        if (active && part == 0) {
            double *dst = isc ? c : phi;
            dst[j0] = a0;
            dst[j0 + 1] = a1;
            dst[j0 + 2] = a2;
            dst[j0 + 3] = a3;
        }
    }
}

// ---- four-step FFT for N = 16 R1 (R1 = 8, 16): two passes of in-register DFTs ----
// cos / sin(2 pi j / 16), j < 8 (correctly rounded; the symmetric pairs exactly equal)
#define NUFI_C1 0x1.d906bcf328d46p-1  // cos(pi/8)
#define NUFI_S1 0x1.87de2a6aea963p-2  // sin(pi/8)
#define NUFI_R2 0x1.6a09e667f3bcdp-1  // sqrt(2)/2
__device__ __forceinline__ constexpr double tw16c(int j) {
    return j == 0 ? 1.0 : j == 1 ? NUFI_C1 : j == 2 ? NUFI_R2 : j == 3 ? NUFI_S1 : j == 4 ? 0.0
         : j == 5 ? -NUFI_S1 : j == 6 ? -NUFI_R2 : -NUFI_C1;
}
__device__ __forceinline__ constexpr double tw16s(int j) {
    return j == 0 ? 0.0 : j == 1 ? NUFI_S1 : j == 2 ? NUFI_R2 : j == 3 ? NUFI_C1 : j == 4 ? 1.0
         : j == 5 ? NUFI_C1 : j == 6 ? NUFI_R2 : NUFI_S1;
}
__device__ __forceinline__ constexpr int brev_c(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
    return r;
}

// In-register R-point DFT (R = 8, 16), X_k = sum_n x_n e^{SIGN 2 pi i n k / R}: radix-2
// decimation in time on a bit-reversed copy, twiddles compile-time constants (the
// trivial ones -- 1 and +-i -- are plain adds).
template <int R, int SIGN>
__device__ __forceinline__ void dft_reg(double (&re)[R], double (&im)[R]) {
    constexpr int LOG = R == 16 ? 4 : 3;
    double ar[R], ai[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
        ar[i] = re[brev_c(i, LOG)];
        ai[i] = im[brev_c(i, LOG)];
    }
#pragma unroll
    for (int h = 1; h < R; h <<= 1) {
#pragma unroll
        for (int b = 0; b < R / 2; ++b) {
            const int pos = b % h, i0 = (b / h) * 2 * h + pos, i1 = i0 + h;
            const int t = pos * (16 / (2 * h));  // e^{SIGN 2 pi i pos / (2h)} = tw16[t]
            double xr, xi;
            if (t == 0) {
                xr = ar[i1];
                xi = ai[i1];
            } else if (t == 4) {  // multiply by SIGN * i
                xr = -SIGN * ai[i1];
                xi = SIGN * ar[i1];
            } else {
                const double wr = tw16c(t), wi = SIGN * tw16s(t);
                xr = fma(ar[i1], wr, -ai[i1] * wi);
                xi = fma(ar[i1], wi, ai[i1] * wr);
            }
            ar[i1] = ar[i0] - xr;
            ai[i1] = ai[i0] - xi;
            ar[i0] = ar[i0] + xr;
            ai[i0] = ai[i0] + xi;
        }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        re[i] = ar[i];
        im[i] = ai[i];
    }
}

// One four-step transform, N = R1 * 16, n = n1 + R1 n2, k = k2 + 16 k1:
//   pass 1 (thread n1 < R1): Y[n1][k2] = e^{SIGN 2 pi i n1 k2 / N} sum_n2 x[n1 + R1 n2] w16^{n2 k2}
//   pass 2 (thread k2 < 16): X[k2 + 16 k1] = sum_n1 Y[n1][k2] w_R1^{n1 k1}
// Y lives in (yr, yi) at k2 R1 + (n1 ^ (k2 & (R1 - 1))) (xor swizzle: both passes
// conflict-free or 2-way); twc / tws: cos / sin(2 pi m / N) in shared memory.
template <int R1, int SIGN>
__device__ __forceinline__ void fft4_pass1(const double *xr, const double *xi, double *yr, double *yi,
                                           const double *twc, const double *tws) {
    const int n1 = threadIdx.x;
    if (n1 >= R1) return;
    double re[16], im[16];
#pragma unroll
    for (int n2 = 0; n2 < 16; ++n2) {
        re[n2] = xr[n1 + R1 * n2];
        im[n2] = xi ? xi[n1 + R1 * n2] : 0.0;
    }
    dft_reg<16, SIGN>(re, im);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
        const int m = n1 * k2;  // < N
        const double wr = twc[m], wi = SIGN * tws[m];
        const int o = k2 * R1 + (n1 ^ (k2 & (R1 - 1)));
        yr[o] = fma(re[k2], wr, -im[k2] * wi);
        yi[o] = fma(re[k2], wi, im[k2] * wr);
    }
}

template <int R1>
__device__ __forceinline__ void fft4_pass2_load(const double *yr, const double *yi, double (&re)[R1],
                                                double (&im)[R1]) {
    const int k2 = threadIdx.x;
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
        const int o = k2 * R1 + (n1 ^ (k2 & (R1 - 1)));
        re[n1] = yr[o];
        im[n1] = yi[o];
    }
}

// c + i phi = IFFT_unscaled( FFT(r) * fac * (1 + i sym) ) by two four-step transforms,
// natural order throughout; wr / wi: 2N doubles of work space.  3 CTA barriers.
template <int R1>
static __device__ __forceinline__ void circulant_fft4(const FieldParams &p, const double *r, double *c, double *phi,
                                                      const double *twc, const double *tws, double *wr,
                                                      double *wi) {
    constexpr int N = 16 * R1;
    fft4_pass1<R1, -1>(r, nullptr, wr, wi, twc, tws);  // forward: r is real
    __syncthreads();
    if (threadIdx.x < 16) {
        const int k2 = threadIdx.x;
        double re[R1], im[R1];
        fft4_pass2_load<R1>(wr, wi, re, im);
        dft_reg<R1, -1>(re, im);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) {  // spectrum * fac * (1 + i sym) -> (c, phi), natural order
            const int k = k2 + 16 * k1;
            const double f = p.fac[k], sy = p.fac[N + k];
            const double a = re[k1] * f, b = im[k1] * f;
            c[k] = fma(-b, sy, a);
            phi[k] = fma(a, sy, b);
        }
    }
    __syncthreads();
    fft4_pass1<R1, 1>(c, phi, wr, wi, twc, tws);  // inverse, unscaled
    __syncthreads();
    if (threadIdx.x < 16) {
        const int k2 = threadIdx.x;
        double re[R1], im[R1];
        fft4_pass2_load<R1>(wr, wi, re, im);
        dft_reg<R1, 1>(re, im);
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) {
            c[k2 + 16 * k1] = re[k1];
            phi[k2 + 16 * k1] = im[k1];
        }
    }
}

// c + i phi = IFFT_unscaled( FFT(r) * fac * (1 + i sym) ): the d = 1 Poisson solve +
// spline fit in O(N log N) (fac = 1 / (N k^2 sym), 0 at the zero / Nyquist modes;
// poisson.py:105-110, spline.py:78-84).  Both products are real-even factors on a
// Hermitian spectrum, so c and phi come out as the real and imaginary parts of ONE
// inverse transform.  twc / tws: the twiddles, already in shared memory; fq: this
// thread's spectral factors (fac[k], fac[N+k], fac[kb], fac[N+kb]) for k = threadIdx.x,
// loaded by the caller with its other global loads.
static __device__ __forceinline__ void circulant_fft(const FieldParams &p, const double *r, double *c, double *phi,
                                                     const double *twc, const double *tws, int N, const double fq[4]) {
    const int logN = 31 - __clz(N);
    for (int m = threadIdx.x; m < N; m += blockDim.x) {
        const int br = (int)(__brev((unsigned)m) >> (32 - logN));
        c[br] = r[m];
        phi[br] = 0.0;
    }
    __syncthreads();
    fft_radix2(c, phi, twc, tws, N, -1.0);
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        const int kb = (int)(__brev((unsigned)k) >> (32 - logN));
        if (k <= kb) {  // multiply and bit-reverse in place (disjoint swap pairs)
            const bool mine = k == (int)threadIdx.x;
            const double f0 = mine ? fq[0] : p.fac[k], s0 = mine ? fq[1] : p.fac[N + k];
            const double f1 = mine ? fq[2] : p.fac[kb], s1 = mine ? fq[3] : p.fac[N + kb];
            const double a0 = c[k] * f0, b0 = phi[k] * f0, a1 = c[kb] * f1, b1 = phi[kb] * f1;
            c[kb] = fma(-b0, s0, a0);
            phi[kb] = fma(a0, s0, b0);
            c[k] = fma(-b1, s1, a1);
            phi[k] = fma(a1, s1, b1);
        }
    }
    __syncthreads();
    fft_radix2(c, phi, twc, tws, N, 1.0);
}

// d = 1 tail: the Poisson solve + spline fit is a circulant operator on the
// nodal density (poisson.py:105-110 + spline.py:78-84 are diagonal in Fourier
// space), so the coefficient slab is one circular convolution c = gc (*) rho'
// and the nodal potential phi = gp (*) rho' another; the electric energy follows
// from Parseval, W = (L/N)/2 sum_i rho'_i phi_i = L/2 sum_alpha k^2 |phi_hat|^2
// (poisson.py:115-120).  This routine sits on the latency-critical path of every
// d = 1 step, so it is built around few dependent round trips:
//   A  all threads: every global load issued before any is consumed (one L2 round
//      trip), block sums of the tile-row partials, per-warp (min, max)      | barrier
//   B  warp 0: rho, its mean, rho', the neutrality check, stats              | barrier
//   C  all threads: the two convolutions (blocked direct N <= 64, else FFT)  | barrier
//   D  last warp: W;  all threads: the appended slabs and E at the nodes.
static __device__ __forceinline__ bool field_update_1d_body(const FieldParams &p, double *sm) {
    const int N = p.N, T = blockDim.x, B = p.B, rpb = p.rows_per_block;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = T >> 5;
    const bool small = N <= 64;  // blocked direct convolution on skewed operands, else FFT
    const int RS = small ? N + (N >> 3) : N, GS = small ? N + (N >> 2) : N;
    // B N + RS + 2 GS + 2 N + 128 <= field_smem_doubles(N, N, true) = 14 N + 128 (B <= 8)
    double *sb = sm;            // B * N block sums
    double *r = sb + B * N;     // rho, then rho' (skewed when small)
    double *gc = r + RS, *gp = gc + GS;  // kernels (skewed) or FFT twiddles
    double *c = gp + GS, *phi = c + N;
    double *scratch = phi + N;  // 128
    NUFI_STAMP(p, 0);
    // ---- A: with in-order issue a load feeding a store stalls the thread, so the kernel
    // taps / twiddles, the spectral factors, the block (min, max) and the tile-row
    // partials are all requested before anything is consumed ----
    const int t0 = threadIdx.x;
    const double *g0src = small ? p.gc : p.twc, *g1src = small ? p.gp : p.tws;
    double ga = 0.0, gb = 0.0, fq[4] = {0.0, 0.0, 0.0, 0.0};
    if (t0 < N) {
        ga = __ldg(g0src + t0);
        gb = __ldg(g1src + t0);
        if (!small) {
            const int kb = (int)(__brev((unsigned)t0) >> (32 - (31 - __clz(N))));
            if (t0 <= kb) {
                fq[0] = __ldg(p.fac + t0);
                fq[1] = __ldg(p.fac + N + t0);
                fq[2] = __ldg(p.fac + kb);
                fq[3] = __ldg(p.fac + N + kb);
            }
        }
    }
    const int nmm = p.sums ? B * p.mm_per_block : 0;
    double mn = DBL_MAX, mx = -DBL_MAX;
    // Staged path: every tile-row partial and (min, max) pair is copied into shared memory
    // with cp.async (16-byte chunks, no registers held, all in flight at once), then summed
    // from there.  The register-load path below is limited by the compiler interleaving
    // each load with its add (one L2 round trip per row).
    const int64_t nsum = (int64_t)B * rpb * N;
    const bool split = p.sums && p.sums_last;  // tile row partial = sums + sums_last
    const int64_t nstage = (nsum + 2 * (int64_t)nmm) * (split ? 2 : 1);
    const bool stage = p.sums && rpb > 1 && p.stage_cap >= nstage &&
                       ((reinterpret_cast<uintptr_t>(p.sums) | reinterpret_cast<uintptr_t>(p.minmax) |
                         reinterpret_cast<uintptr_t>(p.sums_last) | reinterpret_cast<uintptr_t>(p.minmax_last)) &
                        15) == 0;
    double *stg = sm + field_smem_doubles(N, N, true);  // even offset: 16-byte aligned
    double *stg_last = stg + nsum + 2 * (int64_t)nmm;   // split: the last rows and their pairs
    if (stage) {
        for (int64_t q = t0; q < nsum / 2; q += T) cp_async16(stg + 2 * q, p.sums + 2 * q);
        for (int q = t0; q < nmm; q += T) cp_async16(stg + nsum + 2 * q, p.minmax + 2 * q);
        if (split) {
            for (int64_t q = t0; q < nsum / 2; q += T) cp_async16(stg_last + 2 * q, p.sums_last + 2 * q);
            for (int q = t0; q < nmm; q += T) cp_async16(stg_last + nsum + 2 * q, p.minmax_last + 2 * q);
        }
        cp_async_wait_all();
        __syncthreads();
        // rows in order per output; rows in chunks of 8 with every load of a chunk issued
        // before its adds (N a power of two: shifts only)
        // two outputs per thread, their two add chains interleaved
        const int logN = 31 - __clz(N), BN = B * N;
        for (int it = t0; it < BN; it += 2 * T) {
            const int it2 = it + T < BN ? it + T : it;
            const size_t o1 = (size_t)(it >> logN) * rpb * N + (it & (N - 1));
            const size_t o2 = (size_t)(it2 >> logN) * rpb * N + (it2 & (N - 1));
            const double *s1 = stg + o1, *s2 = stg + o2;
            double S1 = 0.0, S2 = 0.0;
            if (split) {  // each tile row partial is its sequential sum's last add: s + last
                const double *l1 = stg_last + o1, *l2 = stg_last + o2;
                for (int q = 0; q < rpb; ++q) {
                    S1 += s1[(size_t)q * N] + l1[(size_t)q * N];
                    S2 += s2[(size_t)q * N] + l2[(size_t)q * N];
                }
            } else {
                int q = 0;
                for (; q + 8 <= rpb; q += 8) {
                    double a[8], b[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        a[u] = s1[(size_t)(q + u) * N];
                        b[u] = s2[(size_t)(q + u) * N];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        S1 += a[u];
                        S2 += b[u];
                    }
                }
                for (; q < rpb; ++q) {
                    S1 += s1[(size_t)q * N];
                    S2 += s2[(size_t)q * N];
                }
            }
            sb[it] = S1;
            if (it + T < BN) sb[it + T] = S2;
        }
        for (int q = t0; q < nmm; q += T) {
            mn = fmin(mn, stg[nsum + 2 * q]);
            mx = fmax(mx, stg[nsum + 2 * q + 1]);
            if (split) {
                mn = fmin(mn, stg_last[nsum + 2 * q]);
                mx = fmax(mx, stg_last[nsum + 2 * q + 1]);
            }
        }
    } else if (t0 < nmm) {
        mn = __ldcg(p.minmax + 2 * t0);
        mx = __ldcg(p.minmax + 2 * t0 + 1);
        if (split) {
            mn = fmin(mn, __ldcg(p.minmax_last + 2 * t0));
            mx = fmax(mx, __ldcg(p.minmax_last + 2 * t0 + 1));
        }
    }
    // ---- block sums over the block's rows in order (reduce_blocks_kernel order) ----
    if (p.sums && !stage) {
        if (split) {  // each tile row partial is its sequential sum's last add: s + last
            for (int it = threadIdx.x; it < B * N; it += T) {
                const int b = it / N, i = it - b * N;
                const size_t o = (size_t)b * rpb * N + i;
                double Sb = 0.0;
                for (int q = 0; q < rpb; ++q)
                    Sb += __ldcg(p.sums + o + (size_t)q * N) + __ldcg(p.sums_last + o + (size_t)q * N);
                sb[it] = Sb;
            }
        } else if (rpb <= 8) {
            // two outputs per thread per pass: all 2 * rpb loads in flight at once
            for (int it = threadIdx.x; it < B * N; it += 2 * T) {
                const int it2 = it + T;
                const double *s1 = p.sums + (size_t)(it / N) * rpb * N + (it % N);
                const double *s2 = p.sums + (size_t)(it2 / N) * rpb * N + (it2 % N);
                double v1[8], v2[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    v1[u] = u < rpb ? __ldcg(s1 + (size_t)u * N) : 0.0;
                    v2[u] = (u < rpb && it2 < B * N) ? __ldcg(s2 + (size_t)u * N) : 0.0;
                }
                double S1 = 0.0, S2 = 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (u < rpb) {
                        S1 += v1[u];
                        S2 += v2[u];
                    }
                sb[it] = S1;
                if (it2 < B * N) sb[it2] = S2;
            }
        } else {
            for (int it = threadIdx.x; it < B * N; it += T) {
                const int b = it / N, i = it - b * N;
                const double *src = p.sums + (size_t)b * rpb * N + i;
                double Sb = 0.0;
                int q = 0;
                for (; q + 8 <= rpb; q += 8) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (size_t)(q + u) * N);
#pragma unroll
                    for (int u = 0; u < 8; ++u) Sb += v[u];
                }
                for (; q < rpb; ++q) Sb += __ldcg(src + (size_t)q * N);
                sb[it] = Sb;
            }
        }
        for (int q = t0 + T; q < nmm; q += T) {
            mn = fmin(mn, __ldcg(p.minmax + 2 * q));
            mx = fmax(mx, __ldcg(p.minmax + 2 * q + 1));
            if (split) {
                mn = fmin(mn, __ldcg(p.minmax_last + 2 * q));
                mx = fmax(mx, __ldcg(p.minmax_last + 2 * q + 1));
            }
        }
    }
    if (p.sums) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
            scratch[warp] = mn;
            scratch[32 + warp] = mx;
        }
    }
    if (t0 < N) {
        gc[small ? gsk(t0) : t0] = ga;
        gp[small ? gsk(t0) : t0] = gb;
    }
    for (int m = t0 + T; m < N; m += T) {
        gc[small ? gsk(m) : m] = __ldg(g0src + m);
        gp[small ? gsk(m) : m] = __ldg(g1src + m);
    }
    __syncthreads();
    NUFI_STAMP(p, 1);
    // ---- B (warp 0): rho = rho_bar - hv S (density.py:81), c = mean, rho' = rho - c
    // (density.py:84-85), the neutrality check of poisson.py:97-104 on rho', stats ----
    if (warp == 0) {
        double s = 0.0;
        // two nodes per lane per pass (i, i + 32), their chains interleaved; s in node order
        for (int i = lane; i < N; i += 64) {
            const int i2 = i + 32 < N ? i + 32 : i;
            double r1, r2;
            if (p.sums) {
                double S1 = 0.0, S2 = 0.0;
                if (B == 8) {  // the usual block count: every load ahead of the ordered adds
                    double a[8], c2[8];
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        a[b] = sb[b * N + i];
                        c2[b] = sb[b * N + i2];
                    }
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        S1 += a[b];
                        S2 += c2[b];
                    }
                } else {
                    for (int b = 0; b < B; ++b) {
                        S1 += sb[b * N + i];
                        S2 += sb[b * N + i2];
                    }
                }
                r1 = p.rho_bar - p.hv_d * S1;
                r2 = p.rho_bar - p.hv_d * S2;
            } else {
                r1 = p.rho_in[i];
                r2 = p.rho_in[i2];
            }
            r[small ? rsk(i) : i] = r1;
            s += r1;
            if (i + 32 < N) {
                r[small ? rsk(i2) : i2] = r2;
                s += r2;
            }
        }
        s = warp_sum(s);
        // N is a power of two here: s * (1/N) is s / N exactly (no DDIV on the critical path)
        const double neut = p.sums ? s * (1.0 / (double)N) : 0.0;
        double s2 = 0.0, m = 0.0;
        for (int i = lane; i < N; i += 32) {
            const int ix = small ? rsk(i) : i;
            const double v = r[ix] - neut;
            r[ix] = v;
            if (p.rho_out) p.rho_out[i] = v;
            s2 += v;
            m = fmax(m, fabs(v));
        }
        s2 = warp_sum(s2);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (p.stats_out && lane == 0) p.stats_out[0] = neut;
        if (lane == 0) {
            const bool bad = fabs(s2 * (1.0 / (double)N)) > 1e-8 * m;
            scratch[96] = bad ? 1.0 : 0.0;
            if (bad && p.status) *p.status = NUFI_ERR_NUMERICAL;
            if (bad && p.hist_len) *p.hist_len = p.slot;  // the device length: this slot not appended
        }
    }
    // sampled f min / max (the per-warp partials of phase A) in another warp, off warp 0's path
    if (warp == (nw > 1 ? 1 : 0) && p.stats_out) {
        double fmn = (p.sums && lane < nw) ? scratch[lane] : DBL_MAX;
        double fmx = (p.sums && lane < nw) ? scratch[32 + lane] : -DBL_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            fmn = fmin(fmn, __shfl_xor_sync(0xffffffffu, fmn, o));
            fmx = fmax(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
        }
        if (lane == 0) {
            p.stats_out[1] = fmn;
            p.stats_out[2] = fmx;
        }
    }
    if (p.finish_only) return true;
    __syncthreads();
    NUFI_STAMP(p, 2);
    if (scratch[96] != 0.0) return false;  // history unchanged (the reference raises before appending)
    // ---- C: c = gc (*) rho', phi = gp (*) rho' ----
    if (small)
        circulant_blocked(gc, gp, r, c, phi, N);
    else if (N == 256)
        circulant_fft4<16>(p, r, c, phi, gc, gp, scratch + 128, scratch + 128 + N);
    else if (N == 128)
        circulant_fft4<8>(p, r, c, phi, gc, gp, scratch + 128, scratch + 128 + N);
    else
        circulant_fft(p, r, c, phi, gc, gp, N, fq);
    __syncthreads();
    NUFI_STAMP(p, 4);
    // ---- D: W (Parseval) in the last warp, which holds no append work for N < T ----
    if (warp == nw - 1 && p.W_out) {
        double w = 0.0;
        for (int i = lane; i < N; i += 32) w = fma(r[small ? rsk(i) : i], phi[i], w);
        w = warp_sum(w);
        if (lane == 0) *p.W_out = 0.5 * (p.L / (double)N) * w;
    }
    // ---- append: raw slab, evaluation slab (trace_common.cuh layout), E at the nodes ----
    const double evs = p.slot == 0 ? 0.5 : 1.0;  // slab 0 stored pre-halved
    double *evg = p.ev_hist ? p.ev_hist + (size_t)p.slot * p.ev_slab_elems : nullptr;
    double *evl = p.ev_local;
    double *hrow = p.hist ? p.hist + (size_t)p.slot * N : nullptr;
    for (int i = threadIdx.x; i < N; i += T) {
        const double e0 = c[(i - 1 + N) & (N - 1)], e1 = c[i], e2 = c[(i + 1) & (N - 1)], e3 = c[(i + 2) & (N - 1)];
        // the stored (and traced) slab; E at the nodes comes from the fit itself
        const double c0 = hist_round(e0, p.f32_hist), c1 = hist_round(e1, p.f32_hist),
                     c2 = hist_round(e2, p.f32_hist), c3 = hist_round(e3, p.f32_hist);
        double A, Bc, C;
        d1_cell_poly(c0, c1, c2, c3, evs * p.K, A, Bc, C);
        if (evg) {
            evg[d1_ia(i, N)] = A;
            evg[d1_ib(i, N)] = Bc;
            evg[d1_ic(i, N)] = C;
        }
        if (evl) {
            evl[d1_ia(i, N)] = A;
            evl[d1_ib(i, N)] = Bc;
            evl[d1_ic(i, N)] = C;
        }
        if (hrow) hrow[i] = c1;
        if (p.coeffs_out) p.coeffs_out[i] = c1;
        // E(x_i) = -(N/L) (-c_{i-1}/2 + c_{i+1}/2)  (f = 0 stencil, kernels.py:102-123)
        if (p.E_out) p.E_out[i] = -(0.5 * (e2 - e0)) * p.inv_h;
    }
    if (threadIdx.x == 0) {
        for (int e = 3 * N; e < p.ev_slab_elems; ++e) {
            if (evg) evg[e] = 0.0;
            if (evl) evl[e] = 0.0;
        }
        if (p.hist_len) *p.hist_len = p.slot + 1;
    }
    NUFI_STAMP(p, 8);
    return true;
}

// E at the nodes: -(N/L) sum over the 3^D f = 0 stencil (w = 1/6, 2/3, 1/6 and
// dw = -1/2, 0, 1/2 on the differentiated axis), taps in x-slowest order, weights
// multiplied in axis order -- the order of the former generic loop, with the
// neighbour indices formed once per node and every loop unrolled (no local memory).
template <int D>
__device__ __forceinline__ void e_at_nodes(const double *c, int N, int nodes, double inv_h, double *E_out) {
    const double w0[3] = {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0};
    const double dw0[3] = {-0.5, 0.0, 0.5};
    for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
        int nb[D][3];
        int r = i;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
            const int ia = r % N;
            r /= N;
            nb[a][0] = ia == 0 ? N - 1 : ia - 1;
            nb[a][1] = ia;
            nb[a][2] = ia == N - 1 ? 0 : ia + 1;
        }
#pragma unroll
        for (int g = 0; g < D; ++g) {
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < (D == 1 ? 3 : (D == 2 ? 9 : 27)); ++t) {
                int o[3] = {t % 3, (t / 3) % 3, t / 9};
                if (o[g] == 1) continue;  // dw = 0 at the centre tap
                int lin = 0;
                double w = 1.0;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    lin = lin * N + nb[a][o[a]];
                    w *= (a == g) ? dw0[o[a]] : w0[o[a]];
                }
                acc = fma(c[lin], w, acc);
            }
            E_out[(size_t)i * D + g] = -acc * inv_h;
        }
    }
}

// The whole tail.  `sm`: field_smem_doubles(nodes, N, rows_per_block > 1) doubles of shared memory
// (B <= 8 when rows_per_block > 1).
__host__ __device__ inline bool field_uses_1d_body(const FieldParams &p) {
    return p.d == 1 && p.gc != nullptr && (p.N & (p.N - 1)) == 0 && p.B <= 8;
}

// WITH_1D = false compiles the generic body only (the d >= 2 tail kernel: without the d = 1
// body's register arrays it fits 1024 threads x 64 registers with no spills)
template <bool WITH_1D = true>
static __device__ __forceinline__ bool field_update_body(const FieldParams &p, double *sm) {
    if constexpr (WITH_1D) {
        if (field_uses_1d_body(p)) return field_update_1d_body(p, sm);
    }
    const int nodes = p.nodes, N = p.N, d = p.d, T = blockDim.x;
    double *re0 = sm, *im0 = re0 + nodes, *re1 = im0 + nodes, *im1 = re1 + nodes;
    double *twc = im1 + nodes, *tws = twc + N, *sb = tws + N;
    double *scratch = sb + (p.rows_per_block > 1 ? 8 * nodes : 0);
    const bool pow2 = (N & (N - 1)) == 0;
    NUFI_STAMP(p, 0);
    for (int m = threadIdx.x; m < N; m += T) {
        twc[m] = p.twc[m];  // tables may live in global or shared memory (generic loads)
        tws[m] = p.tws[m];
    }

    // ---- rho: fixed-order combine of the v-sums (density.py:80-81), neutralise (:84-85) ----
    double neut = 0.0, fmn = 0.0, fmx = 0.0;
    double chk_s = 0.0, chk_m = 0.0;
    if (p.sums) {
        // per-block sums over the block's rows in order (same order as
        // reduce_blocks_kernel), all (block, node) items in parallel, loads batched
        const int rpb = p.rows_per_block;
        if (rpb > 1) {
            for (int it = threadIdx.x; it < p.B * nodes; it += T) {
                const int b = it / nodes, i = it % nodes;
                const double *src = p.sums + (size_t)b * rpb * nodes + i;
                double Sb = 0.0;
                int r = 0;
                for (; r + 8 <= rpb; r += 8) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (size_t)(r + u) * nodes);
#pragma unroll
                    for (int u = 0; u < 8; ++u) Sb += v[u];
                }
                for (; r < rpb; ++r) Sb += __ldcg(src + (size_t)r * nodes);
                sb[it] = Sb;
            }
            __syncthreads();
        }
        NUFI_STAMP(p, 1);
        double local = 0.0;
        if (rpb == 1 && p.B <= 8) {
            // every block sum of 2 nodes requested before any is added (one L2 round trip
            // instead of one per block), then added in block order
            for (int i0 = threadIdx.x; i0 < nodes; i0 += 2 * T) {
                double v[2][8];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int i = i0 + u * T;
#pragma unroll
                    for (int b = 0; b < 8; ++b)
                        v[u][b] = (i < nodes && b < p.B) ? __ldcg(p.sums + (size_t)b * nodes + i) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int i = i0 + u * T;
                    double S = 0.0;
#pragma unroll
                    for (int b = 0; b < 8; ++b)
                        if (b < p.B) S += v[u][b];
                    if (i < nodes) {
                        const double r = p.rho_bar - p.hv_d * S;
                        re1[i] = r;
                        local += r;
                    }
                }
            }
        } else {
            for (int i = threadIdx.x; i < nodes; i += T) {
                double S = 0.0;
                for (int b = 0; b < p.B; ++b) S += rpb > 1 ? sb[b * nodes + i] : __ldcg(p.sums + (size_t)b * nodes + i);
                const double r = p.rho_bar - p.hv_d * S;
                re1[i] = r;
                local += r;
            }
        }
        double mn = DBL_MAX, mx = -DBL_MAX;
        const int mrows = p.B * p.mm_per_block;
        for (int r = threadIdx.x; r < mrows; r += T) {
            mn = fmin(mn, __ldcg(p.minmax + 2 * r));
            mx = fmax(mx, __ldcg(p.minmax + 2 * r + 1));
        }
        double tot;
        cta_sum_min_max(local, mn, mx, scratch, tot, fmn, fmx);
        neut = (nodes & (nodes - 1)) == 0 ? tot * (1.0 / (double)nodes) : tot / (double)nodes;  // exact for 2^k
        for (int i = threadIdx.x; i < nodes; i += T) {
            const double v = re1[i] - neut;
            re0[i] = v;
            im0[i] = 0.0;
            chk_s += v;  // the neutrality check's partials, in its order (poisson.py:97-104)
            chk_m = fmax(chk_m, fabs(v));
        }
    } else {
        for (int i = threadIdx.x; i < nodes; i += T) {
            const double v = p.rho_in[i];
            re0[i] = v;
            im0[i] = 0.0;
            chk_s += v;
            chk_m = fmax(chk_m, fabs(v));
        }
    }
    __syncthreads();
    if (p.rho_out)
        for (int i = threadIdx.x; i < nodes; i += T) p.rho_out[i] = re0[i];
    if (p.stats_out && threadIdx.x == 0) {
        p.stats_out[0] = neut;
        p.stats_out[1] = fmn;
        p.stats_out[2] = fmx;
    }
    if (p.finish_only) return true;
    NUFI_STAMP(p, 2);

    // ---- neutrality check (poisson.py:97-104), partials formed with rho' above ----
    {
        double tot, unused, m;
        cta_sum_min_max(chk_s, DBL_MAX, chk_m, scratch, tot, unused, m);
        const double mean = (nodes & (nodes - 1)) == 0 ? tot * (1.0 / (double)nodes) : tot / (double)nodes;
        const double tol = 1e-8 * m;
        if (fabs(mean) > tol) {
            if (threadIdx.x == 0 && p.status) *p.status = NUFI_ERR_NUMERICAL;
            if (threadIdx.x == 0 && p.hist_len) *p.hist_len = p.slot;  // this slot not appended
            return false;  // history unchanged (the reference raises before appending)
        }
    }

    NUFI_STAMP(p, 3);
    // lanes per DFT output from the grid alone (not the CTA width): fixed summation order
    int G = 1;
    while (G < 32 && 2 * G <= N && (long long)nodes * 2 * G <= 256) G *= 2;

    // ---- forward DFT (poisson.py:77) ----
    double *ar = re0, *ai = im0, *br = re1, *bi = im1;
    for (int axis = d - 1; axis >= 0; --axis) {
        int st = 1;
        for (int a = axis + 1; a < d; ++a) st *= N;
        if (pow2) {
            fft_axis_stockham(ar, ai, br, bi, twc, tws, 31 - __clz(N), nodes, 31 - __clz(st), -1.0);
            continue;  // (ar, ai) already hold the result
        }
        dft_pass(ar, ai, br, bi, twc, tws, N, nodes, st, -1.0, G, pow2);
        double *tr = ar, *ti = ai;
        ar = br, ai = bi, br = tr, bi = ti;
    }
    NUFI_STAMP(p, 4);
    // ---- phi_hat = rho_hat / k^2, Nyquist / zero mode dropped (poisson.py:105-110);
    //      W = L^d/2 sum k^2 |phi_hat|^2 (poisson.py:119-120); coefficient spectrum ----
    double wsum = 0.0;
    for (int e = threadIdx.x; e < nodes; e += T) {
        // fac = 1 / (N^d k^2 prod_a sym(alpha_a)) (0 for the zero / Nyquist modes):
        // (pr, pi) is the coefficient spectrum, (pr, pi) * prod sym is phi_hat
        const double f = p.fac[e], k2 = p.k2[e], sp = p.fac[nodes + e];
        const double pr = ar[e] * f, pi = ai[e] * f;
        ar[e] = pr;
        ai[e] = pi;
        const double hr = pr * sp, hi = pi * sp;
        wsum += k2 * (hr * hr + hi * hi);
    }
    const double W = 0.5 * p.L_d * cta_sum(wsum, scratch);
    if (p.W_out && threadIdx.x == 0) *p.W_out = W;

    NUFI_STAMP(p, 5);
    // ---- inverse DFT (unscaled) -> spline coefficients (spline.py:84 .real) ----
    for (int axis = d - 1; axis >= 0; --axis) {
        int st = 1;
        for (int a = axis + 1; a < d; ++a) st *= N;
        if (pow2) {
            fft_axis_stockham(ar, ai, br, bi, twc, tws, 31 - __clz(N), nodes, 31 - __clz(st), 1.0);
            continue;
        }
        dft_pass(ar, ai, br, bi, twc, tws, N, nodes, st, 1.0, G, pow2);
        double *tr = ar, *ti = ai;
        ar = br, ai = bi, br = tr, bi = ti;
    }
    const double *c = ar;
    NUFI_STAMP(p, 6);

    // ---- append: raw slab + evaluation slab (spline.py:132-142) ----
    if (p.hist) {
        double *hrow = p.hist + (size_t)p.slot * nodes;
        for (int i = threadIdx.x; i < nodes; i += T) {
            hrow[i] = hist_round(c[i], p.f32_hist);
            if (p.coeffs_out) p.coeffs_out[i] = hrow[i];
        }
    }
    double *evg = p.ev_hist ? p.ev_hist + (size_t)p.slot * p.ev_slab_elems : nullptr;
    double *evl = p.ev_local;
    auto put = [&](int e, double v) {
        if (evg) evg[e] = v;
        if (evl) evl[e] = v;
    };
    // slab 0 is only ever used for the final half kick (kernels.py:203-205): store it halved
    const double evs = p.slot == 0 ? 0.5 : 1.0;
    if (d == 1) {
        for (int i = threadIdx.x; i < N; i += T) {
            const double c0 = hist_round(c[(i - 1 + N) % N], p.f32_hist), c1 = hist_round(c[i], p.f32_hist),
                         c2 = hist_round(c[(i + 1) % N], p.f32_hist), c3 = hist_round(c[(i + 2) % N], p.f32_hist);
            double A, Bc, C;
            d1_cell_poly(c0, c1, c2, c3, evs * p.K, A, Bc, C);
            put(d1_ia(i, N), A);
            put(d1_ib(i, N), Bc);
            put(d1_ic(i, N), C);
        }
    } else {
        const int raw = ev_slab_raw_elems(d, N);
        for (int e = threadIdx.x; e < raw; e += T)
            put(e, evs * hist_round(c[p.halo ? p.halo[e] : ev_halo_source(d, N, e)], p.f32_hist));
    }
    for (int e = ev_slab_raw_elems(d, N) + threadIdx.x; e < p.ev_slab_elems; e += T) put(e, 0.0);
    if (threadIdx.x == 0 && p.hist_len) *p.hist_len = p.slot + 1;

    NUFI_STAMP(p, 7);
    // ---- E at the nodes: -grad of the spline at x_i (f = 0 stencil (1/6, 2/3, 1/6) / (-1/2, 0, 1/2)) ----
    if (p.E_out) {
        if (d == 2)
            e_at_nodes<2>(c, N, nodes, p.inv_h, p.E_out);
        else if (d == 3)
            e_at_nodes<3>(c, N, nodes, p.inv_h, p.E_out);
        else
            e_at_nodes<1>(c, N, nodes, p.inv_h, p.E_out);
    }
    NUFI_STAMP(p, 8);
    return true;
}

}  // namespace nufi
