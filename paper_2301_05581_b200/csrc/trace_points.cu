// trace_points.cu -- kernels.trace_backward on caller-provided points, and eval_f0.
//
// Two arithmetic modes:
//   FAST   the production substep of trace_common.cuh, reading the evaluation
//          slabs from global memory (L2-resident history);
//   PARITY the reference's exact operation sequence (kernels.py:153-387: Python
//          float modulo via fmod + sign fix, int() truncation, weights exactly
//          as written, contraction order m -> q -> w, no FMA contraction:
//          __dmul_rn / __dadd_rn), reading the raw coefficient history.  It
//          reproduces the numba kernels' X, V bit for bit.
#include <algorithm>
#include <cstdlib>

#include "trace_common.cuh"

namespace nufi {

// ---- PARITY helpers (kernels.py:153-228), no contraction ----
#define M_(a, b) __dmul_rn((a), (b))
#define A_(a, b) __dadd_rn((a), (b))
#define S_(a, b) __dsub_rn((a), (b))

__device__ __forceinline__ void cell_1d_exact(double x, double L, int N, double inv_h, int &i, double &f) {
    double u = fmod(x, L);  // numba lowers Python float % to fmod + sign fix
    if (u != 0.0) {
        if ((L < 0.0) != (u < 0.0)) u = A_(u, L);
    } else {
        u = copysign(0.0, L);
    }
    if (u >= L || u < 0.0) u = 0.0;  // kernels.py:156-157
    const double t = M_(u, inv_h);
    long long ii = (long long)t;  // int(t): truncation
    if (ii > N - 1) ii = N - 1;
    i = (int)ii;
    f = S_(t, (double)ii);
}

__device__ __forceinline__ void fill_weights_exact(double f, double *w, double *dw) {
    const double s = S_(1.0, f);
    w[0] = __ddiv_rn(M_(M_(s, s), s), 6.0);
    w[1] = S_(2.0 / 3.0, M_(M_(f, f), S_(1.0, M_(0.5, f))));
    w[2] = S_(2.0 / 3.0, M_(M_(s, s), S_(1.0, M_(0.5, s))));
    w[3] = __ddiv_rn(M_(M_(f, f), f), 6.0);
    dw[0] = M_(M_(-0.5, s), s);
    dw[1] = M_(f, S_(M_(1.5, f), 2.0));
    dw[2] = M_(s, S_(2.0, M_(1.5, s)));
    dw[3] = M_(M_(0.5, f), f);
}

__device__ __forceinline__ void stencil_exact(int i, int N, int *idx) {
    idx[0] = i > 0 ? i - 1 : N - 1;
    idx[1] = i;
    idx[2] = i + 1 < N ? i + 1 : i + 1 - N;
    idx[3] = i + 2 < N ? i + 2 : i + 2 - N;
}

template <int D>
__device__ __forceinline__ void E_exact(const double *__restrict__ c, double L, int N, double inv_h, const double *x,
                                        double *E) {
    if constexpr (D == 1) {  // kernels.py:164-182
        int i;
        double f;
        cell_1d_exact(x[0], L, N, inv_h, i, f);
        double w[4], dw[4];
        fill_weights_exact(f, w, dw);
        int idx[4];
        stencil_exact(i, N, idx);
        const double g = A_(A_(A_(M_(c[idx[0]], dw[0]), M_(c[idx[1]], dw[1])), M_(c[idx[2]], dw[2])),
                            M_(c[idx[3]], dw[3]));
        E[0] = M_(-g, inv_h);
    } else if constexpr (D == 2) {  // kernels.py:230-249
        int i, j;
        double f, g;
        double wx[4], dwx[4], wy[4], dwy[4];
        int ix[4], iy[4];
        cell_1d_exact(x[0], L, N, inv_h, i, f);
        fill_weights_exact(f, wx, dwx);
        stencil_exact(i, N, ix);
        cell_1d_exact(x[1], L, N, inv_h, j, g);
        fill_weights_exact(g, wy, dwy);
        stencil_exact(j, N, iy);
        double gx = 0.0, gy = 0.0;
        for (int m = 0; m < 4; ++m) {
            double r = 0.0, rd = 0.0;
            for (int q = 0; q < 4; ++q) {
                const double cc = c[ix[m] * N + iy[q]];
                r = A_(r, M_(cc, wy[q]));
                rd = A_(rd, M_(cc, dwy[q]));
            }
            gx = A_(gx, M_(dwx[m], r));
            gy = A_(gy, M_(wx[m], rd));
        }
        E[0] = M_(-gx, inv_h);
        E[1] = M_(-gy, inv_h);
    } else {  // kernels.py:296-327
        int i, j, l;
        double f, g, h;
        double wx[4], dwx[4], wy[4], dwy[4], wz[4], dwz[4];
        int ix[4], iy[4], iz[4];
        cell_1d_exact(x[0], L, N, inv_h, i, f);
        fill_weights_exact(f, wx, dwx);
        stencil_exact(i, N, ix);
        cell_1d_exact(x[1], L, N, inv_h, j, g);
        fill_weights_exact(g, wy, dwy);
        stencil_exact(j, N, iy);
        cell_1d_exact(x[2], L, N, inv_h, l, h);
        fill_weights_exact(h, wz, dwz);
        stencil_exact(l, N, iz);
        double gx = 0.0, gy = 0.0, gz = 0.0;
        for (int m = 0; m < 4; ++m) {
            double sy = 0.0, sdy = 0.0, sdz = 0.0;
            for (int q = 0; q < 4; ++q) {
                double r = 0.0, rd = 0.0;
                const double *row = c + (ix[m] * N + iy[q]) * N;
                for (int w = 0; w < 4; ++w) {
                    const double cc = row[iz[w]];
                    r = A_(r, M_(cc, wz[w]));
                    rd = A_(rd, M_(cc, dwz[w]));
                }
                sy = A_(sy, M_(wy[q], r));
                sdy = A_(sdy, M_(dwy[q], r));
                sdz = A_(sdz, M_(wy[q], rd));
            }
            gx = A_(gx, M_(dwx[m], sy));
            gy = A_(gy, M_(wx[m], sdy));
            gz = A_(gz, M_(wx[m], sdz));
        }
        E[0] = M_(-gx, inv_h);
        E[1] = M_(-gy, inv_h);
        E[2] = M_(-gz, inv_h);
    }
}

// kernels.py:184-209 / 251-294 / 329-387 on the raw coefficient history.
template <int D>
__global__ void trace_points_parity(const double *__restrict__ hist, int N, int nodes, double L, int n, double tau,
                                    double *X, double *V, int64_t M, int half_kick) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= M) return;
    const double inv_h = (double)N / L;
    const double half = M_(0.5, tau);
    double x[D], v[D], E[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        x[a] = X[p * D + a];
        v[a] = V[p * D + a];
    }
    if (half_kick) {
        E_exact<D>(hist + (size_t)n * nodes, L, N, inv_h, x, E);
#pragma unroll
        for (int a = 0; a < D; ++a) v[a] = A_(v[a], M_(half, E[a]));
    }
    for (int k = n - 1; k >= 1; --k) {
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = S_(x[a], M_(tau, v[a]));
        E_exact<D>(hist + (size_t)k * nodes, L, N, inv_h, x, E);
#pragma unroll
        for (int a = 0; a < D; ++a) v[a] = A_(v[a], M_(tau, E[a]));
    }
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = S_(x[a], M_(tau, v[a]));
    E_exact<D>(hist, L, N, inv_h, x, E);
#pragma unroll
    for (int a = 0; a < D; ++a) {
        v[a] = A_(v[a], M_(half, E[a]));
        X[p * D + a] = x[a];
        V[p * D + a] = v[a];
    }
}


// Production arithmetic on caller points.  The optional leading half kick
// (Psi, flow.py:106-112) uses slab n.
template <int D, bool POW2>
__global__ void trace_points_fast(const double *__restrict__ ev_hist, int ev_slab_elems, int N, double inv_h,
                                  double tau, double K, int n, double *X, double *V, int64_t M, int half_kick) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= M) return;
    const double s_in = tau * inv_h, s_out = 1.0 / s_in, hx = 1.0 / inv_h;
    double Xs[D], Vs[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        Xs[a] = fma(X[p * D + a], inv_h, D == 1 ? -D1_OFF : -0.5);
        Vs[a] = V[p * D + a] * s_in;
    }
    if (half_kick && n > 0) kick<D, POW2>(Xs, Vs, ev_hist + (size_t)n * ev_slab_elems, N, K, true);
    if (n == 0) return;
    // slab 0 is stored pre-halved: the final tau/2 kick needs no special case
    for (int k = n - 1; k >= 0; --k) substep<D, POW2>(Xs, Vs, ev_hist + (size_t)k * ev_slab_elems, N, K, false);
#pragma unroll
    for (int a = 0; a < D; ++a) {
        X[p * D + a] = (Xs[a] + (D == 1 ? D1_OFF : 0.5)) * hx;
        V[p * D + a] = Vs[a] * s_out;
    }
}

// Production arithmetic on caller points with the evaluation slabs staged in a shared-memory
// TMA ring (d >= 2), as in the density kernel: the CTA's 32 * warps * PPT points (PPT
// interleaved per thread) of each pass share one backward stream of slabs n-1 .. 0, instead
// of every thread gathering from L1/L2 (random caller points keep little slab locality
// there).  The optional leading half kick reads slab n in place.  Same substep arithmetic
// as trace_points_fast, so the two agree bit for bit.
template <int D, int PPT, bool POW2, int NX>
__global__ void __launch_bounds__(256, 2)
    trace_points_ring(const double *__restrict__ ev_hist, int slab_elems, int N_, double inv_h, double tau, double K,
                      int n, double *X, double *V, int64_t M, int half_kick, int passes, int sps, int stages) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int N = NX ? NX : N_;
    const int warps = blockDim.x >> 5, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *ring = reinterpret_cast<double *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)stages * sps * slab_elems);
    uint64_t *empty = full + stages;
    const int stages_per_pass = (n + sps - 1) / sps;
    const int total_it = passes * stages_per_pass;
    auto issue = [&](int it) {
        const int st = it % stages_per_pass, s = it % stages;
        const int k_hi = n - 1 - st * sps, k_lo = max(0, k_hi - sps + 1);
        const uint32_t bytes = (uint32_t)((k_hi - k_lo + 1) * slab_elems * sizeof(double));
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_bulk_g2s(ring + (size_t)s * sps * slab_elems, ev_hist + (size_t)k_lo * slab_elems, bytes, &full[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            reinterpret_cast<unsigned *>(&empty[s])[0] = 0u;  // release counter of stage s
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int it = 0; it < min(stages, total_it); ++it) issue(it);
    const double s_in = tau * inv_h, s_out = 1.0 / s_in, hx = 1.0 / inv_h;
    const int64_t per_pass = (int64_t)32 * warps * PPT;
    int it = 0;
    int s = 0;         // ring stage of iteration it and its fill parity, kept incrementally
    uint32_t ph = 0u;  // (no integer division per stage; trace_rho.cu)
    for (int pass = 0; pass < passes; ++pass) {
        const int64_t base = ((int64_t)blockIdx.x * passes + pass) * per_pass + (int64_t)warp * PPT * 32 + lane;
        double Xs[PPT][D], Vs[PPT][D];
#pragma unroll
        for (int pp = 0; pp < PPT; ++pp) {
            const int64_t q = base + pp * 32;
            const int64_t qq = q < M ? q : M - 1;  // the tail CTA's spare lanes trace a copy, never stored
#pragma unroll
            for (int a = 0; a < D; ++a) {
                Xs[pp][a] = fma(X[qq * D + a], inv_h, D == 1 ? -D1_OFF : -0.5);
                Vs[pp][a] = V[qq * D + a] * s_in;
            }
            if (half_kick) kick<D, POW2, NX>(Xs[pp], Vs[pp], ev_hist + (size_t)n * slab_elems, N, K, true);
        }
        for (int st = 0; st < stages_per_pass; ++st, ++it) {
            const int k_hi = n - 1 - st * sps, k_lo = max(0, k_hi - sps + 1);
            mbar_wait(&full[s], ph);
            const double *buf = ring + (size_t)s * sps * slab_elems;
            for (int k = k_hi; k >= k_lo; --k) {
                const double *slab = buf + (size_t)(k - k_lo) * slab_elems;
#pragma unroll
                for (int pp = 0; pp < PPT; ++pp) substep<D, POW2, NX>(Xs[pp], Vs[pp], slab, N, K, false);
            }
            __syncwarp();
            if (lane == 0) {  // the last warp to finish the stage refills it (trace_rho.cu)
                unsigned *cnt = reinterpret_cast<unsigned *>(&empty[s]);
                __threadfence_block();
                if (atomicAdd(cnt, 1u) == (unsigned)warps - 1u) {
                    *cnt = 0u;
                    __threadfence_block();
                    if (it + stages < total_it) {
                        fence_proxy_async_smem();
                        issue(it + stages);
                    }
                }
            }
            if (++s == stages) s = 0, ph ^= 1u;
        }
#pragma unroll
        for (int pp = 0; pp < PPT; ++pp) {
            const int64_t q = base + pp * 32;
            if (q < M)
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    X[q * D + a] = (Xs[pp][a] + (D == 1 ? D1_OFF : 0.5)) * hx;
                    V[q * D + a] = Vs[pp][a] * s_out;
                }
        }
    }
}

// SplineField.eval_phi_many / eval_E_many (spline.py:46-52 -> kernels.py:84-123, the numpy
// twin): _locate (np.mod, u >= L -> 0), bspline_weights / dweights, the 4^d stencil in
// itertools.product order (x tap slowest), phi += c * prod w, E_g -= c * prod (dw on axis
// g, w elsewhere), E *= N / L; elementwise IEEE operations in numpy's order, no FMA.
template <int D>
__device__ __forceinline__ void field_numpy(const double *__restrict__ c, int N, double L, double inv_h,
                                            const double *x, double *phi_out, double *E_out) {
    int i[D];
    double w[D][4], dw[D][4];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double f;
        cell_1d_exact(x[a], L, N, inv_h, i[a], f);
        fill_weights_exact(f, w[a], dw[a]);
    }
    double phi = 0.0, E[D];
#pragma unroll
    for (int g = 0; g < D; ++g) E[g] = 0.0;
    constexpr int TAPS = D == 1 ? 4 : (D == 2 ? 16 : 64);
    for (int t = 0; t < TAPS; ++t) {
        int o[D];
        int r = t;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
            o[a] = r & 3;
            r >>= 2;
        }
        int idx = 0;
        double wp = 1.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            int j = i[a] + o[a] - 1;
            j = j < 0 ? j + N : (j >= N ? j - N : j);
            idx = a == 0 ? j : idx * N + j;
            wp = a == 0 ? w[0][o[0]] : M_(wp, w[a][o[a]]);
        }
        const double cv = c[idx];
        phi = A_(phi, M_(cv, wp));
#pragma unroll
        for (int g = 0; g < D; ++g) {
            double v = cv;
#pragma unroll
            for (int a = 0; a < D; ++a) v = M_(v, a == g ? dw[a][o[a]] : w[a][o[a]]);
            E[g] = S_(E[g], v);
        }
    }
    if (phi_out) *phi_out = phi;
    if (E_out)
#pragma unroll
        for (int g = 0; g < D; ++g) E_out[g] = M_(E[g], inv_h);
}

// kernels.bspline_weights / bspline_dweights (kernels.py:62-81) at M fractions t:
// w[m * M + p], dw[m * M + p] (the reference's (4,) + t.shape layout), numpy's operations.
__global__ void bspline_weights_kernel(const double *__restrict__ t, int64_t M, double *w, double *dw) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= M) return;
    double a[4], b[4];
    fill_weights_exact(t[p], a, b);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        if (w) w[m * M + p] = a[m];
        if (dw) dw[m * M + p] = b[m];
    }
}

cudaError_t launch_bspline_weights(const double *t, int64_t M, double *w, double *dw, cudaStream_t st) {
    const int threads = 256;
    bspline_weights_kernel<<<(unsigned)((M + threads - 1) / threads), threads, 0, st>>>(t, M, w, dw);
    return cudaGetLastError();
}

template <int D>
__global__ void eval_field_kernel(const double *__restrict__ c, int N, double L, const double *__restrict__ X,
                                  int64_t M, double *__restrict__ phi_out, double *__restrict__ E_out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= M) return;
    double x[D];
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = X[p * D + a];
    field_numpy<D>(c, N, L, (double)N / L, x, phi_out ? phi_out + p : nullptr, E_out ? E_out + p * D : nullptr);
}

// The reference's generic trace (flow.py:65-82), used there whenever a non-spline field is
// installed (FlowContext.install_field, flow.py:44-47): numpy operation order --
// V += (0.5 tau) E_n(X) [half kick]; k = n-1 .. 1: X -= tau V, V += tau E_k(X); X -= tau V,
// V += (0.5 tau) E_0(X) -- where E_k is the installed UniformField (spline.py:55-68,
// ovr[4k] != 0, E0 = ovr[4k+1 ..]) or the stored spline's eval_E_many.
template <int D>
__global__ void trace_points_generic(const double *__restrict__ hist, int nodes, const double *__restrict__ ovr,
                                     const double *__restrict__ ovr_slabs, int N, double L, int n, double tau,
                                     double *X, double *V, int64_t M, int half_kick) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= M) return;
    const double inv_h = (double)N / L;
    const double half = M_(0.5, tau);
    double x[D], v[D], E[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        x[a] = X[p * D + a];
        v[a] = V[p * D + a];
    }
    // slot k: ovr[4k] = 0 the stored spline, 1 a UniformField (E0 = ovr[4k+1..]), 2 an
    // installed SplineField (its slab is ovr_slabs row ovr[4k+1])
    auto field = [&](int k) {
        const double kind = ovr[4 * (size_t)k];
        if (kind == 1.0) {
#pragma unroll
            for (int a = 0; a < D; ++a) E[a] = ovr[4 * (size_t)k + 1 + a];
        } else if (kind == 2.0) {
            field_numpy<D>(ovr_slabs + (size_t)ovr[4 * (size_t)k + 1] * nodes, N, L, inv_h, x, nullptr, E);
        } else {
            field_numpy<D>(hist + (size_t)k * nodes, N, L, inv_h, x, nullptr, E);
        }
    };
    if (half_kick) {
        field(n);
#pragma unroll
        for (int a = 0; a < D; ++a) v[a] = A_(v[a], M_(half, E[a]));
    }
    for (int k = n - 1; k >= 1; --k) {
#pragma unroll
        for (int a = 0; a < D; ++a) x[a] = S_(x[a], M_(tau, v[a]));
        field(k);
#pragma unroll
        for (int a = 0; a < D; ++a) v[a] = A_(v[a], M_(tau, E[a]));
    }
#pragma unroll
    for (int a = 0; a < D; ++a) x[a] = S_(x[a], M_(tau, v[a]));
    field(0);
#pragma unroll
    for (int a = 0; a < D; ++a) {
        v[a] = A_(v[a], M_(half, E[a]));
        X[p * D + a] = x[a];
        V[p * D + a] = v[a];
    }
}

#undef M_
#undef A_
#undef S_

cudaError_t launch_eval_field(int d, const double *c, int N, double L, const double *X, int64_t M, double *phi,
                              double *E, cudaStream_t st) {
    const int threads = 128;
    const int ctas = (int)((M + threads - 1) / threads);
    if (d == 1) eval_field_kernel<1><<<ctas, threads, 0, st>>>(c, N, L, X, M, phi, E);
    if (d == 2) eval_field_kernel<2><<<ctas, threads, 0, st>>>(c, N, L, X, M, phi, E);
    if (d == 3) eval_field_kernel<3><<<ctas, threads, 0, st>>>(c, N, L, X, M, phi, E);
    return cudaGetLastError();
}

template <int D>
__global__ void eval_f0_kernel(const F0Params f0, const double *X, const double *V, int64_t M, double *F) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= M) return;
    double x[D], v[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        x[a] = X[p * D + a];
        v[a] = V[p * D + a];
    }
    F[p] = eval_f0<D>(f0, x, v);
}

cudaError_t launch_trace_points(int d, int mode, bool pow2, const double *hist, const double *ev_hist,
                                int ev_slab_elems, int N, int nodes, double L, int n, double tau, double K, double *X,
                                double *V, int64_t M, int half_kick, cudaStream_t st) {
    const int threads = 128;
    const int ctas = (int)((M + threads - 1) / threads);
    const double inv_h = (double)N / L;
    if (mode == NUFI_TRACE_PARITY) {
        if (d == 1) trace_points_parity<1><<<ctas, threads, 0, st>>>(hist, N, nodes, L, n, tau, X, V, M, half_kick);
        if (d == 2) trace_points_parity<2><<<ctas, threads, 0, st>>>(hist, N, nodes, L, n, tau, X, V, M, half_kick);
        if (d == 3) trace_points_parity<3><<<ctas, threads, 0, st>>>(hist, N, nodes, L, n, tau, X, V, M, half_kick);
    } else {
#define NUFI_TP(DD)                                                                                              \
    if (d == DD) {                                                                                               \
        if (pow2)                                                                                                \
            trace_points_fast<DD, true>                                                                          \
                <<<ctas, threads, 0, st>>>(ev_hist, ev_slab_elems, N, inv_h, tau, K, n, X, V, M, half_kick);     \
        else                                                                                                     \
            trace_points_fast<DD, false>                                                                         \
                <<<ctas, threads, 0, st>>>(ev_hist, ev_slab_elems, N, inv_h, tau, K, n, X, V, M, half_kick);     \
    }
        NUFI_TP(1)
        NUFI_TP(2)
        NUFI_TP(3)
#undef NUFI_TP
    }
    return cudaGetLastError();
}

cudaError_t launch_trace_points_generic(int d, const double *hist, int nodes, const double *ovr,
                                        const double *ovr_slabs, int N, double L, int n, double tau, double *X,
                                        double *V, int64_t M, int half_kick, cudaStream_t st) {
    const int threads = 128;
    const int ctas = (int)((M + threads - 1) / threads);
#define NUFI_TPG(DD)                                                                                        \
    if (d == DD)                                                                                            \
        trace_points_generic<DD><<<ctas, threads, 0, st>>>(hist, nodes, ovr, ovr_slabs, N, L, n, tau, X, V, M, \
                                                           half_kick);
    NUFI_TPG(1)
    NUFI_TPG(2)
    NUFI_TPG(3)
#undef NUFI_TPG
    return cudaGetLastError();
}

// d >= 2 FAST trace on caller points through a staged slab ring (trace_points_ring);
// returns cudaErrorNotSupported when the ring would not fit (the caller then uses the
// in-place kernel).
cudaError_t launch_trace_points_ring(int d, bool pow2, const double *ev_hist, int ev_slab_elems, int N, double L,
                                     int n, double tau, double K, double *X, double *V, int64_t M, int half_kick,
                                     cudaStream_t st) {
    if (d < 2 || n < 1) return cudaErrorNotSupported;
    const int threads = 256, ppt = 2, warps = threads / 32;
    const size_t slab_bytes = (size_t)ev_slab_elems * sizeof(double);
    const int sps = std::max<int>(1, (int)(40960 / slab_bytes)), stages = 2;
    const size_t smem = (size_t)stages * sps * slab_bytes + 2 * stages * sizeof(uint64_t);
    if (smem > 110 * 1024) return cudaErrorNotSupported;  // two CTAs per SM, as the density kernel
    const int64_t per_cta_pass = (int64_t)32 * warps * ppt;
    const int64_t chunks = (M + per_cta_pass - 1) / per_cta_pass;
    const int passes = chunks >= 4 * 296 ? 4 : (chunks >= 2 * 296 ? 2 : 1);  // amortise the stream
    const int ctas = (int)((chunks + passes - 1) / passes);
    const double inv_h = (double)N / L;
#define NUFI_TPR(DD, NN, P2)                                                                                 \
    {                                                                                                        \
        auto kern = trace_points_ring<DD, 2, P2, NN>;                                                        \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  \
        if (e != cudaSuccess) return e;                                                                      \
        kern<<<ctas, threads, smem, st>>>(ev_hist, ev_slab_elems, N, inv_h, tau, K, n, X, V, M, half_kick,  \
                                          passes, sps, stages);                                              \
        return cudaGetLastError();                                                                           \
    }
    if (d == 2) {
        if (N == 32) NUFI_TPR(2, 32, true)
        if (pow2) NUFI_TPR(2, 0, true)
        NUFI_TPR(2, 0, false)
    }
    if (N == 16) NUFI_TPR(3, 16, true)
    if (pow2) NUFI_TPR(3, 0, true)
    NUFI_TPR(3, 0, false)
#undef NUFI_TPR
}

cudaError_t launch_eval_f0(int d, const F0Params &f0, const double *X, const double *V, int64_t M, double *F,
                           cudaStream_t st) {
    const int threads = 128;
    const int ctas = (int)((M + threads - 1) / threads);
    if (d == 1) eval_f0_kernel<1><<<ctas, threads, 0, st>>>(f0, X, V, M, F);
    if (d == 2) eval_f0_kernel<2><<<ctas, threads, 0, st>>>(f0, X, V, M, F);
    if (d == 3) eval_f0_kernel<3><<<ctas, threads, 0, st>>>(f0, X, V, M, F);
    return cudaGetLastError();
}

}  // namespace nufi
