// field_update.cu -- the per-step tail of the NuFI loop on one CTA.
//
// Replaces, per step:
//   density.compute_rho's combine + neutralisation   density.py:80-85
//   poisson.solve_poisson                             poisson.py:90-112
//   spline.fit_spline                                 spline.py:71-86
//   PotentialHistory.append                           spline.py:132-142
//   poisson.electric_energy                           poisson.py:115-120
//   E at the nodes (SplineField.eval_E_many)          spline.py:50-52, kernels.py:102-123
// The spectral steps are separable shared-memory DFTs (Nx^d <= 4096, exact
// integer twiddle indices).  fit_spline's forward FFT of phi is fused away: for
// real rho the spectrum of phi is phi_hat * N^d, so the coefficient slab is
// Re IDFT(phi_hat / prod_a sym(alpha_a)) (same maths as poisson.py:85-87 then
// spline.py:78-84, one transform pair instead of two).
//
// Outputs: coefficient slab -> hist[n], evaluation slab -> ev_hist[n]
// (layouts in trace_common.cuh), rho, W, E, stats, status.
#include <cfloat>

#include "trace_common.cuh"

namespace nufi {



// block-wide fixed-order sum (deterministic for a fixed blockDim)
__device__ double block_sum(double v, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += scratch[w];
    __syncthreads();
    return s;
}

__device__ double block_max(double v, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double s = -DBL_MAX;
    for (int w = 0; w < nw; ++w) s = fmax(s, scratch[w]);
    __syncthreads();
    return s;
}

// One separable DFT pass along `axis` (stride st): out = sum_x in[x] e^{sign i 2 pi alpha x / N}
__device__ void dft_pass(const double *__restrict__ ire, const double *__restrict__ iim, double *__restrict__ ore,
                         double *__restrict__ oim, const double *__restrict__ twc, const double *__restrict__ tws,
                         int N, int nodes, int st, double sign, bool pow2) {
    for (int e = threadIdx.x; e < nodes; e += blockDim.x) {
        const int inner = e % st;
        const int alpha = (e / st) % N;
        const int base = (e / (st * N)) * st * N + inner;
        double re = 0.0, im = 0.0;
        for (int x = 0; x < N; ++x) {
            int m = alpha * x;
            m = pow2 ? (m & (N - 1)) : (m % N);
            const double c = twc[m], s = sign * tws[m];
            const double xr = ire[base + x * st], xi = iim[base + x * st];
            re = fma(xr, c, fma(-xi, s, re));
            im = fma(xr, s, fma(xi, c, im));
        }
        ore[e] = re;
        oim[e] = im;
    }
    __syncthreads();
}

__device__ __forceinline__ int fftfreq(int alpha, int N) { return alpha < (N + 1) / 2 ? alpha : alpha - N; }

// dynamic smem: re0, im0, re1, im1 (nodes each), twc, tws (N each), scratch (32)
__global__ void __launch_bounds__(1024) field_update_kernel(const FieldParams p) {
    extern __shared__ __align__(16) double fsm[];
    const int nodes = p.nodes, N = p.N, d = p.d;
    double *re0 = fsm, *im0 = re0 + nodes, *re1 = im0 + nodes, *im1 = re1 + nodes;
    double *twc = im1 + nodes, *tws = twc + N, *scratch = tws + N;
    const bool pow2 = (N & (N - 1)) == 0;

    for (int m = threadIdx.x; m < N; m += blockDim.x) {
        double s, c;
        sincospi(2.0 * (double)m / (double)N, &s, &c);
        twc[m] = c;
        tws[m] = s;
    }

    // ---- rho: fixed-order combine of the v-block sums, then neutralise ----
    double neut = 0.0, fmn = 0.0, fmx = 0.0;
    if (p.partials) {
        double local = 0.0;
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
            double S = 0.0;
            for (int b = 0; b < p.B; ++b) S += p.partials[(size_t)b * nodes + i];
            const double r = p.rho_bar - p.hv_d * S;  // density.py:81
            re1[i] = r;
            local += r;
        }
        neut = block_sum(local, scratch) / (double)nodes;  // density.py:84 rho.mean()
        fmn = DBL_MAX;
        fmx = -DBL_MAX;
        const double *mm = p.partials + (size_t)p.B * nodes;
        for (int b = 0; b < p.B; ++b) {
            fmn = fmin(fmn, mm[2 * b]);
            fmx = fmax(fmx, mm[2 * b + 1]);
        }
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
            re0[i] = re1[i] - neut;  // density.py:85
            im0[i] = 0.0;
        }
    } else {
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
            re0[i] = p.rho_in[i];
            im0[i] = 0.0;
        }
    }
    __syncthreads();

    if (p.rho_out)
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) p.rho_out[i] = re0[i];
    if (p.stats_out && threadIdx.x == 0) {
        p.stats_out[0] = neut;
        p.stats_out[1] = fmn;
        p.stats_out[2] = fmx;
    }
    if (p.finish_only) return;
    // ---- neutrality check (poisson.py:97-104) ----
    {
        double s = 0.0, mx = 0.0;
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
            s += re0[i];
            mx = fmax(mx, fabs(re0[i]));
        }
        const double mean = block_sum(s, scratch) / (double)nodes;
        const double tol = 1e-8 * block_max(mx, scratch);
        if (fabs(mean) > tol) {
            if (threadIdx.x == 0) *p.status = NUFI_ERR_NUMERICAL;
            return;  // history unchanged (the reference raises before appending)
        }
    }

    // ---- forward DFT of rho over every axis (poisson.py:77) ----
    double *ar = re0, *ai = im0, *br = re1, *bi = im1;
    for (int axis = d - 1; axis >= 0; --axis) {
        int st = 1;
        for (int a = axis + 1; a < d; ++a) st *= N;
        dft_pass(ar, ai, br, bi, twc, tws, N, nodes, st, -1.0, pow2);
        double *tr = ar, *ti = ai;
        ar = br;
        ai = bi;
        br = tr;
        bi = ti;
    }
    // spectrum in (ar, ai); phi_hat = rho_hat / k^2 (poisson.py:105-110), energy, coefficient spectrum
    double wsum = 0.0;
    const double inv_nodes = 1.0 / (double)nodes;
    for (int e = threadIdx.x; e < nodes; e += blockDim.x) {
        double k2 = 0.0, symp = 1.0;
        bool nyq = false;
        int r = e;
        for (int a = d - 1; a >= 0; --a) {
            const int alpha = r % N;
            r /= N;
            const int m = fftfreq(alpha, N);
            const double km = p.k_scale * (double)m;
            k2 += km * km;
            if ((N % 2 == 0) && (m == N / 2 || m == -N / 2)) nyq = true;
            symp *= (4.0 + 2.0 * cospi(2.0 * (double)alpha / (double)N)) / 6.0;  // spline.py:20-25
        }
        double pr = 0.0, pi = 0.0;
        if (k2 > 0.0 && !nyq) {
            pr = ar[e] * inv_nodes / k2;
            pi = ai[e] * inv_nodes / k2;
        }
        wsum += k2 * (pr * pr + pi * pi);  // poisson.py:119
        ar[e] = pr / symp;
        ai[e] = pi / symp;
    }
    const double W = 0.5 * p.L_d * block_sum(wsum, scratch);  // poisson.py:120
    if (p.W_out && threadIdx.x == 0) *p.W_out = W;

    // ---- inverse DFT (unscaled) -> spline coefficients (real part) ----
    for (int axis = d - 1; axis >= 0; --axis) {
        int st = 1;
        for (int a = axis + 1; a < d; ++a) st *= N;
        dft_pass(ar, ai, br, bi, twc, tws, N, nodes, st, 1.0, pow2);
        double *tr = ar, *ti = ai;
        ar = br;
        ai = bi;
        br = tr;
        bi = ti;
    }
    const double *c = ar;  // coefficient slab (Nx,)*d row-major

    // ---- append: raw slab, evaluation slab (spline.py:132-142) ----
    double *hrow = p.hist + (size_t)p.slot * nodes;
    for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
        hrow[i] = c[i];
        if (p.coeffs_out) p.coeffs_out[i] = c[i];
    }
    double *ev = p.ev_hist + (size_t)p.slot * p.ev_slab_elems;
    if (d == 1) {
        // cell i, centred fc: kick = K * g(fc + 1/2), g = sum_taps c * dw  (kernels.py:164-182)
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const double c0 = c[(i - 1 + N) % N], c1 = c[i], c2 = c[(i + 1) % N], c3 = c[(i + 2) % N];
            const double g0 = 0.5 * (c2 - c0);
            const double g1 = (c0 - 2.0 * c1) + c2;
            const double g2 = (1.5 * (c1 - c2)) + 0.5 * (c3 - c0);
            ev[i] = p.K * ((g0 + 0.5 * g1) + 0.25 * g2);
            ev[N + i] = p.K * (g1 + g2);
            ev[2 * N + i] = p.K * g2;
        }
    } else {
        const int row = N + 3;
        const int rows = nodes / N;
        for (int e = threadIdx.x; e < rows * row; e += blockDim.x) {
            const int r = e / row, j = e % row;
            ev[e] = c[r * N + (j - 1 + N) % N];
        }
    }
    if (threadIdx.x == 0) {
        const int raw = ev_slab_raw_elems(d, N);
        for (int e = raw; e < p.ev_slab_elems; ++e) ev[e] = 0.0;
        if (p.hist_len) *p.hist_len = p.slot + 1;
    }

    // ---- E at the nodes: -grad of the spline at x_i (f = 0 stencil) ----
    if (p.E_out) {
        const double w0[3] = {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0};
        const double dw0[3] = {-0.5, 0.0, 0.5};
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) {
            int idx[3] = {0, 0, 0};
            {
                int r = i;
                for (int a = d - 1; a >= 0; --a) {
                    idx[a] = r % N;
                    r /= N;
                }
            }
            for (int g = 0; g < d; ++g) {
                double acc = 0.0;
                const int taps = d == 1 ? 3 : (d == 2 ? 9 : 27);
                for (int t = 0; t < taps; ++t) {
                    int o[3] = {t % 3, (t / 3) % 3, t / 9};
                    int lin = 0;
                    double w = 1.0;
                    for (int a = 0; a < d; ++a) {
                        lin = lin * N + (idx[a] + o[a] - 1 + N) % N;
                        w *= (a == g) ? dw0[o[a]] : w0[o[a]];
                    }
                    acc = fma(c[lin], w, acc);
                }
                p.E_out[(size_t)i * d + g] = -acc * p.inv_h;
            }
        }
    }
}

// Evaluation slabs (trace_common.cuh layouts) for raw rows [r0, r1) of hist.
__global__ void build_ev_slabs_kernel(const double *__restrict__ hist, double *__restrict__ ev_hist, int d, int N,
                                      int nodes, int ev_slab_elems, double K, int64_t r0) {
    const int64_t slot = r0 + blockIdx.x;
    const double *c = hist + (size_t)slot * nodes;
    double *ev = ev_hist + (size_t)slot * ev_slab_elems;
    if (d == 1) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const double c0 = c[(i - 1 + N) % N], c1 = c[i], c2 = c[(i + 1) % N], c3 = c[(i + 2) % N];
            const double g0 = 0.5 * (c2 - c0);
            const double g1 = (c0 - 2.0 * c1) + c2;
            const double g2 = (1.5 * (c1 - c2)) + 0.5 * (c3 - c0);
            ev[i] = K * ((g0 + 0.5 * g1) + 0.25 * g2);
            ev[N + i] = K * (g1 + g2);
            ev[2 * N + i] = K * g2;
        }
    } else {
        const int row = N + 3;
        const int rows = nodes / N;
        for (int e = threadIdx.x; e < rows * row; e += blockDim.x) {
            const int r = e / row, j = e % row;
            ev[e] = c[r * N + (j - 1 + N) % N];
        }
    }
    for (int e = ev_slab_raw_elems(d, N) + threadIdx.x; e < ev_slab_elems; e += blockDim.x) ev[e] = 0.0;
}

cudaError_t launch_build_ev_slabs(const double *hist, double *ev_hist, int d, int N, int nodes, int ev_slab_elems,
                                  double K, int64_t r0, int64_t r1, cudaStream_t st) {
    if (r1 <= r0) return cudaSuccess;
    build_ev_slabs_kernel<<<(unsigned)(r1 - r0), 256, 0, st>>>(hist, ev_hist, d, N, nodes, ev_slab_elems, K, r0);
    return cudaGetLastError();
}

size_t field_update_smem_bytes(int nodes, int N) { return (4 * (size_t)nodes + 2 * N + 32) * sizeof(double); }

cudaError_t launch_field_update(const FieldParams &p, cudaStream_t st) {
    const size_t smem = field_update_smem_bytes(p.nodes, p.N);
    cudaError_t e = cudaFuncSetAttribute(field_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int threads = p.nodes >= 1024 ? 1024 : (p.nodes >= 256 ? 256 : 128);
    field_update_kernel<<<1, threads, smem, st>>>(p);
    return cudaGetLastError();
}

// ---- background density on the device (initial.py:187-208) ----
// sum_v over the Nv^d velocity grid of prod_a factor_a(v_a), sum_x over the
// Nx^d nodes of 1 + alpha * sum_a cos(k x_a); rho_bar = sum_x*sum_v*hx^d*hv^d / L^d.


__global__ void __launch_bounds__(1024) rho_bar_kernel(const RhoBarParams p) {
    __shared__ double scratch[32];
    int64_t V = 1, X = 1;
    for (int a = 0; a < p.d; ++a) {
        V *= p.Nv;
        X *= p.N;
    }
    double sv = 0.0;
    for (int64_t j = threadIdx.x; j < V; j += blockDim.x) {
        int64_t r = j;
        double vel = 1.0;
        for (int a = p.d - 1; a >= 0; --a) {
            const int ja = (int)(r % p.Nv);
            r /= p.Nv;
            const double v = __dadd_rn(-p.vmax, __dmul_rn((double)ja + 0.5, p.hv));
            double acc = 0.0;
            for (int m = 0; m < p.f0.n_centers[a]; ++m) {
                const double t = v - p.f0.centers[a][m];
                acc += p.f0.weights[a][m] * exp(-0.5 * (t * t));
            }
            acc *= GAUSS_NORM;
            if (p.f0.power[a]) acc = acc * (v * v);
            vel *= acc;
        }
        sv += vel;
    }
    const double sum_v = block_sum(sv, scratch);
    double sx = 0.0;
    for (int64_t i = threadIdx.x; i < X; i += blockDim.x) {
        int64_t r = i;
        double pert = 0.0;
        for (int a = p.d - 1; a >= 0; --a) {
            const int ia = (int)(r % p.N);
            r /= p.N;
            pert += cos(p.f0.k * __dmul_rn((double)ia, p.hx));
        }
        sx += 1.0 + p.f0.alpha * pert;
    }
    const double sum_x = block_sum(sx, scratch);
    if (threadIdx.x == 0) *p.out = sum_x * sum_v * p.hx_d * p.hv_d / p.L_d;
}

cudaError_t launch_rho_bar(const RhoBarParams &p, cudaStream_t st) {
    rho_bar_kernel<<<1, 1024, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace nufi
