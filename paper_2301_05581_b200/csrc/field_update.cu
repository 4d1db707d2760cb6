// field_update.cu -- the per-step tail kernel (one CTA) and its constant tables.
//
// The routine itself is field_update_body (field_common.cuh); this file holds
// the standalone launch used for d = 2, 3, multi-rank steps and
// nufi_field_update, the per-handle tables, the evaluation-slab builder for
// loaded / appended histories, and the device background density.
#include <cfloat>

#include "field_common.cuh"

namespace nufi {

// WITH_1D: the d = 1 power-of-two tail (CTA width = the d = 1 trace kernel's, <= 544);
// otherwise the generic tail for up to 1024 threads
template <bool WITH_1D>
__global__ void __launch_bounds__(WITH_1D ? 544 : 1024) field_update_kernel(const FieldParams p) {
    extern __shared__ __align__(16) double fsm[];
    // an earlier step of an asynchronously enqueued sequence failed (non-neutral rho):
    // leave the history untouched, like the reference which raises before appending
    if (p.status && *(volatile int *)p.status != 0) {
        mirror_status(p);
        return;
    }
    if (p.wait_flags) {
        __shared__ int failed;
        if (threadIdx.x == 0) {
            failed = 0;
            const unsigned long long t0 = globaltimer_ns();
            for (int q = 0; q < p.wait_G && !failed; ++q) {
                unsigned v;
                for (;;) {
                    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p.wait_flags + q) : "memory");
                    if (v >= p.wait_target) break;
                    if (globaltimer_ns() - t0 > 4000000000ull) {  // 4 s: a peer is gone
                        failed = 1;
                        if (p.wait_error) atomicExch(p.wait_error, 1);
                        if (p.status) atomicExch(p.status, NUFI_ERR_COMM);
                        break;
                    }
                    __nanosleep(NUFI_BARRIER_SLEEP_NS);
                }
            }
        }
        __syncthreads();
        if (failed) {
            mirror_status(p);
            return;
        }
    }
    field_update_body<WITH_1D>(p, fsm);
    mirror_status(p);
}

// The separate reference operations of the step tail, for callers that use them one by
// one (a single CTA, separable smem DFTs as in field_update_body):
//   mode 0  solve_poisson (poisson.py:90-112): neutrality check (status 2, no output),
//           spec = fftn(rho) / N^d / k^2 with the zero and Nyquist modes dropped,
//           phi = Re ifftn(spec * N^d); W = L^d / 2 sum k^2 |spec|^2 (poisson.py:115-120)
//   mode 1  fit_spline (spline.py:71-86): coeffs = Re ifftn(fftn(phi) / prod sym)
//   mode 2  transform_values (poisson.py:72-78): spec = fftn(in) / N^d -> spec_re, spec_im
//   mode 3  inverse_transform (poisson.py:85-87): out = Re ifftn(spec * N^d), spectrum
//           read from in (real part) and spec_im (imaginary part, an INPUT here)
// in: Nx^d reals; out: Nx^d reals; spec_re / spec_im / W optional (mode 0).
__global__ void __launch_bounds__(1024) poisson_fit_kernel(FieldParams p, int mode, const double *in, double *out,
                                                           double *spec_re, double *spec_im, double *W_out,
                                                           int *status) {
    extern __shared__ __align__(16) double fsm[];
    const int nodes = p.nodes, N = p.N, d = p.d, T = blockDim.x;
    double *ar = fsm, *ai = ar + nodes, *br = ai + nodes, *bi = br + nodes;
    double *twc = bi + nodes, *tws = twc + N, *scratch = tws + N;
    const bool pow2 = (N & (N - 1)) == 0;
    for (int m = threadIdx.x; m < N; m += T) {
        twc[m] = p.twc[m];
        tws[m] = p.tws[m];
    }
    double s = 0.0, mx = 0.0;
    for (int i = threadIdx.x; i < nodes; i += T) {
        const double v = in[i];
        ar[i] = v;
        ai[i] = mode == 3 ? spec_im[i] : 0.0;
        s += v;
        mx = fmax(mx, fabs(v));
    }
    if (mode == 0) {  // poisson.py:98-104
        const double mean = cta_sum(s, scratch) / (double)nodes;
        const double tol = 1e-8 * cta_max(mx, scratch);
        if (fabs(mean) > tol) {
            if (threadIdx.x == 0) *status = NUFI_ERR_NUMERICAL;
            return;
        }
    }
    __syncthreads();
    int G = 1;
    while (G < 32 && 2 * G <= N && (long long)nodes * 2 * G <= 256) G *= 2;
    for (int axis = d - 1; axis >= 0 && mode != 3; --axis) {
        int st = 1;
        for (int a = axis + 1; a < d; ++a) st *= N;
        dft_pass(ar, ai, br, bi, twc, tws, N, nodes, st, -1.0, G, pow2);
        double *tr = ar, *ti = ai;
        ar = br, ai = bi, br = tr, bi = ti;
    }
    if (mode == 2) {  // poisson.py:77: fftn(values) / grid.n_nodes
        for (int e = threadIdx.x; e < nodes; e += T) {
            spec_re[e] = ar[e] / (double)nodes;
            spec_im[e] = ai[e] / (double)nodes;
        }
        return;
    }
    double wsum = 0.0;
    for (int e = threadIdx.x; e < nodes && mode != 3; e += T) {
        const double sym = p.fac[nodes + e];
        double f;
        if (mode == 0) {
            f = p.fac[e] * sym;  // 1 / (N^d k^2), 0 at the zero / Nyquist modes
        } else {
            f = 1.0 / ((double)nodes * sym);
        }
        const double pr = ar[e] * f, pi = ai[e] * f;
        ar[e] = pr;
        ai[e] = pi;
        if (mode == 0) {
            if (spec_re) spec_re[e] = pr;
            if (spec_im) spec_im[e] = pi;
            wsum += p.k2[e] * (pr * pr + pi * pi);
        }
    }
    if (mode == 0) {
        const double W = 0.5 * p.L_d * cta_sum(wsum, scratch);
        if (W_out && threadIdx.x == 0) *W_out = W;
    }
    __syncthreads();
    for (int axis = d - 1; axis >= 0; --axis) {
        int st = 1;
        for (int a = axis + 1; a < d; ++a) st *= N;
        dft_pass(ar, ai, br, bi, twc, tws, N, nodes, st, 1.0, G, pow2);
        double *tr = ar, *ti = ai;
        ar = br, ai = bi, br = tr, bi = ti;
    }
    for (int i = threadIdx.x; i < nodes; i += T) out[i] = ar[i];
}

cudaError_t launch_poisson_fit(const FieldParams &p, int mode, const double *in, double *out, double *spec_re,
                               double *spec_im, double *W, int *status, cudaStream_t st) {
    const size_t smem = (4 * (size_t)p.nodes + 2 * p.N + 128) * sizeof(double);  // scratch: cta_sum uses 97
    cudaError_t e = cudaFuncSetAttribute(poisson_fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int threads = p.nodes >= 1024 ? 1024 : (p.nodes >= 128 ? 512 : 256);
    poisson_fit_kernel<<<1, threads, smem, st>>>(p, mode, in, out, spec_re, spec_im, W, status);
    return cudaGetLastError();
}

// d = 1 (field_update_1d_body) stages up to 8 block-sum rows; d = 2, 3 read the block table directly
size_t field_update_smem_bytes(int d, int nodes, int N) {
    return (size_t)field_smem_doubles(nodes, N, d == 1) * sizeof(double);
}

// threads: 0 = by size; d = 1 handles pass their trace-kernel CTA width so every d = 1
// tail (persistent run kernel, fused step kernel, this kernel) runs with the same
// block size -- the CTA-wide reductions then group identically and the results of
// nufi_run, nufi_step and the multi-rank path are bit-identical.
cudaError_t launch_field_update(const FieldParams &p, cudaStream_t st, int threads_req) {
    const size_t smem = field_update_smem_bytes(p.d, p.nodes, p.N);
    const bool d1 = field_uses_1d_body(p);
    auto kern = d1 ? field_update_kernel<true> : field_update_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int threads = threads_req > 0 ? threads_req : (p.nodes >= 1024 ? 1024 : (p.nodes >= 128 ? 512 : 256));
    if (d1 && threads > 544) threads = 544;
    kern<<<1, threads, smem, st>>>(p);
    return cudaGetLastError();
}

// Constant tables of field_common.cuh: tw[0:N] = cos(2 pi m/N), tw[N:2N] = sin;
// fac[e] = 1 / (N^d k^2 prod_a sym(alpha_a)) with k^2 = sum_a (2 pi m_a / L)^2
// (poisson.py:52-59, m = fftfreq) and sym(alpha) = (4 + 2 cos(2 pi alpha / N)) / 6
// (spline.py:20-25); 0 at the zero mode and wherever an axis carries the
// Nyquist mode (poisson.py:62-69, 106-110); fac[nodes + e] = prod_a sym.
__global__ void field_tables_kernel(double *tw, double *fac, double *k2t, int d, int N, int nodes, double k_scale) {
    for (int m = threadIdx.x + blockIdx.x * blockDim.x; m < N; m += blockDim.x * gridDim.x) {
        double s, c;
        sincospi(2.0 * (double)m / (double)N, &s, &c);
        tw[m] = c;
        tw[N + m] = s;
    }
    for (int e = threadIdx.x + blockIdx.x * blockDim.x; e < nodes; e += blockDim.x * gridDim.x) {
        double k2 = 0.0, symp = 1.0;
        bool nyq = false;
        int r = e;
        for (int a = d - 1; a >= 0; --a) {
            const int alpha = r % N;
            r /= N;
            const int m = alpha < (N + 1) / 2 ? alpha : alpha - N;
            const double km = k_scale * (double)m;
            k2 += km * km;
            if ((N % 2 == 0) && (m == -N / 2)) nyq = true;
            symp *= (4.0 + 2.0 * cospi(2.0 * (double)alpha / (double)N)) / 6.0;
        }
        k2t[e] = k2;
        fac[e] = (k2 > 0.0 && !nyq) ? 1.0 / ((double)nodes * k2 * symp) : 0.0;
        fac[nodes + e] = symp;
    }
}

// d = 1 circulant kernels: gc[m] = sum_alpha fac[alpha] cos(2 pi alpha m / N)
// (coefficients, spline.py:78-84 o poisson.py:105-110) and
// gp[m] = sum_alpha fac[alpha] sym[alpha] cos(2 pi alpha m / N) (nodal potential,
// poisson.py:85-87); fac already carries the 1/N of the inverse transform.
// (grids too large for the staged tables below: the same values, formed per tap)
__global__ void field_conv_kernels_direct(const double *fac, double *gc, double *gp, int N) {
    for (int m = threadIdx.x + blockIdx.x * blockDim.x; m < N; m += blockDim.x * gridDim.x) {
        double a = 0.0, b = 0.0;
        for (int al = 0; al < N; ++al) {
            const double cs = cospi(2.0 * (double)(((int64_t)al * m) % N) / (double)N);
            a = fma(fac[al], cs, a);
            b = fma(fac[al] * fac[N + al], cs, b);
        }
        gc[m] = a;
        gp[m] = b;
    }
}

__global__ void field_conv_kernels_kernel(const double *fac, double *gc, double *gp, int N) {
    // the N distinct cosines, fac and fac * sym staged once (the values and the summation
    // order of the direct form: one cospi per (alpha, m) and an integer modulo per tap
    // made this ~28 us per handle); (alpha m) mod N advanced incrementally
    extern __shared__ double tab[];
    double *cs = tab, *f1 = tab + N, *f2 = tab + 2 * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        cs[j] = cospi(2.0 * (double)j / (double)N);
        f1[j] = fac[j];
        f2[j] = fac[j] * fac[N + j];
    }
    __syncthreads();
    for (int m = threadIdx.x + blockIdx.x * blockDim.x; m < N; m += blockDim.x * gridDim.x) {
        double a = 0.0, b = 0.0;
        int idx = 0;  // (al * m) % N
        for (int al = 0; al < N; ++al) {
            a = fma(f1[al], cs[idx], a);
            b = fma(f2[al], cs[idx], b);
            idx += m;
            if (idx >= N) idx -= N;
        }
        gc[m] = a;
        gp[m] = b;
    }
}

cudaError_t launch_field_tables(double *tw, double *fac, double *k2, int d, int N, int nodes, double k_scale,
                                cudaStream_t st) {
    field_tables_kernel<<<8, 256, 0, st>>>(tw, fac, k2, d, N, nodes, k_scale);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || d != 1) return e;
    // d = 1: gc, gp follow k2 in the table buffer
    const size_t smem = 3 * (size_t)N * sizeof(double);
    if (smem > 200 * 1024) {
        field_conv_kernels_direct<<<(N + 255) / 256, 256, 0, st>>>(fac, k2 + nodes, k2 + nodes + N, N);
        return cudaGetLastError();
    }
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(field_conv_kernels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    field_conv_kernels_kernel<<<1, 256, smem, st>>>(fac, k2 + nodes, k2 + nodes + N, N);
    return cudaGetLastError();
}

// d >= 2: the halo source index of every evaluation-slab element, once per handle
__global__ void halo_table_kernel(int d, int N, int raw, int *halo) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < raw; e += gridDim.x * blockDim.x)
        halo[e] = ev_halo_source(d, N, e);
}

cudaError_t launch_halo_table(int d, int N, int *halo, cudaStream_t st) {
    const int raw = ev_slab_raw_elems(d, N);
    halo_table_kernel<<<(raw + 255) / 256 < 1024 ? (raw + 255) / 256 : 1024, 256, 0, st>>>(d, N, raw, halo);
    return cudaGetLastError();
}

// Evaluation slabs (trace_common.cuh layouts) for raw rows [r0, r1) of hist.
// f32: FP32 history mode -- round the raw row in place first (spline.py:118-125, 140).
__global__ void build_ev_slabs_kernel(double *__restrict__ hist, double *__restrict__ ev_hist, int d, int N,
                                      int nodes, int ev_slab_elems, double K, int64_t r0, int f32) {
    const int64_t slot = r0 + blockIdx.x;
    double *c = hist + (size_t)slot * nodes;
    if (f32) {
        for (int i = threadIdx.x; i < nodes; i += blockDim.x) c[i] = hist_round(c[i], 1);
        __syncthreads();
    }
    double *ev = ev_hist + (size_t)slot * ev_slab_elems;
    const double evs = slot == 0 ? 0.5 : 1.0;  // slab 0 stored pre-halved (field_common.cuh)
    if (d == 1) {
        K *= evs;
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const double c0 = c[(i - 1 + N) % N], c1 = c[i], c2 = c[(i + 1) % N], c3 = c[(i + 2) % N];
            double A, Bc, C;
            d1_cell_poly(c0, c1, c2, c3, K, A, Bc, C);
            ev[d1_ia(i, N)] = A;
            ev[d1_ib(i, N)] = Bc;
            ev[d1_ic(i, N)] = C;
        }
    } else {
        const int raw = ev_slab_raw_elems(d, N);
        for (int e = threadIdx.x; e < raw; e += blockDim.x) ev[e] = evs * c[ev_halo_source(d, N, e)];
    }
    for (int e = ev_slab_raw_elems(d, N) + threadIdx.x; e < ev_slab_elems; e += blockDim.x) ev[e] = 0.0;
}

cudaError_t launch_build_ev_slabs(double *hist, double *ev_hist, int d, int N, int nodes, int ev_slab_elems,
                                  double K, int64_t r0, int64_t r1, int f32, cudaStream_t st) {
    if (r1 <= r0) return cudaSuccess;
    build_ev_slabs_kernel<<<(unsigned)(r1 - r0), 256, 0, st>>>(hist, ev_hist, d, N, nodes, ev_slab_elems, K, r0, f32);
    return cudaGetLastError();
}

// ---- background density on the device (initial.py:187-208) ----
// sum_v over the Nv^d velocity grid of prod_a factor_a(v_a), sum_x over the
// Nx^d nodes of 1 + alpha * sum_a cos(k x_a); rho_bar = sum_x*sum_v*hx^d*hv^d / L^d.


__global__ void __launch_bounds__(1024) rho_bar_kernel(const RhoBarParams p) {
    __shared__ double scratch[128];  // cta_sum: 32 warp slots + result slot 96
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
    const double sum_v = cta_sum(sv, scratch);
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
    const double sum_x = cta_sum(sx, scratch);
    if (threadIdx.x == 0) *p.out = sum_x * sum_v * p.hx_d * p.hv_d / p.L_d;
}

cudaError_t launch_rho_bar(const RhoBarParams &p, cudaStream_t st) {
    rho_bar_kernel<<<1, 1024, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace nufi
