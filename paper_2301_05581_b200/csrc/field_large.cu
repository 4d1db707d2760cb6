// field_large.cu -- the per-step tail for grids beyond one CTA (Nx^d > 4096).
//
// Same operations and order of the reference as field_update_body (field_common.cuh):
// combine the block table (density.py:80-85), neutralise, the neutrality check of
// solve_poisson (poisson.py:98-104), the forward transform (poisson.py:72-78), the
// Poisson / spline-filter division (poisson.py:105-110, spline.py:78-84), W
// (poisson.py:115-120), the inverse transform to the coefficient slab (spline.py:84),
// append (spline.py:132-142) and E at the nodes -- split over multi-CTA kernels that
// work in global memory.  Every reduction has a fixed grid and a fixed order, so the
// results are deterministic run to run.
#include <cfloat>

#include "field_common.cuh"

namespace nufi {

constexpr int kLargeThreads = 256;
constexpr int kLargeCtas = 148 * 2;

// fixed-order block reduction of v into out[blockIdx.x] (sum, or max when MAX)
template <bool MAX>
__device__ __forceinline__ void cta_reduce_to(double v, double *out) {
    __shared__ double sh[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, v, o);
        v = MAX ? fmax(v, y) : v + y;
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = sh[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s = MAX ? fmax(s, sh[w]) : s + sh[w];
        out[blockIdx.x] = s;
    }
}

struct LargeParams {
    FieldParams f;
    double *re, *im, *re2, *im2;  // nodes each
    double *part;                 // per-CTA partials: [0, G) sums, [G, 2G) maxima
    double *scal;                 // [0] neut, [1] fmn, [2] fmx
};

// rho = rho_bar - hv^d sum_b S_b (rows_per_block = 1 block table) or the caller's rho
__global__ void large_rho_kernel(LargeParams P) {
    const FieldParams &p = P.f;
    double s = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.nodes; i += gridDim.x * blockDim.x) {
        double r;
        if (p.sums) {
            double S = 0.0;
            for (int b = 0; b < p.B; ++b) S += __ldcg(p.sums + (size_t)b * p.nodes + i);
            r = p.rho_bar - p.hv_d * S;
        } else {
            r = p.rho_in[i];
        }
        P.re2[i] = r;
        s += r;
    }
    cta_reduce_to<false>(s, P.part);
}

// neutralisation constant and (f_min, f_max) from the block table: one CTA
__global__ void large_stats_kernel(LargeParams P, int ctas) {
    const FieldParams &p = P.f;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int c = 0; c < ctas; ++c) s += P.part[c];
        const double neut = p.sums ? s / (double)p.nodes : 0.0;  // density.py:84
        double mn = DBL_MAX, mx = -DBL_MAX;
        if (p.sums)
            for (int q = 0; q < p.B * p.mm_per_block; ++q) {
                mn = fmin(mn, p.minmax[2 * q]);
                mx = fmax(mx, p.minmax[2 * q + 1]);
            }
        P.scal[0] = neut;
        P.scal[1] = mn;
        P.scal[2] = mx;
        if (p.stats_out) {
            p.stats_out[0] = neut;
            p.stats_out[1] = mn;
            p.stats_out[2] = mx;
        }
    }
}

// rho' = rho - neut (density.py:85) -> re, im = 0; partial sums and max|rho'|
__global__ void large_neutral_kernel(LargeParams P, int ctas) {
    const FieldParams &p = P.f;
    const double neut = P.scal[0];
    double s = 0.0, m = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.nodes; i += gridDim.x * blockDim.x) {
        const double v = P.re2[i] - neut;
        P.re[i] = v;
        P.im[i] = 0.0;
        if (p.rho_out) p.rho_out[i] = v;
        s += v;
        m = fmax(m, fabs(v));
    }
    cta_reduce_to<false>(s, P.part);
    __syncthreads();
    cta_reduce_to<true>(m, P.part + ctas);
}

// solve_poisson's neutrality check (poisson.py:98-104): one CTA
__global__ void large_check_kernel(LargeParams P, int ctas) {
    const FieldParams &p = P.f;
    if (threadIdx.x == 0) {
        double s = 0.0, m = 0.0;
        for (int c = 0; c < ctas; ++c) {
            s += P.part[c];
            m = fmax(m, P.part[ctas + c]);
        }
        if (fabs(s / (double)p.nodes) > 1e-8 * m) {
            if (p.status) *p.status = NUFI_ERR_NUMERICAL;
            if (p.hist_len) *p.hist_len = p.slot;  // the device length: this slot not appended
        }
    }
}

__device__ __forceinline__ bool large_failed(const FieldParams &p) {
    return p.status && *(volatile const int *)p.status != 0;
}

// one separable DFT pass along the axis of stride st: out[e] = sum_x in[.. x ..] e^{sign 2 pi i alpha x / N}
__global__ void large_dft_kernel(LargeParams P, const double *ire, const double *iim, double *ore, double *oim,
                                 int st, double sign) {
    const FieldParams &p = P.f;
    if (large_failed(p)) return;
    const int N = p.N;
    const bool pow2 = (N & (N - 1)) == 0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < p.nodes; e += gridDim.x * blockDim.x) {
        const int inner = e % st;
        const int alpha = (e / st) % N;
        const int base = (e / (st * N)) * st * N + inner;
        double re = 0.0, im = 0.0;
        for (int x = 0; x < N; ++x) {
            int m = alpha * x;
            m = pow2 ? (m & (N - 1)) : (m % N);
            const double c = p.twc[m], s = sign * p.tws[m];
            const double xr = ire[base + x * st], xi = iim[base + x * st];
            re = fma(xr, c, fma(-xi, s, re));
            im = fma(xr, s, fma(xi, c, im));
        }
        ore[e] = re;
        oim[e] = im;
    }
}

// coefficient spectrum (the same factors as field_update_body) and the W partials
__global__ void large_spectrum_kernel(LargeParams P, double *ar, double *ai) {
    const FieldParams &p = P.f;
    if (large_failed(p)) return;
    double w = 0.0;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < p.nodes; e += gridDim.x * blockDim.x) {
        const double f = p.fac[e], k2 = p.k2[e], sp = p.fac[p.nodes + e];
        const double pr = ar[e] * f, pi = ai[e] * f;
        ar[e] = pr;
        ai[e] = pi;
        const double hr = pr * sp, hi = pi * sp;
        w += k2 * (hr * hr + hi * hi);
    }
    cta_reduce_to<false>(w, P.part);
}

__global__ void large_energy_kernel(LargeParams P, int ctas) {
    const FieldParams &p = P.f;
    if (large_failed(p)) return;
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int c = 0; c < ctas; ++c) s += P.part[c];
        if (p.W_out) *p.W_out = 0.5 * p.L_d * s;
    }
}

// append: raw slab (+ FP32 rounding), evaluation slab, E at the nodes, history length
__global__ void large_append_kernel(LargeParams P, const double *c) {
    const FieldParams &p = P.f;
    if (large_failed(p)) return;
    const int nodes = p.nodes, N = p.N, d = p.d;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t t0 = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    double *hrow = p.hist ? p.hist + (size_t)p.slot * nodes : nullptr;
    for (size_t i = t0; i < (size_t)nodes; i += stride) {
        const double v = hist_round(c[i], p.f32_hist);
        if (hrow) hrow[i] = v;
        if (p.coeffs_out) p.coeffs_out[i] = v;
    }
    const double evs = p.slot == 0 ? 0.5 : 1.0;
    double *evg = p.ev_hist ? p.ev_hist + (size_t)p.slot * p.ev_slab_elems : nullptr;
    if (evg) {
        if (d == 1) {
            for (size_t ii = t0; ii < (size_t)N; ii += stride) {
                const int i = (int)ii;
                const double c0 = hist_round(c[(i - 1 + N) % N], p.f32_hist), c1 = hist_round(c[i], p.f32_hist),
                             c2 = hist_round(c[(i + 1) % N], p.f32_hist), c3 = hist_round(c[(i + 2) % N], p.f32_hist);
                double A, Bc, C;
                d1_cell_poly(c0, c1, c2, c3, evs * p.K, A, Bc, C);
                evg[d1_ia(i, N)] = A;
                evg[d1_ib(i, N)] = Bc;
                evg[d1_ic(i, N)] = C;
            }
        } else {
            const int raw = ev_slab_raw_elems(d, N);
            for (size_t e = t0; e < (size_t)raw; e += stride)
                evg[e] = evs * hist_round(c[ev_halo_source(d, N, (int)e)], p.f32_hist);
        }
        for (size_t e = ev_slab_raw_elems(d, N) + t0; e < (size_t)p.ev_slab_elems; e += stride) evg[e] = 0.0;
    }
    if (t0 == 0 && p.hist_len) *p.hist_len = p.slot + 1;
    if (p.E_out) {  // -grad of the spline at the nodes (f = 0 stencil), as field_update_body
        const double w0[3] = {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0};
        const double dw0[3] = {-0.5, 0.0, 0.5};
        for (size_t ii = t0; ii < (size_t)nodes; ii += stride) {
            const int i = (int)ii;
            int idx[3] = {0, 0, 0};
            int r = i;
            for (int a = d - 1; a >= 0; --a) {
                idx[a] = r % N;
                r /= N;
            }
            const int taps = d == 1 ? 3 : (d == 2 ? 9 : 27);
            for (int g = 0; g < d; ++g) {
                double acc = 0.0;
                for (int t = 0; t < taps; ++t) {
                    const int o[3] = {t % 3, (t / 3) % 3, t / 9};
                    if (o[g] == 1) continue;
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

// scratch doubles the large tail needs: 4 node arrays + 2G partials + 4 scalars
size_t field_large_scratch_doubles(int nodes) { return 4 * (size_t)nodes + 2 * kLargeCtas + 8; }

cudaError_t launch_field_large(const FieldParams &f, double *scratch, cudaStream_t st) {
    LargeParams P;
    P.f = f;
    const size_t nodes = f.nodes;
    P.re = scratch;
    P.im = P.re + nodes;
    P.re2 = P.im + nodes;
    P.im2 = P.re2 + nodes;
    P.part = P.im2 + nodes;
    P.scal = P.part + 2 * kLargeCtas;
    const int G = kLargeCtas, T = kLargeThreads;
    large_rho_kernel<<<G, T, 0, st>>>(P);
    large_stats_kernel<<<1, 32, 0, st>>>(P, G);
    large_neutral_kernel<<<G, T, 0, st>>>(P, G);
    if (f.finish_only) return cudaGetLastError();
    large_check_kernel<<<1, 32, 0, st>>>(P, G);
    // forward transform (axis d-1 first, like field_update_body), ping-pong re/im <-> re2/im2
    double *ar = P.re, *ai = P.im, *br = P.re2, *bi = P.im2;
    for (int axis = f.d - 1; axis >= 0; --axis) {
        int stv = 1;
        for (int a = axis + 1; a < f.d; ++a) stv *= f.N;
        large_dft_kernel<<<G, T, 0, st>>>(P, ar, ai, br, bi, stv, -1.0);
        double *tr = ar, *ti = ai;
        ar = br, ai = bi, br = tr, bi = ti;
    }
    large_spectrum_kernel<<<G, T, 0, st>>>(P, ar, ai);
    large_energy_kernel<<<1, 32, 0, st>>>(P, G);
    for (int axis = f.d - 1; axis >= 0; --axis) {
        int stv = 1;
        for (int a = axis + 1; a < f.d; ++a) stv *= f.N;
        large_dft_kernel<<<G, T, 0, st>>>(P, ar, ai, br, bi, stv, 1.0);
        double *tr = ar, *ti = ai;
        ar = br, ai = bi, br = tr, bi = ti;
    }
    large_append_kernel<<<G, T, 0, st>>>(P, ar);
    return cudaGetLastError();
}

}  // namespace nufi
