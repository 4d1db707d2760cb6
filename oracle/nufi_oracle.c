/*
 * nufi_oracle.c -- CPU restatement of the reference's backward-trace kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker (or the timed CPU baseline), never as the product path.
 *
 * Restates, operation for operation, the numba kernels of the reference
 * (/root/reference/pkg/src/vpflow/kernels.py):
 *   _cell_1d      kernels.py:153-162   (Python float % -> fmod + sign fix)
 *   _E_1d         kernels.py:164-182
 *   _trace_1d     kernels.py:184-209
 *   _fill_weights kernels.py:211-221
 *   _stencil_1d   kernels.py:223-228
 *   _E_2d         kernels.py:230-249,  _trace_2d kernels.py:251-294
 *   _E_3d         kernels.py:296-327,  _trace_3d kernels.py:329-387
 * numba emits no FMA, so this file is compiled with
 * -ffp-contract=off and keeps the reference's left-to-right evaluation order;
 * it then reproduces trace_backward's X, V bit for bit (pinned by
 * tests/test_oracle.py against tests/golden/trace_*.npz).
 *
 * Points are independent, so the OpenMP split over points does not change any
 * result bit (same as the reference's numba prange, kernels.py:190,257,335).
 */
#include <math.h>
#include <stdint.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* Python float modulo as numba lowers it: fmod, then move into the sign of L. */
static inline double py_mod(double x, double L) {
    double m = fmod(x, L);
    if (m != 0.0) {
        if ((L < 0.0) != (m < 0.0)) m += L;
    } else {
        m = copysign(0.0, L);
    }
    return m;
}

/* kernels.py:153-162 */
static inline void cell_1d(double x, double L, int64_t N, double inv_h, int64_t *i, double *f) {
    double u = py_mod(x, L);
    if (u >= L || u < 0.0) u = 0.0;
    double t = u * inv_h;
    int64_t ii = (int64_t)t;
    if (ii > N - 1) ii = N - 1;
    *i = ii;
    *f = t - (double)ii;
}

/* kernels.py:164-182 */
static inline double E_1d(const double *c, double L, int64_t N, double inv_h, double x) {
    int64_t i;
    double f;
    cell_1d(x, L, N, inv_h, &i, &f);
    double s = 1.0 - f;
    double dw0 = -0.5 * s * s;
    double dw1 = f * (1.5 * f - 2.0);
    double dw2 = s * (2.0 - 1.5 * s);
    double dw3 = 0.5 * f * f;
    int64_t im = i - 1;
    if (im < 0) im += N;
    int64_t i1 = i + 1;
    if (i1 >= N) i1 -= N;
    int64_t i2 = i + 2;
    if (i2 >= N) i2 -= N;
    double g = c[im] * dw0 + c[i] * dw1 + c[i1] * dw2 + c[i2] * dw3;
    return -g * inv_h;
}

/* kernels.py:211-221 */
static inline void fill_weights(double f, double *w, double *dw) {
    double s = 1.0 - f;
    w[0] = s * s * s / 6.0;
    w[1] = 2.0 / 3.0 - f * f * (1.0 - 0.5 * f);
    w[2] = 2.0 / 3.0 - s * s * (1.0 - 0.5 * s);
    w[3] = f * f * f / 6.0;
    dw[0] = -0.5 * s * s;
    dw[1] = f * (1.5 * f - 2.0);
    dw[2] = s * (2.0 - 1.5 * s);
    dw[3] = 0.5 * f * f;
}

/* kernels.py:223-228 */
static inline void stencil_1d(int64_t i, int64_t N, int64_t *idx) {
    idx[0] = i > 0 ? i - 1 : N - 1;
    idx[1] = i;
    idx[2] = i + 1 < N ? i + 1 : i + 1 - N;
    idx[3] = i + 2 < N ? i + 2 : i + 2 - N;
}

/* kernels.py:230-249 (c points at slab k, row-major (N, N)) */
static inline void E_2d(const double *c, double L, int64_t N, double inv_h, double x, double y,
                        double *ex, double *ey) {
    double wx[4], dwx[4], wy[4], dwy[4];
    int64_t ix[4], iy[4];
    int64_t i, j;
    double f, g;
    cell_1d(x, L, N, inv_h, &i, &f);
    fill_weights(f, wx, dwx);
    stencil_1d(i, N, ix);
    cell_1d(y, L, N, inv_h, &j, &g);
    fill_weights(g, wy, dwy);
    stencil_1d(j, N, iy);
    double gx = 0.0, gy = 0.0;
    for (int m = 0; m < 4; ++m) {
        double r = 0.0, rd = 0.0;
        for (int q = 0; q < 4; ++q) {
            double cc = c[ix[m] * N + iy[q]];
            r += cc * wy[q];
            rd += cc * dwy[q];
        }
        gx += dwx[m] * r;
        gy += wx[m] * rd;
    }
    *ex = -gx * inv_h;
    *ey = -gy * inv_h;
}

/* kernels.py:296-327 */
static inline void E_3d(const double *c, double L, int64_t N, double inv_h, double x, double y,
                        double z, double *ex, double *ey, double *ez) {
    double wx[4], dwx[4], wy[4], dwy[4], wz[4], dwz[4];
    int64_t ix[4], iy[4], iz[4];
    int64_t i, j, l;
    double f, g, h;
    cell_1d(x, L, N, inv_h, &i, &f);
    fill_weights(f, wx, dwx);
    stencil_1d(i, N, ix);
    cell_1d(y, L, N, inv_h, &j, &g);
    fill_weights(g, wy, dwy);
    stencil_1d(j, N, iy);
    cell_1d(z, L, N, inv_h, &l, &h);
    fill_weights(h, wz, dwz);
    stencil_1d(l, N, iz);
    double gx = 0.0, gy = 0.0, gz = 0.0;
    for (int m = 0; m < 4; ++m) {
        double sy = 0.0, sdy = 0.0, sdz = 0.0;
        for (int q = 0; q < 4; ++q) {
            double r = 0.0, rd = 0.0;
            const double *row = c + (ix[m] * N + iy[q]) * N;
            for (int w = 0; w < 4; ++w) {
                double cc = row[iz[w]];
                r += cc * wz[w];
                rd += cc * dwz[w];
            }
            sy += wy[q] * r;
            sdy += dwy[q] * r;
            sdz += wy[q] * rd;
        }
        gx += dwx[m] * sy;
        gy += wx[m] * sdy;
        gz += wx[m] * sdz;
    }
    *ex = -gx * inv_h;
    *ey = -gy * inv_h;
    *ez = -gz * inv_h;
}

/*
 * oracle_trace: kernels.py:390-412 semantics for d = 1, 2, 3.
 * coeffs: (rows, N^d) row-major; X, V: (M, d) row-major, mutated in place.
 * Returns the number of field evaluations (kernels.py:193-209 `cnt`), or -1
 * when the history is too short (trace_backward raises UsageError there).
 */
int64_t oracle_trace(const double *coeffs, int64_t rows, int d, int64_t N, double L, int64_t n,
                     double tau, double *X, double *V, int64_t M, int half_kick, int threads) {
    if (n == 0) return 0;
    int64_t need = half_kick ? n + 1 : n;
    if (rows < need) return -1;
    if (M == 0) return 0;
    const double inv_h = (double)N / L;
    const double half = 0.5 * tau;
    int64_t slab = N;
    if (d >= 2) slab *= N;
    if (d == 3) slab *= N;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#else
    (void)threads;
#endif
    if (d == 1) {
#pragma omp parallel for schedule(static) num_threads(threads)
        for (int64_t p = 0; p < M; ++p) {
            double x = X[p], v = V[p];
            if (half_kick) v += half * E_1d(coeffs + n * slab, L, N, inv_h, x);
            int64_t k = n;
            while (k > 1) {
                k -= 1;
                x -= tau * v;
                v += tau * E_1d(coeffs + k * slab, L, N, inv_h, x);
            }
            x -= tau * v;
            v += half * E_1d(coeffs, L, N, inv_h, x);
            X[p] = x;
            V[p] = v;
        }
    } else if (d == 2) {
#pragma omp parallel for schedule(static) num_threads(threads)
        for (int64_t p = 0; p < M; ++p) {
            double x = X[2 * p], y = X[2 * p + 1], u = V[2 * p], v = V[2 * p + 1];
            double ex, ey;
            if (half_kick) {
                E_2d(coeffs + n * slab, L, N, inv_h, x, y, &ex, &ey);
                u += half * ex;
                v += half * ey;
            }
            int64_t k = n;
            while (k > 1) {
                k -= 1;
                x -= tau * u;
                y -= tau * v;
                E_2d(coeffs + k * slab, L, N, inv_h, x, y, &ex, &ey);
                u += tau * ex;
                v += tau * ey;
            }
            x -= tau * u;
            y -= tau * v;
            E_2d(coeffs, L, N, inv_h, x, y, &ex, &ey);
            u += half * ex;
            v += half * ey;
            X[2 * p] = x;
            X[2 * p + 1] = y;
            V[2 * p] = u;
            V[2 * p + 1] = v;
        }
    } else {
#pragma omp parallel for schedule(static) num_threads(threads)
        for (int64_t p = 0; p < M; ++p) {
            double x = X[3 * p], y = X[3 * p + 1], z = X[3 * p + 2];
            double u = V[3 * p], v = V[3 * p + 1], w = V[3 * p + 2];
            double ex, ey, ez;
            if (half_kick) {
                E_3d(coeffs + n * slab, L, N, inv_h, x, y, z, &ex, &ey, &ez);
                u += half * ex;
                v += half * ey;
                w += half * ez;
            }
            int64_t k = n;
            while (k > 1) {
                k -= 1;
                x -= tau * u;
                y -= tau * v;
                z -= tau * w;
                E_3d(coeffs + k * slab, L, N, inv_h, x, y, z, &ex, &ey, &ez);
                u += tau * ex;
                v += tau * ey;
                w += tau * ez;
            }
            x -= tau * u;
            y -= tau * v;
            z -= tau * w;
            E_3d(coeffs, L, N, inv_h, x, y, z, &ex, &ey, &ez);
            u += half * ex;
            v += half * ey;
            w += half * ez;
            X[3 * p] = x;
            X[3 * p + 1] = y;
            X[3 * p + 2] = z;
            V[3 * p] = u;
            V[3 * p + 1] = v;
            V[3 * p + 2] = w;
        }
    }
    return M * (half_kick ? n + 1 : n);
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
