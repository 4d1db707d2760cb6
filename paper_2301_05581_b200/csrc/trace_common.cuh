// trace_common.cuh -- one backward leapfrog substep of the NuFI characteristic trace.
//
// Reference semantics (kernels.py:184-387): per stored step k
//     x -= tau * v ;  v += tau * E_k(x)        (k = n-1 .. 1)
//     x -= tau * v ;  v += (tau/2) * E_0(x)    (last substep)
// with E_k = -grad of the periodic cubic B-spline whose coefficients are slab k.
//
// Production arithmetic ("fast" mode) works in scaled units
//     X = x * N/L - 1/2  (cell units, centred),   V = v * tau * N/L  (cells/step)
// so a drift is one DADD and the cell lookup is the magic-constant rint of X:
// cell i = rint(X) mod N, centred fraction fc = X - rint(X) in [-1/2, 1/2], and
// the reference's fraction is f = fc + 1/2.  d = 1 shifts the state instead:
//     Y = x * N/L - 1/16,  s8 = Y + 1.5 * 2^49 (ulp 1/8)
// leaves round(8 Y) in the low word of s8, whose bits >= 3 are 8 * floor(x N/L): the cell's
// byte offset in a plane of doubles, OR-able into an aligned slab address with no shift on
// the substep's dependent chain; the local coordinate is u = Y - cell = f - 1/16 (d1_locate).  The kick scale
//     K = -tau^2 (N/L)^2    (V += K * dphi/dt-sum, i.e. tau*N/L * tau*E)
// is folded into the evaluation slabs (d = 1) or applied once (d = 2, 3).
//
// Evaluation-slab layouts (written by field_update.cu, one per stored step):
//   d = 1: three arrays [A | B | C] of N doubles: on cell i the kick is the
//          quadratic A_i + u*(B_i + u*C_i) in u = f - 1/16 (the B-spline derivative
//          restricted to one cell, pre-multiplied by K; d1_cell_poly);
//   d = 2: [R][R], d = 3: [R][R][R] with R = N + 3: raw coefficients with a
//          periodic halo on every axis (halo index j' holds c[(j' - 1) mod N]),
//          so the 4^d stencil of the cell with lower corner i is the block at
//          halo index i .. i+3 per axis: one base address + 4^d compile-time
//          offsets, no per-tap index wrapping.
#pragma once

#include "nufi_internal.cuh"

namespace nufi {

__host__ __device__ constexpr int ev_slab_raw_elems(int d, int N) {
    return d == 1 ? 3 * N : (d == 2 ? (N + 3) * (N + 3) : (N + 3) * (N + 3) * (N + 3));
}

// halo element e of a d >= 2 evaluation slab -> linear index of the raw slab
__host__ __device__ inline int ev_halo_source(int d, int N, int e) {
    const int R = N + 3;
    int lin = 0;
    int div = d == 2 ? R : R * R;
    for (int a = 0; a < d; ++a) {
        const int j = (e / div) % R;
        lin = lin * N + (j - 1 + N) % N;
        div /= R;
    }
    return lin;
}
// d = 1 velocity row of warp slot w of global v-tile vt.  Block b is the residue
// class {j : j mod B == b}; inside a block the tile's rows are strided across the
// whole block (local row l = t + vt_per_block * w), so every CTA tile -- and every
// rank's share of blocks -- mixes trapped (chaotic, bank-conflicted gathers) and
// passing (coherent) particles: equal work per CTA between grid barriers.
__host__ __device__ __forceinline__ int d1_row(int vt, int w, int vt_per_block, int B) {
    const int b = vt / vt_per_block, t = vt - b * vt_per_block;
    return (t + vt_per_block * w) * B + b;
}

// conserved-quantity sweep: sums f, f^2, f ln f, |v|^2 f / 2, v_a f (then f_min, f_max)
__host__ __device__ constexpr int mom_sums(int d) { return 4 + d; }

// padded to a 16-byte multiple (TMA bulk copy granularity)
__host__ __device__ constexpr int ev_slab_elems(int d, int N) {
    return (ev_slab_raw_elems(d, N) + 1) & ~1;
}

// d = 1 evaluation slab: three planes [A | B | C] (three 8-byte shared-memory gathers per
// lookup).  NUFI_D1_PAIRED=1 interleaves the (A_i, B_i) pairs at 2i, 2i + 1 (one 16-byte
// gather + one 8-byte) -- measured slower: 16-byte gathers are served per quarter warp, so
// random cells cost more wavefronts than two 8-byte gathers (ts1 trace 76.5 -> 80.2 ms).
#ifndef NUFI_D1_PAIRED
#define NUFI_D1_PAIRED 0
#endif
__host__ __device__ constexpr int d1_ia(int i, int N) { return NUFI_D1_PAIRED ? 2 * i : i; }
__host__ __device__ constexpr int d1_ib(int i, int N) { return NUFI_D1_PAIRED ? 2 * i + 1 : N + i; }
__host__ __device__ constexpr int d1_ic(int i, int N) { return 2 * N + i; }

__device__ __forceinline__ void d1_fetch(const double *__restrict__ slab, int i, int N, double &A, double &B,
                                         double &C) {
#if NUFI_D1_PAIRED
    const double2 ab = *reinterpret_cast<const double2 *>(slab + 2 * i);
    A = ab.x;
    B = ab.y;
#else
    A = slab[i];
    B = slab[N + i];
#endif
    C = slab[2 * N + i];
}

// The kick polynomial of one d = 1 cell from the four spline coefficients c_{i-1} .. c_{i+2}:
// -(d/dt) of the cubic B-spline sum on the cell is g0 + g1 f + g2 f^2 in the reference's
// fraction f (kernels.py:164-182); stored in u = f - 1/16, pre-multiplied by the kick scale K.
__host__ __device__ __forceinline__ void d1_cell_poly(double c0, double c1, double c2, double c3, double K,
                                                      double &A, double &B, double &C) {
    const double g0 = 0.5 * (c2 - c0);
    const double g1 = (c0 - 2.0 * c1) + c2;
    const double g2 = (1.5 * (c1 - c2)) + 0.5 * (c3 - c0);
    A = K * ((g0 + 0.0625 * g1) + 0.00390625 * g2);
    B = K * (g1 + 0.125 * g2);
    C = K * g2;
}

// d = 1 state offset: Y = x * N/L - D1_OFF
constexpr double D1_OFF = 0.0625;
constexpr double MAGIC8 = 844424930131968.0;  // 1.5 * 2^49: ulp 1/8

// d = 1 cell lookup on the shifted state Y: returns the low word of s8 = Y + MAGIC8, i.e.
// round(8 Y) mod 2^32, whose bits >= 3 hold the cell floor(round(8 Y) / 8) = floor(x N/L)
// (a tie of round(8 Y) only occurs on a cell boundary, where both neighbouring pieces agree);
// u = Y - cell in [-1/16, 15/16) is the local coordinate of the stored polynomial.
__device__ __forceinline__ unsigned d1_locate(double Y, double &u) {
    const long long b = __double_as_longlong(Y + MAGIC8);
    u = Y - (__longlong_as_double(b & ~7ll) - MAGIC8);
    return (unsigned)b;
}

// cell index mod N from d1_locate's word (POW2: mask; else floor division and wrap)
template <bool POW2>
__device__ __forceinline__ int d1_cell(unsigned lo8, int N) {
    if (POW2) return (int)(lo8 >> 3) & (N - 1);
    const int i = ((int)lo8 >> 3) % N;
    return i < 0 ? i + N : i;
}

template <bool POW2>
__device__ __forceinline__ int wrap_idx(int i, int N) {
    if (POW2) return i & (N - 1);
    i %= N;
    return i < 0 ? i + N : i;
}

// Kick through evaluation slab `slab` (smem or global): V += K * g(X), or half of
// it (`half`: the tau/2 kicks of kernels.py:194-196 and 203-205).
template <int D, bool POW2, int NX = 0>
__device__ __forceinline__ void kick(const double (&X)[D], double (&V)[D], const double *__restrict__ slab, int N_,
                                     double K, bool half) {
    const int N = NX ? NX : N_;  // compile-time N makes every stencil offset an immediate
    if constexpr (D == 1) {  // X[0] is the shifted state Y (d1_locate)
        double fc;
        const int i = d1_cell<POW2>(d1_locate(X[0], fc), N);
        double A, B, C;
        d1_fetch(slab, i, N, A, B, C);
        const double kick = fma(fc, fma(fc, C, B), A);
        V[0] = half ? fma(0.5, kick, V[0]) : V[0] + kick;
        (void)K;
    } else if constexpr (D == 2) {
        const int R = N + 3;
        double fx, fy;
        const int ix = locate_centred<POW2>(X[0], N, fx);
        const int iy = locate_centred<POW2>(X[1], N, fy);
        double wx[4], dwx[4], wy[4], dwy[4];
        bspline_w_dw_scaled(fx, wx, dwx);
        bspline_w_dw_scaled(fy, wy, dwy);
        const double *c = slab + ix * R + iy;
        double gx = 0.0, gy = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const double *cm = c + m * R;
            const double c0 = cm[0], c1 = cm[1], c2 = cm[2], c3 = cm[3];
            const double r = fma(c3, wy[3], fma(c2, wy[2], fma(c1, wy[1], c0 * wy[0])));
            const double rd = fma(c3, dwy[3], fma(c2, dwy[2], fma(c1, dwy[1], c0 * dwy[0])));
            gx = fma(dwx[m], r, gx);
            gy = fma(wx[m], rd, gy);
        }
        const double k = (half ? 0.5 : 1.0) * (K * (1.0 / 12.0));  // scaled weights: 2 * 6
        V[0] = fma(k, gx, V[0]);
        V[1] = fma(k, gy, V[1]);
    } else {
        const int R = N + 3;
        double fx, fy, fz;
        const int ix = locate_centred<POW2>(X[0], N, fx);
        const int iy = locate_centred<POW2>(X[1], N, fy);
        const int iz = locate_centred<POW2>(X[2], N, fz);
        double wx[4], dwx[4], wy[4], dwy[4], wz[4], dwz[4];
        bspline_w_dw_scaled(fx, wx, dwx);
        bspline_w_dw_scaled(fy, wy, dwy);
        bspline_w_dw_scaled(fz, wz, dwz);
        const double *c = slab + (ix * R + iy) * R + iz;
        double gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            double sy = 0.0, sdy = 0.0, sdz = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double *cq = c + (m * R + q) * R;
                const double c0 = cq[0], c1 = cq[1], c2 = cq[2], c3 = cq[3];
                const double r = fma(c3, wz[3], fma(c2, wz[2], fma(c1, wz[1], c0 * wz[0])));
                const double rd = fma(c3, dwz[3], fma(c2, dwz[2], fma(c1, dwz[1], c0 * dwz[0])));
                sy = fma(wy[q], r, sy);
                sdy = fma(dwy[q], r, sdy);
                sdz = fma(wy[q], rd, sdz);
            }
            gx = fma(dwx[m], sy, gx);
            gy = fma(wx[m], sdy, gy);
            gz = fma(wx[m], sdz, gz);
        }
        const double k = (half ? 0.5 : 1.0) * (K * (1.0 / 72.0));  // scaled weights: 2 * 6 * 6
        V[0] = fma(k, gx, V[0]);
        V[1] = fma(k, gy, V[1]);
        V[2] = fma(k, gz, V[2]);
    }
}

// The d = 1 folded update from the located cell's coefficients (kick polynomial
// q = A + B fc + C fc^2, pre-scaled): V <- V + q, X <- (X - V) - q.  Two rounding orders,
// chosen by N alone so that every d = 1 path of one grid (run_1d, trace_rho_1d, trace_rho,
// any rank split) computes the same bits:
//  - N <= 64: few points per SM, the run is bound by the substep's dependent chain
//    (profiles/r02_d1_chain_floor.txt).  X = ((X - V) - A - fc B) - fc^2 C puts the
//    last-loaded coefficient C one DFMA from the next cell lookup (two in Horner form),
//    for two more FP64 ops per substep;
//  - N > 64: throughput-bound (FP64 pipe and shared-memory wavefronts), the 5-op Horner form.
__host__ __device__ constexpr bool d1_wform(int N) { return N <= 64; }

__device__ __forceinline__ void d1_fold(double &X, double &V, double fc, double A, double B, double C, bool wform) {
    const double XmV = X - V;
    if (wform) {
        const double w = fc * fc;
        X = fma(-w, C, fma(-fc, B, XmV - A));
        V = fma(w, C, fma(fc, B, V + A));
    } else {
        const double t = fma(fc, C, B);
        X = fma(-fc, t, XmV - A);
        V = fma(fc, t, V + A);
    }
}

// d = 1 substep with the drift folded into the kick (every d = 1 path outside the shared-memory
// ring fast path kick1s, which has the same lookup and arithmetic): on entry X is the
// already drifted position of this substep, on exit the drifted position of the next one,
// X - V_new = (X - V) - A - fc (B + fc C): the next cell lookup does not wait for a DADD.
template <bool POW2, int NX = 0>
__device__ __forceinline__ void kick1_folded(double &X, double &V, const double *__restrict__ slab, int N_) {
    const int N = NX ? NX : N_;
    double fc;
    const int i = d1_cell<POW2>(d1_locate(X, fc), N);
    double A, B, C;
    d1_fetch(slab, i, N, A, B, C);
    d1_fold(X, V, fc, A, B, C, d1_wform(N));
}

// shared-window alignment of the d = 1 slab rings: a multiple of 8 N for every N with a
// compile-time kernel (slab = 3 N doubles: 8 N divides the slab and stage offsets too)
constexpr unsigned D1_RING_ALIGN = 2048;

// the d = 1 ring start: smem aligned up to D1_RING_ALIGN in the shared window (the
// kernels reserve D1_RING_ALIGN extra bytes)
__device__ __forceinline__ double *d1_ring_base(unsigned char *smem) {
    const unsigned raw32 = (unsigned)__cvta_generic_to_shared(smem);
    return reinterpret_cast<double *>(smem + (((raw32 + D1_RING_ALIGN - 1) & ~(D1_RING_ALIGN - 1)) - raw32));
}

// kick1 with the cell address formed by ONE 3-input LOP3: the slab's shared-window address
// sbase is a multiple of N*8 (the ring is aligned to D1_RING_ALIGN bytes and every slab / stage
// offset is a multiple of N*8), and d1_locate's word already holds 8 * cell in its bits >= 3,
// so base + 8*(i mod N) == (word & (8N-8)) | sbase: DADD -> LOP3 -> LDS on the substep's
// dependent chain (the centred rint form needed a shift and an add as well).
template <int NX>
__device__ __forceinline__ void kick1s(double &X, double &V, unsigned sbase) {
    static_assert(NX > 0 && (NX & (NX - 1)) == 0, "power-of-two N");
    double fc;
    const unsigned addr = (d1_locate(X, fc) & (unsigned)(8 * NX - 8)) | sbase;
    double A, B, C;  // issued A, B, C: C (loaded last) is the one the W form consumes last
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(A) : "r"(addr));
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(B) : "r"(addr), "n"(8 * NX));
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(C) : "r"(addr), "n"(16 * NX));
    d1_fold(X, V, fc, A, B, C, d1_wform(NX));
}

// One backward substep: drift x -= tau v, then kick through slab.
template <int D, bool POW2, int NX = 0>
__device__ __forceinline__ void substep(double (&X)[D], double (&V)[D], const double *__restrict__ slab,
                                        int N, double K, bool half) {
#pragma unroll
    for (int a = 0; a < D; ++a) X[a] -= V[a];
    kick<D, POW2, NX>(X, V, slab, N, K, half);
}

}  // namespace nufi
