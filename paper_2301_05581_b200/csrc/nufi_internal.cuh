// nufi_internal.cuh -- device-side helpers shared by the NuFI sm_100a kernels.
//
// TMA bulk copies (cp.async.bulk -> SASS UBLKCP) completing on shared-memory
// mbarriers, the magic-constant cell locator used by the production trace,
// and the kernel parameter blocks.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "nufi.h"

namespace nufi {

// ----------------------------------------------------------------------------
// constants
// ----------------------------------------------------------------------------

// 1.5 * 2^52: x + MAGIC rounds x to the nearest integer in the low mantissa bits
// (|x| < 2^51); (x + MAGIC) - MAGIC is rint(x) and the low 32 bits of the sum's
// bit pattern are rint(x) as a two's-complement int32.
constexpr double MAGIC = 6755399441055744.0;
constexpr double GAUSS_NORM = 0.3989422804014327;  // 1/sqrt(2*pi), initial.py:22

constexpr int MAX_D = 3;
#ifndef NUFI_BARRIER_SLEEP_NS
#define NUFI_BARRIER_SLEEP_NS 32
#endif
constexpr int MAX_FIELD_NODES = 4096;  // single-CTA field update limit (Nx^d); beyond: field_large.cu
constexpr int MAX_GRID_NODES = 1 << 21;  // supported Nx^d (128^3)

// ----------------------------------------------------------------------------
// f0 descriptor (initial.py:25-56, 165-180)
// ----------------------------------------------------------------------------

struct F0Params {
    int d;
    int n_centers[MAX_D];
    int power[MAX_D];
    double centers[MAX_D][NUFI_MAX_CENTERS];
    double weights[MAX_D][NUFI_MAX_CENTERS];
    double alpha;
    double k;
};

// eval_f0 at one point (initial.py:41-49,165-180): x is NOT wrapped.
template <int D>
__device__ __forceinline__ double eval_f0(const F0Params &P, const double *x, const double *v) {
    double vel = 1.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double acc = 0.0;
        for (int m = 0; m < P.n_centers[a]; ++m) {
            double t = v[a] - P.centers[a][m];
            acc += P.weights[a][m] * exp(-0.5 * (t * t));
        }
        acc *= GAUSS_NORM;
        if (P.power[a]) acc = acc * (v[a] * v[a]);
        vel = (a == 0) ? acc : vel * acc;
    }
    double pert = cos(P.k * x[0]);
#pragma unroll
    for (int a = 1; a < D; ++a) pert = pert + cos(P.k * x[a]);
    return vel * (1.0 + P.alpha * pert);
}

// ----------------------------------------------------------------------------
// cell location (production arithmetic)
// ----------------------------------------------------------------------------

// X is a position in cell units shifted by -1/2 (X = x*N/L - 1/2, unwrapped).
// Returns the cell index in [0, N) and the centred offset fc in [-1/2, 1/2];
// the reference's fraction is f = fc + 1/2 (kernels.py:153-162).
template <bool POW2>
__device__ __forceinline__ int locate_centred(double X, int N, double &fc) {
    double s = X + MAGIC;
    double r = s - MAGIC;
    fc = X - r;
    int ri = (int)(unsigned)(__double_as_longlong(s) & 0xffffffffull);
    if (POW2) return ri & (N - 1);
    int i = ri % N;
    return i < 0 ? i + N : i;
}

// Cubic B-spline stencil weights and their t-derivatives (kernels.py:62-81 /
// 211-221), SCALED: w'' = 6 w, dw'' = 2 dw, from the centred fraction fc
// (f = fc + 1/2), FMA form.  The scale factors are folded into the kick constant
// (trace_common.cuh: K / 12 in d = 2, K / 72 in d = 3), which saves the four
// constant multiplies per axis of the unscaled form:
//   w0'' = s^3          w1'' = 4 - 6 f^2 + 3 f^3   w2'' = 4 - 6 s^2 + 3 s^3   w3'' = f^3
//   dw0'' = -s^2        dw1'' = f (3 f - 4)        dw2'' = s (4 - 3 s)        dw3'' = f^2
__device__ __forceinline__ void bspline_w_dw_scaled(double fc, double w[4], double dw[4]) {
    const double f = fc + 0.5, s = 0.5 - fc;
    const double f2 = f * f, s2 = s * s;
    w[0] = s2 * s;
    w[1] = fma(f2, fma(3.0, f, -6.0), 4.0);
    w[2] = fma(s2, fma(3.0, s, -6.0), 4.0);
    w[3] = f2 * f;
    dw[0] = -s2;
    dw[1] = f * fma(3.0, f, -4.0);
    dw[2] = s * fma(-3.0, s, 4.0);
    dw[3] = f2;
}

// ----------------------------------------------------------------------------
// TMA bulk copy + mbarrier (PTX; sm_90+ incl. sm_100a)
// ----------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order this thread's (and, after a CTA barrier, the CTA's) generic-proxy shared-memory
// accesses before subsequent async-proxy (TMA) accesses of the same bytes
// multi-rank d >= 2 exchange (reduce_exchange_kernel): this step's parity slot of every
// rank's table, every rank's arrival counters, and the source slot of the sending rank
#ifndef NUFI_MG_MAX
#define NUFI_MG_MAX 8
#endif
struct MgExchange {
    double *tab[NUFI_MG_MAX];
    unsigned *flags[NUFI_MG_MAX];
    int G, src;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// cp.async (Ampere-style LDGSTS): a 16-byte global -> shared copy, L2 only (.cg), that
// holds no registers while in flight; cp_async_wait_all waits for this thread's copies
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared, completion signalled on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).  SASS: UBLKCP.S.G.
__device__ __forceinline__ void tma_bulk_g2s(void *dst_smem, const void *src_gmem, uint32_t bytes,
                                             uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Grid-wide barrier for a cooperative (co-resident) launch: monotonically
// increasing arrival counter, `target` = CTAs x barrier-generation.  Arrival is a
// release-ordered reduction (no returned value, no separate fence); the wait is an
// acquire-load spin.  The CTA barriers on both sides order the other threads.
__device__ __forceinline__ void grid_barrier(unsigned *counter, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        while (v < target) {
            if (NUFI_BARRIER_SLEEP_NS > 0) __nanosleep(NUFI_BARRIER_SLEEP_NS);
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        }
    }
    __syncthreads();
}

// The same barrier for a rank of a fused multi-rank run: gives up (returns) when the
// rank's error flag is raised, so a watchdog timeout cannot strand the other CTAs.
__device__ __forceinline__ void grid_barrier_wd(unsigned *counter, unsigned target, const int *err) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        while (v < target && *(volatile const int *)err == 0) {
            if (NUFI_BARRIER_SLEEP_NS > 0) __nanosleep(NUFI_BARRIER_SLEEP_NS);
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        }
    }
    __syncthreads();
}

// ----------------------------------------------------------------------------
// kernel parameter blocks
// ----------------------------------------------------------------------------

struct TraceRhoParams {
    // geometry
    int N;          // Nx
    int nodes;      // Nx^d
    int Nv;
    int64_t V;      // Nv^d
    int node_tiles; // ceil(nodes / 32)
    int vt_rows;    // v-rows per CTA tile (warps * PPT * passes)
    int passes;
    int vt_lo;      // first global v-tile traced by this launch
    int B;          // velocity blocks (fixed combine order; the multi-rank shard unit)
    int vt_per_block;
    // step
    int n;          // Psi-tilde through slabs n-1 .. 0
    // arithmetic (scaled units: X = x*inv_h - 1/2, V = v*tau*inv_h)
    double hx, inv_h, vmax, hv;
    double vel_to_scaled;  // tau * inv_h
    double scaled_to_vel;  // 1 / (tau * inv_h)
    // history of evaluation slabs (see field_update.cu for layouts)
    const double *ev_hist;
    int ev_slab_elems;     // doubles per evaluation slab (16-byte multiple)
    int slabs_per_stage;
    int stages;
    F0Params f0;
    // outputs: partial[vt][nodes], fminmax[vt * node_tiles + tile][2]
    double *partial;
    double *fminmax;
    // d >= 2 fused block reduce (optional): the last CTA of each node tile sums its nodes'
    // partials per block in fixed v-tile order (reduce_blocks_kernel's order) into
    // block_out[b][node]; the last node tile reduces the per-(block, node tile) (min, max)
    // pairs (block_mm scratch) into block_out[B * nodes + 2 b].  Blocks [b_lo, b_hi).
    double *block_out;
    double *block_mm;        // B * node_tiles * 2
    unsigned *tile_cnt;      // node_tiles + 1 arrival counters (zero between launches)
    int b_lo, b_hi;
};

// background density (field_update.cu)
struct RhoBarParams {
    int d, N, Nv;
    double hx, hv, vmax, hx_d, hv_d, L_d;
    F0Params f0;
    double *out;
};

}  // namespace nufi
