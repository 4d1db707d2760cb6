// trace_rho_1d.cu -- d = 1: one launch per NuFI step.
//
// Fused Psi-tilde trace + f0 at the foot point + v-reduction (density.py:72-91,
// flow.py:115-121, kernels.py:184-209, initial.py:165-180), and — in the last
// CTA to finish — the fixed-order combine + Poisson / spline / append / W / E
// tail (field_common.cuh).  d = 1 runs are latency-bound (16-33k points, a
// serial chain of n substeps per point), so the kernel minimises the
// per-substep dependency chain:
//
//   X -= V                      DADD      (scaled units, trace_common.cuh)
//   s = X + MAGIC               DADD      cell = low bits of s (LOP3)
//   A,B,C = slab[cell]          LDS x3    (SoA slab, compile-time offsets)
//   fc = X - (s - MAGIC)        2 DADD    (off the chain, overlaps the loads)
//   V = fma(fc, fma(fc,C,B), V + A)       2 DFMA on the chain
//
// with the 8-slab stages of the TMA ring fully unrolled so slab addresses are
// immediates.  Slab 0 is stored pre-halved, so the final tau/2 kick needs no
// special case.
#include <cfloat>
#include <cstdlib>

#include "field_common.cuh"

namespace nufi {

// NX: compile-time Nx (power of two) or 0 (runtime N, any value); SPS: slabs per stage.
// Block = C consumer warps (one point per thread) + 1 producer warp that keeps
// the TMA ring full, so no consumer ever waits for a refill it did not need.
template <int NX, int SPS>
__global__ void __launch_bounds__(544) trace_rho_1d_kernel(const TraceRhoParams p, const FieldParams fp, int fuse,
                                                            unsigned *ticket) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int cw = p.vt_rows;  // tracing warps (tile rows); the last warp is the producer
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool producer = warp == (int)(blockDim.x >> 5) - 1;
    const int N = NX ? NX : p.N;
    const int SLAB = NX ? ev_slab_elems(1, NX) : p.ev_slab_elems;
    const int stages = p.stages;

    double *ring = d1_ring_base(smem_raw);  // aligned: kick1s forms addresses by OR
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)stages * SPS * SLAB);
    uint64_t *empty = full + stages;
    double *red = reinterpret_cast<double *>(empty + stages);  // 3 * 32 * cw
    __shared__ int is_last;

    const int tile = blockIdx.x % p.node_tiles;
    const int vt = p.vt_lo + blockIdx.x / p.node_tiles;
    const int node = tile * 32 + lane;
    const bool valid = node < p.nodes && !producer && warp < cw;
    const int n = p.n;
    const int groups = (n + SPS - 1) / SPS;  // slab groups g = k / SPS, consumed g_top .. 0

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], cw);
        }
        fence_mbar_init();
    }
    __syncthreads();

    double acc = 0.0, fmn = DBL_MAX, fmx = -DBL_MAX;
    if (producer) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int it = 0; it < groups; ++it) {
                if (it >= stages) mbar_wait(&empty[s], ph ^ 1u);  // consumers released this buffer's last use
                const int k_lo = (groups - 1 - it) * SPS, k_hi = min(n - 1, k_lo + SPS - 1);
                const uint32_t bytes = (uint32_t)((k_hi - k_lo + 1) * SLAB * sizeof(double));
                mbar_arrive_expect_tx(&full[s], bytes);
                tma_bulk_g2s(ring + (size_t)s * SPS * SLAB, p.ev_hist + (size_t)k_lo * SLAB, bytes, &full[s]);
                if (++s == stages) s = 0, ph ^= 1u;
            }
        }
    } else if (warp < cw) {
        // point (x_i, v_j): grids.py:104-115
        const int j = d1_row(vt, warp, p.vt_per_block, p.B);
        const double v0 = __dadd_rn(-p.vmax, __dmul_rn((double)j + 0.5, p.hv));
        double V = v0 * p.vel_to_scaled;
        double X = ((double)(valid ? node : 0) - D1_OFF) - V;  // shifted state (d1_locate), first drift folded
        int s = 0;
        uint32_t ph = 0;
        const int top_cnt = n - (groups - 1) * SPS;  // slabs in the (partial) top group
        for (int it = 0; it < groups; ++it) {
            mbar_wait(&full[s], ph);
            const double *buf = ring + (size_t)s * SPS * SLAB;
            if (NX != 0 && (it > 0 || top_cnt == SPS)) {
                const unsigned b32 = (unsigned)__cvta_generic_to_shared(buf);
#pragma unroll
                for (int q = SPS - 1; q >= 0; --q) kick1s<NX ? NX : 64>(X, V, b32 + q * SLAB * 8);
            } else {
                const int cnt = it == 0 ? top_cnt : SPS;
                for (int q = cnt - 1; q >= 0; --q) {
                    if (NX != 0)
                        kick1_folded<true, NX>(X, V, buf + q * SLAB, N);
                    else
                        kick1_folded<false>(X, V, buf + q * SLAB, N);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == stages) s = 0, ph ^= 1u;
        }
        // f0 at the foot point (x unwrapped)
        double x, v;
        if (n == 0) {
            x = __dmul_rn((double)node, p.hx);
            v = v0;
        } else {
            x = ((X + V) + D1_OFF) * p.hx;  // undo the look-ahead drift of the last kick
            v = V * p.scaled_to_vel;
        }
        const double f = eval_f0<1>(p.f0, &x, &v);
        if (valid) {
            acc = f;
            fmn = f;
            fmx = f;
        }
        red[threadIdx.x] = acc;
        red[32 * cw + threadIdx.x] = fmn;
        red[64 * cw + threadIdx.x] = fmx;
    }
    __syncthreads();

    // fixed-order CTA reduction over the consumer warps (same node per lane)
    if (warp == 0) {
        double sum = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
        for (int w = 0; w < cw; ++w) {
            sum += red[w * 32 + lane];
            mn = fmin(mn, red[32 * cw + w * 32 + lane]);
            mx = fmax(mx, red[64 * cw + w * 32 + lane]);
        }
        if (node < p.nodes) p.partial[(size_t)vt * p.nodes + node] = sum;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
            const size_t c = (size_t)vt * p.node_tiles + tile;
            p.fminmax[2 * c] = mn;
            p.fminmax[2 * c + 1] = mx;
        }
    }
    if (!fuse) return;

    // ---- last CTA to finish runs the step tail (threadfence reduction pattern) ----
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // an earlier asynchronously enqueued tail failed: leave the history untouched
    if (fp.finish_only || !fp.status || *(volatile int *)fp.status == 0)
        field_update_body(fp, reinterpret_cast<double *>(smem_raw));
    mirror_status(fp);
    if (threadIdx.x == 0) *ticket = 0u;
}

size_t trace_rho_1d_smem_bytes(const TraceRhoParams &p, int threads, int nodes) {
    const size_t ring = D1_RING_ALIGN + (size_t)p.stages * p.slabs_per_stage * p.ev_slab_elems * sizeof(double) +
                        2 * p.stages * sizeof(uint64_t) + 3 * (size_t)(threads - 32) * sizeof(double);
    const size_t tail = (size_t)field_smem_doubles(nodes, p.N, true) * sizeof(double);
    return ring > tail ? ring : tail;
}

// slabs per stage for a given N (must match the template instantiations below)
int trace_rho_1d_sps(int N, bool wide) {
    if (N == 64) {
        if (const char *e = getenv("NUFI_D1_SPS"))
            if (atoi(e) == 16 || atoi(e) == 32) return atoi(e);
        return 64;  // 2 stages x 64 slabs (192 KB, one CTA per SM): ts1 87.8 -> 80.9 ms vs 6 x 16
    }
    if (N == 32) return 16;
    if (N == 128) return 8;
    if (N == 256) {
        if (wide) return 16;  // the WIDE run kernel is instantiated for 2 x 16 slabs only
        if (const char *e = getenv("NUFI_D1_SPS")) {
            const int v = atoi(e);
            if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) return v;
        }
        // 2 stages x 8 slabs for two 8-warp CTAs per SM (sl1 248 -> 218 ms vs 4 x 4), 2 x 16 for
        // one 16-warp CTA per SM (218 -> 203 ms)
        return wide ? 16 : 8;
    }
    return 1;
}

template <int NX, int SPS>
static cudaError_t launch1(const TraceRhoParams &p, const FieldParams &fp, int fuse, unsigned *ticket, int ctas,
                           int threads, size_t smem, cudaStream_t st) {
    auto kern = trace_rho_1d_kernel<NX, SPS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<ctas, threads, smem, st>>>(p, fp, fuse, ticket);
    return cudaGetLastError();
}

cudaError_t launch_trace_rho_1d(const TraceRhoParams &p, const FieldParams &fp, int fuse, unsigned *ticket, int ctas,
                                int threads, cudaStream_t st) {
    const size_t smem = trace_rho_1d_smem_bytes(p, threads, p.nodes);
    switch (p.N) {
        case 32: return launch1<32, 16>(p, fp, fuse, ticket, ctas, threads, smem, st);
        case 64:
            if (p.slabs_per_stage == 32) return launch1<64, 32>(p, fp, fuse, ticket, ctas, threads, smem, st);
            if (p.slabs_per_stage == 64) return launch1<64, 64>(p, fp, fuse, ticket, ctas, threads, smem, st);
            return launch1<64, 16>(p, fp, fuse, ticket, ctas, threads, smem, st);
        case 128: return launch1<128, 8>(p, fp, fuse, ticket, ctas, threads, smem, st);
        case 256:
            if (p.slabs_per_stage == 1) return launch1<256, 1>(p, fp, fuse, ticket, ctas, threads, smem, st);
            if (p.slabs_per_stage == 2) return launch1<256, 2>(p, fp, fuse, ticket, ctas, threads, smem, st);
            if (p.slabs_per_stage == 8) return launch1<256, 8>(p, fp, fuse, ticket, ctas, threads, smem, st);
            if (p.slabs_per_stage == 16) return launch1<256, 16>(p, fp, fuse, ticket, ctas, threads, smem, st);
            return launch1<256, 4>(p, fp, fuse, ticket, ctas, threads, smem, st);
        default: return launch1<0, 1>(p, fp, fuse, ticket, ctas, threads, smem, st);
    }
}

}  // namespace nufi
