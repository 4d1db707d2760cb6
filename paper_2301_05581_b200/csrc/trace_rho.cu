// trace_rho.cu -- fused Psi-tilde trace + f0 at the foot point + v-reduction.
//
// Replaces density.compute_rho's point loop (density.py:72-91) ->
// flow.psi_tilde_batch (flow.py:115-121) -> kernels.trace_backward
// (kernels.py:390-412, _trace_1d/2d/3d kernels.py:184-387) -> initial.eval_f0
// (initial.py:165-180) -> np.add.reduce over v (density.py:80-81).
//
// One thread per quadrature point (x_i, v_j) with (x, v) in registers; no point
// arrays exist (they are decoded from the thread index, unlike
// density.py:32-42).  Warp lanes take 32 consecutive x nodes at the same v
// (x-fastest), so the stencil gathers of neighbouring lanes hit neighbouring
// coefficients.  The coefficient history is streamed backwards (slab n-1 first)
// through a shared-memory ring filled by TMA bulk copies (cp.async.bulk,
// mbarrier complete_tx) that the whole CTA shares.  The v-sum is a fixed-order
// per-thread accumulation then a fixed-order CTA sum over warps: deterministic,
// no atomics.
//
// CTA tile: 32 nodes x vt_rows v-rows (warps * PPT rows per pass).  Output:
// partial[vt][node] (vt = global v-tile) and per-CTA (f_min, f_max).
#include <cfloat>

#include "trace_common.cuh"

namespace nufi {

// MOM = false: compute_rho (Psi-tilde, per-node v-sums).
// MOM = true:  the observable sweep of density.quadrature_sweep_many
// (density.py:94-120) for the fixed conserved-quantity weights: Psi (leading
// half kick through slab n, kernels.py:194-196), f = f0(foot), and per-CTA sums
// of f, f^2, f ln f, |v|^2 f / 2, v_a f at the UNTRACED quadrature point plus
// (f_min, f_max) -> p.partial[cta][mom_count(D)].
// GL = true: slabs too large for a shared-memory ring (large grids) are read in place
// from the (L2-resident where it fits) global history instead of being staged.
// The block reduce fused into the trace (threadfence-reduction pattern, two levels): the
// last CTA to finish a node tile forms that tile's block sums, the last node tile the
// block (min, max).  Same fixed order as reduce_blocks_kernel, so bit-identical to it.
__device__ __forceinline__ void fused_block_reduce(const TraceRhoParams &p, int tile, int node, bool valid, int lane,
                                                int warp, int warps) {
    __shared__ unsigned last;
    const int nblk = p.b_hi - p.b_lo, vpb = p.vt_per_block, nt = p.node_tiles;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(p.tile_cnt + tile, 1u) == (unsigned)(nblk * vpb) - 1u;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int bb = warp; bb < nblk; bb += warps) {
        const int b = p.b_lo + bb;
        const double *src = p.partial + (size_t)b * vpb * p.nodes + (valid ? node : 0);
        double s = 0.0;
        int t = 0;
        for (; t + 8 <= vpb; t += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (size_t)(t + u) * p.nodes);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; t < vpb; ++t) s += __ldcg(src + (size_t)t * p.nodes);
        if (valid) p.block_out[(size_t)b * p.nodes + node] = s;
        double mn = DBL_MAX, mx = -DBL_MAX;
        for (int q = lane; q < vpb; q += 32) {
            const size_t c = ((size_t)b * vpb + q) * nt + tile;
            mn = fmin(mn, __ldcg(p.fminmax + 2 * c));
            mx = fmax(mx, __ldcg(p.fminmax + 2 * c + 1));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
            p.block_mm[2 * ((size_t)b * nt + tile)] = mn;
            p.block_mm[2 * ((size_t)b * nt + tile) + 1] = mx;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        p.tile_cnt[tile] = 0u;  // ready for the next launch
        last = atomicAdd(p.tile_cnt + nt, 1u) == (unsigned)nt - 1u;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int bb = warp; bb < nblk; bb += warps) {
        const int b = p.b_lo + bb;
        double mn = DBL_MAX, mx = -DBL_MAX;
        for (int q = lane; q < nt; q += 32) {
            mn = fmin(mn, __ldcg(p.block_mm + 2 * ((size_t)b * nt + q)));
            mx = fmax(mx, __ldcg(p.block_mm + 2 * ((size_t)b * nt + q) + 1));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
            p.block_out[(size_t)p.B * p.nodes + 2 * b] = mn;
            p.block_out[(size_t)p.B * p.nodes + 2 * b + 1] = mx;
        }
    }
    if (threadIdx.x == 0) p.tile_cnt[nt] = 0u;
}

template <int D, int PPT, bool POW2, int NX, bool MOM, bool GL = false>
__global__ void __launch_bounds__(256, 2) trace_rho_kernel(const TraceRhoParams p, const double K) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warps = blockDim.x >> 5;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int N = p.N;
    const int sps = p.slabs_per_stage;
    const int stages = p.stages;
    const int slab_elems = p.ev_slab_elems;

    double *ring = reinterpret_cast<double *>(smem_raw);
    // the mbarriers sit after max(ring, red) -- the CTA reduction below may need more
    // room than the ring (MOM sweeps on small grids) and must never overwrite them
    // (same layout as trace_rho_smem_bytes)
    const size_t ring_elems = GL ? 0 : (size_t)stages * sps * slab_elems;
    const size_t red_elems = (size_t)(mom_sums(3) + 2) * blockDim.x;
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + (ring_elems > red_elems ? ring_elems : red_elems));
    uint64_t *empty = full + stages;
    double *red = ring;  // aliases the ring once every stage is consumed

    const int tile = blockIdx.x % p.node_tiles;
    const int vt = p.vt_lo + blockIdx.x / p.node_tiles;
    const int node = tile * 32 + lane;
    const bool valid = node < p.nodes;

    int ni[D];
    {
        int r = valid ? node : 0;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
            ni[a] = r % N;
            r /= N;
        }
    }

    const int n = p.n;
    const int stages_per_pass = (n + sps - 1) / sps;
    const int total_it = p.passes * stages_per_pass;

    // Issue the bulk copy for ring iteration `it` (pass-agnostic: stage index
    // it % stages_per_pass covers slabs [k_lo, k_hi], k_hi = n-1 - st*sps).
    auto issue = [&](int it) {
        const int st = it % stages_per_pass;
        const int s = it % stages;
        const int k_hi = n - 1 - st * sps;
        const int k_lo = max(0, k_hi - sps + 1);
        const uint32_t bytes = (uint32_t)((k_hi - k_lo + 1) * slab_elems * sizeof(double));
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_bulk_g2s(ring + (size_t)s * sps * slab_elems, p.ev_hist + (size_t)k_lo * slab_elems, bytes, &full[s]);
    };

    if (!GL) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < stages; ++s) {
                mbar_init(&full[s], 1);
                reinterpret_cast<unsigned *>(&empty[s])[0] = 0u;  // release counter of stage s
            }
            fence_mbar_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int it = 0; it < min(stages, total_it); ++it) issue(it);
        }
    }

    double acc = 0.0, fmn = DBL_MAX, fmx = -DBL_MAX;
    constexpr int NS = MOM ? mom_sums(D) : 1;
    double mom[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) mom[q] = 0.0;
    int it = 0;
    int s = 0;         // ring stage of iteration it (= it % stages), kept incrementally:
    uint32_t ph = 0u;  // and its fill parity ((it / stages) & 1) -- no integer division per stage
    for (int pass = 0; pass < p.passes; ++pass) {
        double X[PPT][D], V[PPT][D];
        int64_t jrow[PPT];
#pragma unroll
        for (int pp = 0; pp < PPT; ++pp) {
            jrow[pp] = D == 1 ? (int64_t)d1_row(vt, (pass * warps + warp) * PPT + pp, p.vt_per_block, p.B)
                              : (int64_t)vt * p.vt_rows + (int64_t)(pass * warps + warp) * PPT + pp;
            int64_t r = jrow[pp];
#pragma unroll
            for (int a = D - 1; a >= 0; --a) {
                const int ja = (int)(r % p.Nv);
                r /= p.Nv;
                // grids.py:110-115: -vmax + (j + 0.5) * hv
                const double v = __dadd_rn(-p.vmax, __dmul_rn((double)ja + 0.5, p.hv));
                X[pp][a] = (double)ni[a] - (D == 1 ? D1_OFF : 0.5);  // d = 1: shifted state (d1_locate)
                V[pp][a] = v * p.vel_to_scaled;
            }
            // Psi's leading half kick through the step's own field (slab n, read in place)
            if (MOM && n >= 1) kick<D, POW2, NX>(X[pp], V[pp], p.ev_hist + (size_t)n * slab_elems, N, K, true);
        }

        for (int st = 0; st < stages_per_pass; ++st, ++it) {
            const int k_hi = n - 1 - st * sps;
            const int k_lo = max(0, k_hi - sps + 1);
            if (!GL) mbar_wait(&full[s], ph);
            const double *buf = GL ? p.ev_hist + (size_t)k_lo * slab_elems : ring + (size_t)s * sps * slab_elems;
            // slab 0 is stored pre-halved (field_common.cuh), so every kick is uniform
            if constexpr (D == 1) {
                // drift folded into the kick (X carries the look-ahead drift inside the stream)
                if (st == 0)
#pragma unroll
                    for (int pp = 0; pp < PPT; ++pp) X[pp][0] -= V[pp][0];
                for (int k = k_hi; k >= k_lo; --k) {
                    const double *slab = buf + (size_t)(k - k_lo) * slab_elems;
#pragma unroll
                    for (int pp = 0; pp < PPT; ++pp) kick1_folded<POW2, NX>(X[pp][0], V[pp][0], slab, N);
                }
                if (st == stages_per_pass - 1)
#pragma unroll
                    for (int pp = 0; pp < PPT; ++pp) X[pp][0] += V[pp][0];
            } else {
                for (int k = k_hi; k >= k_lo; --k) {
                    const double *slab = buf + (size_t)(k - k_lo) * slab_elems;
#pragma unroll
                    for (int pp = 0; pp < PPT; ++pp) substep<D, POW2, NX>(X[pp], V[pp], slab, N, K, false);
                }
            }
            if (!GL) {
                // the LAST warp to finish the stage refills it (no warp waits for the others;
                // a fixed refilling warp would stall on the slowest one every stage)
                __syncwarp();
                if (lane == 0) {
                    unsigned *cnt = reinterpret_cast<unsigned *>(&empty[s]);
                    __threadfence_block();
                    if (atomicAdd(cnt, 1u) == (unsigned)warps - 1u) {
                        *cnt = 0u;
                        __threadfence_block();
                        if (it + stages < total_it) {
                            fence_proxy_async_smem();  // generic reads of the stage -> async-proxy refill
                            issue(it + stages);
                        }
                    }
                }
            }
            if (++s == stages) s = 0, ph ^= 1u;
        }

#pragma unroll
        for (int pp = 0; pp < PPT; ++pp) {
            double x[D], v[D];
            if (n == 0) {
                int64_t r = jrow[pp];
#pragma unroll
                for (int a = D - 1; a >= 0; --a) {
                    const int ja = (int)(r % p.Nv);
                    r /= p.Nv;
                    x[a] = __dmul_rn((double)ni[a], p.hx);  // grids.py:104-108
                    v[a] = __dadd_rn(-p.vmax, __dmul_rn((double)ja + 0.5, p.hv));
                }
            } else {
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    x[a] = (X[pp][a] + (D == 1 ? D1_OFF : 0.5)) * p.hx;
                    v[a] = V[pp][a] * p.scaled_to_vel;
                }
            }
            const double f = eval_f0<D>(p.f0, x, v);
            if (valid) {
                fmn = fmin(fmn, f);
                fmx = fmax(fmx, f);
                if constexpr (MOM) {
                    // weights at the untraced point (density.py:57-60): v0 of row jrow
                    double v0[D], v2 = 0.0;
                    int64_t r = jrow[pp];
#pragma unroll
                    for (int a = D - 1; a >= 0; --a) {
                        v0[a] = __dadd_rn(-p.vmax, __dmul_rn((double)(int)(r % p.Nv) + 0.5, p.hv));
                        r /= p.Nv;
                    }
#pragma unroll
                    for (int a = 0; a < D; ++a) v2 = fma(v0[a], v0[a], v2);
                    mom[0] += f;
                    mom[1] = fma(f, f, mom[1]);
                    mom[2] += f > 0.0 ? f * log(f) : 0.0;  // 0 ln 0 := 0 (SPEC diagnostics)
                    mom[3] = fma(0.5 * v2, f, mom[3]);
#pragma unroll
                    for (int a = 0; a < D; ++a) mom[4 + a] = fma(v0[a], f, mom[4 + a]);
                } else {
                    acc += f;
                }
            }
        }
    }

    if constexpr (MOM) {
        // fixed-order CTA reduction of the moment sums and (min, max)
        constexpr int NM = NS + 2;
        const int T = blockDim.x;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NS; ++q) red[q * T + threadIdx.x] = mom[q];
        red[NS * T + threadIdx.x] = fmn;
        red[(NS + 1) * T + threadIdx.x] = fmx;
        __syncthreads();
        if (warp == 0) {
            double* out = p.partial + (size_t)blockIdx.x * NM;
#pragma unroll
            for (int q = 0; q < NM; ++q) {
                double s = q < NS ? 0.0 : (q == NS ? DBL_MAX : -DBL_MAX);
                for (int w = 0; w < warps; ++w) {
                    const double x = red[q * T + w * 32 + lane];
                    s = q < NS ? s + x : (q == NS ? fmin(s, x) : fmax(s, x));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double y = __shfl_xor_sync(0xffffffffu, s, o);
                    s = q < NS ? s + y : (q == NS ? fmin(s, y) : fmax(s, y));
                }
                if (lane == 0) out[q] = s;
            }
        }
        return;
    }

    // fixed-order CTA reduction over warps (same v-tile, same node per lane)
    const int T = blockDim.x;
    __syncthreads();  // every warp is done with the ring before it is reused as `red`
    red[threadIdx.x] = acc;
    red[T + threadIdx.x] = fmn;
    red[2 * T + threadIdx.x] = fmx;
    __syncthreads();
    if (warp == 0) {
        double s = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
        for (int w = 0; w < warps; ++w) {
            s += red[w * 32 + lane];
            mn = fmin(mn, red[T + w * 32 + lane]);
            mx = fmax(mx, red[2 * T + w * 32 + lane]);
        }
        if (valid) p.partial[(size_t)vt * p.nodes + node] = s;
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
    if (p.block_out) fused_block_reduce(p, tile, node, valid, lane, warp, warps);
}

// partial[vt][node] -> blocks[b][node] (fixed order over the block's v-tiles);
// per-block (min, max) after the Nx^d * B sums.  Grid: one thread per (b, node)
// of this rank's blocks; CTA 0 additionally reduces the min / max.
__global__ void reduce_blocks_kernel(const double *__restrict__ partial, const double *__restrict__ fminmax,
                                     double *__restrict__ out, int nodes, int node_tiles, int vt_per_block,
                                     int b_lo, int b_hi, int B, int sum_ctas) {
    if ((int)blockIdx.x < sum_ctas) {
        const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const int64_t count = (int64_t)(b_hi - b_lo) * nodes;
        if (tid < count) {
            const int b = b_lo + (int)(tid / nodes);
            const int node = (int)(tid % nodes);
            const double *src = partial + (size_t)b * vt_per_block * nodes + node;
            double s = 0.0;
            for (int t = 0; t < vt_per_block; ++t) s += src[(size_t)t * nodes];
            out[(size_t)b * nodes + node] = s;
        }
        return;
    }
    // one CTA per block of this rank: (min, max) over the block's tile pairs
    const int b = b_lo + (int)blockIdx.x - sum_ctas;
    double *mm = out + (size_t)B * nodes;
    double mn = DBL_MAX, mx = -DBL_MAX;
    const int64_t c0 = (int64_t)b * vt_per_block * node_tiles;
    const int64_t c1 = c0 + (int64_t)vt_per_block * node_tiles;
    for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
        mn = fmin(mn, fminmax[2 * c]);
        mx = fmax(mx, fminmax[2 * c + 1]);
    }
    __shared__ double smn[32], smx[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        smn[threadIdx.x >> 5] = mn;
        smx[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mn = fmin(mn, smn[w]);
            mx = fmax(mx, smx[w]);
        }
        mm[2 * b] = mn;
        mm[2 * b + 1] = mx;
    }
}

// Multi-rank d >= 2: the block reduce of this rank's blocks fused with the exchange --
// every block sum and block (min, max) is STORED into every rank's exchange table (peer
// memory over NVLink, CUDA IPC; the same fixed order as reduce_blocks_kernel), then each
// CTA makes its stores visible with one cumulative system-scope fence and adds 1 to slot
// `src` of every rank's arrival counters.  The receiving rank's field update waits for
// the counters (field_update_kernel) instead of an NCCL allreduce.
__global__ void reduce_exchange_kernel(const double *__restrict__ partial, const double *__restrict__ fminmax,
                                       int nodes, int node_tiles, int vt_per_block, int b_lo, int b_hi, int B,
                                       int sum_ctas, MgExchange x) {
    if ((int)blockIdx.x < sum_ctas) {
        const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const int64_t count = (int64_t)(b_hi - b_lo) * nodes;
        if (tid < count) {
            const int b = b_lo + (int)(tid / nodes);
            const int node = (int)(tid % nodes);
            const double *src = partial + (size_t)b * vt_per_block * nodes + node;
            double s = 0.0;
            for (int t = 0; t < vt_per_block; ++t) s += src[(size_t)t * nodes];
            for (int r = 0; r < x.G; ++r) x.tab[r][(size_t)b * nodes + node] = s;
        }
    } else {
        const int b = b_lo + (int)blockIdx.x - sum_ctas;
        double mn = DBL_MAX, mx = -DBL_MAX;
        const int64_t c0 = (int64_t)b * vt_per_block * node_tiles;
        const int64_t c1 = c0 + (int64_t)vt_per_block * node_tiles;
        for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
            mn = fmin(mn, fminmax[2 * c]);
            mx = fmax(mx, fminmax[2 * c + 1]);
        }
        __shared__ double smn[32], smx[32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if ((threadIdx.x & 31) == 0) {
            smn[threadIdx.x >> 5] = mn;
            smx[threadIdx.x >> 5] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                mn = fmin(mn, smn[w]);
                mx = fmax(mx, smx[w]);
            }
            for (int r = 0; r < x.G; ++r) {
                x.tab[r][(size_t)B * nodes + 2 * b] = mn;
                x.tab[r][(size_t)B * nodes + 2 * b + 1] = mx;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.sc.sys;" ::: "memory");
        for (int r = 0; r < x.G; ++r)
            asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(x.flags[r] + x.src) : "memory");
    }
}

// ----------------------------------------------------------------------------
// host-side launch helpers
// ----------------------------------------------------------------------------

size_t trace_rho_smem_bytes(const TraceRhoParams &p, int threads) {
    const size_t ring = (size_t)p.stages * p.slabs_per_stage * p.ev_slab_elems * sizeof(double);
    const size_t red = (size_t)(mom_sums(3) + 2) * (size_t)threads * sizeof(double);
    return (ring > red ? ring : red) + 2 * p.stages * sizeof(uint64_t);
}

template <int D, int PPT, bool POW2, int NX, bool MOM = false, bool GL = false>
static cudaError_t launch_one(const TraceRhoParams &p, double K, int ctas, int threads, size_t smem,
                              cudaStream_t st) {
    auto kern = trace_rho_kernel<D, PPT, POW2, NX, MOM, GL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<ctas, threads, smem, st>>>(p, K);
    return cudaGetLastError();
}

// large grids: slabs read in place from global memory (no ring), one point per thread
cudaError_t launch_trace_rho_global(int d, bool mom, bool pow2, const TraceRhoParams &p, double K, int ctas,
                                    int threads, cudaStream_t st) {
    const size_t smem = (size_t)(mom_sums(3) + 2) * (size_t)threads * sizeof(double) + 64;
#define NUFI_GL(DD)                                                                                           \
    if (d == DD) {                                                                                            \
        if (mom)                                                                                              \
            return pow2 ? launch_one<DD, 1, true, 0, true, true>(p, K, ctas, threads, smem, st)             \
                        : launch_one<DD, 1, false, 0, true, true>(p, K, ctas, threads, smem, st);           \
        return pow2 ? launch_one<DD, 1, true, 0, false, true>(p, K, ctas, threads, smem, st)                \
                    : launch_one<DD, 1, false, 0, false, true>(p, K, ctas, threads, smem, st);              \
    }
    NUFI_GL(1)
    NUFI_GL(2)
    NUFI_GL(3)
#undef NUFI_GL
    return cudaErrorInvalidValue;
}

cudaError_t launch_trace_rho(int d, int ppt, bool pow2, const TraceRhoParams &p, double K, int ctas, int threads,
                             cudaStream_t st) {
    const size_t smem = trace_rho_smem_bytes(p, threads);
#define NUFI_TR(DD, PP)                                                                              \
    if (d == DD && ppt == PP) {                                                                      \
        if (p.N == 8) return launch_one<DD, PP, true, 8, false>(p, K, ctas, threads, smem, st);             \
        if (p.N == 16) return launch_one<DD, PP, true, 16, false>(p, K, ctas, threads, smem, st);           \
        if (p.N == 32) return launch_one<DD, PP, true, 32, false>(p, K, ctas, threads, smem, st);           \
        return pow2 ? launch_one<DD, PP, true, 0, false>(p, K, ctas, threads, smem, st)                     \
                    : launch_one<DD, PP, false, 0, false>(p, K, ctas, threads, smem, st);                   \
    }
    NUFI_TR(2, 1)
    NUFI_TR(3, 1)
    NUFI_TR(2, 2)
    NUFI_TR(3, 2)
#undef NUFI_TR
    return cudaErrorInvalidValue;
}

// Observable sweep (MOM = true): one CTA per tile, outputs p.partial[cta][mom_count(d)].
cudaError_t launch_sweep_moments(int d, int ppt, bool pow2, const TraceRhoParams &p, double K, int ctas, int threads,
                                 cudaStream_t st) {
    const size_t smem = trace_rho_smem_bytes(p, threads);
#define NUFI_SW(DD, PP)                                                                               \
    if (d == DD && ppt == PP) {                                                                       \
        if (p.N == 16) return launch_one<DD, PP, true, 16, true>(p, K, ctas, threads, smem, st);      \
        if (p.N == 32) return launch_one<DD, PP, true, 32, true>(p, K, ctas, threads, smem, st);      \
        return pow2 ? launch_one<DD, PP, true, 0, true>(p, K, ctas, threads, smem, st)                \
                    : launch_one<DD, PP, false, 0, true>(p, K, ctas, threads, smem, st);              \
    }
    if (d == 1 && ppt == 1) {  // the BASELINE d = 1 grids: compile-time plane offsets in the kick
        if (p.N == 64) return launch_one<1, 1, true, 64, true>(p, K, ctas, threads, smem, st);
        if (p.N == 256) return launch_one<1, 1, true, 256, true>(p, K, ctas, threads, smem, st);
    }
    NUFI_SW(1, 1)
    NUFI_SW(2, 1)
    NUFI_SW(3, 1)
#undef NUFI_SW
    return cudaErrorInvalidValue;
}

// per-CTA moment rows -> out[mom_count(d)] in a fixed order (one CTA)
__global__ void reduce_moments_kernel(const double *__restrict__ part, int rows, int nm, int nsums, double measure,
                                      double *__restrict__ out) {
    __shared__ double sh[32];
    for (int q = 0; q < nm; ++q) {
        const bool is_sum = q < nsums, is_min = q == nsums;
        double s = is_sum ? 0.0 : (is_min ? DBL_MAX : -DBL_MAX);
        for (int r = threadIdx.x; r < rows; r += blockDim.x) {
            const double x = part[(size_t)r * nm + q];
            s = is_sum ? s + x : (is_min ? fmin(s, x) : fmax(s, x));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, s, o);
            s = is_sum ? s + y : (is_min ? fmin(s, y) : fmax(s, y));
        }
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = sh[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                t = is_sum ? t + sh[w] : (is_min ? fmin(t, sh[w]) : fmax(t, sh[w]));
            out[q] = is_sum ? t * measure : t;
        }
        __syncthreads();
    }
}

cudaError_t launch_reduce_moments(const double *part, int rows, int d, double measure, double *out, cudaStream_t st) {
    reduce_moments_kernel<<<1, 256, 0, st>>>(part, rows, mom_sums(d) + 2, mom_sums(d), measure, out);
    return cudaGetLastError();
}

int launch_reduce_exchange(const double *partial, const double *fminmax, int nodes, int node_tiles, int vt_per_block,
                           int b_lo, int b_hi, int B, const MgExchange &x, cudaStream_t st) {
    const int64_t count = (int64_t)(b_hi - b_lo) * nodes;
    const int threads = 256;
    const int sum_ctas = (int)((count + threads - 1) / threads);
    reduce_exchange_kernel<<<sum_ctas + (b_hi - b_lo), threads, 0, st>>>(partial, fminmax, nodes, node_tiles,
                                                                         vt_per_block, b_lo, b_hi, B, sum_ctas, x);
    return cudaGetLastError() == cudaSuccess ? sum_ctas + (b_hi - b_lo) : -1;
}

cudaError_t launch_reduce_blocks(const double *partial, const double *fminmax, double *out, int nodes,
                                 int node_tiles, int vt_per_block, int b_lo, int b_hi, int B, cudaStream_t st) {
    const int64_t count = (int64_t)(b_hi - b_lo) * nodes;
    const int threads = 256;
    const int sum_ctas = (int)((count + threads - 1) / threads);
    reduce_blocks_kernel<<<sum_ctas + (b_hi - b_lo), threads, 0, st>>>(partial, fminmax, out, nodes, node_tiles,
                                                                       vt_per_block, b_lo, b_hi, B, sum_ctas);
    return cudaGetLastError();
}

}  // namespace nufi
