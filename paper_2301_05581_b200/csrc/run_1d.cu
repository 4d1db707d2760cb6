// run_1d.cu -- d = 1 whole-run persistent kernel: every step of the NuFI loop
// in ONE cooperative launch.
//
// d = 1 runs are latency-bound: 16-33k points, each step a serial chain of n
// substeps per point, then a global v-sum, then the Poisson / spline tail whose
// result the very first substep of the next step needs.  Launch gaps and a
// serial single-CTA tail would dominate, so:
//
//   for n = n_first .. n_last:
//     trace   every CTA traces its tiles of points through slabs n-1 .. 0:
//             slab n-1 from its own shared-memory copy, slabs n-2 .. 0 streamed
//             by the TMA ring (producer warp, cp.async.bulk + mbarriers);
//             f0 at the foot point; fixed-order CTA v-sum -> partial[vt][node]
//     barrier grid-wide (co-resident CTAs, monotonic arrival counter)
//     tail    EVERY CTA runs the same fixed-order combine + Poisson / spline /
//             W / E (field_common.cuh) on the partials -- redundant but parallel,
//             so no second barrier: each CTA keeps evaluation slab n in shared
//             memory for its next step; CTA 0 alone writes the history and the
//             per-step outputs.
//
// Deterministic: every CTA executes the identical tail on identical data.
#include <cfloat>

#include "field_common.cuh"

namespace nufi {


__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// doubles of the ring / tail-workspace union (16-byte aligned end for the barriers)
__host__ __device__ inline size_t run_1d_ring_doubles(int stages, int sps, int slab, int nodes, int N) {
    const size_t ring = (size_t)stages * sps * slab, tail = (size_t)field_smem_doubles(nodes, N, true);
    return ((ring > tail ? ring : tail) + 1) & ~(size_t)1;
}

// WIDE: 16 tracing warps + producer in one CTA per SM (experiment knob NUFI_D1_WARPS=16)
// N = 32, 64 run one CTA per SM (the 2 x 64-slab ring fills the SM's shared memory), so their
// register budget is not halved for a second resident CTA
template <int NX, int SPS, int WIDE = 0, int SPLIT = 0>
__global__ void __launch_bounds__(WIDE ? 544 : 288, (WIDE || NX == 64 || NX == 32) ? 1 : 2)
    run_1d_kernel(const Run1DParams P) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const TraceRhoParams &p = P.tp;
    // warps [0, cw) trace (cw = tile rows), the last warp is the TMA producer, any
    // warps in between only help with the tail (the CTA is 9 warps wide for it)
    const int cw = p.vt_rows;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool producer = warp == (int)(blockDim.x >> 5) - 1;
    const int N = NX ? NX : p.N;
    const int SLAB = NX ? ev_slab_elems(1, NX) : p.ev_slab_elems;
    const int stages = p.stages;
    const int nodes = p.nodes;

    // multi-rank context: rank rk of G traces its blocks' tiles with nct CTAs (lc local index)
    const int G = P.mg_ranks > 1 ? P.mg_ranks : 1;
    const bool mg = G > 1, emu = mg && P.mg_emulated;
    const int rk = !mg ? 0 : (emu ? (int)blockIdx.x / P.mg_ctas : P.mg_rank);
    const int lc = emu ? (int)blockIdx.x % P.mg_ctas : (int)blockIdx.x;
    const int nct = emu ? P.mg_ctas : (int)gridDim.x;
    double *const my_partial = emu ? P.mg_partial[rk] : p.partial;
    double *const my_fminmax = emu ? P.mg_fminmax[rk] : p.fminmax;
    unsigned *const my_barrier = emu ? P.mg_barrier[rk] : P.barrier;
    const int tiles_r = P.tiles / G, tile_lo = rk * tiles_r;
    // split (single rank, one tile per CTA, P.split_helpers > 0): owners trace rows 0 .. cw-2 of
    // their tile, CTAs tiles .. tiles + helpers - 1 trace every tile's last row (<= cw - 1 rows
    // each), so no SM holds more than cw - 1 tracing warps; the tail completes each tile's
    // sequential sum with + last row (the same operations, so bit-identical to no split)
    const bool split = SPLIT && P.split_helpers > 0 && !mg;  // compile-time off for other kernels
    const bool helper = split && lc >= tiles_r;

    // shared memory: [ring | tail workspace (aliased)] | barriers | red | local slab.
    // The tail runs between grid barriers when no bulk copy is in flight (every copy
    // of a step is consumed before its barrier), so it reuses the ring's bytes;
    // the ring is re-armed behind a proxy fence (generic writes -> async-proxy writes).
    const size_t ring_doubles = run_1d_ring_doubles(stages, SPS, SLAB, nodes, N);
    double *ring = d1_ring_base(smem_raw);  // aligned: kick1s forms addresses by OR
    double *tail = ring;                                                   // field_smem_doubles(nodes, N, true)
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + ring_doubles);
    uint64_t *empty = full + stages;
    double *red = reinterpret_cast<double *>(empty + stages);  // 3 * 32 * cw
    double *slabN = red + 3 * 32 * cw;                          // evaluation slab n-1 (SLAB)

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], cw);
        }
        fence_mbar_init();
    }
    if (P.n_first >= 1)
        for (int e = threadIdx.x; e < SLAB; e += blockDim.x)
            slabN[e] = __ldcg(p.ev_hist + (size_t)(P.n_first - 1) * SLAB + e);
    __syncthreads();

    // ring state (identical sequence on the producer and the consumers)
    int s_ring = 0;
    uint32_t ph_ring = 0;
    int fills = 0;
    unsigned gen = 0;
    // groups consumed so far by this CTA (uniform over its threads): the ring stage the next
    // group lands in is gs_mod (= groups so far mod stages, kept incrementally: a 64-bit modulo
    // on the path from the barrier into the tail cost ~130 ns per step)
    unsigned gs_mod = 0;
    const int my_tiles = lc < tiles_r ? (tiles_r - lc + nct - 1) / nct : 0;
    const size_t stage_doubles = (size_t)SPS * SLAB;
    bool pref_ready = false;  // this step's first group was issued before the previous tail

    for (int n = P.n_first; n <= P.n_last; ++n) {
        const int m = n >= 1 ? n - 1 : 0;  // slabs streamed by TMA: m-1 .. 0
        const int groups = (m + SPS - 1) / SPS;
        // partials double-buffered by step parity: a CTA that finished the tail of
        // step n may write step n+1's partials while a slower one still reads step n's
        double *part = my_partial + (size_t)(n & 1) * P.tiles * 32;
        double *fmm = my_fminmax + (size_t)(n & 1) * P.tiles * 2;
        double *row_last = split ? P.row_last + (size_t)(n & 1) * P.tiles * 32 : nullptr;
        double *row_last_mm = split ? P.row_last_mm + (size_t)(n & 1) * P.tiles * 2 : nullptr;
        const int top_cnt = m - (groups - 1) * SPS;

        const bool pref_now = pref_ready;
        pref_ready = false;
        // PAIR (the WIDE, many-tiles-per-CTA kernel): two tiles per pass share one stream of
        // the history through the ring (half the ring-fill traffic into shared memory, which
        // the gathers of this shared-memory-bound kernel compete with) and give every thread
        // two independent chains.  Each point's arithmetic and each tile's fixed-order CTA
        // v-sum are unchanged, so the results are bit-identical to one tile per pass.
        constexpr bool PAIR = WIDE != 0;
        // (a helper makes exactly one pass: t_loc = lc >= tiles_r)
        for (int t_loc = lc; t_loc < tiles_r || (helper && t_loc == lc); t_loc += (PAIR ? 2 : 1) * nct) {
            const bool first_tile = t_loc == lc;
            const bool hasB = PAIR && !helper && t_loc + nct < tiles_r;
            static constexpr bool kAlt = false;  // tile mapping: v-tile-major (true) or node-tile-major
            const int vts = P.tiles / p.node_tiles;
            // a helper's warp w traces the last row of item lc - tiles + w * helpers (split)
            const int item = helper ? (lc - tiles_r) + warp * P.split_helpers : 0;
            const bool tracing = helper ? (warp < cw - 1 && item < tiles_r) : (!split || warp < cw - 1);
            const int row = helper ? cw - 1 : warp;
            int nt2[2], vt2[2], node2[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int tile = tile_lo + (helper ? (item < tiles_r ? item : 0) : t_loc + (u ? nct : 0));
                nt2[u] = kAlt ? tile / vts : tile % p.node_tiles;
                vt2[u] = kAlt ? tile % vts : tile / p.node_tiles;
                node2[u] = nt2[u] * 32 + lane;
            }
            double f2[2] = {0.0, 0.0};
            bool valid2[2] = {false, false};
            if (producer) {
                const int it0 = (pref_now && first_tile) ? 1 : 0;  // group 0 already in flight
                if (lane == 0) {
                    auto issue = [&](int g, int mm) {
                        if (fills >= stages) mbar_wait(&empty[s_ring], ph_ring ^ 1u);
                        const int gg = (mm + SPS - 1) / SPS;
                        const int k_lo = (gg - 1 - g) * SPS, k_hi = min(mm - 1, k_lo + SPS - 1);
                        const uint32_t bytes = (uint32_t)((k_hi - k_lo + 1) * SLAB * sizeof(double));
                        mbar_arrive_expect_tx(&full[s_ring], bytes);
                        tma_bulk_g2s(ring + (size_t)s_ring * SPS * SLAB, p.ev_hist + (size_t)k_lo * SLAB, bytes,
                                     &full[s_ring]);
                        ++fills;
                        if (++s_ring == stages) s_ring = 0, ph_ring ^= 1u;
                    };
                    for (int it = it0; it < groups; ++it) issue(it, m);
                } else {
                    // keep the warp's copy of the ring state in step with lane 0
                    for (int it = it0; it < groups; ++it) {
                        ++fills;
                        if (++s_ring == stages) s_ring = 0, ph_ring ^= 1u;
                    }
                }
            } else if (warp < cw) {
                double X2[2], V2[2], v02[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    valid2[u] = tracing && node2[u] < nodes && (u == 0 || hasB);
                    const int j = d1_row(vt2[u], row, p.vt_per_block, p.B);
                    v02[u] = __dadd_rn(-p.vmax, __dmul_rn((double)j + 0.5, p.hv));  // grids.py:110-115
                    V2[u] = v02[u] * p.vel_to_scaled;
                    // shifted state (d1_locate), first drift folded
                    X2[u] = ((double)(node2[u] < nodes ? node2[u] : 0) - D1_OFF) - V2[u];
                }
                if (n >= 1 && tracing) {
#pragma unroll
                    for (int u = 0; u < (PAIR ? 2 : 1); ++u) {
                        if (u == 1 && !hasB) break;
                        if (NX)
                            kick1_folded<true, NX>(X2[u], V2[u], slabN, N);
                        else
                            kick1_folded<false>(X2[u], V2[u], slabN, N);
                    }
                }
                long long wait_cyc = 0, t_start = clock64();
                for (int it = 0; it < groups; ++it) {
                    const long long tw0 = clock64();
                    mbar_wait(&full[s_ring], ph_ring);
                    wait_cyc += clock64() - tw0;
                    const double *buf = ring + (size_t)s_ring * SPS * SLAB;
                    if (!tracing) {
                        // split: a warp without a row keeps the ring protocol only
                    } else if (NX != 0 && (it > 0 || top_cnt == SPS)) {
                        const unsigned b32 = (unsigned)__cvta_generic_to_shared(buf);
                        if (PAIR && hasB) {
#pragma unroll
                            for (int q = SPS - 1; q >= 0; --q) {
                                kick1s<NX ? NX : 64>(X2[0], V2[0], b32 + q * SLAB * 8);
                                kick1s<NX ? NX : 64>(X2[1], V2[1], b32 + q * SLAB * 8);
                            }
                        } else {
#pragma unroll
                            for (int q = SPS - 1; q >= 0; --q) kick1s<NX ? NX : 64>(X2[0], V2[0], b32 + q * SLAB * 8);
                        }
                    } else {
                        const int cnt = it == 0 ? top_cnt : SPS;
                        for (int q = cnt - 1; q >= 0; --q) {
#pragma unroll
                            for (int u = 0; u < (PAIR ? 2 : 1); ++u) {
                                if (u == 1 && !hasB) break;
                                if (NX)
                                    kick1_folded<true, NX>(X2[u], V2[u], buf + q * SLAB, N);
                                else
                                    kick1_folded<false>(X2[u], V2[u], buf + q * SLAB, N);
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s_ring]);
                    ++fills;
                    if (++s_ring == stages) s_ring = 0, ph_ring ^= 1u;
                }
                if (P.stamps && n == P.n_last && lane == 0 && warp == 0) {
                    const size_t o = 3 * (size_t)(P.n_last - P.n_first + 1) + 10 + 4 * 1024 + 2 * blockIdx.x;
                    P.stamps[o] = (unsigned long long)wait_cyc;
                    P.stamps[o + 1] = (unsigned long long)(clock64() - t_start);
                }
#pragma unroll
                for (int u = 0; u < (PAIR ? 2 : 1); ++u) {
                    double x, v;
                    if (n == 0) {
                        x = __dmul_rn((double)node2[u], p.hx);  // grids.py:104-108
                        v = v02[u];
                    } else {
                        x = ((X2[u] + V2[u]) + D1_OFF) * p.hx;  // undo the look-ahead drift of the last kick
                        v = V2[u] * p.scaled_to_vel;
                    }
                    f2[u] = eval_f0<1>(p.f0, &x, &v);
                }
            }
            if (helper) {
                // split: each tracing warp's row goes to the last-row table as is (the tile's
                // sequential sum ends with + this row; the tail adds it), its (min, max) alongside
                if (tracing) {
                    const double f = f2[0];
                    if (node2[0] < nodes) row_last[(size_t)vt2[0] * nodes + node2[0]] = valid2[0] ? f : 0.0;
                    double mn = valid2[0] ? f : DBL_MAX, mx = valid2[0] ? f : -DBL_MAX;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    }
                    if (lane == 0) {
                        const size_t c = (size_t)vt2[0] * p.node_tiles + nt2[0];
                        row_last_mm[2 * c] = mn;
                        row_last_mm[2 * c + 1] = mx;
                    }
                }
                continue;
            }
            // per tile: the fixed-order CTA v-sum in warp 0 (on the critical path to the
            // barrier), the sampled (min, max) in another warp alongside (split: over the
            // rows this CTA traced -- the tail adds the last row)
            const int mmw = cw > 1 ? 1 : 0;
            const int tr = split ? cw - 1 : cw;
#pragma unroll
            for (int u = 0; u < (PAIR ? 2 : 1); ++u) {
                if (u == 1 && !hasB) break;
                if (warp < cw) {
                    const double acc = valid2[u] ? f2[u] : 0.0;
                    red[threadIdx.x] = acc;
                    red[32 * cw + threadIdx.x] = valid2[u] ? f2[u] : DBL_MAX;
                    red[64 * cw + threadIdx.x] = valid2[u] ? f2[u] : -DBL_MAX;
                }
                __syncthreads();
                if (warp == 0) {
                    double sum = 0.0;
                    for (int w = 0; w < tr; ++w) sum += red[w * 32 + lane];
                    if (node2[u] < nodes) part[(size_t)vt2[u] * nodes + node2[u]] = sum;
                }
                if (warp == mmw) {
                    double mn = DBL_MAX, mx = -DBL_MAX;
                    for (int w = 0; w < tr; ++w) {
                        mn = fmin(mn, red[32 * cw + w * 32 + lane]);
                        mx = fmax(mx, red[64 * cw + w * 32 + lane]);
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    }
                    if (lane == 0) {
                        const size_t c = (size_t)vt2[u] * p.node_tiles + nt2[u];
                        fmm[2 * c] = mn;
                        fmm[2 * c + 1] = mx;
                    }
                }
                __syncthreads();
            }
        }

        {
            const int my_passes = helper ? 1 : (WIDE ? (my_tiles + 1) / 2 : my_tiles);  // ring streams this step
            gs_mod = (gs_mod + (unsigned)(my_passes * groups) % (unsigned)stages) % (unsigned)stages;
        }
        pref_ready = P.prefetch && (my_tiles > 0 || helper) && n < P.n_last && n >= 1;  // (groups_next > 0 iff n >= 1)
        // all partials of step n are written
        if (P.stamps && blockIdx.x == 0 && threadIdx.x == 0) P.stamps[3 * (n - P.n_first)] = globaltimer();
        if (P.stamps && threadIdx.x == 0 && (n % 400) == 0 && n > 0 && n / 400 <= 4 && blockIdx.x < 1024) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            P.stamps[3 * (P.n_last - P.n_first + 1) + 10 + (n / 400 - 1) * 1024 + blockIdx.x] =
                (globaltimer() << 8) | (smid & 0xff);
        }
        if (mg) {
            grid_barrier_wd(my_barrier, ++gen * nct, P.mg_error);
            if (*(volatile int *)P.mg_error) break;
        } else {
            grid_barrier(my_barrier, ++gen * nct);
        }
        if (P.stamps && blockIdx.x == 0 && threadIdx.x == 0) P.stamps[3 * (n - P.n_first) + 1] = globaltimer();

        FieldParams fp = P.fp;
        fp.sums = part;
        fp.minmax = fmm;
        fp.sums_last = row_last;
        fp.minmax_last = row_last_mm;
        if (mg) {
            // ---- fused exchange over peer memory: this rank's block sums (the canonical
            // sequential order over the block's tile rows) and block (min, max) are stored
            // straight into EVERY rank's exchange table (NVLink stores; parity-buffered by
            // step), then one arrival flag per peer (release, system scope) and a wait for
            // all peers' flags (acquire).  Every rank then runs the identical tail on the
            // identical table, so all ranks hold bit-identical histories.
            const int B = fp.B, rpb = fp.rows_per_block, nb = B / G, b_lo = rk * nb;
            const size_t xstride = (size_t)B * nodes + 2 * (size_t)B, xoff = (size_t)(n & 1) * xstride;
            bool wrote = false;
            for (int64_t o = (int64_t)lc * blockDim.x + threadIdx.x; o < (int64_t)nb * nodes;
                 o += (int64_t)nct * blockDim.x) {
                const int b = b_lo + (int)(o / nodes), i = (int)(o - (o / nodes) * nodes);
                const double *src = part + (size_t)b * rpb * nodes + i;
                double Sb = 0.0;
                int q = 0;
                for (; q + 8 <= rpb; q += 8) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (size_t)(q + u) * nodes);
#pragma unroll
                    for (int u = 0; u < 8; ++u) Sb += v[u];
                }
                for (; q < rpb; ++q) Sb += __ldcg(src + (size_t)q * nodes);
                for (int r = 0; r < G; ++r) P.mg_xtab[r][xoff + (size_t)b * nodes + i] = Sb;
                wrote = true;
            }
            for (int bb = lc; bb < nb; bb += nct) {
                const int b = b_lo + bb;
                double mn = DBL_MAX, mx = -DBL_MAX;
                for (int q = threadIdx.x; q < fp.mm_per_block; q += blockDim.x) {
                    mn = fmin(mn, __ldcg(fmm + 2 * ((size_t)b * fp.mm_per_block + q)));
                    mx = fmax(mx, __ldcg(fmm + 2 * ((size_t)b * fp.mm_per_block + q) + 1));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                }
                if (lane == 0) {
                    red[warp] = mn;
                    red[32 + warp] = mx;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                        mn = fmin(mn, red[w]);
                        mx = fmax(mx, red[32 + w]);
                    }
                    for (int r = 0; r < G; ++r) {
                        P.mg_xtab[r][xoff + (size_t)B * nodes + 2 * b] = mn;
                        P.mg_xtab[r][xoff + (size_t)B * nodes + 2 * b + 1] = mx;
                    }
                    wrote = true;
                }
                __syncthreads();
            }
            // Cross-rank arrival without further grid barriers: after its peer stores (ordered
            // by the CTA barrier and one cumulative system-scope fence) every CTA adds 1 to its
            // rank's slot of EVERY rank's arrival counter, then waits until each slot of its
            // own rank's counters shows all nct CTAs of that peer for this step.
            (void)wrote;
            __syncthreads();
            if (threadIdx.x == 0) {
                asm volatile("fence.sc.sys;" ::: "memory");
                for (int r = 0; r < G; ++r)
                    asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(P.mg_flags[r] + rk) : "memory");
                const unsigned target = (P.mg_base + (unsigned)(n - P.n_first) + 1u) * (unsigned)nct;
                const unsigned long long t0 = globaltimer();
                for (int q = 0; q < G; ++q) {
                    unsigned v;
                    for (;;) {
                        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(P.mg_flags[rk] + q)
                                     : "memory");
                        if (v >= target) break;
                        if (globaltimer() - t0 > 4000000000ull) {  // 4 s: a peer is gone
                            atomicExch(P.mg_error, 1);
                            break;
                        }
                        if (NUFI_BARRIER_SLEEP_NS > 0) __nanosleep(NUFI_BARRIER_SLEEP_NS);
                    }
                }
            }
            __syncthreads();
            if (*(volatile int *)P.mg_error) break;  // identical decision in every CTA of the rank
            fp.sums = P.mg_xtab[rk] + xoff;
            fp.rows_per_block = 1;
            fp.minmax = fp.sums + (size_t)B * nodes;
            fp.mm_per_block = 1;
        } else if (P.two_level) {
            // level 1, spread over the grid: tile partials -> block sums in the SAME
            // sequential order the tail uses (field_update_1d_body), block (min, max)
            const int B = fp.B, rpb = fp.rows_per_block;
            const int64_t outs = (int64_t)B * nodes;
            for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < outs;
                 o += (int64_t)gridDim.x * blockDim.x) {
                const int b = (int)(o / nodes), i = (int)(o - (int64_t)b * nodes);
                const double *src = fp.sums + (size_t)b * rpb * nodes + i;
                double Sb = 0.0;
                int q = 0;
                for (; q + 8 <= rpb; q += 8) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (size_t)(q + u) * nodes);
#pragma unroll
                    for (int u = 0; u < 8; ++u) Sb += v[u];
                }
                for (; q < rpb; ++q) Sb += __ldcg(src + (size_t)q * nodes);
                P.blocks[o] = Sb;
            }
            for (int b = blockIdx.x; b < B; b += gridDim.x) {
                double mn = DBL_MAX, mx = -DBL_MAX;
                for (int q = threadIdx.x; q < fp.mm_per_block; q += blockDim.x) {
                    mn = fmin(mn, __ldcg(fp.minmax + 2 * ((size_t)b * fp.mm_per_block + q)));
                    mx = fmax(mx, __ldcg(fp.minmax + 2 * ((size_t)b * fp.mm_per_block + q) + 1));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                }
                if (lane == 0) {
                    red[warp] = mn;
                    red[32 + warp] = mx;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                        mn = fmin(mn, red[w]);
                        mx = fmax(mx, red[32 + w]);
                    }
                    P.blocks[outs + 2 * b] = mn;
                    P.blocks[outs + 2 * b + 1] = mx;
                }
                __syncthreads();
            }
            grid_barrier(P.barrier, ++gen * gridDim.x);
            fp.sums = P.blocks;
            fp.rows_per_block = 1;
            fp.minmax = P.blocks + outs;
            fp.mm_per_block = 1;
        }

        // The next step's newest ring group (slabs n-1 .. ; slab n-1 became visible with this
        // step's barrier) is issued now, so its copy overlaps the tail, which then works in
        // another ring stage.
        if (pref_ready && producer) {
            if (lane == 0) {
                if (fills >= stages) mbar_wait(&empty[s_ring], ph_ring ^ 1u);  // released before the barrier
                const int gg = (n + SPS - 1) / SPS;  // step n + 1 streams slabs n - 1 .. 0
                const int k_lo = (gg - 1) * SPS, k_hi = min(n - 1, k_lo + SPS - 1);
                const uint32_t bytes = (uint32_t)((k_hi - k_lo + 1) * SLAB * sizeof(double));
                mbar_arrive_expect_tx(&full[s_ring], bytes);
                tma_bulk_g2s(ring + (size_t)s_ring * SPS * SLAB, p.ev_hist + (size_t)k_lo * SLAB, bytes,
                             &full[s_ring]);
            }
            ++fills;
            if (++s_ring == stages) s_ring = 0, ph_ring ^= 1u;
        }

        // redundant tail in every CTA; CTA 0 publishes
        fp.slot = n;
        fp.ev_local = slabN;
        double *tail_ws = tail;
        if (pref_ready) {
            // the next step's first group is landing in stage gs_mod: work in the next one
            tail_ws = ring + (size_t)(gs_mod + 1 == (unsigned)stages ? 0u : gs_mod + 1) * stage_doubles;
            fp.stage_cap = (int64_t)stage_doubles - field_smem_doubles(nodes, N, true);
        } else {
            fp.stage_cap = (int64_t)ring_doubles - field_smem_doubles(nodes, N, true);  // rest of the ring
        }
        const int64_t row = n - P.n_first;
        if (lc == 0 && !(emu && rk != 0)) {  // one publisher per rank (emulated: rank 0 only)
            fp.rho_out = P.rho_hist ? P.rho_hist + row * nodes : nullptr;
            fp.E_out = P.E_hist ? P.E_hist + row * nodes : nullptr;
            fp.W_out = P.W_hist ? P.W_hist + row : nullptr;
            fp.stats_out = P.stats_hist ? P.stats_hist + row * 3 : nullptr;
        } else {
            fp.rho_out = fp.E_out = fp.W_out = fp.stats_out = fp.coeffs_out = nullptr;
            fp.hist = fp.ev_hist = nullptr;
            fp.hist_len = nullptr;
            fp.status = nullptr;
        }
        fp.tstamps = (P.stamps && blockIdx.x == 0 && n == P.n_last) ? P.stamps + 3 * (P.n_last - P.n_first + 1) : nullptr;
        const bool ok = field_update_body(fp, tail_ws);
        __syncthreads();
        // the tail's generic-proxy writes to the ring bytes must be ordered before the
        // next step's bulk copies (async proxy) into them
        if (producer && lane == 0) fence_proxy_async_smem();
        if (P.stamps && blockIdx.x == 0 && threadIdx.x == 0) P.stamps[3 * (n - P.n_first) + 2] = globaltimer();
        if (!ok) {  // identical decision in every CTA
            // no CTA may exit with the prefetched bulk copy still landing in its shared memory
            if (pref_ready && warp == 0 && lane == 0) mbar_wait(&full[s_ring], ph_ring);
            break;
        }
    }
}

size_t run_1d_smem_bytes(const TraceRhoParams &p, int threads) {
    const int cw = threads / 32 - 1;
    return D1_RING_ALIGN +
           run_1d_ring_doubles(p.stages, p.slabs_per_stage, p.ev_slab_elems, p.nodes, p.N) * sizeof(double) +
           2 * p.stages * sizeof(uint64_t) + (3 * 32 * (size_t)cw + p.ev_slab_elems) * sizeof(double);
}

template <int NX, int SPS, int WIDE = 0, int SPLIT = 0>
static cudaError_t launch_run(const Run1DParams &P, int threads, int device, cudaStream_t st, int *grid_out) {
    auto kern = run_1d_kernel<NX, SPS, WIDE, SPLIT>;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int G = P.mg_ranks > 1 ? P.mg_ranks : 1;
    const bool emu = G > 1 && P.mg_emulated;
    // tiles this launch traces (emulated: all ranks' tiles in one launch)
    const int tiles_launch = (G > 1 && !emu) ? P.tiles / G : P.tiles;
    size_t smem = run_1d_smem_bytes(P.tp, threads);
    // latency-bound (tiles <= SMs): one CTA per SM -- reserve more than half the
    // SM's shared memory so the scheduler cannot double up CTAs on one SM
    if (tiles_launch <= sms && smem < 120 * 1024) smem = 120 * 1024;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    Run1DParams args = P;
    int grid;
    if (emu) {  // G equal CTA groups, every CTA co-resident
        args.mg_ctas = std::min(P.tiles / G, (per_sm * sms) / G);
        if (args.mg_ctas < 1) return cudaErrorInvalidConfiguration;
        grid = G * args.mg_ctas;
    } else {
        grid = std::min(tiles_launch, per_sm * sms);
        if (SPLIT) grid = tiles_launch + args.split_helpers;  // helpers after the tiles' CTAs (checked by the caller)
        args.mg_ctas = grid;
    }
    if (grid_out) *grid_out = grid;
    void *kargs[] = {&args};
    return cudaLaunchCooperativeKernel((const void *)kern, dim3(grid), dim3(threads), kargs, smem, st);
}

cudaError_t launch_run_1d(const Run1DParams &P_in, int threads, int device, cudaStream_t st, int *grid_out) {
    // the split (helper CTAs) exists for the N = 64, 2 x 64-slab kernel only (ts1)
    Run1DParams P = P_in;
    if (!(P.tp.N == 64 && P.tp.slabs_per_stage == 64)) P.split_helpers = 0;
    switch (P.tp.N) {
        case 32: return launch_run<32, 16>(P, threads, device, st, grid_out);
        case 64:
            if (P.tp.slabs_per_stage == 32) return launch_run<64, 32>(P, threads, device, st, grid_out);
            if (P.tp.slabs_per_stage == 64) {
                // split only when every CTA (tiles + helpers, one per SM) can be co-resident
                int sms = 0;
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
                if (P.split_helpers > 0 && P.mg_ranks <= 1 && P.tiles + P.split_helpers <= sms)
                    return launch_run<64, 64, 0, 1>(P, threads, device, st, grid_out);
                Run1DParams q = P;
                q.split_helpers = 0;
                return launch_run<64, 64>(q, threads, device, st, grid_out);
            }
            return launch_run<64, 16>(P, threads, device, st, grid_out);
        case 128: return launch_run<128, 8>(P, threads, device, st, grid_out);
        case 256:
            if (P.tp.slabs_per_stage == 1) return launch_run<256, 1>(P, threads, device, st, grid_out);
            if (P.tp.slabs_per_stage == 2) return launch_run<256, 2>(P, threads, device, st, grid_out);
            if (P.tp.slabs_per_stage == 8) return launch_run<256, 8>(P, threads, device, st, grid_out);
            if (P.tp.slabs_per_stage == 16)
                return threads > 288 ? launch_run<256, 16, 1>(P, threads, device, st, grid_out)
                                     : launch_run<256, 16>(P, threads, device, st, grid_out);
            return launch_run<256, 4>(P, threads, device, st, grid_out);
        default: return launch_run<0, 1>(P, threads, device, st, grid_out);
    }
}

}  // namespace nufi
