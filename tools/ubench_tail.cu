// The real d = 1 step tail (field_update_1d_body) on synthetic partials, one CTA of
// 288 threads or G CTAs at once, phase times from the NUFI_STAMP hook (globaltimer).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//      -I paper_2301_05581_b200/csrc -o tools/bin/ubench_tail tools/ubench_tail.cu
#include <cstdio>
#include <vector>

#include "field_common.cuh"

using namespace nufi;

__global__ void tail_kernel(FieldParams p, int reps, unsigned long long *stamps, int getenv_twice) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *sm = reinterpret_cast<double *>(smem_raw);
    for (int r = 0; r < reps; ++r) {
        FieldParams q = p;
        q.tstamps = (blockIdx.x == 0 && r == reps - 1) ? stamps : nullptr;
        if (blockIdx.x != 0) q.rho_out = q.stats_out = q.W_out = q.E_out = q.coeffs_out = nullptr;
        if (blockIdx.x != 0) q.hist = q.ev_hist = nullptr;
        if (threadIdx.x == 0 && r == reps - 1) {
            long long c0 = clock64();
            int j = 0;
            for (int k = 0; k < 16; ++k) j = (int)__ldcg(p.sums + ((j + 97 * k) & 4095)) + j;
            long long c1 = clock64();
            int jj = 0;
            for (int k = 0; k < 16; ++k) jj = (int)__ldg(p.gc + ((jj + 7 * k) & 63)) + jj;
            long long c2 = clock64();
            stamps[12] = (c1 - c0) / 16 + (j == 12345);
            stamps[13] = (c2 - c1) / 16 + (jj == 12345);
        }
        if (getenv_twice) {
            FieldParams q2 = q;
            q2.tstamps = nullptr;
            field_update_body(q2, sm);
            __syncthreads();
        }
        unsigned long long t0, t1;
        const long long k0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0)::"memory");
        field_update_body(q, sm);
        __syncthreads();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)::"memory");
        const long long k1 = clock64();
        if (q.tstamps && threadIdx.x == 0) {
            stamps[10] = t0;
            stamps[11] = t1;
            stamps[14] = (unsigned long long)(k1 - k0);
        }
    }
}

int main(int argc, char **argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 64;
    const int ctas = argc > 2 ? atoi(argv[2]) : 1;
    const int B = 8, rpb = 8, mm = 16, SLAB = ev_slab_elems(1, N);
    std::vector<double> h(16 * 4096, 0.0);
    auto dbuf = [&](size_t n, double fill) {
        double *p;
        cudaMalloc(&p, n * sizeof(double));
        for (size_t i = 0; i < n && i < h.size(); ++i) h[i] = fill * (1.0 + 1e-3 * (double)(i % 97));
        cudaMemcpy(p, h.data(), std::min(n, h.size()) * sizeof(double), cudaMemcpyHostToDevice);
        return p;
    };
    FieldParams p{};
    p.d = 1;
    p.N = N;
    p.nodes = N;
    p.B = B;
    p.L = 12.566370614359172;
    p.inv_h = N / p.L;
    p.hv_d = 1.0 / 512;
    p.rho_bar = 1.0;
    p.L_d = p.L;
    p.K = -0.01;
    p.twc = dbuf(N, 0.5);
    p.tws = dbuf(N, 0.25);
    p.fac = dbuf(2 * N, 0.1);
    p.k2 = dbuf(N, 1.0);
    p.gc = dbuf(N, 0.01);
    p.gp = dbuf(N, 0.02);
    p.sums = dbuf((size_t)B * rpb * N, 1.0);
    p.rows_per_block = rpb;
    p.minmax = dbuf((size_t)B * mm * 2, 0.5);
    p.mm_per_block = mm;
    p.slot = 3;
    p.hist = dbuf(8 * N, 0.0);
    p.ev_hist = dbuf(8 * SLAB, 0.0);
    p.ev_slab_elems = SLAB;
    p.rho_out = dbuf(N, 0.0);
    p.stats_out = dbuf(4, 0.0);
    p.W_out = dbuf(4, 0.0);
    p.E_out = dbuf(N, 0.0);
    cudaMalloc(&p.status, sizeof(int));
    cudaMemset(p.status, 0, sizeof(int));
    cudaMalloc(&p.hist_len, sizeof(int64_t));
    unsigned long long *st, *dst;
    st = new unsigned long long[16];
    cudaMalloc(&dst, 16 * sizeof(unsigned long long));
    const bool stage = argc > 3 && atoi(argv[3]);
    p.stage_cap = stage ? (int64_t)B * rpb * N + 2 * B * mm : 0;
    const size_t smem = (field_smem_doubles(N, N, true) + p.stage_cap) * sizeof(double);
    cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0.f;
    for (int it = 0; it < 3; ++it) {
        cudaMemset(dst, 0, 16 * sizeof(unsigned long long));
        cudaEventRecord(e0);
        tail_kernel<<<ctas, 288, smem>>>(p, 200, dst, argc > 4 ? atoi(argv[4]) : 0);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(st, dst, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    }
    printf("kernel: %.2f us per tail\n", ms * 1e3 / 200);
    printf("N=%d ctas=%d stage=%d:", N, ctas, (int)stage);
    for (int k = 0; k < 10; ++k)
        if (st[k]) printf(" %d:%.2f", k, (double)(st[k] - st[10]) * 1e-3);
    printf(" end:%.2f  ldcg-chain %llu cyc, ldg-chain %llu cyc, tail %llu cyc = %.0f MHz", (double)(st[11] - st[10]) * 1e-3, st[12], st[13], st[14], (double)st[14] / (double)(st[11] - st[10]) * 1e3);
    printf(" us   (%s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
