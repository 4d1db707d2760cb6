// Cycle count of the d = 1 tail's phase B (warp 0: rho from 8 block sums, mean, rho',
// neutrality reductions) in isolation, one CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ubench_phaseb tools/ubench_phaseb.cu
#include <cfloat>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct Prm {
    double rho_bar, hv_d;
    double *rho_out, *stats_out;
    int N, B;
};

__global__ void phaseb(Prm p, long long *cyc, double *out) {
    __shared__ double sm[8 * 256 + 512];
    double *sb = sm, *r = sm + 8 * 256;
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) sb[i] = 1e-3 * i;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int N = p.N, B = p.B;
    for (int rep = 0; rep < 4; ++rep) {
        __syncthreads();
        long long c0 = clock64(), c1 = 0, c2 = 0, c3 = 0;
        if (warp == 0) {
            double s = 0.0;
            for (int i = lane; i < N; i += 32) {
                double S = 0.0;
                for (int b = 0; b < B; ++b) S += sb[b * N + i];
                const double ri = p.rho_bar - p.hv_d * S;
                r[i] = ri;
                s += ri;
            }
            s = warp_sum(s);
            const double neut = s / (double)N;
            c1 = clock64();
            double s2 = 0.0, m = 0.0;
            for (int i = lane; i < N; i += 32) {
                const double v = r[i] - neut;
                r[i] = v;
                p.rho_out[i] = v;
                s2 += v;
                m = fmax(m, fabs(v));
            }
            c2 = clock64();
            s2 = warp_sum(s2);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) {
                p.stats_out[0] = neut;
                p.stats_out[1] = s2 / (double)N > 1e-8 * m ? 1.0 : 0.0;
            }
            c3 = clock64();
        }
        __syncthreads();
        long long c4 = clock64();
        if (threadIdx.x == 0 && (rep == 3 || rep == 0)) { if (rep == 0) { cyc[4] = c1 - c0; cyc[5] = c4 - c0; } else {
            cyc[0] = c1 - c0;
            cyc[1] = c2 - c1;
            cyc[2] = c3 - c2;
            cyc[3] = c4 - c0; }
        }
    }
}

int main() {
    long long *cyc;
    double *buf;
    cudaMallocManaged(&cyc, 8 * sizeof(long long));
    cudaMalloc(&buf, 1024 * sizeof(double));
    for (int N : {64, 256}) {
        Prm p{1.0, 0.01, buf, buf + 512, N, 8};
        phaseb<<<1, 288>>>(p, cyc, buf);
        cudaDeviceSynchronize();
        printf("N=%d: rho+mean %lld, rho loop %lld, reductions %lld, total %lld | cold: rho+mean %lld total %lld\n", N, cyc[0],
               cyc[1], cyc[2], cyc[3], cyc[4], cyc[5]);
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock rate attr %d kHz; err %s\n", clk, cudaGetErrorString(cudaGetLastError()));
}
