// Shared-memory wavefronts of 8-byte warp loads by address pattern (throughput, 16 warps/SM):
//   32 distinct consecutive doubles (256 B), 16 distinct (128 B, pairs of lanes share),
//   8 distinct (64 B, groups of 4 lanes share), 1 (broadcast), and the rotated-tap pattern
//   of a 4-tap stencil (lane L reads tap (s - L) mod 4 of cell base + L).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ubench_bcast tools/ubench_bcast.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) lds_kernel(double *out, int iters, long long *cyc) {
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 1e-3 * i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    int base = (threadIdx.x >> 5) * 64;
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            int idx;
            if (MODE == 0) idx = base + 40 * t + lane;                 // 32 distinct
            else if (MODE == 1) idx = base + 40 * t + (lane >> 1);     // 16 distinct
            else if (MODE == 2) idx = base + 40 * t + (lane >> 2);     // 8 distinct
            else if (MODE == 3) idx = base + 40 * t;                   // broadcast
            else if (MODE == 4) idx = base + lane + ((t - lane) & 3);  // rotated taps, consecutive cells
            else if (MODE == 6) idx = base + 40 * t + (lane & 15);     // halves identical (L, L+16 share)
            else idx = base + lane + t;                                // plain taps, consecutive cells
            const double v = s[idx & 4095];
            if (t == 0) a0 += v; else if (t == 1) a1 += v; else if (t == 2) a2 += v; else a3 += v;
        }
        base += 37;
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = c1 - c0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

int main() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 2 * 256 * sizeof(double));
    cudaMallocManaged(&cyc, sizeof(long long));
    const int iters = 4096;
    const char *names[] = {"32 distinct (256 B)", "16 distinct (128 B)", "8 distinct (64 B)", "broadcast",
                           "rotated 4-tap", "plain 4-tap", "halves identical"};
    for (int mode = 0; mode < 7; ++mode) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (mode) {
                case 0: lds_kernel<0><<<296, 256>>>(out, iters, cyc); break;
                case 1: lds_kernel<1><<<296, 256>>>(out, iters, cyc); break;
                case 2: lds_kernel<2><<<296, 256>>>(out, iters, cyc); break;
                case 3: lds_kernel<3><<<296, 256>>>(out, iters, cyc); break;
                case 4: lds_kernel<4><<<296, 256>>>(out, iters, cyc); break;
                case 6: lds_kernel<6><<<296, 256>>>(out, iters, cyc); break;
                default: lds_kernel<5><<<296, 256>>>(out, iters, cyc); break;
            }
            cudaEventRecord(e1);
            cudaDeviceSynchronize();
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        // per SM: 16 warps x iters x 4 LDS
        const double lds_per_sm = 16.0 * iters * 4;
        printf("%-22s %8.3f ms  %.2f SM-cycles per warp-LDS\n", names[mode], ms, (double)*cyc / (lds_per_sm));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
