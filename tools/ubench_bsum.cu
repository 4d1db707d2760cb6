// Cycle cost of the tail's block-sum pass from staged shared memory: 512 outputs, 8 rows
// each, 288 threads (2 outputs per thread), then a (min, max) warp reduction.
#include <cfloat>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void bsum(long long *cyc, double *out, int N, int B, int rpb) {
    __shared__ double stg[4096 + 256];
    __shared__ double sb[512];
    for (int i = threadIdx.x; i < 4096 + 256; i += blockDim.x) stg[i] = 1e-3 * i;
    __syncthreads();
    const int T = blockDim.x, t0 = threadIdx.x;
    long long c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    for (int rep = 0; rep < 4; ++rep) {
        __syncthreads();
        c0 = clock64();
        const int logN = 31 - __clz(N);
        for (int it = t0; it < B * N; it += T) {
            const double *src = stg + (size_t)(it >> logN) * rpb * N + (it & (N - 1));
            double Sb = 0.0;
            for (int q0 = 0; q0 < rpb; q0 += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = src[(size_t)(q0 + u < rpb ? q0 + u : rpb - 1) * N];
#pragma unroll
                for (int u = 0; u < 8; ++u) Sb = q0 + u < rpb ? Sb + v[u] : Sb;
            }
            sb[it] = Sb;
        }
        c1 = clock64();
        double mn = DBL_MAX, mx = -DBL_MAX;
        for (int q = t0; q < 128; q += T) {
            mn = fmin(mn, stg[4096 + 2 * q]);
            mx = fmax(mx, stg[4096 + 2 * q + 1]);
        }
        c2 = clock64();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = mn + mx;
        c3 = clock64();
    }
    if (threadIdx.x == 0) {
        cyc[0] = c1 - c0;
        cyc[1] = c2 - c1;
        cyc[2] = c3 - c2;
    }
    out[threadIdx.x] = sb[threadIdx.x % 512];
}

int main() {
    long long *cyc;
    double *out;
    cudaMallocManaged(&cyc, 8 * sizeof(long long));
    cudaMalloc(&out, 1024 * sizeof(double));
    bsum<<<1, 288>>>(cyc, out, 64, 8, 8);
    cudaDeviceSynchronize();
    printf("block sums %lld cyc, minmax loads %lld cyc, shuffles %lld cyc (%s)\n", cyc[0], cyc[1], cyc[2],
           cudaGetErrorString(cudaGetLastError()));
}
