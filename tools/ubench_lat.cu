// Latency microbenchmarks for the d = 1 step tail design (one CTA / SM):
// dependent DFMA / DADD chains, a double warp-shuffle reduction, __syncthreads with
// 9 warps, DDIV, shared-memory load, and L2 (ld.global.cg) round trips on a line that
// every CTA of the grid reads at the same time.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_lat tools/ubench_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double *out, long long *cyc, const double *__restrict__ g, int iters) {
    __shared__ double sm[1024];
    const int t = threadIdx.x;
    for (int i = t; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-3;
    __syncthreads();
    double a = out[t] + 1.0, b = 0.999999;
    long long c0, c1;
    // 1. DFMA chain
    c0 = clock64();
    for (int i = 0; i < iters; ++i) a = fma(a, b, 1e-9);
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[0] = (c1 - c0) / iters;
    // 2. DADD chain
    c0 = clock64();
    for (int i = 0; i < iters; ++i) a = a + b;
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[1] = (c1 - c0) / iters;
    // 3. warp_sum of a double (5 shuffle steps)
    c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double s = a;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        a = s * 1e-30 + a;
    }
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[2] = (c1 - c0) / iters;
    // 4. __syncthreads
    c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
    }
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[3] = (c1 - c0) / iters;
    // 5. DDIV chain
    c0 = clock64();
    for (int i = 0; i < iters; ++i) a = 1.0 / a;
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[4] = (c1 - c0) / iters;
    // 6. dependent LDS.64 chain
    int idx = t;
    c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const double v = sm[idx & 1023];
        idx = (int)v + t;
    }
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[5] = (c1 - c0) / iters;
    a += idx;
    // 7. dependent ld.global.cg chain over a shared 32 KB region (all CTAs)
    int gi = t;
    c0 = clock64();
    for (int i = 0; i < 64; ++i) {
        const double v = __ldcg(g + (gi & 4095));
        gi = (int)v + t + 37 * i;
    }
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[6] = (c1 - c0) / 64;
    a += gi;
    // 8. one LDS + STS round (smem write then barrier then read), as in a tail phase
    c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        sm[t] = a;
        __syncthreads();
        a = sm[(t + 1) % blockDim.x] * 1e-30 + a;
        __syncthreads();
    }
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[7] = (c1 - c0) / iters;
    // 9. 16 independent ld.global.cg then use (one round trip with 16 in flight), all CTAs
    c0 = clock64();
    double acc = 0.0;
    for (int r = 0; r < 8; ++r) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcg(g + ((t + 288 * u + 64 * r + (int)acc) & 4095));
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += v[u];
        acc *= 1e-30;
    }
    c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[8] = (c1 - c0) / 8;
    out[blockIdx.x * blockDim.x + t] = a + acc;
}

int main() {
    double *out, *g;
    long long *cyc;
    cudaMalloc(&out, 148 * 288 * sizeof(double));
    cudaMalloc(&g, 4096 * sizeof(double));
    cudaMemset(g, 0, 4096 * sizeof(double));
    cudaMemset(out, 0, 148 * 288 * sizeof(double));
    cudaMallocManaged(&cyc, 16 * sizeof(long long));
    for (int rep = 0; rep < 2; ++rep) {
        lat_kernel<<<148, 288>>>(out, cyc, g, 256);
        cudaDeviceSynchronize();
    }
    const char *names[] = {"DFMA chain", "DADD chain", "warp_sum(double)", "__syncthreads (9 warps)", "DDIV chain",
                           "LDS.64 dependent", "ld.cg dependent (148 CTAs, 32 KB)", "STS+bar+LDS+bar round",
                           "16x ld.cg in flight + sum (148 CTAs)"};
    for (int i = 0; i < 9; ++i) printf("%-40s %lld cycles\n", names[i], cyc[i]);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
