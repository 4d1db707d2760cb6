// microbench.cu -- dependent-chain latencies on the B200 (cycles, clock64):
// DADD, DFMA, DMUL, LDS.64, magic-rint+index+LDS (the d=1 substep chain).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double *out, long long *cyc, int iters, double a, double b) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7) & 1023) * 1e-300 + 0.0;
    __syncthreads();
    double x = threadIdx.x * 1e-9 + 1.0;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = x + a; x = x + b; x = x + a; x = x + b;
    }
    t1 = clock64();
    cyc[0] = (t1 - t0);
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b);
    }
    t1 = clock64();
    cyc[1] = (t1 - t0);
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        x = x * a; x = x * b; x = x * a; x = x * b;
    }
    t1 = clock64();
    cyc[2] = (t1 - t0);
    // LDS.64 pointer chase (index from value)
    int idx = threadIdx.x & 1;
    double acc = 0;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        double v = sm[idx]; idx = (int)(__double_as_longlong(v) & 1); acc += v;
        v = sm[idx]; idx = (int)(__double_as_longlong(v) & 1);
        v = sm[idx]; idx = (int)(__double_as_longlong(v) & 1);
        v = sm[idx]; idx = (int)(__double_as_longlong(v) & 1);
    }
    t1 = clock64();
    cyc[3] = (t1 - t0);
    // substep-like chain: X -= V; s = X + M; i = lo(s)&63; y = sm[i]; V = fma(f, y, V)
    double X = 3.25 + threadIdx.x, V = 1e-3, M = 6755399441055744.0;
    t0 = clock64();
    for (int i = 0; i < iters * 4; ++i) {
        X = X - V;
        double s = X + M;
        double r = s - M;
        double f = X - r;
        int ii = (int)(__double_as_longlong(s) & 63);
        double A = sm[ii], B = sm[64 + ii], C = sm[128 + ii];
        double t = fma(f, C, B);
        V = fma(f, t, V + A);
    }
    t1 = clock64();
    cyc[4] = (t1 - t0);
    out[threadIdx.x] = x + acc + X + V;
}

int main() {
    double *out; long long *cyc;
    cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 8 * 8);
    const int iters = 4096;
    lat_kernel<<<1, 32>>>(out, cyc, 64, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    lat_kernel<<<1, 32>>>(out, cyc, iters, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    const char *names[5] = {"DADD", "DFMA", "DMUL", "LDS.64 chase", "d1 substep"};
    for (int i = 0; i < 5; ++i) printf("%-14s %.2f cycles/op\n", names[i], (double)cyc[i] / (4.0 * iters));
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock %d kHz\n", clk);
    return 0;
}
