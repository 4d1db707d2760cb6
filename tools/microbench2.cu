// microbench2.cu -- d=1 substep chain vs warps per SM (smem slabs, no TMA).
#include <cstdio>
#include <cuda_runtime.h>

template <int LAYOUT>  // 0: SoA 3xLDS.64, 1: AoS LDS.128 + LDS.64, 2: SoA, drift folded into the kick
__global__ void sub_kernel(double *out, long long *cyc, int steps) {
    extern __shared__ double sm[];
    const int N = 64, SL = 16;
    for (int i = threadIdx.x; i < SL * 4 * N; i += blockDim.x) sm[i] = 1e-6 * ((i * 37) % 101) - 5e-5;
    __syncthreads();
    double X = (threadIdx.x & 31) - 0.5 + 0.123 * (threadIdx.x >> 5), V = 0.3 + 0.01 * (threadIdx.x >> 5);
    const double M = 6755399441055744.0;
    long long t0 = clock64();
    for (int k = 0; k < steps; k += SL) {
#pragma unroll
        for (int q = SL - 1; q >= 0; --q) {
            if (LAYOUT == 2) {
                // X already drifted; the kick also produces the next drifted position
                const double s = X + M;
                const double fc = X - (s - M);
                const char *b = reinterpret_cast<const char *>(sm + q * 3 * N);
                const double *p = reinterpret_cast<const double *>(b + (((unsigned)__double_as_longlong(s) & 63u) << 3));
                const double XmV = X - V;
                const double A = p[0], B = p[N], C = p[2 * N];
                const double t = fma(fc, C, B);
                X = fma(-fc, t, XmV - A);
                V = fma(fc, t, V + A);
                continue;
            }
            X -= V;
            const double s = X + M;
            const int i = (int)((unsigned)__double_as_longlong(s) & 63u);
            const double fc = X - (s - M);
            if (LAYOUT == 0) {
                const double *sl = sm + q * 3 * N;
                V = fma(fc, fma(fc, sl[2 * N + i], sl[N + i]), V + sl[i]);
            } else {
                const double *sl = sm + q * 4 * N + 4 * i;
                const double2 ab = *reinterpret_cast<const double2 *>(sl);
                V = fma(fc, fma(fc, sl[2], ab.y), V + ab.x);
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = X + V;
}

int main() {
    double *out; long long *cyc;
    cudaMalloc(&out, 148 * 1024 * 8); cudaMallocManaged(&cyc, 148 * 8);
    const int steps = 4096;
    for (int layout = 0; layout < 3; ++layout)
        for (int w : {1, 2, 4, 8, 12, 16, 24, 32}) {
            auto k = layout == 2 ? sub_kernel<2> : (layout ? sub_kernel<1> : sub_kernel<0>);
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 4 * 64 * 8);
            k<<<148, 32 * w, 16 * 4 * 64 * 8>>>(out, cyc, 64);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k<<<148, 32 * w, 16 * 4 * 64 * 8>>>(out, cyc, steps);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            cudaDeviceSynchronize();
            printf("layout %d warps/SM %2d: %.1f cycles/substep (clock64), %.2f ns/substep (events), %.3e point-steps/s\n",
                   layout, w, (double)cyc[0] / steps, ms * 1e6 / steps, 148.0 * 32 * w * steps / (ms * 1e-3));
        }
    return 0;
}
