// peak.cu -- FP64 vector (DFMA) throughput microbenchmark, the roofline
// denominator for the trace kernel (MEASURED_PEAKS.json has no FP64 entry).
// 8 independent DFMA chains per thread, grid = 4 CTAs x 256 threads per SM.
#include <cuda_runtime.h>

#include "nufi.h"

namespace nufi {

__global__ void __launch_bounds__(256) dfma_peak_kernel(double *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 123.456) out[0] = s;  // never true; keeps the chains alive
}

}  // namespace nufi

extern "C" int nufi_fp64_peak(int device, double *tflops, double *ms) {
    if (cudaSetDevice(device) != cudaSuccess) return NUFI_ERR_CUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double *out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return NUFI_ERR_CUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int ctas = sms * 4, threads = 256, iters = 2048;
    nufi::dfma_peak_kernel<<<ctas, threads>>>(out, 64, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        nufi::dfma_peak_kernel<<<ctas, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t = 0;
        cudaEventElapsedTime(&t, e0, e1);
        if (t < best) best = t;
    }
    const double flops = 2.0 * 8 * 16 * (double)iters * ctas * threads;
    *tflops = flops / (best * 1e-3) / 1e12;
    if (ms) *ms = best;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? NUFI_OK : NUFI_ERR_CUDA;
}
