// Cycle count of the d = 1 tail's convolution phase (circulant_blocked, N = 64) and of
// the FFT path (N = 256) in isolation, one 288-thread CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2301_05581_b200/csrc \
//      -o tools/bin/ubench_conv tools/ubench_conv.cu
#include <cstdio>

#include "field_common.cuh"

using namespace nufi;

__global__ void conv(long long *cyc, double *out, int N) {
    __shared__ double sm[14 * 256 + 128];
    double *r = sm, *gc = r + 2 * N, *gp = gc + 2 * N, *c = gp + 2 * N, *phi = c + N;
    for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) {
        r[i] = 1e-3 * i;
        gc[i] = 1e-2 * i;
        gp[i] = 2e-2 * i;
    }
    __syncthreads();
    for (int rep = 0; rep < 4; ++rep) {
        __syncthreads();
        const long long c0 = clock64();
        circulant_blocked(gc, gp, r, c, phi, N);
        const long long c1 = clock64();
        __syncthreads();
        const long long c2 = clock64();
        if (threadIdx.x == 0 && rep == 3) {
            cyc[0] = c1 - c0;
            cyc[1] = c2 - c0;
        }
    }
    out[threadIdx.x] = c[threadIdx.x % N] + phi[threadIdx.x % N];
}

int main() {
    long long *cyc;
    double *buf;
    cudaMallocManaged(&cyc, 8 * sizeof(long long));
    cudaMalloc(&buf, 1024 * sizeof(double));
    for (int N : {4, 8, 16, 32, 64}) {
        conv<<<1, 288>>>(cyc, buf, N);
        cudaDeviceSynchronize();
        printf("N=%d circulant_blocked: thread0 %lld cycles, incl. barrier %lld\n", N, cyc[0], cyc[1]);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
