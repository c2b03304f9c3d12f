// FP64 FMA issue probe: TFLOP/s for W warps per SM, C independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fma_probe fma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k(double* out, int iters, double a, double b) {
    double v[C];
#pragma unroll
    for (int i = 0; i < C; ++i) v[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) v[i] = fma(v[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += v[i];
    if (s == -1.2345) out[0] = s;
}

template <int C>
void run(int warps_per_sm) {
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 1 << 14;
    const int threads = 32 * warps_per_sm;  // one CTA per SM
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<C><<<148, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    k<C><<<148, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * C * iters * 148.0 * threads;
    printf("warps/SM %2d chains %2d: %6.2f TF/s\n", warps_per_sm, C, fl / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    for (int w : {4, 8, 12, 16, 32}) {
        run<1>(w);
        run<2>(w);
        run<4>(w);
        run<8>(w);
        run<16>(w);
    }
    return 0;
}
