// peak.cu -- on-box FMA-pipe peak (the ALU roofline denominator of bench.py).
//
// the spread / interp are bound by the floating-point FMA pipe
// at w >= 5; the datasheet-derived peak (148 SM x lanes x 2 x clock) is checked
// by measuring it on the GPU that runs the bench: every thread runs 8
// independent FMA chains (enough to cover the pipe latency at full occupancy)
// over a grid of 148 x 8 CTAs of 256 threads, timed with CUDA events.
#include <cuda_runtime.h>

#include "plan_state.h"

namespace nufft {

template <typename T>
__global__ void __launch_bounds__(256) fma_peak_kernel(T* out, int iters, T a, T b) {
    T v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (T)(threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fma(v[k], a, b);
    }
    T s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == (T)-1.2345) out[0] = s;  // keeps the chains live
}

template <typename T>
static int fma_peak_t(double* tflops, cudaStream_t st) {
    int dev = 0, sms = 0;
    NUFFT_CK(cudaGetDevice(&dev));
    NUFFT_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    T* out = nullptr;
    NUFFT_CK(cudaMallocAsync(&out, sizeof(T), st));
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t e0, e1;
    NUFFT_CK(cudaEventCreate(&e0));
    NUFFT_CK(cudaEventCreate(&e1));
    fma_peak_kernel<T><<<blocks, threads, 0, st>>>(out, iters, (T)0.999999, (T)1e-7);  // warm
    NUFFT_CK(cudaEventRecord(e0, st));
    const int reps = 5;
    for (int r = 0; r < reps; ++r)
        fma_peak_kernel<T><<<blocks, threads, 0, st>>>(out, iters, (T)0.999999, (T)1e-7);
    NUFFT_CK(cudaEventRecord(e1, st));
    NUFFT_CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    NUFFT_CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    NUFFT_CK(cudaFreeAsync(out, st));
    NUFFT_CK(cudaStreamSynchronize(st));
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads * reps;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return NUFFT_OK;
}

}  // namespace nufft

extern "C" int nufft_fma_peak(int precision, void* stream, double* tflops) {
    if (!tflops || (precision != NUFFT_F32 && precision != NUFFT_F64)) return NUFFT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    return precision == NUFFT_F64 ? nufft::fma_peak_t<double>(tflops, st)
                                  : nufft::fma_peak_t<float>(tflops, st);
}
