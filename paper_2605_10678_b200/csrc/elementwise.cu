// elementwise.cu -- the fused, coalesced elementwise passes of Eq. (3)/(4).
//
// truncate_deconv (type 1, Steps 3 + 4):
//     fk[n] = B[n mod nf] * p1(n1) p2(n2) p3(n3)
//   chi keeps the index set {0..N/2-1} U {nf-N/2..nf-1} per axis;
//   one thread per retained mode, consecutive threads read consecutive x cells
//   of the grid row (two contiguous segments per row) and write consecutive modes.
// pad_precorrect (type 2, D then chi^T, "pre-correction"
//   PAPER.md:382): one thread per FINE cell writes every cell of the grid,
//   fk[n] * p(n) on the retained set and zero elsewhere -- the zero fill and the
//   pre-correction are a single streaming pass, no separate memset.
#include "internal.cuh"

namespace nufft {

namespace {

constexpr int kEwThreads = 256;

__device__ __forceinline__ double2 cmul_real(double2 a, double s) { return {a.x * s, a.y * s}; }
__device__ __forceinline__ float2 cmul_real(float2 a, float s) { return {a.x * s, a.y * s}; }

// mode storage index i -> signed mode n (modeord 0: centered, 1: FFT order)
__device__ __forceinline__ int64_t mode_of(int64_t i, int64_t N, int modeord) {
    return modeord == 0 ? i - N / 2 : (i < N / 2 ? i : i - N);
}
// signed mode -> storage index
__device__ __forceinline__ int64_t index_of(int64_t n, int64_t N, int modeord) {
    return modeord == 0 ? n + N / 2 : (n >= 0 ? n : n + N);
}

template <typename T>
__global__ void __launch_bounds__(kEwThreads)
    truncate_deconv_kernel(const typename Cx<T>::type* __restrict__ grid, int64_t nf1,
                           int64_t nf2, int64_t nf3, int64_t N1, int64_t N2, int64_t N3,
                           const T* __restrict__ p1, const T* __restrict__ p2,
                           const T* __restrict__ p3, int modeord,
                           typename Cx<T>::type* __restrict__ fk) {
    const int64_t total = N1 * N2 * N3;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i1 = i % N1, i2 = (i / N1) % N2, i3 = i / (N1 * N2);
        const int64_t n1 = mode_of(i1, N1, modeord), n2 = mode_of(i2, N2, modeord),
                      n3 = mode_of(i3, N3, modeord);
        const int64_t m1 = n1 < 0 ? n1 + nf1 : n1, m2 = n2 < 0 ? n2 + nf2 : n2,
                      m3 = n3 < 0 ? n3 + nf3 : n3;
        const T s = p1[n1 + N1 / 2] * p2[n2 + N2 / 2] * p3[n3 + N3 / 2];
        fk[i] = cmul_real(grid[m1 + nf1 * (m2 + nf2 * m3)], s);
    }
}

template <typename T>
__global__ void __launch_bounds__(kEwThreads)
    pad_precorrect_kernel(const typename Cx<T>::type* __restrict__ fk, int64_t N1, int64_t N2,
                          int64_t N3, const T* __restrict__ p1, const T* __restrict__ p2,
                          const T* __restrict__ p3, int modeord, int64_t nf1, int64_t nf2,
                          int64_t nf3, typename Cx<T>::type* __restrict__ grid) {
    using C = typename Cx<T>::type;
    const int64_t total = nf1 * nf2 * nf3;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < total;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m1 = m % nf1, m2 = (m / nf1) % nf2, m3 = m / (nf1 * nf2);
        // retained iff m < N/2 (n = m) or m >= nf - N/2 (n = m - nf)
        const bool k1 = m1 < N1 / 2 || m1 >= nf1 - N1 / 2;
        const bool k2 = m2 < N2 / 2 || m2 >= nf2 - N2 / 2;
        const bool k3 = m3 < N3 / 2 || m3 >= nf3 - N3 / 2;
        C v{0, 0};
        if (k1 && k2 && k3) {
            const int64_t n1 = m1 < N1 / 2 ? m1 : m1 - nf1;
            const int64_t n2 = m2 < N2 / 2 ? m2 : m2 - nf2;
            const int64_t n3 = m3 < N3 / 2 ? m3 : m3 - nf3;
            const T s = p1[n1 + N1 / 2] * p2[n2 + N2 / 2] * p3[n3 + N3 / 2];
            const int64_t i = index_of(n1, N1, modeord) +
                              N1 * (index_of(n2, N2, modeord) + N2 * index_of(n3, N3, modeord));
            v = cmul_real(fk[i], s);
        }
        grid[m] = v;
    }
}

inline unsigned ew_grid(int64_t n) {
    int64_t b = (n + kEwThreads - 1) / kEwThreads;
    const int64_t cap = 148 * 32;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

template <typename T>
cudaError_t launch_truncate_deconv(const typename Cx<T>::type* grid, const int64_t nf[3],
                                   const int64_t N[3], const T* p1, const T* p2, const T* p3,
                                   int modeord, typename Cx<T>::type* fk, cudaStream_t s) {
    truncate_deconv_kernel<T><<<ew_grid(N[0] * N[1] * N[2]), kEwThreads, 0, s>>>(
        grid, nf[0], nf[1], nf[2], N[0], N[1], N[2], p1, p2, p3, modeord, fk);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pad_precorrect(const typename Cx<T>::type* fk, const int64_t N[3],
                                  const T* p1, const T* p2, const T* p3, int modeord,
                                  const int64_t nf[3], typename Cx<T>::type* grid,
                                  cudaStream_t s) {
    pad_precorrect_kernel<T><<<ew_grid(nf[0] * nf[1] * nf[2]), kEwThreads, 0, s>>>(
        fk, N[0], N[1], N[2], p1, p2, p3, modeord, nf[0], nf[1], nf[2], grid);
    return cudaGetLastError();
}

template cudaError_t launch_truncate_deconv<float>(const float2*, const int64_t*, const int64_t*,
                                                   const float*, const float*, const float*, int,
                                                   float2*, cudaStream_t);
template cudaError_t launch_truncate_deconv<double>(const double2*, const int64_t*,
                                                    const int64_t*, const double*, const double*,
                                                    const double*, int, double2*, cudaStream_t);
template cudaError_t launch_pad_precorrect<float>(const float2*, const int64_t*, const float*,
                                                  const float*, const float*, int,
                                                  const int64_t*, float2*, cudaStream_t);
template cudaError_t launch_pad_precorrect<double>(const double2*, const int64_t*, const double*,
                                                   const double*, const double*, int,
                                                   const int64_t*, double2*, cudaStream_t);

}  // namespace nufft
