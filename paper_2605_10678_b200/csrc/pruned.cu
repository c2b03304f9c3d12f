// pruned.cu -- the paper's sigma = 2 split of the fine-grid FFT (PAPER.md:237-247,
// Eq. (7)), an option of the complex transforms
// (opts.fft_method = 1).
//
// With nf = 2N per axis and fine index j = 2m + p (p in {0, 1}^3 the parity of
// each coordinate), the fine-grid DFT with sign s at a retained mode k (|k| < N/2)
// factors into eight DFTs of size N^3, one per parity sub-grid G_p[m] = G[2m + p]:
//
//     sum_j G[j] e^{s i 2 pi j.k / (2N)}
//         = sum_p e^{s i pi p.k / N} S_p[k mod N],
//     S_p[k'] = sum_m G_p[m] e^{s i 2 pi m.k' / N}.
//
// Type 1: the eight S_p are cuFFT N^3 transforms read straight from the strided
// fine grid (input stride 2, no copy); pruned_combine applies the twiddles of
// each retained mode, sums the eight terms and deconvolves (chi and D fused, one
// thread per output mode).  Type 2 is the mirror (the conjugate-twiddle zero pad):
// pruned_split writes H_p[k mod N] = P[k] e^{-s i pi p.k / N} for the
// pre-corrected modes P = D f, and eight inverse N^3 transforms write the parity
// sub-grids of the fine grid (output stride 2).  Only the N^3 retained modes of
// each sub-grid transform are ever formed: the zero padding of chi^T and the
// discarded modes of chi are never touched.
#include "internal.cuh"

namespace nufft {

namespace {

constexpr int kPrunedThreads = 256;

// signed mode k of storage index i (modeord 0: centered, 1: FFT order)
__device__ __forceinline__ int64_t mode_of(int64_t i, int64_t n, int modeord) {
    return modeord ? (i < n / 2 ? i : i - n) : i - n / 2;
}

template <typename T> struct CxOps;
template <> struct CxOps<double> {
    using C = double2;
    __device__ static C tw(double s, int64_t k, int64_t n) {  // e^{s i pi k / n}
        double sn, cs;
        sincospi(s * (double)k / (double)n, &sn, &cs);
        return C{cs, sn};
    }
    __device__ static C mul(C a, C b) { return C{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
    __device__ static C add(C a, C b) { return C{a.x + b.x, a.y + b.y}; }
    __device__ static C scale(C a, double r) { return C{a.x * r, a.y * r}; }
};
template <> struct CxOps<float> {
    using C = float2;
    __device__ static C tw(double s, int64_t k, int64_t n) {  // twiddles in fp64, rounded
        double sn, cs;
        sincospi(s * (double)k / (double)n, &sn, &cs);
        return C{(float)cs, (float)sn};
    }
    __device__ static C mul(C a, C b) { return C{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
    __device__ static C add(C a, C b) { return C{a.x + b.x, a.y + b.y}; }
    __device__ static C scale(C a, float r) { return C{a.x * r, a.y * r}; }
};

// fk[i] = p1 p2 p3 (k) sum_p t(k)^p S_p[k mod N]; S = 8 contiguous N^3 blocks, p = px + 2 py + 4 pz
template <typename T>
__global__ void __launch_bounds__(kPrunedThreads) pruned_combine_kernel(
    const typename Cx<T>::type* __restrict__ S, int64_t N1, int64_t N2, int64_t N3,
    const T* __restrict__ p1, const T* __restrict__ p2, const T* __restrict__ p3, int modeord,
    double s, typename Cx<T>::type* __restrict__ fk) {
    using O = CxOps<T>;
    using C = typename Cx<T>::type;
    const int64_t nm = N1 * N2 * N3;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i1 = i % N1, i2 = (i / N1) % N2, i3 = i / (N1 * N2);
        const int64_t k1 = mode_of(i1, N1, modeord), k2 = mode_of(i2, N2, modeord),
                      k3 = mode_of(i3, N3, modeord);
        const int64_t r = ((((k3 + N3) % N3) * N2 + (k2 + N2) % N2) * N1) + (k1 + N1) % N1;
        const C tx = O::tw(s, k1, N1), ty = O::tw(s, k2, N2), tz = O::tw(s, k3, N3);
        C a[4];  // sum over px first, then py, then pz (Horner in the twiddles)
#pragma unroll
        for (int q = 0; q < 4; ++q) a[q] = O::add(S[(2 * q) * nm + r], O::mul(tx, S[(2 * q + 1) * nm + r]));
        const C b0 = O::add(a[0], O::mul(ty, a[1])), b1 = O::add(a[2], O::mul(ty, a[3]));
        const C f = O::add(b0, O::mul(tz, b1));
        fk[i] = O::scale(f, p1[k1 + N1 / 2] * p2[k2 + N2 / 2] * p3[k3 + N3 / 2]);
    }
}

// H_p[k mod N] = P[k] e^{s i pi p.k / N}, P = D fk (the sign s is the type-2 FFT's)
template <typename T>
__global__ void __launch_bounds__(kPrunedThreads) pruned_split_kernel(
    const typename Cx<T>::type* __restrict__ fk, int64_t N1, int64_t N2, int64_t N3,
    const T* __restrict__ p1, const T* __restrict__ p2, const T* __restrict__ p3, int modeord,
    double s, typename Cx<T>::type* __restrict__ H) {
    using O = CxOps<T>;
    using C = typename Cx<T>::type;
    const int64_t nm = N1 * N2 * N3;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i1 = i % N1, i2 = (i / N1) % N2, i3 = i / (N1 * N2);
        const int64_t k1 = mode_of(i1, N1, modeord), k2 = mode_of(i2, N2, modeord),
                      k3 = mode_of(i3, N3, modeord);
        const int64_t r = ((((k3 + N3) % N3) * N2 + (k2 + N2) % N2) * N1) + (k1 + N1) % N1;
        const C P = O::scale(fk[i], p1[k1 + N1 / 2] * p2[k2 + N2 / 2] * p3[k3 + N3 / 2]);
        const C tx = O::tw(s, k1, N1), ty = O::tw(s, k2, N2), tz = O::tw(s, k3, N3);
        const C px[2] = {P, O::mul(P, tx)};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const C y0 = px[q], y1 = O::mul(px[q], ty);
            H[(q + 0) * nm + r] = y0;
            H[(q + 2) * nm + r] = y1;
            H[(q + 4) * nm + r] = O::mul(y0, tz);
            H[(q + 6) * nm + r] = O::mul(y1, tz);
        }
    }
}

inline int grid_for(int64_t n) {
    int64_t b = (n + kPrunedThreads - 1) / kPrunedThreads;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

template <typename T>
cudaError_t launch_pruned_combine(const typename Cx<T>::type* S, const int64_t N[3], const T* p1,
                                  const T* p2, const T* p3, int modeord, int sign,
                                  typename Cx<T>::type* fk, cudaStream_t st) {
    const int64_t nm = N[0] * N[1] * N[2];
    if (nm > 0)
        pruned_combine_kernel<T><<<grid_for(nm), kPrunedThreads, 0, st>>>(
            S, N[0], N[1], N[2], p1, p2, p3, modeord, sign < 0 ? -1.0 : 1.0, fk);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pruned_split(const typename Cx<T>::type* fk, const int64_t N[3], const T* p1,
                                const T* p2, const T* p3, int modeord, int sign,
                                typename Cx<T>::type* H, cudaStream_t st) {
    const int64_t nm = N[0] * N[1] * N[2];
    if (nm > 0)
        pruned_split_kernel<T><<<grid_for(nm), kPrunedThreads, 0, st>>>(
            fk, N[0], N[1], N[2], p1, p2, p3, modeord, sign < 0 ? -1.0 : 1.0, H);
    return cudaGetLastError();
}

template cudaError_t launch_pruned_combine<double>(const double2*, const int64_t*, const double*,
                                                   const double*, const double*, int, int,
                                                   double2*, cudaStream_t);
template cudaError_t launch_pruned_combine<float>(const float2*, const int64_t*, const float*,
                                                  const float*, const float*, int, int, float2*,
                                                  cudaStream_t);
template cudaError_t launch_pruned_split<double>(const double2*, const int64_t*, const double*,
                                                 const double*, const double*, int, int, double2*,
                                                 cudaStream_t);
template cudaError_t launch_pruned_split<float>(const float2*, const int64_t*, const float*,
                                                const float*, const float*, int, int, float2*,
                                                cudaStream_t);

}  // namespace nufft
