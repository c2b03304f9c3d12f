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
// Real-valued transforms run the FFT on the
// half spectrum H (nf3 x nf2 x (nf1/2 + 1), x fastest) of a real fine grid:
// truncate_deconv_r2c completes the retained modes by Hermitian symmetry
// (B[q] = conj(B[-q]) for a real grid); pad_precorrect_c2r writes the half
// spectrum of the Hermitian part of the pre-corrected modes, whose C2R
// transform is Re(sum_n fk[n] p(n) e^{s i n x}) exactly.
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

// Row-blocked launch of the pad pass: a block walks fine-grid rows (fixed y, z) with
// L = 32..256 threads per row and kEwThreads / L rows at a time, so the per-row index
// arithmetic (64-bit divisions) is done once per row, not once per cell, and rows
// outside the retained set are a plain zero stream (C2b 74 -> 64 us, C3 529 -> 414 us)
__host__ __device__ __forceinline__ int row_lanes(int64_t n1) {
    return n1 <= 32 ? 32 : n1 <= 64 ? 64 : n1 <= 128 ? 128 : 256;
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
    const int L = row_lanes(nf1), RB = kEwThreads / L;
    const int tx = threadIdx.x % L, ty = threadIdx.x / L;
    const int64_t rows = nf2 * nf3;
    for (int64_t r = (int64_t)blockIdx.x * RB + ty; r < rows; r += (int64_t)gridDim.x * RB) {
        const int64_t m2 = r % nf2, m3 = r / nf2;
        C* grow = grid + nf1 * r;
        // retained iff m < N/2 (n = m) or m >= nf - N/2 (n = m - nf)
        const bool k23 = (m2 < N2 / 2 || m2 >= nf2 - N2 / 2) && (m3 < N3 / 2 || m3 >= nf3 - N3 / 2);
        if (!k23) {
            for (int64_t m1 = tx; m1 < nf1; m1 += L) grow[m1] = C{0, 0};
            continue;
        }
        const int64_t n2 = m2 < N2 / 2 ? m2 : m2 - nf2;
        const int64_t n3 = m3 < N3 / 2 ? m3 : m3 - nf3;
        const T s23 = p2[n2 + N2 / 2] * p3[n3 + N3 / 2];
        const C* frow =
            fk + N1 * (index_of(n2, N2, modeord) + N2 * index_of(n3, N3, modeord));
        for (int64_t m1 = tx; m1 < nf1; m1 += L) {
            C v{0, 0};
            if (m1 < N1 / 2 || m1 >= nf1 - N1 / 2) {
                const int64_t n1 = m1 < N1 / 2 ? m1 : m1 - nf1;
                v = cmul_real(frow[index_of(n1, N1, modeord)], p1[n1 + N1 / 2] * s23);
            }
            grow[m1] = v;
        }
    }
}

__device__ __forceinline__ double2 cconj(double2 a) { return {a.x, -a.y}; }
__device__ __forceinline__ float2 cconj(float2 a) { return {a.x, -a.y}; }

// type 1, real strengths.  H = R2C(G) (exponent -).  conj_all: the type-1 sign is +
// (iflag = +1), whose transform of a real grid is conj(H).
template <typename T>
__global__ void __launch_bounds__(kEwThreads)
    truncate_deconv_r2c_kernel(const typename Cx<T>::type* __restrict__ H, int64_t nf1,
                               int64_t nf2, int64_t nf3, int64_t N1, int64_t N2, int64_t N3,
                               const T* __restrict__ p1, const T* __restrict__ p2,
                               const T* __restrict__ p3, int modeord, int conj_all,
                               typename Cx<T>::type* __restrict__ fk) {
    using C = typename Cx<T>::type;
    const int64_t hx = nf1 / 2 + 1;
    const int64_t total = N1 * N2 * N3;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i1 = i % N1, i2 = (i / N1) % N2, i3 = i / (N1 * N2);
        const int64_t n1 = mode_of(i1, N1, modeord), n2 = mode_of(i2, N2, modeord),
                      n3 = mode_of(i3, N3, modeord);
        const bool mirror = n1 < 0;  // read the conjugate partner -n in the stored half
        const int64_t a1 = mirror ? -n1 : n1, a2 = mirror ? -n2 : n2, a3 = mirror ? -n3 : n3;
        const int64_t m2 = a2 < 0 ? a2 + nf2 : a2, m3 = a3 < 0 ? a3 + nf3 : a3;
        C v = H[a1 + hx * (m2 + nf2 * m3)];
        if (mirror != (conj_all != 0)) v = cconj(v);
        const T sc = p1[n1 + N1 / 2] * p2[n2 + N2 / 2] * p3[n3 + N3 / 2];
        fk[i] = cmul_real(v, sc);
    }
}

// type 2, real outputs.  One thread per half-spectrum cell q (k = (q1, signed q2,
// signed q3)); F(k) = fk[k] p(k) on the retained box, 0 elsewhere.  C2R applies
// exponent +: for the type-2 sign s = +1 H[q] = (F(k) + conj F(-k)) / 2, for s = -1
// (F(-k) + conj F(k)) / 2 -- in both cases C2R(H) = Re(sum F(k) e^{s i k x}).
template <typename T>
__global__ void __launch_bounds__(kEwThreads)
    pad_precorrect_c2r_kernel(const typename Cx<T>::type* __restrict__ fk, int64_t N1,
                              int64_t N2, int64_t N3, const T* __restrict__ p1,
                              const T* __restrict__ p2, const T* __restrict__ p3, int modeord,
                              int sign_plus, int64_t nf1, int64_t nf2, int64_t nf3,
                              typename Cx<T>::type* __restrict__ H) {
    using C = typename Cx<T>::type;
    const int64_t hx = nf1 / 2 + 1;
    const int64_t total = hx * nf2 * nf3;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < total;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q1 = m % hx, q2 = (m / hx) % nf2, q3 = m / (hx * nf2);
        const int64_t k1 = q1, k2 = q2 < nf2 / 2 ? q2 : q2 - nf2, k3 = q3 < nf3 / 2 ? q3 : q3 - nf3;
        C a{0, 0}, b{0, 0};  // F(k), F(-k)
        if (k1 < N1 / 2 && k2 >= -N2 / 2 && k2 < N2 / 2 && k3 >= -N3 / 2 && k3 < N3 / 2) {
            const T sc = p1[k1 + N1 / 2] * p2[k2 + N2 / 2] * p3[k3 + N3 / 2];
            a = cmul_real(fk[index_of(k1, N1, modeord) +
                             N1 * (index_of(k2, N2, modeord) + N2 * index_of(k3, N3, modeord))],
                          sc);
        }
        if (k1 <= N1 / 2 && k2 > -N2 / 2 && k2 <= N2 / 2 && k3 > -N3 / 2 && k3 <= N3 / 2) {
            const T sc = p1[-k1 + N1 / 2] * p2[-k2 + N2 / 2] * p3[-k3 + N3 / 2];
            b = cmul_real(fk[index_of(-k1, N1, modeord) +
                             N1 * (index_of(-k2, N2, modeord) + N2 * index_of(-k3, N3, modeord))],
                          sc);
        }
        const C u = sign_plus ? a : b, v = sign_plus ? b : a;  // H = (u + conj v) / 2
        H[m] = C{(T)0.5 * (u.x + v.x), (T)0.5 * (u.y - v.y)};
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
    pad_precorrect_kernel<T><<<ew_grid(nf[1] * nf[2] * row_lanes(nf[0])), kEwThreads, 0, s>>>(
        fk, N[0], N[1], N[2], p1, p2, p3, modeord, nf[0], nf[1], nf[2], grid);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_truncate_deconv_r2c(const typename Cx<T>::type* H, const int64_t nf[3],
                                       const int64_t N[3], const T* p1, const T* p2, const T* p3,
                                       int modeord, int conj_all, typename Cx<T>::type* fk,
                                       cudaStream_t s) {
    truncate_deconv_r2c_kernel<T><<<ew_grid(N[0] * N[1] * N[2]), kEwThreads, 0, s>>>(
        H, nf[0], nf[1], nf[2], N[0], N[1], N[2], p1, p2, p3, modeord, conj_all, fk);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pad_precorrect_c2r(const typename Cx<T>::type* fk, const int64_t N[3],
                                      const T* p1, const T* p2, const T* p3, int modeord,
                                      int sign_plus, const int64_t nf[3],
                                      typename Cx<T>::type* H, cudaStream_t s) {
    pad_precorrect_c2r_kernel<T><<<ew_grid((nf[0] / 2 + 1) * nf[1] * nf[2]), kEwThreads, 0, s>>>(
        fk, N[0], N[1], N[2], p1, p2, p3, modeord, sign_plus, nf[0], nf[1], nf[2], H);
    return cudaGetLastError();
}

template cudaError_t launch_truncate_deconv_r2c<float>(const float2*, const int64_t*,
                                                       const int64_t*, const float*, const float*,
                                                       const float*, int, int, float2*,
                                                       cudaStream_t);
template cudaError_t launch_truncate_deconv_r2c<double>(const double2*, const int64_t*,
                                                        const int64_t*, const double*,
                                                        const double*, const double*, int, int,
                                                        double2*, cudaStream_t);
template cudaError_t launch_pad_precorrect_c2r<float>(const float2*, const int64_t*, const float*,
                                                      const float*, const float*, int, int,
                                                      const int64_t*, float2*, cudaStream_t);
template cudaError_t launch_pad_precorrect_c2r<double>(const double2*, const int64_t*,
                                                       const double*, const double*, const double*,
                                                       int, int, const int64_t*, double2*,
                                                       cudaStream_t);
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
