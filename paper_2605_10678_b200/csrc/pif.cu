// pif.cu -- elementwise kernels of the Particle-in-Fourier step (PAPER.md:486-492,
// §4): the Poisson solve in Fourier space and the leapfrog push.
// Not hot; coalesced single passes.
//
//   poisson  E_k = -i k rho_k / |k|^2, k = 2 pi n / L, E_0 = 0, E = 0 on the Nyquist
//            planes (reading R15) (Gauss's law
//            i k . E_k = rho_k; the neutralising ion background cancels k = 0)
//   kick     v_d += s Re(E_d(x_j)),   s = (q/m) dt / L^3  (E(x) = L^-3 sum_k E_k e^{ikx})
//   drift    x += v dt, folded onto [0, L)
#include "internal.cuh"

namespace nufft {

namespace {

constexpr int kThreads = 256;

inline unsigned grid1d(int64_t n) {
    int64_t b = (n + kThreads - 1) / kThreads;
    const int64_t cap = 148 * 32;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

__device__ __forceinline__ int64_t mode_of(int64_t i, int64_t N, int modeord) {
    return modeord == 0 ? i - N / 2 : (i < N / 2 ? i : i - N);
}

template <typename T>
__global__ void poisson_kernel(const typename Cx<T>::type* __restrict__ rho, int64_t N1, int64_t N2,
                               int64_t N3, int64_t lo1, int64_t lo2, int64_t lo3, int64_t n1l,
                               int64_t n2l, int64_t n3l, double kscale, int modeord, int xhalf,
                               typename Cx<T>::type* __restrict__ ex,
                               typename Cx<T>::type* __restrict__ ey,
                               typename Cx<T>::type* __restrict__ ez) {
    using C = typename Cx<T>::type;
    const int64_t total = n1l * n2l * n3l;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = t % n1l, b = (t / n1l) % n2l, cc = t / (n1l * n2l);
        // xhalf: half-spectrum layout of a slab plan's real transforms (x index = k1 >= 0)
        const int64_t m1 = xhalf ? lo1 + a : mode_of(lo1 + a, N1, modeord);
        const int64_t m2 = mode_of(lo2 + b, N2, modeord), m3 = mode_of(lo3 + cc, N3, modeord);
        const double k1 = kscale * (double)m1, k2 = kscale * (double)m2, k3 = kscale * (double)m3;
        // Nyquist planes (k_d = -N_d/2, or k1 = +N1/2 in the half layout) carry no field:
        // a real field's odd derivative vanishes there (reading R15)
        const bool nyq = (xhalf ? m1 == N1 / 2 : m1 == -N1 / 2) || m2 == -N2 / 2 || m3 == -N3 / 2;
        const double kk = nyq ? 0.0 : k1 * k1 + k2 * k2 + k3 * k3;
        const C r = rho[t];
        // -i k rho / |k|^2 = (k / |k|^2) (Im rho, -Re rho)
        const double inv = kk > 0.0 ? 1.0 / kk : 0.0;
        const T re = (T)((double)r.y * inv), im = (T)(-(double)r.x * inv);
        ex[t] = C{(T)k1 * re, (T)k1 * im};
        ey[t] = C{(T)k2 * re, (T)k2 * im};
        ez[t] = C{(T)k3 * re, (T)k3 * im};
    }
}

// v += s Re(e): e complex (stride 2, real parts) or real (stride 1, a type2_real output)
template <typename T>
__global__ void kick_kernel(int64_t Np, T* __restrict__ v, const T* __restrict__ e, int stride,
                            T s) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < Np;
         j += (int64_t)gridDim.x * blockDim.x)
        v[j] += s * e[j * stride];
}

template <typename T>
__global__ void drift_kernel(int64_t Np, T* __restrict__ x, T* __restrict__ y, T* __restrict__ z,
                             const T* __restrict__ vx, const T* __restrict__ vy,
                             const T* __restrict__ vz, T dt, T L) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < Np;
         j += (int64_t)gridDim.x * blockDim.x) {
        T p[3] = {x[j] + vx[j] * dt, y[j] + vy[j] * dt, z[j] + vz[j] * dt};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            T q = p[d] - L * floor(p[d] / L);
            if (q >= L) q -= L;
            if (q < (T)0) q = (T)0;
            p[d] = q;
        }
        x[j] = p[0];
        y[j] = p[1];
        z[j] = p[2];
    }
}

}  // namespace

template <typename T>
cudaError_t launch_pif_poisson(const typename Cx<T>::type* rho, const int64_t N[3],
                               const int64_t lo[3], const int64_t hi[3], double L, int modeord, int xhalf,
                               typename Cx<T>::type* ex, typename Cx<T>::type* ey,
                               typename Cx<T>::type* ez, cudaStream_t s) {
    const int64_t n1 = hi[0] - lo[0], n2 = hi[1] - lo[1], n3 = hi[2] - lo[2];
    poisson_kernel<T><<<grid1d(n1 * n2 * n3), kThreads, 0, s>>>(
        rho, N[0], N[1], N[2], lo[0], lo[1], lo[2], n1, n2, n3, 2.0 * M_PI / L, modeord, xhalf, ex, ey, ez);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pif_kick(int64_t Np, T* v, const typename Cx<T>::type* e, double s,
                            cudaStream_t st) {
    if (Np > 0)
        kick_kernel<T><<<grid1d(Np), kThreads, 0, st>>>(Np, v, reinterpret_cast<const T*>(e), 2,
                                                        (T)s);
    return cudaGetLastError();
}
template <typename T>
cudaError_t launch_pif_kick_real(int64_t Np, T* v, const T* e, double s, cudaStream_t st) {
    if (Np > 0) kick_kernel<T><<<grid1d(Np), kThreads, 0, st>>>(Np, v, e, 1, (T)s);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_pif_drift(int64_t Np, T* x, T* y, T* z, const T* vx, const T* vy, const T* vz,
                             double dt, double L, cudaStream_t s) {
    if (Np > 0)
        drift_kernel<T><<<grid1d(Np), kThreads, 0, s>>>(Np, x, y, z, vx, vy, vz, (T)dt, (T)L);
    return cudaGetLastError();
}

#define NUFFT_PIF_INST(T)                                                                        \
    template cudaError_t launch_pif_poisson<T>(const Cx<T>::type*, const int64_t*, const int64_t*, \
                                               const int64_t*, double, int, int, Cx<T>::type*,     \
                                               Cx<T>::type*, Cx<T>::type*, cudaStream_t);          \
    template cudaError_t launch_pif_kick<T>(int64_t, T*, const Cx<T>::type*, double, cudaStream_t); \
    template cudaError_t launch_pif_kick_real<T>(int64_t, T*, const T*, double, cudaStream_t);      \
    template cudaError_t launch_pif_drift<T>(int64_t, T*, T*, T*, const T*, const T*, const T*,    \
                                             double, double, cudaStream_t);
NUFFT_PIF_INST(float)
NUFFT_PIF_INST(double)
#undef NUFFT_PIF_INST

}  // namespace nufft
