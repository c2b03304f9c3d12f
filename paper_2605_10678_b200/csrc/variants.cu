// variants.cu -- the paper's baseline spread / interpolation algorithms, kept for
// the design-space ablation; never the default.
//
//   Atomic Spread: one thread per point evaluates its 3w ES
//     weights and adds c_j wx wy wz to the w^3 fine-grid cells
//     of its stencil with global atomics (periodic wrap).
//   Direct Interpolation: one thread per point reads the w^3
//     cells of its stencil straight from global memory and accumulates
//     sum wx wy wz G (the operator C^T of Eq. (3)).
//
// Both walk the points either in the caller's order (`order` = the slot of caller
// point t, so thread t handles caller point t: the paper's unsorted variants) or
// in bin-sorted order (order == nullptr: "sorted" Atomic / Direct).
// They read the setpts records (bin-local stencil base + phase), so the bin of a
// sorted slot is found by a binary search of the bin offsets.
#include "device_util.cuh"
#include "internal.cuh"

namespace nufft {

namespace {

using namespace dev;

constexpr int kVarThreads = 256;

template <typename T> struct VarPoint {
    int g0[3];  // global fine index of stencil node 0 per axis (before the periodic wrap)
    T wt[3][16];
    uint32_t perm;
};

template <typename T, int W>
__device__ __forceinline__ void load_point(const Geom& g, const PtsView<T>& p, int nbins,
                                           uint32_t s, T beta, VarPoint<T>& v) {
    // bin b of sorted slot s: offset[b] <= s < offset[b + 1]
    int lo = 0, hi = nbins;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (p.offset[mid] <= s) lo = mid;
        else hi = mid;
    }
    const int bx = lo % g.nb[0], by = (lo / g.nb[0]) % g.nb[1], bz = lo / (g.nb[0] * g.nb[1]);
    const PtRec<T> r = p.rec[s];
    v.perm = r.perm;
    v.g0[0] = bx * g.T[0] - W / 2 + (int)(r.la & 0xff);
    v.g0[1] = by * g.T[1] - W / 2 + (int)((r.la >> 8) & 0xff);
    v.g0[2] = bz * g.T[2] - W / 2 + (int)(r.la >> 16);
    const T two_over_w = (T)2 / (T)W;
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int k = 0; k < W; ++k)
            v.wt[d][k] = p.w ? p.w[(size_t)s * (3 * W) + W * d + k]
                             : es_weight<T>(((T)k - r.d[d]) * two_over_w, beta);
}

__device__ __forceinline__ void atomic_add_v(float2* a, float2 v) {
    atomicAdd(&a->x, v.x);
    atomicAdd(&a->y, v.y);
}
__device__ __forceinline__ void atomic_add_v(double2* a, double2 v) {
    atomicAdd(&a->x, v.x);
    atomicAdd(&a->y, v.y);
}

template <typename T, int W>
__global__ void __launch_bounds__(kVarThreads)
    spread_atomic_kernel(Geom g, PtsView<T> p, int nbins, const uint32_t* __restrict__ order,
                         int64_t Np, const typename Cx<T>::type* __restrict__ c,
                         typename Cx<T>::type* __restrict__ grid, T beta) {
    using C = typename Cx<T>::type;
    const int64_t t = (int64_t)blockIdx.x * kVarThreads + threadIdx.x;
    if (t >= Np) return;
    VarPoint<T> v;
    load_point<T, W>(g, p, nbins, order ? order[t] : (uint32_t)t, beta, v);
    const C cv = c[v.perm];
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    int gx[W];
#pragma unroll
    for (int i = 0; i < W; ++i) gx[i] = wrap1(v.g0[0] + i, nfx);
    for (int k = 0; k < W; ++k) {
        const int gz = z_row(v.g0[2] + k, g);
        if (gz < -g.hz_lo) continue;  // outside the halo-extended slab (never on one GPU)
        const C cz = vscale(cv, v.wt[2][k]);
        for (int j = 0; j < W; ++j) {
            const int gy = wrap1(v.g0[1] + j, nfy);
            C* row = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
            const C cy = vscale(cz, v.wt[1][j]);
#pragma unroll
            for (int i = 0; i < W; ++i) atomic_add_v(row + gx[i], vscale(cy, v.wt[0][i]));
        }
    }
}

template <typename T, int W>
__global__ void __launch_bounds__(kVarThreads)
    interp_direct_kernel(Geom g, PtsView<T> p, int nbins, const uint32_t* __restrict__ order,
                         int64_t Np, const typename Cx<T>::type* __restrict__ grid,
                         typename Cx<T>::type* __restrict__ c, T beta) {
    using C = typename Cx<T>::type;
    const int64_t t = (int64_t)blockIdx.x * kVarThreads + threadIdx.x;
    if (t >= Np) return;
    VarPoint<T> v;
    load_point<T, W>(g, p, nbins, order ? order[t] : (uint32_t)t, beta, v);
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    int gx[W];
#pragma unroll
    for (int i = 0; i < W; ++i) gx[i] = wrap1(v.g0[0] + i, nfx);
    C acc = vzero<C>();
    for (int k = 0; k < W; ++k) {
        const int gz = z_row(v.g0[2] + k, g);
        if (gz < -g.hz_lo) continue;
        C az = vzero<C>();
        for (int j = 0; j < W; ++j) {
            const int gy = wrap1(v.g0[1] + j, nfy);
            const C* row = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
            C ay = vzero<C>();
#pragma unroll
            for (int i = 0; i < W; ++i) vfma(ay, __ldg(row + gx[i]), v.wt[0][i]);
            vfma(az, ay, v.wt[1][j]);
        }
        vfma(acc, az, v.wt[2][k]);
    }
    c[v.perm] = acc;
}

// order[perm] = sorted slot (the caller-order walk of the unsorted variants)
template <typename T>
__global__ void caller_order_kernel(const PtRec<T>* __restrict__ rec, int64_t Np,
                                    uint32_t* __restrict__ order) {
    const int64_t s = (int64_t)blockIdx.x * kVarThreads + threadIdx.x;
    if (s < Np) order[rec[s].perm] = (uint32_t)s;
}

}  // namespace

template <typename T>
cudaError_t launch_spread_atomic(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                 const uint32_t* order, int64_t Np, const typename Cx<T>::type* c,
                                 typename Cx<T>::type* grid, double beta, cudaStream_t s) {
    if (Np <= 0) return cudaSuccess;
    const unsigned nb = (unsigned)((Np + kVarThreads - 1) / kVarThreads);
#define CASE(WW)                                                                        \
    case WW:                                                                           \
        spread_atomic_kernel<T, WW><<<nb, kVarThreads, 0, s>>>(g, p, (int)nbins, order, Np, c, \
                                                              grid, (T)beta);           \
        break;
    switch (g.w) {
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11)
        CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
        default: return cudaErrorInvalidValue;
    }
#undef CASE
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_interp_direct(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                 const uint32_t* order, int64_t Np,
                                 const typename Cx<T>::type* grid, typename Cx<T>::type* c,
                                 double beta, cudaStream_t s) {
    if (Np <= 0) return cudaSuccess;
    const unsigned nb = (unsigned)((Np + kVarThreads - 1) / kVarThreads);
#define CASE(WW)                                                                        \
    case WW:                                                                           \
        interp_direct_kernel<T, WW><<<nb, kVarThreads, 0, s>>>(g, p, (int)nbins, order, Np, grid, \
                                                              c, (T)beta);              \
        break;
    switch (g.w) {
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11)
        CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
        default: return cudaErrorInvalidValue;
    }
#undef CASE
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_caller_order(const PtRec<T>* rec, int64_t Np, uint32_t* order,
                                cudaStream_t s) {
    if (Np <= 0) return cudaSuccess;
    caller_order_kernel<T><<<(unsigned)((Np + kVarThreads - 1) / kVarThreads), kVarThreads, 0, s>>>(
        rec, Np, order);
    return cudaGetLastError();
}

template cudaError_t launch_spread_atomic<float>(const Geom&, const PtsView<float>&, int64_t,
                                                 const uint32_t*, int64_t, const float2*, float2*,
                                                 double, cudaStream_t);
template cudaError_t launch_spread_atomic<double>(const Geom&, const PtsView<double>&, int64_t,
                                                  const uint32_t*, int64_t, const double2*,
                                                  double2*, double, cudaStream_t);
template cudaError_t launch_interp_direct<float>(const Geom&, const PtsView<float>&, int64_t,
                                                 const uint32_t*, int64_t, const float2*, float2*,
                                                 double, cudaStream_t);
template cudaError_t launch_interp_direct<double>(const Geom&, const PtsView<double>&, int64_t,
                                                  const uint32_t*, int64_t, const double2*,
                                                  double2*, double, cudaStream_t);
template cudaError_t launch_caller_order<float>(const PtRec<float>*, int64_t, uint32_t*,
                                                cudaStream_t);
template cudaError_t launch_caller_order<double>(const PtRec<double>*, int64_t, uint32_t*,
                                                 cudaStream_t);

}  // namespace nufft
