// interp.cu -- the interpolation operator C^T of Eq. (4).
//
// "Sorted interpolation" taken to its B200 form: one CTA per
// bin stages the bin's (T + w)^3 subgrid from the periodic fine grid into
// shared memory once (coalesced wrapped loads along x rows), then every point
// of the bin gathers its w^3 stencil from shared memory.
//
// Per point (one warp): lanes 0..3w-1 evaluate the 3w ES weights (separability,
// PAPER.md:193-196) into a per-warp buffer; the 32 lanes then cover the w x w
// (x, y) columns, each summing its w z-cells against the z weights, scale by
// wx * wy, and a shuffle reduction produces c_j, written to the caller's order
// (c[perm[slot]], "reported in input particle order").
#include "internal.cuh"

namespace nufft {

namespace {

constexpr int kInterpThreads = 256;

template <typename T> __device__ __forceinline__ T es_weight(T zz, T beta);
template <> __device__ __forceinline__ double es_weight<double>(double zz, double beta) {
    const double t = 1.0 - zz * zz;
    return t >= 0.0 ? exp(beta * (sqrt(t) - 1.0)) : 0.0;
}
template <> __device__ __forceinline__ float es_weight<float>(float zz, float beta) {
    const float t = 1.0f - zz * zz;
    return t >= 0.0f ? expf(beta * (sqrtf(t) - 1.0f)) : 0.0f;
}

__device__ __forceinline__ int64_t wrap_idx(int64_t i, int64_t n) {
    while (i < 0) i += n;
    while (i >= n) i -= n;
    return i;
}

template <typename T, int W>
__global__ void __launch_bounds__(kInterpThreads, 2)
    interp_tile_kernel(Geom g, PtsView<T> p, const typename Cx<T>::type* __restrict__ grid,
                       typename Cx<T>::type* __restrict__ out, T beta) {
    using C = typename Cx<T>::type;
    constexpr int NQ = (W * W + 31) / 32;
    extern __shared__ __align__(16) unsigned char smem[];

    const int b = blockIdx.x;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int Ex = g.T[0] + W, Ey = g.T[1] + W, Ez = g.T[2] + W;
    const int ncell = Ex * Ey * Ez;
    C* tile = reinterpret_cast<C*>(smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    T* wb = reinterpret_cast<T*>(tile + ncell) + warp * 3 * W;  // per-warp weights

    // ---- stage the subgrid (wrapped, coalesced along x rows)
    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const int64_t ox = (int64_t)bx * g.T[0] - W / 2;
    const int64_t oy = (int64_t)by * g.T[1] - W / 2;
    const int64_t oz = (int64_t)bz * g.T[2] - W / 2;
    for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
        const int cx = i % Ex, cy = (i / Ex) % Ey, cz = i / (Ex * Ey);
        const int64_t gx = wrap_idx(ox + cx, g.nf[0]);
        const int64_t gy = wrap_idx(oy + cy, g.nf[1]);
        const int64_t gz = wrap_idx(oz + cz, g.nz_loc);
        tile[i] = grid[gx + g.nf[0] * (gy + g.nf[1] * gz)];
    }
    __syncthreads();

    int qx[NQ], qy[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int e = lane + 32 * q;
        qx[q] = e % W;
        qy[q] = e < W * W ? e / W : -1;
    }
    const T two_over_w = (T)2 / (T)W;
    const int plane = Ex * Ey;

    for (uint32_t slot = beg + warp; slot < end; slot += nwarps) {
        if (lane < 3 * W) {
            const int d = lane / W, k = lane - d * W;
            const T dd = d == 0 ? p.dx[slot] : (d == 1 ? p.dy[slot] : p.dz[slot]);
            wb[lane] = es_weight<T>(((T)k - dd) * two_over_w, beta);
        }
        const uint32_t la = p.la[slot];
        __syncwarp();
        const int lx = la & 0xff, ly = (la >> 8) & 0xff, lz = la >> 16;
        T ar = 0, ai = 0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (qy[q] >= 0) {
                const C* col = tile + lz * plane + (ly + qy[q]) * Ex + lx + qx[q];
                T sr = 0, si = 0;
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const C v = col[k * plane];
                    const T wz = wb[2 * W + k];
                    sr += v.x * wz;
                    si += v.y * wz;
                }
                const T wxy = wb[qx[q]] * wb[W + qy[q]];
                ar += sr * wxy;
                ai += si * wxy;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ar += __shfl_xor_sync(0xffffffffu, ar, o);
            ai += __shfl_xor_sync(0xffffffffu, ai, o);
        }
        if (lane == 0) out[p.perm[slot]] = C{ar, ai};
        __syncwarp();
    }
}

template <typename T, int W>
cudaError_t launch_w(const Geom& g, const PtsView<T>& p, int64_t nbins,
                     const typename Cx<T>::type* grid, typename Cx<T>::type* c, double beta,
                     cudaStream_t s) {
    using C = typename Cx<T>::type;
    const size_t ncell = (size_t)(g.T[0] + W) * (g.T[1] + W) * (g.T[2] + W);
    const size_t smem = ncell * sizeof(C) + (size_t)(kInterpThreads / 32) * 3 * W * sizeof(T);
    auto kern = interp_tile_kernel<T, W>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (nbins > 0) kern<<<(unsigned)nbins, kInterpThreads, smem, s>>>(g, p, grid, c, (T)beta);
    return cudaGetLastError();
}

}  // namespace

template <typename T>
cudaError_t launch_interp(const Geom& g, const PtsView<T>& p, int64_t nbins,
                          const typename Cx<T>::type* grid, typename Cx<T>::type* c, double beta,
                          cudaStream_t s) {
    switch (g.w) {
#define NUFFT_W_CASE(WW) \
    case WW:             \
        return launch_w<T, WW>(g, p, nbins, grid, c, beta, s);
        NUFFT_W_CASE(2) NUFFT_W_CASE(3) NUFFT_W_CASE(4) NUFFT_W_CASE(5) NUFFT_W_CASE(6)
        NUFFT_W_CASE(7) NUFFT_W_CASE(8) NUFFT_W_CASE(9) NUFFT_W_CASE(10) NUFFT_W_CASE(11)
        NUFFT_W_CASE(12) NUFFT_W_CASE(13) NUFFT_W_CASE(14) NUFFT_W_CASE(15) NUFFT_W_CASE(16)
#undef NUFFT_W_CASE
        default:
            return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_interp<float>(const Geom&, const PtsView<float>&, int64_t,
                                          const float2*, float2*, double, cudaStream_t);
template cudaError_t launch_interp<double>(const Geom&, const PtsView<double>&, int64_t,
                                           const double2*, double2*, double, cudaStream_t);

}  // namespace nufft
