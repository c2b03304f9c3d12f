// spread.cu -- Step 1 of Eq. (3), the spreading operator C.
//
// One CTA per bin (tile of T^3 fine cells).  The CTA owns a shared-memory
// subgrid of (T + w)^3 complex cells ("a shared memory histogram of size
// prod(T_i + w)") and processes the bin's points in batches:
//
//   phase A  every thread evaluates the w ES weights of one (point, axis) pair
//            in registers -- d w evaluations per point thanks to separability
//            (PAPER.md:193-196), phi evaluated directly -- and
//            stages them with the point's strength in shared memory;
//   phase B  accumulation WITHOUT shared-memory atomics: warp k owns the
//            subgrid z-planes {k, k + nwarps, ...}; for each point whose
//            z-stencil covers an owned plane, the 32 lanes cover the w x w
//            (x, y) cells of that plane.  No two threads ever write the same
//            cell concurrently (cf. the paper's Grid-Parallel ownership,
//            PAPER.md:209, and its z-split of the stencil).
//            On sm_100a shared-memory float atomics are CAS loops, so owning
//            planes is the B200-native choice.
//   flush    the subgrid is added into the periodic fine grid in HBM with one
//            vector/scalar global reduction per cell (fp32: red.global.add.v2.f32,
//            fp64: red.global.add.f64 x 2); periodic ghost cells wrap directly
//            (PAPER.md:213), so no separate ghost-fold pass exists on one GPU.
#include "internal.cuh"

namespace nufft {

namespace {

constexpr int kSpreadThreads = 256;
constexpr int kBatch = 64;  // points staged per phase-A/phase-B round

template <typename T> __device__ __forceinline__ T es_weight(T zz, T beta);
template <> __device__ __forceinline__ double es_weight<double>(double zz, double beta) {
    // PAPER.md:168-173; |z| <= 1 inside (reading R5)
    const double t = 1.0 - zz * zz;
    return t >= 0.0 ? exp(beta * (sqrt(t) - 1.0)) : 0.0;
}
template <> __device__ __forceinline__ float es_weight<float>(float zz, float beta) {
    const float t = 1.0f - zz * zz;
    return t >= 0.0f ? expf(beta * (sqrtf(t) - 1.0f)) : 0.0f;
}

__device__ __forceinline__ void red_add(double2* p, double2 v) {
    atomicAdd(&p->x, v.x);
    atomicAdd(&p->y, v.y);
}
__device__ __forceinline__ void red_add(float2* p, float2 v) {
    atomicAdd(p, v);  // sm_90+: red.global.add.v2.f32
}

__device__ __forceinline__ int64_t wrap_idx(int64_t i, int64_t n) {
    while (i < 0) i += n;
    while (i >= n) i -= n;
    return i;
}

template <typename T, int W>
__global__ void __launch_bounds__(kSpreadThreads, 2)
    spread_tile_kernel(Geom g, PtsView<T> p, const typename Cx<T>::type* __restrict__ c,
                       typename Cx<T>::type* __restrict__ grid, T beta) {
    using C = typename Cx<T>::type;
    constexpr int NQ = (W * W + 31) / 32;  // lane passes over a w x w plane
    extern __shared__ __align__(16) unsigned char smem[];

    const int b = blockIdx.x;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int Ex = g.T[0] + W, Ey = g.T[1] + W, Ez = g.T[2] + W;
    const int ncell = Ex * Ey * Ez;
    C* tile = reinterpret_cast<C*>(smem);
    T* wts = reinterpret_cast<T*>(tile + ncell);         // [kBatch][3][W]
    C* cval = reinterpret_cast<C*>(wts + kBatch * 3 * W);  // [kBatch]
    uint32_t* lav = reinterpret_cast<uint32_t*>(cval + kBatch);

    for (int i = threadIdx.x; i < ncell; i += blockDim.x) tile[i] = C{0, 0};

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    int qx[NQ], qy[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int e = lane + 32 * q;
        qx[q] = e % W;
        qy[q] = e < W * W ? e / W : -1;
    }
    const T two_over_w = (T)2 / (T)W;

    for (uint32_t p0 = beg; p0 < end; p0 += kBatch) {
        const int n = (int)min((uint32_t)kBatch, end - p0);
        __syncthreads();  // previous batch fully consumed (and tile zeroed)
        // ---- phase A: weights of (point, axis) pairs, strengths, bases
        for (int t = threadIdx.x; t < 3 * n; t += blockDim.x) {
            const int i = t / 3, d = t - 3 * i;
            const uint32_t slot = p0 + i;
            const T dd = d == 0 ? p.dx[slot] : (d == 1 ? p.dy[slot] : p.dz[slot]);
            T* wd = wts + (i * 3 + d) * W;
#pragma unroll
            for (int k = 0; k < W; ++k) wd[k] = es_weight<T>(((T)k - dd) * two_over_w, beta);
            if (d == 0) {
                cval[i] = c[p.perm[slot]];
                lav[i] = p.la[slot];
            }
        }
        __syncthreads();
        // ---- phase B: warp-owned z-planes, lanes over the w x w (x, y) cells
        for (int i = 0; i < n; ++i) {
            const uint32_t la = lav[i];
            const int lx = la & 0xff, ly = (la >> 8) & 0xff, lz = la >> 16;
            // planes of this warp inside [lz, lz + W)
            int pz = lz + ((warp - lz) % nwarps + nwarps) % nwarps;
            if (pz >= lz + W) continue;
            const T* wx = wts + (i * 3 + 0) * W;
            const T* wy = wts + (i * 3 + 1) * W;
            const T* wz = wts + (i * 3 + 2) * W;
            const C cv = cval[i];
            T wxy[NQ];
            int off[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                wxy[q] = qy[q] >= 0 ? wx[qx[q]] * wy[qy[q]] : (T)0;
                off[q] = (ly + (qy[q] >= 0 ? qy[q] : 0)) * Ex + lx + qx[q];
            }
            for (; pz < lz + W; pz += nwarps) {
                const T wzz = wz[pz - lz];
                const T cr = cv.x * wzz, ci = cv.y * wzz;
                C* plane = tile + pz * Ey * Ex;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    if (qy[q] >= 0) {
                        C v = plane[off[q]];
                        v.x += cr * wxy[q];
                        v.y += ci * wxy[q];
                        plane[off[q]] = v;
                    }
                }
            }
        }
    }
    __syncthreads();
    // ---- flush: subgrid -> periodic fine grid (HBM), one reduction per nonzero cell
    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const int64_t ox = (int64_t)bx * g.T[0] - W / 2;
    const int64_t oy = (int64_t)by * g.T[1] - W / 2;
    const int64_t oz = (int64_t)bz * g.T[2] - W / 2;
    for (int i = threadIdx.x; i < ncell; i += blockDim.x) {
        const C v = tile[i];
        if (v.x == (T)0 && v.y == (T)0) continue;
        const int cx = i % Ex, cy = (i / Ex) % Ey, cz = i / (Ex * Ey);
        const int64_t gx = wrap_idx(ox + cx, g.nf[0]);
        const int64_t gy = wrap_idx(oy + cy, g.nf[1]);
        const int64_t gz = wrap_idx(oz + cz, g.nz_loc);
        red_add(grid + gx + g.nf[0] * (gy + g.nf[1] * gz), v);
    }
}

template <typename T, int W>
cudaError_t launch_w(const Geom& g, const PtsView<T>& p, int64_t nbins,
                     const typename Cx<T>::type* c, typename Cx<T>::type* grid, double beta,
                     cudaStream_t s) {
    using C = typename Cx<T>::type;
    const size_t ncell = (size_t)(g.T[0] + W) * (g.T[1] + W) * (g.T[2] + W);
    const size_t smem = ncell * sizeof(C) + (size_t)kBatch * 3 * W * sizeof(T) +
                        kBatch * sizeof(C) + kBatch * sizeof(uint32_t);
    auto kern = spread_tile_kernel<T, W>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (nbins > 0) kern<<<(unsigned)nbins, kSpreadThreads, smem, s>>>(g, p, c, grid, (T)beta);
    return cudaGetLastError();
}

}  // namespace

template <typename T>
cudaError_t launch_spread(const Geom& g, const PtsView<T>& p, int64_t nbins,
                          const typename Cx<T>::type* c, typename Cx<T>::type* grid, double beta,
                          cudaStream_t s) {
    switch (g.w) {
#define NUFFT_W_CASE(WW) \
    case WW:             \
        return launch_w<T, WW>(g, p, nbins, c, grid, beta, s);
        NUFFT_W_CASE(2) NUFFT_W_CASE(3) NUFFT_W_CASE(4) NUFFT_W_CASE(5) NUFFT_W_CASE(6)
        NUFFT_W_CASE(7) NUFFT_W_CASE(8) NUFFT_W_CASE(9) NUFFT_W_CASE(10) NUFFT_W_CASE(11)
        NUFFT_W_CASE(12) NUFFT_W_CASE(13) NUFFT_W_CASE(14) NUFFT_W_CASE(15) NUFFT_W_CASE(16)
#undef NUFFT_W_CASE
        default:
            return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_spread<float>(const Geom&, const PtsView<float>&, int64_t,
                                          const float2*, float2*, double, cudaStream_t);
template cudaError_t launch_spread<double>(const Geom&, const PtsView<double>&, int64_t,
                                           const double2*, double2*, double, cudaStream_t);

}  // namespace nufft
