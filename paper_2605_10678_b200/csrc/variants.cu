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
// in bin-sorted order (order == nullptr: "sorted" Atomic / Direct),
// or -- Direct Interpolation only -- along the Morton (Z-order) curve of the bins
// (launch_morton_order).
// They read the setpts records (bin-local stencil base + phase), so the bin of a
// sorted slot is found by a binary search of the bin offsets.
#include "device_util.cuh"
#include "internal.cuh"

#include <algorithm>

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

// ---- Tiled Spread: the bin's points accumulated into a
// shared-memory histogram of the (T + w)^3 subgrid with shared ATOMIC additions,
// one point per thread; the subgrid is split along z into Z slices ("multiple
// teams process the same tile but operate on disjoint z-slices of the output"), one
// CTA (team) per (bin, slice), so the histogram is (T + w)^2 x ceil((T + w) / Z)
// cells; after the bin each slice row is added to the fine grid with one bulk
// reduction (UBLKRED).  On sm_100a the fp32 / fp64 shared adds are CAS loops.
constexpr int kTiledZ = 4;  // z-oversubscription: teams per bin

template <typename T, int W>
__global__ void __launch_bounds__(kVarThreads)
    spread_tiled_kernel(Geom g, PtsView<T> p, const typename Cx<T>::type* __restrict__ c,
                        typename Cx<T>::type* __restrict__ grid, T beta) {
    using C = typename Cx<T>::type;
    extern __shared__ __align__(16) unsigned char smem[];
    const int b = blockIdx.x / kTiledZ, zk = blockIdx.x % kTiledZ;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;
    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const TileX tx = tile_x<sizeof(C)>(bx, g.T[0], W);
    const int P = tx.pitch, Ey = g.T[1] + W, Ez = g.T[2] + W;
    const int S = (Ez + kTiledZ - 1) / kTiledZ, z0 = zk * S, z1 = min(Ez, z0 + S);
    if (z0 >= z1) return;
    C* hist = reinterpret_cast<C*>(smem);  // [S][Ey][P]
    {
        float4* z4 = reinterpret_cast<float4*>(hist);
        const int n4 = (int)(((size_t)S * Ey * P * sizeof(C)) / 16);
        for (int i = threadIdx.x; i < n4; i += kVarThreads) z4[i] = float4{0.f, 0.f, 0.f, 0.f};
    }
    __syncthreads();
    const T two_over_w = (T)2 / (T)W;
    for (uint32_t s = beg + threadIdx.x; s < end; s += kVarThreads) {
        const PtRec<T> r = p.rec[s];
        const int lx = (int)(r.la & 0xff), ly = (int)((r.la >> 8) & 0xff), lz = (int)(r.la >> 16);
        if (lz + W <= z0 || lz >= z1) continue;  // no stencil plane in this team's slice
        T wt[3][W];
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int k = 0; k < W; ++k)
                wt[d][k] = p.w ? p.w[(size_t)s * (3 * W) + W * d + k]
                               : es_weight<T>(((T)k - r.d[d]) * two_over_w, beta);
        const C cv = c[r.perm];
#pragma unroll 1
        for (int k = 0; k < W; ++k) {
            const int z = lz + k;
            if (z < z0 || z >= z1) continue;
            const C cz = vscale(cv, wt[2][k]);
            for (int j = 0; j < W; ++j) {
                C* row = hist + ((size_t)(z - z0) * Ey + ly + j) * P + tx.shift + lx;
                const C cy = vscale(cz, wt[1][j]);
#pragma unroll
                for (int i = 0; i < W; ++i) atomic_add_v(row + i, vscale(cy, wt[0][i]));
            }
        }
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int oy = by * g.T[1] - W / 2, oz = bz * g.T[2] - W / 2;
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    int sg[2], ss[2], sn[2];
    const int nseg = row_segments(tx.gx0, tx.len, nfx, sg, ss, sn);
    for (int rr = threadIdx.x; rr < (z1 - z0) * Ey; rr += kVarThreads) {
        const int cz = rr / Ey, cy = rr - cz * Ey;
        const int gy = wrap1(oy + cy, nfy), gz = z_row(oz + z0 + cz, g);
        C* grow = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
        const C* trow = hist + (size_t)rr * P;
        for (int k = 0; k < (gz < -g.hz_lo ? 0 : nseg); ++k)
            bulk_red_add(reinterpret_cast<T*>(grow + sg[k]), trow + ss[k],
                         (unsigned)(sn[k] * sizeof(C)));
    }
    bulk_commit();
    bulk_wait_read();
}

// ---- Morton-ordered walk ("Morton code ordering"): the bins are
// visited along the Z-order curve of their coordinates (bits interleaved x fastest,
// coordinates coarsened by `shift` so the key space stays <= 2^24), the points of a
// bin in its sorted order.  Built from the bin-sorted records without another sort:
// per-key point counts (an atomic cursor places the bins sharing a coarsened key),
// an exclusive scan of the keys, then each sorted slot's rank along the curve.
__device__ __forceinline__ uint32_t spread_bits(uint32_t v) {  // 10 bits -> every 3rd bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__device__ __forceinline__ uint32_t morton_key(const Geom& g, int b, int shift) {
    const uint32_t bx = (uint32_t)(b % g.nb[0]) >> shift,
                   by = (uint32_t)((b / g.nb[0]) % g.nb[1]) >> shift,
                   bz = (uint32_t)(b / (g.nb[0] * g.nb[1])) >> shift;
    return spread_bits(bx) | (spread_bits(by) << 1) | (spread_bits(bz) << 2);
}
__global__ void morton_bin_count_kernel(Geom g, int nbins, int shift,
                                        const uint32_t* __restrict__ offset,
                                        uint32_t* __restrict__ key_count,
                                        uint32_t* __restrict__ bin_base) {
    const int b = blockIdx.x * kVarThreads + threadIdx.x;
    if (b >= nbins) return;
    const uint32_t n = offset[b + 1] - offset[b];
    bin_base[b] = n ? atomicAdd(&key_count[morton_key(g, b, shift)], n) : 0u;
}
__global__ void morton_slot_kernel(Geom g, int nbins, int shift, int64_t Np,
                                   const uint32_t* __restrict__ offset,
                                   const uint32_t* __restrict__ key_off,
                                   const uint32_t* __restrict__ bin_base,
                                   uint32_t* __restrict__ order) {
    const int64_t s = (int64_t)blockIdx.x * kVarThreads + threadIdx.x;
    if (s >= Np) return;
    int lo = 0, hi = nbins;  // bin of sorted slot s
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (offset[mid] <= (uint32_t)s) lo = mid;
        else hi = mid;
    }
    order[key_off[morton_key(g, lo, shift)] + bin_base[lo] + ((uint32_t)s - offset[lo])] =
        (uint32_t)s;
}

}  // namespace

size_t spread_tiled_smem_bytes(const Geom& g, int cell_bytes) {
    const int P = cell_bytes == 16 ? tile_pitch<16>(g.T[0], g.w) : tile_pitch<8>(g.T[0], g.w);
    const int Ez = g.T[2] + g.w, S = (Ez + kTiledZ - 1) / kTiledZ;
    return (size_t)S * (g.T[1] + g.w) * P * cell_bytes;
}

template <typename T>
cudaError_t launch_spread_tiled(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                const typename Cx<T>::type* c, typename Cx<T>::type* grid,
                                double beta, cudaStream_t s) {
    const size_t smem = spread_tiled_smem_bytes(g, (int)sizeof(typename Cx<T>::type));
    const unsigned nb = (unsigned)(nbins * kTiledZ);
#define CASE(WW)                                                                             \
    case WW: {                                                                               \
        auto kern = spread_tiled_kernel<T, WW>;                                              \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)smem);                                     \
        if (e != cudaSuccess) return e;                                                      \
        if (nb) kern<<<nb, kVarThreads, smem, s>>>(g, p, c, grid, (T)beta);                  \
        break;                                                                               \
    }
    switch (g.w) {
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11)
        CASE(12) CASE(13) CASE(14) CASE(15) CASE(16)
        default: return cudaErrorInvalidValue;
    }
#undef CASE
    return cudaGetLastError();
}
template cudaError_t launch_spread_tiled<float>(const Geom&, const PtsView<float>&, int64_t,
                                                const float2*, float2*, double, cudaStream_t);
template cudaError_t launch_spread_tiled<double>(const Geom&, const PtsView<double>&, int64_t,
                                                 const double2*, double2*, double, cudaStream_t);

int morton_shift(const Geom& g) {
    int m = std::max(g.nb[0], std::max(g.nb[1], g.nb[2])), bits = 0;
    while ((1 << bits) < m) ++bits;
    return bits > 8 ? bits - 8 : 0;  // 3 x 8 bits: a 2^24-entry key space
}
size_t morton_keys(const Geom& g) { return (size_t)1 << (3 * (std::min(8, [&] {
    int m = std::max(g.nb[0], std::max(g.nb[1], g.nb[2])), bits = 0;
    while ((1 << bits) < m) ++bits;
    return bits;
}()))); }

cudaError_t launch_morton_order(const Geom& g, const uint32_t* offset, int64_t nbins, int64_t Np,
                                uint32_t* key_count, uint32_t* key_off, uint32_t* blocksum,
                                uint32_t* bin_base, uint32_t* order, cudaStream_t s) {
    const int shift = morton_shift(g);
    const size_t nk = morton_keys(g);
    cudaError_t e = cudaMemsetAsync(key_count, 0, sizeof(uint32_t) * nk, s);
    if (e != cudaSuccess) return e;
    if (nbins > 0)
        morton_bin_count_kernel<<<(unsigned)((nbins + kVarThreads - 1) / kVarThreads), kVarThreads,
                                  0, s>>>(g, (int)nbins, shift, offset, key_count, bin_base);
    if ((e = launch_exclusive_scan(key_count, (int64_t)nk, blocksum, key_off, s)) != cudaSuccess)
        return e;
    if (Np > 0)
        morton_slot_kernel<<<(unsigned)((Np + kVarThreads - 1) / kVarThreads), kVarThreads, 0, s>>>(
            g, (int)nbins, shift, Np, offset, key_off, bin_base, order);
    return cudaGetLastError();
}

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
