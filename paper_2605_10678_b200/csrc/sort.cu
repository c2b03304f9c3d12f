// sort.cu -- setpts: fold + bin count, exclusive scan, scatter (counting sort).
//
// PAPER.md:204 ("sort particles into spatial tiles of tunable size") and
// PAPER.md:226-227 (bin sorting for interpolation locality).  north_star (1):
// "a bin-sort of points by subgrid cell, using a counting sort built from
// warp-level prefix scans".
//
//   k1 bin_count : per point, fold onto the torus and rescale in fp64
//                  (s = x * nf / L), bin = tile of floor(s); an atomicAdd on
//                  count[bin] returns each point's rank inside its bin.
//   k2 scan      : exclusive prefix sum of count[] -> offset[] with warp
//                  __shfl_up_sync scans, three phases (tile sums, scan of sums,
//                  tile scans + carry-in).
//   k3 scatter   : slot = offset[bin] + rank; the sorted 32-byte stencil record
//                  (phase offsets d, local base la, caller index) is written
//                  to the slot as one full DRAM sector.
#include "device_util.cuh"
#include "internal.cuh"

namespace nufft {

namespace {

constexpr int kSortThreads = 256;
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;                        // per thread
constexpr int kScanTile = kScanThreads * kScanItems;  // counts per scan tile

constexpr int kScatterILP = 4;  // points per thread per scatter round

// L2 residency of setpts: the per-point streams (coordinates, bin_of / rank_of)
// are read or written once, so they go with the streaming / evict-first hints,
// while the key arrays (count, offset_key: 4 B per key, 68 MB at C4) -- hit at
// random by every point -- are accessed under an evict-last policy, so the
// coordinate stream does not push them out of L2 between two hits.
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint32_t atomic_add_keep(uint32_t* a, uint32_t v, uint64_t pol) {
    uint32_t r;
    asm volatile("atom.global.add.L2::cache_hint.u32 %0, [%1], %2, %3;"
                 : "=r"(r)
                 : "l"(a), "r"(v), "l"(pol)
                 : "memory");
    return r;
}
__device__ __forceinline__ uint32_t ld_keep(const uint32_t* a, uint64_t pol) {
    uint32_t r;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
    return r;
}

// Fold onto [0, L) and rescale to fine-grid units (reading R10), fp64.  For x in
// [0, L) the quotient x / L rounds to at most 1 - 2^-53, so floor(x / L) = 0 and
// the fold is the identity: the fp64 division runs only for x outside [0, L).
__device__ __forceinline__ double fold_rescale(double x, double L, double scale, int64_t nf) {
    double xf = (x >= 0.0 && x < L) ? x : x - L * floor(x / L);
    double s = xf * scale;
    if (s >= (double)nf) s -= (double)nf;
    if (s < 0.0) s += (double)nf;
    return s;
}

__device__ __forceinline__ int cell_of(double s, int64_t nf) {
    int64_t c = (int64_t)s;  // s >= 0: truncation == floor
    return (int)(c >= nf ? nf - 1 : c);
}

// Bin-local stencil record of one coordinate (reading R4: a = ceil(s - w/2)).
//   r  = s - (bin origin)          exact in fp64
//   ls = r + floor(w/2)            coordinate relative to the tile origin
//   la = ceil(ls - w/2)            local stencil base, in [0, T]
//   d  = ls - la                   phase offset, z_k = 2 (k - d) / w
__device__ __forceinline__ void local_stencil(double s, int c, int T, int w, int* la, double* d) {
    const int origin = (c / T) * T;
    const double ls = (s - (double)origin) + (double)(w / 2);
    const double a = ceil(ls - 0.5 * (double)w);
    *la = (int)a;
    *d = ls - a;
}

// Sub-bin of a point from its bin-local stencil bases (Geom::nsub > 1): the same
// la the scatter stores, so the sub-bin kernel sees la - G * sub in [0, G).
__device__ __forceinline__ uint32_t sub_of(const Geom& g, double sx, int cx, double sy, int cy,
                                           double sz, int cz) {
    int lax, lay, laz;
    double dd;
    local_stencil(sx, cx, g.T[0], g.w, &lax, &dd);
    local_stencil(sy, cy, g.T[1], g.w, &lay, &dd);
    local_stencil(sz, cz, g.T[2], g.w, &laz, &dd);
    return (uint32_t)((laz / g.Gs[2] * g.ns[1] + lay / g.Gs[1]) * g.ns[0] + lax / g.Gs[0]);
}

// slab-local z coordinate exactly as the scatter uses it (clamped into the slab)
__device__ __forceinline__ double slab_z(const Geom& g, double szg) {
    double sz = szg - (double)g.z_lo;
    if (!(sz >= 0.0)) sz = 0.0;  // outside the slab: clamp (see bin_count_kernel)
    if (sz >= (double)g.nz_loc) sz = (double)g.nz_loc - 0.5;
    return sz;
}

// sort key of one point: bin, or (bin, sub-bin) for sub-bin plans (the scatter's la)
template <typename T>
__device__ __forceinline__ uint32_t sort_key(const Geom& g, T xv, T yv, T zv) {
    const double sx = fold_rescale((double)xv, g.L, g.scale[0], g.nf[0]);
    const double sy = fold_rescale((double)yv, g.L, g.scale[1], g.nf[1]);
    const double szg = fold_rescale((double)zv, g.L, g.scale[2], g.nf[2]);
    const int cx = cell_of(sx, g.nf[0]);
    const int cy = cell_of(sy, g.nf[1]);
    int cz = cell_of(szg, g.nf[2]) - (int)g.z_lo;
    // a slab plan given a point outside its slab (points_owned misuse): keep memory
    // safe by clamping to the slab (the caller's contract is broken)
    cz = cz < 0 ? 0 : (cz >= (int)g.nz_loc ? (int)g.nz_loc - 1 : cz);
    uint32_t bin = (uint32_t)(cx / g.T[0]) +
                   (uint32_t)g.nb[0] *
                       ((uint32_t)(cy / g.T[1]) + (uint32_t)g.nb[1] * (uint32_t)(cz / g.T[2]));
    if (g.nsub > 1) {
        const double sz = slab_z(g, szg);
        bin = bin * (uint32_t)g.nsub +
              sub_of(g, sx, cx, sy, cy, sz, cell_of(sz + (double)g.z_lo, g.nf[2]) - (int)g.z_lo);
    }
    return bin;
}

// kScatterILP points per thread per round, every load issued before any use and the
// atomics of the round in flight together (the atomic's return -- the rank -- is
// the latency that bounds this kernel)
template <typename T>
__global__ void __launch_bounds__(kSortThreads) bin_count_kernel(
    Geom g, int64_t Np, const T* __restrict__ x, const T* __restrict__ y,
    const T* __restrict__ z, uint32_t* __restrict__ count, uint32_t* __restrict__ bin_of,
    uint32_t* __restrict__ rank_of) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint64_t keep = l2_evict_last();
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < Np;
         i0 += kScatterILP * stride) {
        T xv[kScatterILP], yv[kScatterILP], zv[kScatterILP];
#pragma unroll
        for (int u = 0; u < kScatterILP; ++u) {
            const int64_t i = i0 + u * stride;
            const bool ok = i < Np;
            xv[u] = ok ? __ldcs(x + i) : (T)0;
            yv[u] = ok ? __ldcs(y + i) : (T)0;
            zv[u] = ok ? __ldcs(z + i) : (T)0;
        }
        uint32_t key[kScatterILP], rank[kScatterILP];
#pragma unroll
        for (int u = 0; u < kScatterILP; ++u) key[u] = sort_key<T>(g, xv[u], yv[u], zv[u]);
        // one atomicAdd per point: the rank of the point in its bin.  (A warp-
        // aggregated __match_any_sync version was measured slower on B200 for the
        // paper's near-uniform workloads: setpts C2b 0.170 -> 0.152 ms, C3 18.0 ->
        // 16.5 ms without it; collisions inside a warp are rare at ~1e4-1e5 bins.)
#pragma unroll
        for (int u = 0; u < kScatterILP; ++u)
            if (i0 + u * stride < Np) rank[u] = atomic_add_keep(&count[key[u]], 1u, keep);
#pragma unroll
        for (int u = 0; u < kScatterILP; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < Np) {
                __stcs(bin_of + i, key[u]);
                __stcs(rank_of + i, rank[u]);
            }
        }
    }
}

// Inclusive warp scan with __shfl_up_sync.
__device__ __forceinline__ uint32_t warp_inclusive_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_sums[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    uint32_t inc = warp_inclusive_scan(v);
    if (lane == 31) warp_sums[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = lane < nwarps ? warp_sums[lane] : 0u;
        uint32_t si = warp_inclusive_scan(s);
        if (lane < nwarps) warp_sums[lane] = si - s;  // exclusive warp offsets
        if (lane == nwarps - 1) *total = si;
    }
    __syncthreads();
    uint32_t r = inc - v + warp_sums[warp];
    __syncthreads();
    return r;
}

// phase 1: per scan tile, the sum of its counts
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums(const uint32_t* __restrict__ count,
                                                               int64_t n,
                                                               uint32_t* __restrict__ sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < n) v += count[base + k];
    // warp reduce, then block reduce via the scan helper's total
    __shared__ uint32_t total;
    (void)block_exclusive_scan(v, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// phase 2: one block scans the tile sums in place (exclusive), any length
__global__ void __launch_bounds__(kScanThreads) scan_sums(uint32_t* __restrict__ sums,
                                                          int64_t nsums) {
    __shared__ uint32_t total;
    uint32_t carry = 0;
    for (int64_t base = 0; base < nsums; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        uint32_t v = i < nsums ? sums[i] : 0u;
        uint32_t ex = block_exclusive_scan(v, &total);
        if (i < nsums) sums[i] = ex + carry;
        carry += total;
        __syncthreads();
    }
}

// phase 3: each tile re-scans its counts and adds its carry-in; offset[n] = total
__global__ void __launch_bounds__(kScanThreads) scan_tiles(const uint32_t* __restrict__ count,
                                                           int64_t n,
                                                           const uint32_t* __restrict__ sums,
                                                           uint32_t* __restrict__ offset) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t tsum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < n ? count[base + k] : 0u;
        tsum += v[k];
    }
    __shared__ uint32_t total;
    uint32_t ex = block_exclusive_scan(tsum, &total) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) offset[base + k] = ex;
        ex += v[k];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) offset[n] = ex;
}

// slot = offset[bin] + rank; the whole 32-byte record (one full DRAM sector, one
// 256-bit streaming store) goes to the slot: the only random access of setpts.
template <typename T>
__global__ void __launch_bounds__(kSortThreads) scatter_kernel(
    Geom g, int64_t Np, const T* __restrict__ x, const T* __restrict__ y,
    const T* __restrict__ z, const uint32_t* __restrict__ bin_of,
    const uint32_t* __restrict__ rank_of, const uint32_t* __restrict__ offset,
    PtRec<T>* __restrict__ rec) {
    // kScatterILP points per thread per round, every load issued before any use:
    // the dependent offset[bin] lookups and the random stores overlap across points
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const uint64_t keep = l2_evict_last();
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < Np;
         i0 += kScatterILP * stride) {
        uint32_t slot[kScatterILP], rk[kScatterILP];
        T xv[kScatterILP], yv[kScatterILP], zv[kScatterILP];
#pragma unroll
        for (int u = 0; u < kScatterILP; ++u) {
            const int64_t i = i0 + u * stride;
            const bool ok = i < Np;
            slot[u] = ok ? __ldcs(bin_of + i) : 0u;
            rk[u] = ok ? __ldcs(rank_of + i) : 0u;
            xv[u] = ok ? __ldcs(x + i) : (T)0;
            yv[u] = ok ? __ldcs(y + i) : (T)0;
            zv[u] = ok ? __ldcs(z + i) : (T)0;
        }
#pragma unroll
        for (int u = 0; u < kScatterILP; ++u) {
            const int64_t i = i0 + u * stride;
            if (i < Np) {
                slot[u] = ld_keep(offset + slot[u], keep) + rk[u];
                NUFFT_CHECK(slot[u] < (uint32_t)Np);
            }
        }
#pragma unroll
        for (int u = 0; u < kScatterILP; ++u) {
            const int64_t i = i0 + u * stride;
            if (i >= Np) break;
            const double sx = fold_rescale((double)xv[u], g.L, g.scale[0], g.nf[0]);
            const double sy = fold_rescale((double)yv[u], g.L, g.scale[1], g.nf[1]);
            const double sz = slab_z(g, fold_rescale((double)zv[u], g.L, g.scale[2], g.nf[2]));
            int lax, lay, laz;
            double ddx, ddy, ddz;
            local_stencil(sx, cell_of(sx, g.nf[0]), g.T[0], g.w, &lax, &ddx);
            local_stencil(sy, cell_of(sy, g.nf[1]), g.T[1], g.w, &lay, &ddy);
            local_stencil(sz, cell_of(sz + (double)g.z_lo, g.nf[2]) - (int)g.z_lo, g.T[2], g.w,
                          &laz, &ddz);
            PtRec<T> r;
            r.d[0] = (T)ddx;
            r.d[1] = (T)ddy;
            r.d[2] = (T)ddz;
            r.la = (uint32_t)lax | ((uint32_t)lay << 8) | ((uint32_t)laz << 16);
            r.perm = (uint32_t)i;
            store_rec_cs(&rec[slot[u]], r);
        }
    }
}

// Per-point ES weights in sorted order (opts.precompute): one thread per point
// evaluates its 3w weights (3w independent evaluations: no dependent chain) and
// stages them in shared memory; the block then writes its points' rows as one
// contiguous, coalesced run.
constexpr int kWThreads = 128;  // 128 x 3w x 8 B <= 48 KB of static shared memory

template <typename T, int W>
__global__ void __launch_bounds__(kWThreads) weights_kernel(const PtRec<T>* __restrict__ rec,
                                                             int64_t Np, T beta,
                                                             T* __restrict__ out) {
    constexpr int R = 3 * W;
    __shared__ T stage[kWThreads * R];
    const T two_over_w = (T)2 / (T)W;
    for (int64_t base = (int64_t)blockIdx.x * kWThreads; base < Np;
         base += (int64_t)gridDim.x * kWThreads) {
        const int64_t i = base + threadIdx.x;
        if (i < Np) {
            const PtRec<T> r = rec[i];
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int k = 0; k < W; ++k)
                    stage[threadIdx.x * R + d * W + k] =
                        dev::es_weight<T>(((T)k - r.d[d]) * two_over_w, beta);
        }
        __syncthreads();
        const int64_t n = min((int64_t)kWThreads, Np - base);
        T* dst = out + base * R;
        for (int e = threadIdx.x; e < (int)(n * R); e += kWThreads) dst[e] = stage[e];
        __syncthreads();
    }
}

// per-bin starts from the (bin, sub-bin) key starts: offset[b] = offset_key[b nsub]
__global__ void bin_offsets_kernel(const uint32_t* __restrict__ offset_key, int64_t nbins,
                                   int nsub, uint32_t* __restrict__ offset) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= nbins;
         b += (int64_t)gridDim.x * blockDim.x)
        offset[b] = offset_key[b * nsub];
}

inline int grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    const int64_t cap = 148 * 16;  // persistent-style cap: 16 resident CTAs per SM
    if (b > cap) b = cap;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

size_t scan_blocksum_elems(int64_t nbins) { return (size_t)((nbins + kScanTile - 1) / kScanTile) + 1; }

template <typename T>
cudaError_t launch_bin_sort(const Geom& g, int64_t Np, const T* x, const T* y, const T* z,
                            uint32_t* count, uint32_t* offset_key, uint32_t* offset,
                            uint32_t* blocksum, uint32_t* bin_of, uint32_t* rank_of,
                            PtRec<T>* rec, int64_t nbins_, cudaStream_t s) {
    const int64_t nbins = nbins_ * (g.nsub > 1 ? g.nsub : 1);  // sort keys
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(uint32_t) * (size_t)nbins, s);
    if (e != cudaSuccess) return e;
    if (Np > 0) {
        bin_count_kernel<T><<<grid_for(Np, kSortThreads), kSortThreads, 0, s>>>(
            g, Np, x, y, z, count, bin_of, rank_of);
    }
    const int64_t ntiles = (nbins + kScanTile - 1) / kScanTile;
    scan_tile_sums<<<(unsigned)ntiles, kScanThreads, 0, s>>>(count, nbins, blocksum);
    scan_sums<<<1, kScanThreads, 0, s>>>(blocksum, ntiles);
    scan_tiles<<<(unsigned)ntiles, kScanThreads, 0, s>>>(count, nbins, blocksum, offset_key);
    if (Np > 0) {
        scatter_kernel<T><<<grid_for(Np, kSortThreads), kSortThreads, 0, s>>>(
            g, Np, x, y, z, bin_of, rank_of, offset_key, rec);
    }
    if (g.nsub > 1)
        bin_offsets_kernel<<<grid_for(nbins_ + 1, kSortThreads), kSortThreads, 0, s>>>(
            offset_key, nbins_, g.nsub, offset);
    return cudaGetLastError();
}

// out = exclusive prefix sum of count[0, n) (n + 1 entries: out[n] = total), the same
// three-phase warp-shuffle scan as setpts; blocksum: scan_blocksum_elems(n) entries
cudaError_t launch_exclusive_scan(const uint32_t* count, int64_t n, uint32_t* blocksum,
                                  uint32_t* out, cudaStream_t s) {
    const int64_t ntiles = (n + kScanTile - 1) / kScanTile;
    if (ntiles == 0) return cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
    scan_tile_sums<<<(unsigned)ntiles, kScanThreads, 0, s>>>(count, n, blocksum);
    scan_sums<<<1, kScanThreads, 0, s>>>(blocksum, ntiles);
    scan_tiles<<<(unsigned)ntiles, kScanThreads, 0, s>>>(count, n, blocksum, out);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_weights(const PtRec<T>* rec, int64_t Np, int w, double beta, T* out,
                           cudaStream_t s) {
    if (Np <= 0) return cudaSuccess;
    int64_t blocks = (Np + kWThreads - 1) / kWThreads;
    if (blocks > 148 * 32) blocks = 148 * 32;
    switch (w) {
#define NUFFT_WK(WW)                                                                       \
    case WW:                                                                               \
        weights_kernel<T, WW><<<(unsigned)blocks, kWThreads, 0, s>>>(rec, Np, (T)beta, out); \
        break;
        NUFFT_WK(2) NUFFT_WK(3) NUFFT_WK(4) NUFFT_WK(5) NUFFT_WK(6) NUFFT_WK(7) NUFFT_WK(8)
        NUFFT_WK(9) NUFFT_WK(10) NUFFT_WK(11) NUFFT_WK(12) NUFFT_WK(13) NUFFT_WK(14)
        NUFFT_WK(15) NUFFT_WK(16)
#undef NUFFT_WK
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
template cudaError_t launch_weights<float>(const PtRec<float>*, int64_t, int, double, float*,
                                           cudaStream_t);
template cudaError_t launch_weights<double>(const PtRec<double>*, int64_t, int, double, double*,
                                            cudaStream_t);

template cudaError_t launch_bin_sort<float>(const Geom&, int64_t, const float*, const float*,
                                            const float*, uint32_t*, uint32_t*, uint32_t*, uint32_t*,
                                            uint32_t*, uint32_t*, PtRec<float>*, int64_t,
                                            cudaStream_t);
template cudaError_t launch_bin_sort<double>(const Geom&, int64_t, const double*, const double*,
                                             const double*, uint32_t*, uint32_t*, uint32_t*, uint32_t*,
                                             uint32_t*, uint32_t*, PtRec<double>*, int64_t,
                                             cudaStream_t);

}  // namespace nufft
