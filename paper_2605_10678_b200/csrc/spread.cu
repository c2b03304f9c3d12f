// spread.cu -- Step 1 of Eq. (3), the spreading operator C.
//
// One CTA per bin (tile of T^3 fine cells).  The CTA owns a shared-memory
// subgrid of (T + w)^3 complex cells ("a shared memory histogram of size
// prod(T_i + w)") and processes the bin's sorted points in
// batches:
//
//   phase A  one thread per point evaluates the 3w ES weights in registers --
//            d w evaluations per point thanks to separability
//            (PAPER.md:193-196), phi evaluated directly -- and
//            stages, per point, the w x w products wx*wy laid out by lane slot
//            and the complex z-profile c*wz;
//   phase B  accumulation WITHOUT atomics: warp k owns the subgrid z-planes
//            {z : z mod NW == k} (absolute ownership, so no barrier or point
//            order is needed between points); for every point, the warp takes
//            the planes of the point's stencil that it owns and its 32 lanes
//            cover the w x w (x, y) cells of each such plane -- one shared
//            load, two FMAs and one shared store per cell.  No two threads ever
//            touch the same cell concurrently (the paper's Grid-Parallel
//            ownership, with its z-split of the stencil across
//            teams).  On sm_100a shared-memory float atomics are
//            CAS loops (ATOMS.CAST.SPIN), so ownership beats atomics;
//   flush    each subgrid row is added into the periodic fine grid in HBM by
//            the bulk-async engine: cp.reduce.async.bulk ... .add.f32/.f64
//            (SASS UBLKRED), one instruction per contiguous row segment; rows
//            that cross the periodic boundary split into two segments, so the
//            ghost cells wrap directly and no separate
//            ghost-fold pass exists on one GPU.
#include "device_util.cuh"
#include "internal.cuh"

namespace nufft {

namespace {

using namespace dev;

// NW = warps per CTA (4 or 8): the plane owners; compile-time, so plane ownership is
// a mask, not a modulo.  Chosen per plan (opts spread_warps / built-in heuristic).
// points staged per batch
template <typename T> struct Batch;
template <> struct Batch<float> { static constexpr int value = 64; };
template <> struct Batch<double> { static constexpr int value = 32; };

// V: value type of strengths and grid cells, Cx<T> (complex) or T (real)
template <typename T, typename V, int W>
struct SpreadSmem {
    using C = V;
    static constexpr int B = Batch<T>::value;
    static constexpr int NQ = (W * W + 31) / 32;
    // per point: wxy[NQ*32] reals (by lane slot), cwz[W] complex, strength, 1D weights
    // [3][W] reals, base + lz ints
    static constexpr size_t batch_bytes() {
        return (size_t)B * NQ * 32 * sizeof(T) + (size_t)B * W * sizeof(C) + (size_t)B * sizeof(C) +
               (size_t)B * 3 * W * sizeof(T) + (size_t)B * 2 * sizeof(int);
    }
    static size_t bytes(int ncell) { return (size_t)ncell * sizeof(C) + batch_bytes(); }
};

template <typename T, typename V, int W, int NW>
__global__ void __launch_bounds__(32 * NW)
    spread_tile_kernel(Geom g, PtsView<T> p, const V* __restrict__ c, V* __restrict__ grid,
                       T beta) {
    using C = V;
    using S = SpreadSmem<T, V, W>;
    constexpr int B = S::B;
    constexpr int NQ = S::NQ;
    constexpr int kSpreadThreads = 32 * NW;
    extern __shared__ __align__(16) unsigned char smem[];

    const int b = blockIdx.x;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const TileX tx = tile_x<sizeof(C)>(bx, g.T[0], W);
    const int Ey = g.T[1] + W, Ez = g.T[2] + W;
    const int pitch = tx.pitch, plane = pitch * Ey, ncell = plane * Ez;
    C* tile = reinterpret_cast<C*>(smem);
    T* swxy = reinterpret_cast<T*>(tile + ncell);          // [B][NQ*32]
    C* scwz = reinterpret_cast<C*>(swxy + B * NQ * 32);   // [B][W]
    C* scv = scwz + B * W;                                 // [B] strengths
    T* sw1d = reinterpret_cast<T*>(scv + B);               // [B][3][W] 1D weights
    int* sbase = reinterpret_cast<int*>(sw1d + B * 3 * W); // [B]
    int* slz = sbase + B;                                  // [B]

    for (int i = threadIdx.x; i < ncell; i += kSpreadThreads) tile[i] = vzero<C>();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int qoff[NQ];
    bool qok[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int s = lane + 32 * q;
        qok[q] = s < W * W;
        qoff[q] = qok[q] ? (s / W) * pitch + (s % W) : 0;
    }
    const T two_over_w = (T)2 / (T)W;

    for (uint32_t p0 = beg; p0 < end; p0 += B) {
        const int n = (int)min((uint32_t)B, end - p0);
        __syncthreads();  // previous batch consumed (first round: tile zeroed)
        // ---- phase A1: one thread per (point, axis, node): ES weight; strength; base
        for (int e = threadIdx.x; e < 3 * W * n; e += kSpreadThreads) {
            const int t = e / W, k = e - t * W;
            const int i = t / 3, d = t - 3 * i;
            const PtRec<T>& rr = p.rec[p0 + i];
            sw1d[e] = p.w ? p.w[(size_t)p0 * (3 * W) + e]  // precomputed at setpts
                          : es_weight<T>(((T)k - rr.d[d]) * two_over_w, beta);
            if (d == 2 && k == 0) {
                const uint32_t la = rr.la;
                const int lz = (int)(la >> 16);
                sbase[i] = (lz * Ey + (int)((la >> 8) & 0xff)) * pitch + (int)(la & 0xff) + tx.shift;
                slz[i] = lz;
                scv[i] = c[rr.perm];
            }
        }
        __syncthreads();
        // ---- phase A2: wx*wy by lane slot, c*wz
        for (int e = threadIdx.x; e < n * NQ * 32; e += kSpreadThreads) {
            const int i = e / (NQ * 32), s = e - i * (NQ * 32);
            const T* wd = sw1d + i * 3 * W;
            swxy[e] = s < W * W ? wd[W + s / W] * wd[s % W] : (T)0;
        }
        for (int e = threadIdx.x; e < n * W; e += kSpreadThreads) {
            const int i = e / W, k = e - i * W;
            const T wz = sw1d[i * 3 * W + 2 * W + k];
            const C cv = scv[i];
            scwz[e] = vscale(cv, wz);
        }
        __syncthreads();
        // ---- phase B: warp-owned z-planes {z : z % NW == warp}
        for (int i = 0; i < n; ++i) {
            const int lz = slz[i];
            int k = (warp - lz) & (NW - 1);  // first owned plane offset in the stencil
            if (k >= W) continue;
            T wq[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) wq[q] = swxy[i * NQ * 32 + lane + 32 * q];
            const C* cz = scwz + i * W;
            C* row = tile + sbase[i] + k * plane;
            for (; k < W; k += NW, row += NW * plane) {
                const C cv = cz[k];
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    if (qok[q]) {
                        C* cell = row + qoff[q];
                        C v = *cell;
                        vfma(v, cv, wq[q]);
                        *cell = v;
                    }
                }
            }
        }
    }
    fence_proxy_async_smem();
    __syncthreads();
    // ---- flush: every subgrid row -> periodic fine grid, bulk reductions (UBLKRED)
    const int oy = by * g.T[1] - W / 2, oz = bz * g.T[2] - W / 2;
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    int sg[2], ss[2], sn[2];
    const int nseg = row_segments(tx.gx0, tx.len, nfx, sg, ss, sn);
    for (int r = threadIdx.x; r < Ey * Ez; r += kSpreadThreads) {
        const int cz = r / Ey, cy = r - cz * Ey;
        const int gy = wrap1(oy + cy, nfy), gz = z_row(oz + cz, g);
        if (gz < -g.hz_lo) continue;  // outside the halo-extended slab: all zero
        C* grow = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
        const C* trow = tile + r * pitch;
        for (int k = 0; k < nseg; ++k)
            bulk_red_add(reinterpret_cast<T*>(grow + sg[k]), trow + ss[k],
                         (unsigned)(sn[k] * sizeof(C)));
    }
    bulk_commit();
    bulk_wait_read();  // the subgrid must outlive the bulk reads
}

template <typename T, typename V, int W>
size_t smem_w(const Geom& g) {
    return SpreadSmem<T, V, W>::bytes(tile_pitch<sizeof(V)>(g.T[0], W) * (g.T[1] + W) *
                                      (g.T[2] + W));
}

template <typename T, typename V, int W, int NW>
cudaError_t launch_nw(const Geom& g, const PtsView<T>& p, int64_t nbins, const V* c, V* grid,
                      double beta, cudaStream_t s) {
    const size_t smem = smem_w<T, V, W>(g);
    auto kern = spread_tile_kernel<T, V, W, NW>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
    }
    if (nbins > 0) kern<<<(unsigned)nbins, 32 * NW, smem, s>>>(g, p, c, grid, (T)beta);
    return cudaGetLastError();
}

template <typename T, typename V, int W>
cudaError_t launch_w(const Geom& g, const PtsView<T>& p, int64_t nbins, const V* c, V* grid,
                     double beta, cudaStream_t s) {
    return g.spread_warps == 8 ? launch_nw<T, V, W, 8>(g, p, nbins, c, grid, beta, s)
                               : launch_nw<T, V, W, 4>(g, p, nbins, c, grid, beta, s);
}

}  // namespace

#define NUFFT_W_SWITCH(CALL)                                                              \
    switch (g.w) {                                                                        \
        case 2: return CALL(2); case 3: return CALL(3); case 4: return CALL(4);          \
        case 5: return CALL(5); case 6: return CALL(6); case 7: return CALL(7);          \
        case 8: return CALL(8); case 9: return CALL(9); case 10: return CALL(10);        \
        case 11: return CALL(11); case 12: return CALL(12); case 13: return CALL(13);    \
        case 14: return CALL(14); case 15: return CALL(15); case 16: return CALL(16);    \
        default: break;                                                                   \
    }

template <typename T>
cudaError_t launch_spread(const Geom& g, const PtsView<T>& p, int64_t nbins,
                          const typename Cx<T>::type* c, typename Cx<T>::type* grid, double beta,
                          cudaStream_t s) {
#define CALL(WW) launch_w<T, typename Cx<T>::type, WW>(g, p, nbins, c, grid, beta, s)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t launch_spread_real(const Geom& g, const PtsView<T>& p, int64_t nbins, const T* c,
                               T* grid, double beta, cudaStream_t s) {
#define CALL(WW) launch_w<T, T, WW>(g, p, nbins, c, grid, beta, s)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}

template <typename T>
size_t spread_smem_bytes(const Geom& g) {
#define CALL(WW) smem_w<T, typename Cx<T>::type, WW>(g)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return 0;
}

template cudaError_t launch_spread<float>(const Geom&, const PtsView<float>&, int64_t,
                                          const float2*, float2*, double, cudaStream_t);
template cudaError_t launch_spread<double>(const Geom&, const PtsView<double>&, int64_t,
                                           const double2*, double2*, double, cudaStream_t);
template cudaError_t launch_spread_real<float>(const Geom&, const PtsView<float>&, int64_t,
                                               const float*, float*, double, cudaStream_t);
template cudaError_t launch_spread_real<double>(const Geom&, const PtsView<double>&, int64_t,
                                                const double*, double*, double, cudaStream_t);
template size_t spread_smem_bytes<float>(const Geom&);
template size_t spread_smem_bytes<double>(const Geom&);

}  // namespace nufft
