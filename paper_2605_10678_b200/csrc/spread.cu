// spread.cu -- Step 1 of Eq. (3), the spreading operator C.
//
// One CTA per bin (tile of T^3 fine cells).  The CTA owns a shared-memory
// subgrid of (T + w)^3 complex cells ("a shared memory histogram of size
// prod(T_i + w)").  The bin's sorted points are split evenly
// over the warps, which then work independently (no CTA barrier between the
// zero fill and the flush):
//
//   weights  lane l loads point l of a 32-point chunk (sorted record, strength
//            gathered through perm) and evaluates its 3w ES weights in
//            registers -- d w evaluations per point thanks to separability
//            (PAPER.md:193-196), phi evaluated directly --
//            parked in a per-warp buffer as wx, wy and the complex z-profile
//            c * wz;
//   deposit  the warp walks the chunk's points; lane slots cover the w x w
//            (x, y) columns of the stencil, each adds c wz wx wy into its w
//            z-cells.  A shared-memory cell update is ONE packed compare-and-
//            swap of the whole complex value (fp32: 64-bit CAS of (re, im);
//            fp64: atom.shared.cas.b128).  On sm_100a shared-memory float
//            atomics are CAS loops anyway (ATOMS.CAST.SPIN), so packing both
//            components into one CAS halves the atomic count of the paper's
//            Tiled spread without the per-warp ownership
//            bookkeeping of its Grid-Parallel variant;
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

constexpr int kSpreadThreads = 256;
constexpr int kSpreadWarps = kSpreadThreads / 32;
// points per warp chunk (fp64 halves it to keep the per-warp buffers small)
template <typename T> struct Chunk;
template <> struct Chunk<float> { static constexpr int value = 32; };
template <> struct Chunk<double> { static constexpr int value = 16; };

// cell += a * s with one packed 64-bit CAS of (re, im); retries are rare
__device__ __forceinline__ void smem_cas_add(float2* cell, float2 a, float s) {
    unsigned long long* p = reinterpret_cast<unsigned long long*>(cell);
    unsigned long long seen = *reinterpret_cast<volatile unsigned long long*>(p);
    float2 v = *reinterpret_cast<float2*>(&seen);
    v.x = fmaf(a.x, s, v.x);
    v.y = fmaf(a.y, s, v.y);
    unsigned long long old = atomicCAS(p, seen, *reinterpret_cast<unsigned long long*>(&v));
    while (__builtin_expect(old != seen, 0)) {
        seen = old;
        v = *reinterpret_cast<float2*>(&seen);
        v.x = fmaf(a.x, s, v.x);
        v.y = fmaf(a.y, s, v.y);
        old = atomicCAS(p, seen, *reinterpret_cast<unsigned long long*>(&v));
    }
}

__device__ __forceinline__ bool cas128(unsigned addr, double2& cur, double nx, double ny) {
    unsigned long long o0, o1;
    asm volatile(
        "{\n\t.reg .b128 cmp, nw, old;\n\t"
        "mov.b128 cmp, {%2, %3};\n\t"
        "mov.b128 nw, {%4, %5};\n\t"
        "atom.shared.cas.b128 old, [%6], cmp, nw;\n\t"
        "mov.b128 {%0, %1}, old;\n\t}"
        : "=l"(o0), "=l"(o1)
        : "l"(__double_as_longlong(cur.x)), "l"(__double_as_longlong(cur.y)),
          "l"(__double_as_longlong(nx)), "l"(__double_as_longlong(ny)), "r"(addr)
        : "memory");
    const bool ok = o0 == (unsigned long long)__double_as_longlong(cur.x) &&
                    o1 == (unsigned long long)__double_as_longlong(cur.y);
    cur.x = __longlong_as_double((long long)o0);
    cur.y = __longlong_as_double((long long)o1);
    return ok;
}

__device__ __forceinline__ void smem_cas_add(double2* cell, double2 a, double s) {
    const unsigned addr = smem_addr(cell);
    const volatile double* vc = reinterpret_cast<volatile double*>(cell);
    double2 cur = make_double2(vc[0], vc[1]);
    bool ok = cas128(addr, cur, fma(a.x, s, cur.x), fma(a.y, s, cur.y));
    while (__builtin_expect(!ok, 0)) ok = cas128(addr, cur, fma(a.x, s, cur.x), fma(a.y, s, cur.y));
}

template <typename T, int W>
struct SpreadSmem {
    using C = typename Cx<T>::type;
    static constexpr int CH = Chunk<T>::value;
    // per point: cwz[W] complex, wx|wy [2W] reals, base int
    static constexpr size_t per_warp() {
        return (size_t)CH * W * sizeof(C) + (size_t)CH * 2 * W * sizeof(T) + CH * sizeof(int);
    }
    static size_t bytes(int ncell) { return (size_t)ncell * sizeof(C) + kSpreadWarps * per_warp(); }
};

template <typename T, int W>
__global__ void __launch_bounds__(kSpreadThreads, 2)
    spread_tile_kernel(Geom g, PtsView<T> p, const typename Cx<T>::type* __restrict__ c,
                       typename Cx<T>::type* __restrict__ grid, T beta) {
    using C = typename Cx<T>::type;
    using S = SpreadSmem<T, W>;
    constexpr int CH = S::CH;
    constexpr int NQ = (W * W + 31) / 32;
    constexpr int NW = kSpreadWarps;
    extern __shared__ __align__(16) unsigned char smem[];

    const int b = blockIdx.x;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const TileX tx = tile_x<sizeof(C)>(bx, g.T[0], W);
    const int Ey = g.T[1] + W, Ez = g.T[2] + W;
    const int pitch = tx.pitch, plane = pitch * Ey, ncell = plane * Ez;
    C* tile = reinterpret_cast<C*>(smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* wsm = smem + (size_t)ncell * sizeof(C) + warp * S::per_warp();
    C* cwz = reinterpret_cast<C*>(wsm);                       // [CH][W]
    T* wxy1 = reinterpret_cast<T*>(cwz + CH * W);            // [CH][2W]: wx | wy
    int* sbase = reinterpret_cast<int*>(wxy1 + CH * 2 * W);  // [CH]

    for (int i = threadIdx.x; i < ncell; i += kSpreadThreads) tile[i] = C{0, 0};

    int qoff[NQ], qx[NQ], qy[NQ];
    bool qok[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int s = lane + 32 * q;
        qok[q] = s < W * W;
        qx[q] = qok[q] ? s % W : 0;
        qy[q] = qok[q] ? s / W : 0;
        qoff[q] = qy[q] * pitch + qx[q];
    }
    const T two_over_w = (T)2 / (T)W;
    // even split of the bin's points over the warps
    const uint32_t n = end - beg;
    const uint32_t wbeg = beg + (uint32_t)(((uint64_t)n * warp) / NW);
    const uint32_t wend = beg + (uint32_t)(((uint64_t)n * (warp + 1)) / NW);
    __syncthreads();

    for (uint32_t c0 = wbeg; c0 < wend; c0 += CH) {
        const int np = (int)min((uint32_t)CH, wend - c0);
        // ---- weights: lane l < np owns point c0 + l
        if (lane < np) {
            const uint32_t slot = c0 + lane;
            const T dx = p.dx[slot], dy = p.dy[slot], dz = p.dz[slot];
            const uint32_t la = p.la[slot];
            const C cv = c[p.perm[slot]];
            sbase[lane] = (int)(((la >> 16) * Ey + ((la >> 8) & 0xff)) * pitch + (la & 0xff)) +
                          tx.shift;
            T* wl = wxy1 + lane * 2 * W;
            C* cl = cwz + lane * W;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const T kk = (T)k;
                wl[k] = es_weight<T>((kk - dx) * two_over_w, beta);
                wl[W + k] = es_weight<T>((kk - dy) * two_over_w, beta);
                const T wz = es_weight<T>((kk - dz) * two_over_w, beta);
                cl[k] = C{cv.x * wz, cv.y * wz};
            }
        }
        __syncwarp();
        // ---- deposit the chunk's points
        for (int j = 0; j < np; ++j) {
            const int base = sbase[j];
            const T* wl = wxy1 + j * 2 * W;
            const C* cl = cwz + j * W;
            T wq[NQ];
            C* cq[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                wq[q] = wl[qx[q]] * wl[W + qy[q]];
                cq[q] = tile + base + qoff[q];
            }
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const C cz = cl[k];
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    if (qok[q]) smem_cas_add(cq[q] + k * plane, cz, wq[q]);
            }
        }
        __syncwarp();
    }
    fence_proxy_async_smem();
    __syncthreads();
    // ---- flush: every subgrid row -> periodic fine grid, bulk reductions (UBLKRED)
    const int oy = by * g.T[1] - W / 2, oz = bz * g.T[2] - W / 2;
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1], nfz = (int)g.nz_loc;
    int sg[2], ss[2], sn[2];
    const int nseg = row_segments(tx.gx0, pitch, nfx, sg, ss, sn);
    for (int r = threadIdx.x; r < Ey * Ez; r += kSpreadThreads) {
        const int cz = r / Ey, cy = r - cz * Ey;
        const int gy = wrap1(oy + cy, nfy), gz = wrap1(oz + cz, nfz);
        C* grow = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
        const C* trow = tile + r * pitch;
        for (int k = 0; k < nseg; ++k)
            bulk_red_add(reinterpret_cast<T*>(grow + sg[k]), trow + ss[k],
                         (unsigned)(sn[k] * sizeof(C)));
    }
    bulk_commit();
    bulk_wait_read();  // the subgrid must outlive the bulk reads
}

template <typename T, int W>
size_t smem_w(const Geom& g) {
    using C = typename Cx<T>::type;
    return SpreadSmem<T, W>::bytes(tile_pitch<sizeof(C)>(g.T[0], W) * (g.T[1] + W) *
                                   (g.T[2] + W));
}

template <typename T, int W>
cudaError_t launch_w(const Geom& g, const PtsView<T>& p, int64_t nbins,
                     const typename Cx<T>::type* c, typename Cx<T>::type* grid, double beta,
                     cudaStream_t s) {
    const size_t smem = smem_w<T, W>(g);
    auto kern = spread_tile_kernel<T, W>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
    }
    if (nbins > 0) kern<<<(unsigned)nbins, kSpreadThreads, smem, s>>>(g, p, c, grid, (T)beta);
    return cudaGetLastError();
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
#define CALL(WW) launch_w<T, WW>(g, p, nbins, c, grid, beta, s)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}

template <typename T>
size_t spread_smem_bytes(const Geom& g) {
#define CALL(WW) smem_w<T, WW>(g)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return 0;
}

template cudaError_t launch_spread<float>(const Geom&, const PtsView<float>&, int64_t,
                                          const float2*, float2*, double, cudaStream_t);
template cudaError_t launch_spread<double>(const Geom&, const PtsView<double>&, int64_t,
                                           const double2*, double2*, double, cudaStream_t);
template size_t spread_smem_bytes<float>(const Geom&);
template size_t spread_smem_bytes<double>(const Geom&);

}  // namespace nufft
