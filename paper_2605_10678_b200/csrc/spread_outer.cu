// spread_outer.cu -- spreading (Step 1 of Eq. (3), the operator C, PAPER.md:141-142,
// 187-213) as sums of separable outer products, accumulated in registers.
//
// For one bin with a subgrid of E x E x E cells (E = T + w = 16), by separability
// of the ES kernel the spread is
//
//     G[z][y][x] += sum_j  wz_j[z] wy_j[y] b_j[x],     b_j[x] = c_j wx_j[x]
//
// with every 1-D profile zero-padded to the E cells of the subgrid (wx_j[x] =
// phi(2 (x - lx_j - d_j) / w) on the stencil, 0 elsewhere).  Dense padding costs
// more multiply-adds than the w^3 nonzeros, but every one is a register FMA: no
// per-cell shared-memory read-modify-write, atomic, address computation or
// branch (the costs that bound the Tiled / Grid-Parallel spreads of
// PAPER.md:204-209 on sm_100a).
//
// Work split (one CTA of 8 warps per bin): warp k owns the block y in
// [8 (k & 1), +8), z in [4 (k >> 1), +4); lane l owns x = l & 15 and the four
// rows y0 = 8 (k & 1) + 4 (l >> 4) .. y0 + 3 of those four planes: 16 complex
// accumulators per thread, private.  Per visited point a lane loads b[x] (one
// complex), wy[y0..y0+3] and wz[z0..z0+3] (80 B in fp64, conflict-free: a
// quarter-warp reads 8 consecutive b's, the rest is broadcast), forms
// bz = b wz (8 multiplies) and does 32 FMAs -- 2 B of shared memory per FP64
// op, the sm_100a balance point of the LSU (128 B/clk/SM) and the FP64 pipe.
//
// Batches of B sorted points are double-buffered.  The four warps owning the
// edge z-blocks (0 and 3) see about half the points of the centre blocks, so
// they also PRODUCE batch k+1 while every warp consumes batch k -- one CTA
// barrier per batch, no idle warps:
//   produce  counting-sort the batch by (lz, y-class) in shared memory -- y-class
//            0 / 2 = stencil inside the lower / upper 8 rows, 1 = both -- so each
//            warp's visits are contiguous runs; evaluate the 3w weights per
//            point, one (point, axis, node) per thread, phi evaluated directly
//            (PAPER.md:176), into zero-padded rows;
//   consume  each warp walks the (lz, class) runs that intersect its block;
//   flush    registers -> shared-memory subgrid -> periodic fine grid with
//            cp.reduce.async.bulk .add (SASS UBLKRED), split at the periodic
//            boundary (ghost cells wrap directly).
#include "device_util.cuh"
#include "internal.cuh"

namespace nufft {

namespace {

using namespace dev;

constexpr int kOutE = 16;         // subgrid edge, = T + w on every axis
constexpr int kOutThreads = 256;  // 8 warps
constexpr int kProducers = 128;   // warps 0, 1, 6, 7 (edge z-blocks)
constexpr int kMaxKeys = 48;      // 3 (T + 1) <= 45 sort keys (lz, y-class)
template <typename T> struct OuterBatch;
template <> struct OuterBatch<float> { static constexpr int value = 128; };
template <> struct OuterBatch<double> { static constexpr int value = 64; };

// V: value type of strengths and grid cells, Cx<T> (complex) or T (real)
template <typename T, typename V, int W>
struct OuterSmem {
    using C = V;
    static constexpr int E = kOutE;
    static constexpr int B = OuterBatch<T>::value;
    // staging x pitch: cells of < 16 bytes start the row at a 16-byte aligned global x
    // (shift < A = 16 / cell bytes columns), so the row gets A extra cells
    static constexpr int A = sizeof(C) >= 16 ? 1 : 16 / (int)sizeof(C);
    static constexpr int P = A == 1 ? E : E + A;
    static constexpr size_t tile_bytes = (size_t)E * E * P * sizeof(C);
    // one buffer: b = c wx [B][E] complex | wy [B][E] | wz [B][E]
    static constexpr size_t buf_bytes = (size_t)B * E * (sizeof(C) + 2 * sizeof(T));
    static constexpr size_t meta_bytes = (size_t)B * sizeof(C)        // c
                                         + (size_t)B * 4 * sizeof(T)  // d[3]
                                         + (size_t)B * 3 * sizeof(int);  // la, key, rank
    static constexpr size_t staging = 2 * buf_bytes + meta_bytes;
    static constexpr size_t region = tile_bytes > staging ? tile_bytes : staging;
    static constexpr size_t bytes() { return region + 3 * (kMaxKeys + 2) * sizeof(int); }
};

template <typename T> struct Vec4;
template <> struct Vec4<float> {
    __device__ static void load(float (&v)[4], const float* s) {
        const float4 a = *reinterpret_cast<const float4*>(s);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
};
template <> struct Vec4<double> {
    __device__ static void load(double (&v)[4], const double* s) {
        const double2 a = reinterpret_cast<const double2*>(s)[0];
        const double2 b = reinterpret_cast<const double2*>(s)[1];
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
};

#ifdef NUFFT_OUTER_PROF
// debug builds only (-DNUFFT_OUTER_PROF): per warp, clock cycles spent producing,
// consuming and waiting at the batch barrier, summed over all CTAs
__device__ unsigned long long g_outer_prof[8][8];  // [warp][produce, consume, barrier, p.zero, p.load, p.scan, p.weights, -]
#define OUTER_PROF_T(v) const long long v = clock64()
#define OUTER_PROF_ADD(w, k, d) \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_outer_prof[w][k], (unsigned long long)(d))
#else
#define OUTER_PROF_T(v)
#define OUTER_PROF_ADD(w, k, d)
#endif

template <int BAR, int NT>
__device__ __forceinline__ void group_sync() {
    if constexpr (BAR == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}

template <typename T, typename V>
struct OuterPtrs {
    using C = V;
    C* sc;       // [B]    strength
    T* sd;       // [B][4] phase offsets
    int* sla;    // [B]    packed stencil base
    int* skey;   // [B]    sort key
    int* srank;  // [B]    rank within key
    int* gcnt;   // [NK]   key counts
};

// Produce one batch into buffer `buf` (b | wy | wz) and its key starts `goff`,
// using NT threads (tid in [0, NT)) synchronised by barrier BAR.  No trailing
// barrier: the caller's CTA barrier publishes the batch.
template <typename T, typename V, int W, int NT, int BAR>
__device__ __forceinline__ void produce(int tid, const PtsView<T>& p, const V* __restrict__ c,
                                        uint32_t p0, int n, T* buf, int* goff,
                                        const OuterPtrs<T, V>& m, T beta) {
    using C = V;
    using S = OuterSmem<T, V, W>;
    constexpr int E = kOutE, B = S::B, TT = E - W, NK = 3 * (TT + 1);
    C* sb = reinterpret_cast<C*>(buf);
    T* swy = reinterpret_cast<T*>(sb + B * E);
    OUTER_PROF_T(q0);
    // zero the profiles (every row is written densely below only on its stencil)
    float4* z4 = reinterpret_cast<float4*>(buf);
    for (int i = tid; i < (int)(S::buf_bytes / 16); i += NT) z4[i] = float4{0.f, 0.f, 0.f, 0.f};
    for (int i = tid; i < NK; i += NT) m.gcnt[i] = 0;
    group_sync<BAR, NT>();
    OUTER_PROF_T(q1);
    for (int t = tid; t < n; t += NT) {
        const PtRec<T> r = load_rec(&p.rec[p0 + t]);
        const int la = (int)r.la;
        const int ly = (la >> 8) & 0xff, lz = la >> 16;
        const int yc = ly + W <= 8 ? 0 : (ly >= 8 ? 2 : 1);
        const int key = 3 * lz + yc;
        m.sla[t] = la;
        m.skey[t] = key;
        m.sd[4 * t + 0] = r.d[0];
        m.sd[4 * t + 1] = r.d[1];
        m.sd[4 * t + 2] = r.d[2];
        m.sc[t] = c[r.perm];
        m.srank[t] = atomicAdd(&m.gcnt[key], 1);
    }
    group_sync<BAR, NT>();
    OUTER_PROF_T(q2);
    if (tid < 32) {  // exclusive scan of the NK <= 45 key counts, 2 per lane
        const int lane = tid;
        const int a0 = 2 * lane < NK ? m.gcnt[2 * lane] : 0;
        const int a1 = 2 * lane + 1 < NK ? m.gcnt[2 * lane + 1] : 0;
        int s = a0 + a1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += u;
        }
        const int ex = s - a0 - a1;
        if (2 * lane <= NK) goff[2 * lane] = ex;
        if (2 * lane + 1 <= NK) goff[2 * lane + 1] = ex + a0;
    }
    group_sync<BAR, NT>();
    OUTER_PROF_T(q3);
    // weights: one (point, axis) per thread, its w nodes as w independent
    // evaluations (the producer warps are latency-bound on one dependent
    // sqrt / exp chain per thread otherwise: measured, scripts/outer_prof.py)
    const T two_over_w = (T)2 / (T)W;
    for (int e = tid; e < n * 3; e += NT) {
        const int t = e / 3, d = e - 3 * t;
        const int la = m.sla[t];
        const int pos = goff[m.skey[t]] + m.srank[t];
        const int x0 = (la >> (8 * d)) & 0xff;
        const T dd = m.sd[4 * t + d];
        T wk[W];
#pragma unroll
        for (int k = 0; k < W; ++k)
            wk[k] = p.w ? p.w[(size_t)(p0 + t) * (3 * W) + d * W + k]  // precomputed at setpts
                        : es_weight<T>(((T)k - dd) * two_over_w, beta);
        if (d == 0) {
            const C cv = m.sc[t];
            C* row = sb + pos * E + x0;
#pragma unroll
            for (int k = 0; k < W; ++k) row[k] = vscale(cv, wk[k]);
        } else {
            T* row = swy + (d - 1) * B * E + pos * E + x0;  // d = 1: wy, d = 2: wz
#pragma unroll
            for (int k = 0; k < W; ++k) row[k] = wk[k];
        }
    }
#ifdef NUFFT_OUTER_PROF
    if (BAR == 1) {
        OUTER_PROF_T(q4);
        const int wp = threadIdx.x >> 5;
        OUTER_PROF_ADD(wp, 3, q1 - q0);
        OUTER_PROF_ADD(wp, 4, q2 - q1);
        OUTER_PROF_ADD(wp, 5, q3 - q2);
        OUTER_PROF_ADD(wp, 6, q4 - q3);
    }
#endif
}

// resident CTAs per SM: fp64 needs 128 registers (2 CTAs); fp32 fits 3 (<= 85
// registers, 3 x 71 KB shared memory), which hides the per-bin prologue latency
// at low density (one batch per bin)
template <typename T> struct OuterMinBlocks { static constexpr int value = sizeof(T) == 4 ? 3 : 2; };

template <typename T, typename V, int W>
__global__ void __launch_bounds__(kOutThreads, OuterMinBlocks<T>::value)
    spread_outer_kernel(Geom g, PtsView<T> p, const V* __restrict__ c, V* __restrict__ grid,
                        T beta) {
    using C = V;
    using S = OuterSmem<T, V, W>;
    constexpr int E = kOutE;
    constexpr int P = S::P;
    constexpr int B = S::B;
    constexpr int TT = E - W;  // bin edge; lz, ly in [0, TT]
    static_assert(3 * (TT + 1) <= kMaxKeys, "sort keys");
    extern __shared__ __align__(16) unsigned char smem[];

    OUTER_PROF_T(tk0);
    const int b = blockIdx.x;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    // double-buffered staging: buffer i at smem + i * buf_bytes, key starts goff0 + i * stride
    OuterPtrs<T, V> m;
    m.sc = reinterpret_cast<C*>(smem + 2 * S::buf_bytes);
    m.sd = reinterpret_cast<T*>(m.sc + B);
    m.sla = reinterpret_cast<int*>(m.sd + 4 * B);
    m.skey = m.sla + B;
    m.srank = m.skey + B;
    m.gcnt = reinterpret_cast<int*>(smem + S::region);
    int* goff0 = m.gcnt + kMaxKeys + 2;
    constexpr int kGoffStride = kMaxKeys + 2;
    C* tile = reinterpret_cast<C*>(smem);  // [E][E][P] (flush only; aliases the staging)

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = warp & 1, zb = warp >> 1, z0 = 4 * zb;
    const int x = lane & 15, y0 = 8 * h + 4 * (lane >> 4);
    const bool producer = zb == 0 || zb == 3;
    const int ptid = (warp < 2 ? warp : warp - 4) * 32 + lane;  // producers: 0..127

    C acc[4][4];  // [z0 + k][y0 + i] at column x
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[k][i] = vzero<C>();

    // this warp's runs: lz whose stencil [lz, lz + w) meets [z0, z0 + 4), and the
    // y-classes meeting its half: {0, 1} for the lower, {1, 2} for the upper rows
    const int lz_lo = max(0, z0 - W + 1), lz_hi = min(TT, z0 + 3);
    const int c_lo = h, c_hi = h + 1;

    const int nbatch = (int)((end - beg + B - 1) / B);
    produce<T, V, W, kOutThreads, 0>(threadIdx.x, p, c, beg, (int)min((uint32_t)B, end - beg),
                                  reinterpret_cast<T*>(smem), goff0, m, beta);
    __syncthreads();
    for (int kb = 0; kb < nbatch; ++kb) {
        OUTER_PROF_T(t0);
        if (producer && kb + 1 < nbatch) {
            const uint32_t p1 = beg + (uint32_t)(kb + 1) * B;
            produce<T, V, W, kProducers, 1>(ptid, p, c, p1, (int)min((uint32_t)B, end - p1),
                                         reinterpret_cast<T*>(smem + ((kb + 1) & 1) * S::buf_bytes),
                                         goff0 + ((kb + 1) & 1) * kGoffStride, m, beta);
        }
        OUTER_PROF_T(t1);
        // ---- consume: register accumulation over this warp's runs
        const C* sb = reinterpret_cast<const C*>(smem + (kb & 1) * S::buf_bytes);
        const T* swy = reinterpret_cast<const T*>(sb + B * E);
        const T* swz = swy + B * E;
        const int* goff = goff0 + (kb & 1) * kGoffStride;
        for (int lz = lz_lo; lz <= lz_hi; ++lz) {
            const int j1 = goff[3 * lz + c_hi + 1];
            for (int j = goff[3 * lz + c_lo]; j < j1; ++j) {
                const C bxv = sb[j * E + x];
                T wy[4], wz[4];
                Vec4<T>::load(wy, swy + j * E + y0);
                Vec4<T>::load(wz, swz + j * E + z0);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const C z = vscale(bxv, wz[k]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) vfma(acc[k][i], z, wy[i]);
                }
            }
        }
        OUTER_PROF_T(t2);
        __syncthreads();  // batch kb consumed, batch kb + 1 produced
        OUTER_PROF_T(t3);
        OUTER_PROF_ADD(warp, 0, t1 - t0);
        OUTER_PROF_ADD(warp, 1, t2 - t1);
        OUTER_PROF_ADD(warp, 2, t3 - t2);
    }
    // ---- flush: registers -> smem subgrid -> periodic fine grid (bulk reductions)
    const TileX tx = tile_x<sizeof(C)>(bx, TT, W);
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            NUFFT_CHECK(tx.shift + x < P);
            tile[((z0 + k) * E + y0 + i) * P + tx.shift + x] = acc[k][i];
        }
    if constexpr (P > E) {  // zero the P - E pad columns outside the shifted window
        const int rr = threadIdx.x;  // E*E == kOutThreads rows
#pragma unroll
        for (int q = 0; q < P - E; ++q) {
            const int col = q < tx.shift ? q : E + q;
            tile[rr * P + col] = vzero<C>();
        }
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int oy = by * TT - W / 2, oz = bz * TT - W / 2;
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    int sg[2], ss[2], sn[2];
    const int nseg = row_segments(tx.gx0, P, nfx, sg, ss, sn);
    {
        const int r = threadIdx.x;  // one row per thread
        const int cz = r / E, cy = r - cz * E;
        const int gy = wrap1(oy + cy, nfy), gz = z_row(oz + cz, g);
        C* grow = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
        const C* trow = tile + r * P;
        for (int k = 0; k < (gz < -g.hz_lo ? 0 : nseg); ++k)
            bulk_red_add(reinterpret_cast<T*>(grow + sg[k]), trow + ss[k],
                         (unsigned)(sn[k] * sizeof(C)));
    }
    bulk_commit();
    bulk_wait_read();  // the staged rows must outlive the bulk reads
#ifdef NUFFT_OUTER_PROF
    OUTER_PROF_T(tk1);
    OUTER_PROF_ADD(threadIdx.x >> 5, 7, tk1 - tk0);
#endif
}

template <typename T, typename V, int W>
cudaError_t launch_outer_w(const Geom& g, const PtsView<T>& p, int64_t nbins, const V* c,
                           V* grid, double beta, cudaStream_t s) {
    const size_t smem = OuterSmem<T, V, W>::bytes();
    auto kern = spread_outer_kernel<T, V, W>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
    }
    if (nbins > 0) kern<<<(unsigned)nbins, kOutThreads, smem, s>>>(g, p, c, grid, (T)beta);
    return cudaGetLastError();
}

}  // namespace

bool spread_outer_applies(const Geom& g) {
    return g.w >= 2 && g.w <= 12 && g.T[0] == kOutE - g.w && g.T[1] == kOutE - g.w &&
           g.T[2] == kOutE - g.w;
}

template <typename T>
size_t spread_outer_smem_bytes(const Geom& g) {
    switch (g.w) {
#define NUFFT_OS(WW) OuterSmem<T, typename Cx<T>::type, WW>::bytes()
        case 2: return NUFFT_OS(2);   case 3: return NUFFT_OS(3);   case 4: return NUFFT_OS(4);
        case 5: return NUFFT_OS(5);   case 6: return NUFFT_OS(6);   case 7: return NUFFT_OS(7);
        case 8: return NUFFT_OS(8);   case 9: return NUFFT_OS(9);   case 10: return NUFFT_OS(10);
        case 11: return NUFFT_OS(11); case 12: return NUFFT_OS(12);
#undef NUFFT_OS
        default: return 0;
    }
}

template <typename T, typename V>
cudaError_t launch_outer_v(const Geom& g, const PtsView<T>& p, int64_t nbins, const V* c,
                           V* grid, double beta, cudaStream_t s) {
    if (!spread_outer_applies(g)) return cudaErrorNotSupported;
    switch (g.w) {
#define NUFFT_OW(WW) \
    case WW:         \
        return launch_outer_w<T, V, WW>(g, p, nbins, c, grid, beta, s);
        NUFFT_OW(2) NUFFT_OW(3) NUFFT_OW(4) NUFFT_OW(5) NUFFT_OW(6) NUFFT_OW(7) NUFFT_OW(8)
        NUFFT_OW(9) NUFFT_OW(10) NUFFT_OW(11) NUFFT_OW(12)
#undef NUFFT_OW
        default:
            return cudaErrorNotSupported;
    }
}

template <typename T>
cudaError_t launch_spread_outer(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                const typename Cx<T>::type* c, typename Cx<T>::type* grid,
                                double beta, cudaStream_t s) {
    return launch_outer_v<T, typename Cx<T>::type>(g, p, nbins, c, grid, beta, s);
}
template <typename T>
cudaError_t launch_spread_outer_real(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                     const T* c, T* grid, double beta, cudaStream_t s) {
    return launch_outer_v<T, T>(g, p, nbins, c, grid, beta, s);
}

template cudaError_t launch_spread_outer<float>(const Geom&, const PtsView<float>&, int64_t,
                                                const float2*, float2*, double, cudaStream_t);
template cudaError_t launch_spread_outer<double>(const Geom&, const PtsView<double>&, int64_t,
                                                 const double2*, double2*, double, cudaStream_t);
template cudaError_t launch_spread_outer_real<float>(const Geom&, const PtsView<float>&, int64_t,
                                                     const float*, float*, double, cudaStream_t);
template cudaError_t launch_spread_outer_real<double>(const Geom&, const PtsView<double>&, int64_t,
                                                      const double*, double*, double,
                                                      cudaStream_t);
template size_t spread_outer_smem_bytes<float>(const Geom&);
template size_t spread_outer_smem_bytes<double>(const Geom&);

}  // namespace nufft

#ifdef NUFFT_OUTER_PROF
// debug builds only: read (and reset) the per-warp produce / consume / barrier cycles
extern "C" int nufft_debug_outer_prof(unsigned long long out[64]) {
    if (cudaMemcpyFromSymbol(out, nufft::g_outer_prof, sizeof(unsigned long long) * 64) !=
        cudaSuccess)
        return NUFFT_ERR_CUDA;
    unsigned long long z[64] = {};
    return cudaMemcpyToSymbol(nufft::g_outer_prof, z, sizeof(z)) == cudaSuccess ? NUFFT_OK
                                                                                 : NUFFT_ERR_CUDA;
}
#endif
