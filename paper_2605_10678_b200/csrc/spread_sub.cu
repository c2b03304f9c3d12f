// spread_sub.cu -- spreading (Step 1 of Eq. (3), the operator C, PAPER.md:141-142,
// 187-213) with sub-bin register rows: the stencil-exact register layout.
//
// The register outer-product spread (spread_outer.cu) pads every 1-D profile to a
// fixed 16-cell subgrid, so at small widths most of its FMAs multiply zeros
// (fp64 w = 5: 12x the w^3 useful updates).  Here the accumulators follow the
// points instead:
//
//   sub-bin   setpts sorts every bin's points by sub-bin: cubes of G = 9 - w
//             stencil bases per axis (Geom::G / ns / nsub), so the stencils of a
//             sub-bin's points all lie in one 8 x 8 x 8 cell block.
//   warp      one warp accumulates one sub-bin at a time, in REGISTERS: lane l
//             owns the two x-rows (y = l & 7, z = l >> 3) and (y, z + 4) of the
//             block, 8 cells each (2 x 8 complex accumulators).  Per point the
//             x extent of the stencil is EXACT: the point's x base dx in [0, G) is
//             warp-uniform, so a branch on dx selects w fixed registers per row
//             (w FMAs per row and component, no zero padding in x); only the
//             (y, z) rows outside the point's w x w stencil idle: 64 row slots for
//             w^2 useful rows (fp64 w = 5: 2.56x instead of 12x).
//   weights   per batch of 32 points lane l evaluates point l's 3w ES weights
//             (separability; phi direct, by the
//             table-assisted es_weight_tab) and stages b = c wx and wy, wz
//             zero-padded to the block's 8 rows in shared memory; the warp then
//             walks the 32 points with broadcast reads (no per-lane index math).
//   flush     the block (its 8 x 8 rows) is added into the CTA's shared-memory
//             subgrid of the bin, (T + w)^3 cells, with shared atomics (blocks of
//             neighbouring sub-bins overlap by w - 1 cells); after the bin the
//             subgrid goes to the periodic fine grid with cp.reduce.async.bulk
//             .add (SASS UBLKRED), rows split at the periodic boundary (ghost
//             cells wrap directly), as in the other spreads.
//
// One CTA of 16 warps per bin; warp k takes the k-th sixteenth of the bin's points
// (sorted by sub-bin), flushing its registers whenever the sub-bin changes.
#include "device_util.cuh"
#include "sub_common.cuh"
#include "internal.cuh"

#include <algorithm>
#include <cstdlib>

namespace nufft {

namespace {

using namespace dev;

template <typename T, typename V, int W, int NW>
struct SubSmem {
    static constexpr int G = kBlk + 1 - W;
    // per warp, 32 staged points: b = c wx [32][W] values | wy, wz zero-padded to the
    // block's 8 rows [32][kYS] reals
    static constexpr size_t stage_bytes =
        ((32 * W * sizeof(V) + 2 * 32 * kYS * sizeof(T)) + 15) / 16 * 16;
    static constexpr size_t fixed = kExpTab * sizeof(double) + NW * stage_bytes;
    static size_t bytes(size_t ncell) { return fixed + ncell * sizeof(V); }
};

// Shared-memory add of one block cell.  fp64 / fp32 adds in shared memory are CAS
// loops on sm_100a (ATOMS.CAST.SPIN): lanes whose words share a bank in one pass
// retry.  The flush therefore runs in rounds of lanes that are conflict-free by
// construction (odd row pitch P / plane stride PS, sub_pitch / sub_plane): complex
// cells take two rounds of 16 lanes (the odd-z lanes add the imaginary part first:
// a select, no branch), real cells four rounds of the 8 lanes of one z.
template <typename V> struct Atom;
template <> struct Atom<double2> {
    static constexpr int rounds = 2;  // 16 lanes x 8 bytes per 128-byte pass
    __device__ static void add(double2* d, const double2& v, bool flip) {
        double* p = reinterpret_cast<double*>(d);
        atomicAdd(p + (flip ? 1 : 0), flip ? v.y : v.x);
        atomicAdd(p + (flip ? 0 : 1), flip ? v.x : v.y);
    }
};
template <> struct Atom<float2> {
    static constexpr int rounds = 2;
    __device__ static void add(float2* d, const float2& v, bool flip) {
        float* p = reinterpret_cast<float*>(d);
        atomicAdd(p + (flip ? 1 : 0), flip ? v.y : v.x);
        atomicAdd(p + (flip ? 0 : 1), flip ? v.x : v.y);
    }
};
template <> struct Atom<double> {
    static constexpr int rounds = 4;  // 8-byte cells, 16-byte aligned rows: one z per pass
    __device__ static void add(double* d, double v, bool) { atomicAdd(d, v); }
};
template <> struct Atom<float> {
    static constexpr int rounds = 4;
    __device__ static void add(float* d, float v, bool) { atomicAdd(d, v); }
};

// acc[r][D + k] += b[k] f_r, k < W, r < R: one point whose x base is D
template <typename V, typename T, int W, int D, int R>
__device__ __forceinline__ void fma_rows(V (&acc)[R][kBlk], const V* b, const T (&f)[R]) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const V bk = b[k];
#pragma unroll
        for (int r = 0; r < R; ++r) vfma(acc[r][D + k], bk, f[r]);
    }
}

// one staged point in registers: b = c wx (W values) and its R row weights wy wz
template <typename V, typename T, int W, int R>
struct PtLoad {
    V b[W];
    T f[R];
    __device__ __forceinline__ void load(int j, const V* sb, const T* wyp, const T* wzp, int zs) {
#pragma unroll
        for (int k = 0; k < W; ++k) b[k] = sb[j * W + k];
        const T wyv = wyp[j * kYS];
#pragma unroll
        for (int r = 0; r < R; ++r) f[r] = wyv * wzp[j * zs + 4 * r];
    }
    template <int D>
    __device__ __forceinline__ void apply(V (&acc)[R][kBlk]) const {
#pragma unroll
        for (int k = 0; k < W; ++k)
#pragma unroll
            for (int r = 0; r < R; ++r) vfma(acc[r][D + k], b[k], f[r]);
    }
};

// Every point of the current run, grouped by x base: for D = 0 .. GX-1 the points
// whose bit is set in dmask[D] & run (warp-uniform masks), so the register indices
// of each group are compile-time constants and no per-point branch is taken.
template <typename V, typename T, int W, int GX, int D, int R, int ZS>
__device__ __forceinline__ void run_points(V (&acc)[R][kBlk], const unsigned (&dmask)[GX],
                                           unsigned run, const V* sb, const T* swy,
                                           const T* swz, int ry, int rz) {
    if constexpr (D < GX) {
        unsigned msk = dmask[D] & run;
        const T* wyp = swy + ry;
        const T* wzp = swz + rz;
        // software-pipelined: the next point's shared loads are issued before the
        // current point's FMAs (two register sets, A / B, alternate)
        if (msk) {
            PtLoad<V, T, W, R> a, b;
            int ja = __ffs(msk) - 1;
            msk &= msk - 1;
            a.load(ja, sb, wyp, wzp, ZS);
            for (;;) {
                const bool hb = msk != 0;
                const int jb = hb ? __ffs(msk) - 1 : ja;
                msk &= msk - 1;
                b.load(jb, sb, wyp, wzp, ZS);
                a.apply<D>(acc);
                if (!hb) break;
                const bool ha = msk != 0;
                ja = ha ? __ffs(msk) - 1 : jb;
                msk &= msk - 1;
                a.load(ja, sb, wyp, wzp, ZS);
                b.apply<D>(acc);
                if (!ha) break;
            }
        }
        run_points<V, T, W, GX, D + 1, R, ZS>(acc, dmask, run, sb, swy, swz, ry, rz);
    }
}

// the block of sub-bin `sub` (sx | sy << 8 | sz << 16) -> the shared subgrid, in
// conflict-free rounds of lanes
template <typename V, int G>
__device__ __forceinline__ void flush_block(V* tile, int sub, int PS, int P, int shift, int ry,
                                            int rz, V (&acc)[2][kBlk]) {
    const int sx = sub & 0xff, sy = (sub >> 8) & 0xff, sz = sub >> 16;
    NUFFT_CHECK(sz * G + rz + 4 < PS && sy * G + ry < PS / P && shift + sx * G + kBlk <= P);
    const bool flip = rz & 1;
    constexpr int R = Atom<V>::rounds;
#pragma unroll
    for (int round = 0; round < R; ++round) {
        if ((rz * R) / 4 == round) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                V* row = tile + (size_t)(sz * G + rz + 4 * r) * PS + (sy * G + ry) * P + shift +
                         sx * G;
#pragma unroll
                for (int k = 0; k < kBlk; ++k) Atom<V>::add(row + k, acc[r][k], flip);
            }
        }
        __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < kBlk; ++k) acc[r][k] = vzero<V>();
}

template <typename T, typename V, int W, int NW>
__global__ void __launch_bounds__(32 * NW, 1)
    spread_sub_kernel(Geom g, PtsView<T> p, const V* __restrict__ c, V* __restrict__ grid,
                      T beta) {
    using S = SubSmem<T, V, W, NW>;
    constexpr int G = S::G;
    constexpr int NT = 32 * NW;
    extern __shared__ __align__(16) unsigned char smem[];

    const int b = super_bin(g.nb, blockIdx.x);
    if (b < 0) return;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const TileX tx = tile_x<sizeof(V)>(bx, g.T[0], W);
    const int Ey = g.T[1] + W, Ez = g.T[2] + W;
    const int P = sub_pitch<sizeof(V)>(tx.len), PS = sub_plane<sizeof(V)>(P * Ey);
    double* tab = reinterpret_cast<double*>(smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* st = smem + kExpTab * sizeof(double) + warp * S::stage_bytes;
    V* sb = reinterpret_cast<V*>(st);           // [32][W]
    T* swy = reinterpret_cast<T*>(sb + 32 * W);  // [32][kYS]
    T* swz = swy + 32 * kYS;                     // [32][kYS]
    V* tile = reinterpret_cast<V*>(smem + S::fixed);

    {  // zero the subgrid, build the exp table
        float4* z4 = reinterpret_cast<float4*>(tile);
        const int n4 = (int)(((size_t)PS * Ez * sizeof(V)) / 16);
        for (int i = threadIdx.x; i < n4; i += NT) z4[i] = float4{0.f, 0.f, 0.f, 0.f};
        exp_tab_init(tab, threadIdx.x, NT);
    }
    __syncthreads();

    // this warp's share of the bin: a contiguous run of the (sub-bin sorted) points,
    // the bin split evenly over the warps (a sub-bin cut between two warps is
    // flushed by both: the flush is an atomic add)
    const uint32_t n = end - beg;
    const uint32_t wbeg = beg + (uint32_t)(((uint64_t)n * warp) / NW);
    const uint32_t wend = beg + (uint32_t)(((uint64_t)n * (warp + 1)) / NW);
    const int ry = lane & 7, rz = lane >> 3;  // this lane's rows: (ry, rz) and (ry, rz + 4)
    int cur = -1;  // sub-bin whose block the registers hold
    V acc[2][kBlk];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int k = 0; k < kBlk; ++k) acc[r][k] = vzero<V>();

    for (uint32_t c0 = wbeg; c0 < wend; c0 += 32) {
        const int np = (int)min(32u, wend - c0);
        int my_sub = -1, my_dx = -1;
        if (lane < np) {  // lane: weights of point c0 + lane
            const PtRec<T> rr = load_rec(&p.rec[c0 + lane]);
            const uint32_t la = rr.la;
            const int lx = (int)(la & 0xff), ly = (int)((la >> 8) & 0xff), lz = (int)(la >> 16);
            const int sx = lx / G, sy = ly / G, sz = lz / G;
            const int dy = ly - sy * G, dz = lz - sz * G;
            my_dx = lx - sx * G;
            NUFFT_CHECK(sx < g.ns[0] && sy < g.ns[1] && sz < g.ns[2] && dy + W <= kBlk &&
                        dz + W <= kBlk && my_dx + W <= kBlk);
            my_sub = sx | (sy << 8) | (sz << 16);
            const V cv = c[rr.perm];
            T wt[3][W];
            if (p.w) {  // precomputed at setpts (opts.precompute)
                const T* pw = p.w + (size_t)(c0 + lane) * (3 * W);
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int k = 0; k < W; ++k) wt[a][k] = pw[a * W + k];
            } else {
                const T dd[3] = {rr.d[0], rr.d[1], rr.d[2]};
                es_weights3<T, W>(dd, beta, tab, wt);
            }
            T* wyl = swy + lane * kYS;
            T* wzl = swz + lane * kYS;
#pragma unroll
            for (int k = 0; k < kBlk; ++k) {
                wyl[k] = (T)0;
                wzl[k] = (T)0;
            }
#pragma unroll
            for (int k = 0; k < W; ++k) {
                sb[lane * W + k] = vscale(cv, wt[0][k]);
                wyl[dy + k] = wt[1][k];
                wzl[dz + k] = wt[2][k];
            }
        }
        unsigned dmask[G];
#pragma unroll
        for (int d = 0; d < G; ++d) dmask[d] = __ballot_sync(0xffffffffu, my_dx == d);
        __syncwarp();
        // runs of equal sub-bin (contiguous: the points are sorted by sub-bin)
        for (int j = 0; j < np;) {
            const int sub = __shfl_sync(0xffffffffu, my_sub, j);
            if (sub != cur) {  // warp-uniform: a new sub-bin starts
                if (cur >= 0) flush_block<V, G>(tile, cur, PS, P, tx.shift, ry, rz, acc);
                cur = sub;
            }
            const unsigned run = __ballot_sync(0xffffffffu, my_sub == sub);
            run_points<V, T, W, G, 0, 2, kYS>(acc, dmask, run, sb, swy, swz, ry, rz);
            j += __popc(run);
        }
        __syncwarp();
    }
    if (cur >= 0) flush_block<V, G>(tile, cur, PS, P, tx.shift, ry, rz, acc);
    fence_proxy_async_smem();
    __syncthreads();
    // subgrid -> periodic fine grid (bulk reductions, one per row segment)
    const int oy = by * g.T[1] - W / 2, oz = bz * g.T[2] - W / 2;
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    int sg[2], ss[2], sn[2];
    const int nseg = row_segments(tx.gx0, tx.len, nfx, sg, ss, sn);
    for (int r = threadIdx.x; r < Ey * Ez; r += NT) {
        const int cz = r / Ey, cy = r - cz * Ey;
        const int gy = wrap1(oy + cy, nfy), gz = z_row(oz + cz, g);
        V* grow = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
        const V* trow = tile + (size_t)cz * PS + (size_t)cy * P;
        for (int k = 0; k < (gz < -g.hz_lo ? 0 : nseg); ++k)
            bulk_red_add(reinterpret_cast<T*>(grow + sg[k]), trow + ss[k],
                         (unsigned)(sn[k] * sizeof(V)));
    }
    bulk_commit();
    bulk_wait_read();  // the staged rows must outlive the bulk reads
}

// ---------------------------------------------------------------------------
// Variant with the block flushed straight to the fine grid in HBM/L2: no shared
// subgrid and no shared atomics.  On a sub-bin change the warp writes its 8 x 8
// register rows into a private shared-memory buffer and issues one bulk reduction
// (cp.reduce.async.bulk .add, UBLKRED) per block row -- the L2 performs the adds.
// Rows start 16-byte aligned in HBM: cells smaller than 16 bytes shift the row by
// the misalignment and zero-pad it (A = 16 / cell bytes).
template <typename T, typename V, int W, int NW>
struct SubgSmem {
    using SG = SubGeom<W>;
    static constexpr int A = sizeof(V) >= 16 ? 1 : 16 / (int)sizeof(V);
    // flush row pitch (cells): 16-byte aligned rows, consecutive rows in distinct banks
    static constexpr int FP = A == 1 ? kBlk + 1 : (A == 2 ? kBlk + 2 : kBlk + 4);
    // per warp: b = c wx [32][W] values | wy zero-padded [32][kYS] | wz zero-padded [32][ZS]
    static constexpr size_t stage_bytes =
        ((32 * W * sizeof(V) + 32 * (kYS + SG::ZS) * sizeof(T)) + 15) / 16 * 16;
    static constexpr size_t flush_bytes = (size_t)32 * FP * sizeof(V);  // one row per lane
    static constexpr size_t warp_bytes = stage_bytes + flush_bytes;
    static constexpr size_t bytes() { return kExpTab * sizeof(double) + NW * warp_bytes; }
};

// this lane's R block rows -> (one at a time) its row of the warp's flush buffer ->
// bulk reductions into the periodic fine grid (one or two segments per row)
template <typename T, typename V, int W, int NW>
__device__ __forceinline__ void flush_global(const Geom& g, V* grid, V* fb, int sub, int ox,
                                             int oy, int oz, int ry, int rz,
                                             V (&acc)[SubGeom<W>::R][kBlk]) {
    using S = SubgSmem<T, V, W, NW>;
    using SG = SubGeom<W>;
    constexpr int A = S::A, FP = S::FP;
    const int sx = sub & 0xff, sy = (sub >> 8) & 0xff, sz = sub >> 16;
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    const int gxw = wrap1(ox + sx * SG::GX, nfx);  // block x origin, wrapped
    const int shift = gxw & (A - 1);
    const int len = A == 1 ? kBlk : ((shift + kBlk + A - 1) / A) * A;
    int sg[2], ss[2], sn[2];
    const int nseg = row_segments(gxw - shift, len, nfx, sg, ss, sn);
    NUFFT_CHECK(shift + kBlk <= FP && sg[0] >= 0 && sg[nseg - 1] + sn[nseg - 1] <= nfx);
    const int gy = wrap1(oy + sy * SG::GY + ry, nfy);
    V* row = fb + (size_t)(rz * 8 + ry) * FP;
#pragma unroll
    for (int r = 0; r < SG::R; ++r) {
        bulk_wait_read();  // the bulk engine has read this lane's previous row
        if constexpr (A > 1) {
#pragma unroll
            for (int k = 0; k < FP; ++k) row[k] = vzero<V>();
        }
#pragma unroll
        for (int k = 0; k < kBlk; ++k) {
            if constexpr (A > 1)
                row[shift + k] = acc[r][k];
            else
                row[k] = acc[r][k];
            acc[r][k] = vzero<V>();
        }
        fence_proxy_async_smem();
        const int gz = z_row(oz + sz * SG::GZ + rz + 4 * r, g);
        if (gz >= -g.hz_lo) {  // beyond the halo-extended slab: no stencil
            V* grow = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
            for (int k = 0; k < nseg; ++k)
                bulk_red_add(reinterpret_cast<T*>(grow + sg[k]), row + ss[k],
                             (unsigned)(sn[k] * sizeof(V)));
        }
        bulk_commit();
    }
}

// R = 2 (w <= 6): 16 warps per SM at 128 registers; R = 3 (w = 7): 12 at 168
template <typename T, typename V, int W, int NW>
__global__ void __launch_bounds__(32 * NW, (SubGeom<W>::R == 2 ? 16 : 12) / NW)
    spread_subg_kernel(Geom g, PtsView<T> p, const V* __restrict__ c, V* __restrict__ grid,
                       T beta) {
    using S = SubgSmem<T, V, W, NW>;
    using SG = SubGeom<W>;
    constexpr int R = SG::R, GX = SG::GX, GY = SG::GY, GZ = SG::GZ, ZS = SG::ZS;
    constexpr int NT = 32 * NW;
    extern __shared__ __align__(16) unsigned char smem[];

    const int b = super_bin(g.nb, blockIdx.x);
    if (b < 0) return;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;
    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const int ox = bx * g.T[0] - W / 2, oy = by * g.T[1] - W / 2, oz = bz * g.T[2] - W / 2;
    double* tab = reinterpret_cast<double*>(smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* st = smem + kExpTab * sizeof(double) + warp * S::warp_bytes;
    V* sb = reinterpret_cast<V*>(st);                    // [32][W]
    T* swy = reinterpret_cast<T*>(sb + 32 * W);           // [32][kYS]
    T* swz = swy + 32 * kYS;                              // [32][ZS]
    V* fb = reinterpret_cast<V*>(st + S::stage_bytes);    // [32][FP]
    exp_tab_init(tab, threadIdx.x, NT);
    __syncthreads();

    const uint32_t n = end - beg;
    const uint32_t wbeg = beg + (uint32_t)(((uint64_t)n * warp) / NW);
    const uint32_t wend = beg + (uint32_t)(((uint64_t)n * (warp + 1)) / NW);
    const int ry = lane & 7, rz = lane >> 3;
    int cur = -1;
    V acc[R][kBlk];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < kBlk; ++k) acc[r][k] = vzero<V>();

    for (uint32_t c0 = wbeg; c0 < wend; c0 += 32) {
        const int np = (int)min(32u, wend - c0);
        int my_sub = -1, my_dx = -1;
        if (lane < np) {
            const PtRec<T> rr = load_rec(&p.rec[c0 + lane]);
            const uint32_t la = rr.la;
            const int lx = (int)(la & 0xff), ly = (int)((la >> 8) & 0xff), lz = (int)(la >> 16);
            const int sx = lx / GX, sy = ly / GY, sz = lz / GZ;
            const int dy = ly - sy * GY, dz = lz - sz * GZ;
            my_dx = lx - sx * GX;
            my_sub = sx | (sy << 8) | (sz << 16);
            NUFFT_CHECK(sx < g.ns[0] && sy < g.ns[1] && sz < g.ns[2] && dy + W <= kBlk &&
                        dz + W <= SG::BZ && my_dx + W <= kBlk);
            const V cv = c[rr.perm];
            T wt[3][W];
            if (p.w) {  // precomputed at setpts (opts.precompute)
                const T* pw = p.w + (size_t)(c0 + lane) * (3 * W);
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int k = 0; k < W; ++k) wt[a][k] = pw[a * W + k];
            } else {
                const T dd[3] = {rr.d[0], rr.d[1], rr.d[2]};
                es_weights3<T, W>(dd, beta, tab, wt);
            }
            T* wyl = swy + lane * kYS;
            T* wzl = swz + lane * ZS;
#pragma unroll
            for (int k = 0; k < kBlk; ++k) wyl[k] = (T)0;
#pragma unroll
            for (int k = 0; k < SG::BZ; ++k) wzl[k] = (T)0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                sb[lane * W + k] = vscale(cv, wt[0][k]);
                wyl[dy + k] = wt[1][k];
                wzl[dz + k] = wt[2][k];
            }
        }
        unsigned dmask[GX];
#pragma unroll
        for (int d = 0; d < GX; ++d) dmask[d] = __ballot_sync(0xffffffffu, my_dx == d);
        __syncwarp();
        for (int j = 0; j < np;) {
            const int sub = __shfl_sync(0xffffffffu, my_sub, j);
            if (sub != cur) {
                if (cur >= 0) flush_global<T, V, W, NW>(g, grid, fb, cur, ox, oy, oz, ry, rz, acc);
                cur = sub;
            }
            const unsigned run = __ballot_sync(0xffffffffu, my_sub == sub);
            run_points<V, T, W, GX, 0, R, ZS>(acc, dmask, run, sb, swy, swz, ry, rz);
            j += __popc(run);
        }
        __syncwarp();
    }
    if (cur >= 0) flush_global<T, V, W, NW>(g, grid, fb, cur, ox, oy, oz, ry, rz, acc);
    bulk_wait_read();  // the flush buffers must outlive the bulk reads
}

// warps per CTA: 16 (128 registers per thread, one CTA per SM) or 8 (up to 255);
// NUFFT_SUB_WARPS=8 selects the latter (measurement switch)
inline int sub_warps() {
    static const int nw = [] {
        const char* e = std::getenv("NUFFT_SUB_WARPS");
        return (e && std::atoi(e) == 8) ? 8 : 16;
    }();
    return nw;
}

template <typename T, typename V, int W, int NW>
size_t smem_nw(const Geom& g) {
    const int P = sub_pitch<sizeof(V)>(tile_len<sizeof(V)>(g.T[0], W));
    return SubSmem<T, V, W, NW>::bytes((size_t)sub_plane<sizeof(V)>(P * (g.T[1] + W)) *
                                       (g.T[2] + W));
}
template <typename T, typename V, int W>
size_t smem_w(const Geom& g) {
    if constexpr (W <= 6)  // the tile-flush variant exists for R = 2 only
        return std::max(SubgSmem<T, V, W, 4>::bytes(),
                        std::max(smem_nw<T, V, W, 8>(g), smem_nw<T, V, W, 16>(g)));
    else
        return SubgSmem<T, V, W, 4>::bytes();
}

template <typename T, typename V, int W, int NW>
cudaError_t launch_nw(const Geom& g, const PtsView<T>& p, int64_t nbins, const V* c, V* grid,
                      double beta, cudaStream_t s) {
    const size_t smem = smem_nw<T, V, W, NW>(g);
    auto kern = spread_sub_kernel<T, V, W, NW>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
    }
    if (nbins > 0) kern<<<(unsigned)super_ctas(g.nb), 32 * NW, smem, s>>>(g, p, c, grid, (T)beta);
    return cudaGetLastError();
}
// the block flush: straight to the fine grid (default; spread_subg_kernel) or
// NUFFT_SUB_TILE=1 through a shared subgrid of the bin with shared atomics
// (spread_sub_kernel, measured slower: C3e4 25.0 vs 18.5 ms) -- a measurement switch
inline bool sub_global() {
    static const bool on = [] {
        const char* e = std::getenv("NUFFT_SUB_TILE");
        return !(e && std::atoi(e) == 1);
    }();
    return on;
}

template <typename T, typename V, int W, int NW>
cudaError_t launch_g(const Geom& g, const PtsView<T>& p, int64_t nbins, const V* c, V* grid,
                     double beta, cudaStream_t s) {
    const size_t smem = SubgSmem<T, V, W, NW>::bytes();
    auto kern = spread_subg_kernel<T, V, W, NW>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
    }
    if (nbins > 0) kern<<<(unsigned)super_ctas(g.nb), 32 * NW, smem, s>>>(g, p, c, grid, (T)beta);
    return cudaGetLastError();
}

template <typename T, typename V, int W>
cudaError_t launch_w(const Geom& g, const PtsView<T>& p, int64_t nbins, const V* c, V* grid,
                     double beta, cudaStream_t s) {
    if constexpr (W <= 6) {
        if (!sub_global())
            return sub_warps() == 8 ? launch_nw<T, V, W, 8>(g, p, nbins, c, grid, beta, s)
                                    : launch_nw<T, V, W, 16>(g, p, nbins, c, grid, beta, s);
    }
    return launch_g<T, V, W, 4>(g, p, nbins, c, grid, beta, s);
}

template <typename T, typename V>
cudaError_t launch_v(const Geom& g, const PtsView<T>& p, int64_t nbins, const V* c, V* grid,
                     double beta, cudaStream_t s) {
    if (!spread_sub_applies(g)) return cudaErrorNotSupported;
    switch (g.w) {
        case 2: return launch_w<T, V, 2>(g, p, nbins, c, grid, beta, s);
        case 3: return launch_w<T, V, 3>(g, p, nbins, c, grid, beta, s);
        case 4: return launch_w<T, V, 4>(g, p, nbins, c, grid, beta, s);
        case 5: return launch_w<T, V, 5>(g, p, nbins, c, grid, beta, s);
        case 6: return launch_w<T, V, 6>(g, p, nbins, c, grid, beta, s);
        case 7: return launch_w<T, V, 7>(g, p, nbins, c, grid, beta, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace

bool spread_sub_applies(const Geom& g) {
    if (g.w < 2 || g.w > 7 || g.nsub <= 1) return false;
    int G[3];
    sub_extents(g.w, G);
    for (int d = 0; d < 3; ++d)
        if (g.Gs[d] != G[d] || g.ns[d] < 1 || g.ns[d] * G[d] != g.T[d] + 1) return false;
    return true;
}

template <typename T>
size_t spread_sub_smem_bytes(const Geom& g) {
    using C = typename Cx<T>::type;
    switch (g.w) {
        case 2: return smem_w<T, C, 2>(g);
        case 3: return smem_w<T, C, 3>(g);
        case 4: return smem_w<T, C, 4>(g);
        case 5: return smem_w<T, C, 5>(g);
        case 6: return smem_w<T, C, 6>(g);
        case 7: return smem_w<T, C, 7>(g);
        default: return 0;
    }
}

template <typename T>
cudaError_t launch_spread_sub(const Geom& g, const PtsView<T>& p, int64_t nbins,
                              const typename Cx<T>::type* c, typename Cx<T>::type* grid,
                              double beta, cudaStream_t s) {
    return launch_v<T, typename Cx<T>::type>(g, p, nbins, c, grid, beta, s);
}
template <typename T>
cudaError_t launch_spread_sub_real(const Geom& g, const PtsView<T>& p, int64_t nbins, const T* c,
                                   T* grid, double beta, cudaStream_t s) {
    return launch_v<T, T>(g, p, nbins, c, grid, beta, s);
}

template cudaError_t launch_spread_sub<float>(const Geom&, const PtsView<float>&, int64_t,
                                              const float2*, float2*, double, cudaStream_t);
template cudaError_t launch_spread_sub<double>(const Geom&, const PtsView<double>&, int64_t,
                                               const double2*, double2*, double, cudaStream_t);
template cudaError_t launch_spread_sub_real<float>(const Geom&, const PtsView<float>&, int64_t,
                                                   const float*, float*, double, cudaStream_t);
template cudaError_t launch_spread_sub_real<double>(const Geom&, const PtsView<double>&, int64_t,
                                                    const double*, double*, double, cudaStream_t);
template size_t spread_sub_smem_bytes<float>(const Geom&);
template size_t spread_sub_smem_bytes<double>(const Geom&);

}  // namespace nufft
