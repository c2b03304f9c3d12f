// interp_impl.cuh -- the interpolation operator C^T of Eq. (4).
//
// "Sorted interpolation" taken to its B200 form: one CTA per
// bin stages the bin's (T + w)^3 subgrid from the periodic fine grid into
// shared memory once, with the bulk-async (TMA) engine: one
// cp.async.bulk.shared::cta.global (SASS UBLKCP) per contiguous row segment,
// all completing on a single mbarrier transaction count; rows that cross the
// periodic boundary split into two segments.  Every point of the bin then
// gathers its w^3 stencil from shared memory, so each grid cell is read from
// HBM about ((T + w) / T)^3 times per transform instead of w^3 / (points per
// cell) times as in direct interpolation.
//
// Points are handled in chunks of 32 per warp (the bin split evenly over the
// warps): lane l loads point l's sorted record (coalesced) and evaluates its
// 3w ES weights in registers (separability; phi direct,
// PAPER.md:176), parking them in a per-warp shared buffer.  The warp then
// walks the 32 points: lane slots cover the w x w (x, y) columns of the
// stencil, each sums its w z-cells against wz, scales by wx*wy, and a shuffle
// reduction yields c_j, written in the caller's order (c[perm[slot]]).  The
// kernel is bound by shared-memory wavefronts (one 8- or 16-byte cell load per
// stencil cell), so the slot map is chosen for them: for w >= 6 a quarter-warp
// reads 8 consecutive cells of ONE row (x = lane % 8, y = lane / 8 + 4 pass),
// conflict-free for any row pitch; for w <= 5 the flat map over the w^2 columns
// wastes fewer lanes.
#pragma once

#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <type_traits>

#include "device_util.cuh"
#include "internal.cuh"
#include "sub_common.cuh"

namespace nufft {

namespace {

using namespace dev;

constexpr int kInterpThreads = 256;
constexpr int kInterpWarps = kInterpThreads / 32;

// V: value type of the grid and of the outputs, Cx<T> (complex) or T (real)
template <typename T, typename V, int W>
struct InterpSmem {
    using C = V;
    // per-point weight stride in elements, ODD: lane l stores its point's weights
    // at l * WS, so the 32 (fp32) / 16 (fp64 half-warp) lanes of a store hit
    // distinct banks (an even stride such as 16 at w = 5 serialises them 16-32 way)
    static constexpr int WS = (3 * W + 1) | 1;
    static size_t bytes(int ncell) {
        return (size_t)ncell * sizeof(C) + (size_t)kInterpWarps * 32 * WS * sizeof(T) + 16;
    }
};

// Grid values with NC real components: complex (2), real (1), or a real 3-vector
// (3: the three field components of the PIF gather, sharing one weight evaluation).
template <typename T> struct Vec3 { T c[3]; };
template <typename V> struct VT;
template <> struct VT<float2> {
    static constexpr int n = 2;
    __device__ static float get(const float2& v, int k) { return k ? v.y : v.x; }
    __device__ static float2 make(const float (&a)[2]) { return float2{a[0], a[1]}; }
};
template <> struct VT<double2> {
    static constexpr int n = 2;
    __device__ static double get(const double2& v, int k) { return k ? v.y : v.x; }
    __device__ static double2 make(const double (&a)[2]) { return double2{a[0], a[1]}; }
};
template <> struct VT<float> {
    static constexpr int n = 1;
    __device__ static float get(const float& v, int) { return v; }
    __device__ static float make(const float (&a)[1]) { return a[0]; }
};
template <> struct VT<double> {
    static constexpr int n = 1;
    __device__ static double get(const double& v, int) { return v; }
    __device__ static double make(const double (&a)[1]) { return a[0]; }
};
template <typename T> struct VT<Vec3<T>> {
    static constexpr int n = 3;
    __device__ static T get(const Vec3<T>& v, int k) { return v.c[k]; }
    __device__ static Vec3<T> make(const T (&a)[3]) { return Vec3<T>{{a[0], a[1], a[2]}}; }
};
// Grid / shared-memory layout per value type: one tile of V cells, or -- for the
// 3-vector -- three component grids (SoA, gstride reals apart in HBM) staged into
// three consecutive component tiles (cell = one real).
template <typename V> struct Layout {
    using Cell = V;
    static constexpr int comps = 1;
    __device__ static V load(const Cell* t, int o, int) { return t[o]; }
};
template <typename T> struct Layout<Vec3<T>> {
    using Cell = T;
    static constexpr int comps = 3;
    __device__ static Vec3<T> load(const T* t, int o, int nc) {
        return Vec3<T>{{t[o], t[o + nc], t[o + 2 * nc]}};
    }
};

// sv[m] = sum_k G[col + k plane].m wz[k] over the w planes of one stencil column;
// complex fp32 cells take one packed FFMA2 per cell (device_util.cuh vfma)
template <typename V, int W, typename T, int NC>
__device__ __forceinline__ void zsum(T (&sv)[NC], const typename Layout<V>::Cell* tile, int col,
                                     int plane, int ncell, const T (&wz)[W]) {
    if constexpr (std::is_same<V, float2>::value) {
        float2 a = float2{0.0f, 0.0f};
#pragma unroll
        for (int k = 0; k < W; ++k) vfma(a, tile[col + k * plane], wz[k]);
        sv[0] = a.x;
        sv[1] = a.y;
    } else {
#pragma unroll
        for (int m = 0; m < NC; ++m) sv[m] = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const V v = Layout<V>::load(tile, col + k * plane, ncell);
#pragma unroll
            for (int m = 0; m < NC; ++m) sv[m] += VT<V>::get(v, m) * wz[k];
        }
    }
}

// Output stage of the gather: store the value at the caller's index ...
template <typename V> struct StoreOut {
    V* out;
    template <typename T, int NC>
    __device__ void operator()(uint32_t pj, const T (&tot)[NC]) const { out[pj] = VT<V>::make(tot); }
};
// ... or, for the PIF field gather, fuse the leapfrog kick:
// v_d[pj] += s E_d(x_pj) for the three components (no field array in HBM)
template <typename T> struct KickOut {
    T* v0;
    T* v1;
    T* v2;
    T s;
    template <int NC>
    __device__ void operator()(uint32_t pj, const T (&tot)[NC]) const {
        static_assert(NC == 3, "a 3-component gather");
        v0[pj] += s * tot[0];
        v1[pj] += s * tot[1];
        v2[pj] += s * tot[2];
    }
};

// Four per-lane partial sums (points j0 .. j0 + 3) -> the total of point
// j0 + (lane & 16 ? 1 : 0) + (lane & 8 ? 2 : 0) on every lane: a transposing
// butterfly (offsets 16, 8 split the 4 sums over lane octets, 4, 2, 1 finish).
template <typename T>
__device__ __forceinline__ T reduce4(const T (&v)[4], int lane) {
    const bool h16 = lane & 16, h8 = lane & 8;
    T r0 = h16 ? v[1] : v[0], r1 = h16 ? v[3] : v[2];
    r0 += __shfl_xor_sync(0xffffffffu, h16 ? v[0] : v[1], 16);
    r1 += __shfl_xor_sync(0xffffffffu, h16 ? v[2] : v[3], 16);
    T rr = h8 ? r1 : r0;
    rr += __shfl_xor_sync(0xffffffffu, h8 ? r0 : r1, 8);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) rr += __shfl_xor_sync(0xffffffffu, rr, o);
    return rr;
}

template <typename T, typename V, int W, typename Out>
__global__ void __launch_bounds__(kInterpThreads, 2)
    interp_tile_kernel(Geom g, PtsView<T> p, const typename Layout<V>::Cell* __restrict__ grid,
                       int64_t gstride, Out out, T beta, const __grid_constant__ CUtensorMap tmap,
                       int use_tmap) {
    using C = V;
    using Cell = typename Layout<V>::Cell;
    constexpr int NCOMP = Layout<V>::comps;  // component tiles (3 for the SoA 3-vector)
    constexpr int NC = VT<V>::n;  // real components per value
    constexpr bool kFlat = W <= 5;
    constexpr int NQ = kFlat ? (W * W + 31) / 32 : 1;
    constexpr int XS = W <= 8 ? 8 : 16, YS = 32 / XS, NPASS = (W + YS - 1) / YS;
    constexpr int WS = InterpSmem<T, V, W>::WS;
    constexpr int NW = kInterpWarps;
    extern __shared__ __align__(1024) unsigned char smem[];  // TMA tensor destination

    const int b = blockIdx.x;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const TileX tx = tile_x<sizeof(Cell)>(bx, g.T[0], W);
    const int Ey = g.T[1] + W, Ez = g.T[2] + W;
    const int pitch = tx.pitch, plane = pitch * Ey, ncell = plane * Ez;
    Cell* tile = reinterpret_cast<Cell*>(smem);  // NCOMP tiles of ncell cells
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T* wb = reinterpret_cast<T*>(tile + NCOMP * ncell) + warp * 32 * WS;  // [32][WS] per warp
    uint64_t* bar = reinterpret_cast<uint64_t*>(
        (reinterpret_cast<uintptr_t>(reinterpret_cast<T*>(tile + NCOMP * ncell) + NW * 32 * WS) + 15) &
        ~(uintptr_t)15);

    // ---- stage the subgrid (one mbarrier transaction).  A bin whose subgrid lies
    // inside the grid (no periodic wrap) is ONE 3D TMA tensor copy of the whole box;
    // the others take one bulk copy per row segment, split at the periodic boundary.
    const int oy0 = by * g.T[1] - W / 2, oz0 = bz * g.T[2] - W / 2;
    const bool interior = use_tmap && tx.gx0 >= 0 && tx.gx0 + tx.len <= (int)g.nf[0] &&
                          oy0 >= 0 && oy0 + Ey <= (int)g.nf[1] && oz0 >= 0 &&
                          oz0 + Ez <= (int)g.nz_loc;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_arrive_expect_tx(bar, interior ? (unsigned)(Ez * Ey * pitch * sizeof(Cell))
                                            : (unsigned)(NCOMP * Ey * Ez * tx.len * sizeof(Cell)));
    }
    __syncthreads();
    if (interior) {
        if (threadIdx.x == 0) {
            constexpr int R = (int)(sizeof(Cell) / sizeof(T));  // map elements per cell
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(tile)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(tx.gx0 * R), "r"(oy0), "r"(oz0),
                "r"(smem_addr(bar))
                : "memory");
        }
    } else {
        const int oy = by * g.T[1] - W / 2, oz = bz * g.T[2] - W / 2;
        const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
        int sg[2], ss[2], sn[2];
        const int nseg = row_segments(tx.gx0, tx.len, nfx, sg, ss, sn);
        for (int r = threadIdx.x; r < Ey * Ez; r += kInterpThreads) {
            const int cz = r / Ey, cy = r - cz * Ey;
            int gz = z_row(oz + cz, g);
            // a row beyond the halo-extended slab is read by no stencil: stage any
            // valid row there (the transaction count stays one full subgrid)
            if (gz < -g.hz_lo) gz = 0;
            const int gy = wrap1(oy + cy, nfy);
#pragma unroll
            for (int cc = 0; cc < NCOMP; ++cc) {
                const Cell* grow = grid + cc * gstride + (int64_t)nfx * ((int64_t)gz * nfy + gy);
                Cell* trow = tile + cc * ncell + r * pitch;
                for (int k = 0; k < nseg; ++k)
                    bulk_g2s(trow + ss[k], grow + sg[k], (unsigned)(sn[k] * sizeof(Cell)), bar);
            }
        }
    }

    // lane slots.  w <= 5: flat slots s = lane + 32 q over the w x w columns
    // (x = s % w, y = s / w); w >= 6: x = lane % XS, y = lane / XS + YS * pass
    // (one 8-cell row per 128-bit quarter-warp phase: no bank conflicts)
    const int sx = lane % XS, sy0 = lane / XS;
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
    const uint32_t n = end - beg;
    const uint32_t wbeg = beg + (uint32_t)(((uint64_t)n * warp) / NW);
    const uint32_t wend = beg + (uint32_t)(((uint64_t)n * (warp + 1)) / NW);
    bool staged = false;

    for (uint32_t c0 = wbeg; c0 < wend; c0 += 32) {
        // ---- lane l: record + 3w weights of point c0 + l (overlaps the tile load)
        const uint32_t slot = c0 + lane;
        uint32_t my_perm = 0;
        int my_base = 0;
        if (slot < wend) {
            const PtRec<T> rr = load_rec(&p.rec[slot]);
            const T d3[3] = {rr.d[0], rr.d[1], rr.d[2]};
            const uint32_t la = rr.la;
            my_perm = rr.perm;
            my_base = (int)(((la >> 16) * Ey + ((la >> 8) & 0xff)) * pitch + (la & 0xff)) +
                      tx.shift;
            if (!p.w) {
                T* wl = wb + lane * WS;
#pragma unroll
                for (int d = 0; d < 3; ++d)
#pragma unroll
                    for (int k = 0; k < W; ++k)
                        wl[d * W + k] = es_weight<T>(((T)k - d3[d]) * two_over_w, beta);
            }
        }
        if (p.w) {  // precomputed at setpts: the chunk's rows are contiguous, copy coalesced
            const T* src = p.w + (size_t)c0 * (3 * W);
            const int ne = (int)min(32u, wend - c0) * (3 * W);
            for (int e = lane; e < ne; e += 32) {
                const int j = e / (3 * W);
                wb[j * WS + (e - j * (3 * W))] = src[e];
            }
        }
        if (!staged) {
            mbar_wait(bar, 0);
            staged = true;
        }
        __syncwarp();
        const int np = (int)min(32u, wend - c0);
        // four points at a time: independent accumulations, then a transposing
        // butterfly (offsets 16, 8 split the 4 sums over lane octets, 4, 2, 1 finish)
        for (int j0 = 0; j0 < np; j0 += 4) {
            T acc[NC][4];
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) {
                const int j = j0 + g4;
#pragma unroll
                for (int q = 0; q < NC; ++q) acc[q][g4] = 0;
                if (j < np) {
                    const int base = __shfl_sync(0xffffffffu, my_base, j);
                    const T* wj = wb + j * WS;
                    T wz[W];
#pragma unroll
                    for (int k = 0; k < W; ++k) wz[k] = wj[2 * W + k];
                    if constexpr (kFlat) {
#pragma unroll
                        for (int q = 0; q < NQ; ++q) {
                            if (qok[q]) {
                                const int col = base + qoff[q];
                                T sv[NC];
                                zsum<C, W>(sv, tile, col, plane, ncell, wz);
                                const T wxy = wj[qx[q]] * wj[W + qy[q]];
#pragma unroll
                                for (int m = 0; m < NC; ++m) acc[m][g4] += sv[m] * wxy;
                            }
                        }
                    } else {
                        const int col0 = base + sx;
#pragma unroll
                        for (int ps = 0; ps < NPASS; ++ps) {
                            const int y = sy0 + YS * ps;
                            if (sx < W && y < W) {
                                const int col = col0 + y * pitch;
                                T sv[NC];
                                zsum<C, W>(sv, tile, col, plane, ncell, wz);
                                const T wy = wj[W + y];
#pragma unroll
                                for (int m = 0; m < NC; ++m) acc[m][g4] += sv[m] * wy;
                            }
                        }
                        const T wx = sx < W ? wj[sx] : (T)0;
#pragma unroll
                        for (int m = 0; m < NC; ++m) acc[m][g4] *= wx;
                    }
                }
            }
            T tot[NC];
#pragma unroll
            for (int m = 0; m < NC; ++m) tot[m] = reduce4<T>(acc[m], lane);
            const int j = j0 + ((lane & 16) ? 1 : 0) + ((lane & 8) ? 2 : 0);
            const uint32_t pj = __shfl_sync(0xffffffffu, my_perm, j & 31);
            if ((lane & 7) == 0 && j < np) out(pj, tot);
        }
        __syncwarp();
    }
    // a warp without points must not exit before the bulk copies into this CTA's
    // shared memory have landed
    if (!staged) mbar_wait(bar, 0);
}

// ---------------------------------------------------------------------------
// Sub-bin interpolation (plans with Geom::nsub > 1, w <= 6): the mirror of
// spread_sub.cu.  The bin's (T + w)^3 subgrid is staged once (TMA / bulk rows, as
// above); each warp walks a contiguous run of the bin's sub-bin sorted points and
// keeps the 8 x 8 x 8 cell block of the current sub-bin in REGISTERS (lane l: the
// x-rows (y = l & 7, z = l >> 3) and (y, z + 4), reloaded from shared memory only
// when the sub-bin changes).  Per point the x sum is exact -- a warp-uniform branch
// on the point's x base picks w fixed registers per row -- then each lane weights
// its two row sums by wy wz (zero outside the stencil) and a transposing butterfly
// over 4 points sums the 32 lanes.  Shared memory carries only the block reloads
// and broadcast weights, not the w^3 cells of every point (the bound of the
// per-point gather above).
template <typename T, typename V, int W, int NW>
struct InterpSubSmem {
    using Cell = typename Layout<V>::Cell;
    // per warp: wx [32][W] | wy, wz zero-padded [32][kYS] | perm [32]
    static constexpr size_t stage_bytes =
        ((32 * W + 2 * 32 * kYS) * sizeof(T) + 32 * sizeof(int) + 15) / 16 * 16;
    static constexpr size_t fixed = kExpTab * sizeof(double) + NW * stage_bytes + 16;
    static size_t bytes(size_t ncell) {
        return fixed + (size_t)Layout<V>::comps * ncell * sizeof(Cell);
    }
};

template <typename Cell> struct CellGet;
template <> struct CellGet<double2> {
    __device__ static double get(const double2& v, int m) { return m ? v.y : v.x; }
};
template <> struct CellGet<float2> {
    __device__ static float get(const float2& v, int m) { return m ? v.y : v.x; }
};
template <> struct CellGet<double> {
    __device__ static double get(const double& v, int) { return v; }
};
template <> struct CellGet<float> {
    __device__ static float get(const float& v, int) { return v; }
};

// val[m] = sum_r f_r sum_k blk[q(m)][r][D + k] wx[k] for the x base D (warp-uniform)
template <typename T, typename Cell, int NCOMP, int NC, int W, int D, int R>
__device__ __forceinline__ void row_sums(const Cell (&blk)[NCOMP][R][kBlk], const T* wx,
                                         const T (&f)[R], T (&val)[NC]) {
#pragma unroll
    for (int m = 0; m < NC; ++m) {
        const int q = NCOMP == 1 ? 0 : m, cm = NCOMP == 1 ? m : 0;
        T v = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            T sr = 0;
#pragma unroll
            for (int k = 0; k < W; ++k) sr = fma(CellGet<Cell>::get(blk[q][r][D + k], cm), wx[k], sr);
            v = fma(sr, f[r], v);
        }
        val[m] = v;
    }
}

template <typename T, typename Cell, int NCOMP, int NC, int W, int G, int D, typename Out>
__device__ __forceinline__ void run_gather(const Cell (&blk)[NCOMP][2][kBlk],
                                           const unsigned (&dmask)[G], unsigned run, const T* swx,
                                           const T* swy, const T* swz, const uint32_t* sperm,
                                           int lane, int ry, int rz, const Out& out) {
    if constexpr (D < G) {
        unsigned msk = dmask[D] & run;
        while (msk) {
            int jj[4];
            T acc[NC][4];
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) {
                jj[g4] = msk ? __ffs(msk) - 1 : -1;
                msk &= msk - 1;
#pragma unroll
                for (int m = 0; m < NC; ++m) acc[m][g4] = 0;
                if (jj[g4] >= 0) {
                    const int j = jj[g4];
                    const T wyv = swy[j * kYS + ry];
                    const T f[2] = {wyv * swz[j * kYS + rz], wyv * swz[j * kYS + rz + 4]};
                    T val[NC];
                    row_sums<T, Cell, NCOMP, NC, W, D, 2>(blk, swx + j * W, f, val);
#pragma unroll
                    for (int m = 0; m < NC; ++m) acc[m][g4] = val[m];
                }
            }
            T tot[NC];
#pragma unroll
            for (int m = 0; m < NC; ++m) tot[m] = reduce4<T>(acc[m], lane);
            const int sel = ((lane & 16) ? 1 : 0) + ((lane & 8) ? 2 : 0);  // reduce4's point
            const int j = sel == 0 ? jj[0] : sel == 1 ? jj[1] : sel == 2 ? jj[2] : jj[3];
            if ((lane & 7) == 0 && j >= 0) out(sperm[j], tot);
        }
        run_gather<T, Cell, NCOMP, NC, W, G, D + 1, Out>(blk, dmask, run, swx, swy, swz, sperm,
                                                         lane, ry, rz, out);
    }
}

template <typename T, typename V, int W, int NW, typename Out>
__global__ void __launch_bounds__(32 * NW, 1)
    interp_sub_kernel(Geom g, PtsView<T> p, const typename Layout<V>::Cell* __restrict__ grid,
                      int64_t gstride, Out out, T beta, const __grid_constant__ CUtensorMap tmap,
                      int use_tmap) {
    using S = InterpSubSmem<T, V, W, NW>;
    using Cell = typename Layout<V>::Cell;
    constexpr int NCOMP = Layout<V>::comps;
    constexpr int NC = VT<V>::n;
    constexpr int G = kBlk + 1 - W;
    constexpr int NT = 32 * NW;
    extern __shared__ __align__(1024) unsigned char smem[];  // TMA tensor destination

    const int b = super_bin(g.nb, blockIdx.x);
    if (b < 0) return;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const TileX tx = tile_x<sizeof(Cell)>(bx, g.T[0], W);
    const int P = sub_pitch<sizeof(Cell)>(tx.len), Ey = g.T[1] + W, Ez = g.T[2] + W;
    const int PS = P * Ey;  // plane stride of the TMA box
    const int ncell = PS * Ez;
    Cell* tile = reinterpret_cast<Cell*>(smem);  // NCOMP tiles of ncell cells
    unsigned char* after = smem + ((size_t)NCOMP * ncell * sizeof(Cell) + 15) / 16 * 16;
    double* tab = reinterpret_cast<double*>(after);
    uint64_t* bar = reinterpret_cast<uint64_t*>(tab + kExpTab);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* st = after + kExpTab * sizeof(double) + 16 + warp * S::stage_bytes;
    T* swx = reinterpret_cast<T*>(st);                     // [32][W]
    T* swy = swx + 32 * W;                                 // [32][kYS]
    T* swz = swy + 32 * kYS;                               // [32][kYS]
    uint32_t* sperm = reinterpret_cast<uint32_t*>(swz + 32 * kYS);  // [32]

    // ---- stage the subgrid on one mbarrier (TMA box for interior bins, else rows)
    const int oy0 = by * g.T[1] - W / 2, oz0 = bz * g.T[2] - W / 2;
    const bool interior = use_tmap && tx.gx0 >= 0 && tx.gx0 + tx.len <= (int)g.nf[0] && oy0 >= 0 &&
                          oy0 + Ey <= (int)g.nf[1] && oz0 >= 0 && oz0 + Ez <= (int)g.nz_loc;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_arrive_expect_tx(bar, interior ? (unsigned)(Ez * Ey * P * sizeof(Cell))
                                            : (unsigned)(NCOMP * Ey * Ez * tx.len * sizeof(Cell)));
    }
    exp_tab_init(tab, threadIdx.x, NT);
    __syncthreads();
    if (interior) {
        if (threadIdx.x == 0) {
            constexpr int R = (int)(sizeof(Cell) / sizeof(T));
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(tile)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(tx.gx0 * R), "r"(oy0), "r"(oz0),
                "r"(smem_addr(bar))
                : "memory");
        }
    } else {
        const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
        int sg[2], ss[2], sn[2];
        const int nseg = row_segments(tx.gx0, tx.len, nfx, sg, ss, sn);
        for (int r = threadIdx.x; r < Ey * Ez; r += NT) {
            const int cz = r / Ey, cy = r - cz * Ey;
            int gz = z_row(oz0 + cz, g);
            if (gz < -g.hz_lo) gz = 0;  // read by no stencil: any valid row
            const int gy = wrap1(oy0 + cy, nfy);
#pragma unroll
            for (int cc = 0; cc < NCOMP; ++cc) {
                const Cell* grow = grid + cc * gstride + (int64_t)nfx * ((int64_t)gz * nfy + gy);
                Cell* trow = tile + cc * ncell + r * P;
                for (int k = 0; k < nseg; ++k)
                    bulk_g2s(trow + ss[k], grow + sg[k], (unsigned)(sn[k] * sizeof(Cell)), bar);
            }
        }
    }

    const uint32_t n = end - beg;
    const uint32_t wbeg = beg + (uint32_t)(((uint64_t)n * warp) / NW);
    const uint32_t wend = beg + (uint32_t)(((uint64_t)n * (warp + 1)) / NW);
    const int ry = lane & 7, rz = lane >> 3;
    int cur = -1;
    bool staged = false;
    Cell blk[NCOMP][2][kBlk];

    for (uint32_t c0 = wbeg; c0 < wend; c0 += 32) {
        const int np = (int)min(32u, wend - c0);
        int my_sub = -1, my_dx = -1;
        if (lane < np) {  // lane: weights of point c0 + lane (overlaps the staging)
            const PtRec<T> rr = load_rec(&p.rec[c0 + lane]);
            const uint32_t la = rr.la;
            const int lx = (int)(la & 0xff), ly = (int)((la >> 8) & 0xff), lz = (int)(la >> 16);
            const int sx = lx / G, sy = ly / G, sz = lz / G;
            const int dy = ly - sy * G, dz = lz - sz * G;
            my_dx = lx - sx * G;
            NUFFT_CHECK(dy + W <= kBlk && dz + W <= kBlk && my_dx + W <= kBlk &&
                        sz * G + kBlk <= Ez && sy * G + kBlk <= Ey);
            my_sub = sx | (sy << 8) | (sz << 16);
            T wt[3][W];
            if (p.w) {
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
                swx[lane * W + k] = wt[0][k];
                wyl[dy + k] = wt[1][k];
                wzl[dz + k] = wt[2][k];
            }
            sperm[lane] = rr.perm;
        }
        unsigned dmask[G];
#pragma unroll
        for (int d = 0; d < G; ++d) dmask[d] = __ballot_sync(0xffffffffu, my_dx == d);
        if (!staged) {
            mbar_wait(bar, 0);
            staged = true;
        }
        __syncwarp();
        for (int j = 0; j < np;) {
            const int sub = __shfl_sync(0xffffffffu, my_sub, j);
            if (sub != cur) {  // warp-uniform: load the new sub-bin's block
                cur = sub;
                const int sx = sub & 0xff, sy = (sub >> 8) & 0xff, sz = sub >> 16;
#pragma unroll
                for (int q = 0; q < NCOMP; ++q)
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const Cell* row = tile + q * ncell + (sz * G + rz + 4 * r) * PS +
                                          (sy * G + ry) * P + tx.shift + sx * G;
#pragma unroll
                        NUFFT_CHECK(tx.shift + sx * G + kBlk <= P &&
                                    (sz * G + rz + 4 * r) * PS + (sy * G + ry) * P < ncell);
                        for (int k = 0; k < kBlk; ++k) blk[q][r][k] = row[k];
                    }
            }
            const unsigned run = __ballot_sync(0xffffffffu, my_sub == sub);
            run_gather<T, Cell, NCOMP, NC, W, G, 0, Out>(blk, dmask, run, swx, swy, swz, sperm,
                                                         lane, ry, rz, out);
            j += __popc(run);
        }
        __syncwarp();
    }
    if (!staged) mbar_wait(bar, 0);  // the bulk copies must land before the CTA exits
}

template <typename T, typename V, int W, int NW>
size_t sub_smem_nw(const Geom& g) {
    using Cell = typename Layout<V>::Cell;
    const int P = sub_pitch<sizeof(Cell)>(tile_len<sizeof(Cell)>(g.T[0], W));
    return InterpSubSmem<T, V, W, NW>::bytes((size_t)P * (g.T[1] + W) * (g.T[2] + W));
}

// ---------------------------------------------------------------------------
// Sub-bin interpolation WITHOUT a staged subgrid (the default for sub-bin plans):
// each warp loads the current sub-bin's 8^3 block straight from the fine grid in
// HBM / L2 into registers (2 rows x 8 cells per lane, periodic wrap per cell) --
// no (T + w)^3 shared tile, so 16 warps per SM at 128 registers -- and the lanes'
// partial sums go through a small shared buffer instead of a shuffle butterfly:
// every point's 32 lane partials are stored in one slot of red[8][32] (swizzled,
// conflict-free both ways) and every 8 points lane l sums 8 partials of slot l / 4,
// two xor-shuffles finish the slot.  ~5 instructions of reduction per point instead
// of ~20.
template <typename T, typename V, int W, int NW>
struct InterpSubgSmem {
    static constexpr int NC = VT<V>::n;
    // per warp: wx [32][W] | wy, wz zero-padded [32][kYS] | perm [32] | slot point [8] |
    // red [8][32][NC]
    static constexpr size_t stage_bytes =
        ((32 * W + 32 * (kYS + SubGeom<W>::ZS)) * sizeof(T) + 32 * sizeof(int) +
         8 * sizeof(int) + 15) / 16 * 16;
    static constexpr size_t red_bytes = (8 * 32 * NC * sizeof(T) + 15) / 16 * 16;
    static constexpr size_t warp_bytes = stage_bytes + red_bytes;
    static constexpr size_t bytes() { return kExpTab * sizeof(double) + NW * warp_bytes; }
};

// column of lane k's partial in slot j: a bijection in k; conflict-free for the
// stores (slot j, lanes 8q .. 8q + 7) and for the reads (lanes 4 js + q, k = 8 q + i)
__device__ __forceinline__ int red_col(int j, int k) {
    return (k & ~7) | ((k & 7) ^ ((2 * (k >> 3) + (j & 1)) & 7));
}

// sum the n (<= 8) filled slots and hand each total to the output stage
template <typename T, int NC, typename Out>
__device__ __forceinline__ void reduce_slots(const T* red, const int* sj, const uint32_t* sperm,
                                             int n, int lane, const Out& out) {
    const int js = lane >> 2, q = lane & 3;
    T tot[NC];
#pragma unroll
    for (int m = 0; m < NC; ++m) tot[m] = 0;
    if (js < n) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const T* e = red + (size_t)(js * 32 + red_col(js, 8 * q + i)) * NC;
#pragma unroll
            for (int m = 0; m < NC; ++m) tot[m] += e[m];
        }
    }
#pragma unroll
    for (int m = 0; m < NC; ++m) {
        tot[m] += __shfl_xor_sync(0xffffffffu, tot[m], 1);
        tot[m] += __shfl_xor_sync(0xffffffffu, tot[m], 2);
    }
    if (q == 0 && js < n) out(sperm[sj[js]], tot);
}

template <typename T, typename Cell, int NCOMP, int NC, int W, int GX, int D, int R, int ZS,
          typename Out>
__device__ __forceinline__ void run_gather_slots(const Cell (&blk)[NCOMP][R][kBlk],
                                                 const unsigned (&dmask)[GX], unsigned run,
                                                 const T* swx, const T* swy, const T* swz,
                                                 const uint32_t* sperm, T* red, int* sj, int& cnt,
                                                 int lane, int ry, int rz, int cole, int colo,
                                                 const Out& out) {
    if constexpr (D < GX) {
        unsigned msk = dmask[D] & run;
        // two points per step: both points' shared loads and row-sum chains are
        // independent, so their latencies overlap (the second slot repeats the first
        // point when the group has an odd count, and is not stored)
        while (msk) {
            const int j0 = __ffs(msk) - 1;
            msk &= msk - 1;
            const bool two = msk != 0;
            const int j1 = two ? __ffs(msk) - 1 : j0;
            msk &= msk - 1;
            const T wy0 = swy[j0 * kYS + ry], wy1 = swy[j1 * kYS + ry];
            T f0[R], f1[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                f0[r] = wy0 * swz[j0 * ZS + rz + 4 * r];
                f1[r] = wy1 * swz[j1 * ZS + rz + 4 * r];
            }
            T v0[NC], v1[NC];
            row_sums<T, Cell, NCOMP, NC, W, D, R>(blk, swx + j0 * W, f0, v0);
            row_sums<T, Cell, NCOMP, NC, W, D, R>(blk, swx + j1 * W, f1, v1);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (u == 1 && !two) break;
                // red_col(cnt, lane) depends on cnt only through its parity
                T* e = red + (size_t)(cnt * 32 + ((cnt & 1) ? colo : cole)) * NC;
#pragma unroll
                for (int m = 0; m < NC; ++m) e[m] = u ? v1[m] : v0[m];
                if (lane == 0) sj[cnt] = u ? j1 : j0;
                if (++cnt == 8) {
                    __syncwarp();
                    reduce_slots<T, NC>(red, sj, sperm, 8, lane, out);
                    cnt = 0;
                    __syncwarp();
                }
            }
        }
        run_gather_slots<T, Cell, NCOMP, NC, W, GX, D + 1, R, ZS, Out>(
            blk, dmask, run, swx, swy, swz, sperm, red, sj, cnt, lane, ry, rz, cole, colo, out);
    }
}

// MINW resident warps per SM: 16 (128 registers) for one-block fields, 8 for the
// three component blocks of the PIF field gather
template <typename T, typename V, int W, int NW, int MINW, typename Out>
__global__ void __launch_bounds__(32 * NW, (SubGeom<W>::R == 2 ? MINW : (MINW * 3) / 4) / NW)
    interp_subg_kernel(Geom g, PtsView<T> p, const typename Layout<V>::Cell* __restrict__ grid,
                       int64_t gstride, Out out, T beta) {
    using S = InterpSubgSmem<T, V, W, NW>;
    using Cell = typename Layout<V>::Cell;
    constexpr int NCOMP = Layout<V>::comps;
    constexpr int NC = VT<V>::n;
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
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    double* tab = reinterpret_cast<double*>(smem);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* st = smem + kExpTab * sizeof(double) + warp * S::warp_bytes;
    T* swx = reinterpret_cast<T*>(st);                                // [32][W]
    T* swy = swx + 32 * W;                                            // [32][kYS]
    T* swz = swy + 32 * kYS;                                          // [32][ZS]
    uint32_t* sperm = reinterpret_cast<uint32_t*>(swz + 32 * ZS);     // [32]
    int* sj = reinterpret_cast<int*>(sperm + 32);                     // [8]
    T* red = reinterpret_cast<T*>(st + S::stage_bytes);               // [8][32][NC]
    exp_tab_init(tab, threadIdx.x, NT);
    __syncthreads();

    const uint32_t n = end - beg;
    const uint32_t wbeg = beg + (uint32_t)(((uint64_t)n * warp) / NW);
    const uint32_t wend = beg + (uint32_t)(((uint64_t)n * (warp + 1)) / NW);
    const int ry = lane & 7, rz = lane >> 3;
    const int cole = red_col(0, lane), colo = red_col(1, lane);
    int cur = -1, cnt = 0;
    Cell blk[NCOMP][R][kBlk];

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
            NUFFT_CHECK(dy + W <= kBlk && dz + W <= SG::BZ && my_dx + W <= kBlk);
            T wt[3][W];
            if (p.w) {
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
                swx[lane * W + k] = wt[0][k];
                wyl[dy + k] = wt[1][k];
                wzl[dz + k] = wt[2][k];
            }
            sperm[lane] = rr.perm;
        }
        unsigned dmask[GX];
#pragma unroll
        for (int d = 0; d < GX; ++d) dmask[d] = __ballot_sync(0xffffffffu, my_dx == d);
        __syncwarp();
        for (int j = 0; j < np;) {
            const int sub = __shfl_sync(0xffffffffu, my_sub, j);
            if (sub != cur) {  // warp-uniform: the new sub-bin's block from the fine grid
                cur = sub;
                const int sx = sub & 0xff, sy = (sub >> 8) & 0xff, sz = sub >> 16;
                const int gy = wrap1(oy + sy * GY + ry, nfy);
                int gx[kBlk];
#pragma unroll
                for (int k = 0; k < kBlk; ++k) gx[k] = wrap1(ox + sx * GX + k, nfx);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int gz = z_row(oz + sz * GZ + rz + 4 * r, g);
                    const bool ok = gz >= -g.hz_lo;  // beyond the halo-extended slab: unused
#pragma unroll
                    for (int q = 0; q < NCOMP; ++q) {
                        const Cell* row =
                            grid + q * gstride + (int64_t)nfx * ((int64_t)(ok ? gz : 0) * nfy + gy);
#pragma unroll
                        for (int k = 0; k < kBlk; ++k) blk[q][r][k] = row[gx[k]];
                    }
                }
            }
            const unsigned run = __ballot_sync(0xffffffffu, my_sub == sub);
            run_gather_slots<T, Cell, NCOMP, NC, W, GX, 0, R, ZS, Out>(
                blk, dmask, run, swx, swy, swz, sperm, red, sj, cnt, lane, ry, rz, cole, colo, out);
            j += __popc(run);
        }
        if (cnt) {  // the batch's last, partial group of slots (sperm is per batch)
            __syncwarp();
            reduce_slots<T, NC>(red, sj, sperm, cnt, lane, out);
            cnt = 0;
        }
        __syncwarp();
    }
}

template <typename T, typename V, int W, int NW, int MINW, typename Out>
cudaError_t launch_subg(const Geom& g, const PtsView<T>& p, const typename Layout<V>::Cell* grid,
                        Out c, double beta, cudaStream_t s, int64_t gstride) {
    const size_t smem = InterpSubgSmem<T, V, W, NW>::bytes();
    auto kern = interp_subg_kernel<T, V, W, NW, MINW, Out>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
    }
    kern<<<(unsigned)super_ctas(g.nb), 32 * NW, smem, s>>>(g, p, grid, gstride, c, (T)beta);
    return cudaGetLastError();
}

// the staged-subgrid variant (interp_sub_kernel) instead: NUFFT_SUB_TILE=1
inline bool interp_sub_tile() {
    static const bool on = [] {
        const char* e = std::getenv("NUFFT_SUB_TILE");
        return e && std::atoi(e) == 1;
    }();
    return on;
}

inline int interp_sub_warps() {
    static const int nw = [] {
        const char* e = std::getenv("NUFFT_SUB_WARPS");
        return (e && std::atoi(e) == 8) ? 8 : 16;
    }();
    return nw;
}

template <typename T, typename V, int W, int NW, typename Out>
cudaError_t launch_sub_nw(const Geom& g, const PtsView<T>& p, int64_t nbins,
                          const typename Layout<V>::Cell* grid, Out c, double beta, cudaStream_t s,
                          int64_t gstride, const void* tmap) {
    const size_t smem = sub_smem_nw<T, V, W, NW>(g);
    auto kern = interp_sub_kernel<T, V, W, NW, Out>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
    }
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (tmap) std::memcpy(&map, tmap, sizeof(map));
    if (nbins > 0)
        kern<<<(unsigned)super_ctas(g.nb), 32 * NW, smem, s>>>(g, p, grid, gstride, c, (T)beta, map,
                                                    tmap ? 1 : 0);
    return cudaGetLastError();
}

template <typename T, typename V, int W>
size_t smem_w(const Geom& g) {
    using Cell = typename Layout<V>::Cell;
    if constexpr (W <= 6) {
        if (g.nsub > 1)
            return Layout<V>::comps == 3 ? sub_smem_nw<T, V, W, 8>(g)
                                         : std::max(sub_smem_nw<T, V, W, 8>(g),
                                                    sub_smem_nw<T, V, W, 16>(g));
    }
    return InterpSmem<T, V, W>::bytes(tile_pitch<sizeof(Cell)>(g.T[0], W) * (g.T[1] + W) *
                                      (g.T[2] + W));
}

template <typename T, typename V, int W, typename Out = StoreOut<V>>
cudaError_t launch_w(const Geom& g, const PtsView<T>& p, int64_t nbins,
                     const typename Layout<V>::Cell* grid, Out c, double beta, cudaStream_t s,
                     int64_t gstride = 0, const void* tmap = nullptr) {
    if constexpr (W <= 7) {  // plans sorted by sub-bin: the register-block gather
        if (g.nsub > 1) {
            if constexpr (W <= 6) {  // NUFFT_SUB_TILE=1: the staged-subgrid variant
                if (interp_sub_tile()) {
                    if constexpr (Layout<V>::comps == 3)
                        return launch_sub_nw<T, V, W, 8, Out>(g, p, nbins, grid, c, beta, s,
                                                              gstride, tmap);
                    else
                        return interp_sub_warps() == 8
                                   ? launch_sub_nw<T, V, W, 8, Out>(g, p, nbins, grid, c, beta, s,
                                                                    gstride, tmap)
                                   : launch_sub_nw<T, V, W, 16, Out>(g, p, nbins, grid, c, beta,
                                                                     s, gstride, tmap);
                }
            }
            // default: blocks straight from the fine grid
            if constexpr (Layout<V>::comps == 3)
                return launch_subg<T, V, W, 4, 8, Out>(g, p, grid, c, beta, s, gstride);
            else
                return launch_subg<T, V, W, 4, 16, Out>(g, p, grid, c, beta, s, gstride);
        }
    }
    const size_t smem = smem_w<T, V, W>(g);
    auto kern = interp_tile_kernel<T, V, W, Out>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
    }
    CUtensorMap map;
    std::memset(&map, 0, sizeof(map));
    if (tmap) std::memcpy(&map, tmap, sizeof(map));
    if (nbins > 0)
        kern<<<(unsigned)nbins, kInterpThreads, smem, s>>>(g, p, grid, gstride, c, (T)beta, map,
                                                           tmap ? 1 : 0);
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


}  // namespace nufft
