// sub_common.cuh -- shared by the sub-bin kernels (spread_sub.cu, interp.cu's
// interp_sub_kernel): the 8-cell register block geometry, the subgrid row pitch and
// the ES window evaluated branch-free with a table-assisted exp (3w weights per
// point per call).
#pragma once

#include "device_util.cuh"

namespace nufft {
namespace dev {

constexpr int kBlk = 8;  // register block edge in x and y: G + w - 1 cells (G = 9 - w)
constexpr int kYS = 9;   // staging stride of a zero-padded 8-row profile (odd: conflict-free)

// Register block of the sub-bin kernels per width: lane l owns the x-rows (y = l & 7,
// z = (l >> 3) + 4 r), r < R, of an 8 (x) x 8 (y) x 4R (z) cell block; a sub-bin is
// the G = block - w + 1 stencil bases per axis whose stencils fit the block.  R = 2
// for w <= 6 (G = 9 - w per axis), R = 3 for w = 7 (G = 2, 2, 6: 24 bases per
// sub-bin instead of 8, so a block is flushed / reloaded every ~24 points).
template <int W> struct SubGeom {
    static constexpr int R = W <= 6 ? 2 : 3;
    static constexpr int BZ = 4 * R;
    static constexpr int GX = kBlk + 1 - W, GY = kBlk + 1 - W, GZ = BZ + 1 - W;
    static constexpr int ZS = BZ + 1;  // staging stride of the zero-padded z profile (odd)
};

// shared-memory row pitch of a sub-bin kernel's subgrid (cells): rows start 16-byte
// aligned (bulk copies / reductions) and the 8 block rows of a quarter- / half-warp
// fall in different banks -- odd for 16-byte cells, 2 mod 4 for 8-byte, 4 mod 8 for
// 4-byte cells
template <int CB>
__host__ __device__ __forceinline__ int sub_pitch(int len) {
    if (CB >= 16) return len | 1;
    if (CB == 8) {
        const int q = (len + 1) & ~1;
        return (q & 3) == 2 ? q : q + 2;
    }
    const int q = (len + 3) & ~3;
    return (q & 7) == 4 ? q : q + 4;
}
// Super-tiled CTA order of the sub-bin kernels: consecutive CTAs walk 8 x 8 x 8
// blocks of bins (x fastest inside a block, then the blocks row-major), so the bins
// resident at once form a compact region whose overlapping halos meet in L2 (the
// row-major order puts the z-neighbour of a bin nb0 x nb1 bins later).  CTAs past
// the bin grid (ragged blocks) exit at once.
constexpr int kSuper = 8;
inline int64_t super_ctas(const int nb[3]) {
    int64_t n = 1;
    for (int d = 0; d < 3; ++d) n *= (nb[d] + kSuper - 1) / kSuper;
    return n * kSuper * kSuper * kSuper;
}
__device__ __forceinline__ int super_bin(const int nb[3], int64_t blk) {
    const int64_t st = blk / (kSuper * kSuper * kSuper);
    const int w = (int)(blk % (kSuper * kSuper * kSuper));
    const int s0 = (nb[0] + kSuper - 1) / kSuper, s1 = (nb[1] + kSuper - 1) / kSuper;
    const int bx = (int)(st % s0) * kSuper + (w % kSuper);
    const int by = (int)((st / s0) % s1) * kSuper + (w / kSuper) % kSuper;
    const int bz = (int)(st / ((int64_t)s0 * s1)) * kSuper + w / (kSuper * kSuper);
    if (bx >= nb[0] || by >= nb[1] || bz >= nb[2]) return -1;
    return bx + nb[0] * (by + nb[1] * bz);
}

// plane stride (cells) for a plane of `cells` = pitch x rows: 16-byte aligned, and for
// 8 / 4-byte cells odd in 8-byte / 4-byte words modulo 4 so that the block rows of
// consecutive z fall in different banks (16-byte cells: any stride)
template <int CB>
__host__ __device__ __forceinline__ int sub_plane(int cells) {
    if (CB >= 16) return cells;
    if (CB == 8) {  // even (16-byte rows), == 2 mod 4 in cells
        const int q = (cells + 1) & ~1;
        return (q & 3) == 2 ? q : q + 2;
    }
    const int q = (cells + 3) & ~3;  // multiple of 4 cells, == 4 mod 8
    return (q & 7) == 4 ? q : q + 4;
}

// The same window, branch-free and table-assisted (kernels that evaluate many
// weights per point: spread_sub.cu).  fp64: s = sqrt(max(t, 0)) as above; exp(y) as
// y = n ln2 / 64 + r, |r| <= ln2 / 128, exp(r) by its degree-5 Taylor polynomial
// (truncation < 4e-17 relative), times 2^(n mod 64 / 64) from a 64-entry table
// (kExpTab entries of shared memory, filled by exp_tab_init) and 2^(n div 64) added
// into the exponent field; n is read from the low word of the rounding sum.
constexpr int kExpTab = 64;
__device__ __forceinline__ void exp_tab_init(double* tab, int tid, int nthreads) {
    for (int i = tid; i < kExpTab; i += nthreads) tab[i] = exp2((double)i / kExpTab);
}
template <typename T> __device__ __forceinline__ T es_weight_tab(T zz, T beta, const double* tab);
template <> __device__ __forceinline__ float es_weight_tab<float>(float zz, float beta,
                                                                  const double*) {
    return es_weight<float>(zz, beta);
}
template <> __device__ __forceinline__ double es_weight_tab<double>(double zz, double beta,
                                                                    const double* tab) {
    // |z| > 1 (t < 0) computes a finite or non-finite value that the final select
    // discards: no branch, no clamp of t in fp64
    const double t = fma(-zz, zz, 1.0);
    const double tc = t;
    float yf;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(fmaxf((float)t, 1e-30f)));
    double y = (double)yf;
    const double ht = -0.5 * tc;
    double h = fma(ht, y * y, 0.5);
    y = fma(y, h, y);
    h = fma(ht, y * y, 0.5);
    y = fma(y, h, y);
    const double a = fma(beta, tc * y, -beta);  // beta (s - 1) in [-beta, 0]
    const double kMagic = 6755399441055744.0;   // 1.5 * 2^52: round-to-nearest integer
    const double m = fma(a, 92.332482616893657, kMagic);  // 64 / ln2
    const double nd = m - kMagic;
    const int n = __double2loint(m);  // nd as an integer, in [-64 beta / ln2, 0]
    double r = fma(-nd, 6.93147180369123816490e-01 / 64.0, a);  // exact n * hi
    r = fma(-nd, 1.90821492927058770002e-10 / 64.0, r);
    double q = 1.0 / 120.0;
    q = fma(q, r, 1.0 / 24.0);
    q = fma(q, r, 1.0 / 6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    q = fma(q, r, 1.0);
    const double v = q * tab[n & (kExpTab - 1)];
    const double e = __hiloint2double(__double2hiint(v) + ((n >> 6) << 20), __double2loint(v));
    return t >= 0.0 ? e : 0.0;
}

// The 3w weights of one point, phi(2 (k - d_a) / w) for axis a and node k, into
// registers.  All table reads happen here, before the caller's shared-memory
// stores: a store that may alias the table would otherwise order every later
// evaluation after it and serialise the 3w independent chains.
template <typename T, int W>
__device__ __forceinline__ void es_weights3(const T (&d)[3], T beta, const double* tab,
                                            T (&w)[3][W]) {
    const T two_over_w = (T)2 / (T)W;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int k = 0; k < W; ++k) w[a][k] = es_weight_tab<T>(((T)k - d[a]) * two_over_w, beta, tab);
}

}  // namespace dev
}  // namespace nufft
