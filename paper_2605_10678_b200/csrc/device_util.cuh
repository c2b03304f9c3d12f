// device_util.cuh -- device helpers shared by the spread / interp kernels:
// the ES window, periodic index wrap, and the sm_90+/sm_100a bulk-async (TMA
// engine) copy / reduce primitives with their mbarrier plumbing.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

// NUFFT_CHECK(cond): a device-side bounds assertion, compiled only into the
// bounds-checked build (NUFFT_DEBUG_BOUNDS, build.py); traps the kernel with the
// failing file / line.  A no-op in the product build.
#ifdef NUFFT_DEBUG_BOUNDS
#include <cstdio>
#define NUFFT_CHECK(cond)                                                              \
    do {                                                                               \
        if (!(cond)) {                                                                 \
            printf("NUFFT_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__,     \
                   __LINE__, #cond, (int)blockIdx.x, (int)threadIdx.x);                \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define NUFFT_CHECK(cond) \
    do {                  \
    } while (0)
#endif

namespace nufft {
namespace dev {

// ES window:  phi(z) = exp(beta (sqrt(1 - z^2) - 1)) for |z| <= 1
// (the endpoint is inside the support, reading R5), 0 otherwise.
//
// fp64: the weight evaluation is a large share of the spread / interp work
// (libm exp + sqrt cost ~100 instructions per weight), so it is specialised to
// the range it is used on.  s = sqrt(t), t in (0, 1]: fp32 rsqrt seed (2^-23)
// and two fp64 Newton steps (error ~2^-92 before rounding).  exp(y), y = beta
// (s - 1) in [-beta, 0], beta <= 2.3 * 16: y = n ln2 + r with |r| <= ln2 / 2
// (Cody-Waite split of ln2), exp(r) by its degree-13 Taylor polynomial
// (truncation < 6e-18 relative), times 2^n built in the exponent field (no
// overflow / underflow / NaN cases exist on this range).  Relative error
// ~2e-16 against the correctly rounded value -- far inside the 1e-10 parity bar.
template <typename T> __device__ __forceinline__ T es_weight(T zz, T beta);
template <> __device__ __forceinline__ double es_weight<double>(double zz, double beta) {
    const double t = 1.0 - zz * zz;
    if (!(t >= 0.0)) return 0.0;
    double s = 0.0;
    if (t > 0.0) {
        double y = (double)rsqrtf((float)t);
        double h = fma(-0.5 * t, y * y, 0.5);
        y = fma(y, h, y);
        h = fma(-0.5 * t, y * y, 0.5);
        y = fma(y, h, y);
        s = t * y;
    }
    const double a = beta * (s - 1.0);
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52: round-to-nearest integer
    const double nd = fma(a, 1.4426950408889634, kMagic) - kMagic;
    double r = fma(-nd, 6.93147180369123816490e-01, a);  // ln2 high part (exact n * hi)
    r = fma(-nd, 1.90821492927058770002e-10, r);          // ln2 low part
    double p = 1.0 / 6227020800.0;                        // 1/13!
    p = fma(p, r, 1.0 / 479001600.0);
    p = fma(p, r, 1.0 / 39916800.0);
    p = fma(p, r, 1.0 / 3628800.0);
    p = fma(p, r, 1.0 / 362880.0);
    p = fma(p, r, 1.0 / 40320.0);
    p = fma(p, r, 1.0 / 5040.0);
    p = fma(p, r, 1.0 / 720.0);
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const int n = (int)nd;  // in [-54, 0]
    return p * __hiloint2double((n + 1023) << 20, 0);
}
template <> __device__ __forceinline__ float es_weight<float>(float zz, float beta) {
    const float t = 1.0f - zz * zz;
    return t >= 0.0f ? expf(beta * (sqrtf(t) - 1.0f)) : 0.0f;
}

// one conditional step each way: valid for -n <= i < 2n (the plan guarantees T + w <= nf)
__device__ __forceinline__ int wrap1(int i, int n) {
    i += i < 0 ? n : 0;
    return i >= n ? i - n : i;
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

// ---- mbarrier (transaction-count barrier for bulk copies)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// ---- 1D bulk copy global -> shared, completion counted on an mbarrier (UBLKCP)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, unsigned bytes,
                                         uint64_t* bar) {
    NUFFT_CHECK((reinterpret_cast<uintptr_t>(src_gmem) & 15) == 0 && (bytes & 15) == 0 &&
                (smem_addr(dst_smem) & 15) == 0);
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// ---- 1D bulk reduction shared -> global (UBLKRED ... ADD): dst[i] += src[i]
__device__ __forceinline__ void bulk_red_add(float* dst_gmem, const void* src_smem,
                                             unsigned bytes) {
    NUFFT_CHECK((reinterpret_cast<uintptr_t>(dst_gmem) & 15) == 0 && (bytes & 15) == 0 &&
                (smem_addr(src_smem) & 15) == 0);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                     dst_gmem),
                 "r"(smem_addr(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_red_add(double* dst_gmem, const void* src_smem,
                                             unsigned bytes) {
    NUFFT_CHECK((reinterpret_cast<uintptr_t>(dst_gmem) & 15) == 0 && (bytes & 15) == 0 &&
                (smem_addr(src_smem) & 15) == 0);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(
                     dst_gmem),
                 "r"(smem_addr(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// per-thread asynchronous global -> shared copies (SASS LDGSTS), no register staging
__device__ __forceinline__ void cp_async16(void* dst_smem, const void* src_gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst_smem)),
                 "l"(src_gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src_gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst_smem)),
                 "l"(src_gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// generic-proxy shared-memory writes -> visible to the async (bulk) proxy
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Tile x-geometry shared by spread and interp.  Bulk copies need 16-byte
// aligned rows and lengths.  fp64 complex cells are 16 bytes, so any origin
// works (row length = pitch = T + w).  Smaller cells (fp32 complex / fp64 real:
// 8 bytes, fp32 real: 4 bytes) start the subgrid row at a global x that is a
// multiple of A = 16 / cell_bytes (shift = ox mod A) with a length that is a
// multiple of A and covers every shift; the smem pitch is = 8 (mod 16) cells, so
// the 2 (8-byte) or 4 (4-byte) consecutive 8-cell row segments of one 128-byte
// wavefront fall into distinct banks.
struct TileX {
    int gx0;    // global x of smem column 0 (may be negative: periodic)
    int shift;  // smem column of the nominal tile origin bx*T - w/2 (< 16 / cell bytes)
    int len;    // cells per row copied to / from the grid
    int pitch;  // smem row stride in cells (>= len)
};
// cells per 16-byte alignment unit: 16 / gcd(cell bytes, 16) (1 for 16 / 32 B cells,
// 2 for 8 / 24 B, 4 for 4 / 12 B)
template <int CELL_BYTES> struct AlignCells {
    static constexpr int g = (CELL_BYTES % 16 == 0) ? 16 : (CELL_BYTES % 8 == 0) ? 8 : (CELL_BYTES % 4 == 0) ? 4 : 1;
    static constexpr int value = 16 / g;
};
template <int CELL_BYTES>
__host__ __device__ __forceinline__ int tile_len(int T, int W) {
    constexpr int A = AlignCells<CELL_BYTES>::value;
    return A == 1 ? T + W : ((T + W + (A - 1) + (A - 1)) / A) * A;
}
template <int CELL_BYTES>
__host__ __device__ __forceinline__ int tile_pitch(int T, int W) {
    const int len = tile_len<CELL_BYTES>(T, W);
    if (CELL_BYTES != 4 && CELL_BYTES != 8) return len;
    return len <= 8 ? 8 : 16 * ((len - 8 + 15) / 16) + 8;
}
template <int CELL_BYTES>
__device__ __forceinline__ TileX tile_x(int bx, int T, int W) {
    constexpr int A = AlignCells<CELL_BYTES>::value;
    const int ox = bx * T - W / 2;
    TileX t;
    t.shift = ox & (A - 1);
    t.gx0 = ox - t.shift;
    t.len = tile_len<CELL_BYTES>(T, W);
    t.pitch = tile_pitch<CELL_BYTES>(T, W);
    return t;
}

// ---- grid / strength value types: complex (Eq. 1-2) or real
// complex x real in fp32 uses the packed 2-wide FP32 pipe of sm_100 (SASS FFMA2 /
// FMUL2, PTX fma.rn.f32x2 / mul.rn.f32x2): one instruction per complex update
__device__ __forceinline__ uint64_t f2_bits(float2 v) {
    return (uint64_t)__float_as_uint(v.x) | ((uint64_t)__float_as_uint(v.y) << 32);
}
__device__ __forceinline__ float2 f2_from(uint64_t b) {
    return float2{__uint_as_float((uint32_t)b), __uint_as_float((uint32_t)(b >> 32))};
}
__device__ __forceinline__ float2 vscale(float2 a, float s) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(float2{s, s})));
    return f2_from(r);
}
__device__ __forceinline__ double2 vscale(double2 a, double s) { return double2{a.x * s, a.y * s}; }
__device__ __forceinline__ float vscale(float a, float s) { return a * s; }
__device__ __forceinline__ double vscale(double a, double s) { return a * s; }
// acc += z * w
__device__ __forceinline__ void vfma(float2& acc, float2 z, float w) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(f2_bits(z)), "l"(f2_bits(float2{w, w})), "l"(f2_bits(acc)));
    acc = f2_from(r);
}
__device__ __forceinline__ void vfma(double2& acc, double2 z, double w) {
    acc.x = fma(z.x, w, acc.x);
    acc.y = fma(z.y, w, acc.y);
}
__device__ __forceinline__ void vfma(float& acc, float z, float w) { acc = fmaf(z, w, acc); }
__device__ __forceinline__ void vfma(double& acc, double z, double w) { acc = fma(z, w, acc); }
template <typename V> __device__ __forceinline__ V vzero() { return V{}; }

// Split a periodic row [gx0, gx0 + len) of a row of length nf into at most two
// contiguous segments; returns the count.  seg_g = global start, seg_s = smem
// offset, seg_n = length (cells).  Requires -nf <= gx0 and gx0 + len <= 2 nf.
__device__ __forceinline__ int row_segments(int gx0, int len, int nf, int seg_g[2], int seg_s[2],
                                            int seg_n[2]) {
    if (gx0 < 0) {
        seg_g[0] = gx0 + nf; seg_s[0] = 0; seg_n[0] = -gx0;
        seg_g[1] = 0; seg_s[1] = -gx0; seg_n[1] = len + gx0;
        return 2;
    }
    if (gx0 + len > nf) {
        seg_g[0] = gx0; seg_s[0] = 0; seg_n[0] = nf - gx0;
        seg_g[1] = 0; seg_s[1] = nf - gx0; seg_n[1] = gx0 + len - nf;
        return 2;
    }
    seg_g[0] = gx0; seg_s[0] = 0; seg_n[0] = len;
    return 1;
}

}  // namespace dev
}  // namespace nufft
