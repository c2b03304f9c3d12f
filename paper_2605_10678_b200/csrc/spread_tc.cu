// spread_tc.cu -- fp32 spreading (Step 1 of Eq. (3), the operator C, PAPER.md:141-142,
// 187-213) on the 5th-generation tensor cores (tcgen05, accumulators in TMEM).
//
// With the zero-padded separable profiles of spread_outer.cu, the 16^3 subgrid of
// one bin is a dense contraction over the bin's points j:
//
//     G[(z,y)][x] = sum_j  A[(z,y)][j] B[x][j],   A = wz_j[z] wy_j[y],  B = c_j wx_j[x]
//
// an M = 256 ((z,y) rows) x N = 32 (16 complex x) x K = points GEMM.  Per batch of
// KB = 16 points the CTA writes A and B into shared memory in the canonical
// no-swizzle K-major UMMA layout, and one thread issues tcgen05.mma kind::tf32
// (two M = 128 halves x two K = 8 steps) into a 64-column fp32 TMEM accumulator.
// TF32 keeps 10 mantissa bits, so every operand is split x = hi + lo (hi = tf32(x),
// lo = tf32(x - hi)) and the product is hi*hi + hi*lo + lo*hi ("3xTF32"): the
// dropped lo*lo term and the split residue are ~2^-22 relative, the accuracy of the
// fp32 FMA path.  Operand buffers are double-buffered on tcgen05.commit mbarriers.
// Epilogue: tcgen05.ld (one TMEM lane = one (z,y) row per thread) -> shared-memory
// subgrid -> cp.reduce.async.bulk .add into the periodic fine grid (as the other
// spread kernels).  Plan option spread_warps = 3 (fp32 complex, T = 16 - w).
//
// Status (B200, C2b fp32 w = 7): parity-green but 1.12 ms vs 0.78 ms for the
// register outer products; with the MMAs removed the kernel still takes 0.99 ms,
// so the tensor cores are not the limit -- building the operands (zero-padded
// profiles, the 256-row Kronecker A = wz (x) wy and its hi / lo split, two CTA
// barriers per 16-point batch, 2 CTAs per SM) is.  Kept as an option, not the default.
#include "device_util.cuh"
#include "internal.cuh"

namespace nufft {

namespace {

using namespace dev;

constexpr int kTcThreads = 256;
constexpr int kTcE = 16;   // subgrid edge
constexpr int kKB = 16;    // points per batch = 2 MMA K-steps of 8 (tf32)
constexpr int kM = 256;    // (z,y) rows
constexpr int kN = 32;     // 16 complex x as (re, im) columns

// shared-memory carve (bytes)
constexpr int kAbytes = 2 * kM * kKB * 4;                 // hi | lo, one buffer
constexpr int kBbytes = 2 * kN * kKB * 4;
constexpr int kOffA = 0;                                   // [2 buffers]
constexpr int kOffB = kOffA + 2 * kAbytes;                 // [2 buffers]
constexpr int kPS = kKB + 4;                               // profile row stride (floats): 2-way stores
constexpr int kOffProf = kOffB + 2 * kBbytes;              // [3][16 cells][kPS] floats, by point
constexpr int kOffC = kOffProf + 3 * kTcE * kPS * 4;       // [KB] float2
constexpr int kOffBar = kOffC + kKB * 8;                   // 2 mbarriers + tmem address
constexpr int kSmemTc = kOffBar + 32;
constexpr int kTilePitch = kTcE + 2;                       // float2 cells: 16-byte aligned rows
static_assert(kTcE * kTcE * kTilePitch * 8 <= 2 * kAbytes, "flush tile aliases the A buffers");

// x = hi + lo: hi = x rounded to the 10-bit TF32 mantissa (integer round-half-up on
// the bit pattern, exact for the finite values here), lo = x - hi exactly in fp32
// (|lo| <= 2^-11 |x|); the tensor core reads lo's top 19 bits, a further 2^-10
// relative of lo, so hi*hi + hi*lo + lo*hi carries ~2^-20 relative error per product
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

// UMMA shared-memory descriptor, SWIZZLE_NONE, K-major: core matrices of 8 rows x
// 16 bytes; lbo = bytes between the two 16-byte K chunks of one K = 8 step, sbo =
// bytes between 8-row groups along M / N; version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// instruction descriptor: D f32, A / B tf32, both K-major, N = 32, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kN >> 3) << 17) |
                            ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

template <int W>
__global__ void __launch_bounds__(kTcThreads, 2)
    spread_tc_kernel(Geom g, PtsView<float> p, const float2* __restrict__ c,
                     float2* __restrict__ grid, float beta) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const int b = blockIdx.x;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;
    const int n = (int)(end - beg);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);

    float* prof = reinterpret_cast<float*>(smem + kOffProf);
    float2* pc = reinterpret_cast<float2*>(smem + kOffC);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kOffBar);
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(smem + kOffBar + 16);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                         smem_addr(s_tmem))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        mbar_init(bar + 0, 1);
        mbar_init(bar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    const float two_over_w = 2.0f / (float)W;
    const int nbat = (n + kKB - 1) / kKB;
    // the batch's (point, axis, cell) items, kItems per thread; their point records
    // (and strengths) are loaded one batch ahead so the global latency overlaps the
    // current batch's operand build and MMAs
    constexpr int kItems = kKB * 3 * kTcE / kTcThreads;
    static_assert(kItems * kTcThreads == kKB * 3 * kTcE, "whole items per thread");
    float nd[kItems];
    uint32_t nla[kItems];
    float2 ncv = make_float2(0.0f, 0.0f);
    // item q of this thread: point jq, axis dq, cell iq (batch-invariant)
    int jq[kItems], dq[kItems], iq[kItems];
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
        const int e = tid + q * kTcThreads;
        jq[q] = e / (3 * kTcE);
        dq[q] = (e / kTcE) % 3;
        iq[q] = e % kTcE;
    }
    auto fetch = [&](int kb) {
        const uint32_t p0 = beg + kb * kKB;
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            if (p0 + jq[q] < end) {
                nd[q] = p.rec[p0 + jq[q]].d[dq[q]];
                nla[q] = p.rec[p0 + jq[q]].la;
            }
        }
        if (tid < kKB) ncv = p0 + tid < end ? c[p.rec[p0 + tid].perm] : make_float2(0.0f, 0.0f);
    };
    fetch(0);
    for (int kb = 0; kb < nbat; ++kb) {
        const int buf = kb & 1;
        const uint32_t p0 = beg + kb * kKB;
        const int nv = min(kKB, (int)(end - p0));
        float cd[kItems];
        uint32_t cla[kItems];
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            cd[q] = nd[q];
            cla[q] = nla[q];
        }
        if (tid < kKB) pc[tid] = ncv;
        if (kb + 1 < nbat) fetch(kb + 1);
        // ---- zero-padded 16-cell profiles of the batch, one thread per (point, axis,
        // cell): phi of the node the cell holds, 0 off the stencil and for padding points
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            const int j = jq[q], d = dq[q];
            float v = 0.0f;
            if (j < nv) {
                const int k = iq[q] - (int)((cla[q] >> (8 * d)) & 0xff);
                if (k >= 0 && k < W)
                    v = p.w ? p.w[(size_t)(p0 + j) * (3 * W) + d * W + k]
                            : es_weight<float>(((float)k - cd[q]) * two_over_w, beta);
            }
            prof[(d * kTcE + iq[q]) * kPS + j] = v;  // [axis][cell][point]
        }
        // the MMAs of batch kb - 2 read this operand buffer: wait for their commit
        if (kb >= 2) mbar_wait(bar + buf, ((kb - 2) >> 1) & 1);
        __syncthreads();
        // ---- A[(z,y)][j] = wz_j[z] wy_j[y] (hi | lo): thread = row m, 4 points per 16-byte store
        {
            uint32_t* Ahi = reinterpret_cast<uint32_t*>(smem + kOffA + buf * kAbytes);
            uint32_t* Alo = Ahi + kM * kKB;
            const int m = tid, z = m >> 4, y = m & 15;
            const float* wz = prof + (2 * kTcE + z) * kPS;
            const float* wy = prof + (1 * kTcE + y) * kPS;
#pragma unroll
            for (int kc = 0; kc < kKB / 4; ++kc) {
                const float4 a = *reinterpret_cast<const float4*>(wz + 4 * kc);
                const float4 bq = *reinterpret_cast<const float4*>(wy + 4 * kc);
                uint32_t h[4], l[4];
                split_tf32(a.x * bq.x, h[0], l[0]);
                split_tf32(a.y * bq.y, h[1], l[1]);
                split_tf32(a.z * bq.z, h[2], l[2]);
                split_tf32(a.w * bq.w, h[3], l[3]);
                const int off = ((kc * (kM / 8) + (m >> 3)) * 8 + (m & 7)) * 4;
                *reinterpret_cast<uint4*>(Ahi + off) = make_uint4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<uint4*>(Alo + off) = make_uint4(l[0], l[1], l[2], l[3]);
            }
        }
        // ---- B[(x, re/im)][j] = (c_j wx_j[x]) (hi | lo)
        if (tid < kN * (kKB / 4)) {
            uint32_t* Bhi = reinterpret_cast<uint32_t*>(smem + kOffB + buf * kBbytes);
            uint32_t* Blo = Bhi + kN * kKB;
            const int nn = tid & (kN - 1), kc = tid / kN, x = nn >> 1;
            const float4 wx = *reinterpret_cast<const float4*>(prof + x * kPS + 4 * kc);
            const float wq[4] = {wx.x, wx.y, wx.z, wx.w};
            uint32_t h[4], l[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 cv = pc[4 * kc + q];
                split_tf32((nn & 1 ? cv.y : cv.x) * wq[q], h[q], l[q]);
            }
            const int off = ((kc * (kN / 8) + (nn >> 3)) * 8 + (nn & 7)) * 4;
            *reinterpret_cast<uint4*>(Bhi + off) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(Blo + off) = make_uint4(l[0], l[1], l[2], l[3]);
        }
        fence_proxy_async_smem();  // generic-proxy operand stores -> tensor-core (async) reads
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t a0 = smem_addr(smem + kOffA + buf * kAbytes);
            const uint32_t b0 = smem_addr(smem + kOffB + buf * kBbytes);
            const uint32_t alo = a0 + kM * kKB * 4, blo = b0 + kN * kKB * 4;
            constexpr uint32_t ALBO = (kM / 8) * 128, BLBO = (kN / 8) * 128;
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int ks = 0; ks < kKB / 8; ++ks) {
                    const uint32_t ao = h * (128 / 8) * 128 + ks * 2 * ALBO, bo = ks * 2 * BLBO;
                    const uint32_t d = tmem + h * kN;
                    mma_tf32(d, umma_desc(a0 + ao, ALBO, 128), umma_desc(b0 + bo, BLBO, 128),
                             (kb | ks) ? 1u : 0u);
                    mma_tf32(d, umma_desc(a0 + ao, ALBO, 128), umma_desc(blo + bo, BLBO, 128), 1u);
                    mma_tf32(d, umma_desc(alo + ao, ALBO, 128), umma_desc(b0 + bo, BLBO, 128), 1u);
                }
            mma_commit(bar + buf);
        }
    }
    // ---- epilogue: the last commit covers every MMA of the CTA
    mbar_wait(bar + ((nbat - 1) & 1), ((nbat - 1) >> 1) & 1);
    tc_fence_after();
    uint32_t r[32];
    {
        const int h = warp >> 2, lg = warp & 3;
        const uint32_t ta = tmem + ((uint32_t)(32 * lg) << 16) + (uint32_t)(h * kN);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
            "%28, %29, %30, %31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();  // every TMEM read done; the A buffers become the flush tile
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");

    const TileX tx = tile_x<sizeof(float2)>(bx, g.T[0], W);
    float2* tile = reinterpret_cast<float2*>(smem + kOffA);
    {
        const int m = 128 * (warp >> 2) + 32 * (warp & 3) + lane;  // (z,y) row of this thread
        float2* trow = tile + m * kTilePitch;
#pragma unroll
        for (int x = 0; x < kTcE; ++x)
            trow[tx.shift + x] = make_float2(__uint_as_float(r[2 * x]), __uint_as_float(r[2 * x + 1]));
#pragma unroll
        for (int q = 0; q < kTilePitch - kTcE; ++q)
            trow[q < tx.shift ? q : kTcE + q] = make_float2(0.0f, 0.0f);
    }
    fence_proxy_async_smem();
    __syncthreads();
    const int oy = by * g.T[1] - W / 2, oz = bz * g.T[2] - W / 2;
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    int sg[2], ss[2], sn[2];
    const int nseg = row_segments(tx.gx0, kTilePitch, nfx, sg, ss, sn);
    {
        const int rr = tid;  // one (z,y) row per thread
        const int cz = rr / kTcE, cy = rr - cz * kTcE;
        const int gy = wrap1(oy + cy, nfy), gz = z_row(oz + cz, g);
        float2* grow = grid + (int64_t)nfx * ((int64_t)gz * nfy + gy);
        const float2* trow = tile + rr * kTilePitch;
        for (int k = 0; k < (gz < -g.hz_lo ? 0 : nseg); ++k)
            bulk_red_add(reinterpret_cast<float*>(grow + sg[k]), trow + ss[k],
                         (unsigned)(sn[k] * sizeof(float2)));
    }
    bulk_commit();
    bulk_wait_read();
}

}  // namespace

bool spread_tc_applies(const Geom& g) {
    return g.w >= 2 && g.w <= 12 && g.T[0] == kTcE - g.w && g.T[1] == kTcE - g.w &&
           g.T[2] == kTcE - g.w;
}

cudaError_t launch_spread_tc(const Geom& g, const PtsView<float>& p, int64_t nbins,
                             const float2* c, float2* grid, double beta, cudaStream_t s) {
    if (nbins <= 0) return cudaSuccess;
#define CASE(WW)                                                                              \
    case WW: {                                                                               \
        auto k = spread_tc_kernel<WW>;                                                       \
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             kSmemTc);                                       \
        if (e != cudaSuccess) return e;                                                      \
        k<<<(unsigned)nbins, kTcThreads, kSmemTc, s>>>(g, p, c, grid, (float)beta);          \
        break;                                                                               \
    }
    switch (g.w) {
        CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12)
        default: return cudaErrorInvalidValue;
    }
#undef CASE
    return cudaGetLastError();
}

}  // namespace nufft
