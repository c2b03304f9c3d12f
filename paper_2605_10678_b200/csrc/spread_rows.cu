// spread_rows.cu -- the default spreading kernel (Step 1 of Eq. (3), the operator C,
// PAPER.md:141-142, 187-213) for w <= 12: register-resident subgrid rows.
//
// One CTA (8 warps, 256 threads) per bin.  The bin's subgrid is E x E x E cells
// with E = T + w = 16 (so the bin edge is T = 16 - w).  Its E*E = 256 (y, z)
// rows are owned one per thread -- lane l of warp k owns row y = l mod 16,
// z = 2k + l / 16 -- and each thread keeps its whole row of complex cells in
// REGISTERS for the lifetime of the CTA.  Accumulation therefore never touches
// shared memory (the smem read-modify-write of the paper's Tiled / Grid-
// Parallel spreads, is latency- and bandwidth-bound at ~4
// fp64 cells per clock per SM on sm_100a):
//
//   phase A  (per batch of points, all threads) the 3w ES weights of every
//            (point, axis) in registers -- d w evaluations per point by
//            separability, phi evaluated directly
//             -- staged in shared memory as wx, wy and the
//            complex z-profile c * wz;
//   phase B  every warp walks the batch; a point whose z-stencil misses the
//            warp's two z-planes is skipped (warp-uniform); otherwise each
//            thread forms f = c wz[z - lz] wy[y - ly] for its row (zero
//            outside the stencil) and a warp-uniform switch on the stencil's
//            x-base selects w complex FMAs on FIXED registers of the row:
//            row[lx + m] += f wx[m].  Rows are thread-private, so there are no
//            conflicts, atomics or barriers inside the batch;
//   flush    each thread writes its row to shared memory and the subgrid rows
//            are added into the periodic fine grid in HBM by the bulk-async
//            engine (cp.reduce.async.bulk .add, SASS UBLKRED), split at the
//            periodic boundary (ghost cells wrap directly).
#include "device_util.cuh"
#include "internal.cuh"

namespace nufft {

namespace {

using namespace dev;

constexpr int kRowsE = 16;          // subgrid edge (y and z), = T + w
constexpr int kRowsThreads = 256;   // one thread per (y, z) row
template <typename T> struct RowsBatch;
template <> struct RowsBatch<float> { static constexpr int value = 128; };
template <> struct RowsBatch<double> { static constexpr int value = 64; };

template <typename T, int W>
struct RowsSmem {
    using C = typename Cx<T>::type;
    static constexpr int P = sizeof(C) >= 16 ? kRowsE : kRowsE + 2;  // x pitch (even-x alignment in fp32)
    static constexpr int B = RowsBatch<T>::value;
    static constexpr size_t bytes() {
        return (size_t)kRowsE * kRowsE * P * sizeof(C)     // flush staging (rows)
               + (size_t)B * W * sizeof(C)                 // cwz
               + (size_t)B * 2 * W * sizeof(T)             // wx | wy
               + (size_t)B * sizeof(int);                  // la
    }
};

// row[K + m] += f * wx[m], m < W, on compile-time register indices
template <int K, int W, int P, typename C, typename T>
__device__ __forceinline__ void row_fma(C (&row)[P], const C f, const T (&wx)[W]) {
    if constexpr (K + W <= P) {
#pragma unroll
        for (int m = 0; m < W; ++m) {
            row[K + m].x = fma(f.x, wx[m], row[K + m].x);
            row[K + m].y = fma(f.y, wx[m], row[K + m].y);
        }
    }
}

template <typename T, int W>
__global__ void __launch_bounds__(kRowsThreads, 2)
    spread_rows_kernel(Geom g, PtsView<T> p, const typename Cx<T>::type* __restrict__ c,
                       typename Cx<T>::type* __restrict__ grid, T beta) {
    using C = typename Cx<T>::type;
    using S = RowsSmem<T, W>;
    constexpr int P = S::P;
    constexpr int B = S::B;
    constexpr int E = kRowsE;
    constexpr int TT = E - W;
    extern __shared__ __align__(16) unsigned char smem[];

    const int b = blockIdx.x;
    const uint32_t beg = p.offset[b], end = p.offset[b + 1];
    if (beg == end) return;

    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const TileX tx = tile_x<sizeof(C)>(bx, TT, W);
    C* tile = reinterpret_cast<C*>(smem);                 // [E*E][P] (flush only)
    C* scwz = tile + E * E * P;                           // [B][W]
    T* swxy = reinterpret_cast<T*>(scwz + B * W);         // [B][2W]: wx | wy
    int* sla = reinterpret_cast<int*>(swxy + B * 2 * W);  // [B]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int my_y = lane & 15, my_z = 2 * warp + (lane >> 4);
    const int z0 = 2 * warp;  // this warp's planes: z0, z0 + 1
    const T two_over_w = (T)2 / (T)W;

    C row[P];
#pragma unroll
    for (int i = 0; i < P; ++i) row[i] = C{0, 0};

    for (uint32_t p0 = beg; p0 < end; p0 += B) {
        const int n = (int)min((uint32_t)B, end - p0);
        __syncthreads();  // previous batch consumed
        // ---- phase A: one thread per (point, axis, node) weight
        for (int e = threadIdx.x; e < 3 * W * n; e += kRowsThreads) {
            const int i = e / (3 * W), r3 = e - i * (3 * W), d = r3 / W, k = r3 - d * W;
            const PtRec<T>& r = p.rec[p0 + i];
            const T wk = p.w ? p.w[(size_t)p0 * (3 * W) + e]  // precomputed at setpts
                             : es_weight<T>(((T)k - r.d[d]) * two_over_w, beta);
            if (d < 2) {
                swxy[i * 2 * W + d * W + k] = wk;
            } else {
                const C cv = c[r.perm];
                scwz[i * W + k] = C{cv.x * wk, cv.y * wk};
                if (k == 0) sla[i] = (int)r.la;
            }
        }
        __syncthreads();
        // ---- phase B: thread-private register rows
        for (int i = 0; i < n; ++i) {
            const int la = sla[i];
            const int lz = la >> 16;
            if (z0 + 1 < lz || z0 >= lz + W) continue;  // warp-uniform: no plane of ours
            const int ly = (la >> 8) & 0xff, lx = (la & 0xff) + tx.shift;
            const int zi = my_z - lz, yi = my_y - ly;
            const bool act = (unsigned)zi < (unsigned)W && (unsigned)yi < (unsigned)W;
            const T* wl = swxy + i * 2 * W;
            C f{0, 0};
            if (act) {
                const C cz = scwz[i * W + zi];
                const T wy = wl[W + yi];
                f = C{cz.x * wy, cz.y * wy};
            }
            T wx[W];
#pragma unroll
            for (int m = 0; m < W; ++m) wx[m] = wl[m];
            switch (lx) {
#define NUFFT_ROW_CASE(K) \
    case K:               \
        row_fma<K, W, P>(row, f, wx); \
        break;
                NUFFT_ROW_CASE(0) NUFFT_ROW_CASE(1) NUFFT_ROW_CASE(2) NUFFT_ROW_CASE(3)
                NUFFT_ROW_CASE(4) NUFFT_ROW_CASE(5) NUFFT_ROW_CASE(6) NUFFT_ROW_CASE(7)
                NUFFT_ROW_CASE(8) NUFFT_ROW_CASE(9) NUFFT_ROW_CASE(10) NUFFT_ROW_CASE(11)
                NUFFT_ROW_CASE(12) NUFFT_ROW_CASE(13) NUFFT_ROW_CASE(14) NUFFT_ROW_CASE(15)
                NUFFT_ROW_CASE(16)
#undef NUFFT_ROW_CASE
                default:
                    break;
            }
        }
    }
    // ---- flush: rows -> shared memory -> periodic fine grid (bulk reductions)
    const int r_me = my_z * E + my_y;
#pragma unroll
    for (int i = 0; i < P; ++i) tile[r_me * P + i] = row[i];
    fence_proxy_async_smem();
    __syncthreads();
    const int oy = by * TT - W / 2, oz = bz * TT - W / 2;
    const int nfx = (int)g.nf[0], nfy = (int)g.nf[1];
    int sg[2], ss[2], sn[2];
    const int nseg = row_segments(tx.gx0, P, nfx, sg, ss, sn);
    {
        const int r = threadIdx.x;  // one row per thread (E*E == kRowsThreads)
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
}

template <typename T, int W>
cudaError_t launch_rows_w(const Geom& g, const PtsView<T>& p, int64_t nbins,
                          const typename Cx<T>::type* c, typename Cx<T>::type* grid, double beta,
                          cudaStream_t s) {
    if constexpr (W > 12) {
        return cudaErrorNotSupported;
    } else {
        const size_t smem = RowsSmem<T, W>::bytes();
        auto kern = spread_rows_kernel<T, W>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return e;
        }
        if (nbins > 0) kern<<<(unsigned)nbins, kRowsThreads, smem, s>>>(g, p, c, grid, (T)beta);
        return cudaGetLastError();
    }
}

}  // namespace

bool spread_rows_applies(const Geom& g) {
    return g.w <= 12 && g.T[0] == kRowsE - g.w && g.T[1] == kRowsE - g.w && g.T[2] == kRowsE - g.w;
}

template <typename T>
size_t spread_rows_smem_bytes(const Geom& g) {
    switch (g.w) {
        case 2: return RowsSmem<T, 2>::bytes();   case 3: return RowsSmem<T, 3>::bytes();
        case 4: return RowsSmem<T, 4>::bytes();   case 5: return RowsSmem<T, 5>::bytes();
        case 6: return RowsSmem<T, 6>::bytes();   case 7: return RowsSmem<T, 7>::bytes();
        case 8: return RowsSmem<T, 8>::bytes();   case 9: return RowsSmem<T, 9>::bytes();
        case 10: return RowsSmem<T, 10>::bytes(); case 11: return RowsSmem<T, 11>::bytes();
        case 12: return RowsSmem<T, 12>::bytes();
        default: return 0;
    }
}

template <typename T>
cudaError_t launch_spread_rows(const Geom& g, const PtsView<T>& p, int64_t nbins,
                               const typename Cx<T>::type* c, typename Cx<T>::type* grid,
                               double beta, cudaStream_t s) {
    if (!spread_rows_applies(g)) return cudaErrorNotSupported;
    switch (g.w) {
#define NUFFT_RW(WW) \
    case WW:         \
        return launch_rows_w<T, WW>(g, p, nbins, c, grid, beta, s);
        NUFFT_RW(2) NUFFT_RW(3) NUFFT_RW(4) NUFFT_RW(5) NUFFT_RW(6) NUFFT_RW(7) NUFFT_RW(8)
        NUFFT_RW(9) NUFFT_RW(10) NUFFT_RW(11) NUFFT_RW(12)
#undef NUFFT_RW
        default:
            return cudaErrorNotSupported;
    }
}

template cudaError_t launch_spread_rows<float>(const Geom&, const PtsView<float>&, int64_t,
                                               const float2*, float2*, double, cudaStream_t);
template cudaError_t launch_spread_rows<double>(const Geom&, const PtsView<double>&, int64_t,
                                                const double2*, double2*, double, cudaStream_t);
template size_t spread_rows_smem_bytes<float>(const Geom&);
template size_t spread_rows_smem_bytes<double>(const Geom&);

}  // namespace nufft
