// internal.cuh -- shared internals of libnufft.so (the CUDA product path).
// Nothing here is visible through the C ABI (include/nufft.h).  The CPU oracle
// (oracle/) shares none of this code.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <vector>

#include "../../include/nufft.h"

namespace nufft {

// ---------------------------------------------------------------- complex types
template <typename T> struct Cx;
template <> struct Cx<float> { using type = float2; };
template <> struct Cx<double> { using type = double2; };

// ---------------------------------------------------------------- geometry
// Fine grid, bins and the fold/rescale map shared by all point kernels.
struct Geom {
    int64_t nf[3];      // fine grid cells per axis (nf = 2 N)
    int T[3];           // bin / tile edge (fine cells)
    int nb[3];          // bins per axis = ceil(nf / T)
    int64_t z_lo;       // first fine z-plane owned by this rank (0 on one GPU)
    int64_t nz_loc;     // fine z-planes owned by this rank (nf[2] on one GPU)
    double L;           // period
    double scale[3];    // nf / L
    int w;              // kernel width
    int spread_warps;   // spread kernel: 1 = register rows, 2 = plane outer products,
                        // 4 / 8 = smem z-plane owners
    // z boundary: 1 = periodic over nz_loc (one GPU); 0 = z-slab of a distributed
    // plan, the grid pointer addresses local plane 0 and planes [-hz_lo, nz_loc + hz_hi)
    // exist (ghost halos accumulated / filled over NCCL)
    int zper;
    int hz_lo, hz_hi;
    // sub-bins (spread_warps = 5): every bin is split into ns[0] x ns[1] x ns[2]
    // boxes of Gs[d] stencil-base values per axis (sub_common.cuh SubGeom: a sub-bin's
    // stencils fit one register block); setpts sorts by (bin, sub-bin).  nsub = 1:
    // no sub-bins
    int Gs[3];
    int ns[3];
    int nsub;
};

// Sub-bin extents Gs[3] (stencil bases per sub-bin and axis) of width w: the
// register block of the sub-bin kernels is 8 x 8 x 4R cells, R = 2 for w <= 6, 3 for
// w = 7 (sub_common.cuh SubGeom).
__host__ __device__ inline void sub_extents(int w, int G[3]) {
    const int R = w <= 6 ? 2 : 3;
    G[0] = G[1] = 9 - w;
    G[2] = 4 * R + 1 - w;
}

// Local z row of a subgrid: periodic wrap on one GPU; on a slab, -1e9 marks a
// row outside the halo-extended slab (never touched by any stencil).
__host__ __device__ __forceinline__ int z_row(int gz, const Geom& g) {
    if (g.zper) {
        const int n = (int)g.nz_loc;
        gz += gz < 0 ? n : 0;
        return gz >= n ? gz - n : gz;
    }
    return (gz < -g.hz_lo || gz >= (int)g.nz_loc + g.hz_hi) ? -1000000000 : gz;
}

// Sorted point record written by setpts, one 32-byte (one DRAM sector) AoS
// record per sorted slot:
//   d[0..2] : ls - la, the stencil phase offset in cells per axis, in [w/2 - 1, w/2]
//   la      : packed bin-local stencil base (8 bits per axis), la in [0, T]
//   perm    : original (caller) index of the point
// The weight of stencil node k on axis d is phi(2 (k - d[d]) / w).
template <typename T> struct alignas(32) PtRec {
    T d[3];
    uint32_t la;
    uint32_t perm;
};
static_assert(sizeof(PtRec<double>) == 32 && sizeof(PtRec<float>) == 32, "one sector per point");

#ifdef __CUDACC__
// One record = one 256-bit global access (SASS LDG.E.ENL2.256 / STG.E.ENL2.256 on
// sm_100a): half the load / store instructions of two 128-bit accesses.
template <typename T>
__device__ __forceinline__ PtRec<T> load_rec(const PtRec<T>* p) {
    union {
        PtRec<T> r;
        unsigned long long q[4];
    } u;
    asm("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
        : "=l"(u.q[0]), "=l"(u.q[1]), "=l"(u.q[2]), "=l"(u.q[3])
        : "l"(p));
    return u.r;
}
// streaming store (.cs: written once, read by a later kernel from HBM)
template <typename T>
__device__ __forceinline__ void store_rec_cs(PtRec<T>* p, const PtRec<T>& r) {
    union {
        PtRec<T> r;
        unsigned long long q[4];
    } u;
    u.r = r;
    asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(u.q[0]), "l"(u.q[1]),
                 "l"(u.q[2]), "l"(u.q[3])
                 : "memory");
}
#endif

template <typename T> struct PtsView {
    const uint32_t* offset;  // nbins + 1 bin starts (exclusive scan of counts)
    const uint32_t* offset_sub;  // nbins nsub + 1 sub-bin starts (Geom::nsub > 1), else = offset
    const PtRec<T>* rec;     // Np sorted records
    const T* w;              // Np x 3w ES weights in sorted order ([x | y | z] per point,
                             // node k of axis d at 3w i + w d + k), or nullptr: evaluate phi
};

// ---------------------------------------------------------------- kernel launchers
// sort.cu
// sort keys = nbins nsub (bin-major, sub-bin minor); offset_key: nkeys + 1 starts;
// offset (nbins + 1 bin starts) is gathered from it when nsub > 1 (else the same array)
template <typename T>
cudaError_t launch_bin_sort(const Geom& g, int64_t Np, const T* x, const T* y, const T* z,
                            uint32_t* count, uint32_t* offset_key, uint32_t* offset,
                            uint32_t* blocksum, uint32_t* bin_of, uint32_t* rank_of,
                            PtRec<T>* rec, int64_t nbins, cudaStream_t s);
size_t scan_blocksum_elems(int64_t nbins);
// setpts (precompute): w[3w i + w d + k] = phi(2 (k - rec[i].d[d]) / w)
template <typename T>
cudaError_t launch_weights(const PtRec<T>* rec, int64_t Np, int w, double beta, T* out,
                           cudaStream_t s);

// spread.cu: grid (nf[0] x nf[1] x nz_loc complex, x fastest) += C c
template <typename T>
cudaError_t launch_spread(const Geom& g, const PtsView<T>& p, int64_t nbins,
                          const typename Cx<T>::type* c, typename Cx<T>::type* grid, double beta,
                          cudaStream_t s);
// interp.cu: c = C^T grid.  tmap (optional): a CUtensorMap of `grid` (reals, box =
// pitch x (T1 + w) x (T2 + w) cells, interp_tile_pitch): interior bins stage their
// subgrid with one TMA tensor copy
template <typename T>
cudaError_t launch_interp(const Geom& g, const PtsView<T>& p, int64_t nbins,
                          const typename Cx<T>::type* grid, typename Cx<T>::type* c, double beta,
                          cudaStream_t s, const void* tmap = nullptr);
// spread_tc.cu: fp32 complex spread as a tcgen05 3xTF32 GEMM per bin (T = 16 - w)
bool spread_tc_applies(const Geom& g);
cudaError_t launch_spread_tc(const Geom& g, const PtsView<float>& p, int64_t nbins,
                             const float2* c, float2* grid, double beta, cudaStream_t s);
// variants.cu (ablation only): the paper's Atomic Spread and
// Direct Interpolation, one thread per point; order =
// sorted slot of caller point t (caller-order walk) or nullptr (bin-sorted walk)
template <typename T>
cudaError_t launch_spread_atomic(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                 const uint32_t* order, int64_t Np, const typename Cx<T>::type* c,
                                 typename Cx<T>::type* grid, double beta, cudaStream_t s);
template <typename T>
cudaError_t launch_interp_direct(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                 const uint32_t* order, int64_t Np,
                                 const typename Cx<T>::type* grid, typename Cx<T>::type* c,
                                 double beta, cudaStream_t s);
template <typename T>
cudaError_t launch_caller_order(const PtRec<T>* rec, int64_t Np, uint32_t* order,
                                cudaStream_t s);
// the Morton (Z-order) walk of the bins for Direct Interpolation (interp_method = 3):
// order[t] = sorted slot of the t-th point along the curve; key_count / key_off hold
// morton_keys(g) (+ 1) entries, blocksum scan_blocksum_elems(morton_keys(g)), bin_base nbins
// the paper's Tiled Spread (spread_warps = -3): shared-memory histogram with shared
// atomics, kTiledZ z-slice teams per bin
template <typename T>
cudaError_t launch_spread_tiled(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                const typename Cx<T>::type* c, typename Cx<T>::type* grid,
                                double beta, cudaStream_t s);
size_t spread_tiled_smem_bytes(const Geom& g, int cell_bytes);
size_t morton_keys(const Geom& g);
cudaError_t launch_morton_order(const Geom& g, const uint32_t* offset, int64_t nbins, int64_t Np,
                                uint32_t* key_count, uint32_t* key_off, uint32_t* blocksum,
                                uint32_t* bin_base, uint32_t* order, cudaStream_t s);
cudaError_t launch_exclusive_scan(const uint32_t* count, int64_t n, uint32_t* blocksum,
                                  uint32_t* out, cudaStream_t s);
// smem row pitch (cells) of the interp's subgrid for complex cells of cell_bytes
int interp_tile_pitch(int cell_bytes, int T, int W, bool sub = false);
template <typename T>
cudaError_t launch_spread_real(const Geom& g, const PtsView<T>& p, int64_t nbins, const T* c,
                               T* grid, double beta, cudaStream_t s);
template <typename T>
cudaError_t launch_interp_real(const Geom& g, const PtsView<T>& p, int64_t nbins, const T* grid,
                               T* c, double beta, cudaStream_t s);
// three real fields (x, y, z components: grids gstride reals apart) -> Np 3-vectors
template <typename T>
cudaError_t launch_interp_vec3(const Geom& g, const PtsView<T>& p, int64_t nbins, const T* grid,
                               int64_t gstride, T* c, double beta, cudaStream_t s);
template <typename T>
cudaError_t launch_interp_vec3_kick(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                    const T* grid, int64_t gstride, T* v0, T* v1, T* v2,
                                    double scale, double beta, cudaStream_t s);
template <typename T> size_t spread_smem_bytes(const Geom& g);
// spread_rows.cu: register-row spread (default when w <= 12 and T = 16 - w on every axis)
bool spread_rows_applies(const Geom& g);
template <typename T>
cudaError_t launch_spread_rows(const Geom& g, const PtsView<T>& p, int64_t nbins,
                               const typename Cx<T>::type* c, typename Cx<T>::type* grid,
                               double beta, cudaStream_t s);
template <typename T> size_t spread_rows_smem_bytes(const Geom& g);
// spread_sub.cu: sub-bin register-row spread (Geom::nsub > 1, w <= 6)
bool spread_sub_applies(const Geom& g);
template <typename T>
cudaError_t launch_spread_sub(const Geom& g, const PtsView<T>& p, int64_t nbins,
                              const typename Cx<T>::type* c, typename Cx<T>::type* grid,
                              double beta, cudaStream_t s);
template <typename T>
cudaError_t launch_spread_sub_real(const Geom& g, const PtsView<T>& p, int64_t nbins, const T* c,
                                   T* grid, double beta, cudaStream_t s);
template <typename T> size_t spread_sub_smem_bytes(const Geom& g);
// spread_outer.cu: per-plane outer-product spread (w <= 12 and T = 16 - w on every axis)
bool spread_outer_applies(const Geom& g);
template <typename T>
cudaError_t launch_spread_outer(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                const typename Cx<T>::type* c, typename Cx<T>::type* grid,
                                double beta, cudaStream_t s);
template <typename T>
cudaError_t launch_spread_outer_real(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                     const T* c, T* grid, double beta, cudaStream_t s);
template <typename T> size_t spread_outer_smem_bytes(const Geom& g);
template <typename T> size_t interp_smem_bytes(const Geom& g);
// elementwise.cu
template <typename T>
cudaError_t launch_truncate_deconv(const typename Cx<T>::type* grid, const int64_t nf[3],
                                   const int64_t N[3], const T* p1, const T* p2, const T* p3,
                                   int modeord, typename Cx<T>::type* fk, cudaStream_t s);
template <typename T>
cudaError_t launch_pad_precorrect(const typename Cx<T>::type* fk, const int64_t N[3],
                                  const T* p1, const T* p2, const T* p3, int modeord,
                                  const int64_t nf[3], typename Cx<T>::type* grid,
                                  cudaStream_t s);

// pruned.cu: the paper's sigma = 2 split FFT (opts.fft_method = 1): S = 8 contiguous
// N^3 parity-sub-grid spectra (p = px + 2 py + 4 pz) -> retained modes (twiddles, chi,
// D); and the mirror fk -> 8 pre-corrected, twiddled sub-spectra H
template <typename T>
cudaError_t launch_pruned_combine(const typename Cx<T>::type* S, const int64_t N[3], const T* p1,
                                  const T* p2, const T* p3, int modeord, int sign,
                                  typename Cx<T>::type* fk, cudaStream_t st);
template <typename T>
cudaError_t launch_pruned_split(const typename Cx<T>::type* fk, const int64_t N[3], const T* p1,
                                const T* p2, const T* p3, int modeord, int sign,
                                typename Cx<T>::type* H, cudaStream_t st);

// real-valued transforms: R2C half spectrum H (nf3 x nf2 x (nf1/2 + 1), x fastest)
template <typename T>
cudaError_t launch_truncate_deconv_r2c(const typename Cx<T>::type* H, const int64_t nf[3],
                                       const int64_t N[3], const T* p1, const T* p2, const T* p3,
                                       int modeord, int conj_all, typename Cx<T>::type* fk,
                                       cudaStream_t s);
template <typename T>
cudaError_t launch_pad_precorrect_c2r(const typename Cx<T>::type* fk, const int64_t N[3],
                                      const T* p1, const T* p2, const T* p3, int modeord,
                                      int sign_plus, const int64_t nf[3],
                                      typename Cx<T>::type* H, cudaStream_t s);

// host-side window helpers (plan.cu)
int select_width(double eps, int precision, int* w, double* beta, double* eps_used);
double es_phihat(double xi, double beta);

}  // namespace nufft
