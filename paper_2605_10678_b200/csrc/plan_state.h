// plan_state.h -- the plan object behind `nufft_handle` and the host helpers
// shared by plan.cpp (single GPU + ABI) and dist.cpp (z-slab decomposition).
// Private to libnufft.so.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace nufft {
struct DistState;  // dist.cpp
}

struct nufft_plan_s {
    int prec = NUFFT_F64;
    int iflag = -1;
    double eps = 0;
    int w = 0;
    double beta = 0;
    int modeord = 0;
    int64_t N[3] = {0, 0, 0};
    int64_t nf[3] = {0, 0, 0};
    nufft::Geom geom{};
    int64_t nbins = 0;
    cudaStream_t stream = nullptr;
    size_t real_size = 8;
    size_t cplx_size = 16;

    void* d_p[3] = {nullptr, nullptr, nullptr};  // deconvolution factors, precision type
    void* d_grid = nullptr;   // fine grid (one GPU: nf1 nf2 nf3; slab: nf1 nf2 (hz_lo + nzl + hz_hi))
    size_t grid_bytes = 0;    // bytes of d_grid
    void* grid0 = nullptr;    // local plane 0 of the grid (== d_grid on one GPU)
    cufftHandle fft = 0;      // one GPU: 3D plan
    bool fft_ok = false;
    // real-valued transforms (one GPU): R2C / C2R plans, created on first use; the
    // real grid is d_grid[0, nf^3) reals, the half spectrum follows it
    cufftHandle fft_r2c = 0, fft_c2r = 0;
    bool fft_r_ok = false;
    // the paper's pruned sigma = 2 FFT (opts.fft_method = 1, complex transforms): the
    // eight N^3 parity-sub-grid spectra (fft_aux, = the fine grid's size) and the
    // strided sub-grid cuFFT plans (type 1: strided in, type 2: strided out)
    int fft_method = 0;
    void* fft_aux = nullptr;
    size_t fft_aux_bytes = 0;
    cufftHandle fft_sub1 = 0, fft_sub2 = 0;
    bool fft_sub_ok = false;
    // three real fields, SoA (nufft_execute_type2_real3 / nufft_pif_gather_kick)
    void* vgrid = nullptr;  // = d_grid (grown to 3 fields + half spectrum)

    // points (this rank's, after redistribution)
    int64_t Np = -1;
    int64_t cap = 0;
    uint32_t* count = nullptr;
    uint32_t* offset = nullptr;
    uint32_t* offset_key = nullptr;  // (bin, sub-bin) starts when geom.nsub > 1
    uint32_t* blocksum = nullptr;
    uint32_t* bin_of = nullptr;   // setpts scratch when the grid buffer cannot host it
    uint32_t* rank_of = nullptr;
    size_t scratch_cap = 0;
    // TMA tensor map of the complex grid the interp last read (CUtensorMap, 128 B,
    // opaque here): rebuilt when the grid address changes; tmap_state -1 = the driver
    // entry point is unavailable (the interp keeps its row copies)
    alignas(64) unsigned char tmap[128] = {};
    const void* tmap_grid = nullptr;
    int tmap_state = 0;
    void* rec = nullptr;  // Np sorted 32-byte records (PtRec)
    // ablation variants (variants.cu, opts.spread_warps < 0 / opts.interp_method > 0):
    // sorted slot of every caller point, built on first use after each setpts
    int interp_method = 0;
    void* order = nullptr;
    int64_t order_cap = 0;
    bool order_ok = false;
    // interp_method = 3: the Morton walk of the bins (order | key counts | key offsets |
    // scan block sums | bin bases, one allocation), rebuilt after each setpts
    void* morton = nullptr;
    size_t morton_bytes = 0;
    bool morton_ok = false;
    // per-point ES weights (opts.precompute): Np x 3w reals in sorted order
    int precompute = 0;     // opts value: 0 auto, 1 always, -1 never
    void* wts = nullptr;
    size_t wts_bytes = 0;
    bool wts_on = false;    // the last setpts filled wts

    // host staging
    void* stage_in = nullptr;
    size_t stage_in_bytes = 0;
    void* stage_out = nullptr;
    size_t stage_out_bytes = 0;

    // timing
    bool timing = false;
    cudaEvent_t ev0[8] = {};
    cudaEvent_t ev[8] = {};
    bool ev_used[8] = {};

    // distributed (opts.comm != NULL)
    void* comm = nullptr;                 // NufftComm*
    nufft::DistState* dist = nullptr;
    int points_owned = 0;

    size_t bytes = 0;
};

namespace nufft {

enum { EV_SETPTS = 0, EV_SPREAD, EV_FFT, EV_DECONV, EV_PAD, EV_INTERP, EV_COMM, EV_COUNT };

struct StageTimer {
    nufft_plan_s* p;
    int id;
    StageTimer(nufft_plan_s* pl, int i) : p(pl), id(i) {
        if (p->timing) cudaEventRecord(p->ev0[id], p->stream);
    }
    ~StageTimer() {
        if (p->timing) {
            cudaEventRecord(p->ev[id], p->stream);
            p->ev_used[id] = true;
        }
    }
};

inline int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return NUFFT_OK;
    if (e == cudaErrorMemoryAllocation) return NUFFT_ERR_ALLOC;
    return NUFFT_ERR_CUDA;
}

#define NUFFT_CK(expr)                                        \
    do {                                                      \
        cudaError_t e__ = (expr);                             \
        if (e__ != cudaSuccess) return nufft::cuda_status(e__); \
    } while (0)

bool is_device_ptr(const void* ptr);
int dev_alloc(nufft_plan_s* p, void** ptr, size_t bytes);
void dev_free(nufft_plan_s* p, void** ptr, size_t bytes);
// device view of a caller input (host arrays staged into the input buffer at `off`)
int input_view(nufft_plan_s* p, const void* src, size_t bytes, size_t off, size_t total,
               const void** dev);
// device view of a caller output (host arrays staged; finish_output copies back + syncs)
int output_view(nufft_plan_s* p, void* dst, size_t bytes, void** dev, bool* staged);
int finish_output(nufft_plan_s* p, void* dst, const void* dev, size_t bytes, bool staged);

// counting sort of this rank's points (device arrays) into p->rec
int local_sort(nufft_plan_s* p, int64_t Np, const void* x, const void* y, const void* z);
// C: grid0 += C c (grid must be zeroed by the caller); C^T: c = C^T grid0
int do_spread(nufft_plan_s* p, const void* c_dev, void* grid0);
int do_interp(nufft_plan_s* p, const void* grid0, void* c_dev);
// real-valued spread / interp (grid of reals)
int do_spread_real(nufft_plan_s* p, const void* c_dev, void* grid);
int do_interp_real(nufft_plan_s* p, const void* grid, void* c_dev);

// dist.cpp: the z-slab plan
int dist_init(nufft_plan_s* p);
int dist_setpts(nufft_plan_s* p, int64_t Np, const void* x, const void* y, const void* z);
int dist_type1(nufft_plan_s* p, const void* c, void* fk);
int dist_type2(nufft_plan_s* p, const void* fk, void* c);
int dist_type1_real(nufft_plan_s* p, const void* c, void* fk);  // half-spectrum modes
int dist_type2_real(nufft_plan_s* p, const void* fk, void* c);
void dist_destroy(nufft_plan_s* p);
int dist_local_modes(nufft_plan_s* p, int64_t lo[3], int64_t hi[3]);
int64_t dist_user_np(nufft_plan_s* p);  // points the caller passed (before redistribution)

// pif.cu launchers
template <typename T>
cudaError_t launch_pif_poisson(const typename Cx<T>::type* rho, const int64_t N[3],
                               const int64_t lo[3], const int64_t hi[3], double L, int modeord,
                               int xhalf, typename Cx<T>::type* ex, typename Cx<T>::type* ey,
                               typename Cx<T>::type* ez, cudaStream_t s);
template <typename T>
cudaError_t launch_pif_kick(int64_t Np, T* v, const typename Cx<T>::type* e, double s,
                            cudaStream_t st);
template <typename T>
cudaError_t launch_pif_kick_real(int64_t Np, T* v, const T* e, double s, cudaStream_t st);
template <typename T>
cudaError_t launch_pif_drift(int64_t Np, T* x, T* y, T* z, const T* vx, const T* vy, const T* vz,
                             double dt, double L, cudaStream_t s);

// dist_kernels.cu launchers
template <typename T>
cudaError_t launch_owner_count(int64_t Np, const T* z, double L, double scale, int64_t nf3,
                               int nzl, uint32_t* owner, uint32_t* rank_in,
                               unsigned long long* counts, cudaStream_t s);
// PIF particle migration (nufft_pif_migrate): per-destination counts of the
// particles outside this rank's slab; then phase 0 = pack leavers into `send`
// (6 values each, grouped by destination at `off`), compact the staying ones into
// [0, n - nleave); phase 1 = append the nrecv received records there
template <typename T>
cudaError_t launch_migrate_count(int64_t n, const T* z, double L, double scale, int64_t nf3,
                                 int nzl, int me, unsigned long long* counts, cudaStream_t s);
template <typename T>
cudaError_t launch_migrate_move(int64_t n, int64_t nleave, int64_t nrecv, T* const st[6],
                                double L, double scale, int64_t nf3, int nzl, int me,
                                const unsigned long long* off, unsigned long long* cursor,
                                T* send, const T* recv, int64_t* hole, int64_t* lo,
                                int64_t* tail, unsigned long long* nlo_ntail, int phase,
                                cudaStream_t s);
// real transforms on a slab plan (half-spectrum mode layout, x index = k1 in [0, N1/2])
template <typename T>
cudaError_t launch_xy_pack_half(const typename Cx<T>::type* H, const int64_t nf[3], int64_t nzl,
                                const int64_t N[3], int P, int modeord,
                                typename Cx<T>::type* send, cudaStream_t s);
template <typename T>
cudaError_t launch_z_deconv_half(const typename Cx<T>::type* Z, const int64_t nf[3],
                                 const int64_t N[3], int64_t NY, int64_t y0, const T* p1,
                                 const T* p2, const T* p3, int modeord, int conj,
                                 typename Cx<T>::type* fk, cudaStream_t s);
template <typename T>
cudaError_t launch_z_pad_half(const typename Cx<T>::type* fk, const int64_t nf[3],
                              const int64_t N[3], int64_t NY, int64_t y0, const T* p1, const T* p2,
                              const T* p3, int modeord, int conj, typename Cx<T>::type* Z,
                              cudaStream_t s);
template <typename T>
cudaError_t launch_xy_unpad_half(const typename Cx<T>::type* recv, const int64_t nf[3],
                                 int64_t nzl, const int64_t N[3], int P, int modeord,
                                 typename Cx<T>::type* H, cudaStream_t s);
cudaError_t launch_pack_bytes(int64_t Np, int elem_bytes, const void* src, const uint32_t* owner,
                              const uint32_t* rank_in, const unsigned long long* off, void* dst,
                              bool unpack, cudaStream_t s);
template <typename T>
cudaError_t launch_halo_add(int64_t n, typename Cx<T>::type* dst, const typename Cx<T>::type* src,
                            cudaStream_t s);
template <typename T>
cudaError_t launch_xy_pack(const typename Cx<T>::type* G, const int64_t nf[3], int64_t nzl,
                           const int64_t N[3], int P, int modeord, typename Cx<T>::type* send,
                           cudaStream_t s);
template <typename T>
cudaError_t launch_z_deconv(const typename Cx<T>::type* Z, const int64_t nf[3], const int64_t N[3],
                            int64_t NY, int64_t y0, const T* p1, const T* p2, const T* p3,
                            int modeord, typename Cx<T>::type* fk, cudaStream_t s);
template <typename T>
cudaError_t launch_z_pad(const typename Cx<T>::type* fk, const int64_t nf[3], const int64_t N[3],
                         int64_t NY, int64_t y0, const T* p1, const T* p2, const T* p3,
                         int modeord, typename Cx<T>::type* Z, cudaStream_t s);
template <typename T>
cudaError_t launch_xy_unpad(const typename Cx<T>::type* recv, const int64_t nf[3], int64_t nzl,
                            const int64_t N[3], int P, int modeord, typename Cx<T>::type* G,
                            cudaStream_t s);

}  // namespace nufft
