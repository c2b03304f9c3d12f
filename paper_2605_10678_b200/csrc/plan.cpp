// plan.cpp -- the C ABI of libnufft.so (include/nufft.h): plan, setpts,
// execute type 1 / type 2, spread / interp, destroy, info.
//
// Host-side orchestration only: parameter choice, the deconvolution table by
// Gauss-Legendre quadrature (once per plan), device buffers,
// the cuFFT plan, host<->device staging, CUDA-event stage timing.  Every step
// of the NUFFT itself runs in the kernels of sort.cu / spread*.cu / interp.cu /
// elementwise.cu (and cuFFT for the uniform FFT).  Plans with
// opts.comm are z-slab plans whose execute path lives in dist.cpp.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "plan_state.h"

using namespace nufft;

namespace nufft {

// Width rule (reading R1; PAPER.md:181 defers to Barnett 2019):
// w = ceil(log10(1/eps)) + 1 clamped to [2, 16], beta = 2.30 w, sigma = 2.
// fp32 plans clamp eps to >= 1e-7 (single precision cannot resolve less).
int select_width(double eps, int precision, int* w, double* beta, double* eps_used) {
    int st = NUFFT_OK;
    const double lo = precision == NUFFT_F32 ? 1e-7 : 1e-15;
    if (!(eps >= lo)) {
        eps = lo;
        st = NUFFT_WARN_EPS_CLAMPED;
    }
    if (eps > 1e-1) {
        eps = 1e-1;
        st = NUFFT_WARN_EPS_CLAMPED;
    }
    int ww = (int)std::ceil(std::log10(1.0 / eps)) + 1;
    ww = ww < 2 ? 2 : (ww > 16 ? 16 : ww);
    *w = ww;
    *beta = 2.30 * (double)ww;
    *eps_used = eps;
    return st;
}

// phihat(xi) = int_{-1}^{1} exp(beta (sqrt(1 - z^2) - 1)) cos(xi z) dz
// (PAPER.md:178-179), evaluated on theta = asin(z) with a 100-node
// Gauss-Legendre rule whose nodes come from std::legendre + Newton.
namespace {
struct GaussLegendre100 {
    static constexpr int n = 100;
    double nodes[n], weights[n];
    GaussLegendre100() {
        for (int k = 0; k < n; ++k) {
            double t = std::cos(M_PI * (k + 0.75) / (n + 0.5));
            double dp = 1.0;
            for (int it = 0; it < 50; ++it) {
                const double pn = std::legendre(n, t), pm = std::legendre(n - 1, t);
                dp = n * (pm - t * pn) / (1.0 - t * t);
                const double step = pn / dp;
                t -= step;
                if (std::fabs(step) < 1e-16) break;
            }
            const double pn = std::legendre(n, t), pm = std::legendre(n - 1, t);
            dp = n * (pm - t * pn) / (1.0 - t * t);
            nodes[k] = t;
            weights[k] = 2.0 / ((1.0 - t * t) * dp * dp);
        }
    }
};
}  // namespace

double es_phihat(double xi, double beta) {
    // built once, thread-safely (C++11 magic static): plans may be created
    // concurrently from several host threads (one per GPU)
    static const GaussLegendre100 gl;
    const int n = GaussLegendre100::n;
    const double* nodes = gl.nodes;
    const double* weights = gl.weights;
    const double h = 0.5 * M_PI;
    double acc = 0.0;
    for (int k = 0; k < n; ++k) {
        const double th = h * nodes[k];
        const double ct = std::cos(th);
        acc += weights[k] * std::exp(beta * (ct - 1.0)) * std::cos(xi * std::sin(th)) * ct;
    }
    return h * acc;
}

bool is_device_ptr(const void* ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int dev_alloc(nufft_plan_s* p, void** ptr, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *ptr = nullptr;
        return NUFFT_ERR_ALLOC;
    }
    p->bytes += bytes;
    return NUFFT_OK;
}

void dev_free(nufft_plan_s* p, void** ptr, size_t bytes) {
    if (*ptr) {
        cudaFree(*ptr);
        p->bytes -= bytes;
        *ptr = nullptr;
    }
}

int input_view(nufft_plan_s* p, const void* src, size_t bytes, size_t off, size_t total,
               const void** dev) {
    if (bytes == 0 || is_device_ptr(src)) {
        *dev = src;
        return NUFFT_OK;
    }
    if (p->stage_in_bytes < total) {
        dev_free(p, &p->stage_in, p->stage_in_bytes);
        p->stage_in_bytes = 0;
        int st = dev_alloc(p, &p->stage_in, total);
        if (st) return st;
        p->stage_in_bytes = total;
    }
    char* d = static_cast<char*>(p->stage_in) + off;
    NUFFT_CK(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, p->stream));
    *dev = d;
    return NUFFT_OK;
}

int output_view(nufft_plan_s* p, void* dst, size_t bytes, void** dev, bool* staged) {
    *staged = false;
    if (bytes == 0 || is_device_ptr(dst)) {
        *dev = dst;
        return NUFFT_OK;
    }
    if (p->stage_out_bytes < bytes) {
        dev_free(p, &p->stage_out, p->stage_out_bytes);
        p->stage_out_bytes = 0;
        int st = dev_alloc(p, &p->stage_out, bytes);
        if (st) return st;
        p->stage_out_bytes = bytes;
    }
    *dev = p->stage_out;
    *staged = true;
    return NUFFT_OK;
}

int finish_output(nufft_plan_s* p, void* dst, const void* dev, size_t bytes, bool staged) {
    if (!staged) return NUFFT_OK;
    NUFFT_CK(cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDeviceToHost, p->stream));
    NUFFT_CK(cudaStreamSynchronize(p->stream));
    return NUFFT_OK;
}

template <typename T>
PtsView<T> pts_view(nufft_plan_s* p) {
    PtsView<T> v;
    v.offset = p->offset;
    v.offset_sub = p->offset_key ? p->offset_key : p->offset;
    v.rec = static_cast<const PtRec<T>*>(p->rec);
    v.w = p->wts_on ? static_cast<const T*>(p->wts) : nullptr;
    return v;
}

int local_sort(nufft_plan_s* p, int64_t Np, const void* xd, const void* yd, const void* zd) {
    if (Np >= (int64_t)1 << 31) return NUFFT_ERR_NPTS;
    int st = NUFFT_OK;
    if (Np > p->cap) {
        dev_free(p, &p->rec, 32 * p->cap);
        p->cap = 0;
        // a slab plan's local count drifts step to step (migration): 6 % slack there
        const size_t n = (size_t)(p->dist ? Np + Np / 16 : Np);
        if ((st = dev_alloc(p, &p->rec, 32 * n))) {
            p->Np = -1;
            return st;
        }
        p->cap = (int64_t)n;
    }
    // bin / rank scratch (dead once the records are written): inside the grid buffer
    // when it is large enough -- no grid is live during setpts -- else own buffers
    uint32_t* bin_of;
    uint32_t* rank_of;
    if (p->grid_bytes >= 8 * (size_t)Np) {
        bin_of = static_cast<uint32_t*>(p->d_grid);
        rank_of = bin_of + Np;
    } else {
        if ((size_t)Np > p->scratch_cap) {
            dev_free(p, (void**)&p->bin_of, 4 * p->scratch_cap);
            dev_free(p, (void**)&p->rank_of, 4 * p->scratch_cap);
            p->scratch_cap = 0;
            const size_t n = (size_t)(p->dist ? Np + Np / 16 : Np);
            st = dev_alloc(p, (void**)&p->bin_of, 4 * n);
            if (!st) st = dev_alloc(p, (void**)&p->rank_of, 4 * n);
            if (st) {
                p->Np = -1;
                return st;
            }
            p->scratch_cap = n;
        }
        bin_of = p->bin_of;
        rank_of = p->rank_of;
    }
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_bin_sort<double>(p->geom, Np, static_cast<const double*>(xd),
                                         static_cast<const double*>(yd),
                                         static_cast<const double*>(zd), p->count,
                                         p->offset_key ? p->offset_key : p->offset, p->offset,
                                         p->blocksum, bin_of, rank_of,
                                         static_cast<PtRec<double>*>(p->rec), p->nbins, p->stream));
    else
        NUFFT_CK(launch_bin_sort<float>(p->geom, Np, static_cast<const float*>(xd),
                                        static_cast<const float*>(yd),
                                        static_cast<const float*>(zd), p->count,
                                         p->offset_key ? p->offset_key : p->offset, p->offset,
                                        p->blocksum, bin_of, rank_of,
                                        static_cast<PtRec<float>*>(p->rec), p->nbins, p->stream));
    p->Np = Np;
    p->order_ok = false;
    p->morton_ok = false;
    // per-point ES weights, reused by every execute on these points
    p->wts_on = false;
    // auto (0): widths w >= 6 (B200, scripts/gpu_precompute.sh, step ms table / in-kernel
    // phi: C2b fp32 w=7 1.723 / 1.749, C3 fp64 w=7 124.3 / 132.3; at w = 5 the table
    // does not pay: C2a fp32 1.314 / 1.286, C3e4 fp64 89.3 / 88.8); 1 forces it, -1 never
    if ((p->precompute > 0 || (p->precompute == 0 && p->w >= 6)) && Np > 0) {
        const size_t need = (size_t)Np * 3 * (size_t)p->w * p->real_size;
        bool want = p->precompute > 0 || p->wts_bytes >= need;  // no query when it fits
        if (!want) {  // auto: when the table fits in a quarter of the device memory
            // (cudaMemGetInfo synchronises: asked only when a (re)allocation is needed)
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
                want = need <= tot / 4 && (p->wts_bytes >= need || need + (64u << 20) < fr);
            else
                cudaGetLastError();
        }
        if (want) {
            if (p->wts_bytes < need) {
                dev_free(p, &p->wts, p->wts_bytes);
                p->wts_bytes = 0;
                const size_t n = p->dist ? need + need / 16 : need;
                if ((st = dev_alloc(p, &p->wts, n))) {
                    if (p->precompute > 0) return st;
                    st = NUFFT_OK;  // auto: fall back to evaluating phi in the kernels
                } else {
                    p->wts_bytes = n;
                }
            }
            if (p->wts_bytes >= need) {
                if (p->prec == NUFFT_F64)
                    NUFFT_CK(launch_weights<double>(static_cast<const PtRec<double>*>(p->rec), Np,
                                                    p->w, p->beta, static_cast<double*>(p->wts),
                                                    p->stream));
                else
                    NUFFT_CK(launch_weights<float>(static_cast<const PtRec<float>*>(p->rec), Np,
                                                   p->w, p->beta, static_cast<float*>(p->wts),
                                                   p->stream));
                p->wts_on = true;
            }
        }
    }
    return NUFFT_OK;
}

// caller-order walk of the ablation variants: order[t] = sorted slot of caller point t
static int caller_order(nufft_plan_s* p, const uint32_t** out) {
    if (!p->order_ok) {
        if (p->Np > p->order_cap) {
            dev_free(p, &p->order, 4 * p->order_cap);
            p->order_cap = 0;
            int st = dev_alloc(p, &p->order, 4 * (size_t)p->Np);
            if (st) return st;
            p->order_cap = p->Np;
        }
        NUFFT_CK(p->prec == NUFFT_F64
                     ? launch_caller_order<double>(static_cast<const PtRec<double>*>(p->rec), p->Np,
                                                   static_cast<uint32_t*>(p->order), p->stream)
                     : launch_caller_order<float>(static_cast<const PtRec<float>*>(p->rec), p->Np,
                                                  static_cast<uint32_t*>(p->order), p->stream));
        p->order_ok = true;
    }
    *out = static_cast<const uint32_t*>(p->order);
    return NUFFT_OK;
}

int do_spread(nufft_plan_s* p, const void* c_dev, void* grid0) {
    StageTimer tm(p, EV_SPREAD);
    if (p->geom.spread_warps == -3) {  // the paper's Tiled Spread (shared atomics)
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_spread_tiled<double>(p->geom, pts_view<double>(p), p->nbins,
                                                 static_cast<const double2*>(c_dev),
                                                 static_cast<double2*>(grid0), p->beta, p->stream));
        else
            NUFFT_CK(launch_spread_tiled<float>(p->geom, pts_view<float>(p), p->nbins,
                                                static_cast<const float2*>(c_dev),
                                                static_cast<float2*>(grid0), p->beta, p->stream));
        return NUFFT_OK;
    }
    if (p->geom.spread_warps < 0) {  // Atomic Spread (-1 caller order, -2 bin-sorted)
        const uint32_t* order = nullptr;
        if (p->geom.spread_warps == -1) {
            int st = caller_order(p, &order);
            if (st) return st;
        }
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_spread_atomic<double>(p->geom, pts_view<double>(p), p->nbins, order,
                                                  p->Np, static_cast<const double2*>(c_dev),
                                                  static_cast<double2*>(grid0), p->beta, p->stream));
        else
            NUFFT_CK(launch_spread_atomic<float>(p->geom, pts_view<float>(p), p->nbins, order,
                                                 p->Np, static_cast<const float2*>(c_dev),
                                                 static_cast<float2*>(grid0), p->beta, p->stream));
        return NUFFT_OK;
    }
    if (p->geom.spread_warps == 3) {  // tensor-core GEMM spread (plan checked: fp32, T = 16 - w)
        NUFFT_CK(launch_spread_tc(p->geom, pts_view<float>(p), p->nbins,
                                  static_cast<const float2*>(c_dev), static_cast<float2*>(grid0),
                                  p->beta, p->stream));
        return NUFFT_OK;
    }
    if (p->geom.spread_warps == 5) {  // sub-bin register rows (plan checked the geometry)
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_spread_sub<double>(p->geom, pts_view<double>(p), p->nbins,
                                               static_cast<const double2*>(c_dev),
                                               static_cast<double2*>(grid0), p->beta, p->stream));
        else
            NUFFT_CK(launch_spread_sub<float>(p->geom, pts_view<float>(p), p->nbins,
                                              static_cast<const float2*>(c_dev),
                                              static_cast<float2*>(grid0), p->beta, p->stream));
        return NUFFT_OK;
    }
    const bool rows = p->geom.spread_warps == 1;  // register-row kernel (plan checked it applies)
    const bool outer = p->geom.spread_warps == 2;  // plane outer-product kernel (ditto)
    if (outer && p->prec == NUFFT_F64)
        NUFFT_CK(launch_spread_outer<double>(p->geom, pts_view<double>(p), p->nbins,
                                             static_cast<const double2*>(c_dev),
                                             static_cast<double2*>(grid0), p->beta, p->stream));
    else if (outer)
        NUFFT_CK(launch_spread_outer<float>(p->geom, pts_view<float>(p), p->nbins,
                                            static_cast<const float2*>(c_dev),
                                            static_cast<float2*>(grid0), p->beta, p->stream));
    else if (rows && p->prec == NUFFT_F64)
        NUFFT_CK(launch_spread_rows<double>(p->geom, pts_view<double>(p), p->nbins,
                                            static_cast<const double2*>(c_dev),
                                            static_cast<double2*>(grid0), p->beta, p->stream));
    else if (rows)
        NUFFT_CK(launch_spread_rows<float>(p->geom, pts_view<float>(p), p->nbins,
                                           static_cast<const float2*>(c_dev),
                                           static_cast<float2*>(grid0), p->beta, p->stream));
    else if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_spread<double>(p->geom, pts_view<double>(p), p->nbins,
                                       static_cast<const double2*>(c_dev),
                                       static_cast<double2*>(grid0), p->beta, p->stream));
    else
        NUFFT_CK(launch_spread<float>(p->geom, pts_view<float>(p), p->nbins,
                                      static_cast<const float2*>(c_dev),
                                      static_cast<float2*>(grid0), p->beta, p->stream));
    return NUFFT_OK;
}

// real-valued transforms: real strengths / grid / outputs
int do_spread_real(nufft_plan_s* p, const void* c_dev, void* grid) {
    StageTimer tm(p, EV_SPREAD);
    Geom g = p->geom;
    // no real register-row or ablation kernels: real transforms take the z-plane owners
    if (g.spread_warps == 1 || g.spread_warps < 0) g.spread_warps = 8;
    if (g.spread_warps == 3) g.spread_warps = 2;  // the register outer products
    if (g.spread_warps == 5 && p->prec == NUFFT_F64)
        NUFFT_CK(launch_spread_sub_real<double>(g, pts_view<double>(p), p->nbins,
                                                static_cast<const double*>(c_dev),
                                                static_cast<double*>(grid), p->beta, p->stream));
    else if (g.spread_warps == 5)
        NUFFT_CK(launch_spread_sub_real<float>(g, pts_view<float>(p), p->nbins,
                                               static_cast<const float*>(c_dev),
                                               static_cast<float*>(grid), p->beta, p->stream));
    else if (g.spread_warps == 2 && p->prec == NUFFT_F64)
        NUFFT_CK(launch_spread_outer_real<double>(g, pts_view<double>(p), p->nbins,
                                                  static_cast<const double*>(c_dev),
                                                  static_cast<double*>(grid), p->beta, p->stream));
    else if (g.spread_warps == 2)
        NUFFT_CK(launch_spread_outer_real<float>(g, pts_view<float>(p), p->nbins,
                                                 static_cast<const float*>(c_dev),
                                                 static_cast<float*>(grid), p->beta, p->stream));
    else if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_spread_real<double>(g, pts_view<double>(p), p->nbins,
                                            static_cast<const double*>(c_dev),
                                            static_cast<double*>(grid), p->beta, p->stream));
    else
        NUFFT_CK(launch_spread_real<float>(g, pts_view<float>(p), p->nbins,
                                           static_cast<const float*>(c_dev),
                                           static_cast<float*>(grid), p->beta, p->stream));
    return NUFFT_OK;
}

int do_interp_real(nufft_plan_s* p, const void* grid, void* c_dev) {
    StageTimer tm(p, EV_INTERP);
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_interp_real<double>(p->geom, pts_view<double>(p), p->nbins,
                                            static_cast<const double*>(grid),
                                            static_cast<double*>(c_dev), p->beta, p->stream));
    else
        NUFFT_CK(launch_interp_real<float>(p->geom, pts_view<float>(p), p->nbins,
                                           static_cast<const float*>(grid),
                                           static_cast<float*>(c_dev), p->beta, p->stream));
    return NUFFT_OK;
}

int ensure_real_fft(nufft_plan_s* p) {
    if (p->fft_r_ok) return NUFFT_OK;
    const bool f64 = p->prec == NUFFT_F64;
    const int n3 = (int)p->nf[2], n2 = (int)p->nf[1], n1 = (int)p->nf[0];
    if (cufftPlan3d(&p->fft_r2c, n3, n2, n1, f64 ? CUFFT_D2Z : CUFFT_R2C) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    if (cufftPlan3d(&p->fft_c2r, n3, n2, n1, f64 ? CUFFT_Z2D : CUFFT_C2R) != CUFFT_SUCCESS) {
        cufftDestroy(p->fft_r2c);
        return NUFFT_ERR_CUFFT;
    }
    p->fft_r_ok = true;
    size_t w1 = 0, w2 = 0;
    cufftGetSize(p->fft_r2c, &w1);
    cufftGetSize(p->fft_c2r, &w2);
    p->bytes += w1 + w2;
    if (cufftSetStream(p->fft_r2c, p->stream) != CUFFT_SUCCESS ||
        cufftSetStream(p->fft_c2r, p->stream) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    return NUFFT_OK;
}

void* half_spectrum(nufft_plan_s* p) {
    return static_cast<char*>(p->d_grid) + (size_t)(p->nf[0] * p->nf[1] * p->nf[2]) * p->real_size;
}

// The interp's subgrid box as a TMA tensor map over the complex grid at grid0
// (reals: {2 nf1, nf2, nz_loc}, box {2 pitch, T2 + w, T3 + w}; the box row is the
// kernel's padded smem row, columns past the grid are zero-filled and unused).
// Returns the map, or nullptr (the kernel then stages every bin row by row).
static const void* interp_tmap(nufft_plan_s* p, const void* grid0) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    // resolved once, thread-safely; NUFFT_NO_TMAP=1 is the ablation switch
    // (profiles/README.md)
    static const Encode encode = []() -> Encode {
        if (std::getenv("NUFFT_NO_TMAP")) return nullptr;
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<Encode>(fn);
        return nullptr;
    }();
    if (p->tmap_state < 0 || grid0 == nullptr) return nullptr;
    if (p->tmap_state == 1 && p->tmap_grid == grid0) return p->tmap;
    const int w = p->w, r = (int)p->real_size;
    const int pitch = interp_tile_pitch(2 * r, p->geom.T[0], w,
                                        p->geom.nsub > 1 && w <= 6);  // the sub-bin gather's rows
    const cuuint64_t dim[3] = {(cuuint64_t)(2 * p->nf[0]), (cuuint64_t)p->nf[1],
                               (cuuint64_t)p->geom.nz_loc};
    const cuuint64_t stride[2] = {(cuuint64_t)(2 * p->nf[0] * r),
                                  (cuuint64_t)(2 * p->nf[0] * p->nf[1] * r)};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * pitch), (cuuint32_t)(p->geom.T[1] + w),
                               (cuuint32_t)(p->geom.T[2] + w)};
    const cuuint32_t estride[3] = {1, 1, 1};
    // plan-level impossibility (no driver entry point, box or pitch out of range):
    // latch TMA staging off for this plan
    if (!encode || box[0] > 256 || box[1] > 256 || box[2] > 256 || (box[0] * r) % 16 ||
        (stride[0] % 16)) {
        p->tmap_state = -1;
        return nullptr;
    }
    // per-grid failure (a misaligned caller grid, an encode refused for this address):
    // stage this call row by row, keep TMA for later grids
    if (reinterpret_cast<uintptr_t>(grid0) % 16) return nullptr;
    if (encode(reinterpret_cast<CUtensorMap*>(p->tmap),
               r == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
               const_cast<void*>(grid0), dim, stride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        if (p->tmap_state == 1) p->tmap_state = 0;  // the cached map belongs to another grid
        return nullptr;
    }
    p->tmap_state = 1;
    p->tmap_grid = grid0;
    return p->tmap;
}

// Morton walk of the bins (interp_method = 3): order[t] = sorted slot of point t
static int morton_order(nufft_plan_s* p, const uint32_t** out) {
    const size_t nk = morton_keys(p->geom);
    const size_t n_order = (size_t)p->Np, n_blk = scan_blocksum_elems((int64_t)nk);
    const size_t need = 4 * (n_order + nk + (nk + 1) + n_blk + (size_t)p->nbins) + 64;
    if (!p->morton_ok) {
        if (need > p->morton_bytes) {
            dev_free(p, &p->morton, p->morton_bytes);
            p->morton_bytes = 0;
            int st = dev_alloc(p, &p->morton, need);
            if (st) return st;
            p->morton_bytes = need;
        }
        uint32_t* order = static_cast<uint32_t*>(p->morton);
        uint32_t* kc = order + n_order;
        uint32_t* ko = kc + nk;
        uint32_t* bs = ko + nk + 1;
        uint32_t* bb = bs + n_blk;
        NUFFT_CK(launch_morton_order(p->geom, p->offset, p->nbins, p->Np, kc, ko, bs, bb, order,
                                     p->stream));
        p->morton_ok = true;
    }
    *out = static_cast<const uint32_t*>(p->morton);
    return NUFFT_OK;
}

int do_interp(nufft_plan_s* p, const void* grid0, void* c_dev) {
    StageTimer tm(p, EV_INTERP);
    if (p->interp_method > 0) {  // Direct Interpolation (1 caller order, 2 bin-sorted, 3 Morton)
        const uint32_t* order = nullptr;
        if (p->interp_method == 1) {
            int st = caller_order(p, &order);
            if (st) return st;
        } else if (p->interp_method == 3) {
            int st = morton_order(p, &order);
            if (st) return st;
        }
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_interp_direct<double>(p->geom, pts_view<double>(p), p->nbins, order,
                                                  p->Np, static_cast<const double2*>(grid0),
                                                  static_cast<double2*>(c_dev), p->beta, p->stream));
        else
            NUFFT_CK(launch_interp_direct<float>(p->geom, pts_view<float>(p), p->nbins, order,
                                                 p->Np, static_cast<const float2*>(grid0),
                                                 static_cast<float2*>(c_dev), p->beta, p->stream));
        return NUFFT_OK;
    }
    const void* tmap = interp_tmap(p, grid0);
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_interp<double>(p->geom, pts_view<double>(p), p->nbins,
                                       static_cast<const double2*>(grid0),
                                       static_cast<double2*>(c_dev), p->beta, p->stream, tmap));
    else
        NUFFT_CK(launch_interp<float>(p->geom, pts_view<float>(p), p->nbins,
                                      static_cast<const float2*>(grid0),
                                      static_cast<float2*>(c_dev), p->beta, p->stream, tmap));
    return NUFFT_OK;
}

}  // namespace nufft

namespace {

// Default bin edge by width (measured on B200: profiles/tile_sweep_r01.txt, the
// exhaustive sweep of scripts/tile_sweep.py): the register outer-product spread
// takes a 16 x 16 x 16 subgrid (T = 16 - w) -- the default for fp32 and for fp64
// with 6 <= w <= 12; fp64 with w <= 5 and every w >= 13 use the shared-memory
// z-plane spread with T = 8 (w = 13: 93 vs 122 ms at 1 point per cell, T = 4);
// never larger than the grid allows.
int default_tile(int w, int prec, int64_t nf) {
    int t = ((prec == NUFFT_F64 && w <= 5) || w >= 13) ? 8 : 16 - w;
    if (t < 4) t = 4;
    if (t > 64) t = 64;
    if (t > nf - w - 2) t = (int)(nf - w - 2);  // T + w + 2 <= nf: one-step periodic wraps, <= 2 row segments
    return t;
}

bool spread_sub_width(int w) { return w >= 2 && w <= 7; }

// Sub-bin kernels (spread_warps = 5): Gs[d] stencil bases per sub-bin and axis
// (SubGeom in sub_common.cuh: 9 - w, and 6 in z for w = 7), ns sub-bins per bin
// axis, T = ns G - 1 (la in [0, T] covers ns G values); ns chosen so that the bin
// edge T + w stays <= 20 cells (points per bin ~ (T + 1)^3)
int sub_default_tile(int w, int axis, int64_t nf) {
    int Gs[3];
    sub_extents(w, Gs);
    const int G = Gs[axis];
    int ns = 1;
    while ((ns + 1) * G - 1 + w <= 20) ++ns;
    int t = ns * G - 1;
    while (t > 0 && t + w + 2 > nf) t -= G;  // tiny grids
    return t;
}

int ensure_complex_fft(nufft_plan_s* p) {
    if (p->fft_ok) return NUFFT_OK;
    if (cufftPlan3d(&p->fft, (int)p->nf[2], (int)p->nf[1], (int)p->nf[0],
                    p->prec == NUFFT_F64 ? CUFFT_Z2Z : CUFFT_C2C) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    p->fft_ok = true;
    size_t ws = 0;
    cufftGetSize(p->fft, &ws);
    p->bytes += ws;
    return cufftSetStream(p->fft, p->stream) == CUFFT_SUCCESS ? NUFFT_OK : NUFFT_ERR_CUFFT;
}

int do_fft(nufft_plan_s* p, int sign) {
    int st = ensure_complex_fft(p);
    if (st) return st;
    StageTimer tm(p, EV_FFT);
    const int dir = sign < 0 ? CUFFT_FORWARD : CUFFT_INVERSE;
    cufftResult r;
    if (p->prec == NUFFT_F64)
        r = cufftExecZ2Z(p->fft, static_cast<cufftDoubleComplex*>(p->d_grid),
                         static_cast<cufftDoubleComplex*>(p->d_grid), dir);
    else
        r = cufftExecC2C(p->fft, static_cast<cufftComplex*>(p->d_grid),
                         static_cast<cufftComplex*>(p->d_grid), dir);
    return r == CUFFT_SUCCESS ? NUFFT_OK : NUFFT_ERR_CUFFT;
}

// The paper's pruned sigma = 2 FFT (pruned.cu): two strided cuFFT N^3 plans and the
// buffer of the eight parity-sub-grid spectra, created on first use.
int ensure_pruned(nufft_plan_s* p) {
    if (p->fft_sub_ok) return NUFFT_OK;
    const int64_t nm = p->N[0] * p->N[1] * p->N[2];
    const size_t need = (size_t)(8 * nm) * p->cplx_size;
    if (p->fft_aux_bytes < need) {
        dev_free(p, &p->fft_aux, p->fft_aux_bytes);
    dev_free(p, &p->morton, p->morton_bytes);
        p->fft_aux_bytes = 0;
        int st = dev_alloc(p, &p->fft_aux, need);
        if (st) return st;
        p->fft_aux_bytes = need;
    }
    int n[3] = {(int)p->N[2], (int)p->N[1], (int)p->N[0]};
    // sub-grid element (z, y, x) of parity p sits at fine index 2 (x + nf1 (y + nf2 z)) + off(p)
    int strided[3] = {(int)p->N[2], (int)p->nf[1], (int)p->nf[0]};
    const cufftType ty = p->prec == NUFFT_F64 ? CUFFT_Z2Z : CUFFT_C2C;
    if (cufftPlanMany(&p->fft_sub1, 3, n, strided, 2, 1, n, 1, (int)nm, ty, 1) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    if (cufftPlanMany(&p->fft_sub2, 3, n, n, 1, (int)nm, strided, 2, 1, ty, 1) != CUFFT_SUCCESS) {
        cufftDestroy(p->fft_sub1);
        return NUFFT_ERR_CUFFT;
    }
    p->fft_sub_ok = true;
    size_t w1 = 0, w2 = 0;
    cufftGetSize(p->fft_sub1, &w1);
    cufftGetSize(p->fft_sub2, &w2);
    p->bytes += w1 + w2;
    if (cufftSetStream(p->fft_sub1, p->stream) != CUFFT_SUCCESS ||
        cufftSetStream(p->fft_sub2, p->stream) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    return NUFFT_OK;
}

// fine-grid offset of parity sub-grid q = px + 2 py + 4 pz
size_t parity_offset(const nufft_plan_s* p, int q) {
    return (size_t)((q & 1) + ((q >> 1) & 1) * p->nf[0] + ((q >> 2) & 1) * p->nf[0] * p->nf[1]);
}

int sub_fft(nufft_plan_s* p, cufftHandle h, void* in, void* out, int sign) {
    const int dir = sign < 0 ? CUFFT_FORWARD : CUFFT_INVERSE;
    cufftResult r;
    if (p->prec == NUFFT_F64)
        r = cufftExecZ2Z(h, static_cast<cufftDoubleComplex*>(in),
                         static_cast<cufftDoubleComplex*>(out), dir);
    else
        r = cufftExecC2C(h, static_cast<cufftComplex*>(in), static_cast<cufftComplex*>(out), dir);
    return r == CUFFT_SUCCESS ? NUFFT_OK : NUFFT_ERR_CUFFT;
}

// type 1 after the spread: eight strided N^3 FFTs of the fine grid's parity sub-grids,
// then twiddle combine + truncation + deconvolution
int pruned_type1(nufft_plan_s* p, void* fkd) {
    int st = ensure_pruned(p);
    if (st) return st;
    const int64_t nm = p->N[0] * p->N[1] * p->N[2];
    {
        StageTimer tm(p, EV_FFT);
        for (int q = 0; q < 8; ++q) {
            char* in = static_cast<char*>(p->d_grid) + parity_offset(p, q) * p->cplx_size;
            char* out = static_cast<char*>(p->fft_aux) + (size_t)(q * nm) * p->cplx_size;
            if ((st = sub_fft(p, p->fft_sub1, in, out, p->iflag))) return st;
        }
    }
    StageTimer tm(p, EV_DECONV);
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_pruned_combine<double>(
            static_cast<const double2*>(p->fft_aux), p->N, static_cast<const double*>(p->d_p[0]),
            static_cast<const double*>(p->d_p[1]), static_cast<const double*>(p->d_p[2]),
            p->modeord, p->iflag, static_cast<double2*>(fkd), p->stream));
    else
        NUFFT_CK(launch_pruned_combine<float>(
            static_cast<const float2*>(p->fft_aux), p->N, static_cast<const float*>(p->d_p[0]),
            static_cast<const float*>(p->d_p[1]), static_cast<const float*>(p->d_p[2]),
            p->modeord, p->iflag, static_cast<float2*>(fkd), p->stream));
    return NUFFT_OK;
}

// type 2 before the interp: D + conjugate twiddles into eight N^3 sub-spectra, then
// eight inverse N^3 FFTs writing the fine grid's parity sub-grids (stride 2)
int pruned_type2(nufft_plan_s* p, const void* fkd) {
    int st = ensure_pruned(p);
    if (st) return st;
    const int64_t nm = p->N[0] * p->N[1] * p->N[2];
    {
        StageTimer tm(p, EV_PAD);
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_pruned_split<double>(
                static_cast<const double2*>(fkd), p->N, static_cast<const double*>(p->d_p[0]),
                static_cast<const double*>(p->d_p[1]), static_cast<const double*>(p->d_p[2]),
                p->modeord, -p->iflag, static_cast<double2*>(p->fft_aux), p->stream));
        else
            NUFFT_CK(launch_pruned_split<float>(
                static_cast<const float2*>(fkd), p->N, static_cast<const float*>(p->d_p[0]),
                static_cast<const float*>(p->d_p[1]), static_cast<const float*>(p->d_p[2]),
                p->modeord, -p->iflag, static_cast<float2*>(p->fft_aux), p->stream));
    }
    StageTimer tm(p, EV_FFT);
    for (int q = 0; q < 8; ++q) {
        char* in = static_cast<char*>(p->fft_aux) + (size_t)(q * nm) * p->cplx_size;
        char* out = static_cast<char*>(p->d_grid) + parity_offset(p, q) * p->cplx_size;
        if ((st = sub_fft(p, p->fft_sub2, in, out, -p->iflag))) return st;
    }
    return NUFFT_OK;
}

int64_t user_np(nufft_plan_s* p) { return p->dist ? dist_user_np(p) : p->Np; }

// bytes of one complex fine grid nf1 nf2 nf3 (the caller's grid of nufft_spread /
// nufft_interp; p->grid_bytes is the plan's grid buffer, which may be larger)
size_t cgrid_bytes(const nufft_plan_s* p) {
    return (size_t)(p->nf[0] * p->nf[1] * p->nf[2]) * p->cplx_size;
}

}  // namespace

extern "C" {

int nufft_default_opts(nufft_opts* o) {
    if (!o) return NUFFT_ERR_ARG;
    std::memset(o, 0, sizeof(*o));
    o->L = 2.0 * M_PI;
    return NUFFT_OK;
}

const char* nufft_strerror(int code) {
    switch (code) {
        case NUFFT_OK: return "ok";
        case NUFFT_WARN_EPS_CLAMPED: return "warning: eps clamped to the supported range";
        case NUFFT_ERR_ARG: return "invalid argument";
        case NUFFT_ERR_MODES: return "invalid mode counts (need even N >= 2 with 2N >= w + 3)";
        case NUFFT_ERR_NPTS: return "invalid number of points";
        case NUFFT_ERR_NOT_SET: return "points not set (call nufft_setpts first)";
        case NUFFT_ERR_ALLOC: return "device allocation failed";
        case NUFFT_ERR_CUDA: return "CUDA error";
        case NUFFT_ERR_CUFFT: return "cuFFT error";
        case NUFFT_ERR_NCCL: return "NCCL error";
        case NUFFT_ERR_UNSUPPORTED: return "unsupported option";
        default: return "unknown status";
    }
}

int nufft_plan(int64_t N1, int64_t N2, int64_t N3, int iflag, double eps, int precision,
               const nufft_opts* opts, nufft_handle* out) {
    if (!out) return NUFFT_ERR_ARG;
    *out = nullptr;
    if (precision != NUFFT_F32 && precision != NUFFT_F64) return NUFFT_ERR_ARG;
    nufft_opts o;
    if (opts) o = *opts;
    else nufft_default_opts(&o);
    if (!(o.L > 0) || (o.modeord != 0 && o.modeord != 1)) return NUFFT_ERR_ARG;
    if (o.spread_warps != 0 && o.spread_warps != 1 && o.spread_warps != 2 &&
        o.spread_warps != 3 && o.spread_warps != 4 && o.spread_warps != 5 && o.spread_warps != 8 &&
        o.spread_warps != -1 && o.spread_warps != -2 && o.spread_warps != -3)
        return NUFFT_ERR_ARG;
    if (o.interp_method < 0 || o.interp_method > 3) return NUFFT_ERR_ARG;
    if (o.fft_method < 0 || o.fft_method > 1 || (o.fft_method == 1 && o.comm))
        return o.fft_method == 1 && o.comm ? NUFFT_ERR_UNSUPPORTED : NUFFT_ERR_ARG;

    nufft_plan_s* p = new (std::nothrow) nufft_plan_s();
    if (!p) return NUFFT_ERR_ALLOC;
    int status = select_width(eps, precision, &p->w, &p->beta, &p->eps);
    const int64_t Nv[3] = {N1, N2, N3};
    for (int d = 0; d < 3; ++d) {
        if (Nv[d] < 2 || (Nv[d] & 1) || 2 * Nv[d] < p->w + 3) {
            delete p;
            return NUFFT_ERR_MODES;
        }
        p->N[d] = Nv[d];
        p->nf[d] = 2 * Nv[d];  // sigma = 2 (reading R8)
    }
    p->prec = precision;
    p->iflag = iflag >= 0 ? 1 : -1;
    p->modeord = o.modeord;
    p->stream = static_cast<cudaStream_t>(o.stream);
    p->real_size = precision == NUFFT_F64 ? 8 : 4;
    p->cplx_size = 2 * p->real_size;
    p->timing = o.timing != 0;
    p->comm = o.comm;
    p->points_owned = o.points_owned;
    if (o.precompute < -1 || o.precompute > 1) {
        delete p;
        return NUFFT_ERR_ARG;
    }
    p->precompute = o.precompute;
    p->interp_method = o.interp_method;
    p->fft_method = o.fft_method;

    Geom& g = p->geom;
    g.nsub = 1;
    g.Gs[0] = g.Gs[1] = g.Gs[2] = 0;
    // sub-bin register-row spread (spread_sub.cu): opts.spread_warps = 5, and the
    // default for fp64 at w <= 6 (C3e4 / C4 on B200: spread 51.9 -> 18.5 ms, 416 -> 155 ms)
    // (a caller's tile that is not a whole number of sub-bins keeps the other kernels)
    bool sub_tiles = true;
    int Gs[3];
    sub_extents(p->w, Gs);
    for (int d = 0; d < 3; ++d)
        if (o.tile[d] > 0 && (o.tile[d] + 1) % Gs[d] != 0) sub_tiles = false;
    const bool sub = o.spread_warps == 5 || (o.spread_warps == 0 && precision == NUFFT_F64 &&
                                             spread_sub_width(p->w) && sub_tiles);
    if (sub && !spread_sub_width(p->w)) {
        delete p;
        return NUFFT_ERR_UNSUPPORTED;
    }
    for (int d = 0; d < 3; ++d) {
        g.nf[d] = p->nf[d];
        int t = o.tile[d] > 0 ? o.tile[d]
                : sub         ? sub_default_tile(p->w, d, p->nf[d])
                              : default_tile(p->w, precision, p->nf[d]);
        if (t < 1 || t > 255 || t + p->w + 2 > p->nf[d]) {
            delete p;
            return NUFFT_ERR_ARG;
        }
        g.T[d] = t;
        g.nb[d] = (int)((p->nf[d] + t - 1) / t);
        g.scale[d] = (double)p->nf[d] / o.L;
    }
    if (sub) {  // bins of ns_d sub-bins of Gs_d stencil bases: T_d + 1 = ns_d Gs_d
        sub_extents(p->w, g.Gs);
        g.nsub = 1;
        for (int d = 0; d < 3; ++d) {
            if ((g.T[d] + 1) % g.Gs[d]) {
                delete p;
                return NUFFT_ERR_ARG;
            }
            g.ns[d] = (g.T[d] + 1) / g.Gs[d];
            g.nsub *= g.ns[d];
        }
    }
    g.L = o.L;
    g.w = p->w;
    g.z_lo = 0;
    g.nz_loc = p->nf[2];
    g.zper = 1;
    g.hz_lo = 0;
    g.hz_hi = 0;
    // spread kernel: 1 = register rows, 2 = register outer products (both need
    // w <= 12 and T = 16 - w), 4 / 8 = shared-memory z-plane owners with that many
    // warps; 0 = outer products when they apply, else 8 z-plane owners (the
    // fastest on B200 per precision and width, profiles/README.md)
    g.spread_warps = sub ? 5 : o.spread_warps;
    if (g.spread_warps == 0) g.spread_warps = spread_outer_applies(g) ? 2 : 8;
    if ((g.spread_warps == 1 && !spread_rows_applies(g)) ||
        (g.spread_warps == 2 && !spread_outer_applies(g)) ||
        (g.spread_warps == 3 && (precision != NUFFT_F32 || !spread_tc_applies(g)))) {
        delete p;
        return NUFFT_ERR_UNSUPPORTED;
    }

    // the (T + w)^3 subgrid (+ staging) of the spread / interp kernels must fit in
    // the opt-in shared memory of one CTA
    {
        int dev = 0, smem_max = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) !=
            cudaSuccess) {
            cudaGetLastError();
            delete p;
            return NUFFT_ERR_CUDA;
        }
        const bool rows = g.spread_warps == 1, outer = g.spread_warps == 2 || g.spread_warps == 3;
        const bool subk = g.spread_warps == 5;
        const bool auto_tile = o.tile[0] <= 0 && o.tile[1] <= 0 && o.tile[2] <= 0;
        for (;;) {
            const size_t sp =
                subk ? (precision == NUFFT_F64 ? spread_sub_smem_bytes<double>(g)
                                               : spread_sub_smem_bytes<float>(g))
                : precision == NUFFT_F64
                    ? (outer  ? spread_outer_smem_bytes<double>(g)
                       : rows ? spread_rows_smem_bytes<double>(g)
                              : spread_smem_bytes<double>(g))
                    : (outer  ? spread_outer_smem_bytes<float>(g)
                       : rows ? spread_rows_smem_bytes<float>(g)
                              : spread_smem_bytes<float>(g));
            const size_t need = std::max(sp, precision == NUFFT_F64 ? interp_smem_bytes<double>(g)
                                                                    : interp_smem_bytes<float>(g));
            if (need <= (size_t)smem_max) break;
            // a built-in tile too large for one CTA (the widest kernels) shrinks to fit;
            // a caller's tile is refused
            if (subk && auto_tile && g.nsub > 1) {  // one sub-bin less per axis
                g.nsub = 1;
                for (int d = 0; d < 3; ++d) {
                    if (g.ns[d] > 1) {
                        --g.ns[d];
                        g.T[d] -= g.Gs[d];
                    }
                    g.nb[d] = (int)((p->nf[d] + g.T[d] - 1) / g.T[d]);
                    g.nsub *= g.ns[d];
                }
                continue;
            }
            if (!auto_tile || outer || rows || subk || g.T[0] <= 2) {
                delete p;
                return NUFFT_ERR_ARG;
            }
            for (int d = 0; d < 3; ++d) {
                if (g.T[d] > 2) --g.T[d];
                g.nb[d] = (int)((p->nf[d] + g.T[d] - 1) / g.T[d]);
            }
        }
    }
    int st = NUFFT_OK;
    // deconvolution factors p_d(n) = 2 / (w phihat(pi n w / nf_d)) (R6)
    for (int d = 0; d < 3 && !st; ++d) {
        std::vector<double> pd((size_t)p->N[d]);
        for (int64_t i = 0; i < p->N[d]; ++i) {
            const double n = (double)(i - p->N[d] / 2);
            pd[(size_t)i] = 2.0 / ((double)p->w *
                                   es_phihat(M_PI * n * (double)p->w / (double)p->nf[d], p->beta));
        }
        st = dev_alloc(p, &p->d_p[d], (size_t)p->N[d] * p->real_size);
        if (st) break;
        if (precision == NUFFT_F64) {
            st = cuda_status(cudaMemcpy(p->d_p[d], pd.data(), pd.size() * 8, cudaMemcpyHostToDevice));
        } else {
            std::vector<float> pf(pd.begin(), pd.end());
            st = cuda_status(cudaMemcpy(p->d_p[d], pf.data(), pf.size() * 4, cudaMemcpyHostToDevice));
        }
    }
    if (!st && p->comm) {
        st = dist_init(p);  // z-slab geometry, halo grid, buffers, slab FFT plans
    } else if (!st) {
        p->nbins = (int64_t)g.nb[0] * g.nb[1] * g.nb[2];
        // complex grid, or (real transforms) real grid + R2C half spectrum: nf^3 r +
        // nf3 nf2 (nf1/2 + 1) 2r bytes = complex size + 2 nf2 nf3 r
        p->grid_bytes = (size_t)(p->nf[0] * p->nf[1] * p->nf[2]) * p->cplx_size +
                        (size_t)(2 * p->nf[1] * p->nf[2]) * p->real_size;
        st = dev_alloc(p, &p->d_grid, p->grid_bytes);
        p->grid0 = p->d_grid;
        // the complex 3D cuFFT plan (and its workspace) is created on the first complex
        // execute: a plan used only through the real transforms never holds it
    }
    // sort keys: bins, or (bin, sub-bin) pairs for the sub-bin spread
    const int64_t nkeys = p->nbins * (int64_t)g.nsub;
    if (!st && nkeys >= ((int64_t)1 << 31)) st = NUFFT_ERR_UNSUPPORTED;
    if (!st) st = dev_alloc(p, (void**)&p->count, sizeof(uint32_t) * (size_t)nkeys);
    if (!st) st = dev_alloc(p, (void**)&p->offset, sizeof(uint32_t) * (size_t)(p->nbins + 1));
    if (!st && g.nsub > 1)
        st = dev_alloc(p, (void**)&p->offset_key, sizeof(uint32_t) * (size_t)(nkeys + 1));
    if (!st) st = dev_alloc(p, (void**)&p->blocksum, sizeof(uint32_t) * scan_blocksum_elems(nkeys));
    if (!st && p->timing)
        for (int i = 0; i < 8; ++i) {
            cudaEventCreate(&p->ev0[i]);
            cudaEventCreate(&p->ev[i]);
        }
    if (st) {
        nufft_destroy(p);
        return st;
    }
    *out = p;
    return status;
}

int nufft_setpts(nufft_handle p, int64_t Np, const void* x, const void* y, const void* z) {
    cudaGetLastError();  // a stale non-sticky error of another caller is not ours
    if (!p) return NUFFT_ERR_ARG;
    if (Np < 0 || Np >= (int64_t)1 << 31) return NUFFT_ERR_NPTS;
    if (Np > 0 && (!x || !y || !z)) return NUFFT_ERR_ARG;
    StageTimer tm(p, EV_SETPTS);
    int st = NUFFT_OK;
    const size_t b = (size_t)Np * p->real_size;
    const void *xd = nullptr, *yd = nullptr, *zd = nullptr;
    if ((st = input_view(p, x, b, 0, 3 * b, &xd))) return st;
    if ((st = input_view(p, y, b, b, 3 * b, &yd))) return st;
    if ((st = input_view(p, z, b, 2 * b, 3 * b, &zd))) return st;
    if (p->dist) return dist_setpts(p, Np, xd, yd, zd);
    return local_sort(p, Np, xd, yd, zd);
}

int nufft_execute_type1(nufft_handle p, const void* c, void* fk) {
    cudaGetLastError();  // a stale non-sticky error of another caller is not ours
    if (!p || !fk) return NUFFT_ERR_ARG;
    if (p->Np < 0) return NUFFT_ERR_NOT_SET;
    if (!c && user_np(p) > 0) return NUFFT_ERR_ARG;
    if (p->dist) return dist_type1(p, c, fk);
    int st;
    const void* cd = nullptr;
    if ((st = input_view(p, c, (size_t)p->Np * p->cplx_size, 0, (size_t)p->Np * p->cplx_size, &cd)))
        return st;
    const size_t fk_bytes = (size_t)(p->N[0] * p->N[1] * p->N[2]) * p->cplx_size;
    void* fkd = nullptr;
    bool staged = false;
    if ((st = output_view(p, fk, fk_bytes, &fkd, &staged))) return st;
    NUFFT_CK(cudaMemsetAsync(p->d_grid, 0, cgrid_bytes(p), p->stream));
    if ((st = do_spread(p, cd, p->grid0))) return st;                   // Step 1: C
    if (p->fft_method == 1) {                                           // Steps 2-4, Eq. (7)
        if ((st = pruned_type1(p, fkd))) return st;
        return finish_output(p, fk, fkd, fk_bytes, staged);
    }
    if ((st = do_fft(p, p->iflag))) return st;                          // Step 2: F
    {
        StageTimer tm(p, EV_DECONV);                                    // Steps 3, 4: chi, D
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_truncate_deconv<double>(
                static_cast<const double2*>(p->d_grid), p->nf, p->N,
                static_cast<const double*>(p->d_p[0]), static_cast<const double*>(p->d_p[1]),
                static_cast<const double*>(p->d_p[2]), p->modeord, static_cast<double2*>(fkd),
                p->stream));
        else
            NUFFT_CK(launch_truncate_deconv<float>(
                static_cast<const float2*>(p->d_grid), p->nf, p->N,
                static_cast<const float*>(p->d_p[0]), static_cast<const float*>(p->d_p[1]),
                static_cast<const float*>(p->d_p[2]), p->modeord, static_cast<float2*>(fkd),
                p->stream));
    }
    return finish_output(p, fk, fkd, fk_bytes, staged);
}

int nufft_execute_type2(nufft_handle p, const void* fk, void* c) {
    cudaGetLastError();  // a stale non-sticky error of another caller is not ours
    if (!p || !fk) return NUFFT_ERR_ARG;
    if (p->Np < 0) return NUFFT_ERR_NOT_SET;
    if (!c && user_np(p) > 0) return NUFFT_ERR_ARG;
    if (p->dist) return dist_type2(p, fk, c);
    int st;
    const size_t fk_bytes = (size_t)(p->N[0] * p->N[1] * p->N[2]) * p->cplx_size;
    const void* fkd = nullptr;
    if ((st = input_view(p, fk, fk_bytes, 0, fk_bytes, &fkd))) return st;
    const size_t c_bytes = (size_t)p->Np * p->cplx_size;
    void* cd = nullptr;
    bool staged = false;
    if ((st = output_view(p, c, c_bytes, &cd, &staged))) return st;
    if (p->fft_method == 1) {                                           // D, chi^T, F^-1 (Eq. 7)
        if ((st = pruned_type2(p, fkd))) return st;
        if ((st = do_interp(p, p->grid0, cd))) return st;               // C^T
        return finish_output(p, c, cd, c_bytes, staged);
    }
    {
        StageTimer tm(p, EV_PAD);                                       // D, chi^T
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_pad_precorrect<double>(
                static_cast<const double2*>(fkd), p->N, static_cast<const double*>(p->d_p[0]),
                static_cast<const double*>(p->d_p[1]), static_cast<const double*>(p->d_p[2]),
                p->modeord, p->nf, static_cast<double2*>(p->d_grid), p->stream));
        else
            NUFFT_CK(launch_pad_precorrect<float>(
                static_cast<const float2*>(fkd), p->N, static_cast<const float*>(p->d_p[0]),
                static_cast<const float*>(p->d_p[1]), static_cast<const float*>(p->d_p[2]),
                p->modeord, p->nf, static_cast<float2*>(p->d_grid), p->stream));
    }
    if ((st = do_fft(p, -p->iflag))) return st;                         // F^-1
    if ((st = do_interp(p, p->grid0, cd))) return st;                   // C^T
    return finish_output(p, c, cd, c_bytes, staged);
}

int nufft_execute_type1_real(nufft_handle p, const void* c, void* fk) {
    cudaGetLastError();
    if (!p || !fk) return NUFFT_ERR_ARG;
    if (p->Np < 0) return NUFFT_ERR_NOT_SET;
    if (!c && user_np(p) > 0) return NUFFT_ERR_ARG;
    if (p->dist) return dist_type1_real(p, c, fk);
    int st;
    if ((st = ensure_real_fft(p))) return st;
    const void* cd = nullptr;
    if ((st = input_view(p, c, (size_t)p->Np * p->real_size, 0, (size_t)p->Np * p->real_size, &cd)))
        return st;
    const size_t fk_bytes = (size_t)(p->N[0] * p->N[1] * p->N[2]) * p->cplx_size;
    void* fkd = nullptr;
    bool staged = false;
    if ((st = output_view(p, fk, fk_bytes, &fkd, &staged))) return st;
    const size_t rg = (size_t)(p->nf[0] * p->nf[1] * p->nf[2]) * p->real_size;
    NUFFT_CK(cudaMemsetAsync(p->d_grid, 0, rg, p->stream));
    if ((st = do_spread_real(p, cd, p->d_grid))) return st;              // Step 1: C
    {
        StageTimer tm(p, EV_FFT);                                        // Step 2: F (R2C)
        const cufftResult r =
            p->prec == NUFFT_F64
                ? cufftExecD2Z(p->fft_r2c, static_cast<cufftDoubleReal*>(p->d_grid),
                               static_cast<cufftDoubleComplex*>(half_spectrum(p)))
                : cufftExecR2C(p->fft_r2c, static_cast<cufftReal*>(p->d_grid),
                               static_cast<cufftComplex*>(half_spectrum(p)));
        if (r != CUFFT_SUCCESS) return NUFFT_ERR_CUFFT;
    }
    {
        StageTimer tm(p, EV_DECONV);                                     // Steps 3, 4
        const int conj_all = p->iflag > 0 ? 1 : 0;
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_truncate_deconv_r2c<double>(
                static_cast<const double2*>(half_spectrum(p)), p->nf, p->N,
                static_cast<const double*>(p->d_p[0]), static_cast<const double*>(p->d_p[1]),
                static_cast<const double*>(p->d_p[2]), p->modeord, conj_all,
                static_cast<double2*>(fkd), p->stream));
        else
            NUFFT_CK(launch_truncate_deconv_r2c<float>(
                static_cast<const float2*>(half_spectrum(p)), p->nf, p->N,
                static_cast<const float*>(p->d_p[0]), static_cast<const float*>(p->d_p[1]),
                static_cast<const float*>(p->d_p[2]), p->modeord, conj_all,
                static_cast<float2*>(fkd), p->stream));
    }
    return finish_output(p, fk, fkd, fk_bytes, staged);
}

int nufft_execute_type2_real(nufft_handle p, const void* fk, void* c) {
    cudaGetLastError();
    if (!p || !fk) return NUFFT_ERR_ARG;
    if (p->Np < 0) return NUFFT_ERR_NOT_SET;
    if (!c && user_np(p) > 0) return NUFFT_ERR_ARG;
    if (p->dist) return dist_type2_real(p, fk, c);
    int st;
    if ((st = ensure_real_fft(p))) return st;
    const size_t fk_bytes = (size_t)(p->N[0] * p->N[1] * p->N[2]) * p->cplx_size;
    const void* fkd = nullptr;
    if ((st = input_view(p, fk, fk_bytes, 0, fk_bytes, &fkd))) return st;
    const size_t c_bytes = (size_t)p->Np * p->real_size;
    void* cd = nullptr;
    bool staged = false;
    if ((st = output_view(p, c, c_bytes, &cd, &staged))) return st;
    {
        StageTimer tm(p, EV_PAD);                                        // D, chi^T, Hermitian part
        const int sign_plus = p->iflag < 0 ? 1 : 0;                      // type-2 sign = -iflag
        if (p->prec == NUFFT_F64)
            NUFFT_CK(launch_pad_precorrect_c2r<double>(
                static_cast<const double2*>(fkd), p->N, static_cast<const double*>(p->d_p[0]),
                static_cast<const double*>(p->d_p[1]), static_cast<const double*>(p->d_p[2]),
                p->modeord, sign_plus, p->nf, static_cast<double2*>(half_spectrum(p)),
                p->stream));
        else
            NUFFT_CK(launch_pad_precorrect_c2r<float>(
                static_cast<const float2*>(fkd), p->N, static_cast<const float*>(p->d_p[0]),
                static_cast<const float*>(p->d_p[1]), static_cast<const float*>(p->d_p[2]),
                p->modeord, sign_plus, p->nf, static_cast<float2*>(half_spectrum(p)),
                p->stream));
    }
    {
        StageTimer tm(p, EV_FFT);                                        // F^-1 (C2R)
        const cufftResult r =
            p->prec == NUFFT_F64
                ? cufftExecZ2D(p->fft_c2r, static_cast<cufftDoubleComplex*>(half_spectrum(p)),
                               static_cast<cufftDoubleReal*>(p->d_grid))
                : cufftExecC2R(p->fft_c2r, static_cast<cufftComplex*>(half_spectrum(p)),
                               static_cast<cufftReal*>(p->d_grid));
        if (r != CUFFT_SUCCESS) return NUFFT_ERR_CUFFT;
    }
    if ((st = do_interp_real(p, p->d_grid, cd))) return st;              // C^T
    return finish_output(p, c, cd, c_bytes, staged);
}

namespace {
int64_t nf3_of(const nufft_plan_s* p) { return p->nf[0] * p->nf[1] * p->nf[2]; }
// three real fields (PIF E field) as three consecutive real fine grids (SoA) in the
// grid buffer, each filled by the plan's C2R transform
int real3_fields(nufft_plan_s* p, const void* fk0, const void* fk1, const void* fk2) {
    // the three fields + a half spectrum live in the grid buffer (grown once): no
    // other grid is live during the gather
    const size_t nf3 = (size_t)(p->nf[0] * p->nf[1] * p->nf[2]);
    const size_t half = (size_t)((p->nf[0] / 2 + 1) * p->nf[1] * p->nf[2]) * p->cplx_size;
    const size_t need = 3 * nf3 * p->real_size + half;
    if (p->grid_bytes < need) {
        dev_free(p, &p->d_grid, p->grid_bytes);
        p->grid_bytes = 0;
        p->grid0 = nullptr;
        int st = dev_alloc(p, &p->d_grid, need);
        if (st) return st;
        p->grid_bytes = need;
        p->grid0 = p->d_grid;
    }
    p->vgrid = p->d_grid;
    void* half3 = static_cast<char*>(p->d_grid) + 3 * nf3 * p->real_size;
    int st0;
    if ((st0 = ensure_real_fft(p))) return st0;
    const void* fks[3] = {fk0, fk1, fk2};
    const int sign_plus = p->iflag < 0 ? 1 : 0;
    for (int d = 0; d < 3; ++d) {
        {
            StageTimer tm(p, EV_PAD);
            if (p->prec == NUFFT_F64)
                NUFFT_CK(launch_pad_precorrect_c2r<double>(
                    static_cast<const double2*>(fks[d]), p->N,
                    static_cast<const double*>(p->d_p[0]), static_cast<const double*>(p->d_p[1]),
                    static_cast<const double*>(p->d_p[2]), p->modeord, sign_plus, p->nf,
                    static_cast<double2*>(half3), p->stream));
            else
                NUFFT_CK(launch_pad_precorrect_c2r<float>(
                    static_cast<const float2*>(fks[d]), p->N,
                    static_cast<const float*>(p->d_p[0]), static_cast<const float*>(p->d_p[1]),
                    static_cast<const float*>(p->d_p[2]), p->modeord, sign_plus, p->nf,
                    static_cast<float2*>(half3), p->stream));
        }
        StageTimer tm(p, EV_FFT);
        const cufftResult r =
            p->prec == NUFFT_F64
                ? cufftExecZ2D(p->fft_c2r, static_cast<cufftDoubleComplex*>(half3),
                               static_cast<cufftDoubleReal*>(p->vgrid) + d * nf3)
                : cufftExecC2R(p->fft_c2r, static_cast<cufftComplex*>(half3),
                               static_cast<cufftReal*>(p->vgrid) + d * nf3);
        if (r != CUFFT_SUCCESS) return NUFFT_ERR_CUFFT;
    }
    return NUFFT_OK;
}
}  // namespace

int nufft_execute_type2_real3(nufft_handle p, const void* fk0, const void* fk1, const void* fk2,
                              void* c) {
    cudaGetLastError();
    if (!p || !fk0 || !fk1 || !fk2) return NUFFT_ERR_ARG;
    if (p->Np < 0) return NUFFT_ERR_NOT_SET;
    if (!c && p->Np > 0) return NUFFT_ERR_ARG;
    if (p->dist) return NUFFT_ERR_UNSUPPORTED;
    if (!is_device_ptr(fk0) || !is_device_ptr(fk1) || !is_device_ptr(fk2) ||
        (p->Np > 0 && !is_device_ptr(c)))
        return NUFFT_ERR_ARG;
    int st;
    if ((st = real3_fields(p, fk0, fk1, fk2))) return st;
    StageTimer tm(p, EV_INTERP);
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_interp_vec3<double>(p->geom, pts_view<double>(p), p->nbins,
                                            static_cast<const double*>(p->vgrid), nf3_of(p),
                                            static_cast<double*>(c), p->beta, p->stream));
    else
        NUFFT_CK(launch_interp_vec3<float>(p->geom, pts_view<float>(p), p->nbins,
                                           static_cast<const float*>(p->vgrid), nf3_of(p),
                                           static_cast<float*>(c), p->beta, p->stream));
    return NUFFT_OK;
}

int nufft_pif_gather_kick(nufft_handle p, const void* ex_k, const void* ey_k, const void* ez_k,
                          void* vx, void* vy, void* vz, double scale) {
    cudaGetLastError();
    if (!p || !ex_k || !ey_k || !ez_k) return NUFFT_ERR_ARG;
    if (p->Np < 0) return NUFFT_ERR_NOT_SET;
    if (p->Np > 0 && (!vx || !vy || !vz)) return NUFFT_ERR_ARG;
    if (p->dist) return NUFFT_ERR_UNSUPPORTED;
    if (!is_device_ptr(ex_k) || !is_device_ptr(ey_k) || !is_device_ptr(ez_k) ||
        (p->Np > 0 && (!is_device_ptr(vx) || !is_device_ptr(vy) || !is_device_ptr(vz))))
        return NUFFT_ERR_ARG;
    int st;
    if ((st = real3_fields(p, ex_k, ey_k, ez_k))) return st;
    StageTimer tm(p, EV_INTERP);
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_interp_vec3_kick<double>(
            p->geom, pts_view<double>(p), p->nbins, static_cast<const double*>(p->vgrid),
            nf3_of(p), static_cast<double*>(vx), static_cast<double*>(vy), static_cast<double*>(vz), scale,
            p->beta, p->stream));
    else
        NUFFT_CK(launch_interp_vec3_kick<float>(
            p->geom, pts_view<float>(p), p->nbins, static_cast<const float*>(p->vgrid),
            nf3_of(p), static_cast<float*>(vx), static_cast<float*>(vy), static_cast<float*>(vz), scale,
            p->beta, p->stream));
    return NUFFT_OK;
}

int nufft_spread(nufft_handle p, const void* c, void* grid) {
    cudaGetLastError();  // a stale non-sticky error of another caller is not ours
    if (!p || !grid || (!c && p->Np > 0)) return NUFFT_ERR_ARG;
    if (p->dist) return NUFFT_ERR_UNSUPPORTED;
    if (p->Np < 0) return NUFFT_ERR_NOT_SET;
    int st;
    const void* cd = nullptr;
    if ((st = input_view(p, c, (size_t)p->Np * p->cplx_size, 0, (size_t)p->Np * p->cplx_size, &cd)))
        return st;
    void* gd = nullptr;
    bool staged = false;
    if ((st = output_view(p, grid, cgrid_bytes(p), &gd, &staged))) return st;
    NUFFT_CK(cudaMemsetAsync(gd, 0, cgrid_bytes(p), p->stream));
    if ((st = do_spread(p, cd, gd))) return st;
    return finish_output(p, grid, gd, cgrid_bytes(p), staged);
}

int nufft_interp(nufft_handle p, const void* grid, void* c) {
    cudaGetLastError();  // a stale non-sticky error of another caller is not ours
    if (!p || !grid || (!c && p->Np > 0)) return NUFFT_ERR_ARG;
    if (p->dist) return NUFFT_ERR_UNSUPPORTED;
    if (p->Np < 0) return NUFFT_ERR_NOT_SET;
    int st;
    const void* gd = nullptr;
    if ((st = input_view(p, grid, cgrid_bytes(p), 0, cgrid_bytes(p), &gd))) return st;
    const size_t c_bytes = (size_t)p->Np * p->cplx_size;
    void* cd = nullptr;
    bool staged = false;
    if ((st = output_view(p, c, c_bytes, &cd, &staged))) return st;
    if ((st = do_interp(p, gd, cd))) return st;
    return finish_output(p, c, cd, c_bytes, staged);
}

int nufft_destroy(nufft_handle p) {
    if (!p) return NUFFT_OK;
    if (p->stream) cudaStreamSynchronize(p->stream);
    else cudaDeviceSynchronize();
    if (p->dist) dist_destroy(p);
    if (p->fft_ok) cufftDestroy(p->fft);
    if (p->fft_r_ok) {
        cufftDestroy(p->fft_r2c);
        cufftDestroy(p->fft_c2r);
    }
    for (int d = 0; d < 3; ++d) dev_free(p, &p->d_p[d], 0);
    dev_free(p, &p->d_grid, 0);
    dev_free(p, (void**)&p->count, 0);
    dev_free(p, (void**)&p->offset, 0);
    dev_free(p, (void**)&p->offset_key, 0);
    if (p->fft_sub_ok) {
        cufftDestroy(p->fft_sub1);
        cufftDestroy(p->fft_sub2);
    }
    dev_free(p, &p->fft_aux, p->fft_aux_bytes);
    dev_free(p, &p->morton, p->morton_bytes);
    dev_free(p, (void**)&p->blocksum, 0);
    dev_free(p, (void**)&p->bin_of, 0);
    dev_free(p, (void**)&p->rank_of, 0);
    dev_free(p, &p->rec, 0);
    dev_free(p, &p->wts, 0);
    dev_free(p, &p->order, 0);
    dev_free(p, &p->stage_in, 0);
    dev_free(p, &p->stage_out, 0);
    if (p->timing)
        for (int i = 0; i < 8; ++i) {
            if (p->ev0[i]) cudaEventDestroy(p->ev0[i]);
            if (p->ev[i]) cudaEventDestroy(p->ev[i]);
        }
    delete p;
    return NUFFT_OK;
}

int nufft_get_info(nufft_handle p, nufft_info* info) {
    if (!p || !info) return NUFFT_ERR_ARG;
    std::memset(info, 0, sizeof(*info));
    info->precision = p->prec;
    info->w = p->w;
    info->beta = p->beta;
    info->eps = p->eps;
    for (int d = 0; d < 3; ++d) {
        info->N[d] = p->N[d];
        info->nf[d] = p->nf[d];
        info->tile[d] = p->geom.T[d];
    }
    info->nbins = p->nbins;
    info->Np = p->Np;
    info->device_bytes = p->bytes;
    info->nranks = 1;
    info->rank = 0;
    info->slab_lo = p->geom.z_lo;
    info->slab_hi = p->geom.z_lo + p->geom.nz_loc;
    if (p->dist) {
        int64_t lo[3], hi[3];
        dist_local_modes(p, lo, hi);
        info->nranks = (int)(p->nf[2] / p->geom.nz_loc);
        info->rank = (int)(p->geom.z_lo / p->geom.nz_loc);
    }
    float ms[8];
    for (int i = 0; i < 8; ++i) {
        ms[i] = -1.0f;
        if (p->timing && p->ev_used[i] && cudaEventSynchronize(p->ev[i]) == cudaSuccess)
            cudaEventElapsedTime(&ms[i], p->ev0[i], p->ev[i]);
    }
    info->ms_setpts = ms[EV_SETPTS];
    info->ms_spread = ms[EV_SPREAD];
    info->ms_fold = -1;
    info->ms_fft = ms[EV_FFT];
    info->ms_deconv = ms[EV_DECONV];
    info->ms_pad = ms[EV_PAD];
    info->ms_interp = ms[EV_INTERP];
    info->ms_comm = ms[EV_COMM];
    info->weights_precomputed = p->wts_on ? 1 : 0;
    info->sub_bins = p->geom.nsub;
    return NUFFT_OK;
}

int nufft_local_modes(nufft_handle p, int64_t lo[3], int64_t hi[3]) {
    if (!p || !lo || !hi) return NUFFT_ERR_ARG;
    if (p->dist) return dist_local_modes(p, lo, hi);
    for (int d = 0; d < 3; ++d) {
        lo[d] = 0;
        hi[d] = p->N[d];
    }
    return NUFFT_OK;
}

static int pif_poisson(nufft_handle p, const void* rho_k, void* ex_k, void* ey_k, void* ez_k,
                       bool real_layout) {
    cudaGetLastError();
    if (!p || !rho_k || !ex_k || !ey_k || !ez_k) return NUFFT_ERR_ARG;
    if (!is_device_ptr(rho_k) || !is_device_ptr(ex_k) || !is_device_ptr(ey_k) || !is_device_ptr(ez_k))
        return NUFFT_ERR_ARG;
    int64_t lo[3], hi[3];
    nufft_local_modes(p, lo, hi);
    // a slab plan's real transforms hold x modes k1 = 0 .. N1/2 (half spectrum)
    const int xhalf = (real_layout && p->dist) ? 1 : 0;
    if (xhalf) {
        lo[0] = 0;
        hi[0] = p->N[0] / 2 + 1;
    }
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_pif_poisson<double>(static_cast<const double2*>(rho_k), p->N, lo, hi,
                                            p->geom.L, p->modeord, xhalf,
                                            static_cast<double2*>(ex_k), static_cast<double2*>(ey_k),
                                            static_cast<double2*>(ez_k), p->stream));
    else
        NUFFT_CK(launch_pif_poisson<float>(static_cast<const float2*>(rho_k), p->N, lo, hi,
                                           p->geom.L, p->modeord, xhalf,
                                           static_cast<float2*>(ex_k), static_cast<float2*>(ey_k),
                                           static_cast<float2*>(ez_k), p->stream));
    return NUFFT_OK;
}

int nufft_pif_poisson(nufft_handle p, const void* rho_k, void* ex_k, void* ey_k, void* ez_k) {
    return pif_poisson(p, rho_k, ex_k, ey_k, ez_k, false);
}

int nufft_pif_poisson_real(nufft_handle p, const void* rho_k, void* ex_k, void* ey_k,
                           void* ez_k) {
    return pif_poisson(p, rho_k, ex_k, ey_k, ez_k, true);
}

int nufft_pif_kick(nufft_handle p, int64_t Np, void* v, const void* e, double scale) {
    cudaGetLastError();
    if (!p || Np < 0 || (Np > 0 && (!v || !e))) return NUFFT_ERR_ARG;
    if (Np > 0 && (!is_device_ptr(v) || !is_device_ptr(e))) return NUFFT_ERR_ARG;
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_pif_kick<double>(Np, static_cast<double*>(v), static_cast<const double2*>(e),
                                         scale, p->stream));
    else
        NUFFT_CK(launch_pif_kick<float>(Np, static_cast<float*>(v), static_cast<const float2*>(e),
                                        scale, p->stream));
    return NUFFT_OK;
}

int nufft_pif_kick_real(nufft_handle p, int64_t Np, void* v, const void* e, double scale) {
    cudaGetLastError();
    if (!p || Np < 0 || (Np > 0 && (!v || !e))) return NUFFT_ERR_ARG;
    if (Np > 0 && (!is_device_ptr(v) || !is_device_ptr(e))) return NUFFT_ERR_ARG;
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_pif_kick_real<double>(Np, static_cast<double*>(v),
                                              static_cast<const double*>(e), scale, p->stream));
    else
        NUFFT_CK(launch_pif_kick_real<float>(Np, static_cast<float*>(v),
                                             static_cast<const float*>(e), scale, p->stream));
    return NUFFT_OK;
}

int nufft_pif_drift(nufft_handle p, int64_t Np, void* x, void* y, void* z, const void* vx,
                    const void* vy, const void* vz, double dt) {
    cudaGetLastError();
    if (!p || Np < 0 || (Np > 0 && (!x || !y || !z || !vx || !vy || !vz))) return NUFFT_ERR_ARG;
    if (Np > 0 && !is_device_ptr(x)) return NUFFT_ERR_ARG;
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_pif_drift<double>(Np, static_cast<double*>(x), static_cast<double*>(y),
                                          static_cast<double*>(z), static_cast<const double*>(vx),
                                          static_cast<const double*>(vy),
                                          static_cast<const double*>(vz), dt, p->geom.L, p->stream));
    else
        NUFFT_CK(launch_pif_drift<float>(Np, static_cast<float*>(x), static_cast<float*>(y),
                                         static_cast<float*>(z), static_cast<const float*>(vx),
                                         static_cast<const float*>(vy),
                                         static_cast<const float*>(vz), dt, p->geom.L, p->stream));
    return NUFFT_OK;
}

}  // extern "C"
