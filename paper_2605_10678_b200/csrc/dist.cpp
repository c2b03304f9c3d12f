// dist.cpp -- the distributed (multi-GPU) NUFFT: z-slab decomposition over NCCL.
//
// PAPER.md:229-235 (§2.4): grid values and particles share one spatial
// decomposition, each local domain carries a halo of ceil(w/2) planes, halos are
// ACCUMULATED into the owners after spreading and FILLED from the owners before
// interpolation, and the FFT is a distributed FFT.  On one NVSwitch box we use
// z-slabs: rank r owns fine planes [r nf3/P, (r+1) nf3/P) and the
// points whose fine cell lies there.  Every exchange goes through the communicator's
// transport (xport.h): NCCL between GPUs, or loopback for P ranks on one GPU (tests).
//
//   setpts   owner = slab of the fine z-cell; counts all-to-all; points moved
//            with grouped ncclSend/ncclRecv (skipped with opts.points_owned);
//            then the local counting sort (sort.cu) on the slab.
//   type 1   strengths follow the points -> spread into the halo-extended slab ->
//            halo accumulate (ncclSend/Recv with both z-neighbours + add) ->
//            2D (x, y) cuFFT of the owned planes -> keep the retained (x, y)
//            modes and pack them by destination y-block -> ncclAlltoAll
//            (z-slab -> y-slab) -> 1D z cuFFT -> keep retained z modes * D.
//            Truncating before the transpose is exact (chi, F separable per axis)
//            and moves N1 N2 nf3 / P instead of nf1 nf2 nf3 / P values per rank.
//   type 2   the mirror: pad z * D -> 1D z iFFT -> ncclAlltoAll (y-slab -> z-slab)
//            -> zero-pad (x, y) -> 2D iFFT -> halo fill -> interpolate -> results
//            return to the caller's ranks and order.
// Mode layout of a distributed plan: this rank holds storage indices
// [r N2/P, (r+1) N2/P) along y (all of x and z), x fastest (nufft_local_modes).
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "plan_state.h"
#include "xport.h"

// a communicator: the transport (NCCL, or loopback for P ranks on one GPU) and
// this handle's rank
struct NufftComm {
    nufft::Xport* x = nullptr;
    int nranks = 1;
    int rank = 0;
};

namespace nufft {

struct DistState {
    int P = 1, r = 0;
    int64_t nzl = 0;     // owned fine z-planes
    int64_t NY = 0;      // y-modes per rank
    int64_t y0 = 0;      // first y storage index of this rank
    int hlo = 0, hhi = 0;
    int64_t plane = 0;   // nf1 nf2
    Xport* x = nullptr;  // the communicator's transport (xport.h)
    size_t rs = 8;       // bytes per real

    void* xbuf = nullptr;      // nzl N2 N1 complex: x-y-truncated planes / z-lines (two roles)
    void* ybuf = nullptr;      // same size
    size_t xfer_bytes = 0;
    void* halo_a = nullptr;    // accumulate: hlo planes from the upper neighbour
    void* halo_b = nullptr;    // accumulate: hhi planes from the lower neighbour
    cufftHandle fft2 = 0, fft1 = 0;
    bool fft2_ok = false, fft1_ok = false;

    // point redistribution
    bool redist = false;
    int64_t np_user = 0, np_local = 0, cap_user = 0, cap_local = 0;
    uint32_t* owner = nullptr;
    uint32_t* rank_in = nullptr;
    unsigned long long* d_counts = nullptr;  // [P] this rank's per-destination counts, then recv
    unsigned long long* d_rcounts = nullptr; // [P]
    unsigned long long* d_off = nullptr;     // [P] send offsets
    std::vector<unsigned long long> scount, soff, rcount, roff;
    void* sbuf = nullptr;  // send staging (3 coords or complex values), np_user elements
    void* rbuf = nullptr;  // receive staging, np_local elements
    size_t sbuf_bytes = 0, rbuf_bytes = 0;

    // real transforms (half-spectrum modes): batched 2D R2C / C2R of the owned planes,
    // 1D z transforms of the NY (N1/2 + 1) lines, half planes nzl x nf2 x (nf1/2 + 1)
    cufftHandle fft2r = 0, fft2c = 0, fft1h = 0;
    bool real_ok = false;
    void* hbuf = nullptr;
    size_t hbuf_bytes = 0;

    // PIF particle migration (nufft_pif_migrate)
    unsigned long long* d_mig = nullptr;  // [P] pack cursors, [2] hole / tail counters, [1] flag
    void* mig_send = nullptr;             // leavers, 6 values each
    void* mig_recv = nullptr;             // arrivals, 6 values each
    void* mig_idx = nullptr;              // 3 nleave int64: vacated slots, holes, tail stayers
    size_t mig_send_bytes = 0, mig_recv_bytes = 0, mig_idx_bytes = 0;
};

namespace {



// grow-only staging buffers with 12.5 % slack: per-step particle migration changes
// the counts slightly, and a cudaFree/cudaMalloc of GBs every step would dominate
int ensure(nufft_plan_s* p, void** buf, size_t* have, size_t need) {
    if (*have >= need && *buf) return NUFFT_OK;
    dev_free(p, buf, *have);
    *have = 0;
    need += need / 8;
    int st = dev_alloc(p, buf, need);
    if (!st) *have = need;
    return st;
}

// grouped point-to-point all-to-all-v of `elem` bytes per item
int alltoallv(DistState* d, const void* send, const std::vector<unsigned long long>& sc,
              const std::vector<unsigned long long>& so, void* recv,
              const std::vector<unsigned long long>& rc, const std::vector<unsigned long long>& ro,
              size_t elem, cudaStream_t s) {
    int st;
    if ((st = d->x->group_start())) return st;
    for (int q = 0; q < d->P; ++q) {
        if (sc[q] && (st = d->x->send(static_cast<const char*>(send) + so[q] * elem, sc[q] * elem,
                                      q, s)))
            return st;
        if (rc[q] &&
            (st = d->x->recv(static_cast<char*>(recv) + ro[q] * elem, rc[q] * elem, q, s)))
            return st;
    }
    return d->x->group_end(s);
}

// Ghost planes of the slab grid whose cells hold K reals (K = 2: complex, 1: real).
template <typename T>
int halo_accumulate(nufft_plan_s* p, void* grid0, int K) {
    using C = typename Cx<T>::type;
    DistState* d = p->dist;
    T* g0 = static_cast<T*>(grid0);
    const int prev = (d->r + d->P - 1) % d->P, next = (d->r + 1) % d->P;
    const size_t pl = (size_t)d->plane * K;  // reals per plane
    const size_t rs = sizeof(T);
    int st;
    Xport* x = d->x;
    if ((st = x->group_start())) return st;
    // my lower halo (hlo planes below plane 0) belongs to prev's top owned planes
    if ((st = x->send(g0 - d->hlo * pl, d->hlo * pl * rs, prev, p->stream))) return st;
    if ((st = x->recv(d->halo_a, d->hlo * pl * rs, next, p->stream))) return st;
    // my upper halo (hhi planes above the slab) belongs to next's bottom owned planes
    if ((st = x->send(g0 + d->nzl * pl, d->hhi * pl * rs, next, p->stream))) return st;
    if ((st = x->recv(d->halo_b, d->hhi * pl * rs, prev, p->stream))) return st;
    if ((st = x->group_end(p->stream))) return st;
    // the adds run on complex pairs (plane sizes are even)
    NUFFT_CK(launch_halo_add<T>((int64_t)(d->hlo * pl / 2),
                                reinterpret_cast<C*>(g0 + (d->nzl - d->hlo) * pl),
                                static_cast<const C*>(d->halo_a), p->stream));
    NUFFT_CK(launch_halo_add<T>((int64_t)(d->hhi * pl / 2), reinterpret_cast<C*>(g0),
                                static_cast<const C*>(d->halo_b), p->stream));
    return NUFFT_OK;
}
template <typename T>
int halo_fill(nufft_plan_s* p, void* grid0, int K) {
    DistState* d = p->dist;
    T* g0 = static_cast<T*>(grid0);
    const int prev = (d->r + d->P - 1) % d->P, next = (d->r + 1) % d->P;
    const size_t pl = (size_t)d->plane * K;
    const size_t rs = sizeof(T);
    int st;
    Xport* x = d->x;
    if ((st = x->group_start())) return st;
    // my bottom hhi owned planes are prev's upper halo; next's bottom planes are mine
    if ((st = x->send(g0, d->hhi * pl * rs, prev, p->stream))) return st;
    if ((st = x->recv(g0 + d->nzl * pl, d->hhi * pl * rs, next, p->stream))) return st;
    // my top hlo owned planes are next's lower halo; prev's top planes fill my lower halo
    if ((st = x->send(g0 + (d->nzl - d->hlo) * pl, d->hlo * pl * rs, next, p->stream))) return st;
    if ((st = x->recv(g0 - d->hlo * pl, d->hlo * pl * rs, prev, p->stream))) return st;
    return x->group_end(p->stream);
}
int fft_exec(nufft_plan_s* p, cufftHandle h, void* data, int sign) {
    const int dir = sign < 0 ? CUFFT_FORWARD : CUFFT_INVERSE;
    cufftResult r;
    if (p->prec == NUFFT_F64)
        r = cufftExecZ2Z(h, static_cast<cufftDoubleComplex*>(data),
                         static_cast<cufftDoubleComplex*>(data), dir);
    else
        r = cufftExecC2C(h, static_cast<cufftComplex*>(data), static_cast<cufftComplex*>(data), dir);
    return r == CUFFT_SUCCESS ? NUFFT_OK : NUFFT_ERR_CUFFT;
}

template <typename T>
int type1_t(nufft_plan_s* p, const void* c_local, void* fk_local) {
    using C = typename Cx<T>::type;
    DistState* d = p->dist;
    int st;
    NUFFT_CK(cudaMemsetAsync(p->d_grid, 0, p->grid_bytes, p->stream));
    if ((st = do_spread(p, c_local, p->grid0))) return st;                         // C
    {
        StageTimer tm(p, EV_COMM);
        if ((st = halo_accumulate<T>(p, p->grid0, 2))) return st;                 // halos
    }
    {
        StageTimer tm(p, EV_FFT);
        if ((st = fft_exec(p, d->fft2, p->grid0, p->iflag))) return st;            // F (x, y)
        NUFFT_CK(launch_xy_pack<T>(static_cast<const C*>(p->grid0), p->nf, d->nzl, p->N, d->P,
                                   p->modeord, static_cast<C*>(d->xbuf), p->stream));  // chi (x, y)
        if ((st = d->x->alltoall(d->xbuf, d->ybuf, 2 * (size_t)(d->nzl * d->NY * p->N[0]) * d->rs,
                                 p->stream)))
            return st;                                                             // transpose
        if ((st = fft_exec(p, d->fft1, d->ybuf, p->iflag))) return st;             // F (z)
    }
    StageTimer tm(p, EV_DECONV);
    NUFFT_CK(launch_z_deconv<T>(static_cast<const C*>(d->ybuf), p->nf, p->N, d->NY, d->y0,
                                static_cast<const T*>(p->d_p[0]), static_cast<const T*>(p->d_p[1]),
                                static_cast<const T*>(p->d_p[2]), p->modeord,
                                static_cast<C*>(fk_local), p->stream));          // chi (z), D
    return NUFFT_OK;
}

template <typename T>
int type2_t(nufft_plan_s* p, const void* fk_local, void* c_local) {
    using C = typename Cx<T>::type;
    DistState* d = p->dist;
    int st;
    {
        StageTimer tm(p, EV_PAD);
        NUFFT_CK(launch_z_pad<T>(static_cast<const C*>(fk_local), p->nf, p->N, d->NY, d->y0,
                                 static_cast<const T*>(p->d_p[0]), static_cast<const T*>(p->d_p[1]),
                                 static_cast<const T*>(p->d_p[2]), p->modeord,
                                 static_cast<C*>(d->ybuf), p->stream));          // D, chi^T (z)
    }
    {
        StageTimer tm(p, EV_FFT);
        if ((st = fft_exec(p, d->fft1, d->ybuf, -p->iflag))) return st;            // F^-1 (z)
        if ((st = d->x->alltoall(d->ybuf, d->xbuf, 2 * (size_t)(d->nzl * d->NY * p->N[0]) * d->rs,
                                 p->stream)))
            return st;                                                             // transpose
        NUFFT_CK(launch_xy_unpad<T>(static_cast<const C*>(d->xbuf), p->nf, d->nzl, p->N, d->P,
                                    p->modeord, static_cast<C*>(p->grid0), p->stream));  // chi^T
        if ((st = fft_exec(p, d->fft2, p->grid0, -p->iflag))) return st;           // F^-1 (x, y)
    }
    {
        StageTimer tm(p, EV_COMM);
        if ((st = halo_fill<T>(p, p->grid0, 2))) return st;                       // halos
    }
    return do_interp(p, p->grid0, c_local);                                        // C^T
}

int ensure_real_dist(nufft_plan_s* p) {
    DistState* d = p->dist;
    if (d->real_ok) return NUFFT_OK;
    const bool f64 = p->prec == NUFFT_F64;
    const int nf1 = (int)p->nf[0], nf2 = (int)p->nf[1], hx = nf1 / 2 + 1;
    int n2[2] = {nf2, nf1};
    int rembed[2] = {nf2, nf1}, cembed[2] = {nf2, hx};
    if (cufftPlanMany(&d->fft2r, 2, n2, rembed, 1, nf2 * nf1, cembed, 1, nf2 * hx,
                      f64 ? CUFFT_D2Z : CUFFT_R2C, (int)d->nzl) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    if (cufftPlanMany(&d->fft2c, 2, n2, cembed, 1, nf2 * hx, rembed, 1, nf2 * nf1,
                      f64 ? CUFFT_Z2D : CUFFT_C2R, (int)d->nzl) != CUFFT_SUCCESS) {
        cufftDestroy(d->fft2r);
        return NUFFT_ERR_CUFFT;
    }
    const int S = (int)(d->NY * (p->N[0] / 2 + 1));
    int n1[1] = {(int)p->nf[2]};
    int emb[1] = {(int)p->nf[2]};
    if (cufftPlanMany(&d->fft1h, 1, n1, emb, S, 1, emb, S, 1, f64 ? CUFFT_Z2Z : CUFFT_C2C, S) !=
        CUFFT_SUCCESS) {
        cufftDestroy(d->fft2r);
        cufftDestroy(d->fft2c);
        return NUFFT_ERR_CUFFT;
    }
    d->real_ok = true;
    size_t ws = 0;
    cufftGetSize(d->fft2r, &ws);
    p->bytes += ws;
    cufftGetSize(d->fft2c, &ws);
    p->bytes += ws;
    cufftGetSize(d->fft1h, &ws);
    p->bytes += ws;
    if (cufftSetStream(d->fft2r, p->stream) != CUFFT_SUCCESS ||
        cufftSetStream(d->fft2c, p->stream) != CUFFT_SUCCESS ||
        cufftSetStream(d->fft1h, p->stream) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    return ensure(p, &d->hbuf, &d->hbuf_bytes,
                  (size_t)(d->nzl * p->nf[1] * (p->nf[0] / 2 + 1)) * p->cplx_size);
}

// real slab grid: (hlo + nzl + hhi) planes of reals at d_grid, plane 0 after hlo
template <typename T>
T* real_grid0(nufft_plan_s* p) {
    return static_cast<T*>(p->d_grid) + p->dist->hlo * p->dist->plane;
}

template <typename T>
int type1_real_t(nufft_plan_s* p, const void* c_local, void* fk_local) {
    using C = typename Cx<T>::type;
    DistState* d = p->dist;
    int st;
    const size_t rg = (size_t)((d->hlo + d->nzl + d->hhi) * d->plane) * sizeof(T);
    NUFFT_CK(cudaMemsetAsync(p->d_grid, 0, rg, p->stream));
    T* g0 = real_grid0<T>(p);
    if ((st = do_spread_real(p, c_local, g0))) return st;                          // C
    {
        StageTimer tm(p, EV_COMM);
        if ((st = halo_accumulate<T>(p, g0, 1))) return st;                        // halos
    }
    const int64_t H1 = p->N[0] / 2 + 1;
    {
        StageTimer tm(p, EV_FFT);
        const cufftResult r =
            p->prec == NUFFT_F64
                ? cufftExecD2Z(d->fft2r, reinterpret_cast<cufftDoubleReal*>(g0),
                               static_cast<cufftDoubleComplex*>(d->hbuf))
                : cufftExecR2C(d->fft2r, reinterpret_cast<cufftReal*>(g0),
                               static_cast<cufftComplex*>(d->hbuf));                // F (x, y)
        if (r != CUFFT_SUCCESS) return NUFFT_ERR_CUFFT;
        NUFFT_CK(launch_xy_pack_half<T>(static_cast<const C*>(d->hbuf), p->nf, d->nzl, p->N, d->P,
                                        p->modeord, static_cast<C*>(d->xbuf), p->stream));
        if ((st = d->x->alltoall(d->xbuf, d->ybuf, 2 * (size_t)(d->nzl * d->NY * H1) * d->rs,
                                 p->stream)))
            return st;                                                              // transpose
        if ((st = fft_exec(p, d->fft1h, d->ybuf, -1))) return st;                   // F (z), sign -
    }
    StageTimer tm(p, EV_DECONV);
    NUFFT_CK(launch_z_deconv_half<T>(static_cast<const C*>(d->ybuf), p->nf, p->N, d->NY, d->y0,
                                     static_cast<const T*>(p->d_p[0]),
                                     static_cast<const T*>(p->d_p[1]),
                                     static_cast<const T*>(p->d_p[2]), p->modeord,
                                     p->iflag > 0 ? 1 : 0, static_cast<C*>(fk_local),
                                     p->stream));                                  // chi (z), D
    return NUFFT_OK;
}

template <typename T>
int type2_real_t(nufft_plan_s* p, const void* fk_local, void* c_local) {
    using C = typename Cx<T>::type;
    DistState* d = p->dist;
    int st;
    const int64_t H1 = p->N[0] / 2 + 1;
    {
        StageTimer tm(p, EV_PAD);
        // type-2 sign -iflag; the C2R path applies +, so a - sign conjugates the input
        NUFFT_CK(launch_z_pad_half<T>(static_cast<const C*>(fk_local), p->nf, p->N, d->NY, d->y0,
                                      static_cast<const T*>(p->d_p[0]),
                                      static_cast<const T*>(p->d_p[1]),
                                      static_cast<const T*>(p->d_p[2]), p->modeord,
                                      p->iflag > 0 ? 1 : 0, static_cast<C*>(d->ybuf),
                                      p->stream));                                 // D, chi^T (z)
    }
    T* g0 = real_grid0<T>(p);
    {
        StageTimer tm(p, EV_FFT);
        if ((st = fft_exec(p, d->fft1h, d->ybuf, +1))) return st;                   // F^-1 (z)
        if ((st = d->x->alltoall(d->ybuf, d->xbuf, 2 * (size_t)(d->nzl * d->NY * H1) * d->rs,
                                 p->stream)))
            return st;                                                              // transpose
        NUFFT_CK(launch_xy_unpad_half<T>(static_cast<const C*>(d->xbuf), p->nf, d->nzl, p->N,
                                         d->P, p->modeord, static_cast<C*>(d->hbuf), p->stream));
        const cufftResult r =
            p->prec == NUFFT_F64
                ? cufftExecZ2D(d->fft2c, static_cast<cufftDoubleComplex*>(d->hbuf),
                               reinterpret_cast<cufftDoubleReal*>(g0))
                : cufftExecC2R(d->fft2c, static_cast<cufftComplex*>(d->hbuf),
                               reinterpret_cast<cufftReal*>(g0));                  // F^-1 (x, y)
        if (r != CUFFT_SUCCESS) return NUFFT_ERR_CUFFT;
    }
    {
        StageTimer tm(p, EV_COMM);
        if ((st = halo_fill<T>(p, g0, 1))) return st;                              // halos
    }
    return do_interp_real(p, g0, c_local);                                         // C^T
}

}  // namespace

int dist_init(nufft_plan_s* p) {
    NufftComm* cm = static_cast<NufftComm*>(p->comm);
    const int P = cm->nranks, r = cm->rank;
    if (P < 2 || p->nf[2] % P != 0 || p->N[1] % P != 0) return NUFFT_ERR_UNSUPPORTED;
    DistState* d = new (std::nothrow) DistState();
    if (!d) return NUFFT_ERR_ALLOC;
    p->dist = d;
    d->P = P;
    d->r = r;
    d->x = cm->x;
    d->rs = p->real_size;
    d->nzl = p->nf[2] / P;
    d->NY = p->N[1] / P;
    d->y0 = (int64_t)r * d->NY;
    // halo planes: a stencil of a point whose cell lies in [z_lo, z_hi) reaches
    // [z_lo - floor(w/2), z_hi - 1 + ceil(w/2)] (reading R4)
    d->hlo = p->w / 2;
    d->hhi = (p->w + 1) / 2;
    if (d->nzl < d->hhi) return NUFFT_ERR_UNSUPPORTED;  // halos reach only the two neighbours
    d->plane = p->nf[0] * p->nf[1];
    Geom& g = p->geom;
    g.z_lo = (int64_t)r * d->nzl;
    g.nz_loc = d->nzl;
    g.zper = 0;
    g.hz_lo = d->hlo;
    g.hz_hi = d->hhi;
    if (g.T[2] > d->nzl) {
        if (g.nsub > 1) {  // sub-bin plans keep T + 1 = ns G: drop whole sub-bins in z
            g.ns[2] = std::max(1, (int)((d->nzl + 1) / g.Gs[2]));
            g.T[2] = g.ns[2] * g.Gs[2] - 1;
            g.nsub = g.ns[0] * g.ns[1] * g.ns[2];
        } else {
            g.T[2] = (int)d->nzl;
        }
        // rows / outer products need T = 16 - w on every axis
        if (g.spread_warps >= 1 && g.spread_warps <= 3) g.spread_warps = 8;
    }
    g.nb[2] = (int)((d->nzl + g.T[2] - 1) / g.T[2]);
    p->nbins = (int64_t)g.nb[0] * g.nb[1] * g.nb[2];

    int st = NUFFT_OK;
    const size_t cs = p->cplx_size;
    p->grid_bytes = (size_t)(d->plane * (d->hlo + d->nzl + d->hhi)) * cs;
    if ((st = dev_alloc(p, &p->d_grid, p->grid_bytes))) return st;
    p->grid0 = static_cast<char*>(p->d_grid) + (size_t)(d->plane * d->hlo) * cs;
    d->xfer_bytes = (size_t)(d->nzl * p->N[1] * p->N[0]) * cs;
    if ((st = dev_alloc(p, &d->xbuf, d->xfer_bytes))) return st;
    if ((st = dev_alloc(p, &d->ybuf, d->xfer_bytes))) return st;
    if ((st = dev_alloc(p, &d->halo_a, (size_t)(d->plane * d->hlo) * cs))) return st;
    if ((st = dev_alloc(p, &d->halo_b, (size_t)(d->plane * d->hhi) * cs))) return st;
    if ((st = dev_alloc(p, (void**)&d->d_counts, sizeof(unsigned long long) * P))) return st;
    if ((st = dev_alloc(p, (void**)&d->d_rcounts, sizeof(unsigned long long) * P))) return st;
    if ((st = dev_alloc(p, (void**)&d->d_off, sizeof(unsigned long long) * P))) return st;
    if ((st = dev_alloc(p, (void**)&d->d_mig, sizeof(unsigned long long) * (P + 3)))) return st;
    d->scount.assign(P, 0);
    d->soff.assign(P, 0);
    d->rcount.assign(P, 0);
    d->roff.assign(P, 0);

    const cufftType ty = p->prec == NUFFT_F64 ? CUFFT_Z2Z : CUFFT_C2C;
    // 2D (x, y) transforms of the nzl owned planes
    int n2[2] = {(int)p->nf[1], (int)p->nf[0]};
    if (cufftPlanMany(&d->fft2, 2, n2, nullptr, 1, (int)d->plane, nullptr, 1, (int)d->plane, ty,
                      (int)d->nzl) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    d->fft2_ok = true;
    // 1D z transforms of the S = NY N1 lines of this rank's y-block: element
    // (m3, line) at m3 S + line
    const int S = (int)(d->NY * p->N[0]);
    int n1[1] = {(int)p->nf[2]};
    int emb[1] = {(int)p->nf[2]};
    if (cufftPlanMany(&d->fft1, 1, n1, emb, S, 1, emb, S, 1, ty, S) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    d->fft1_ok = true;
    size_t ws = 0;
    cufftGetSize(d->fft2, &ws);
    p->bytes += ws;
    cufftGetSize(d->fft1, &ws);
    p->bytes += ws;
    if (cufftSetStream(d->fft2, p->stream) != CUFFT_SUCCESS ||
        cufftSetStream(d->fft1, p->stream) != CUFFT_SUCCESS)
        return NUFFT_ERR_CUFFT;
    return NUFFT_OK;
}

int64_t dist_user_np(nufft_plan_s* p) { return p->dist->redist ? p->dist->np_user : p->Np; }

int dist_local_modes(nufft_plan_s* p, int64_t lo[3], int64_t hi[3]) {
    DistState* d = p->dist;
    lo[0] = 0;
    hi[0] = p->N[0];
    lo[1] = d->y0;
    hi[1] = d->y0 + d->NY;
    lo[2] = 0;
    hi[2] = p->N[2];
    return NUFFT_OK;
}

// Collective agreement on a local status before an exchange: every rank learns
// whether ANY rank failed (allocation, size check), and all of them return an
// error together -- no rank is left waiting in a later ncclSend / ncclRecv.  A
// rank that did not fail itself reports NUFFT_ERR_NCCL ("a peer failed").
static int agree(nufft_plan_s* p, int local) {
    DistState* d = p->dist;
    unsigned long long flag = local >= 2 ? 1ull : 0ull;
    unsigned long long* f = d->d_mig + d->P + 2;
    NUFFT_CK(cudaMemcpyAsync(f, &flag, sizeof(flag), cudaMemcpyHostToDevice, p->stream));
    {
        const int e = d->x->allreduce_max_u64(f, p->stream);
        if (e) return e;
    }
    NUFFT_CK(cudaMemcpyAsync(&flag, f, sizeof(flag), cudaMemcpyDeviceToHost, p->stream));
    NUFFT_CK(cudaStreamSynchronize(p->stream));
    if (local >= 2) return local;
    return flag ? NUFFT_ERR_NCCL : NUFFT_OK;
}

int dist_setpts(nufft_plan_s* p, int64_t Np, const void* x, const void* y, const void* z) {
    DistState* d = p->dist;
    if (p->points_owned) {
        d->redist = false;
        d->np_user = Np;
        return local_sort(p, Np, x, y, z);
    }
    d->redist = true;
    int st;
    const int P = d->P;
    const size_t rs = p->real_size;
    // ---- owners and per-destination counts
    st = NUFFT_OK;
    if (Np > d->cap_user) {
        dev_free(p, (void**)&d->owner, 4 * d->cap_user);
        dev_free(p, (void**)&d->rank_in, 4 * d->cap_user);
        d->cap_user = 0;
        const int64_t cap = Np + Np / 8;
        st = dev_alloc(p, (void**)&d->owner, 4 * (size_t)cap);
        if (!st) st = dev_alloc(p, (void**)&d->rank_in, 4 * (size_t)cap);
        if (!st) d->cap_user = cap;
    }
    if ((st = agree(p, st))) return st;  // before the count all-to-all
    NUFFT_CK(cudaMemsetAsync(d->d_counts, 0, sizeof(unsigned long long) * P, p->stream));
    const Geom& g = p->geom;
    if (p->prec == NUFFT_F64)
        NUFFT_CK(launch_owner_count<double>(Np, static_cast<const double*>(z), g.L, g.scale[2],
                                            p->nf[2], (int)d->nzl, d->owner, d->rank_in,
                                            d->d_counts, p->stream));
    else
        NUFFT_CK(launch_owner_count<float>(Np, static_cast<const float*>(z), g.L, g.scale[2],
                                           p->nf[2], (int)d->nzl, d->owner, d->rank_in,
                                           d->d_counts, p->stream));
    {
        const int e = d->x->alltoall(d->d_counts, d->d_rcounts, sizeof(unsigned long long),
                                     p->stream);
        if (e) return e;
    }
    NUFFT_CK(cudaMemcpyAsync(d->scount.data(), d->d_counts, sizeof(unsigned long long) * P,
                             cudaMemcpyDeviceToHost, p->stream));
    NUFFT_CK(cudaMemcpyAsync(d->rcount.data(), d->d_rcounts, sizeof(unsigned long long) * P,
                             cudaMemcpyDeviceToHost, p->stream));
    NUFFT_CK(cudaStreamSynchronize(p->stream));  // receive sizes must be known on the host
    unsigned long long so = 0, ro = 0;
    for (int q = 0; q < P; ++q) {
        d->soff[q] = so;
        d->roff[q] = ro;
        so += d->scount[q];
        ro += d->rcount[q];
    }
    d->np_user = Np;
    d->np_local = (int64_t)ro;
    // ---- size check and staging buffers, agreed by every rank before any point moves
    st = d->np_local >= (int64_t)1 << 31 ? NUFFT_ERR_NPTS : NUFFT_OK;
    const size_t need_s = 3 * (size_t)Np * rs + 16, need_r = 3 * (size_t)d->np_local * rs + 16;
    if (!st) st = ensure(p, &d->sbuf, &d->sbuf_bytes, std::max(need_s, (size_t)Np * p->cplx_size + 16));
    if (!st)
        st = ensure(p, &d->rbuf, &d->rbuf_bytes,
                    std::max(need_r, (size_t)d->np_local * p->cplx_size + 16));
    if ((st = agree(p, st))) {
        d->np_local = 0;
        return st;
    }
    NUFFT_CK(cudaMemcpyAsync(d->d_off, d->soff.data(), sizeof(unsigned long long) * P,
                             cudaMemcpyHostToDevice, p->stream));
    // ---- move x, y, z (three rounds through the staging buffers)
    const void* src[3] = {x, y, z};
    for (int k = 0; k < 3; ++k) {
        char* sb = static_cast<char*>(d->sbuf) + (size_t)k * Np * rs;
        NUFFT_CK(launch_pack_bytes(Np, (int)rs, src[k], d->owner, d->rank_in, d->d_off, sb, false,
                                   p->stream));
    }
    if ((st = d->x->group_start())) return st;
    for (int k = 0; k < 3; ++k) {
        const char* sb = static_cast<const char*>(d->sbuf) + (size_t)k * Np * rs;
        char* rb = static_cast<char*>(d->rbuf) + (size_t)k * d->np_local * rs;
        for (int q = 0; q < P; ++q) {
            if (d->scount[q] &&
                (st = d->x->send(sb + d->soff[q] * rs, d->scount[q] * rs, q, p->stream)))
                return st;
            if (d->rcount[q] &&
                (st = d->x->recv(rb + d->roff[q] * rs, d->rcount[q] * rs, q, p->stream)))
                return st;
        }
    }
    if ((st = d->x->group_end(p->stream))) return st;
    const char* rb = static_cast<const char*>(d->rbuf);
    st = local_sort(p, d->np_local, rb, rb + (size_t)d->np_local * rs,
                    rb + 2 * (size_t)d->np_local * rs);
    return agree(p, st);  // later executes exchange again: fail together here
}

int dist_type1(nufft_plan_s* p, const void* c, void* fk) {
    DistState* d = p->dist;
    int st;
    const int64_t npu = dist_user_np(p);
    const void* cd = nullptr;
    if ((st = input_view(p, c, (size_t)npu * p->cplx_size, 0, (size_t)npu * p->cplx_size, &cd)))
        return st;
    const size_t fk_bytes = (size_t)(p->N[0] * d->NY * p->N[2]) * p->cplx_size;
    void* fkd = nullptr;
    bool staged = false;
    if ((st = output_view(p, fk, fk_bytes, &fkd, &staged))) return st;
    const void* c_local = cd;
    if (d->redist) {  // strengths follow their points
        StageTimer tm(p, EV_COMM);
        NUFFT_CK(launch_pack_bytes(npu, (int)p->cplx_size, cd, d->owner, d->rank_in, d->d_off,
                                   d->sbuf, false, p->stream));
        if ((st = alltoallv(d, d->sbuf, d->scount, d->soff, d->rbuf, d->rcount, d->roff,
                            p->cplx_size, p->stream)))
            return st;
        c_local = d->rbuf;
    }
    st = p->prec == NUFFT_F64 ? type1_t<double>(p, c_local, fkd) : type1_t<float>(p, c_local, fkd);
    if (st) return st;
    return finish_output(p, fk, fkd, fk_bytes, staged);
}

int dist_type2(nufft_plan_s* p, const void* fk, void* c) {
    DistState* d = p->dist;
    int st;
    const int64_t npu = dist_user_np(p);
    const size_t fk_bytes = (size_t)(p->N[0] * d->NY * p->N[2]) * p->cplx_size;
    const void* fkd = nullptr;
    if ((st = input_view(p, fk, fk_bytes, 0, fk_bytes, &fkd))) return st;
    const size_t c_bytes = (size_t)npu * p->cplx_size;
    void* cd = nullptr;
    bool staged = false;
    if ((st = output_view(p, c, c_bytes, &cd, &staged))) return st;
    void* c_local = d->redist ? d->rbuf : cd;
    st = p->prec == NUFFT_F64 ? type2_t<double>(p, fkd, c_local) : type2_t<float>(p, fkd, c_local);
    if (st) return st;
    if (d->redist) {  // results return to the caller's ranks and order
        StageTimer tm(p, EV_COMM);
        if ((st = alltoallv(d, d->rbuf, d->rcount, d->roff, d->sbuf, d->scount, d->soff,
                            p->cplx_size, p->stream)))
            return st;
        NUFFT_CK(launch_pack_bytes(npu, (int)p->cplx_size, d->sbuf, d->owner, d->rank_in,
                                   d->d_off, cd, true, p->stream));
    }
    return finish_output(p, c, cd, c_bytes, staged);
}

int dist_type1_real(nufft_plan_s* p, const void* c, void* fk) {
    DistState* d = p->dist;
    int st;
    if ((st = ensure_real_dist(p))) return st;
    const int64_t npu = dist_user_np(p);
    const size_t rs = p->real_size;
    const void* cd = nullptr;
    if ((st = input_view(p, c, (size_t)npu * rs, 0, (size_t)npu * rs, &cd))) return st;
    const size_t fk_bytes = (size_t)((p->N[0] / 2 + 1) * d->NY * p->N[2]) * p->cplx_size;
    void* fkd = nullptr;
    bool staged = false;
    if ((st = output_view(p, fk, fk_bytes, &fkd, &staged))) return st;
    const void* c_local = cd;
    if (d->redist) {  // strengths follow their points
        StageTimer tm(p, EV_COMM);
        NUFFT_CK(launch_pack_bytes(npu, (int)rs, cd, d->owner, d->rank_in, d->d_off, d->sbuf,
                                   false, p->stream));
        if ((st = alltoallv(d, d->sbuf, d->scount, d->soff, d->rbuf, d->rcount, d->roff, rs,
                            p->stream)))
            return st;
        c_local = d->rbuf;
    }
    st = p->prec == NUFFT_F64 ? type1_real_t<double>(p, c_local, fkd)
                              : type1_real_t<float>(p, c_local, fkd);
    if (st) return st;
    return finish_output(p, fk, fkd, fk_bytes, staged);
}

int dist_type2_real(nufft_plan_s* p, const void* fk, void* c) {
    DistState* d = p->dist;
    int st;
    if ((st = ensure_real_dist(p))) return st;
    const int64_t npu = dist_user_np(p);
    const size_t rs = p->real_size;
    const size_t fk_bytes = (size_t)((p->N[0] / 2 + 1) * d->NY * p->N[2]) * p->cplx_size;
    const void* fkd = nullptr;
    if ((st = input_view(p, fk, fk_bytes, 0, fk_bytes, &fkd))) return st;
    const size_t c_bytes = (size_t)npu * rs;
    void* cd = nullptr;
    bool staged = false;
    if ((st = output_view(p, c, c_bytes, &cd, &staged))) return st;
    void* c_local = d->redist ? d->rbuf : cd;
    st = p->prec == NUFFT_F64 ? type2_real_t<double>(p, fkd, c_local)
                              : type2_real_t<float>(p, fkd, c_local);
    if (st) return st;
    if (d->redist) {  // results return to the caller's ranks and order
        StageTimer tm(p, EV_COMM);
        if ((st = alltoallv(d, d->rbuf, d->rcount, d->roff, d->sbuf, d->scount, d->soff, rs,
                            p->stream)))
            return st;
        NUFFT_CK(launch_pack_bytes(npu, (int)rs, d->sbuf, d->owner, d->rank_in, d->d_off, cd,
                                   true, p->stream));
    }
    return finish_output(p, c, cd, c_bytes, staged);
}

void dist_destroy(nufft_plan_s* p) {
    DistState* d = p->dist;
    if (!d) return;
    if (d->fft2_ok) cufftDestroy(d->fft2);
    if (d->fft1_ok) cufftDestroy(d->fft1);
    if (d->real_ok) {
        cufftDestroy(d->fft2r);
        cufftDestroy(d->fft2c);
        cufftDestroy(d->fft1h);
    }
    dev_free(p, &d->hbuf, 0);
    dev_free(p, &d->xbuf, 0);
    dev_free(p, &d->ybuf, 0);
    dev_free(p, &d->halo_a, 0);
    dev_free(p, &d->halo_b, 0);
    dev_free(p, (void**)&d->d_counts, 0);
    dev_free(p, (void**)&d->d_rcounts, 0);
    dev_free(p, (void**)&d->d_off, 0);
    dev_free(p, (void**)&d->owner, 0);
    dev_free(p, (void**)&d->rank_in, 0);
    dev_free(p, &d->sbuf, 0);
    dev_free(p, &d->rbuf, 0);
    dev_free(p, (void**)&d->d_mig, 0);
    dev_free(p, &d->mig_send, 0);
    dev_free(p, &d->mig_recv, 0);
    dev_free(p, &d->mig_idx, 0);
    delete d;
    p->dist = nullptr;
}

// PIF particle migration: particles that drifted out of this rank's slab move to
// their owner; the rest are compacted in place.  Only the leavers (a small
// fraction per step) are copied or sent.
template <typename T>
int migrate_t(nufft_plan_s* p, int64_t* np, int64_t cap, T* const st[6]) {
    DistState* d = p->dist;
    const int P = d->P;
    const int64_t n = *np;
    const Geom& g = p->geom;
    const size_t rs = sizeof(T);
    NUFFT_CK(cudaMemsetAsync(d->d_counts, 0, sizeof(unsigned long long) * P, p->stream));
    NUFFT_CK(launch_migrate_count<T>(n, st[2], g.L, g.scale[2], p->nf[2], (int)d->nzl, d->r,
                                     d->d_counts, p->stream));
    {
        const int e = d->x->alltoall(d->d_counts, d->d_rcounts, sizeof(unsigned long long),
                                     p->stream);
        if (e) return e;
    }
    NUFFT_CK(cudaMemcpyAsync(d->scount.data(), d->d_counts, sizeof(unsigned long long) * P,
                             cudaMemcpyDeviceToHost, p->stream));
    NUFFT_CK(cudaMemcpyAsync(d->rcount.data(), d->d_rcounts, sizeof(unsigned long long) * P,
                             cudaMemcpyDeviceToHost, p->stream));
    NUFFT_CK(cudaStreamSynchronize(p->stream));
    unsigned long long so = 0, ro = 0;
    for (int q = 0; q < P; ++q) {
        d->soff[q] = so;
        d->roff[q] = ro;
        so += d->scount[q];
        ro += d->rcount[q];
    }
    const int64_t nleave = (int64_t)so, nrecv = (int64_t)ro;
    // every rank must agree before any particle moves: a rank without room (or
    // without staging memory) fails the call on ALL ranks, state untouched
    int s = (n - nleave + nrecv > cap) ? NUFFT_ERR_NPTS : NUFFT_OK;
    if (!s) s = ensure(p, &d->mig_send, &d->mig_send_bytes, 6 * (size_t)nleave * rs + 16);
    if (!s) s = ensure(p, &d->mig_recv, &d->mig_recv_bytes, 6 * (size_t)nrecv * rs + 16);
    if (!s) s = ensure(p, &d->mig_idx, &d->mig_idx_bytes, 3 * (size_t)nleave * 8 + 16);
    if ((s = agree(p, s))) return s == NUFFT_ERR_NCCL ? NUFFT_ERR_NPTS : s;
    NUFFT_CK(cudaMemcpyAsync(d->d_off, d->soff.data(), sizeof(unsigned long long) * P,
                             cudaMemcpyHostToDevice, p->stream));
    NUFFT_CK(cudaMemsetAsync(d->d_mig, 0, sizeof(unsigned long long) * (P + 2), p->stream));
    int64_t* idx = static_cast<int64_t*>(d->mig_idx);
    T* send = static_cast<T*>(d->mig_send);
    T* recv = static_cast<T*>(d->mig_recv);
    NUFFT_CK(launch_migrate_move<T>(n, nleave, nrecv, st, g.L, g.scale[2], p->nf[2], (int)d->nzl,
                                    d->r, d->d_off, d->d_mig, send, recv, idx, idx + nleave,
                                    idx + 2 * nleave, d->d_mig + P, 0, p->stream));
    {
        int e;
        if ((e = d->x->group_start())) return e;
        for (int q = 0; q < P; ++q) {
            if (d->scount[q] &&
                (e = d->x->send(send + 6 * d->soff[q], 6 * d->scount[q] * rs, q, p->stream)))
                return e;
            if (d->rcount[q] &&
                (e = d->x->recv(recv + 6 * d->roff[q], 6 * d->rcount[q] * rs, q, p->stream)))
                return e;
        }
        if ((e = d->x->group_end(p->stream))) return e;
    }
    NUFFT_CK(launch_migrate_move<T>(n, nleave, nrecv, st, g.L, g.scale[2], p->nf[2], (int)d->nzl,
                                    d->r, d->d_off, d->d_mig, send, recv, idx, idx + nleave,
                                    idx + 2 * nleave, d->d_mig + P, 1, p->stream));
    *np = n - nleave + nrecv;
    return NUFFT_OK;
}

}  // namespace nufft

extern "C" {

int nufft_pif_migrate(nufft_handle p, int64_t* np, int64_t cap, void* x, void* y, void* z,
                      void* vx, void* vy, void* vz) {
    if (!p || !np || *np < 0 || cap < *np) return NUFFT_ERR_ARG;
    if (!p->dist) return NUFFT_OK;  // one GPU: every particle is local
    if (*np > 0 && (!x || !y || !z || !vx || !vy || !vz)) return NUFFT_ERR_ARG;
    cudaGetLastError();
    if (p->prec == NUFFT_F64) {
        double* st[6] = {static_cast<double*>(x), static_cast<double*>(y), static_cast<double*>(z),
                         static_cast<double*>(vx), static_cast<double*>(vy), static_cast<double*>(vz)};
        return nufft::migrate_t<double>(p, np, cap, st);
    }
    float* st[6] = {static_cast<float*>(x), static_cast<float*>(y), static_cast<float*>(z),
                    static_cast<float*>(vx), static_cast<float*>(vy), static_cast<float*>(vz)};
    return nufft::migrate_t<float>(p, np, cap, st);
}

int nufft_comm_unique_id(char id[128]) {
    if (!id) return NUFFT_ERR_ARG;
    int st = NUFFT_OK;
    nufft::xport_nccl_unique_id(id, &st);
    return st;
}

int nufft_comm_init(const char id[128], int nranks, int rank, void** comm) {
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return NUFFT_ERR_ARG;
    NufftComm* c = new (std::nothrow) NufftComm();
    if (!c) return NUFFT_ERR_ALLOC;
    c->x = nufft::xport_nccl(id, nranks, rank);
    if (!c->x) {
        delete c;
        return NUFFT_ERR_NCCL;
    }
    c->nranks = nranks;
    c->rank = rank;
    *comm = c;
    return NUFFT_OK;
}

int nufft_comm_init_loopback(int nranks, void** comms) {
    if (!comms || nranks < 1) return NUFFT_ERR_ARG;
    std::vector<nufft::Xport*> xs((size_t)nranks, nullptr);
    int st = nufft::xport_loopback(nranks, xs.data());
    if (st) return st;
    for (int q = 0; q < nranks; ++q) {
        NufftComm* c = new (std::nothrow) NufftComm();
        if (!c) {
            for (int k = 0; k < q; ++k) delete static_cast<NufftComm*>(comms[k]);
            for (auto* x : xs) delete x;
            return NUFFT_ERR_ALLOC;
        }
        c->x = xs[(size_t)q];
        c->nranks = nranks;
        c->rank = q;
        comms[q] = c;
    }
    return NUFFT_OK;
}

int nufft_comm_destroy(void* comm) {
    if (!comm) return NUFFT_OK;
    NufftComm* c = static_cast<NufftComm*>(comm);
    delete c->x;  // NCCL: ncclCommDestroy; loopback: this rank's events
    delete c;
    return NUFFT_OK;
}

}  // extern "C"
