/*
 * nufft.h -- C ABI of libnufft.so, the B200-native (sm_100a) hot path of the
 * distributed 3D NUFFT of arXiv 2605.10678.
 *
 * The problem (§2, Eq. 1-2), points x_j in [0, L)^3, N_d even,
 * modes n in {-N_d/2 .. N_d/2-1}:
 *   type 1:  fk[n] = sum_j c_j exp(iflag * i (2 pi / L) n . x_j)
 *   type 2:  c_j   = sum_n fk[n] exp(-iflag * i (2 pi / L) n . x_j)
 * With iflag = -1 these are exactly Eq. (1) and Eq. (2) and the pair is adjoint
 * (PAPER.md:95, 123).  The library evaluates them by the paper's factorisation
 *   type 1 = D chi F C   (Eq. 3)
 *   type 2 = C^T F^-1 chi^T D   (Eq. 4)
 * with the ES window, sigma = 2 (fine grid nf_d = 2 N_d,
 * PAPER.md:141, 181) and w chosen from eps (reading R1).
 *
 * Conventions common to all calls
 * -------------------------------
 * Pointers.  Every array argument may be DEVICE memory (cudaMalloc / torch CUDA
 *   tensor) or HOST memory (pinned or pageable).  Host arrays are staged through
 *   plan-owned device buffers with cudaMemcpyAsync on the plan stream; when an
 *   OUTPUT is host memory the call returns only after the result is in it.  With
 *   device arrays every call is asynchronous (stream-ordered on opts.stream).
 * Layout.  Complex values are interleaved (re, im) pairs of the plan precision
 *   (float2 / double2 = torch.complex64 / complex128).  Coordinates are three
 *   separate real arrays (SoA) of the plan precision.  Mode arrays are
 *   N1 x N2 x N3 with x fastest: flat index (n1+N1/2) + N1 ((n2+N2/2) + N2 (n3+N3/2))
 *   for modeord 0 (centered, default); for modeord 1 (FFT order) index i_d holds
 *   n_d = i_d for i_d < N_d/2 and i_d - N_d otherwise.  Fine grids (nufft_spread /
 *   nufft_interp) are nf1 x nf2 x nf3 complex, x fastest, nf_d = 2 N_d.
 * Ownership.  The caller owns every array it passes and the stream.  setpts
 *   COPIES what it needs (sorted point records), so x, y, z may be reused once the
 *   stream has passed the call.  The plan owns its fine grid, bins, tables, cuFFT
 *   plan and staging buffers; nufft_destroy frees them.
 * Errors.  Every call returns an int status: 0 = NUFFT_OK, 1 = a warning
 *   (NUFFT_WARN_EPS_CLAMPED), >= 2 an error (enum below; nufft_strerror names it).
 *   No exception or exit() crosses the ABI.  Asynchronous CUDA faults surface as
 *   NUFFT_ERR_CUDA at a later call.  A handle is not re-entrant; distinct handles
 *   on distinct streams are independent.
 */
#ifndef NUFFT_B200_H
#define NUFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nufft_plan_s* nufft_handle;

enum { NUFFT_F32 = 0, NUFFT_F64 = 1 };

enum {
    NUFFT_OK = 0,
    NUFFT_WARN_EPS_CLAMPED = 1, /* eps outside [1e-15, 1e-1] (fp64) / [1e-7, 1e-1] (fp32): clamped */
    NUFFT_ERR_ARG = 2,          /* null handle / pointer, bad enum, bad option                      */
    NUFFT_ERR_MODES = 3,        /* some N_d odd, < 2, or 2 N_d < w + 3                               */
    NUFFT_ERR_NPTS = 4,         /* Np < 0 or Np >= 2^31 on one GPU                                  */
    NUFFT_ERR_NOT_SET = 5,      /* execute / spread / interp before setpts                           */
    NUFFT_ERR_ALLOC = 6,        /* device allocation failed                                          */
    NUFFT_ERR_CUDA = 7,         /* a CUDA runtime error (launch, copy, or an earlier async fault)    */
    NUFFT_ERR_CUFFT = 8,        /* cuFFT plan / exec failure                                         */
    NUFFT_ERR_NCCL = 9,         /* NCCL failure (distributed plans)                                  */
    NUFFT_ERR_UNSUPPORTED = 10  /* option combination not built                                      */
};

typedef struct {
    double L;          /* period of the torus [0, L)^3; default 2 pi                   */
    int modeord;       /* 0 = centered modes (default), 1 = FFT order                                 */
    void* stream;      /* cudaStream_t for every call of the plan; NULL = the legacy default stream */
    void* comm;        /* NULL = single GPU; else a communicator from nufft_comm_init (slab mode)    */
    int points_owned;  /* distributed: 1 = caller guarantees each point lies in this rank's z-slab   */
    int tile[3];       /* bin edge T_d (fine cells); 0 = built-in table by w; T_d + w + 2 <= 2 N_d  */
    int timing;        /* 1 = record per-stage CUDA events (read back by nufft_get_info)              */
    int spread_warps;  /* spread kernel: 0 = built-in choice; 1 = register rows, 2 = register outer   *
                        * products, 3 = tcgen05 tensor-core GEMM (3xTF32, fp32 complex only; all three   *
                        * need T_d = 16 - w); 4 / 8 = smem z-plane owners, that many warps;               *
                        * ablation only (complex transforms; real ones use 8): -1 = the paper's Atomic    *
                        * Spread, one thread per point in caller order, global atomics;*
                        * -2 = the same over the bin-sorted points; -3 = the paper's Tiled Spread       *
                        * (PAPER.md:203-206): shared-memory histogram, shared atomics, 4 z-slice teams/bin */
    int precompute;    /* ES weights of every point (3 w reals, sorted order) computed once by setpts and
                        * read by every execute / spread / interp instead of re-evaluating phi:
                        * 0 = auto (widths w >= 6, when the table fits in 1/4 of the device memory),
                        * 1 = always, -1 = never */
    int interp_method; /* 0 = tiled (subgrid staged in shared memory, default); ablation only (complex *
                        * type 2 / nufft_interp): 1 = the paper's Direct Interpolation, one thread per    *
                        * point in caller order reading global memory; 2 = the same   *
                        * over the bin-sorted points; 3 = the same along the Morton   *
                        * (Z-order) curve of the bins                                   */
    int fft_method;    /* fine-grid FFT of the complex transforms (one GPU): 0 = one (2N)^3 cuFFT + mode *
                        * truncation (default); 1 = the paper's pruned sigma = 2 split (PAPER.md:237-247,  *
                        * Eq. 7): eight N^3 transforms of the parity sub-grids read / written with stride *
                        * 2, twiddle combine (type 1) / conjugate-twiddle split (type 2) fused with D;     *
                        * needs one extra fine-grid-sized buffer.  Slab plans and real transforms: 0 only */
    int reserved[3];
} nufft_opts;

typedef struct {
    int precision;          /* NUFFT_F32 / NUFFT_F64                                  */
    int w;                  /* ES kernel width (cells)                                */
    double beta;            /* ES shape parameter                                     */
    double eps;             /* tolerance after clamping                               */
    int64_t N[3];           /* modes per axis                                         */
    int64_t nf[3];          /* fine grid per axis (= 2 N)                             */
    int tile[3];            /* bin edge per axis                                      */
    int64_t nbins;          /* number of bins                                         */
    int64_t Np;             /* points after setpts (this rank)                        */
    size_t device_bytes;    /* device memory owned by the plan                        */
    int nranks, rank;       /* 1, 0 on a single GPU                                   */
    int64_t slab_lo, slab_hi; /* fine z-planes owned by this rank                     */
    /* per-stage device milliseconds of the most recent calls (opts.timing = 1), else -1 */
    float ms_setpts, ms_spread, ms_fold, ms_fft, ms_deconv, ms_pad, ms_interp, ms_comm;
    int weights_precomputed; /* 1 if the last setpts stored the per-point ES weights     */
    int sub_bins;           /* sub-bins per bin (sub-bin sorted plans: spread_warps 5), else 1 */
} nufft_info;

/* Fills *o with the defaults (L = 2 pi, centered modes, default stream, single GPU). */
int nufft_default_opts(nufft_opts* o);

/* Create a plan (all precomputation "once during initialization").
 * N1, N2, N3: modes per axis (even, >= 2, 2 N_d >= w + 3).  iflag: sign of the type-1
 * exponent (-1 reproduces Eq. 1); type 2 uses -iflag.  eps: requested relative
 * l2 tolerance.  precision: NUFFT_F32 or NUFFT_F64.  opts may be NULL (defaults).
 * Host: computes w, beta, the deconvolution factors p_d(n) = 2 / (w phihat(pi n w / nf_d))
 * by Gauss-Legendre quadrature, allocates the fine grid and the cuFFT plan.
 * Blocks the host.  On success *out is a new handle. */
int nufft_plan(int64_t N1, int64_t N2, int64_t N3, int iflag, double eps, int precision,
               const nufft_opts* opts, nufft_handle* out);

/* Set the nonuniform points: fold onto [0, L)^3, bin-sort
 * them by tile (counting sort with warp-level prefix scans), store sorted per-point
 * stencil records.  x, y, z: Np reals each of the plan precision, device or host.
 * Distributed plans: collective over the communicator; points are redistributed
 * to their owning z-slab unless opts.points_owned (blocks the host for the counts).
 * A local failure (allocation, >= 2^31 points arriving on one rank) is agreed by an
 * all-reduce before any point moves: the failing rank returns its own code, every
 * other rank NUFFT_ERR_NCCL, and no rank is left waiting in the exchange. */
int nufft_setpts(nufft_handle h, int64_t Np, const void* x, const void* y, const void* z);

/* Type-1 NUFFT (Eq. 3): c = Np complex strengths (caller order), fk = N1 N2 N3 complex out.
 * Spread (C) -> FFT with sign iflag (F) -> truncate (chi) + deconvolve (D), fused. */
int nufft_execute_type1(nufft_handle h, const void* c, void* fk);

/* Type-2 NUFFT (Eq. 4): fk = N1 N2 N3 complex in, c = Np complex out in caller order.
 * Pre-correct (D) + zero-pad (chi^T), fused -> FFT with sign -iflag -> interpolate (C^T). */
int nufft_execute_type2(nufft_handle h, const void* fk, void* c);

/* Real-valued transforms ("all implementations support real and complex-valued inputs",
 * PAPER.md:198).  Same plan, same points; the spread / interp grid is REAL and the FFT
 * runs on its half spectrum (R2C / C2R), halving grid bytes, FFT work and FMAs.
 * One GPU (full mode layout, N1 N2 N3 as for the complex calls):
 *   type1_real: c = Np REAL strengths; fk = N1 N2 N3 complex out, identical in value to
 *               nufft_execute_type1 with c + 0i (Hermitian where n and -n are stored).
 *   type2_real: fk = N1 N2 N3 complex in; c = Np REAL out, c_j = Re(sum_n fk[n]
 *               exp(-iflag i (2 pi / L) n . x_j)) -- the real part of nufft_execute_type2.
 * Slab plan (HALF-SPECTRUM layout: x index i1 = k1 in [0, N1/2] (N1/2 + 1 values), the
 * rank's y-block and all z as in nufft_local_modes, x fastest) -- nothing crosses ranks:
 *   type1_real: fk holds the type-1 values at k1 = 0 .. N1/2 (k1 = N1/2 is the conjugate
 *               partner of -N1/2; the k1 < 0 half is conj fk[-k]).
 *   type2_real: fk is the k1 >= 0 half of a Hermitian spectrum; c_j = the sum over its
 *               Hermitian completion (the k1 = 0 plane enters through its Hermitian part). */
int nufft_execute_type1_real(nufft_handle h, const void* c, void* fk);
int nufft_execute_type2_real(nufft_handle h, const void* fk, void* c);
/* Three real type-2 transforms on the same points at once (a vector field, e.g. the PIF
 * E field): fk0, fk1, fk2 as for type2_real; c = Np 3-vectors of reals,
 * interleaved (c[3j + d] = component d at point j).  The three C2R outputs are kept as
 * three real fine grids and gathered together with ONE evaluation of each point's weights.
 * DEVICE pointers only.  Single-GPU plans (NUFFT_ERR_UNSUPPORTED on a slab plan). */
int nufft_execute_type2_real3(nufft_handle h, const void* fk0, const void* fk1, const void* fk2,
                              void* c);

/* The spreading operator alone (Step 1): grid = C c on the periodic
 * nf1 x nf2 x nf3 fine grid (overwritten).  Single-GPU plans only. */
int nufft_spread(nufft_handle h, const void* c, void* grid);

/* The interpolation operator alone (C^T): c = C^T grid, caller order. */
int nufft_interp(nufft_handle h, const void* grid, void* c);

/* Free everything the plan owns.  Accepts NULL. */
int nufft_destroy(nufft_handle h);

/* Plan parameters and, with opts.timing, the last per-stage device times.  Blocks. */
int nufft_get_info(nufft_handle h, nufft_info* info);

/* Diagnostics (not a step of the method): the measured FMA-pipe peak of this GPU in
 * TFLOP/s (2 flops per FMA) for precision NUFFT_F32 / NUFFT_F64 -- the ALU roofline
 * denominator of bench.py ("measure on the box with an FMA
 * microbenchmark").  8 independent FMA chains per thread, 8 CTAs of 256 threads per SM,
 * CUDA-event timed on `stream` (cudaStream_t, NULL = default).  Blocks the host.
 * *tflops is host memory.  NUFFT_ERR_ARG for a bad precision / NULL tflops. */
int nufft_fma_peak(int precision, void* stream, double* tflops);

/* Static string for a status code (host). */
const char* nufft_strerror(int code);

/* ---- multi-GPU (one process per GPU; z-slab decomposition, §2.4) ----
 * nufft_comm_unique_id: rank 0 makes the 128-byte NCCL id (host); PyTorch only carries
 * it through its process group.  nufft_comm_init: collective over the nranks processes;
 * *comm is passed as opts.comm to nufft_plan; the caller destroys it after its plans.
 * A slab plan (opts.comm != NULL) needs nranks >= 2, 2 N3 and N2 divisible by nranks
 * and 2 N3 / nranks >= ceil(w/2).  Rank r owns fine z-planes [r 2N3/P, (r+1) 2N3/P);
 * nufft_setpts then moves every point to the rank owning its fine z-cell (unless
 * opts.points_owned) and type 2 returns values to the caller's rank and order.
 * Errors: NUFFT_ERR_NCCL for a failed NCCL call, NUFFT_ERR_UNSUPPORTED for a shape
 * that cannot be slab-decomposed.  nufft_spread / nufft_interp are single-GPU only. */
int nufft_comm_unique_id(char id[128]);                                    /* rank 0, host */
int nufft_comm_init(const char id[128], int nranks, int rank, void** comm); /* collective   */
int nufft_comm_destroy(void* comm);
/* Loopback communicators: nranks handles comms[0 .. nranks-1] (host array, filled) on
 * the CURRENT device, one per rank of a z-slab decomposition that runs entirely on one
 * GPU.  Each rank's plan calls must be issued from its own host thread (the calls are
 * collective: every exchange meets the other ranks' threads), on the rank's own
 * stream; messages are device-to-device copies.  Same plan semantics and results as
 * NCCL communicators at any nranks -- a test / validation transport, not a
 * performance path.  Destroy each handle with nufft_comm_destroy after its plan. */
int nufft_comm_init_loopback(int nranks, void** comms);
/* This rank's [lo, hi) range of mode STORAGE indices per axis (x, y, z): the whole
 * N1 N2 N3 block on one GPU; on a slab plan all of x and z and the y-slab
 * [r N2/P, (r+1) N2/P).  fk arguments of a slab plan are that block, x fastest. */
int nufft_local_modes(nufft_handle h, int64_t lo[3], int64_t hi[3]);

/* ---- Particle-in-Fourier step helpers (§4) ----
 * DEVICE pointers only; stream-ordered on the plan stream; precision of the plan. */
/* Gauss's law in Fourier space on this rank's mode block (nufft_local_modes layout):
 *   E_k = -i k rho_k / |k|^2, k = 2 pi n / L, E_0 = 0.  rho_k, ex_k, ey_k, ez_k: complex. */
int nufft_pif_poisson(nufft_handle h, const void* rho_k, void* ex_k, void* ey_k, void* ez_k);
/* The same on the mode layout of the plan's REAL transforms (the half spectrum on a slab
 * plan, the full box on one GPU). */
int nufft_pif_poisson_real(nufft_handle h, const void* rho_k, void* ex_k, void* ey_k, void* ez_k);
/* Leapfrog kick of one velocity component: v[j] += scale * Re(e[j]), j < Np (e complex,
 * e.g. a type-2 output; scale = (q/m) dt / L^3). */
int nufft_pif_kick(nufft_handle h, int64_t Np, void* v, const void* e, double scale);
/* Field gather fused with the kick: v_d[j] += scale E_d(x_j) for
 * d = x, y, z, where E_d = type2_real(e_k[d]) -- nufft_execute_type2_real3 whose output
 * stage adds into the velocities (no field array).  Single-GPU plans.  Measured slower
 * than three nufft_execute_type2_real + nufft_pif_kick_real at C4 on B200 (the three
 * component tiles halve the resident CTAs), so the PIF driver does not use it by default. */
int nufft_pif_gather_kick(nufft_handle h, const void* ex_k, const void* ey_k, const void* ez_k,
                          void* vx, void* vy, void* vz, double scale);
/* The same kick from a REAL field sample e (Np reals, e.g. a nufft_execute_type2_real output). */
int nufft_pif_kick_real(nufft_handle h, int64_t Np, void* v, const void* e, double scale);
/* Drift: x += v dt on each axis, folded onto [0, L). */
int nufft_pif_drift(nufft_handle h, int64_t Np, void* x, void* y, void* z, const void* vx,
                    const void* vy, const void* vz, double dt);
/* Particle migration for a slab plan created with opts.points_owned = 1 (PAPER.md:229-235:
 * "particles are partitioned according to the same spatial decomposition" as the grid).
 * Collective over the plan's ranks.  In: this rank's *np particles (x y z vx vy vz, six
 * device arrays of capacity cap >= *np).  Every particle whose fine z-cell lies outside
 * this rank's slab is sent to its owner (NCCL send/recv of the leavers only); the staying
 * particles are compacted into [0, *np - leavers) in place (their order may change) and
 * the arrivals appended.  Out: *np = the new local count.  An error on EVERY rank if any
 * rank's new count would exceed its cap or its staging allocation fails (agreed
 * collectively before anything moves, all particles stay where they were):
 * NUFFT_ERR_NPTS, or NUFFT_ERR_ALLOC on the rank whose allocation failed.  On a one-GPU
 * plan: no-op. */
int nufft_pif_migrate(nufft_handle h, int64_t* np, int64_t cap, void* x, void* y, void* z,
                      void* vx, void* vy, void* vz);

#ifdef __cplusplus
}
#endif
#endif /* NUFFT_B200_H */
