/*
 * oracle/nufft_oracle.cpp -- plain, slow, obviously-correct CPU oracle for the
 * 3D type-1 / type-2 NUFFT of arXiv 2605.10678 ("A Performance-Portable,
 * Massively Parallel Distributed Nonuniform FFT", PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  It
 * shares no code, header, table or constant generator with the CUDA product
 * path (paper_2605_10678_b200/), and neither side includes the other.
 *
 * Everything is fp64 (the paper's precision).  Each function
 * cites the passage it follows; readings of silent / ambiguous points are
 * numbered R1..R12 and listed in DESIGN.md section "Readings of the paper".
 *
 * Two parts:
 *   O-NUDFT -- the exact definitions, Eq. (1) and Eq. (2);
 *   O-NUFFT -- the window-based approximation step by step in the paper's order:
 *              type 1 = D chi F C  (Eq. 3, Steps 1-4),
 *              type 2 = C^T F^-1 chi^T D (Eq. 4).
 *
 * Pins (tests/test_oracle_*.py, all `-m "not gpu"`): closed forms of phi and
 * phihat(beta=0); phihat against scipy.integrate.quad; the FFT against
 * numpy.fft; the NUDFT against numpy.fft for on-grid points and against the
 * one-particle closed form; the NUFFT against the NUDFT within 10*eps over an
 * eps sweep; type-1/type-2 adjointness; truncate/pad index sets.
 *
 * Parallelism (OpenMP) never changes results: spreading is partitioned by
 * OUTPUT z-plane (each thread owns disjoint planes and visits points in index
 * order), every other loop is over independent outputs.  Wrapped node indices
 * are computed once per point (not per cell); the sums are unchanged.  The
 * sampled NUDFT evaluates only the per-axis phases its modes use.
 * Build: g++ -O2 -ffp-contract=off -fno-fast-math -fcx-limited-range (the last
 * drops only the NaN/Inf recovery path of complex multiplication, which finite
 * inputs never take).
 */
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef std::complex<double> cplx;

static const double kPi = 3.14159265358979323846264338327950288;

extern "C" {

/* ---------------------------------------------------------------------------
 * Threads
 * ------------------------------------------------------------------------- */
int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---------------------------------------------------------------------------
 * Window parameters.  PAPER.md:181 (§2.1): "we use sigma = 2 and select w such
 * that the aliasing error satisfies the tolerance" (deferring to Barnett 2019).
 * Reading R1: w = ceil(log10(1/eps)) + 1 clamped to [2, 16]; beta = 2.30 * w.
 * Returns 0 on success, 1 if eps was outside [1e-15, 1e-1] and was clamped.
 * ------------------------------------------------------------------------- */
int orc_select_params(double eps, int* w_out, double* beta_out) {
    int status = 0;
    if (!(eps >= 1e-15)) { eps = 1e-15; status = 1; }
    if (eps > 1e-1) { eps = 1e-1; status = 1; }
    int w = (int)std::ceil(std::log10(1.0 / eps)) + 1;
    if (w < 2) w = 2;
    if (w > 16) w = 16;
    *w_out = w;
    *beta_out = 2.30 * (double)w;
    return status;
}

/* ---------------------------------------------------------------------------
 * ES window, PAPER.md:167-173 (§2.1):
 *   phi(z) = exp(beta (sqrt(1 - z^2) - 1))  for |z| <= 1,  0 otherwise.
 * Reading R5: the endpoint |z| = 1 is inside the support (phi(+-1) = e^-beta).
 * ------------------------------------------------------------------------- */
double orc_phi(double z, double beta) {
    if (std::fabs(z) <= 1.0) return std::exp(beta * (std::sqrt(1.0 - z * z) - 1.0));
    return 0.0;
}

/* ---------------------------------------------------------------------------
 * Gauss-Legendre nodes / weights on [-1, 1] by Newton iteration on P_n
 * (textbook construction; used only by orc_phihat).
 * ------------------------------------------------------------------------- */
static void gauss_legendre(int n, std::vector<double>& t, std::vector<double>& wt) {
    t.assign(n, 0.0);
    wt.assign(n, 0.0);
    for (int i = 0; i < n; ++i) {
        double x = std::cos(kPi * (i + 0.75) / (n + 0.5));  /* initial guess */
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;                        /* P_0, P_1 */
            for (int k = 2; k <= n; ++k) {                  /* three-term recurrence */
                double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1.0);         /* P_n'(x) */
            double dx = p1 / dp;
            x -= dx;
            if (std::fabs(dx) < 1e-16) break;
        }
        /* recompute derivative at the converged node */
        double p0 = 1.0, p1 = x;
        for (int k = 2; k <= n; ++k) {
            double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
            p0 = p1;
            p1 = p2;
        }
        dp = n * (x * p1 - p0) / (x * x - 1.0);
        t[i] = x;
        wt[i] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
}

/* ---------------------------------------------------------------------------
 * Fourier transform of the window, PAPER.md:178-179 (§2.1): "we compute phihat
 * numerically via Gauss-Legendre quadrature to machine precision".
 *   phihat(xi) = int_{-1}^{1} phi(z) cos(xi z) dz          (phi real and even)
 * Reading R7: the quadrature is done after the substitution z = sin(theta),
 *   phihat(xi) = int_{-pi/2}^{pi/2} e^{beta (cos theta - 1)} cos(xi sin theta) cos theta dtheta,
 * which removes the sqrt endpoint singularity (plain z-space GL at 64 nodes is
 * only ~1e-8 accurate at w = 3).  n_nodes <= 0 selects 128.
 * ------------------------------------------------------------------------- */
double orc_phihat(double xi, double beta, int n_nodes) {
    if (n_nodes <= 0) n_nodes = 128;
    std::vector<double> t, wt;
    gauss_legendre(n_nodes, t, wt);
    double sum = 0.0;
    for (int i = 0; i < n_nodes; ++i) {
        double theta = 0.5 * kPi * t[i];                    /* map [-1,1] -> [-pi/2, pi/2] */
        double f = std::exp(beta * (std::cos(theta) - 1.0)) * std::cos(xi * std::sin(theta)) *
                   std::cos(theta);
        sum += wt[i] * f;
    }
    return 0.5 * kPi * sum;                                 /* d theta = (pi/2) dt */
}

/* ---------------------------------------------------------------------------
 * Deconvolution factors D, PAPER.md:149-152 (Step 4): "entries proportional to
 * 1/phihat(k), including the normalization constants associated with the FFT
 * convention".  Reading R6: with the grid coordinate
 * s = x nf / L, psi(t) = phi(2t/w) and unnormalised FFTs,
 *     p(n) = 2 / (w * phihat(pi * n * w / nf)),   n = -N/2 .. N/2-1.
 * p[0..N-1] holds n = -N/2 .. N/2-1 in order.
 * ------------------------------------------------------------------------- */
void orc_deconv_factors(int64_t N, int64_t nf, int w, double beta, double* p) {
    for (int64_t i = 0; i < N; ++i) {
        int64_t n = i - N / 2;
        double xi = kPi * (double)n * (double)w / (double)nf;
        p[i] = 2.0 / ((double)w * orc_phihat(xi, beta, 0));
    }
}

/* ---------------------------------------------------------------------------
 * Fold a coordinate onto the torus and rescale to fine-grid units.
 * x_j in [0, L)^3.  Reading R10: any finite x is folded with
 * x - L floor(x/L); s = x * (nf / L); s >= nf is mapped to s - nf (guards
 * x = L - ulp).  Points already in [0, L) are unchanged by the fold.
 * ------------------------------------------------------------------------- */
static inline double fold_rescale(double x, double L, int64_t nf) {
    double xf = x - L * std::floor(x / L);
    double s = xf * ((double)nf / L);
    if (s >= (double)nf) s -= (double)nf;
    if (s < 0.0) s += (double)nf;
    return s;
}

static inline int64_t wrap(int64_t i, int64_t n) {
    int64_t r = i % n;
    return r < 0 ? r + n : r;
}

/* Per-axis stencil of one point, PAPER.md:187-196 (Eq. 6):
 * "a = i0 - ceil((w-1)/2)", support [a, a+w-1], separable weights.
 * Reading R4: a = ceil(s - w/2) (i0 = nearest node for odd w, ceil(s) for even w;
 * on a tie the left endpoint z = -1 is included).  Weight of node a+i is
 * phi(2 (a + i - s) / w).                                                     */
static inline int64_t stencil_1d(double s, int w, double beta, double* wts) {
    int64_t a = (int64_t)std::ceil(s - 0.5 * (double)w);
    for (int i = 0; i < w; ++i) {
        double zz = 2.0 * ((double)(a + i) - s) / (double)w;
        wts[i] = orc_phi(zz, beta);
    }
    return a;
}

/* ---------------------------------------------------------------------------
 * Step 1, spreading C (periodic ghost handling
 * PAPER.md:213): dense periodic accumulation onto the nf1 x nf2 x nf3 grid,
 *   b[(a1+i1) mod nf1, (a2+i2) mod nf2, (a3+i3) mod nf3] += c_j w1[i1] w2[i2] w3[i3].
 * Layout: grid index = m1 + nf1 (m2 + nf2 m3) (x fastest), interleaved complex.
 * Deterministic: threads own disjoint output z-planes and add in point order.
 * ------------------------------------------------------------------------- */
void orc_spread(int64_t Np, const double* x, const double* y, const double* z,
                const double* c, int64_t nf1, int64_t nf2, int64_t nf3, int w, double beta,
                double L, double* grid_out) {
    cplx* grid = reinterpret_cast<cplx*>(grid_out);
    const cplx* cc = reinterpret_cast<const cplx*>(c);
    std::memset(grid_out, 0, sizeof(cplx) * (size_t)(nf1 * nf2 * nf3));
    /* z stencil start of every point (a_3 = ceil(s_3 - w/2), the same expression
     * stencil_1d uses), so each thread can find the points that reach its planes
     * without evaluating weights for the others.                                 */
    std::vector<int64_t> a3v((size_t)Np);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < Np; ++j)
        a3v[(size_t)j] = (int64_t)std::ceil(fold_rescale(z[j], L, nf3) - 0.5 * (double)w);
#pragma omp parallel
    {
        int nth = 1, tid = 0;
#ifdef _OPENMP
        nth = omp_get_num_threads();
        tid = omp_get_thread_num();
#endif
        int64_t z0 = nf3 * tid / nth, z1 = nf3 * (tid + 1) / nth;   /* owned planes */
        std::vector<double> w1(w), w2(w), w3(w);
        std::vector<int64_t> m1(w), m2(w), m3(w);                    /* wrapped node indices */
        for (int64_t j = 0; j < Np; ++j) {
            /* does [a3, a3 + w) meet the owned planes, periodically?  (a3 lies in
             * [-w, nf3), so shifts by -nf3, 0, +nf3 cover every wrap)            */
            int64_t lo = a3v[(size_t)j], hi = lo + w;
            bool hit = false;
            for (int64_t sh = -nf3; sh <= nf3; sh += nf3)
                if (lo < z1 + sh && hi > z0 + sh) hit = true;
            if (!hit) continue;
            double s1 = fold_rescale(x[j], L, nf1);
            double s2 = fold_rescale(y[j], L, nf2);
            double s3 = fold_rescale(z[j], L, nf3);
            int64_t a1 = stencil_1d(s1, w, beta, w1.data());
            int64_t a2 = stencil_1d(s2, w, beta, w2.data());
            int64_t a3 = stencil_1d(s3, w, beta, w3.data());
            for (int i = 0; i < w; ++i) {
                m1[i] = wrap(a1 + i, nf1);
                m2[i] = wrap(a2 + i, nf2);
                m3[i] = wrap(a3 + i, nf3);
            }
            for (int i3 = 0; i3 < w; ++i3) {
                if (m3[i3] < z0 || m3[i3] >= z1) continue;
                for (int i2 = 0; i2 < w; ++i2) {
                    cplx* row = grid + nf1 * (m2[i2] + nf2 * m3[i3]);
                    for (int i1 = 0; i1 < w; ++i1)
                        row[m1[i1]] += cc[j] * (w1[i1] * w2[i2] * w3[i3]);
                }
            }
        }
    }
}

/* ---------------------------------------------------------------------------
 * Interpolation C^T: c_j = sum over the same stencil of
 * b[...] w1 w2 w3 -- exactly the transpose of orc_spread.
 * ------------------------------------------------------------------------- */
void orc_interp(int64_t Np, const double* x, const double* y, const double* z,
                const double* grid_in, int64_t nf1, int64_t nf2, int64_t nf3, int w,
                double beta, double L, double* c_out) {
    const cplx* grid = reinterpret_cast<const cplx*>(grid_in);
    cplx* out = reinterpret_cast<cplx*>(c_out);
#pragma omp parallel
    {
        std::vector<double> w1(w), w2(w), w3(w);
        std::vector<int64_t> m1(w), m2(w), m3(w);                    /* wrapped node indices */
#pragma omp for schedule(static)
        for (int64_t j = 0; j < Np; ++j) {
            int64_t a1 = stencil_1d(fold_rescale(x[j], L, nf1), w, beta, w1.data());
            int64_t a2 = stencil_1d(fold_rescale(y[j], L, nf2), w, beta, w2.data());
            int64_t a3 = stencil_1d(fold_rescale(z[j], L, nf3), w, beta, w3.data());
            for (int i = 0; i < w; ++i) {
                m1[i] = wrap(a1 + i, nf1);
                m2[i] = wrap(a2 + i, nf2);
                m3[i] = wrap(a3 + i, nf3);
            }
            cplx acc(0.0, 0.0);
            for (int i3 = 0; i3 < w; ++i3) {
                for (int i2 = 0; i2 < w; ++i2) {
                    const cplx* row = grid + nf1 * (m2[i2] + nf2 * m3[i3]);
                    for (int i1 = 0; i1 < w; ++i1)
                        acc += row[m1[i1]] * (w1[i1] * w2[i2] * w3[i3]);
                }
            }
            out[j] = acc;
        }
    }
}

/* ---------------------------------------------------------------------------
 * Step 2, the uniform FFT F, unnormalised, sign = +1 or -1:
 *   B[m] = sum_l b[l] exp(sign * 2 pi i m.l / nf).
 * Done axis by axis.  Each 1D line: textbook iterative radix-2 (bit reversal +
 * butterflies) when n is a power of two, otherwise the direct O(n^2) DFT.
 * Twiddles are computed directly with cos/sin (no recurrences).
 * ------------------------------------------------------------------------- */
static void dft_1d_direct(cplx* v, int64_t n, int sign) {
    std::vector<cplx> out(n);
    for (int64_t m = 0; m < n; ++m) {
        cplx acc(0.0, 0.0);
        for (int64_t l = 0; l < n; ++l) {
            double ang = (double)sign * 2.0 * kPi * (double)((m * l) % n) / (double)n;
            acc += v[l] * cplx(std::cos(ang), std::sin(ang));
        }
        out[m] = acc;
    }
    for (int64_t m = 0; m < n; ++m) v[m] = out[m];
}

static void fft_1d_radix2(cplx* v, int64_t n, int sign) {
    /* bit-reversal permutation */
    for (int64_t i = 1, j = 0; i < n; ++i) {
        int64_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(v[i], v[j]);
    }
    /* butterflies: len = 2, 4, ..., n */
    for (int64_t len = 2; len <= n; len <<= 1) {
        int64_t half = len >> 1;
        for (int64_t k = 0; k < half; ++k) {
            double ang = (double)sign * 2.0 * kPi * (double)k / (double)len;
            cplx tw(std::cos(ang), std::sin(ang));
            for (int64_t st = 0; st < n; st += len) {
                cplx u = v[st + k];
                cplx t = tw * v[st + k + half];
                v[st + k] = u + t;
                v[st + k + half] = u - t;
            }
        }
    }
}

static void transform_line(cplx* v, int64_t n, int sign) {
    if (n > 1 && (n & (n - 1)) == 0) fft_1d_radix2(v, n, sign);
    else dft_1d_direct(v, n, sign);
}

void orc_fft3d(double* data, int64_t n1, int64_t n2, int64_t n3, int sign) {
    cplx* g = reinterpret_cast<cplx*>(data);
    /* axis 1 (x, contiguous lines) */
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < n2 * n3; ++l) transform_line(g + l * n1, n1, sign);
    /* axis 2 (y) */
#pragma omp parallel
    {
        std::vector<cplx> line(n2);
#pragma omp for schedule(static)
        for (int64_t l = 0; l < n1 * n3; ++l) {
            int64_t i1 = l % n1, i3 = l / n1;
            for (int64_t i2 = 0; i2 < n2; ++i2) line[i2] = g[i1 + n1 * (i2 + n2 * i3)];
            transform_line(line.data(), n2, sign);
            for (int64_t i2 = 0; i2 < n2; ++i2) g[i1 + n1 * (i2 + n2 * i3)] = line[i2];
        }
    }
    /* axis 3 (z) */
#pragma omp parallel
    {
        std::vector<cplx> line(n3);
#pragma omp for schedule(static)
        for (int64_t l = 0; l < n1 * n2; ++l) {
            for (int64_t i3 = 0; i3 < n3; ++i3) line[i3] = g[l + n1 * n2 * i3];
            transform_line(line.data(), n3, sign);
            for (int64_t i3 = 0; i3 < n3; ++i3) g[l + n1 * n2 * i3] = line[i3];
        }
    }
}

/* ---------------------------------------------------------------------------
 * Steps 3 + 4: chi (mode extraction, index set of PAPER.md:245
 * {0..N/2-1} U {nf-N/2..nf-1}) and D:
 *   fk[n] = B[n mod nf] * p1(n1) p2(n2) p3(n3).
 * Mode layout (reading R9): centered n in [-N/2, N/2), flat index
 *   (n1+N1/2) + N1 ((n2+N2/2) + N2 (n3+N3/2))   (x fastest).
 * ------------------------------------------------------------------------- */
void orc_truncate_deconv(const double* grid_in, int64_t nf1, int64_t nf2, int64_t nf3,
                         int64_t N1, int64_t N2, int64_t N3, const double* p1,
                         const double* p2, const double* p3, double* fk_out) {
    const cplx* B = reinterpret_cast<const cplx*>(grid_in);
    cplx* fk = reinterpret_cast<cplx*>(fk_out);
#pragma omp parallel for schedule(static)
    for (int64_t i3 = 0; i3 < N3; ++i3) {
        int64_t m3 = wrap(i3 - N3 / 2, nf3);
        for (int64_t i2 = 0; i2 < N2; ++i2) {
            int64_t m2 = wrap(i2 - N2 / 2, nf2);
            for (int64_t i1 = 0; i1 < N1; ++i1) {
                int64_t m1 = wrap(i1 - N1 / 2, nf1);
                fk[i1 + N1 * (i2 + N2 * i3)] =
                    B[m1 + nf1 * (m2 + nf2 * m3)] * (p1[i1] * p2[i2] * p3[i3]);
            }
        }
    }
}

/* Type-2 mirror, Eq. (4) read right to left: D then chi^T
 * (zero padding; every fine cell outside the retained index set is zero).     */
void orc_pad_precorrect(const double* fk_in, int64_t N1, int64_t N2, int64_t N3,
                        const double* p1, const double* p2, const double* p3, int64_t nf1,
                        int64_t nf2, int64_t nf3, double* grid_out) {
    const cplx* fk = reinterpret_cast<const cplx*>(fk_in);
    cplx* B = reinterpret_cast<cplx*>(grid_out);
    std::memset(grid_out, 0, sizeof(cplx) * (size_t)(nf1 * nf2 * nf3));
#pragma omp parallel for schedule(static)
    for (int64_t i3 = 0; i3 < N3; ++i3) {
        int64_t m3 = wrap(i3 - N3 / 2, nf3);
        for (int64_t i2 = 0; i2 < N2; ++i2) {
            int64_t m2 = wrap(i2 - N2 / 2, nf2);
            for (int64_t i1 = 0; i1 < N1; ++i1) {
                int64_t m1 = wrap(i1 - N1 / 2, nf1);
                B[m1 + nf1 * (m2 + nf2 * m3)] =
                    fk[i1 + N1 * (i2 + N2 * i3)] * (p1[i1] * p2[i2] * p3[i3]);
            }
        }
    }
}

/* ---------------------------------------------------------------------------
 * O-NUFFT type 1, Eq. (3): fk = D chi F C c, sigma = 2
 * (nf = 2N, reading R8), FFT sign iflag (reading R11: iflag = -1 is Eq. 1).
 * Returns the orc_select_params status.  grid_scratch may be NULL.
 * ------------------------------------------------------------------------- */
int orc_type1(int64_t Np, const double* x, const double* y, const double* z, const double* c,
              int64_t N1, int64_t N2, int64_t N3, int iflag, double eps, double L,
              double* fk_out) {
    int w;
    double beta;
    int st = orc_select_params(eps, &w, &beta);
    int64_t nf1 = 2 * N1, nf2 = 2 * N2, nf3 = 2 * N3;
    std::vector<double> p1(N1), p2(N2), p3(N3);
    orc_deconv_factors(N1, nf1, w, beta, p1.data());
    orc_deconv_factors(N2, nf2, w, beta, p2.data());
    orc_deconv_factors(N3, nf3, w, beta, p3.data());
    std::vector<double> grid((size_t)(2 * nf1 * nf2 * nf3));
    orc_spread(Np, x, y, z, c, nf1, nf2, nf3, w, beta, L, grid.data());   /* Step 1: C   */
    orc_fft3d(grid.data(), nf1, nf2, nf3, iflag >= 0 ? 1 : -1);             /* Step 2: F   */
    orc_truncate_deconv(grid.data(), nf1, nf2, nf3, N1, N2, N3, p1.data(), /* Steps 3, 4 */
                        p2.data(), p3.data(), fk_out);
    return st;
}

/* O-NUFFT type 2, Eq. (4): c = C^T F^-1 chi^T D fk, the FFT with sign -iflag. */
int orc_type2(int64_t Np, const double* x, const double* y, const double* z, const double* fk,
              int64_t N1, int64_t N2, int64_t N3, int iflag, double eps, double L,
              double* c_out) {
    int w;
    double beta;
    int st = orc_select_params(eps, &w, &beta);
    int64_t nf1 = 2 * N1, nf2 = 2 * N2, nf3 = 2 * N3;
    std::vector<double> p1(N1), p2(N2), p3(N3);
    orc_deconv_factors(N1, nf1, w, beta, p1.data());
    orc_deconv_factors(N2, nf2, w, beta, p2.data());
    orc_deconv_factors(N3, nf3, w, beta, p3.data());
    std::vector<double> grid((size_t)(2 * nf1 * nf2 * nf3));
    orc_pad_precorrect(fk, N1, N2, N3, p1.data(), p2.data(), p3.data(), nf1, nf2, nf3,
                       grid.data());                                          /* D, chi^T */
    orc_fft3d(grid.data(), nf1, nf2, nf3, iflag >= 0 ? -1 : 1);               /* F^-1     */
    orc_interp(Np, x, y, z, grid.data(), nf1, nf2, nf3, w, beta, L, c_out);   /* C^T      */
    return st;
}

/* ---------------------------------------------------------------------------
 * O-NUDFT type 1, Eq. (1) (K_N of PAPER.md:113-120):
 *   fk[n] = sum_j c_j exp(iflag * i * (2 pi / L) n.x_j)
 * Per point and axis the phases exp(iflag i (2pi/L) n_d x_d) are computed
 * directly with cos/sin (no recurrence).  If sel != NULL only the nsel modes with
 * flat indices sel[k] are evaluated, into fk_out[k]; else all N1 N2 N3 modes.
 * ------------------------------------------------------------------------- */
static void phase_table(int64_t n, const double* x, int64_t N, const std::vector<int64_t>& idx,
                        int iflag, double L, std::vector<cplx>& e) {
    /* e[j K + k] = exp(iflag i (2 pi / L) n x_j) for the K centered mode indices
     * n = idx[k] - N/2 (idx = 0..N-1 for the full table).                       */
    int64_t K = (int64_t)idx.size();
    e.resize((size_t)(n * K));
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j)
        for (int64_t k = 0; k < K; ++k) {
            double ang = (double)iflag * (2.0 * kPi / L) * (double)(idx[(size_t)k] - N / 2) * x[j];
            e[(size_t)(j * K + k)] = cplx(std::cos(ang), std::sin(ang));
        }
}

/* Distinct per-axis indices used by the requested modes, and each mode's column in
 * the per-axis phase table (so a sampled NUDFT evaluates only the phases it needs). */
static void axis_columns(int64_t nout, const int64_t* sel, int64_t N, int64_t stride,
                         std::vector<int64_t>& idx, std::vector<int64_t>& col) {
    std::vector<int64_t> where((size_t)N, -1);
    idx.clear();
    col.assign((size_t)nout, 0);
    for (int64_t k = 0; k < nout; ++k) {
        int64_t flat = sel ? sel[k] : k;
        int64_t i = (flat / stride) % N;
        if (where[(size_t)i] < 0) {
            where[(size_t)i] = (int64_t)idx.size();
            idx.push_back(i);
        }
        col[(size_t)k] = where[(size_t)i];
    }
}

void orc_nudft1(int64_t Np, const double* x, const double* y, const double* z,
                const double* c, int64_t N1, int64_t N2, int64_t N3, int iflag, double L,
                int64_t nsel, const int64_t* sel, double* fk_out) {
    const cplx* cc = reinterpret_cast<const cplx*>(c);
    cplx* fk = reinterpret_cast<cplx*>(fk_out);
    int sgn = iflag >= 0 ? 1 : -1;
    int64_t nout = sel ? nsel : N1 * N2 * N3;
    for (int64_t k = 0; k < nout; ++k) fk[k] = cplx(0.0, 0.0);
    std::vector<int64_t> idx1, idx2, idx3, col1, col2, col3;
    axis_columns(nout, sel, N1, 1, idx1, col1);
    axis_columns(nout, sel, N2, N1, idx2, col2);
    axis_columns(nout, sel, N3, N1 * N2, idx3, col3);
    int64_t K1 = (int64_t)idx1.size(), K2 = (int64_t)idx2.size(), K3 = (int64_t)idx3.size();
    /* points in chunks so the phase tables stay small; sum over j in index order */
    const int64_t chunk = 2048;
    std::vector<cplx> e1, e2, e3;
    for (int64_t j0 = 0; j0 < Np; j0 += chunk) {
        int64_t n = Np - j0 < chunk ? Np - j0 : chunk;
        phase_table(n, x + j0, N1, idx1, sgn, L, e1);
        phase_table(n, y + j0, N2, idx2, sgn, L, e2);
        phase_table(n, z + j0, N3, idx3, sgn, L, e3);
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t k = 0; k < nout; ++k) {
            int64_t c1 = col1[(size_t)k], c2 = col2[(size_t)k], c3 = col3[(size_t)k];
            cplx acc(0.0, 0.0);
            for (int64_t j = 0; j < n; ++j)
                acc += cc[j0 + j] * e1[(size_t)(j * K1 + c1)] * e2[(size_t)(j * K2 + c2)] *
                       e3[(size_t)(j * K3 + c3)];
            fk[k] += acc;
        }
    }
}

/* O-NUDFT type 2, Eq. (2), sign -iflag:
 *   c_j = sum_n fk[n] exp(-iflag * i * (2 pi / L) n.x_j)
 * If sel != NULL only points sel[k] are evaluated, into c_out[k].              */
void orc_nudft2(int64_t Np, const double* x, const double* y, const double* z,
                const double* fk_in, int64_t N1, int64_t N2, int64_t N3, int iflag, double L,
                int64_t nsel, const int64_t* sel, double* c_out) {
    const cplx* fk = reinterpret_cast<const cplx*>(fk_in);
    cplx* out = reinterpret_cast<cplx*>(c_out);
    int sgn = iflag >= 0 ? -1 : 1;
    int64_t nout = sel ? nsel : Np;
#pragma omp parallel
    {
        std::vector<cplx> e1(N1), e2(N2), e3(N3);
#pragma omp for schedule(dynamic, 16)
        for (int64_t k = 0; k < nout; ++k) {
            int64_t j = sel ? sel[k] : k;
            for (int64_t i = 0; i < N1; ++i) {
                double a = (double)sgn * (2.0 * kPi / L) * (double)(i - N1 / 2) * x[j];
                e1[i] = cplx(std::cos(a), std::sin(a));
            }
            for (int64_t i = 0; i < N2; ++i) {
                double a = (double)sgn * (2.0 * kPi / L) * (double)(i - N2 / 2) * y[j];
                e2[i] = cplx(std::cos(a), std::sin(a));
            }
            for (int64_t i = 0; i < N3; ++i) {
                double a = (double)sgn * (2.0 * kPi / L) * (double)(i - N3 / 2) * z[j];
                e3[i] = cplx(std::cos(a), std::sin(a));
            }
            cplx acc(0.0, 0.0);
            for (int64_t i3 = 0; i3 < N3; ++i3)
                for (int64_t i2 = 0; i2 < N2; ++i2) {
                    cplx e23 = e2[i2] * e3[i3];
                    for (int64_t i1 = 0; i1 < N1; ++i1)
                        acc += fk[i1 + N1 * (i2 + N2 * i3)] * (e1[i1] * e23);
                }
            out[k] = acc;
        }
    }
}

/* O-NUDFT type 2, Eq. (2), for a rank-one (separable) mode array
 *   fk[n1, n2, n3] = a1[n1] a2[n2] a3[n3]:
 * the triple sum factors exactly into three 1D sums,
 *   c_j = A1(x_j) A2(y_j) A3(z_j),  A_d(t) = sum_n a_d[n] exp(-iflag i (2 pi / L) n t),
 * so the exact type-2 sum at a point costs O(N1 + N2 + N3) instead of O(N1 N2 N3)
 * (used to check full-size configurations, where the triple sum is out of reach).
 * a_d are centered (index n + N_d/2).  If sel != NULL only points sel[k].          */
void orc_nudft2_separable(int64_t Np, const double* x, const double* y, const double* z,
                          const double* a1_in, const double* a2_in, const double* a3_in,
                          int64_t N1, int64_t N2, int64_t N3, int iflag, double L,
                          int64_t nsel, const int64_t* sel, double* c_out) {
    const cplx* a1 = reinterpret_cast<const cplx*>(a1_in);
    const cplx* a2 = reinterpret_cast<const cplx*>(a2_in);
    const cplx* a3 = reinterpret_cast<const cplx*>(a3_in);
    cplx* out = reinterpret_cast<cplx*>(c_out);
    int sgn = iflag >= 0 ? -1 : 1;
    int64_t nout = sel ? nsel : Np;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t k = 0; k < nout; ++k) {
        int64_t j = sel ? sel[k] : k;
        const double* t[3] = {x, y, z};
        const cplx* a[3] = {a1, a2, a3};
        int64_t N[3] = {N1, N2, N3};
        cplx prod(1.0, 0.0);
        for (int d = 0; d < 3; ++d) {
            cplx acc(0.0, 0.0);
            for (int64_t i = 0; i < N[d]; ++i) {
                double ang = (double)sgn * (2.0 * kPi / L) * (double)(i - N[d] / 2) * t[d][j];
                acc += a[d][i] * cplx(std::cos(ang), std::sin(ang));
            }
            prod *= acc;
        }
        out[k] = prod;
    }
}

}  /* extern "C" */
