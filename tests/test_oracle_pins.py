"""Pins of the CPU oracle to things other than itself (all CPU, `-m "not gpu"`).

Each test names what fixes the expected value: a closed form, a library routine
(numpy.fft, scipy.integrate.quad), the exact NUDFT (itself pinned to numpy.fft
on grid-aligned points), an invariant, or a paper passage.  A plausible mistake
in the oracle -- a dropped term, a wrong sign or index, a transposed operand,
a wrong deconvolution constant -- fails at least one of them.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synthetic

TWO_PI = 2 * math.pi


def _pts(Np, L=TWO_PI, seed=1):
    x, y, z = synthetic.uniform_points(Np, L=L, seed=seed)
    return x.numpy(), y.numpy(), z.numpy()


def _c(Np, seed=2):
    return synthetic.strengths(Np, seed=seed).numpy()


# ---------------------------------------------------------------- generator
def test_splitmix64_matches_python_reference():
    cnt = [0, 1, 2, 12345, (1 << 40) ^ 7, (1 << 63) - 1]
    t = torch.tensor([synthetic._s64(c) for c in cnt], dtype=torch.int64)
    got = [int(v) & ((1 << 64) - 1) for v in synthetic.splitmix64(t).tolist()]
    assert got == [synthetic.splitmix64_py(c) for c in cnt]
    u = synthetic.u01(1, 0, 1000)
    assert float(u.min()) >= 0.0 and float(u.max()) < 1.0
    assert abs(float(u.mean()) - 0.5) < 0.05


def test_landau_points_are_distributed_as_the_paper_density():
    # density prop. to 1 + alpha cos(k x); the first Fourier
    # moment <cos(k x)> = alpha / 2 for this density on [0, 2pi/k).
    x, _, _ = synthetic.landau_points(200000, alpha=0.05, k=0.5)
    L = 2 * math.pi / 0.5
    assert float(x.min()) >= 0.0 and float(x.max()) < L
    m1 = float(torch.cos(0.5 * x).mean())
    assert abs(m1 - 0.025) < 0.004


# ---------------------------------------------------------------- window
def test_select_params_rule():
    # reading R1 (PAPER.md:181 defers the table; SPEC.md:60-62 examples)
    assert oracle.select_params(1e-2)[0] == 3
    assert oracle.select_params(1e-4)[0] == 5
    assert oracle.select_params(1e-6)[0] == 7
    assert oracle.select_params(1e-8)[0] == 9
    ws = [oracle.select_params(10.0 ** -k)[0] for k in range(1, 16)]
    assert ws == sorted(ws)
    w, beta, st = oracle.select_params(1e-20)
    assert st == 1 and w == 16
    assert oracle.select_params(1e-6)[1] == pytest.approx(16.1, abs=1e-12)


def test_phi_closed_forms():
    # PAPER.md:168-173
    for beta in (4.0, 11.5, 16.1):
        assert oracle.phi(0.0, beta) == 1.0
        assert oracle.phi(1.0, beta) == pytest.approx(math.exp(-beta), rel=1e-15)
        assert oracle.phi(-1.0, beta) == pytest.approx(math.exp(-beta), rel=1e-15)
        assert oracle.phi(1.5, beta) == 0.0
        assert oracle.phi(-1.0000001, beta) == 0.0
        for zz in (0.1, 0.37, 0.9):
            assert oracle.phi(zz, beta) == oracle.phi(-zz, beta)
        vals = [oracle.phi(t, beta) for t in np.linspace(0, 1, 50)]
        assert all(a > b for a, b in zip(vals, vals[1:]))


def test_phihat_beta0_closed_form():
    # beta = 0: phi = 1 on [-1, 1] -> phihat(xi) = 2 sin(xi)/xi
    assert oracle.phihat(0.0, 0.0) == pytest.approx(2.0, rel=1e-15)
    for xi in (0.3, 1.3, 3.9, 8.6):
        assert oracle.phihat(xi, 0.0) == pytest.approx(2 * math.sin(xi) / xi, rel=1e-13)


@pytest.mark.parametrize("beta", [6.9, 11.5, 16.1, 25.3])
@pytest.mark.parametrize("xi", [0.0, 1.3, 3.9, 8.6])
def test_phihat_against_scipy_quad(beta, xi):
    # library routine (adaptive Gauss-Kronrod, QUADPACK) on the z-space definition
    from scipy.integrate import quad

    def f(zz):
        return math.exp(beta * (math.sqrt(max(0.0, 1 - zz * zz)) - 1.0)) * math.cos(xi * zz)

    ref, err = quad(f, -1.0, 1.0, epsabs=1e-15, epsrel=1e-14, limit=400, points=[0.0])
    got = oracle.phihat(xi, beta)
    assert abs(got - ref) <= 1e-12 * abs(ref) + 1e-15
    # node doubling converged
    assert abs(oracle.phihat(xi, beta, 64) - oracle.phihat(xi, beta, 256)) <= 1e-13 * abs(ref)


def test_deconv_factors_symmetry_and_center():
    w, beta, _ = oracle.select_params(1e-6)
    N, nf = 16, 32
    p = oracle.deconv_factors(N, nf, w, beta)
    assert np.all(p > 0)
    # p(n) = p(-n) for |n| < N/2 (phihat even)
    for n in range(1, N // 2):
        assert p[N // 2 + n] == pytest.approx(p[N // 2 - n], rel=1e-15)
    assert p[N // 2] == pytest.approx(2.0 / (w * oracle.phihat(0.0, beta)), rel=1e-15)


# ---------------------------------------------------------------- FFT
@pytest.mark.parametrize("shape", [(8, 8, 8), (4, 8, 16), (6, 10, 12), (8, 6, 4)])
def test_fft3d_against_numpy(shape):
    rng = np.random.default_rng(0)
    g = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    n = g.size
    fwd = oracle.fft3d(g, -1)
    assert np.max(np.abs(fwd - np.fft.fftn(g))) <= 1e-12 * np.max(np.abs(fwd))
    inv = oracle.fft3d(g, +1)
    assert np.max(np.abs(inv - np.fft.ifftn(g) * n)) <= 1e-12 * np.max(np.abs(inv))


def test_fft3d_delta_constant_parseval():
    g = np.zeros((8, 8, 8), dtype=np.complex128)
    g[0, 0, 0] = 1.0
    assert np.allclose(oracle.fft3d(g, -1), 1.0, atol=1e-15)
    h = oracle.fft3d(np.full((8, 8, 8), 2.0 + 1.0j), 1)
    assert h[0, 0, 0] == pytest.approx((2.0 + 1.0j) * 512)
    h[0, 0, 0] = 0
    assert np.max(np.abs(h)) < 1e-12
    rng = np.random.default_rng(1)
    r = rng.standard_normal((8, 16, 4)) + 0j
    assert np.sum(np.abs(oracle.fft3d(r, -1)) ** 2) == pytest.approx(r.size * np.sum(np.abs(r) ** 2))


# ---------------------------------------------------------------- chi / D
def test_truncate_pad_index_sets_and_inverse():
    # retained indices {0..N/2-1} U {nf-N/2..nf-1} per axis
    N = (4, 6, 8)
    nf = (8, 12, 16)
    ones = [np.ones(n) for n in N]
    fk = np.ones((N[2], N[1], N[0]), dtype=np.complex128)
    g = oracle.pad_precorrect(fk, nf, ones)
    for axis, (n, m) in enumerate(zip(N, nf)):
        keep = set(range(n // 2)) | set(range(m - n // 2, m))
        prof = np.abs(g).sum(axis=tuple(a for a in range(3) if a != 2 - axis))
        assert {i for i in range(m) if prof[i] > 0} == keep
    rng = np.random.default_rng(2)
    f = rng.standard_normal(fk.shape) + 1j * rng.standard_normal(fk.shape)
    p = [rng.uniform(0.5, 2.0, n) for n in N]
    back = oracle.truncate_deconv(oracle.pad_precorrect(f, nf, [np.ones(n) for n in N]), N, p)
    expect = f * p[0][None, None, :] * p[1][None, :, None] * p[2][:, None, None]
    assert np.max(np.abs(back - expect)) < 1e-14
    # centered order: mode n=0 sits at flat index (N1/2, N2/2, N3/2); grid index 0
    g = np.zeros((nf[2], nf[1], nf[0]), dtype=np.complex128)
    g[0, 0, 0] = 3.0
    t = oracle.truncate_deconv(g, N, ones)
    assert t[N[2] // 2, N[1] // 2, N[0] // 2] == 3.0 and np.count_nonzero(t) == 1


# ---------------------------------------------------------------- spread / interp
def test_spread_point_on_node_and_mass_relation():
    # L = nf so that s = x exactly; point on node 3 of each axis, w = 3 (odd):
    # a = ceil(3 - 1.5) = 2, weights phi(-2/3), phi(0) = 1, phi(2/3).
    w, beta = 3, 6.9
    nf = (8, 8, 8)
    c = np.array([0.25 - 0.5j])
    g = oracle.spread([3.0], [3.0], [3.0], c, nf, w, beta, 8.0)
    assert g[3, 3, 3] == c[0]
    assert np.count_nonzero(g) == 27
    side = oracle.phi(2.0 / 3.0, beta)
    assert g[3, 3, 2] == pytest.approx(c[0] * side, rel=1e-15)
    assert g[2, 4, 3] == pytest.approx(c[0] * side * side, rel=1e-15)
    # mass relation: sum(grid) = sum_j c_j prod_d sum_i phi_d
    x, y, z = _pts(50)
    cc = _c(50)
    w, beta, _ = oracle.select_params(1e-5)
    g = oracle.spread(x, y, z, cc, (16, 16, 16), w, beta, TWO_PI)
    tot = 0
    for j in range(50):
        prod = 1.0
        for v in (x[j], y[j], z[j]):
            s = v * (16 / TWO_PI)
            a = math.ceil(s - w / 2)
            prod *= sum(oracle.phi(2 * (a + i - s) / w, beta) for i in range(w))
        tot += cc[j] * prod
    assert abs(g.sum() - tot) < 1e-12 * abs(tot)


def test_spread_wraps_periodically_and_is_linear():
    w, beta, _ = oracle.select_params(1e-6)
    nf = (16, 16, 16)
    # a point near 0 touches cells at the top end (periodic ghost handling)
    g = oracle.spread([0.01], [0.01], [0.01], [1.0], nf, w, beta, TWO_PI)
    assert abs(g[15, 15, 15]) > 0 and abs(g[0, 0, 0]) > 0
    x, y, z = _pts(100)
    c = _c(100)
    g1 = oracle.spread(x, y, z, c, nf, w, beta, TWO_PI)
    g2 = oracle.spread(np.r_[x, x], np.r_[y, y], np.r_[z, z], np.r_[c, c] * 0.5, nf, w, beta, TWO_PI)
    assert np.max(np.abs(g1 - g2)) < 1e-14 * np.max(np.abs(g1))
    # folding: x + L and x - L land on the same cells (L = 8 keeps arithmetic exact)
    xs = np.array([0.5, 3.25, 7.75])
    a = oracle.spread(xs, xs, xs, [1, 2, 3], (8, 8, 8), 3, 6.9, 8.0)
    b = oracle.spread(xs + 8.0, xs - 8.0, xs + 16.0, [1, 2, 3], (8, 8, 8), 3, 6.9, 8.0)
    assert np.array_equal(a, b)


def test_spread_interp_adjoint():
    # <C c, g> = <c, C^T g> (C real): a transposed or mis-indexed interp fails this
    rng = np.random.default_rng(3)
    x, y, z = _pts(300)
    c = _c(300)
    nf = (12, 16, 20)
    w, beta, _ = oracle.select_params(1e-7)
    g = rng.standard_normal((nf[2], nf[1], nf[0])) + 1j * rng.standard_normal((nf[2], nf[1], nf[0]))
    lhs = np.vdot(g, oracle.spread(x, y, z, c, nf, w, beta, TWO_PI))
    rhs = np.vdot(oracle.interp(x, y, z, g, w, beta, TWO_PI), c)
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


# ---------------------------------------------------------------- NUDFT
def test_nudft_grid_aligned_points_equal_numpy_fft():
    # x_j = L m_j / N on the N-point grid: Eq. (1) becomes a DFT -> numpy.fft
    N = (8, 6, 4)
    rng = np.random.default_rng(4)
    Np = 200
    m = [rng.integers(0, n, Np) for n in N]
    L = TWO_PI
    x, y, z = (m[d] * (L / N[d]) for d in range(3))
    c = _c(Np)
    A = np.zeros((N[2], N[1], N[0]), dtype=np.complex128)
    np.add.at(A, (m[2], m[1], m[0]), c)
    ref1 = np.fft.fftshift(np.fft.fftn(A))          # e^{-2 pi i n m / N}, centered
    got1 = oracle.nudft1(x, y, z, c, N, iflag=-1, L=L)
    assert np.max(np.abs(got1 - ref1)) <= 1e-12 * np.max(np.abs(ref1))
    got1p = oracle.nudft1(x, y, z, c, N, iflag=+1, L=L)
    ref1p = np.fft.fftshift(np.fft.ifftn(A)) * A.size
    assert np.max(np.abs(got1p - ref1p)) <= 1e-12 * np.max(np.abs(ref1p))
    # type 2 with iflag=-1 uses exponent +i: c_j = sum_n f_n e^{+2 pi i n m_j/N}
    f = rng.standard_normal(A.shape) + 1j * rng.standard_normal(A.shape)
    G = np.fft.ifftn(np.fft.ifftshift(f)) * A.size
    ref2 = G[m[2], m[1], m[0]]
    got2 = oracle.nudft2(x, y, z, f, iflag=-1, L=L)
    assert np.max(np.abs(got2 - ref2)) <= 1e-12 * np.max(np.abs(ref2))


def test_nudft_one_particle_and_sampling():
    N = (6, 8, 10)
    f = oracle.nudft1([0.0], [0.0], [0.0], [1.0], N)
    assert np.allclose(f, 1.0, atol=0, rtol=1e-15)
    x, y, z = _pts(40)
    c = _c(40)
    full = oracle.nudft1(x, y, z, c, N, L=TWO_PI)
    sel = np.array([0, 5, 77, 479, 123])
    assert np.array_equal(oracle.nudft1(x, y, z, c, N, sel=sel), full.ravel()[sel])
    assert np.allclose(np.abs(oracle.nudft1([1.7], [0.3], [5.0], [1.0], N)), 1.0, rtol=1e-14)
    fk = synthetic.modes(*N).numpy()
    full2 = oracle.nudft2(x, y, z, fk)
    assert np.array_equal(oracle.nudft2(x, y, z, fk, sel=[3, 0, 39]), full2[[3, 0, 39]])


def test_nudft_sampled_modes_span_point_chunks():
    # sampled modes on a tensor product of per-axis indices (the full-size parity
    # tests' layout), with more points than one phase-table chunk: identical to
    # the full evaluation at those modes
    N = (8, 6, 10)
    x, y, z = _pts(5000, seed=11)
    c = _c(5000, seed=12)
    full = oracle.nudft1(x, y, z, c, N)
    ax = [np.array([0, 3, 7]), np.array([1, 5]), np.array([0, 4, 9])]
    sel = ((ax[2][:, None, None] * N[1] + ax[1][None, :, None]) * N[0]
           + ax[0][None, None, :]).ravel()
    assert np.array_equal(oracle.nudft1(x, y, z, c, N, sel=sel), full.ravel()[sel])


def test_nudft2_separable_equals_fft_and_triple_sum():
    # rank-one modes fk[n3, n2, n1] = a1[n1] a2[n2] a3[n3]: on grid-aligned points
    # Eq. (2) is an inverse DFT (numpy.fft); at random points it equals the
    # general triple sum orc_nudft2
    N = (8, 6, 4)
    rng = np.random.default_rng(8)
    a = [rng.standard_normal(n) + 1j * rng.standard_normal(n) for n in N]
    fk = np.einsum("k,j,i->kji", a[2], a[1], a[0])
    m = [rng.integers(0, n, 300) for n in N]
    x, y, z = (m[d] * (TWO_PI / N[d]) for d in range(3))
    G = np.fft.ifftn(np.fft.ifftshift(fk)) * fk.size
    ref = G[m[2], m[1], m[0]]
    got = oracle.nudft2_separable(x, y, z, *a, iflag=-1)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    xr, yr, zr = _pts(500, seed=13)
    for iflag in (-1, 1):
        tri = oracle.nudft2(xr, yr, zr, fk, iflag=iflag)
        sep = oracle.nudft2_separable(xr, yr, zr, *a, iflag=iflag)
        assert oracle.rel_l2(sep, tri) <= 1e-13
    sel = np.array([499, 0, 17])
    assert np.array_equal(oracle.nudft2_separable(xr, yr, zr, *a, sel=sel),
                          oracle.nudft2_separable(xr, yr, zr, *a)[sel])


def test_max_abs_error_helper():
    b = np.array([1.0, -4.0, 2.0j])
    assert oracle.max_abs(b, b) == 0.0
    assert oracle.max_abs(b + np.array([0, 0.5, 0]), b) == 0.5 / 4.0


# ---------------------------------------------------------------- NUFFT vs NUDFT
@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-4, 1e-6, 1e-8, 1e-10])
def test_type1_type2_within_10eps_of_nudft(eps):
    N = (16, 16, 16)
    Np = 2000
    x, y, z = _pts(Np)
    c = _c(Np)
    ex1 = oracle.nudft1(x, y, z, c, N)
    got1 = oracle.type1(x, y, z, c, N, eps)
    e1 = oracle.rel_l2(got1, ex1)
    fk = synthetic.modes(*N).numpy()
    ex2 = oracle.nudft2(x, y, z, fk)
    got2 = oracle.type2(x, y, z, fk, eps)
    e2 = oracle.rel_l2(got2, ex2)
    assert e1 <= 10 * eps, e1
    assert e2 <= 10 * eps, e2
    # and it is a real approximation, not accidentally exact everywhere
    assert e1 > 1e-15


def test_type1_type2_nonuniform_shapes_signs_and_L():
    N = (8, 12, 16)
    L = 4 * math.pi      # Landau box
    Np = 1500
    x, y, z = (v.numpy() for v in synthetic.landau_points(Np))
    c = _c(Np)
    for iflag in (-1, +1):
        ex = oracle.nudft1(x, y, z, c, N, iflag=iflag, L=L)
        assert oracle.rel_l2(oracle.type1(x, y, z, c, N, 1e-7, iflag=iflag, L=L), ex) <= 1e-6
        fk = synthetic.modes(*N).numpy()
        ex2 = oracle.nudft2(x, y, z, fk, iflag=iflag, L=L)
        assert oracle.rel_l2(oracle.type2(x, y, z, fk, 1e-7, iflag=iflag, L=L), ex2) <= 1e-6


def test_error_decreases_with_eps():
    N = (12, 12, 12)
    x, y, z = _pts(800)
    c = _c(800)
    ex = oracle.nudft1(x, y, z, c, N)
    errs = [oracle.rel_l2(oracle.type1(x, y, z, c, N, e), ex) for e in (1e-2, 1e-4, 1e-6, 1e-8)]
    assert all(b < a for a, b in zip(errs, errs[1:]))


def test_single_particle_and_single_mode():
    # SPEC.md:441, 450-451; Eq. (1)/(2) with one term
    N = (16, 16, 16)
    eps = 1e-6
    f = oracle.type1([0.0], [0.0], [0.0], [1.0], N, eps)
    assert np.max(np.abs(f - 1.0)) <= 10 * eps
    x, y, z = _pts(300)
    fk = np.zeros((16, 16, 16), dtype=np.complex128)
    n = (3, -5, 7)
    fk[n[2] + 8, n[1] + 8, n[0] + 8] = 1.0
    got = oracle.type2(x, y, z, fk, eps)
    ref = np.exp(1j * (n[0] * x + n[1] * y + n[2] * z))
    assert np.max(np.abs(got - ref)) <= 10 * eps


def test_type1_type2_adjointness():
    # T2 = T1^H exactly in exact arithmetic: <T1 c, f> = <c, T2 f>
    N = (16, 12, 8)
    rng = np.random.default_rng(5)
    for seed in range(5):
        x, y, z = _pts(700, seed=10 + seed)
        c = rng.standard_normal(700) + 1j * rng.standard_normal(700)
        f = rng.standard_normal((8, 12, 16)) + 1j * rng.standard_normal((8, 12, 16))
        t1 = oracle.type1(x, y, z, c, N, 1e-6)
        t2 = oracle.type2(x, y, z, f, 1e-6)
        lhs = np.vdot(f, t1)
        rhs = np.vdot(t2, c)
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(t1) * np.linalg.norm(f)
