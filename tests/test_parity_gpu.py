"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): relative l2 vs the oracle's O-NUFFT <= 1e-10
(fp64) / <= 1e-4 (fp32); vs the exact NUDFT <= 10 eps; adjointness <= 1e-12
(fp64).  Inputs are the seeded synthetic generators (synthetic/), generated on
the host and copied, so both sides see identical bits.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from errs import err
import synthetic

pytestmark = pytest.mark.gpu

TWO_PI = 2 * math.pi
TOL = {"f64": 1e-10, "f32": 1e-4}


@pytest.fixture(scope="module")
def nb():
    import paper_2605_10678_b200 as nb
    from paper_2605_10678_b200 import build
    build.build()
    return nb


def dev(t):
    return t.to("cuda")


def host_inputs(Np, prec, kind="uniform", L=TWO_PI, seed=1):
    if kind == "uniform":
        pts = synthetic.uniform_points(Np, L=L, seed=seed)
    elif kind == "landau":
        pts = synthetic.landau_points(Np, seed=seed)
    else:
        pts = synthetic.clustered_points(Np, L=L, seed=seed)
    rdt = torch.float64 if prec == "f64" else torch.float32
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    pts = tuple(p.to(rdt) for p in pts)
    c = synthetic.strengths(Np).to(cdt)
    return pts, c


def np64(t):
    return t.detach().cpu().numpy().astype(np.complex128 if t.is_complex() else np.float64)


def run_pair(nb, N, eps, prec, pts, c, fk, L=TWO_PI, iflag=-1, **kw):
    plan = nb.Plan(N, eps, precision=prec, iflag=iflag, L=L, **kw)
    plan.setpts(*(dev(p) for p in pts))
    f1 = plan.type1(dev(c))
    c2 = plan.type2(dev(fk))
    torch.cuda.synchronize()
    return plan, np64(f1), np64(c2)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_config1_parity_vs_oracle_and_nudft(nb, prec):
    # configs[0]: 32^3 modes, 1e5 uniform points, eps = 1e-6
    N, Np, eps = (32, 32, 32), 100_000, 1e-6
    pts, c = host_inputs(Np, prec)
    fk = synthetic.modes(*N).to(c.dtype)
    plan, g1, g2 = run_pair(nb, N, eps, prec, pts, c, fk)
    x, y, z = (np64(p) for p in pts)
    o1 = oracle.type1(x, y, z, np64(c), N, eps)
    o2 = oracle.type2(x, y, z, np64(fk), eps)
    assert err(g1, o1) <= TOL[prec]
    assert err(g2, o2) <= TOL[prec]
    # accuracy vs the exact sums (sampled: 2000 modes / 2000 points)
    rng = np.random.default_rng(0)
    sm = rng.choice(np.prod(N), 2000, replace=False)
    sp = rng.choice(Np, 2000, replace=False)
    e1 = err(g1.ravel()[sm], oracle.nudft1(x, y, z, np64(c), N, sel=sm))
    e2 = err(g2[sp], oracle.nudft2(x, y, z, np64(fk), sel=sp))
    assert e1 <= 10 * eps and e2 <= 10 * eps


@pytest.mark.parametrize("w", list(range(2, 17)))
def test_every_width_fp64(nb, w):
    eps = 10.0 ** (-(w - 1))
    N, Np = (16, 16, 16), 3000
    pts, c = host_inputs(Np, "f64", seed=w)
    fk = synthetic.modes(*N)
    plan, g1, g2 = run_pair(nb, N, eps, "f64", pts, c, fk)
    assert plan.info()["w"] == w
    x, y, z = (np64(p) for p in pts)
    assert err(g1, oracle.type1(x, y, z, np64(c), N, eps)) <= 1e-10
    assert err(g2, oracle.type2(x, y, z, np64(fk), eps)) <= 1e-10


@pytest.mark.parametrize("w", [2, 3, 5, 7, 8])
def test_widths_fp32(nb, w):
    eps = max(10.0 ** (-(w - 1)), 1e-7)
    N, Np = (16, 16, 16), 3000
    pts, c = host_inputs(Np, "f32", seed=w)
    fk = synthetic.modes(*N).to(torch.complex64)
    plan, g1, g2 = run_pair(nb, N, eps, "f32", pts, c, fk)
    x, y, z = (np64(p) for p in pts)
    assert err(g1, oracle.type1(x, y, z, np64(c), N, eps)) <= 1e-4
    assert err(g2, oracle.type2(x, y, z, np64(fk), eps)) <= 1e-4


def test_stage_spread_and_interp_match_oracle(nb):
    N, Np, eps = (16, 24, 32), 20000, 1e-7
    pts, c = host_inputs(Np, "f64", seed=3)
    plan = nb.Plan(N, eps, precision="f64")
    plan.setpts(*(dev(p) for p in pts))
    info = plan.info()
    w, beta = info["w"], info["beta"]
    ow, obeta, _ = oracle.select_params(eps)
    assert (w, beta) == (ow, obeta)
    x, y, z = (np64(p) for p in pts)
    nf = (32, 48, 64)
    g = np64(plan.spread(dev(c)))
    og = oracle.spread(x, y, z, np64(c), nf, w, beta, TWO_PI)
    assert err(g, og) <= 1e-12
    rng = np.random.default_rng(1)
    grid = rng.standard_normal(og.shape) + 1j * rng.standard_normal(og.shape)
    gi = np64(plan.interp(dev(torch.from_numpy(grid))))
    assert err(gi, oracle.interp(x, y, z, grid, w, beta, TWO_PI)) <= 1e-12


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_interp_tensor_map_follows_the_grid_address(nb, prec):
    # interior bins stage their subgrid through a TMA tensor map of the grid the
    # interp reads; alternating the plan's own grid (type 2) with two caller grids
    # (nufft_interp) must re-encode it every time the address changes
    N, Np, eps = (24, 20, 28), 20000, 1e-6
    pts, c = host_inputs(Np, prec, seed=8)
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    plan = nb.Plan(N, eps, precision=prec)
    plan.setpts(*(dev(p) for p in pts))
    info = plan.info()
    w, beta = info["w"], info["beta"]
    x, y, z = (np64(p) for p in pts)
    fk = synthetic.modes(*N).to(cdt)
    o2 = oracle.type2(x, y, z, np64(fk), eps)
    rng = np.random.default_rng(9)
    shape = (2 * N[2], 2 * N[1], 2 * N[0])
    grids = [rng.standard_normal(shape) + 1j * rng.standard_normal(shape) for _ in range(2)]
    refs = [oracle.interp(x, y, z, g, w, beta, TWO_PI) for g in grids]
    dgrids = [dev(torch.from_numpy(g).to(cdt)) for g in grids]
    for _ in range(2):
        assert err(np64(plan.type2(dev(fk))), o2) <= TOL[prec]
        for dg, ref in zip(dgrids, refs):
            assert err(np64(plan.interp(dg)), ref) <= (1e-12 if prec == "f64" else 1e-5)


def test_stage_calls_never_write_past_the_callers_grid(nb):
    # nufft_spread writes exactly nf1 nf2 nf3 complex cells (device and host buffers)
    N, Np, eps = (8, 10, 12), 3000, 1e-6
    pts, c = host_inputs(Np, "f64", seed=5)
    plan = nb.Plan(N, eps, precision="f64")
    plan.setpts(*(dev(p) for p in pts))
    n = 8 * N[0] * N[1] * N[2]
    shape = (2 * N[2], 2 * N[1], 2 * N[0])
    for on_dev in (True, False):
        guard = torch.full((n + 4096,), 7.0 + 7.0j, dtype=torch.complex128)
        if on_dev:
            guard = guard.cuda()
        else:
            guard = guard.pin_memory()
        g = guard[:n].view(shape)
        plan.spread(dev(c) if on_dev else c, out=g)
        torch.cuda.synchronize()
        assert bool((guard[n:] == 7.0 + 7.0j).all())
        assert float(g.abs().max()) > 0


def test_nonuniform_shape_signs_modeord_landau(nb):
    N, Np, eps = (8, 12, 20), 6000, 1e-8
    L = 4 * math.pi
    pts, c = host_inputs(Np, "f64", kind="landau")
    fk = synthetic.modes(*N)
    x, y, z = (np64(p) for p in pts)
    for iflag in (-1, 1):
        plan, g1, g2 = run_pair(nb, N, eps, "f64", pts, c, fk, L=L, iflag=iflag)
        assert err(g1, oracle.type1(x, y, z, np64(c), N, eps, iflag=iflag, L=L)) <= 1e-10
        assert err(g2, oracle.type2(x, y, z, np64(fk), eps, iflag=iflag, L=L)) <= 1e-10
    # FFT-ordered modes are the centered ones rolled by N/2 per axis
    plan, g1f, _ = run_pair(nb, N, eps, "f64", pts, c, fk, L=L, modeord=1)
    _, g1c, _ = run_pair(nb, N, eps, "f64", pts, c, fk, L=L, modeord=0)
    assert np.allclose(np.fft.ifftshift(g1c), g1f, rtol=0, atol=1e-12 * np.abs(g1c).max())


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("kernel", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9])
def test_every_spread_kernel(nb, prec, kernel, eps):
    # 1 = register-row spread, 2 = plane outer products, 3 = tcgen05 3xTF32 GEMM
    # (fp32 only; all three T = 16 - w), 4 / 8 = shared-memory z-plane owners
    if prec == "f32" and eps < 1e-7:
        eps = 1e-7
    if kernel == 3 and prec == "f64":
        pytest.skip("tensor-core spread is fp32-only")
    w = nb.Plan((8, 8, 8), eps, precision=prec).info()["w"]
    tile = 16 - w if kernel in (1, 2, 3) else 8
    N, Np = (24, 24, 24), 20000
    pts, c = host_inputs(Np, prec, seed=11)
    fk = synthetic.modes(*N).to(c.dtype)
    plan, g1, g2 = run_pair(nb, N, eps, prec, pts, c, fk, tile=tile, spread_warps=kernel)
    x, y, z = (np64(p) for p in pts)
    assert err(g1, oracle.type1(x, y, z, np64(c), N, eps)) <= TOL[prec]
    assert err(g2, oracle.type2(x, y, z, np64(fk), eps)) <= TOL[prec]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("eps", [1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6])
def test_sub_bin_spread_every_width(nb, prec, eps):
    # spread_warps = 5: sub-bin register rows, w = 2 .. 7 (w = 7: three rows per lane,
    # 2 x 2 x 6 sub-bins), default tile (T_d + 1 = ns_d G_d)
    N, Np = (32, 24, 40), 40000
    pts, c = host_inputs(Np, prec, seed=21)
    fk = synthetic.modes(*N).to(c.dtype)
    plan, g1, g2 = run_pair(nb, N, eps, prec, pts, c, fk, spread_warps=5)
    w = plan.info()["w"]
    G = (9 - w, 9 - w, (8 if w <= 6 else 12) + 1 - w)
    assert all((t + 1) % Gd == 0 for t, Gd in zip(plan.info()["tile"], G))
    x, y, z = (np64(p) for p in pts)
    assert err(g1, oracle.type1(x, y, z, np64(c), N, eps)) <= TOL[prec]
    assert err(g2, oracle.type2(x, y, z, np64(fk), eps)) <= TOL[prec]


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_sub_bin_spread_tiles_clusters_precompute(nb, prec):
    # ragged / non-cubic tiles, one-hot bins (every point in one cell), precomputed
    # weights, Landau points on [0, 4 pi)^3 -- all against the oracle's spread
    N = (24, 20, 28)
    fk = synthetic.modes(*N)
    cases = []
    for eps in (1e-4, 1e-6):  # w = 5 (G = 4, 4, 4) and w = 7 (G = 2, 2, 6)
        w = nb.Plan((8, 8, 8), eps, precision=prec).info()["w"]
        G = (9 - w, 9 - w, (8 if w <= 6 else 12) + 1 - w)
        cases += [dict(eps=eps, tile=(G[0] - 1, 2 * G[1] - 1, G[2] - 1)),
                  dict(eps=eps, precompute=1),
                  dict(eps=eps, tile=(3 * G[0] - 1, 3 * G[1] - 1, 2 * G[2] - 1), precompute=-1)]
    for kind in ("uniform", "clustered", "one", "landau"):
        L = 4 * math.pi if kind == "landau" else TWO_PI
        if kind == "one":
            pts = tuple(torch.full((3000,), 1.2345, dtype=torch.float64) for _ in range(3))
            c = synthetic.strengths(3000)
        else:
            pts, c = host_inputs(25000, "f64", kind=kind, seed=22)
        rdt = torch.float64 if prec == "f64" else torch.float32
        pts = tuple(p.to(rdt) for p in pts)
        c = c.to(torch.complex128 if prec == "f64" else torch.complex64)
        x, y, z = (np64(p) for p in pts)
        ref = {}
        for eps in (1e-4, 1e-6):
            ref[eps] = (oracle.type1(x, y, z, np64(c), N, eps, L=L),
                        oracle.type2(x, y, z, np64(fk), eps, L=L))
        for kw in cases:
            kw = dict(kw)
            eps = kw.pop("eps")
            _, g1, g2 = run_pair(nb, N, eps, prec, pts, c, fk.to(c.dtype), L=L, spread_warps=5, **kw)
            assert err(g1, ref[eps][0]) <= TOL[prec], (kind, eps, kw)
            assert err(g2, ref[eps][1]) <= TOL[prec], (kind, eps, kw)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("kernel", [1, 2, 8])
@pytest.mark.parametrize("precompute", [-1, 1])
def test_precomputed_weights_both_paths(nb, prec, kernel, precompute):
    # opts.precompute: ES weights stored by setpts (1) or evaluated in the kernels (-1)
    eps = 1e-6
    w = nb.Plan((8, 8, 8), eps, precision=prec).info()["w"]
    tile = 16 - w if kernel in (1, 2) else 8
    N, Np = (24, 20, 28), 30000
    pts, c = host_inputs(Np, prec, seed=12)
    fk = synthetic.modes(*N).to(c.dtype)
    plan, g1, g2 = run_pair(nb, N, eps, prec, pts, c, fk, tile=tile, spread_warps=kernel,
                            precompute=precompute)
    assert plan.info()["weights_precomputed"] == (1 if precompute == 1 else 0)
    x, y, z = (np64(p) for p in pts)
    assert err(g1, oracle.type1(x, y, z, np64(c), N, eps)) <= TOL[prec]
    assert err(g2, oracle.type2(x, y, z, np64(fk), eps)) <= TOL[prec]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("variant", [(-1, 1), (-2, 2), (0, 3), (-3, 0)])
@pytest.mark.parametrize("precompute", [-1, 1])
def test_ablation_variants_atomic_spread_direct_interp(nb, prec, variant, precompute):
    # the paper's Atomic Spread / Direct Interpolation,
    # in caller order (-1 / 1) and bin-sorted order (-2 / 2), Direct Interpolation
    # along the Morton curve of the bins (3), the Tiled Spread (-3), clustered points
    # included (atomic contention), to the same oracle bars as the default kernels
    sw, im = variant
    eps = 1e-9 if prec == "f64" else 1e-5
    N, Np = (20, 24, 16), 25000
    x, y, z = synthetic.clustered_points(Np, seed=13)
    rdt = torch.float64 if prec == "f64" else torch.float32
    pts = (x.to(rdt), y.to(rdt), z.to(rdt))
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    c = synthetic.strengths(Np).to(cdt)
    fk = synthetic.modes(*N).to(cdt)
    plan, g1, g2 = run_pair(nb, N, eps, prec, pts, c, fk, spread_warps=sw, interp_method=im,
                            precompute=precompute)
    xs, ys, zs = (np64(p) for p in pts)
    assert err(g1, oracle.type1(xs, ys, zs, np64(c), N, eps)) <= TOL[prec]
    assert err(g2, oracle.type2(xs, ys, zs, np64(fk), eps)) <= TOL[prec]
    # a second setpts (other points, fewer of them) refreshes the caller-order map
    pts2, c2 = host_inputs(Np // 3, prec, seed=14)
    plan.setpts(*(p.cuda() for p in pts2))
    f = np64(plan.type2(fk.cuda()))
    xs, ys, zs = (np64(p) for p in pts2)
    assert err(f, oracle.type2(xs, ys, zs, np64(fk), eps)) <= TOL[prec]


def test_custom_and_ragged_tiles(nb):
    N, Np, eps = (32, 32, 32), 30000, 1e-5
    pts, c = host_inputs(Np, "f64", seed=7)
    fk = synthetic.modes(*N)
    x, y, z = (np64(p) for p in pts)
    o1 = oracle.type1(x, y, z, np64(c), N, eps)
    o2 = oracle.type2(x, y, z, np64(fk), eps)
    for tile in [(4, 4, 4), (7, 9, 5), (16, 8, 4), (32, 12, 3)]:
        plan, g1, g2 = run_pair(nb, N, eps, "f64", pts, c, fk, tile=tile)
        assert tuple(plan.info()["tile"]) == tile
        assert err(g1, o1) <= 1e-10, tile
        assert err(g2, o2) <= 1e-10, tile
    # a subgrid that cannot fit in one CTA's shared memory is refused at plan time
    with pytest.raises(nb.NufftError):
        nb.Plan(N, eps, tile=(64, 64, 64))


def test_edge_cases(nb):
    N, eps = (16, 16, 16), 1e-6
    fk = synthetic.modes(*N)
    # Np = 0: zero modes out, nothing to write
    plan = nb.Plan(N, eps)
    e = torch.empty(0, dtype=torch.float64, device="cuda")
    plan.setpts(e, e, e)
    f = plan.type1(torch.empty(0, dtype=torch.complex128, device="cuda"))
    assert float(f.abs().max()) == 0.0
    assert plan.type2(dev(fk)).numel() == 0
    # Np = 1 at the origin: all modes ~ 1
    z1 = torch.zeros(1, dtype=torch.float64, device="cuda")
    plan.setpts(z1, z1, z1)
    f = np64(plan.type1(torch.ones(1, dtype=torch.complex128, device="cuda")))
    assert np.max(np.abs(f - 1.0)) <= 10 * eps
    # boundary points, exact node ties (L = 32 = nf: s = x exactly), folded points
    L = 32.0
    xs = np.array([0.0, np.nextafter(L, 0), 16.0, 3.5, 4.0, -0.25, L + 1.75, 2 * L + 0.5, -L - 3.0])
    rng = np.random.default_rng(2)
    pts = [rng.permutation(xs) for _ in range(3)]
    c = rng.standard_normal(len(xs)) + 1j * rng.standard_normal(len(xs))
    for w_eps in (1e-3, 1e-6):   # even and odd widths
        plan = nb.Plan(N, w_eps, L=L)
        plan.setpts(*(dev(torch.from_numpy(p)) for p in pts))
        g1 = np64(plan.type1(dev(torch.from_numpy(c))))
        g2 = np64(plan.type2(dev(fk)))
        assert err(g1, oracle.type1(*pts, c, N, w_eps, L=L)) <= 1e-10
        assert err(g2, oracle.type2(*pts, np64(fk), w_eps, L=L)) <= 1e-10


@pytest.mark.parametrize("kernel", [0, 1, 2, 8])
def test_clustered_points_one_hot_bin(nb, kernel):
    # all points in a few tiles (load imbalance, many batches per bin) and all in
    # ONE cell; every spread kernel (w = 7: the register kernels take T = 9)
    N, Np, eps = (32, 32, 32), 50000, 1e-6
    tile = 9 if kernel in (1, 2) else None
    pts, c = host_inputs(Np, "f64", kind="clustered")
    fk = synthetic.modes(*N)
    x, y, z = (np64(p) for p in pts)
    _, g1, g2 = run_pair(nb, N, eps, "f64", pts, c, fk, tile=tile, spread_warps=kernel)
    assert err(g1, oracle.type1(x, y, z, np64(c), N, eps)) <= 1e-10
    assert err(g2, oracle.type2(x, y, z, np64(fk), eps)) <= 1e-10
    one = tuple(torch.full((5000,), 1.2345, dtype=torch.float64) for _ in range(3))
    c1 = synthetic.strengths(5000)
    _, g1, g2 = run_pair(nb, N, eps, "f64", one, c1, fk, tile=tile, spread_warps=kernel)
    o = [np64(p) for p in one]
    assert err(g1, oracle.type1(*o, np64(c1), N, eps)) <= 1e-10
    assert err(g2, oracle.type2(*o, np64(fk), eps)) <= 1e-10


def test_adjointness_fp64(nb):
    N, Np = (24, 16, 20), 40000
    for seed in range(3):
        pts, c = host_inputs(Np, "f64", seed=20 + seed)
        fk = synthetic.modes(*N, seed=30 + seed)
        _, t1, t2 = run_pair(nb, N, 1e-9, "f64", pts, c, fk)
        lhs = np.vdot(np64(fk).ravel(), t1.ravel())
        rhs = np.vdot(t2, np64(c))
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(t1) * np.linalg.norm(np64(fk))


def test_host_buffers_through_the_abi(nb):
    # the C ABI accepts host arrays (staged internally): same result as device arrays
    N, Np, eps = (16, 16, 16), 10000, 1e-6
    pts, c = host_inputs(Np, "f64", seed=9)
    fk = synthetic.modes(*N)
    plan = nb.Plan(N, eps)
    plan.setpts(*(p.pin_memory() for p in pts))
    h1 = plan.type1(c.pin_memory())
    h2 = plan.type2(fk.pin_memory())
    assert not h1.is_cuda and not h2.is_cuda
    _, g1, g2 = run_pair(nb, N, eps, "f64", pts, c, fk)
    assert err(np64(h1), g1) <= 1e-13
    assert err(np64(h2), g2) <= 1e-13


def test_config2_fp32_full_parity(nb):
    # configs[1] (bench workload): fp32, 128^3 modes, 2^21 points, eps = 1e-4 and 1e-6
    N, Np = (128, 128, 128), 1 << 21
    pts, c = host_inputs(Np, "f32", seed=1)
    fk = synthetic.modes(*N).to(torch.complex64)
    x, y, z = (np64(p) for p in pts)
    for eps in (1e-4, 1e-6):
        _, g1, g2 = run_pair(nb, N, eps, "f32", pts, c, fk)
        assert err(g1, oracle.type1(x, y, z, np64(c), N, eps)) <= 1e-4
        assert err(g2, oracle.type2(x, y, z, np64(fk), eps)) <= 1e-4
        rng = np.random.default_rng(3)
        sm = rng.choice(np.prod(N), 300, replace=False)
        e1 = err(g1.ravel()[sm], oracle.nudft1(x, y, z, np64(c), N, sel=sm))
        assert e1 <= 10 * eps


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("modeord,iflag", [(0, -1), (1, 1)])
def test_pruned_sigma2_fft_option(nb, prec, modeord, iflag):
    # opts.fft_method = 1: the paper's pruned FFT (Eq. 7) -- eight
    # N^3 parity-sub-grid transforms + twiddle combine / split -- equals the full
    # (2N)^3 transform + truncation on the same points, and the oracle
    eps = 1e-9 if prec == "f64" else 1e-5
    N, Np = (24, 32, 20), 30000
    pts, c = host_inputs(Np, prec, seed=23)
    fk = synthetic.modes(*N).to(c.dtype)
    _, a1, a2 = run_pair(nb, N, eps, prec, pts, c, fk, iflag=iflag, modeord=modeord)
    _, b1, b2 = run_pair(nb, N, eps, prec, pts, c, fk, iflag=iflag, modeord=modeord, fft_method=1)
    same = 1e-13 if prec == "f64" else 1e-5
    assert err(b1, a1) <= same
    assert err(b2, a2) <= same
    if modeord == 0:
        x, y, z = (np64(p) for p in pts)
        assert err(b1, oracle.type1(x, y, z, np64(c), N, eps, iflag=iflag)) <= TOL[prec]
        assert err(b2, oracle.type2(x, y, z, np64(fk), eps, iflag=iflag)) <= TOL[prec]
