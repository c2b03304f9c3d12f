"""Real-valued transforms on the CUDA path.

nufft_execute_type1_real(c real) must equal the oracle's type 1 of c + 0i, and
nufft_execute_type2_real(fk) the real part of the oracle's type 2 of fk, to the
north_star bars (rel-l2 <= 1e-10 fp64, <= 1e-4 fp32); the type-1 output of real
strengths is Hermitian (fk[-n] = conj fk[n]) wherever both n and -n are stored.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from errs import err
import synthetic

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-4}


@pytest.fixture(scope="module")
def nb():
    import paper_2605_10678_b200 as nb
    from paper_2605_10678_b200 import build
    build.build()
    return nb


def np64(t):
    return t.detach().cpu().numpy().astype(np.complex128 if t.is_complex() else np.float64)


def inputs(Np, prec, seed=1, L=2 * math.pi, kind="uniform"):
    pts = (synthetic.uniform_points(Np, L=L, seed=seed) if kind == "uniform"
           else synthetic.landau_points(Np, seed=seed))
    rdt = torch.float64 if prec == "f64" else torch.float32
    pts = tuple(p.to(rdt) for p in pts)
    c = synthetic.strengths(Np).real.contiguous().to(rdt)
    return pts, c


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("kernel", [2, 5, 8])
@pytest.mark.parametrize("iflag", [-1, 1])
def test_real_type1_type2_vs_oracle(nb, prec, kernel, iflag):
    eps = 1e-5 if kernel == 5 else 1e-6  # sub-bin rows: w <= 6
    w = nb.Plan((8, 8, 8), eps, precision=prec).info()["w"]
    tile = 16 - w if kernel == 2 else (None if kernel == 5 else 8)
    N, Np = (24, 20, 28), 30000
    pts, c = inputs(Np, prec, seed=21)
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    fk = synthetic.modes(*N).to(cdt)
    plan = nb.Plan(N, eps, precision=prec, iflag=iflag, tile=tile, spread_warps=kernel)
    plan.setpts(*(p.cuda() for p in pts))
    f1 = np64(plan.type1_real(c.cuda()))
    c2 = np64(plan.type2_real(fk.cuda()))
    torch.cuda.synchronize()
    x, y, z = (np64(p) for p in pts)
    ref1 = oracle.type1(x, y, z, np64(c).astype(np.complex128), N, eps, iflag=iflag)
    ref2 = oracle.type2(x, y, z, np64(fk), eps, iflag=iflag).real
    assert err(f1, ref1) <= TOL[prec]
    assert np.linalg.norm(c2 - ref2) / np.linalg.norm(ref2) <= TOL[prec]


@pytest.mark.parametrize("precompute", [-1, 1])
@pytest.mark.parametrize("modeord", [0, 1])
def test_real_matches_complex_path_and_is_hermitian(nb, precompute, modeord):
    eps, N, Np = 1e-9, (16, 24, 20), 25000
    L = 4 * math.pi
    pts, c = inputs(Np, "f64", seed=22, L=L, kind="landau")
    fk = synthetic.modes(*N)
    plan = nb.Plan(N, eps, precision="f64", L=L, modeord=modeord, precompute=precompute)
    plan.setpts(*(p.cuda() for p in pts))
    f_real = np64(plan.type1_real(c.cuda()))
    f_cplx = np64(plan.type1(c.to(torch.complex128).cuda()))
    c_real = np64(plan.type2_real(fk.cuda()))
    c_cplx = np64(plan.type2(fk.cuda()))
    assert err(f_real, f_cplx) <= 1e-12
    assert np.linalg.norm(c_real - c_cplx.real) / np.linalg.norm(c_cplx.real) <= 1e-12
    # Hermitian symmetry: fk[-n] = conj fk[n] for n with -n also stored (centered view)
    fc = f_real if modeord == 0 else np.fft.fftshift(f_real)
    sub = fc[1:, 1:, 1:]            # indices -N/2 + 1 .. N/2 - 1 on every axis
    assert np.max(np.abs(sub - np.conj(sub[::-1, ::-1, ::-1]))) <= 1e-12 * np.abs(sub).max()


def test_real_pif_like_hermitian_field_and_edge_cases(nb):
    # a Hermitian fk (the spectrum of a real field) gives type2 == type2_real exactly
    eps, N, Np = 1e-8, (16, 16, 16), 8000
    pts, c = inputs(Np, "f64", seed=23)
    plan = nb.Plan(N, eps, precision="f64")
    plan.setpts(*(p.cuda() for p in pts))
    fh = plan.type1_real(c.cuda())             # Hermitian where -n is stored too
    # the -N/2 planes have no +N/2 partner in the stored box: zero them, leaving an
    # exactly Hermitian set of modes (the spectrum of a real field)
    fh[0, :, :] = 0
    fh[:, 0, :] = 0
    fh[:, :, 0] = 0
    a = np64(plan.type2(fh))
    b = np64(plan.type2_real(fh))
    assert np.max(np.abs(a.imag)) <= 1e-9 * np.abs(a).max()
    assert np.linalg.norm(b - a.real) / np.linalg.norm(a.real) <= 1e-12
    # zero points: zero modes / empty output
    plan0 = nb.Plan(N, eps, precision="f64")
    e = torch.empty(0, dtype=torch.float64, device="cuda")
    plan0.setpts(e, e, e)
    f0 = plan0.type1_real(e)
    assert float(f0.abs().max()) == 0.0
    assert plan0.type2_real(fh).numel() == 0


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("eps,kernel", [(1e-4, 0), (1e-7, 0), (1e-4, 5), (1e-5, 5)])
def test_three_field_gather_and_fused_kick(nb, prec, eps, kernel):
    # type2_real3 == three type2_real calls; gather_kick == type2_real + kick per component
    # (kernel 5: sub-bin sorted plan -> the register-block gather for all three paths)
    if prec == "f32" and eps < 1e-6:
        eps = 1e-6
    N, Np = (16, 20, 24), 20000
    pts, _ = inputs(Np, prec, seed=24)
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    fks = [synthetic.modes(*N, seed=40 + d).to(cdt).cuda() for d in range(3)]
    plan = nb.Plan(N, eps, precision=prec, spread_warps=kernel)
    plan.setpts(*(p.cuda() for p in pts))
    sep = torch.stack([plan.type2_real(f) for f in fks], dim=1)
    vec = plan.type2_real3(*fks)
    tol = 1e-13 if prec == "f64" else 1e-5
    assert float((vec - sep).abs().max() / sep.abs().max()) <= tol
    # against the oracle too
    x, y, z = (np64(p) for p in pts)
    ref = np.stack([oracle.type2(x, y, z, np64(f), eps).real for f in fks], axis=1)
    assert np.linalg.norm(np64(vec) - ref) / np.linalg.norm(ref) <= TOL[prec]
    rdt = torch.float64 if prec == "f64" else torch.float32
    v = [torch.randn(Np, dtype=rdt, device="cuda") for _ in range(3)]
    v_ref = [a + 0.37 * sep[:, d] for d, a in enumerate(v)]
    lib = nb.lib()
    import ctypes
    rc = lib.nufft_pif_gather_kick(plan._h, *(f.data_ptr() for f in fks),
                                   *(ctypes.c_void_p(a.data_ptr()) for a in v), ctypes.c_double(0.37))
    assert rc == 0
    for a, b in zip(v, v_ref):
        assert float((a - b).abs().max() / b.abs().max()) <= tol
