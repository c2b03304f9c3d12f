"""The z-slab plan (csrc/dist.cpp) at P = 2, 4 and 8 ranks on ONE GPU, through the
loopback transport (csrc/xport.cpp, nufft_comm_init_loopback): every rank is a host
thread with its own stream and plan, every exchange (point redistribution, halo
accumulate / fill, the all-to-all transposes, the failure agreement) runs the same
dist.cpp code as under NCCL.

Checks: the P-rank type 1 / type 2 equal the
one-GPU plan on the same points (<= 1e-12 fp64, 1e-5 fp32 relative; atomics reorder
sums) and the oracle (<= 1e-10 / 1e-4), with points handed to the wrong ranks
(redistributed by setpts) or owned, Landau points on [0, 4 pi)^3, sub-bin plans,
real transforms (half-spectrum layout) and PIF particle migration.
"""
import math
import threading

import numpy as np
import pytest
import torch

import oracle
import synthetic
from errs import err

pytestmark = pytest.mark.gpu

TWO_PI = 2 * math.pi


@pytest.fixture(scope="module")
def nb():
    import paper_2605_10678_b200 as nb
    from paper_2605_10678_b200 import build
    build.build()
    return nb


def run_ranks(nb, P, fn, timeout=300):
    """fn(rank, comm, stream) on P host threads sharing one GPU; results by rank."""
    comms = nb.Comm.loopback(P)
    out, errs = [None] * P, [None] * P

    def work(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r, comms[r], s)
                s.synchronize()
        except BaseException as e:  # reported below
            errs[r] = e

    ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    hung = [r for r, t in enumerate(ts) if t.is_alive()]
    assert not hung, f"ranks {hung} did not finish (a collective was not matched)"
    for e in errs:
        if e is not None:
            raise e
    for c in comms:
        c.close()
    return out


def owner_of(z, L, nf3, P):
    zz = z.double()  # the library's fold (reading R10), bit for bit
    s = (zz - L * torch.floor(zz / L)) * (nf3 / L)
    s = torch.where(s >= nf3, s - nf3, s)
    return torch.clamp(torch.floor(s).long(), max=nf3 - 1) // (nf3 // P)


def complex_case(nb, P, N, Np, eps, prec, owned, kind, L, **kw):
    rdt = torch.float64 if prec == "f64" else torch.float32
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    pts = [p.to(rdt) for p in (synthetic.landau_points(Np) if kind == "landau"
                               else synthetic.uniform_points(Np, L=L))]
    c = synthetic.strengths(Np).to(cdt)
    fk = synthetic.modes(*N).to(cdt)
    own = owner_of(pts[2], L, 2 * N[2], P) if owned else None

    def rank_fn(r, comm, s):
        mine = torch.nonzero(own == r).flatten() if owned else torch.arange(r, Np, P)
        plan = nb.Plan(N, eps, precision=prec, L=L, comm=comm, points_owned=owned,
                       stream=s, **kw)
        lo, hi = plan.local_modes()
        plan.setpts(*(p[mine].contiguous().cuda() for p in pts))
        f_loc = plan.type1(c[mine].contiguous().cuda()).cpu()
        c_loc = plan.type2(fk[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]].contiguous().cuda()).cpu()
        info = plan.info()
        plan.close()
        return lo, hi, f_loc, mine, c_loc, info

    res = run_ranks(nb, P, rank_fn)
    f_all = torch.cat([rr[2] for rr in sorted(res, key=lambda t: t[0][1])], dim=1)
    c_all = torch.empty(Np, dtype=cdt)
    for rr in res:
        c_all[rr[3]] = rr[4]
    assert all(rr[5]["nranks"] == P for rr in res)
    ref = nb.Plan(N, eps, precision=prec, L=L, **kw)
    ref.setpts(*(p.cuda() for p in pts))
    f_ref, c_ref = ref.type1(c.cuda()).cpu(), ref.type2(fk.cuda()).cpu()
    ref.close()
    same = 1e-12 if prec == "f64" else 1e-5
    assert err(f_all.numpy(), f_ref.numpy()) <= same
    assert err(c_all.numpy(), c_ref.numpy()) <= same
    x, y, z = (p.double().numpy() for p in pts)
    tol = 1e-10 if prec == "f64" else 1e-4
    assert err(f_all.numpy(), oracle.type1(x, y, z, c.numpy().astype(np.complex128), N, eps, L=L)) <= tol
    assert err(c_all.numpy(), oracle.type2(x, y, z, fk.numpy().astype(np.complex128), eps, L=L)) <= tol


@pytest.mark.parametrize("P", [2, 4, 8])
def test_loopback_slab_redistribution_fp64(nb, P):
    complex_case(nb, P, (32, 32, 32), 40000, 1e-6, "f64", False, "uniform", TWO_PI)


@pytest.mark.parametrize("P", [2, 8])
def test_loopback_slab_owned_landau(nb, P):
    complex_case(nb, P, (16, 24, 32), 30000, 1e-9, "f64", True, "landau", 4 * math.pi)


@pytest.mark.parametrize("P", [4, 8])
def test_loopback_slab_fp32_and_sub_bins(nb, P):
    complex_case(nb, P, (32, 32, 32), 40000, 1e-4, "f32", False, "uniform", TWO_PI)
    complex_case(nb, P, (32, 32, 64), 60000, 1e-4, "f64", False, "uniform", TWO_PI,
                 spread_warps=5)


@pytest.mark.parametrize("P", [2, 8])
def test_loopback_slab_real_half_spectrum(nb, P):
    # real transforms on the slab plan: the half spectrum (x index k1 in [0, N1/2]) of
    # type 1 against the one-GPU real transform, and type 2 of a Hermitian field
    N, Np, eps, L = (32, 32, 32), 40000, 1e-9, TWO_PI
    pts = [p for p in synthetic.uniform_points(Np, L=L, seed=31)]
    c = synthetic.strengths(Np, seed=32).real.contiguous()

    def rank_fn(r, comm, s):
        mine = torch.arange(r, Np, P)
        plan = nb.Plan(N, eps, precision="f64", L=L, comm=comm, stream=s)
        lo, hi = plan.local_modes()
        plan.setpts(*(p[mine].contiguous().cuda() for p in pts))
        fh = plan.type1_real(c[mine].contiguous().cuda()).cpu()
        plan.close()
        return lo, fh

    res = run_ranks(nb, P, rank_fn)
    fh = torch.cat([rr[1] for rr in sorted(res, key=lambda t: t[0][1])], dim=1)
    ref = nb.Plan(N, eps, precision="f64", L=L)
    ref.setpts(*(p.cuda() for p in pts))
    ff = ref.type1_real(c.cuda()).cpu()
    ref.close()
    h1 = N[0] // 2
    assert err(fh[:, :, :h1].numpy(), ff[:, :, h1:].numpy()) <= 1e-12
    a = fh[1:, 1:, h1]
    b = torch.conj(torch.flip(ff[1:, 1:, 0], dims=(0, 1))).resolve_conj()
    assert err(a.numpy(), b.numpy()) <= 1e-12


def state_sorted(arrs):
    a = torch.stack([t.double().cpu() for t in arrs], 1)
    key = a[:, 0] * 1e6 + a[:, 1] * 1e3 + a[:, 2]
    return a[torch.argsort(key)]


@pytest.mark.parametrize("P", [2, 4, 8])
def test_loopback_pif_migration_matches_one_gpu(nb, P):
    # PIF steps on a slab plan with migration (dt large: many particles cross slab
    # boundaries every step): count conserved, every particle in its owner's slab, and
    # the particle multiset equal to a one-GPU run from the gathered initial state
    from paper_2605_10678_b200.pif import LandauPIF
    N, Np, steps = (16, 16, 32), 30000, 3  # nf3 / P >= ceil(w / 2) at P = 8

    def rank_fn(r, comm, s):
        sim = LandauPIF(N, Np, eps=1e-9, dt=0.4, comm=comm, device=torch.device("cuda", 0),
                        seed=5)
        init = [a.clone() for a in (sim.x, sim.y, sim.z, sim.vx, sim.vy, sim.vz)]
        ok = True
        for _ in range(steps):
            sim.step()
            own = owner_of(sim.z, sim.L, 2 * N[2], P).cuda()
            ok &= bool((own == r).all())
        fin = [a.clone() for a in (sim.x, sim.y, sim.z, sim.vx, sim.vy, sim.vz)]
        sim.plan.close()
        return init, fin, ok

    res = run_ranks(nb, P, rank_fn)
    assert all(rr[2] for rr in res), "a particle outside its owner's slab"
    init = [torch.cat([rr[0][k] for rr in res]) for k in range(6)]
    fin = [torch.cat([rr[1][k] for rr in res]) for k in range(6)]
    assert init[0].numel() == Np and fin[0].numel() == Np
    ref = LandauPIF(N, Np, eps=1e-9, dt=0.4, device=torch.device("cuda", 0), seed=5)
    for dst, src in zip(ref._state, init):
        dst.copy_(src)
    for _ in range(steps):
        ref.step()
    a, b = state_sorted(fin), state_sorted(ref._state)
    assert float((a - b).abs().max() / b.abs().max()) <= 1e-9
    ref.plan.close()
