"""Full-size GPU parity at the paper's precision (fp64): configs[2] (C3) and configs[3] (C4).

SURVEY.md §8(d) plan, BASELINE.json configs:
* C3 -- fp64, 256^3 modes, 8 points per mode = 134,217,728 uniform points, eps sweep
  1e-3 .. 1e-10 (w = 4 .. 11).  The full GPU type 1 and type 2 against the oracle's
  O-NUFFT (Eq. 3 / 4) at eps in {1e-3, 1e-6, 1e-10}: rel-l2 <= 1e-10; against the
  exact NUDFT (Eq. 1 / 2) on sampled modes / points at all eight eps: <= 10 eps.
* C4 -- the PIF workload: fp64, 512^3 modes, 2^30 = 1,073,741,824 Landau-perturbed
  points on [0, 4 pi)^3, eps = 1e-4.  Type 1 on sampled modes
  against the NUDFT; type 2 of a rank-one mode array against the exact separable
  NUDFT (oracle.nudft2_separable) on 10^5 sampled points: <= 10 eps.

These are the conditions the small tests never reach: fine grids of 2.1 / 17.2 GB
(> 2^31 bytes), ~8 points per fine-cell bin neighbourhood times many batches per CTA,
262k / 2.1M bins, 64-bit offsets everywhere.

The GPU gets the points in generation (random) order.  The oracle gets the same
points permuted into bin order (a test-side reordering of its input, so its cache
behaviour lets it finish in minutes on the host): type 1 is a sum over points, so its
value is the same up to rounding order; type-2 outputs are mapped back through the
permutation.  Every comparison reports rel-l2 and max-abs (tests/errs.py); set
NUFFT_PARITY_LOG to a path to get them as JSON lines.
"""
import json
import math
import os
import time

import numpy as np
import pytest
import torch

import oracle
import synthetic
from errs import both

pytestmark = pytest.mark.gpu

TWO_PI = 2 * math.pi


def log(rec):
    print(json.dumps(rec))
    path = os.environ.get("NUFFT_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.fixture(scope="module")
def nb():
    import paper_2605_10678_b200 as nb
    from paper_2605_10678_b200 import build
    build.build()
    return nb


def bin_order(pts, nf, L, T=8):
    """Permutation sorting points by their T^3 fine-cell bin (z, y, x) -- test-side only."""
    key = None
    nb = nf // T
    for v in (pts[2], pts[1], pts[0]):
        b = torch.clamp(torch.floor(v * (nf / L)).to(torch.int64), 0, nf - 1) // T
        key = b if key is None else key * nb + b
    return torch.argsort(key).numpy()


def tensor_modes(N, per_axis, seed):
    """Flat indices of a tensor product of per-axis mode indices (always containing the
    band edges -N/2, N/2 - 1 and the zero mode), for the sampled NUDFT."""
    rng = np.random.default_rng(seed)
    axes = []
    for n in N:
        fixed = [0, n // 2, n - 1]
        rest = rng.choice(np.setdiff1d(np.arange(n), fixed), per_axis - 3, replace=False)
        axes.append(np.sort(np.concatenate([fixed, rest])))
    a1, a2, a3 = axes
    return ((a3[:, None, None] * N[1] + a2[None, :, None]) * N[0] + a1[None, None, :]).ravel()


# ------------------------------------------------------------------------------- C3
C3_N = (256, 256, 256)
C3_NP = 8 * 256 ** 3
C3_EPS = [1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-9, 1e-10]
C3_ORACLE_EPS = (1e-3, 1e-6, 1e-10)


@pytest.fixture(scope="module")
def c3():
    t0 = time.time()
    pts_d = synthetic.uniform_points(C3_NP, device="cuda")           # bit-identical to CPU
    c_d = synthetic.strengths(C3_NP, device="cuda")
    fk_d = synthetic.modes(*C3_N, device="cuda")
    x, y, z = (p.cpu().numpy() for p in pts_d)
    c, fk = c_d.cpu().numpy(), fk_d.cpu().numpy()
    order = bin_order(tuple(torch.from_numpy(v) for v in (x, y, z)), 2 * C3_N[0], TWO_PI)
    xo, yo, zo, co = x[order], y[order], z[order], c[order]
    # exact sums, shared by every eps: 216 tensor-product modes, 1000 points
    sm = tensor_modes(C3_N, 6, seed=31)
    sp = np.sort(np.random.default_rng(32).choice(C3_NP, 1000, replace=False))
    t1 = time.time()
    nudft1 = oracle.nudft1(xo, yo, zo, co, C3_N, sel=sm)
    nudft2 = oracle.nudft2(x, y, z, fk, sel=sp)
    log({"config": "C3", "what": "setup", "gen_s": t1 - t0, "nudft_s": time.time() - t1,
         "oracle_threads": oracle.num_threads()})
    return dict(pts_d=pts_d, c_d=c_d, fk_d=fk_d, x=x, y=y, z=z, c=c, fk=fk, order=order,
                xo=xo, yo=yo, zo=zo, co=co, sm=sm, sp=sp, nudft1=nudft1, nudft2=nudft2)


@pytest.mark.parametrize("eps", C3_EPS)
def test_c3_fp64_full_size(nb, c3, eps):
    plan = nb.Plan(C3_N, eps, precision="f64")
    plan.setpts(*c3["pts_d"])
    g1 = plan.type1(c3["c_d"]).cpu().numpy()
    g2 = plan.type2(c3["fk_d"]).cpu().numpy()
    info = plan.info()
    plan.close()
    w = info["w"]
    rec = {"config": "C3", "eps": eps, "w": w}
    e1 = both(g1.ravel()[c3["sm"]], c3["nudft1"])
    e2 = both(g2[c3["sp"]], c3["nudft2"])
    rec.update(nudft_t1_rel_l2=e1[0], nudft_t1_max_abs=e1[1], nudft_t2_rel_l2=e2[0],
               nudft_t2_max_abs=e2[1])
    if eps in C3_ORACLE_EPS:
        t0 = time.time()
        o1 = oracle.type1(c3["xo"], c3["yo"], c3["zo"], c3["co"], C3_N, eps)
        o2p = oracle.type2(c3["xo"], c3["yo"], c3["zo"], c3["fk"], eps)
        o2 = np.empty_like(o2p)
        o2[c3["order"]] = o2p
        f1, f2 = both(g1, o1), both(g2, o2)
        rec.update(oracle_t1_rel_l2=f1[0], oracle_t1_max_abs=f1[1], oracle_t2_rel_l2=f2[0],
                   oracle_t2_max_abs=f2[1], oracle_s=time.time() - t0)
    log(rec)
    assert e1[0] <= 10 * eps and e2[0] <= 10 * eps
    assert e1[1] <= 100 * eps and e2[1] <= 100 * eps
    if eps in C3_ORACLE_EPS:
        assert f1[0] <= 1e-10 and f2[0] <= 1e-10
        assert f1[1] <= 1e-9 and f2[1] <= 1e-9


# ------------------------------------------------------------------------------- C4
C4_N = (512, 512, 512)
C4_NP = 1 << 30
C4_EPS = 1e-4


def test_c4_fp64_landau_full_size(nb):
    torch.cuda.empty_cache()
    t0 = time.time()
    L = 4 * math.pi
    pts_d = synthetic.landau_points(C4_NP, device="cuda")
    torch.cuda.empty_cache()
    c_d = synthetic.strengths(C4_NP, device="cuda")
    plan = nb.Plan(C4_N, C4_EPS, precision="f64", L=L)
    plan.setpts(*pts_d)
    g1 = plan.type1(c_d).cpu().numpy()
    # type 2 of a rank-one mode array: its exact NUDFT factors into 1D sums
    a = [synthetic.complex_uniform(n, 40 + d, device="cuda") for d, n in enumerate(C4_N)]
    fk_d = torch.einsum("k,j,i->kji", a[2], a[1], a[0]).contiguous()
    sp = np.sort(np.random.default_rng(41).choice(C4_NP, 100_000, replace=False))
    sp_d = torch.from_numpy(sp).to("cuda")
    g2 = plan.type2(fk_d)[sp_d].cpu().numpy()
    info = plan.info()
    plan.close()
    del fk_d
    t1 = time.time()
    x, y, z = (p.cpu().numpy() for p in pts_d)
    del pts_d
    c = c_d.cpu().numpy()
    del c_d
    torch.cuda.empty_cache()
    sm = tensor_modes(C4_N, 4, seed=42)
    o1 = oracle.nudft1(x, y, z, c, C4_N, L=L, sel=sm)
    o2 = oracle.nudft2_separable(x, y, z, *(t.cpu().numpy() for t in a), L=L, sel=sp)
    e1, e2 = both(g1.ravel()[sm], o1), both(g2, o2)
    log({"config": "C4", "eps": C4_EPS, "w": info["w"], "Np": C4_NP, "points": "landau",
         "nudft_t1_rel_l2": e1[0], "nudft_t1_max_abs": e1[1], "nudft_t1_modes": len(sm),
         "nudft_t2_rel_l2": e2[0], "nudft_t2_max_abs": e2[1], "nudft_t2_points": len(sp),
         "gpu_s": t1 - t0, "oracle_s": time.time() - t1})
    assert e1[0] <= 10 * C4_EPS and e2[0] <= 10 * C4_EPS
    assert e1[1] <= 100 * C4_EPS and e2[1] <= 100 * C4_EPS
