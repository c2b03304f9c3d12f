"""C1-sized runs of every kernel family for compute-sanitizer:
    compute-sanitizer --tool {memcheck,racecheck,synccheck} python scripts/sanitize_c1.py
One small type 1 + type 2 per kernel path through the C ABI: the default fp64 path
(sub-bin spread with block flushes to the fine grid, register-block interp on a
TMA-staged subgrid; NUFFT_SUB_TILE=1 for the tile-flush sub-bin spread), the register outer-product and
z-plane spreads with the tiled interp (fp64, fp32), the real and three-field
gathers, the paper's variants (Atomic / Tiled spread, Direct / Morton interp) and
the pruned FFT.  Exits non-zero if a result is off (NaN / error)."""
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthetic  # noqa: E402
import paper_2605_10678_b200 as nb  # noqa: E402

N, Np = (32, 32, 32), 20000


def run(prec, eps, **kw):
    rdt = torch.float64 if prec == "f64" else torch.float32
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    pts = [p.to(rdt).cuda() for p in synthetic.uniform_points(Np)]
    c = synthetic.strengths(Np).to(cdt).cuda()
    fk = synthetic.modes(*N).to(cdt).cuda()
    plan = nb.Plan(N, eps, precision=prec, **kw)
    plan.setpts(*pts)
    f = plan.type1(c)
    v = plan.type2(fk)
    torch.cuda.synchronize()
    ok = bool(torch.isfinite(torch.view_as_real(f)).all() and torch.isfinite(torch.view_as_real(v)).all())
    plan.close()
    print(f"{prec} eps={eps:g} {kw}: {'ok' if ok else 'NON-FINITE'}", flush=True)
    return ok


def run_real(eps, **kw):
    pts = [p.cuda() for p in synthetic.uniform_points(Np)]
    c = synthetic.strengths(Np).real.contiguous().cuda()
    fks = [synthetic.modes(*N, seed=40 + d).cuda() for d in range(3)]
    plan = nb.Plan(N, eps, precision="f64", **kw)
    plan.setpts(*pts)
    plan.type1_real(c)
    plan.type2_real(fks[0])
    plan.type2_real3(*fks)
    torch.cuda.synchronize()
    plan.close()
    print(f"real eps={eps:g} {kw}: ok", flush=True)
    return True


def main():
    only = os.environ.get("SANITIZE_ONLY")
    cases = [
        ("f64", 1e-4, {}),                                  # default: sub-bin kernels
        ("f64", 1e-5, {}),
        ("f64", 1e-6, {}),                                  # outer products + tiled interp
        ("f64", 1e-4, dict(spread_warps=8)),                # z-plane spread
        ("f32", 1e-4, {}),
        ("f32", 1e-4, dict(spread_warps=5)),
        ("f64", 1e-4, dict(spread_warps=-2, interp_method=3)),
        ("f64", 1e-4, dict(spread_warps=-3)),
        ("f64", 1e-4, dict(fft_method=1)),
    ]
    ok = True
    for k, (prec, eps, kw) in enumerate(cases):
        if only is None or str(k) in only.split(","):
            ok &= run(prec, eps, **kw)
    if only is None:
        ok &= run_real(1e-4)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
