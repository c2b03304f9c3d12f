"""Developer probe: per-warp produce / consume / barrier cycles of spread_outer_kernel.

    NUFFT_EXTRA_NVCC_FLAGS=-DNUFFT_OUTER_PROF python -m paper_2605_10678_b200.build --force
    python scripts/outer_prof.py [N] [ppc] [eps] [f64|f32]

Rebuild without the flag afterwards (the product build never defines it).
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
import paper_2605_10678_b200 as nb  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    ppc = float(sys.argv[2]) if len(sys.argv) > 2 else 8
    eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
    prec = sys.argv[4] if len(sys.argv) > 4 else "f64"
    Np = int(ppc * N ** 3)
    dt = torch.float64 if prec == "f64" else torch.float32
    ct = torch.complex128 if prec == "f64" else torch.complex64
    pts = [p.to(dt).cuda() for p in synthetic.uniform_points(Np, seed=1)]
    c = synthetic.strengths(Np).to(ct).cuda()
    w = nb.Plan((8, 8, 8), eps, precision=prec).info()["w"]
    plan = nb.Plan((N, N, N), eps, precision=prec, spread_warps=2, tile=16 - w, timing=True)
    plan.setpts(*pts)
    L = nb.lib()
    L.nufft_debug_outer_prof.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
    buf = (ctypes.c_ulonglong * 64)()
    plan.type1(c)
    torch.cuda.synchronize()
    L.nufft_debug_outer_prof(buf)
    reps = 3
    for _ in range(reps):
        plan.type1(c)
    torch.cuda.synchronize()
    L.nufft_debug_outer_prof(buf)
    info = plan.info()
    print(f"N={N} ppc={ppc} eps={eps} {prec} w={info['w']} tile={info['tile']} "
          f"spread {info['ms_spread']:.3f} ms")
    for w in range(8):
        pr, co, ba = buf[8 * w], buf[8 * w + 1], buf[8 * w + 2]
        tot = pr + co + ba
        ph = [buf[8 * w + k] for k in (3, 4, 5, 6)]
        print(f"warp {w}: produce {100 * pr / tot:5.1f}%  consume {100 * co / tot:5.1f}%  "
              f"barrier {100 * ba / tot:5.1f}%  | produce split: zero+reset {100 * ph[0] / tot:4.1f}% "
              f"load+rank {100 * ph[1] / tot:4.1f}% scan {100 * ph[2] / tot:4.1f}% "
              f"weights {100 * ph[3] / tot:4.1f}% | whole CTA {buf[8 * w + 7] / reps:.3e} cyc "
              f"(loop {tot / reps:.3e})")


if __name__ == "__main__":
    main()
