"""Exhaustive (kernel, tile) sweep per ES width on B200 -- SURVEY §8f row f3, the
measured replacement of the paper's Bayesian tile optimisation.

For each precision and tolerance (-> w) and each candidate spread kernel / bin edge
the script times type 1 + type 2 on one seeded uniform workload (per-stage CUDA
events of the plan, median of 5 after 2 warm-ups, L2 flushed before each) and
prints one line per candidate plus the winner per w; the built-in choice
(tile / kernel 0 = default_tile in csrc/plan.cpp) is marked.

usage (GPU box): python scripts/tile_sweep.py [--n 128] [--ppc 1.0] > gpurun_out/tile_sweep.txt
"""
import argparse
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_10678_b200 as nb  # noqa: E402
import synthetic  # noqa: E402


def time_plan(N, eps, prec, pts, c, fk, flush, **kw):
    try:
        plan = nb.Plan(N, eps, precision=prec, timing=True, **kw)
    except nb.NufftError as e:
        return None, str(e)
    plan.setpts(*pts)
    sp, ip = [], []
    for k in range(7):
        flush.fill_(k & 0xff)
        plan.type1(c)
        i1 = plan.info()
        flush.fill_((k + 1) & 0xff)
        plan.type2(fk)
        i2 = plan.info()
        if k >= 2:
            sp.append(i1["ms_spread"])
            ip.append(i2["ms_interp"])
    info = plan.info()
    del plan
    return (statistics.median(sp), statistics.median(ip), tuple(info["tile"]), info["w"]), None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128, help="modes per axis (fine grid 2n)")
    ap.add_argument("--ppc", type=float, default=1.0, help="points per fine cell")
    ap.add_argument("--precs", default="f32,f64")
    args = ap.parse_args()
    N = (args.n,) * 3
    Np = int(args.ppc * (2 * args.n) ** 3)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    x, y, z = synthetic.uniform_points(Np, seed=1)
    c0 = synthetic.strengths(Np)
    fk0 = synthetic.modes(*N)
    print(f"# tile sweep: N = {N}, Np = {Np} ({args.ppc} per fine cell), uniform points")
    print("# columns: prec w kernel tile | spread ms | interp ms | sum ms")
    for prec in args.precs.split(","):
        rdt = torch.float64 if prec == "f64" else torch.float32
        cdt = torch.complex128 if prec == "f64" else torch.complex64
        pts = tuple(p.to(rdt).cuda() for p in (x, y, z))
        c, fk = c0.to(cdt).cuda(), fk0.to(cdt).cuda()
        eps_list = ([1e-2, 1e-3, 1e-4, 1e-5, 1e-6] if prec == "f32" else
                    [1e-3, 1e-4, 1e-5, 1e-6, 1e-7, 1e-8, 1e-9, 1e-10, 1e-11, 1e-12, 1e-13,
                     1e-14])
        for eps in eps_list:
            w = nb.Plan((16, 16, 16), eps, precision=prec).info()["w"]
            cands = [("default", dict())]
            if w <= 12:
                cands.append(("outer", dict(spread_warps=2, tile=16 - w)))
            for t in (4, 6, 8, 10, 12, 16):
                cands.append((f"plane8", dict(spread_warps=8, tile=t)))
            cands.append(("plane4", dict(spread_warps=4, tile=8)))
            rows = []
            for name, kw in cands:
                r, err = time_plan(N, eps, prec, pts, c, fk, flush, **kw)
                if r is None:
                    continue
                sp, ip, tile, _ = r
                rows.append((sp + ip, name, tile[0], sp, ip))
                print(f"{prec} w={w:2d} {name:8s} T={tile[0]:2d} | {sp:8.3f} | {ip:8.3f} | {sp + ip:8.3f}",
                      flush=True)
            best_sp = min(rows, key=lambda r: r[3])
            best_ip = min(rows, key=lambda r: r[4])
            best = min(rows)
            dflt = [r for r in rows if r[1] == "default"][0]
            print(f"# {prec} w={w}: best sum {best[1]} T={best[2]} {best[0]:.3f} ms | default "
                  f"T={dflt[2]} {dflt[0]:.3f} ms ({dflt[0] / best[0]:.3f}x) | best spread "
                  f"{best_sp[1]} T={best_sp[2]} {best_sp[3]:.3f} | best interp T={best_ip[2]} "
                  f"{best_ip[4]:.3f}", flush=True)


if __name__ == "__main__":
    main()
