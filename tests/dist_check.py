"""Distributed (z-slab) NUFFT check, run under torchrun with P GPUs (one per rank).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tests/dist_check.py

SURVEY.md §8e / SPEC.md:538-540 invariants: the P-rank type 1 / type 2 equal the
one-GPU plan on the same points (<= 1e-12 fp64, <= 1e-5 fp32, atomics reorder
sums) and the CPU oracle (<= 1e-10 fp64 / 1e-4 fp32), with points given to the
"wrong" ranks (redistributed by setpts) and with points_owned.  Prints one
line per case and exits non-zero on failure.
"""
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synthetic  # noqa: E402
import paper_2605_10678_b200 as nb  # noqa: E402


def gather_cat(t, dim=0):
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t.contiguous())
    return torch.cat(parts, dim=dim)


def run_case(comm, N, Np, eps, prec, owned, kind, L, **kw):
    rank, P = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device())
    rdt = torch.float64 if prec == "f64" else torch.float32
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    if kind == "landau":
        pts = [p.to(rdt) for p in synthetic.landau_points(Np)]
    else:
        pts = [p.to(rdt) for p in synthetic.uniform_points(Np, L=L)]
    c = synthetic.strengths(Np).to(cdt)
    fk = synthetic.modes(*N).to(cdt)
    nf3 = 2 * N[2]
    if owned:  # give each rank exactly its slab's points
        zz = pts[2].double()  # the library's fold (reading R10), bit for bit
        s = (zz - L * torch.floor(zz / L)) * (nf3 / L)
        s = torch.where(s >= nf3, s - nf3, s)
        owner = torch.clamp(torch.floor(s).long(), max=nf3 - 1) // (nf3 // P)
        mine = torch.nonzero(owner == rank).flatten()
    else:      # round-robin: most points start on the wrong rank
        mine = torch.arange(rank, Np, P)
    xl, yl, zl = (p[mine].contiguous().to(dev) for p in pts)
    cl = c[mine].contiguous().to(dev)

    dbg = os.environ.get("DIST_DEBUG")
    def mark(s):
        if dbg:
            torch.cuda.synchronize()
            print(f"[rank {rank}] {s}", file=sys.stderr, flush=True)
    mark("plan")
    plan = nb.Plan(N, eps, precision=prec, L=L, comm=comm, points_owned=owned, **kw)
    lo, hi = plan.local_modes()
    mark(f"setpts lo={lo} hi={hi}")
    plan.setpts(xl, yl, zl)
    mark("type1")
    f_loc = plan.type1(cl)
    fk_loc = fk[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]].contiguous().to(dev)
    mark("type2")
    c_loc = plan.type2(fk_loc)
    torch.cuda.synchronize()
    mark("gather")
    f_all = gather_cat(f_loc, dim=1).cpu()               # y-slabs -> full modes
    mark("gathered modes")
    # outputs of type 2 back in caller order on each rank: gather (index, value);
    # per-rank sizes differ (points_owned), so gather as objects
    parts = [None] * P
    dist.all_gather_object(parts, (mine.numpy(), c_loc.cpu().numpy()))
    c2_all = torch.empty(Np, dtype=cdt)
    for idx, val in parts:
        c2_all[torch.from_numpy(idx)] = torch.from_numpy(val)
    mark("gathered values")

    # one-GPU reference plan on all points
    ref = nb.Plan(N, eps, precision=prec, L=L)
    ref.setpts(*(p.to(dev) for p in pts))
    f_ref = ref.type1(c.to(dev)).cpu()
    c_ref = ref.type2(fk.to(dev)).cpu()
    tol_same = 1e-12 if prec == "f64" else 1e-5
    tol_orc = 1e-10 if prec == "f64" else 1e-4
    e1 = oracle.rel_l2(f_all.numpy(), f_ref.numpy())
    e2 = oracle.rel_l2(c2_all.numpy(), c_ref.numpy())
    ok = e1 <= tol_same and e2 <= tol_same
    o1 = o2 = 0.0
    if rank == 0:
        x, y, z = (p.double().numpy() for p in pts)
        o1 = oracle.rel_l2(f_all.numpy(), oracle.type1(x, y, z, c.numpy().astype(np.complex128), N, eps, L=L))
        o2 = oracle.rel_l2(c2_all.numpy(), oracle.type2(x, y, z, fk.numpy().astype(np.complex128), eps, L=L))
        ok = ok and o1 <= tol_orc and o2 <= tol_orc
        print(f"P={P} N={N} Np={Np} eps={eps:g} {prec} owned={owned} {kind} {kw}: "
              f"vs 1-GPU {e1:.2e}/{e2:.2e}  vs oracle {o1:.2e}/{o2:.2e}  {'OK' if ok else 'FAIL'}",
              flush=True)
    plan.close()
    ref.close()
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    return int(flag.item()) == 0


def run_real_case(comm, N, Np, eps, prec, owned, L):
    """Real-valued transforms on the slab plan (half-spectrum layout, nufft.h) against the
    one-GPU real transforms on the same points."""
    rank, P = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", torch.cuda.current_device())
    rdt = torch.float64 if prec == "f64" else torch.float32
    pts = [p.to(rdt) for p in synthetic.uniform_points(Np, L=L, seed=31)]
    c = synthetic.strengths(Np, seed=32).real.contiguous().to(rdt)
    nf3 = 2 * N[2]
    if owned:
        zz = pts[2].double()
        s = (zz - L * torch.floor(zz / L)) * (nf3 / L)
        s = torch.where(s >= nf3, s - nf3, s)
        owner = torch.clamp(torch.floor(s).long(), max=nf3 - 1) // (nf3 // P)
        mine = torch.nonzero(owner == rank).flatten()
    else:
        mine = torch.arange(rank, Np, P)
    xl, yl, zl = (p[mine].contiguous().to(dev) for p in pts)
    plan = nb.Plan(N, eps, precision=prec, L=L, comm=comm, points_owned=owned)
    lo, hi = plan.local_modes()
    plan.setpts(xl, yl, zl)
    fh_loc = plan.type1_real(c[mine].contiguous().to(dev))          # (N3, NY, N1/2 + 1)
    fh = gather_cat(fh_loc, dim=1).cpu().to(torch.complex128)        # (N3, N2, N1/2 + 1)
    ref = nb.Plan(N, eps, precision=prec, L=L)
    ref.setpts(*(p.to(dev) for p in pts))
    ff = ref.type1_real(c.to(dev)).cpu().to(torch.complex128)       # (N3, N2, N1) centered
    h1 = N[0] // 2
    # k1 in [0, N1/2): stored at centered x index N1/2 + k1
    e1 = oracle.rel_l2(fh[:, :, :h1].numpy(), ff[:, :, h1:].numpy())
    # k1 = +N1/2: the conjugate of (-N1/2, -k2, -k3) where -k2, -k3 are stored
    a = fh[1:, 1:, h1]                                   # k2, k3 in (-N/2, N/2)
    b = torch.conj(torch.flip(ff[1:, 1:, 0], dims=(0, 1))).resolve_conj()
    e1b = oracle.rel_l2(a.numpy(), b.numpy())
    # type 2: the slab's own half spectrum with the unpaired planes zeroed, against the
    # one-GPU real transform of its Hermitian completion
    fz = fh.clone()
    fz[:, :, h1] = 0
    fz[0, :, :] = 0
    fz[:, 0, :] = 0
    full = torch.zeros((N[2], N[1], N[0]), dtype=torch.complex128)
    full[:, :, h1:] = fz[:, :, :h1]                                      # k1 >= 0
    mirror = torch.conj(torch.flip(fz[1:, 1:, 1:h1 + 1], dims=(0, 1, 2))).resolve_conj()  # -k, k1 > 0
    full[1:, 1:, 1:h1] = mirror[:, :, 1:]                                # k1 = -N1/2+1 .. -1
    cdt = torch.complex128 if prec == "f64" else torch.complex64
    c2_loc = plan.type2_real(fz[:, lo[1]:hi[1], :].contiguous().to(cdt).to(dev))
    c2_ref = ref.type2_real(full.to(cdt).to(dev)).cpu().double()
    parts = [None] * P
    dist.all_gather_object(parts, (mine.numpy(), c2_loc.cpu().double().numpy()))
    c2_all = torch.empty(Np, dtype=torch.float64)
    for idx, val in parts:
        c2_all[torch.from_numpy(idx)] = torch.from_numpy(val)
    e2 = float(torch.linalg.norm(c2_all - c2_ref) / torch.linalg.norm(c2_ref))
    tol = 1e-12 if prec == "f64" else 1e-5
    ok = e1 <= tol and e1b <= tol and e2 <= tol
    if rank == 0:
        print(f"P={P} N={N} Np={Np} eps={eps:g} {prec} owned={owned} REAL: type1 vs 1-GPU "
              f"{e1:.2e} (k1=N1/2: {e1b:.2e}), type2 {e2:.2e}  {'OK' if ok else 'FAIL'}",
              flush=True)
    plan.close()
    ref.close()
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    return int(flag.item()) == 0


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = nb.Comm()
    cases = [
        ((32, 32, 32), 40000, 1e-6, "f64", False, "uniform", 2 * math.pi),
        ((32, 32, 32), 40000, 1e-6, "f64", True, "uniform", 2 * math.pi),
        ((16, 24, 32), 30000, 1e-9, "f64", False, "landau", 4 * math.pi),
        ((32, 32, 32), 40000, 1e-4, "f32", False, "uniform", 2 * math.pi),
        ((64, 64, 64), 300000, 1e-5, "f64", False, "uniform", 2 * math.pi),
    ]
    ok = all([run_case(comm, *cs) for cs in cases])
    # kernel options on slabs: the paper's Atomic Spread / Direct Interpolation
    # (caller and bin-sorted order) and the tcgen05 spread (fp32)
    opt_cases = [
        (((32, 32, 32), 40000, 1e-6, "f64", False, "uniform", 2 * math.pi),
         dict(spread_warps=-1, interp_method=1)),
        (((32, 32, 32), 40000, 1e-6, "f64", True, "landau", 4 * math.pi),
         dict(spread_warps=-2, interp_method=2)),
        (((64, 64, 64), 200000, 1e-5, "f32", True, "uniform", 2 * math.pi),
         dict(spread_warps=3)),
    ]
    ok = all([run_case(comm, *cs, **kw) for cs, kw in opt_cases]) and ok
    real_cases = [
        ((32, 32, 32), 40000, 1e-9, "f64", True, 2 * math.pi),
        ((16, 24, 32), 30000, 1e-6, "f64", False, 4 * math.pi),
        ((32, 32, 32), 40000, 1e-5, "f32", True, 2 * math.pi),
    ]
    ok = all([run_real_case(comm, *cs) for cs in real_cases]) and ok
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
