"""Distributed PIF step with particle migration, run under torchrun (one GPU per rank).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29512 tests/dist_pif_check.py

PAPER.md:229-235 (particles partitioned like the grid) and PAPER.md:486-491 (one
PIF step).  The slab-decomposed LandauPIF (points owned per rank, leavers
migrated by nufft_pif_migrate after each drift) must evolve the SAME particle
set as a one-GPU LandauPIF started from the gathered initial state:
  * particle count conserved, every particle in its owner's slab after migration;
  * the multiset of (x, y, z, vx, vy, vz) after k steps equal to the one-GPU run
    (matched by sorting; <= 1e-9 relative, spread sums are reordered);
  * a large dt makes many particles cross slab boundaries every step.
Prints one line and exits non-zero on failure.
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_10678_b200 as nb  # noqa: E402
from paper_2605_10678_b200.pif import LandauPIF  # noqa: E402


def gather_var(t):
    """all-gather a 1-D tensor whose length differs per rank"""
    n = torch.tensor([t.numel()], device=t.device)
    ns = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(ns, n)
    m = int(max(int(a.item()) for a in ns))
    pad = torch.zeros(m, dtype=t.dtype, device=t.device)
    pad[:t.numel()] = t
    parts = [torch.empty_like(pad) for _ in ns]
    dist.all_gather(parts, pad)
    return torch.cat([p[:int(k.item())] for p, k in zip(parts, ns)])


def state_sorted(arrs):
    a = torch.stack([t.double() for t in arrs], 1)
    key = a[:, 0] * 1e6 + a[:, 1] * 1e3 + a[:, 2]
    return a[torch.argsort(key)]


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, P = dist.get_rank(), dist.get_world_size()
    comm = nb.Comm()
    dev = torch.device("cuda", local)
    N, Np, steps = (16, 16, 16), 30000, 3
    sim = LandauPIF(N, Np, eps=1e-9, dt=0.4, comm=comm, device=dev, seed=5)
    n0 = int(gather_var(torch.tensor([sim.Np], device=dev)).sum().item())
    init = [gather_var(a) for a in (sim.x, sim.y, sim.z, sim.vx, sim.vy, sim.vz)]
    ok = n0 == Np
    ref = None
    if rank == 0:  # one-GPU run from the same initial particles
        ref = LandauPIF(N, Np, eps=1e-9, dt=0.4, device=dev, seed=5)
        for dst, src in zip(ref._state, init):
            dst.copy_(src)
    crossed = 0
    for _ in range(steps):
        zb = sim.z.clone()
        sim.step()
        if ref is not None:
            ref.step()
        nf3, L = 2 * N[2], sim.L
        cell = torch.floor(torch.remainder(sim.z, L) * (nf3 / L)).clamp(max=nf3 - 1)
        owner = torch.div(cell, nf3 // P, rounding_mode="floor")
        ok &= bool((owner == rank).all().item())
        crossed += int(sim.Np != zb.numel())
    ntot = int(gather_var(torch.tensor([sim.Np], device=dev)).sum().item())
    ok &= ntot == Np
    fin = [gather_var(a) for a in (sim.x, sim.y, sim.z, sim.vx, sim.vy, sim.vz)]
    err = 0.0
    if rank == 0:
        a, b = state_sorted(fin), state_sorted(ref._state)
        err = float(((a - b).abs().max() / b.abs().max()).item())
        ok &= err <= 1e-9
        print(f"pif-migrate P={P}: particles {ntot}/{Np}, rel state diff vs 1 GPU {err:.2e}, "
              f"ranks whose count changed {crossed} step(s) -> {'ok' if ok else 'FAIL'}")
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    sim.plan.close()
    comm.close()
    dist.destroy_process_group()
    sys.exit(0 if int(flag.item()) == 0 else 1)


if __name__ == "__main__":
    main()
