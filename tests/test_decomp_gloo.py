"""World-size-2 gloo test (CPU) of the z-slab decomposition logic of dist.cpp.

A numpy mirror of the distributed algorithm
run on two gloo ranks, built only from pinned oracle primitives (phi, deconv
factors) and numpy FFTs: owner = slab of the fine z-cell; points moved with
all_to_all; local spread into a slab with halos of floor(w/2) below and
ceil(w/2) above; halo accumulate with the two neighbours; 2D (x, y) FFT of the
owned planes, x-y truncation, all-to-all transpose to y-slabs, 1D z FFT,
z truncation + deconvolution; and the type-2 mirror with halo fill.  The
assembled result must equal the one-rank oracle.
"""
import math
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthetic

P = 2
N = (8, 12, 16)
EPS = 1e-5
L = 2 * math.pi


def _stencil(s, w, beta):
    a = math.ceil(s - w / 2)
    return a, [oracle.phi(2 * (a + i - s) / w, beta) for i in range(w)]


def _fold(v, nf):
    s = (v - L * math.floor(v / L)) * (nf / L)
    return s - nf if s >= nf else s


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        q.put((rank, _run(rank)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _a2a(objs):
    """all-to-all of python objects (list indexed by destination)."""
    out = []
    for src in range(P):
        box = [objs if dist.get_rank() == src else None]
        dist.broadcast_object_list(box, src=src)
        out.append(box[0][dist.get_rank()])
    return out


def _run(rank):
    w, beta, _ = oracle.select_params(EPS)
    nf = tuple(2 * n for n in N)
    nzl = nf[2] // P
    hlo, hhi = w // 2, (w + 1) // 2
    NY = N[1] // P
    Np = 900
    x, y, z = (t.numpy() for t in synthetic.uniform_points(Np, L=L, seed=7))
    c = synthetic.strengths(Np, seed=8).numpy()
    fk = synthetic.modes(*N, seed=9).numpy()
    mine = np.arange(rank, Np, P)                     # round-robin: points start on the wrong rank

    # ---- redistribution: owner = z-slab of the fine cell
    owner = {j: min(int(_fold(z[j], nf[2])), nf[2] - 1) // nzl for j in mine}
    recv = _a2a([[j for j in mine if owner[j] == d] for d in range(P)])
    local = [j for part in recv for j in part]        # global indices of this rank's points
    assert all(min(int(_fold(z[j], nf[2])), nf[2] - 1) // nzl == rank for j in local)

    # ---- type 1: spread into the halo-extended slab
    z_lo = rank * nzl
    G = np.zeros((hlo + nzl + hhi, nf[1], nf[0]), dtype=np.complex128)
    for j in local:
        ax, wx = _stencil(_fold(x[j], nf[0]), w, beta)
        ay, wy = _stencil(_fold(y[j], nf[1]), w, beta)
        az, wz = _stencil(_fold(z[j], nf[2]), w, beta)
        for k in range(w):
            zl = az + k - z_lo
            assert -hlo <= zl < nzl + hhi                      # halo widths suffice
            for jj in range(w):
                for ii in range(w):
                    G[zl + hlo, (ay + jj) % nf[1], (ax + ii) % nf[0]] += c[j] * wx[ii] * wy[jj] * wz[k]
    # halo accumulate: lower halo -> prev's top planes, upper halo -> next's bottom planes
    prev, nxt = (rank - 1) % P, (rank + 1) % P
    got = _a2a([(G[:hlo].copy() if d == prev else None, G[hlo + nzl:].copy() if d == nxt else None)
                for d in range(P)])
    for src, (lo_part, hi_part) in enumerate(got):
        if lo_part is not None:                      # neighbour above sent its lower halo
            G[hlo + nzl - hlo:hlo + nzl] += lo_part
        if hi_part is not None:                      # neighbour below sent its upper halo
            G[hlo:hlo + hhi] += hi_part
    own = G[hlo:hlo + nzl]
    # 2D (x, y) FFT of the owned planes (sign -1), keep retained x, y modes
    B = np.fft.fft2(own, axes=(1, 2))
    ix = [(i - N[0] // 2) % nf[0] for i in range(N[0])]
    iy = [(i - N[1] // 2) % nf[1] for i in range(N[1])]
    Bt = B[:, iy][:, :, ix]                               # (nzl, N2, N1)
    # all-to-all: z-slab -> y-slab
    blocks = _a2a([Bt[:, d * NY:(d + 1) * NY] for d in range(P)])
    Z = np.concatenate(blocks, axis=0)                    # (nf3, NY, N1), z in global order
    Zf = np.fft.fft(Z, axis=0)
    iz = [(i - N[2] // 2) % nf[2] for i in range(N[2])]
    p1, p2, p3 = (oracle.deconv_factors(N[d], nf[d], w, beta) for d in range(3))
    f_loc = Zf[iz] * p1[None, None, :] * p2[None, rank * NY:(rank + 1) * NY, None] * p3[:, None, None]

    # ---- type 2 mirror
    fk_loc = fk[:, rank * NY:(rank + 1) * NY, :]
    Zp = np.zeros((nf[2], NY, N[0]), dtype=np.complex128)
    Zp[iz] = fk_loc * p1[None, None, :] * p2[None, rank * NY:(rank + 1) * NY, None] * p3[:, None, None]
    Zi = np.fft.ifft(Zp, axis=0) * nf[2]                 # sign +1, unnormalised
    back = _a2a([Zi[d * nzl:(d + 1) * nzl] for d in range(P)])   # y-block from each rank
    Bp = np.zeros((nzl, nf[1], nf[0]), dtype=np.complex128)
    for src, blk in enumerate(back):
        Bp[np.ix_(range(nzl), iy[src * NY:(src + 1) * NY], ix)] = blk
    own2 = np.fft.ifft2(Bp, axes=(1, 2)) * (nf[0] * nf[1])
    G2 = np.zeros_like(G)
    G2[hlo:hlo + nzl] = own2
    # halo fill: my bottom hhi planes -> prev's upper halo; my top hlo planes -> next's lower halo
    got = _a2a([(own2[:hhi].copy() if d == prev else None, own2[nzl - hlo:].copy() if d == nxt else None)
                for d in range(P)])
    for src, (bot, top) in enumerate(got):
        if bot is not None:
            G2[hlo + nzl:] = bot
        if top is not None:
            G2[:hlo] = top
    c_loc = {}
    for j in local:
        ax, wx = _stencil(_fold(x[j], nf[0]), w, beta)
        ay, wy = _stencil(_fold(y[j], nf[1]), w, beta)
        az, wz = _stencil(_fold(z[j], nf[2]), w, beta)
        acc = 0j
        for k in range(w):
            for jj in range(w):
                for ii in range(w):
                    acc += G2[az + k - z_lo + hlo, (ay + jj) % nf[1], (ax + ii) % nf[0]] * wx[ii] * wy[jj] * wz[k]
        c_loc[j] = acc
    # results travel back to the caller's rank
    ret = _a2a([{j: v for j, v in c_loc.items() if j % P == d} for d in range(P)])
    mine_out = {}
    for part in ret:
        mine_out.update(part)
    assert sorted(mine_out) == sorted(mine.tolist())
    return f_loc, mine_out


def test_slab_algorithm_two_gloo_ranks_equals_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
    for r in range(P):
        assert not isinstance(res[r], str), res[r]
    f_all = np.concatenate([res[r][0] for r in range(P)], axis=1)
    Np = 900
    x, y, z = (t.numpy() for t in synthetic.uniform_points(Np, L=L, seed=7))
    c = synthetic.strengths(Np, seed=8).numpy()
    fk = synthetic.modes(*N, seed=9).numpy()
    ref1 = oracle.type1(x, y, z, c, N, EPS, L=L)
    assert oracle.rel_l2(f_all, ref1) <= 1e-12
    c_all = np.empty(Np, dtype=np.complex128)
    for r in range(P):
        for j, v in res[r][1].items():
            c_all[j] = v
    ref2 = oracle.type2(x, y, z, fk, EPS, L=L)
    assert oracle.rel_l2(c_all, ref2) <= 1e-12
