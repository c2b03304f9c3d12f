"""World-size-2 gloo test (CPU) of the slab REAL-transform algorithm of dist.cpp.

A numpy mirror of the half-spectrum slab transforms (
DESIGN.md §8a) on two gloo ranks, built only from pinned oracle primitives
(phi, deconvolution factors) and numpy FFTs, with each rank owning the points of
its z-slab: real spread into the halo-extended slab, halo accumulate, batched 2D
R2C of the owned planes, keep k1 in [0, N1/2] and the y modes, all-to-all to
y-slabs, 1D z FFT, z truncation + deconvolution (x factor p1(-k1) = p1(k1));
type 2 mirrors it and takes the Hermitian part of the k1 = 0 line of every
z-plane after the transpose, then the 2D C2R.  The half spectrum must equal the
oracle's type 1 of c + 0i (k1 < N1/2; k1 = N1/2 as the conjugate of
(-N1/2, -k2, -k3)), and type 2 the real oracle type 2 of the Hermitian completion.
"""
import math
import os

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthetic

P = 2
N = (8, 12, 16)
EPS = 1e-5
L = 2 * math.pi
NP = 700


def _stencil(s, w, beta):
    a = math.ceil(s - w / 2)
    return a, [oracle.phi(2 * (a + i - s) / w, beta) for i in range(w)]


def _fold(v, nf):
    s = (v - L * math.floor(v / L)) * (nf / L)
    return s - nf if s >= nf else s


def _inputs():
    x, y, z = (t.numpy() for t in synthetic.uniform_points(NP, L=L, seed=17))
    c = synthetic.strengths(NP, seed=18).numpy().real.copy()
    return x, y, z, c


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
    out = []
    for src in range(P):
        box = [objs if dist.get_rank() == src else None]
        dist.broadcast_object_list(box, src=src)
        out.append(box[0][dist.get_rank()])
    return out


def _halo_accumulate(G, hlo, nzl, rank):
    prev, nxt = (rank - 1) % P, (rank + 1) % P
    got = _a2a([(G[:hlo].copy() if d == prev else None, G[hlo + nzl:].copy() if d == nxt else None)
                for d in range(P)])
    for lo_part, hi_part in got:
        if lo_part is not None:
            G[nzl:hlo + nzl] += lo_part
        if hi_part is not None:
            G[hlo:hlo + hi_part.shape[0]] += hi_part


def _run(rank):
    w, beta, _ = oracle.select_params(EPS)
    nf = tuple(2 * n for n in N)
    nzl = nf[2] // P
    hlo, hhi = w // 2, (w + 1) // 2
    NY, H1 = N[1] // P, N[0] // 2 + 1
    x, y, z, c = _inputs()
    local = [j for j in range(NP) if min(int(_fold(z[j], nf[2])), nf[2] - 1) // nzl == rank]
    z_lo = rank * nzl
    stencils = {j: (_stencil(_fold(x[j], nf[0]), w, beta), _stencil(_fold(y[j], nf[1]), w, beta),
                    _stencil(_fold(z[j], nf[2]), w, beta)) for j in local}
    # ---- type 1 (real strengths): real slab with halos
    G = np.zeros((hlo + nzl + hhi, nf[1], nf[0]))
    for j in local:
        (ax, wx), (ay, wy), (az, wz) = stencils[j]
        for k in range(w):
            for jj in range(w):
                for ii in range(w):
                    G[az + k - z_lo + hlo, (ay + jj) % nf[1], (ax + ii) % nf[0]] += \
                        c[j] * wx[ii] * wy[jj] * wz[k]
    _halo_accumulate(G, hlo, nzl, rank)
    H = np.fft.rfft2(G[hlo:hlo + nzl], axes=(1, 2))         # (nzl, nf2, nf1/2 + 1), sign -
    iy = [(i - N[1] // 2) % nf[1] for i in range(N[1])]      # centered y storage -> fine row
    Ht = H[:, iy, :H1]                                        # k1 = 0 .. N1/2
    Z = np.concatenate(_a2a([Ht[:, d * NY:(d + 1) * NY] for d in range(P)]), axis=0)
    Zf = np.fft.fft(Z, axis=0)                                # z, sign -
    iz = [(i - N[2] // 2) % nf[2] for i in range(N[2])]
    p1, p2, p3 = (oracle.deconv_factors(N[d], nf[d], w, beta) for d in range(3))
    px = np.array([p1[N[0] // 2 - k] for k in range(H1)])   # p1(-k1) = p1(k1)
    f_half = Zf[iz] * px[None, None, :] * p2[None, rank * NY:(rank + 1) * NY, None] * p3[:, None, None]
    return f_half, stencils, local, G.shape


def _run_type2(rank, F_half_all):
    w, beta, _ = oracle.select_params(EPS)
    nf = tuple(2 * n for n in N)
    nzl = nf[2] // P
    hlo, hhi = w // 2, (w + 1) // 2
    NY, H1 = N[1] // P, N[0] // 2 + 1
    x, y, z, c = _inputs()
    local = [j for j in range(NP) if min(int(_fold(z[j], nf[2])), nf[2] - 1) // nzl == rank]
    z_lo = rank * nzl
    p1, p2, p3 = (oracle.deconv_factors(N[d], nf[d], w, beta) for d in range(3))
    px = np.array([p1[N[0] // 2 - k] for k in range(H1)])
    iz = [(i - N[2] // 2) % nf[2] for i in range(N[2])]
    iy = [(i - N[1] // 2) % nf[1] for i in range(N[1])]
    F = F_half_all[:, rank * NY:(rank + 1) * NY, :]
    Zp = np.zeros((nf[2], NY, H1), dtype=np.complex128)
    Zp[iz] = F * px[None, None, :] * p2[None, rank * NY:(rank + 1) * NY, None] * p3[:, None, None]
    Zi = np.fft.ifft(Zp, axis=0) * nf[2]                     # sign +, unnormalised
    back = _a2a([Zi[d * nzl:(d + 1) * nzl] for d in range(P)])
    Hp = np.zeros((nzl, nf[1], nf[0] // 2 + 1), dtype=np.complex128)
    for src, blk in enumerate(back):
        Hp[np.ix_(range(nzl), iy[src * NY:(src + 1) * NY], range(H1))] = blk
    # Hermitian part of the k1 = 0 line (all y are local after the transpose)
    mirror = np.conj(Hp[:, (-np.arange(nf[1])) % nf[1], 0])
    Hp[:, :, 0] = 0.5 * (Hp[:, :, 0] + mirror)
    own = np.fft.irfft2(Hp, s=(nf[1], nf[0]), axes=(1, 2)) * (nf[0] * nf[1])
    G2 = np.zeros((hlo + nzl + hhi, nf[1], nf[0]))
    G2[hlo:hlo + nzl] = own
    prev, nxt = (rank - 1) % P, (rank + 1) % P
    got = _a2a([(own[:hhi].copy() if d == prev else None, own[nzl - hlo:].copy() if d == nxt else None)
                for d in range(P)])
    for bot, top in got:
        if bot is not None:
            G2[hlo + nzl:] = bot
        if top is not None:
            G2[:hlo] = top
    out = {}
    for j in local:
        ax, wx = _stencil(_fold(x[j], nf[0]), w, beta)
        ay, wy = _stencil(_fold(y[j], nf[1]), w, beta)
        az, wz = _stencil(_fold(z[j], nf[2]), w, beta)
        acc = 0.0
        for k in range(w):
            for jj in range(w):
                for ii in range(w):
                    acc += G2[az + k - z_lo + hlo, (ay + jj) % nf[1], (ax + ii) % nf[0]] * \
                        wx[ii] * wy[jj] * wz[k]
        out[j] = acc
    return out


def _worker2(rank, port, q, F_half_all):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        q.put((rank, _run_type2(rank, F_half_all)))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _spawn(target, extra=()):
    import socket
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=target, args=(r, port, q) + tuple(extra)) for r in range(P)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
    for r in range(P):
        assert not isinstance(res[r], str), res[r]
    return res


def test_real_slab_algorithm_two_gloo_ranks_equals_oracle():
    res = _spawn(_worker)
    fh = np.concatenate([res[r][0] for r in range(P)], axis=1)   # (N3, N2, N1/2 + 1)
    x, y, z, c = _inputs()
    ref = oracle.type1(x, y, z, c.astype(np.complex128), N, EPS, L=L)   # centered (N3, N2, N1)
    h1 = N[0] // 2
    assert oracle.rel_l2(fh[:, :, :h1], ref[:, :, h1:]) <= 1e-12
    conj_mirror = np.conj(ref[1:, 1:, 0][::-1, ::-1])            # (-N1/2, -k2, -k3)
    assert oracle.rel_l2(fh[1:, 1:, h1], conj_mirror) <= 1e-12
    # type 2 of the half spectrum with its unpaired planes zeroed
    fz = fh.copy()
    fz[:, :, h1] = 0
    fz[0] = 0
    fz[:, 0] = 0
    res2 = _spawn(_worker2, (fz,))
    c2 = np.empty(len(x))
    for r in range(P):
        for j, v in res2[r].items():
            c2[j] = v
    full = np.zeros((N[2], N[1], N[0]), dtype=np.complex128)
    full[:, :, h1:] = fz[:, :, :h1]
    full[1:, 1:, 1:h1] = np.conj(fz[1:, 1:, 1:h1 + 1][::-1, ::-1, ::-1])[:, :, 1:]
    ref2 = oracle.type2(x, y, z, full, EPS, L=L)
    assert np.max(np.abs(ref2.imag)) <= 1e-10 * np.max(np.abs(ref2))   # Hermitian completion
    assert np.linalg.norm(c2 - ref2.real) / np.linalg.norm(ref2.real) <= 1e-12
