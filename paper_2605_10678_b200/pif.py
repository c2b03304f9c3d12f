"""Particle-in-Fourier Landau damping on the NUFFT plan (§4).

One step: (1) scatter the charges to Fourier space with a
type-1 NUFFT, (2) solve Gauss's law E_k = -i k rho_k / |k|^2 (E_0 = 0),
(3) gather each E component at the particles with a type-2 NUFFT, (4) leapfrog
kick v += (q/m) dt Re E / L^3 and drift x += v dt (folded onto [0, L)).
Plasma units, electrons q/m = -1, total charge Q_e = -L^3, L = 2 pi / k
(SPEC.md:660-665 for the Poisson/push conventions).  Every
arithmetic step runs in libnufft kernels (type 1/2, nufft_pif_poisson,
nufft_pif_kick, nufft_pif_drift); this class holds buffers and calls them.

With a Comm the plan is a z-slab plan (particles partitioned
like the grid): each rank samples ITS slab's share of the Landau distribution (z
conditioned on the slab) and OWNS the particles in its slab (opts.points_owned).
After every drift, nufft_pif_migrate sends the few particles that crossed a slab
boundary, with their velocities, to the new owner -- the transforms themselves
never move points.  Particle arrays carry slack capacity for the migration.
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import nufft as _n


class LandauPIF:
    def __init__(self, N, Np, eps=1e-4, dt=0.01, alpha=0.05, k=0.5, precision="f64",
                 comm=None, device=None, seed=1, timing=False, real=None, tile=None,
                 spread_warps=0, fused=False):
        import synthetic
        self.N = tuple(N)
        self.k, self.alpha, self.dt = k, alpha, dt
        self.L = 2 * math.pi / k
        self.qm = -1.0
        self.plan = _n.Plan(N, eps, precision=precision, L=self.L, comm=comm, device=device,
                            timing=timing, points_owned=comm is not None, tile=tile,
                            spread_warps=spread_warps)
        dev = self.plan.device
        rdt, cdt = self.plan.real, self.plan.cplx
        self.Np_total = int(Np)
        if comm is None:
            self.Np = int(Np)
            pts = synthetic.landau_points(self.Np, alpha=alpha, k=k, seed=seed, device=dev, dtype=rdt)
        else:
            P, r = comm.size, comm.rank
            nf3 = 2 * N[2]
            z0, z1 = self.L * r / P, self.L * (r + 1) / P       # slab r of the fine grid
            f0, f1 = synthetic.landau_cdf(z0, alpha, k), synthetic.landau_cdf(z1, alpha, k)
            bounds = [round(Np * synthetic.landau_cdf(self.L * q / P, alpha, k) / self.L)
                      for q in range(P + 1)]
            self.Np = bounds[r + 1] - bounds[r]
            assert nf3 % P == 0 and f1 > f0
            pts = synthetic.landau_points(self.Np, alpha=alpha, k=k, seed=seed + 7919 * r,
                                          device=dev, dtype=rdt, z_range=(z0, z1))
        vel = synthetic.maxwellian_velocities(self.Np, seed=seed + 4 + 104729 * (comm.rank if comm else 0),
                                              device=dev, dtype=rdt)
        # particle state with slack capacity (slab plans: migration changes the count)
        self.cap = self.Np if comm is None else self.Np + self.Np // 8 + 4096
        src = [*pts, *vel]
        del pts, vel
        self._state = []
        while src:                                          # one array at a time (memory)
            a = src.pop(0)
            if self.cap == self.Np:
                self._state.append(a.contiguous())
            else:
                buf = torch.empty(self.cap, dtype=rdt, device=dev)
                buf[:self.Np].copy_(a)
                self._state.append(buf)
            del a
        self.q = -self.L ** 3 / self.Np_total              # Q_e = -L^3 shared equally
        # charges and fields are real: the real-valued transforms
        # (R2C / C2R) by default -- on a slab plan their modes are the k1 = 0 .. N1/2
        # half spectrum (nufft.h), which the Poisson solve handles mode by mode
        self.real = True if real is None else bool(real)
        self.half = self.real and comm is not None
        self.charge = torch.full((self.cap,), self.q, dtype=rdt if self.real else cdt, device=dev)
        shape = self.plan.local_shape_real if self.real else self.plan.local_shape
        self.rho_k = torch.empty(shape, dtype=cdt, device=dev)
        self.e_k = [torch.empty(shape, dtype=cdt, device=dev) for _ in range(3)]
        # per-component field gathers through e_pts; the fused three-field gather +
        # kick (nufft_pif_gather_kick) is correct but measured slower on B200 (C4:
        # 808 ms vs 3 x 144 ms: three component tiles halve the resident CTAs of a
        # shared-memory-latency-bound kernel), so it is opt-in
        self.fused = fused and self.real and comm is None
        self.e_pts = (None if self.fused else
                      torch.empty(self.cap, dtype=rdt if self.real else cdt, device=dev))
        self.t = 0.0
        if comm is not None:
            self.migrate()   # sampling at a slab edge may round into the neighbour's cell

    # views of this rank's particles
    x = property(lambda s: s._state[0][:s.Np])
    y = property(lambda s: s._state[1][:s.Np])
    z = property(lambda s: s._state[2][:s.Np])
    vx = property(lambda s: s._state[3][:s.Np])
    vy = property(lambda s: s._state[4][:s.Np])
    vz = property(lambda s: s._state[5][:s.Np])

    def migrate(self):
        """Hand particles that left this rank's slab to their owners (collective)."""
        n = ctypes.c_int64(self.Np)
        with self.plan._call():
            _n._check(_n.lib().nufft_pif_migrate(self.plan._h, ctypes.byref(n), self.cap,
                                                 *(ctypes.c_void_p(a.data_ptr())
                                                   for a in self._state)),
                      "nufft_pif_migrate")
        self.Np = int(n.value)

    def step(self):
        p, L = self.plan, _n.lib()
        n = self.Np
        with p._call():                      # plan stream, ordered against the caller's
            p.setpts(self.x, self.y, self.z)                                   # sort
            if self.real:
                p.type1_real(self.charge[:n], out=self.rho_k)                  # (1) scatter
            else:
                p.type1(self.charge[:n], out=self.rho_k)
            poisson = L.nufft_pif_poisson_real if self.real else L.nufft_pif_poisson
            _n._check(poisson(p._h, self.rho_k.data_ptr(), *(e.data_ptr() for e in self.e_k)),
                      "nufft_pif_poisson")                                      # (2) field solve
            s = self.qm * self.dt / self.L ** 3
            if self.fused:   # (3) + (4): three-field gather with the kick fused in
                _n._check(L.nufft_pif_gather_kick(p._h, *(e.data_ptr() for e in self.e_k),
                                                  *(ctypes.c_void_p(v.data_ptr()) for v in
                                                    (self.vx, self.vy, self.vz)),
                                                  ctypes.c_double(s)), "nufft_pif_gather_kick")
            else:
                e_pts = self.e_pts[:n]
                kick = L.nufft_pif_kick_real if self.real else L.nufft_pif_kick
                for e_k, v in zip(self.e_k, (self.vx, self.vy, self.vz)):
                    if self.real:
                        p.type2_real(e_k, out=e_pts)                            # (3) gather
                    else:
                        p.type2(e_k, out=e_pts)
                    _n._check(kick(p._h, n, ctypes.c_void_p(v.data_ptr()),
                                   ctypes.c_void_p(e_pts.data_ptr()), ctypes.c_double(s)),
                              "nufft_pif_kick")                                 # (4) push
            _n._check(L.nufft_pif_drift(p._h, n, *(ctypes.c_void_p(a.data_ptr()) for a in
                                                   (self.x, self.y, self.z, self.vx, self.vy, self.vz)),
                                        ctypes.c_double(self.dt)), "nufft_pif_drift")
            if p.comm is not None:
                self.migrate()                                                  # slab ownership
        self.t += self.dt

    def _half_weights(self):
        """sum over the full box = sum over k1 = 0 (x1) and 0 < k1 < N1/2 (x2, conjugate
        partners); the k1 = N1/2 column stands for the box's -N1/2 modes (x1)"""
        h = self.N[0] // 2 + 1
        w = torch.full((h,), 2.0, dtype=torch.float64, device=self.plan.device)
        w[0] = 1.0
        w[-1] = 1.0
        return w

    def field_energy(self) -> float:
        """0.5 int |E|^2 dx = 0.5 L^-3 sum_k |E_k|^2 (this rank's modes; all-reduce for a slab plan)."""
        if self.half:
            wx = self._half_weights()
            w = sum(float(((e.abs() ** 2).double() * wx).sum()) for e in self.e_k) * 0.5 / self.L ** 3
        else:
            w = sum(float((e.abs() ** 2).sum()) for e in self.e_k) * 0.5 / self.L ** 3
        if self.plan.comm is not None:
            import torch.distributed as dist
            t = torch.tensor([w], dtype=torch.float64, device=self.plan.device)
            dist.all_reduce(t)
            w = float(t.item())
        return w

    def mode_amplitude(self, n=(1, 0, 0)) -> float:
        """|E_x|-component amplitude of one mode n, summed over ranks."""
        lo, hi = self.plan.local_modes()
        if self.half:  # x index = k1 >= 0; |E(n)| = |E(-n)| for a real field
            if n[0] < 0:
                n = tuple(-v for v in n)
            lo, hi = (0, lo[1], lo[2]), (self.N[0] // 2 + 1, hi[1], hi[2])
            idx = [n[0], n[1] + self.N[1] // 2, n[2] + self.N[2] // 2]
        else:
            idx = [n[d] + self.N[d] // 2 for d in range(3)]
        val = 0.0
        if all(lo[d] <= idx[d] < hi[d] for d in range(3)):
            e = self.e_k[0][idx[2] - lo[2], idx[1] - lo[1], idx[0] - lo[0]]
            val = float(e.abs())
        if self.plan.comm is not None:
            import torch.distributed as dist
            t = torch.tensor([val], dtype=torch.float64, device=self.plan.device)
            dist.all_reduce(t)
            val = float(t.item())
        return val
