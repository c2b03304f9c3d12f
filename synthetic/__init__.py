"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the NUFFT's arithmetic (no window, no FFT, no
spreading): only a counter-based random generator and the distributions the
paper's workloads use:

* ``u01(seed, stream, n)`` -- splitmix64 of the counter ``seed ^ (stream << 40) ^ i``,
  top 53 bits scaled by 2^-53, in [0, 1).  Pure integer arithmetic, so the
  same numbers come out on the host and on the GPU (torch int64 ops).
* uniform points in [0, L)^3 ("particles are initialized at
  uniformly random positions"), seed 1, streams 0/1/2 for x/y/z;
* Landau-perturbed points, density prop. to prod_d (1 + alpha cos(k x_d)) with
  k = 0.5, alpha = 0.05, L = 2 pi / k, by inverting the
  per-axis CDF ``x + (alpha/k) sin(k x) = u L`` with Newton's method;
* complex strengths / mode coefficients uniform in [-1, 1]^2 (seeds 2 / 3);
* Maxwellian velocities by Box-Muller (seed 4);
* clustered Gaussian blobs (stress case for load imbalance).

Every function takes ``device`` (torch device or string); CPU results are
bitwise-identical to CUDA results for ``u01`` and the uniform positions.
"""
from __future__ import annotations

import math

import torch

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    """Unsigned 64-bit constant -> the int64 with the same bits."""
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_GOLDEN = _s64(0x9E3779B97F4A7C15)
_MIX1 = _s64(0xBF58476D1CE4E5B9)
_MIX2 = _s64(0x94D049BB133111EB)


def _lsr(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bits."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def splitmix64(counter: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (two's-complement wrapping arithmetic)."""
    z = counter + _GOLDEN
    z = (z ^ _lsr(z, 30)) * _MIX1
    z = (z ^ _lsr(z, 27)) * _MIX2
    return z ^ _lsr(z, 31)


def splitmix64_py(x: int) -> int:
    """Pure-Python reference of the same finaliser (used by tests)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def u01(seed: int, stream: int, n: int, start: int = 0, device="cpu",
        chunk: int = 1 << 26) -> torch.Tensor:
    """n uniforms in [0,1) (float64) from counters seed ^ (stream << 40) ^ (start + i)."""
    out = torch.empty(n, dtype=torch.float64, device=device)
    base = _s64((seed & _M64) ^ ((stream & 0xFFFFFF) << 40))
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        i = torch.arange(start + lo, start + hi, dtype=torch.int64, device=device)
        h = splitmix64(i ^ base)
        out[lo:hi] = _lsr(h, 11).to(torch.float64) * (2.0 ** -53)
    return out


def uniform_points(Np: int, L: float = 2 * math.pi, seed: int = 1, device="cpu",
                   dtype=torch.float64):
    """x, y, z uniform in [0, L)."""
    pts = []
    for d in range(3):
        v = u01(seed, d, Np, device=device) * L
        v = torch.where(v >= L, torch.zeros_like(v), v)
        pts.append(v.to(dtype))
    return tuple(pts)


def landau_cdf(x: float, alpha: float = 0.05, k: float = 0.5) -> float:
    """L * F(x) = x + (alpha/k) sin(k x): the unnormalised per-axis CDF."""
    return x + (alpha / k) * math.sin(k * x)


def landau_points(Np: int, alpha: float = 0.05, k: float = 0.5, seed: int = 1, device="cpu",
                  dtype=torch.float64, newton_iters: int = 30, z_range=None):
    """Per-axis inverse-CDF sampling of (1 + alpha cos(k x)) on [0, L), L = 2 pi / k.

    PAPER.md:502-508 (Landau damping initial distribution).  CDF:
    F(x) = (x + (alpha/k) sin(k x)) / L; solve F(x) = u by Newton from x0 = u L
    (F' >= (1 - alpha)/L > 0, so the iteration is monotone and converges).
    z_range = (z0, z1) restricts z to that slab (conditional distribution), for
    ranks that generate their own slab's particles.
    """
    L = 2 * math.pi / k
    pts = []
    for d in range(3):
        target = u01(seed, d, Np, device=device) * L
        if d == 2 and z_range is not None:
            f0, f1 = landau_cdf(z_range[0], alpha, k), landau_cdf(z_range[1], alpha, k)
            target = f0 + target * ((f1 - f0) / L)
        x = target.clone()
        for _ in range(newton_iters):
            f = x + (alpha / k) * torch.sin(k * x) - target
            fp = 1.0 + alpha * torch.cos(k * x)
            x = x - f / fp
        x = torch.remainder(x, L)
        x = torch.where(x >= L, torch.zeros_like(x), x)
        pts.append(x.to(dtype))
    return tuple(pts)


def clustered_points(Np: int, L: float = 2 * math.pi, nblobs: int = 8, sigma: float = 0.05,
                     seed: int = 5, device="cpu", dtype=torch.float64):
    """Gaussian blobs (std sigma*L/ (2 pi) units of L) folded onto the torus: a load-imbalance stress case."""
    centers = [u01(seed, 10 + d, nblobs, device=device) * L for d in range(3)]
    which = torch.floor(u01(seed, 20, Np, device=device) * nblobs).to(torch.int64)
    which = torch.clamp(which, max=nblobs - 1)
    pts = []
    for d in range(3):
        u1 = u01(seed, 30 + 2 * d, Np, device=device)
        u2 = u01(seed, 31 + 2 * d, Np, device=device)
        g = torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos(2 * math.pi * u2)
        v = torch.remainder(centers[d][which] + sigma * L * g, L)
        v = torch.where(v >= L, torch.zeros_like(v), v)
        pts.append(v.to(dtype))
    return tuple(pts)


def complex_uniform(n: int, seed: int, device="cpu", dtype=torch.complex128) -> torch.Tensor:
    """Complex numbers with real and imaginary parts uniform in [-1, 1)."""
    re = 2.0 * u01(seed, 0, n, device=device) - 1.0
    im = 2.0 * u01(seed, 1, n, device=device) - 1.0
    return torch.complex(re, im).to(dtype)


def strengths(Np: int, seed: int = 2, device="cpu", dtype=torch.complex128) -> torch.Tensor:
    return complex_uniform(Np, seed, device=device, dtype=dtype)


def modes(N1: int, N2: int, N3: int, seed: int = 3, device="cpu",
          dtype=torch.complex128) -> torch.Tensor:
    """Mode coefficients shaped (N3, N2, N1) (x fastest), centered ordering."""
    return complex_uniform(N1 * N2 * N3, seed, device=device, dtype=dtype).reshape(N3, N2, N1)


def maxwellian_velocities(Np: int, seed: int = 4, device="cpu", dtype=torch.float64):
    """Three N(0,1) components by Box-Muller (e^{-|v|^2/2})."""
    out = []
    for d in range(3):
        u1 = u01(seed, 2 * d, Np, device=device)
        u2 = u01(seed, 2 * d + 1, Np, device=device)
        out.append((torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos(2 * math.pi * u2)).to(dtype))
    return tuple(out)
