"""Particle-in-Fourier Landau damping on the CUDA path (§4).

* one PIF step against a CPU reference built from the oracle's type 1 / type 2
  and the plain Poisson / leapfrog formulas of SPEC.md:660-665;
* physics: the k = 0.5 Landau mode damps at gamma ~ -0.1533 (linear theory,
  textbook value; within 15 %) and oscillates at omega ~ 1.4156;
* E_0 = 0 and the total charge is Q_e = -L^3.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from errs import err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pifmod():
    from paper_2605_10678_b200 import build
    build.build()
    from paper_2605_10678_b200 import pif
    return pif


@pytest.mark.parametrize("real", [True, False])
def test_one_step_matches_cpu_reference(pifmod, real):
    # real: charges / fields through the R2C / C2R transforms (the one-GPU default)
    N, Np, eps, dt = (8, 10, 12), 6000, 1e-9, 0.05
    sim = pifmod.LandauPIF(N, Np, eps=eps, dt=dt, real=real)
    L = sim.L
    x0, y0, z0, vx0, vy0, vz0 = (t.cpu().numpy().copy() for t in
                                 (sim.x, sim.y, sim.z, sim.vx, sim.vy, sim.vz))
    assert abs(sim.q * Np + L ** 3) < 1e-9 * L ** 3           # Q_e = -L^3
    sim.step()
    torch.cuda.synchronize()
    # CPU reference step
    c = np.full(Np, sim.q, dtype=np.complex128)
    rho = oracle.type1(x0, y0, z0, c, N, eps, L=L)            # (N3, N2, N1)
    n = [np.arange(N[d]) - N[d] // 2 for d in range(3)]
    k1 = (2 * math.pi / L) * n[0][None, None, :]
    k2 = (2 * math.pi / L) * n[1][None, :, None]
    k3 = (2 * math.pi / L) * n[2][:, None, None]
    kk = k1 ** 2 + k2 ** 2 + k3 ** 2
    inv = np.where(kk > 0, 1.0 / np.where(kk > 0, kk, 1.0), 0.0)
    # reading R15: no field on the Nyquist planes (storage index 0 on any axis)
    inv[0, :, :] = 0.0
    inv[:, 0, :] = 0.0
    inv[:, :, 0] = 0.0
    ek = [-1j * kd * rho * inv for kd in (k1, k2, k3)]
    assert np.abs(sim.e_k[0].cpu().numpy()[N[2] // 2, N[1] // 2, N[0] // 2]) == 0.0   # E_0 = 0
    for d in range(3):
        assert err(sim.e_k[d].cpu().numpy(), ek[d]) <= 1e-10
    v = [vx0.copy(), vy0.copy(), vz0.copy()]
    for d in range(3):
        e = oracle.type2(x0, y0, z0, ek[d], eps, L=L)
        v[d] += (-1.0) * dt * e.real / L ** 3
    xs = [np.mod(a + vd * dt, L) for a, vd in zip((x0, y0, z0), v)]
    for got, ref in zip((sim.vx, sim.vy, sim.vz), v):
        assert np.max(np.abs(got.cpu().numpy() - ref)) <= 1e-10 * np.max(np.abs(ref))
    for got, ref in zip((sim.x, sim.y, sim.z), xs):
        diff = np.abs(got.cpu().numpy() - ref)
        diff = np.minimum(diff, L - diff)                      # periodic
        assert np.max(diff) <= 1e-12 * L


def test_landau_damping_rate(pifmod):
    # k = 0.5, alpha = 0.05 (weak Landau damping); linear theory gamma = -0.1533, omega = 1.4156
    sim = pifmod.LandauPIF((16, 16, 16), 1 << 21, eps=1e-4, dt=0.05, precision="f64")
    ts, amp = [], []
    for _ in range(320):
        sim.step()
        ts.append(sim.t)
        # the x-mode n = (1, 0, 0) and its mirror carry the first-order perturbation
        amp.append(sim.mode_amplitude((1, 0, 0)) + sim.mode_amplitude((-1, 0, 0)))
    ts, amp = np.array(ts), np.array(amp)
    peaks = [i for i in range(1, len(amp) - 1) if amp[i] > amp[i - 1] and amp[i] >= amp[i + 1]
             and ts[i] > 0.5]
    assert len(peaks) >= 4, peaks
    tp, ap = ts[peaks], np.log(amp[peaks])
    gamma = np.polyfit(tp, ap, 1)[0]
    omega = math.pi / np.mean(np.diff(tp))      # |E| peaks twice per period
    print(f"gamma = {gamma:.4f} (theory -0.1533), omega = {omega:.4f} (theory 1.4156)")
    assert abs(gamma - (-0.1533)) <= 0.15 * 0.1533
    assert abs(omega - 1.4156) <= 0.05 * 1.4156
