"""CPU oracle for the 3D type-1/type-2 NUFFT of arXiv 2605.10678.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with the CUDA product path
(``paper_2605_10678_b200``) and never imports it.

The arithmetic lives in ``oracle/nufft_oracle.cpp`` (plain C++17 + OpenMP,
fp64); this module is argument marshalling over ctypes.  Each wrapper names the
PAPER.md passage its C function follows.  Parity status: every function is
pinned by ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nufft_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_int64_p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fcx-limited-range",
               "-shared", "-fPIC", _SRC, "-o", _LIB + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_select_params.argtypes = [ctypes.c_double, ctypes.POINTER(ctypes.c_int),
                                        _c_double_p]
        L.orc_select_params.restype = ctypes.c_int
        L.orc_phi.argtypes = [ctypes.c_double, ctypes.c_double]
        L.orc_phi.restype = ctypes.c_double
        L.orc_phihat.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int]
        L.orc_phihat.restype = ctypes.c_double
        L.orc_deconv_factors.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_double, _c_double_p]
        pts = [ctypes.c_int64, _c_double_p, _c_double_p, _c_double_p]
        L.orc_spread.argtypes = pts + [_c_double_p, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                       ctypes.c_double, _c_double_p]
        L.orc_interp.argtypes = L.orc_spread.argtypes
        L.orc_fft3d.argtypes = [_c_double_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int]
        L.orc_truncate_deconv.argtypes = [_c_double_p] + [ctypes.c_int64] * 6 + \
            [_c_double_p] * 3 + [_c_double_p]
        L.orc_pad_precorrect.argtypes = [_c_double_p] + [ctypes.c_int64] * 3 + \
            [_c_double_p] * 3 + [ctypes.c_int64] * 3 + [_c_double_p]
        tx = pts + [_c_double_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                    ctypes.c_double, ctypes.c_double, _c_double_p]
        L.orc_type1.argtypes = tx
        L.orc_type1.restype = ctypes.c_int
        L.orc_type2.argtypes = tx
        L.orc_type2.restype = ctypes.c_int
        nu = pts + [_c_double_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                    ctypes.c_double, ctypes.c_int64, _c_int64_p, _c_double_p]
        L.orc_nudft1.argtypes = nu
        L.orc_nudft2.argtypes = nu
        L.orc_nudft2_separable.argtypes = pts + [_c_double_p] * 3 + \
            [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
             ctypes.c_int64, _c_int64_p, _c_double_p]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(_c_double_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def select_params(eps: float):
    """(w, beta, status) -- PAPER.md:181, reading R1."""
    w = ctypes.c_int()
    beta = ctypes.c_double()
    st = lib().orc_select_params(float(eps), ctypes.byref(w), ctypes.byref(beta))
    return w.value, beta.value, st


def phi(z: float, beta: float) -> float:
    """ES window."""
    return lib().orc_phi(float(z), float(beta))


def phihat(xi: float, beta: float, n_nodes: int = 0) -> float:
    """int_{-1}^{1} phi(z) cos(xi z) dz by theta-substituted Gauss-Legendre (R7)."""
    return lib().orc_phihat(float(xi), float(beta), int(n_nodes))


def deconv_factors(N: int, nf: int, w: int, beta: float) -> np.ndarray:
    """p(n) = 2 / (w phihat(pi n w / nf)), n = -N/2..N/2-1 (R6)."""
    p = np.empty(N, dtype=np.float64)
    lib().orc_deconv_factors(N, nf, w, beta, _d(p))
    return p


def spread(x, y, z, c, nf, w, beta, L):
    """Step 1, C. Returns complex grid shaped (nf3, nf2, nf1)."""
    x, y, z, c = _f64(x), _f64(y), _f64(z), _c128(c)
    nf1, nf2, nf3 = nf
    g = np.empty((nf3, nf2, nf1), dtype=np.complex128)
    lib().orc_spread(len(x), _d(x), _d(y), _d(z), _d(c.view(np.float64)), nf1, nf2, nf3, w,
                     beta, L, _d(g.view(np.float64)))
    return g


def interp(x, y, z, grid, w, beta, L):
    """C^T. grid is complex shaped (nf3, nf2, nf1)."""
    x, y, z, g = _f64(x), _f64(y), _f64(z), _c128(grid)
    nf3, nf2, nf1 = g.shape
    out = np.empty(len(x), dtype=np.complex128)
    lib().orc_interp(len(x), _d(x), _d(y), _d(z), _d(g.view(np.float64)), nf1, nf2, nf3, w,
                     beta, L, _d(out.view(np.float64)))
    return out


def fft3d(grid, sign: int):
    """Unnormalised 3D DFT with exponent sign*2*pi*i*m.l/nf. Returns a new array."""
    g = _c128(grid).copy()
    nf3, nf2, nf1 = g.shape
    lib().orc_fft3d(_d(g.view(np.float64)), nf1, nf2, nf3, int(sign))
    return g


def truncate_deconv(grid, N, p):
    """Steps 3+4. grid (nf3,nf2,nf1) -> fk (N3,N2,N1) centered."""
    g = _c128(grid)
    nf3, nf2, nf1 = g.shape
    N1, N2, N3 = N
    p1, p2, p3 = (_f64(q) for q in p)
    fk = np.empty((N3, N2, N1), dtype=np.complex128)
    lib().orc_truncate_deconv(_d(g.view(np.float64)), nf1, nf2, nf3, N1, N2, N3, _d(p1), _d(p2),
                              _d(p3), _d(fk.view(np.float64)))
    return fk


def pad_precorrect(fk, nf, p):
    """D then chi^T. fk (N3,N2,N1) -> grid (nf3,nf2,nf1)."""
    f = _c128(fk)
    N3, N2, N1 = f.shape
    nf1, nf2, nf3 = nf
    p1, p2, p3 = (_f64(q) for q in p)
    g = np.empty((nf3, nf2, nf1), dtype=np.complex128)
    lib().orc_pad_precorrect(_d(f.view(np.float64)), N1, N2, N3, _d(p1), _d(p2), _d(p3), nf1,
                             nf2, nf3, _d(g.view(np.float64)))
    return g


def type1(x, y, z, c, N, eps, iflag=-1, L=2 * np.pi):
    """O-NUFFT type 1 = D chi F C (Eq. 3). Returns fk shaped (N3, N2, N1), centered modes."""
    x, y, z, c = _f64(x), _f64(y), _f64(z), _c128(c)
    N1, N2, N3 = N
    fk = np.empty((N3, N2, N1), dtype=np.complex128)
    lib().orc_type1(len(x), _d(x), _d(y), _d(z), _d(c.view(np.float64)), N1, N2, N3, int(iflag),
                    float(eps), float(L), _d(fk.view(np.float64)))
    return fk


def type2(x, y, z, fk, eps, iflag=-1, L=2 * np.pi):
    """O-NUFFT type 2 = C^T F^-1 chi^T D (Eq. 4). fk shaped (N3, N2, N1)."""
    x, y, z, f = _f64(x), _f64(y), _f64(z), _c128(fk)
    N3, N2, N1 = f.shape
    out = np.empty(len(x), dtype=np.complex128)
    lib().orc_type2(len(x), _d(x), _d(y), _d(z), _d(f.view(np.float64)), N1, N2, N3, int(iflag),
                    float(eps), float(L), _d(out.view(np.float64)))
    return out


def nudft1(x, y, z, c, N, iflag=-1, L=2 * np.pi, sel=None):
    """Exact Eq. (1). sel: optional flat mode indices; returns (N3,N2,N1) or the selected values."""
    x, y, z, c = _f64(x), _f64(y), _f64(z), _c128(c)
    N1, N2, N3 = N
    if sel is None:
        out = np.empty((N3, N2, N1), dtype=np.complex128)
        lib().orc_nudft1(len(x), _d(x), _d(y), _d(z), _d(c.view(np.float64)), N1, N2, N3,
                         int(iflag), float(L), 0, None, _d(out.view(np.float64)))
    else:
        s = np.ascontiguousarray(sel, dtype=np.int64)
        out = np.empty(len(s), dtype=np.complex128)
        lib().orc_nudft1(len(x), _d(x), _d(y), _d(z), _d(c.view(np.float64)), N1, N2, N3,
                         int(iflag), float(L), len(s), s.ctypes.data_as(_c_int64_p),
                         _d(out.view(np.float64)))
    return out


def nudft2(x, y, z, fk, iflag=-1, L=2 * np.pi, sel=None):
    """Exact Eq. (2) with sign -iflag. sel: optional point indices."""
    x, y, z, f = _f64(x), _f64(y), _f64(z), _c128(fk)
    N3, N2, N1 = f.shape
    if sel is None:
        out = np.empty(len(x), dtype=np.complex128)
        lib().orc_nudft2(len(x), _d(x), _d(y), _d(z), _d(f.view(np.float64)), N1, N2, N3,
                         int(iflag), float(L), 0, None, _d(out.view(np.float64)))
    else:
        s = np.ascontiguousarray(sel, dtype=np.int64)
        out = np.empty(len(s), dtype=np.complex128)
        lib().orc_nudft2(len(x), _d(x), _d(y), _d(z), _d(f.view(np.float64)), N1, N2, N3,
                         int(iflag), float(L), len(s), s.ctypes.data_as(_c_int64_p),
                         _d(out.view(np.float64)))
    return out


def nudft2_separable(x, y, z, a1, a2, a3, iflag=-1, L=2 * np.pi, sel=None):
    """Exact Eq. (2) for the rank-one mode array fk[n3, n2, n1] = a1[n1] a2[n2] a3[n3]
    (the triple sum factored into three 1D sums). a_d centered; sel: optional point indices."""
    x, y, z = _f64(x), _f64(y), _f64(z)
    a1, a2, a3 = _c128(a1), _c128(a2), _c128(a3)
    if sel is None:
        s, ns, sp = None, 0, None
        out = np.empty(len(x), dtype=np.complex128)
    else:
        s = np.ascontiguousarray(sel, dtype=np.int64)
        ns, sp = len(s), s.ctypes.data_as(_c_int64_p)
        out = np.empty(len(s), dtype=np.complex128)
    lib().orc_nudft2_separable(len(x), _d(x), _d(y), _d(z), _d(a1.view(np.float64)),
                               _d(a2.view(np.float64)), _d(a3.view(np.float64)), len(a1),
                               len(a2), len(a3), int(iflag), float(L), ns, sp,
                               _d(out.view(np.float64)))
    return out


def max_abs(a, b) -> float:
    """max_j |a_j - b_j| / max_j |b_j| (element-wise companion of rel_l2)."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    nb = np.abs(b).max() if b.size else 0.0
    return float(np.abs(a - b).max() / (nb if nb > 0 else 1.0)) if a.size else 0.0


def rel_l2(a, b) -> float:
    """||a - b||_2 / ||b||_2 (reading R2: the error norm for eps)."""
    a = np.asarray(a).ravel()
    b = np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
