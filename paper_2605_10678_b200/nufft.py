"""Thin ctypes binding of libnufft.so (include/nufft.h) -- argument marshalling only.

Every step of the NUFFT runs in the library's CUDA kernels (and cuFFT).  This
module converts torch tensors to raw pointers and raises on non-zero status.
The plan runs on the stream current at plan creation (or ``stream=``); every
call is ordered after the caller's CURRENT stream (its inputs are ready) and
the caller's stream waits for the plan stream afterwards (outputs are visible),
with the tensors recorded on the plan stream for the caching allocator.  There is NO CPU fallback: if the shared library
is missing or CUDA is absent the calls fail loudly.

    import torch, paper_2605_10678_b200 as nb
    plan = nb.Plan((N1, N2, N3), eps=1e-6, precision="f64")   # iflag=-1: Eq. (1)
    plan.setpts(x, y, z)          # torch tensors, CUDA (or pinned host) memory
    fk = plan.type1(c)            # (N3, N2, N1) complex, centered modes
    c2 = plan.type2(fk)           # (Np,) complex, caller order
"""
from __future__ import annotations

import contextlib
import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# NUFFT_LIB selects another build of the same library (the bounds-checked
# libnufft_debug.so of build.py); default: the in-tree product build
LIB_PATH = os.environ.get("NUFFT_LIB") or os.path.join(_HERE, "libnufft.so")

F32, F64 = 0, 1


class NufftError(RuntimeError):
    pass


class Opts(ctypes.Structure):
    _fields_ = [("L", ctypes.c_double), ("modeord", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("comm", ctypes.c_void_p), ("points_owned", ctypes.c_int),
                ("tile", ctypes.c_int * 3), ("timing", ctypes.c_int),
                ("spread_warps", ctypes.c_int), ("precompute", ctypes.c_int),
                ("interp_method", ctypes.c_int), ("fft_method", ctypes.c_int),
                ("reserved", ctypes.c_int * 3)]


class Info(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_int), ("w", ctypes.c_int), ("beta", ctypes.c_double),
                ("eps", ctypes.c_double), ("N", ctypes.c_int64 * 3), ("nf", ctypes.c_int64 * 3),
                ("tile", ctypes.c_int * 3), ("nbins", ctypes.c_int64), ("Np", ctypes.c_int64),
                ("device_bytes", ctypes.c_size_t), ("nranks", ctypes.c_int),
                ("rank", ctypes.c_int), ("slab_lo", ctypes.c_int64), ("slab_hi", ctypes.c_int64),
                ("ms_setpts", ctypes.c_float), ("ms_spread", ctypes.c_float),
                ("ms_fold", ctypes.c_float), ("ms_fft", ctypes.c_float),
                ("ms_deconv", ctypes.c_float), ("ms_pad", ctypes.c_float),
                ("ms_interp", ctypes.c_float), ("ms_comm", ctypes.c_float),
                ("weights_precomputed", ctypes.c_int), ("sub_bins", ctypes.c_int)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if hasattr(v, "__len__") else v
        return d


_EXPORTS = ["nufft_default_opts", "nufft_plan", "nufft_setpts", "nufft_execute_type1",
            "nufft_execute_type2", "nufft_spread", "nufft_interp", "nufft_destroy",
            "nufft_get_info", "nufft_strerror", "nufft_comm_unique_id", "nufft_comm_init",
            "nufft_comm_destroy", "nufft_local_modes", "nufft_pif_poisson", "nufft_pif_kick",
            "nufft_pif_drift", "nufft_pif_migrate", "nufft_execute_type1_real",
            "nufft_execute_type2_real", "nufft_pif_kick_real", "nufft_pif_poisson_real",
            "nufft_execute_type2_real3", "nufft_pif_gather_kick", "nufft_fma_peak",
            "nufft_comm_init_loopback"]

_lib = None


def lib():
    """Load libnufft.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NufftError(f"{LIB_PATH} missing: run `python -m paper_2605_10678_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        L.nufft_default_opts.argtypes = [ctypes.POINTER(Opts)]
        L.nufft_plan.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                                        ctypes.POINTER(Opts), ctypes.POINTER(vp)]
        L.nufft_setpts.argtypes = [vp, ctypes.c_int64, vp, vp, vp]
        for f in ("nufft_execute_type1", "nufft_execute_type2", "nufft_spread", "nufft_interp",
                  "nufft_execute_type1_real", "nufft_execute_type2_real"):
            getattr(L, f).argtypes = [vp, vp, vp]
        L.nufft_destroy.argtypes = [vp]
        L.nufft_fma_peak.argtypes = [ctypes.c_int, vp, ctypes.POINTER(ctypes.c_double)]
        L.nufft_get_info.argtypes = [vp, ctypes.POINTER(Info)]
        L.nufft_strerror.argtypes = [ctypes.c_int]
        L.nufft_strerror.restype = ctypes.c_char_p
        L.nufft_comm_unique_id.argtypes = [ctypes.c_char_p]
        L.nufft_comm_init.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(vp)]
        L.nufft_comm_destroy.argtypes = [vp]
        L.nufft_comm_init_loopback.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
        L.nufft_pif_poisson.argtypes = [vp, vp, vp, vp, vp]
        L.nufft_pif_poisson_real.argtypes = [vp, vp, vp, vp, vp]
        L.nufft_execute_type2_real3.argtypes = [vp, vp, vp, vp, vp]
        L.nufft_pif_gather_kick.argtypes = [vp, vp, vp, vp, vp, vp, vp, ctypes.c_double]
        L.nufft_pif_kick.argtypes = [vp, ctypes.c_int64, vp, vp, ctypes.c_double]
        L.nufft_pif_kick_real.argtypes = [vp, ctypes.c_int64, vp, vp, ctypes.c_double]
        L.nufft_pif_drift.argtypes = [vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp, ctypes.c_double]
        L.nufft_pif_migrate.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                        vp, vp, vp, vp, vp, vp]
        L.nufft_local_modes.argtypes = [vp, ctypes.POINTER(ctypes.c_int64),
                                        ctypes.POINTER(ctypes.c_int64)]
        _lib = L
    return _lib


def _check(st: int, what: str) -> int:
    if st >= 2:
        raise NufftError(f"{what}: {lib().nufft_strerror(st).decode()} (status {st})")
    return st


def _ptr(t: torch.Tensor, dtype, n: int, name: str) -> int:
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() != n:
        raise ValueError(f"{name}: expected {n} elements, got {t.numel()}")
    return t.data_ptr()


class Comm:
    """libnufft's NCCL communicator for a z-slab plan (one process per GPU).

    The 128-byte NCCL id made by rank 0 (nufft_comm_unique_id) travels through the
    torch.distributed process group; every rank then calls nufft_comm_init.
    """

    def __init__(self, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(lib().nufft_comm_unique_id(uid), "nufft_comm_unique_id")
        box = [uid.raw if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = ctypes.create_string_buffer(box[0], 128)
        h = ctypes.c_void_p()
        _check(lib().nufft_comm_init(uid, self.size, self.rank, ctypes.byref(h)), "nufft_comm_init")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().nufft_comm_destroy(self._h)
            self._h = None

    @classmethod
    def loopback(cls, nranks: int):
        """nranks loopback communicators on the current GPU (nufft_comm_init_loopback):
        rank r's plan must be driven from its own host thread.  For tests of the
        z-slab path at any rank count on one device."""
        hs = (ctypes.c_void_p * nranks)()
        _check(lib().nufft_comm_init_loopback(nranks, hs), "nufft_comm_init_loopback")
        out = []
        for r in range(nranks):
            c = cls.__new__(cls)
            c.rank, c.size, c._h = r, nranks, ctypes.c_void_p(hs[r])
            out.append(c)
        return out


def fma_peak(precision="f64", stream=None) -> float:
    """Measured FMA-pipe peak of the current GPU in TFLOP/s (nufft_fma_peak)."""
    st = (stream or torch.cuda.current_stream()).cuda_stream
    v = ctypes.c_double()
    prec = F64 if precision in ("f64", "double", torch.float64) else F32
    _check(lib().nufft_fma_peak(prec, ctypes.c_void_p(st), ctypes.byref(v)), "nufft_fma_peak")
    return float(v.value)


class Plan:
    """One NUFFT plan (type 1 and type 2 share the points and the fine grid).

    N        : (N1, N2, N3) even mode counts
    eps      : tolerance (relative l2), selects the ES width w (R1)
    precision: "f32" | "f64"
    iflag    : sign of the type-1 exponent (-1 = PAPER.md Eq. 1); type 2 uses -iflag
    L        : period of the point domain [0, L)^3
    comm     : a Comm -> z-slab plan over its ranks (modes are y-slabs: local_modes())
    points_owned : distributed only; 1 = every point given lies in this rank's z-slab
    precompute : ES weights per point stored by setpts (0 auto, 1 always, -1 never)
    spread_warps : spread kernel (include/nufft.h); 3 = tcgen05 tensor-core GEMM (fp32);
                   -1 / -2 = the paper's Atomic Spread
                   in caller / bin-sorted order (ablation only)
    interp_method: 0 tiled (default); 1 / 2 = the paper's Direct Interpolation in
                   caller / bin-sorted order (ablation only)
    fft_method : 0 one (2N)^3 FFT (default); 1 the paper's pruned sigma = 2 split into
                 eight N^3 parity sub-grid FFTs (complex transforms, one GPU)
    """

    def __init__(self, N, eps, precision="f64", iflag=-1, L=2 * math.pi, modeord=0,
                 device=None, stream=None, tile=None, timing=False, spread_warps=0,
                 comm=None, points_owned=False, precompute=0, interp_method=0, fft_method=0):
        if not torch.cuda.is_available():
            raise NufftError("libnufft requires a CUDA device (no CPU fallback)")
        self.N = tuple(int(n) for n in N)
        self.precision = precision
        self.prec = F64 if precision in ("f64", "double", torch.float64) else F32
        self.real = torch.float64 if self.prec == F64 else torch.float32
        self.cplx = torch.complex128 if self.prec == F64 else torch.complex64
        self.device = torch.device(device) if device is not None else torch.device("cuda",
                                                                                   torch.cuda.current_device())
        self._stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        o = Opts()
        lib().nufft_default_opts(ctypes.byref(o))
        o.L = float(L)
        o.modeord = int(modeord)
        o.stream = self._stream.cuda_stream
        o.timing = 1 if timing else 0
        o.spread_warps = int(spread_warps)
        o.precompute = int(precompute)
        o.interp_method = int(interp_method)
        o.fft_method = int(fft_method)
        if comm is not None:
            o.comm = comm._h
            o.points_owned = 1 if points_owned else 0
        self.comm = comm
        if tile is not None:
            for d in range(3):
                o.tile[d] = int(tile[d] if hasattr(tile, "__len__") else tile)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            st = lib().nufft_plan(self.N[0], self.N[1], self.N[2], int(iflag), float(eps), self.prec,
                                  ctypes.byref(o), ctypes.byref(h))
        _check(st, "nufft_plan")
        self.status = st
        self._h = h
        self.Np = None
        lo = (ctypes.c_int64 * 3)()
        hi = (ctypes.c_int64 * 3)()
        _check(lib().nufft_local_modes(h, lo, hi), "nufft_local_modes")
        self.modes_lo, self.modes_hi = tuple(lo), tuple(hi)
        # this rank's mode block, (z, y, x) storage order, x fastest
        self.local_shape = tuple(hi[d] - lo[d] for d in (2, 1, 0))
        # real transforms: the same on one GPU; the k1 = 0 .. N1/2 half on a slab plan
        self.local_shape_real = (self.local_shape if comm is None else
                                 self.local_shape[:2] + (self.N[0] // 2 + 1,))

    def local_modes(self):
        """[lo, hi) storage-index ranges per axis (x, y, z) of this rank's modes."""
        return self.modes_lo, self.modes_hi

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().nufft_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- calls
    @contextlib.contextmanager
    def _call(self, *tensors):
        """One library call on the plan stream, ordered against the caller's stream."""
        with torch.cuda.device(self.device):
            cur = torch.cuda.current_stream(self.device)
            other = cur.cuda_stream != self._stream.cuda_stream
            if other:
                self._stream.wait_stream(cur)
            yield
            if other:
                for t in tensors:
                    if isinstance(t, torch.Tensor) and t.is_cuda:
                        t.record_stream(self._stream)
                cur.wait_stream(self._stream)

    def info(self) -> dict:
        i = Info()
        _check(lib().nufft_get_info(self._h, ctypes.byref(i)), "nufft_get_info")
        return i.as_dict()

    def setpts(self, x: torch.Tensor, y: torch.Tensor, z: torch.Tensor):
        n = x.numel()
        px = _ptr(x, self.real, n, "x")
        py = _ptr(y, self.real, n, "y")
        pz = _ptr(z, self.real, n, "z")
        with self._call(x, y, z):
            _check(lib().nufft_setpts(self._h, n, px, py, pz), "nufft_setpts")
        self.Np = n
        return self

    def _out(self, out, shape, on_host_like=None):
        if out is not None:
            return out
        dev = self.device if on_host_like is None or on_host_like.is_cuda else torch.device("cpu")
        return torch.empty(shape, dtype=self.cplx, device=dev,
                           pin_memory=(dev.type == "cpu" and torch.cuda.is_available()))

    def type1(self, c: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        fk = self._out(out, self.local_shape, c)
        pc = _ptr(c, self.cplx, self.Np, "c")
        pf = _ptr(fk, self.cplx, math.prod(self.local_shape), "fk")
        with self._call(c, fk):
            _check(lib().nufft_execute_type1(self._h, pc, pf), "nufft_execute_type1")
        return fk

    def type2(self, fk: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        c = self._out(out, (self.Np,), fk)
        pf = _ptr(fk, self.cplx, math.prod(self.local_shape), "fk")
        pc = _ptr(c, self.cplx, self.Np, "c")
        with self._call(fk, c):
            _check(lib().nufft_execute_type2(self._h, pf, pc), "nufft_execute_type2")
        return c

    def type1_real(self, c: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Type 1 of REAL strengths (R2C path); returns the complex (Hermitian) modes."""
        fk = self._out(out, self.local_shape_real, c)
        pc = _ptr(c, self.real, self.Np, "c")
        pf = _ptr(fk, self.cplx, math.prod(self.local_shape_real), "fk")
        with self._call(c, fk):
            _check(lib().nufft_execute_type1_real(self._h, pc, pf), "nufft_execute_type1_real")
        return fk

    def type2_real(self, fk: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Real part of type 2 (C2R path); returns Np reals."""
        if out is None:
            dev = self.device if fk.is_cuda else torch.device("cpu")
            out = torch.empty((self.Np,), dtype=self.real, device=dev,
                              pin_memory=(dev.type == "cpu" and torch.cuda.is_available()))
        pf = _ptr(fk, self.cplx, math.prod(self.local_shape_real), "fk")
        pc = _ptr(out, self.real, self.Np, "c")
        with self._call(fk, out):
            _check(lib().nufft_execute_type2_real(self._h, pf, pc), "nufft_execute_type2_real")
        return out

    def type2_real3(self, fk0, fk1, fk2, out: torch.Tensor | None = None) -> torch.Tensor:
        """Three real type-2 transforms at once (one weight evaluation per point);
        returns (Np, 3) reals."""
        if out is None:
            out = torch.empty((self.Np, 3), dtype=self.real, device=self.device)
        n = math.prod(self.local_shape_real)
        ps = [_ptr(f, self.cplx, n, "fk") for f in (fk0, fk1, fk2)]
        pc = _ptr(out, self.real, 3 * self.Np, "c")
        with self._call(fk0, fk1, fk2, out):
            _check(lib().nufft_execute_type2_real3(self._h, *ps, pc), "nufft_execute_type2_real3")
        return out

    def spread(self, c: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        N1, N2, N3 = self.N
        g = self._out(out, (2 * N3, 2 * N2, 2 * N1), c)
        pc = _ptr(c, self.cplx, self.Np, "c")
        pg = _ptr(g, self.cplx, 8 * N1 * N2 * N3, "grid")
        with self._call(c, g):
            _check(lib().nufft_spread(self._h, pc, pg), "nufft_spread")
        return g

    def interp(self, grid: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        N1, N2, N3 = self.N
        c = self._out(out, (self.Np,), grid)
        pg = _ptr(grid, self.cplx, 8 * N1 * N2 * N3, "grid")
        pc = _ptr(c, self.cplx, self.Np, "c")
        with self._call(grid, c):
            _check(lib().nufft_interp(self._h, pg, pc), "nufft_interp")
        return c
