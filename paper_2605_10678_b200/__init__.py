"""B200-native (sm_100a) hot path of the distributed 3D NUFFT of arXiv 2605.10678.

The product is ``libnufft.so`` (C ABI in ``include/nufft.h``); this package is
its thin Python binding (``nufft.py``) and its in-tree build (``build.py``).
"""
from .nufft import F32, F64, Comm, Info, NufftError, Opts, Plan, fma_peak, lib, LIB_PATH  # noqa: F401

__all__ = ["Plan", "Comm", "fma_peak", "NufftError", "lib", "LIB_PATH", "F32", "F64"]
