"""CPU-side checks of the C ABI library: it builds for sm_100a, loads, and exports
every entry point include/nufft.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nufft.h")


@pytest.fixture(scope="module")
def libpath():
    from paper_2605_10678_b200 import build
    return build.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nufft_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("nufft_plan", "nufft_setpts", "nufft_execute_type1", "nufft_execute_type2",
              "nufft_destroy"):
        assert f in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (nufft_[a-z0-9_]+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out


def test_load_and_host_only_calls(libpath):
    import paper_2605_10678_b200 as nb
    L = nb.lib()
    for f in declared_functions():
        assert hasattr(L, f)
    o = nb.Opts()
    assert L.nufft_default_opts(ctypes.byref(o)) == 0
    assert abs(o.L - 2 * 3.141592653589793) < 1e-15 and o.modeord == 0 and not o.comm
    assert L.nufft_strerror(0) == b"ok"
    assert b"points not set" in L.nufft_strerror(5)
    assert L.nufft_default_opts(None) == 2
    # null handles are rejected without touching the device
    assert L.nufft_setpts(None, 0, None, None, None) == 2
    assert L.nufft_execute_type1(None, None, None) == 2
    assert L.nufft_destroy(None) == 0
    h = ctypes.c_void_p()
    assert L.nufft_plan(16, 16, 16, -1, 1e-6, 7, None, ctypes.byref(h)) == 2  # bad precision


def test_python_binding_refuses_without_cuda():
    import torch
    import paper_2605_10678_b200 as nb
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(nb.NufftError):
        nb.Plan((16, 16, 16), 1e-6)


def test_product_path_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2605_10678_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "nufft_oracle" not in txt, f
