"""Build libnufft.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2605_10678_b200.build [--force] [-j N]

Every CUDA translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo``; the host orchestration
(plan.cpp) with the same nvcc driver; the result is linked with cuFFT into
``paper_2605_10678_b200/libnufft.so`` next to this file.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
# NUFFT_DEBUG_BOUNDS=1: a separate bounds-checked build (device asserts on every
# shared-memory / grid index of the hot kernels, NUFFT_CHECK in device_util.cuh) into
# libnufft_debug.so -- the substitute for compute-sanitizer, which is closed on the
# GPU pool; select it at run time with NUFFT_LIB=.../libnufft_debug.so
DEBUG = os.environ.get("NUFFT_DEBUG_BOUNDS") == "1"
BUILD = os.path.join(HERE, "_build_debug" if DEBUG else "_build")
LIB = os.path.join(HERE, "libnufft_debug.so" if DEBUG else "libnufft.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]
CU_FLAGS = ARCH + COMMON + ["--expt-relaxed-constexpr", "-Xptxas", "-v"]
# developer instrumentation only (e.g. -DNUFFT_OUTER_PROF); never set for the product build
CU_FLAGS += os.environ.get("NUFFT_EXTRA_NVCC_FLAGS", "").split()
if DEBUG:
    CU_FLAGS += ["-DNUFFT_DEBUG_BOUNDS"]

SOURCES = ["sort.cu", "xport.cpp", "spread.cu", "spread_rows.cu", "spread_outer.cu", "spread_sub.cu", "interp.cu", "interp_real.cu", "interp_vec3.cu",
           "elementwise.cu", "pif.cu", "variants.cu", "spread_tc.cu", "pruned.cu", "dist_kernels.cu", "peak.cu", "plan.cpp", "dist.cpp"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch's NCCL wheel (2.28.x)
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return None, None


def _includes(path):
    """Local headers #include-d by `path` (quoted includes resolved in csrc/ or include/)."""
    out = []
    try:
        with open(path) as f:
            for line in f:
                line = line.strip()
                if line.startswith("#include \""):
                    name = line.split('"')[1]
                    for d in (os.path.dirname(path), CSRC, os.path.join(ROOT, "include")):
                        cand = os.path.normpath(os.path.join(d, name))
                        if os.path.exists(cand):
                            out.append(cand)
                            break
    except OSError:
        pass
    return out


def _deps(src):
    """The source and every local header it includes, transitively."""
    seen, todo = [], [os.path.join(CSRC, src)]
    while todo:
        f = todo.pop()
        if f in seen:
            continue
        seen.append(f)
        todo.extend(_includes(f))
    return seen


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src, force, log):
    obj = os.path.join(BUILD, src + ".o")
    if not force and not _stale(obj, _deps(src)):
        return obj, ""
    flags = list(CU_FLAGS) if src.endswith(".cu") else ARCH + COMMON
    inc, _ = _nccl_dirs()
    if inc is None:
        raise RuntimeError("nccl.h not found (expected torch's nvidia-nccl wheel)")
    flags += ["-I", inc]
    cmd = [NVCC] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    out = r.stdout + r.stderr
    if log:
        with open(os.path.join(BUILD, src + ".ptxas.txt"), "w") as f:
            f.write(out)
    return obj, out


def build(force: bool = False, jobs: int = 8, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        futs = {ex.submit(_compile, s, force, True): s for s in SOURCES}
        objs = {}
        for f in cf.as_completed(futs):
            obj, out = f.result()
            objs[futs[f]] = obj
            if verbose and out:
                print(out)
    objs = [objs[s] for s in SOURCES]
    if force or _stale(LIB, objs):
        _, ncl = _nccl_dirs()
        # NCCL: torch's libnccl.so.2 (2.28), resolved through rpath at load time
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + \
            ["-lcufft", "-L", ncl, "-l:libnccl.so.2",
             "-Xlinker", "-rpath," + os.path.join(CUDA, "lib64"), "-Xlinker", "-rpath," + ncl]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.j, a.v))


if __name__ == "__main__":
    sys.exit(main())
