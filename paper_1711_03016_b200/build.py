"""Builds the in-tree native library `libdlvm.so` (C++17 front end + sm_100a
CUDA kernels) with nvcc.  `python -m paper_1711_03016_b200.build` or
`__graft_entry__.build()`.  Object files are rebuilt when a source or header
is newer; the .so travels with the repo snapshot to the GPU box."""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# DLVM_BUILD_VARIANT=trace: a separate libdlvm_trace.so with -DDLVM_GEMM_TRACE
# (GEMM phase stamps, tools/gemm_trace.py); the product library is unchanged
VARIANT = os.environ.get("DLVM_BUILD_VARIANT", "")
OUT = os.path.join(PKG, "libdlvm.so" if not VARIANT else f"libdlvm_{VARIANT}.so")
OBJ = os.path.join(PKG, "build" if not VARIANT else f"build_{VARIANT}")
VARIANT_FLAGS = {"": [], "trace": ["-DDLVM_GEMM_TRACE"], "s4": ["-DDLVM_GEMM_STAGES_PAIR=4"],
                 "s5": ["-DDLVM_GEMM_STAGES_PAIR=5"], "rpi4": ["-DDLVM_EW_RPI=4"],
                 "probe": ["-DDLVM_PROBE_SKIP_B"]}[VARIANT]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", CSRC, "-I", os.path.join(ROOT, "include")] + VARIANT_FLAGS


def sources():
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    cu = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")))
    return cpp, cu


def headers():
    return (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "kernels", "*.h"))
            + glob.glob(os.path.join(CSRC, "kernels", "*.cuh")) + glob.glob(os.path.join(CSRC, "kernels", "*.inc")) + [os.path.join(ROOT, "include", "dlvm.h")])


def _compile(src: str, is_cu: bool, newest_header: float) -> str:
    obj = os.path.join(OBJ, os.path.relpath(src, CSRC).replace(os.sep, "_") + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), newest_header):
        return obj
    if is_cu:
        cmd = [NVCC] + COMMON + ["-c", src, "-o", obj] + ARCH + ["-lineinfo"]
        if os.environ.get("DLVM_PTXAS_V"):
            cmd += ["-Xptxas", "-v"]
    else:  # host-only C++ (front end, planner, C ABI)
        cmd = [CXX, "-O2", "-std=c++17", "-fPIC", "-Wall", "-Wno-unused-function"] + VARIANT_FLAGS + ["-I", CSRC,
               "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and os.environ.get("DLVM_BUILD_VERBOSE"):
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    cpp, cu = sources()
    newest = max(os.path.getmtime(h) for h in headers() if os.path.exists(h))
    jobs = [(s, False) for s in cpp] + [(s, True) for s in cu]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda a: _compile(a[0], a[1], newest), jobs))
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(o) for o in objs):
        return OUT
    cmd = [NVCC, "-shared", "-o", OUT] + objs + ARCH + ["-cudart", "static", "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print("built", OUT)
    return OUT


if __name__ == "__main__":
    build(verbose=True)
