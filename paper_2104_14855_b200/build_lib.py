"""Build libmhdp.so in-tree for sm_100a (nvcc; the host setup with g++ -O3 -fopenmp).

The library is the product: CUDA kernels (csrc/kernels.cu), the C-ABI and drivers
(csrc/api.cu) and the host FE setup (csrc/fe_setup.cpp).  Built objects go to
build/ and the shared library to paper_2104_14855_b200/libmhdp.so (git-ignored, but
shipped to the GPU box by gpurun).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libmhdp.so")
PROBE = os.path.join(ROOT, "tools", "libprobe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU = ["kernels.cu", "k2_small.cu", "k6_patch_lu.cu", "k7_dense_lu.cu", "k8_coarse.cu", "api.cu"]
CPP = ["fe_setup.cpp"]
HEADERS = ["kernels.cuh", "k2_common.cuh", "setup.hpp"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "mhdp.h")]
    jobs = []
    objs = []
    for f in CU:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fopenmp",
                         "-Xptxas", "-warn-spills", "-c", src, "-o", obj])
    for f in CPP:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append(["g++", "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=4) as ex:
        for err in ex.map(run, jobs):
            if verbose and err:
                print(err, file=sys.stderr)
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fopenmp", "-lgomp"])
        os.replace(tmp, LIB)
    # measurement probes (FP64 peak, dependency latencies): tools/libprobe.so
    psrc = os.path.join(ROOT, "tools", "probe.cu")
    if os.path.exists(psrc) and (force or _stale(PROBE, [psrc, os.path.join(CSRC, "k2_common.cuh")])):
        tmp = PROBE + ".tmp"
        run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", psrc, "-o", tmp])
        os.replace(tmp, PROBE)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
