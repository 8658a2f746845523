"""In-tree build of libncsg.so (sm_100a) -- used by __graft_entry__.build(),
the tests' conftest and bench.py.  No JIT cache: the .so lands next to this
file so it travels with the repo snapshot to the GPU box."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libncsg.so")
OBJ = os.path.join(HERE, "_obj")
ROOT = os.path.dirname(HERE)
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SRCS = ["radon_kernels.cu", "fft_kernels.cu", "ncs_kernels.cu", "sparse_kernels.cu", "capi.cu"]
CPP_SRCS = ["geometry.cpp", "fanbeam.cpp", "comm.cpp"]
HDRS = ["ncsg_internal.cuh", "ncs_kernels.cuh", "ncs_device.cuh", "ncsg_comm.hpp"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HDRS] + [os.path.join(ROOT, "include", "ncsg.h")]
    objs = []
    for src in CU_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-warn-spills", "-c", s, "-o", o], verbose)
    for src in CPP_SRCS:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + hdrs):
            _run(["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off",
                  f"-I{CUDA}/include", "-c", s, "-o", o], verbose)
    if force or _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static"], verbose)
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
