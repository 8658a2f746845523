"""Build an experimental libncsg.so with extra -D flags into _variants/<name>/
(git-ignored) for A/B timing: NCSG_LIB=_variants/<name>/libncsg.so python bench.py ...
usage: python scripts/build_variant.py NAME -DNCSG_ORB_WARPS=8 ..."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_13100_b200 import _build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.ROOT, "_variants", name)
os.makedirs(out, exist_ok=True)
B.build()
objs = []
for src in B.CU_SRCS + B.CPP_SRCS:
    o = os.path.join(out, src + ".o")
    if src.endswith(".cu"):
        cmd = [B.NVCC, *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
    else:
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", f"-I{B.CUDA}/include"]
    subprocess.run([*cmd, *defs, "-c", os.path.join(B.CSRC, src), "-o", o], check=True)
    objs.append(o)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(out, "libncsg.so"), *objs,
                "-cudart", "static"], check=True)
print(os.path.join(out, "libncsg.so"))
