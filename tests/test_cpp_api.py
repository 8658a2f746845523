"""The C++ mirror of the reference API (include/ncstomo_gpu.hpp) compiles and
links against libncsg.so (CPU), and its doctest-style cases pass on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_gpu_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_1810_13100_b200")


def _build(tmp_path):
    from paper_1810_13100_b200 import _build as b

    b.build()
    exe = os.path.join(str(tmp_path), "test_gpu_api")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", SRC, f"-L{LIBDIR}",
                    "-lncsg", f"-Wl,-rpath,{LIBDIR}", "-pthread", "-o", exe], check=True)
    return exe


def test_cpp_api_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_cases_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
