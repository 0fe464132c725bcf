"""GPU: the C++ drop-in surface (include/spardl/*.hpp over the C ABI).

tests/cpp/test_dropin.cpp is written against the reference's spardl:: API
(same includes, names, exception classes) and runs the reference's known
answers through the GPU.  Built here with g++ (same image on the GPU box).
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build():
    out = os.path.join(ROOT, "build", "dropin", "test_dropin")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
                    "-L", os.path.join(ROOT, "paper_2304_00737_b200"), "-l:libspardl_cuda.so",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2304_00737_b200"), "-o", out],
                   check=True)
    return out


def test_cpp_dropin(built):
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:], r.stderr[-2000:])
    assert r.returncode == 0
    assert "0 failed" in r.stdout
