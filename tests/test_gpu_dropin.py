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


REF_BIN = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("name", ["sparse", "fabric", "collectives"])
def test_reference_unit_tests_unmodified(built, name):
    """The reference's own unit tests (/root/reference/proj/tests/test_*.cpp,
    unmodified) compiled against include/spardl with the GoogleTest
    stand-in (tests/cpp/gtest_shim) by oracle/Makefile, run on the B200:
    every case passes (17 + 9 + 16 = 42)."""
    exe = os.path.join(REF_BIN, f"ref_test_{name}")
    if not os.path.exists(exe):
        pytest.skip("reference unit tests not built (no /root/reference where built)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0
    expect = {"sparse": 17, "fabric": 9, "collectives": 16}[name]
    assert f"{expect} passed, 0 failed" in r.stdout
