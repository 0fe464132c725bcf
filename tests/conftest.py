import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libspardl_cuda.so)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def built():
    """Build the checkers (and the CUDA library if absent) once per session."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib = os.path.join(ROOT, "paper_2304_00737_b200", "libspardl_cuda.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-j8", "-C",
                        os.path.join(ROOT, "paper_2304_00737_b200", "csrc")], check=True)
    return True
