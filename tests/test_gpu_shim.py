"""GPU: the C++ drop-in header (include/tilemul_gpu.hpp) passes the
reference-style acceptance gates (tests/cpp/shim_acceptance.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_shim_acceptance():
    exe = os.path.join(ROOT, "tests", "cpp", "shim_acceptance")
    if not os.path.exists(exe):
        import __graft_entry__
        __graft_entry__.build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") >= 9
