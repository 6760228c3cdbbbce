"""The reference-shaped C++ adapter (include/bfsim_gpu.hpp) on the GPU against
the unmodified reference in the same binary (tests/cpp/wrapper_test.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin", "wrapper_test")


def test_cpp_adapter_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("wrapper_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
