"""The C++ drop-in shim (include/tetvol_b200.hpp) against the unmodified
reference library: tests/cpp/shim_drop_in renders, builds and marches the same
inputs through tetvol:: (CPU) and tetvol::b200:: (GPU) and requires
bit-identical results."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin", "shim_drop_in")


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim test binary not built (needs /root/reference at build time)")
def test_cpp_shim_is_a_drop_in():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim ok" in r.stdout
