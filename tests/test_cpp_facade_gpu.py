"""GPU: the reference's own par_loop tests restated in C++ through the drop-in
facade (tests/cpp/test_facade.cpp, csrc/loam_gpu.hpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_facade_suite(gpu_lib):
    cpp = os.path.join(HERE, "cpp")
    subprocess.run(["make", "-s", "-C", cpp], check=True)
    r = subprocess.run([os.path.join(cpp, "bin", "test_facade")], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
