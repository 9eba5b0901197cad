"""Host logic of the link / star tile planners (csrc/linkwalk.cuh) on the CPU.

The planners of the edge-link tiles (C4), the fused Taylor-Hood launch (C5)
and the link-walk tiles (C3 matrix) order the cells around a mesh edge or
vertex into one ring or fan and decline anything else; tests/cpp/test_linkwalk.cpp
checks that walk and the window-run builder without a GPU.
"""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_link_walk_and_window_runs():
    d = os.path.join(ROOT, "tests", "cpp")
    subprocess.run(["make", "-s", "-C", d, "bin/test_linkwalk"], check=True)
    r = subprocess.run([os.path.join(d, "bin", "test_linkwalk")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
