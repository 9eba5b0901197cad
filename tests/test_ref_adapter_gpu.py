"""GPU: the reference's OWN objects and fem:: callers routed to the B200
through include/loam_gpu_ref.hpp (loam::Parloop -> loam_gpu_execute_host,
fem::assemble_matrix / assemble_vector / assemble_blocks), compared with the
reference's own CPU execution of the same calls (tests/cpp/test_ref_adapter.cpp).

The binary needs the reference headers, so it is built in the container by
__graft_entry__.build() and shipped with the snapshot (tests/cpp/bin)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "bin", "test_ref_adapter")


def test_reference_objects_through_the_adapter(gpu_lib):
    if os.path.exists("/root/reference/proj/include/loam/loam.hpp"):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp"), "bin/test_ref_adapter"], check=True)
    assert os.path.exists(BIN), "tests/cpp/bin/test_ref_adapter was not built (run __graft_entry__.build())"
    r = subprocess.run([BIN, "96", "10"], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout
