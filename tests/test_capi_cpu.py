"""CPU: the C-ABI library (no compute without a GPU).

* libloam_gpu.so loads and exports every symbol include/loam_gpu.h declares;
* the kernel registry declares the reference's staged shapes
  (parloop.hpp:63-70 staged_extents; form.hpp:229-238 params);
* compute entry points refuse to run without an sm_100 device (no CPU
  fallback) -- checked only where no device is present;
* the host-side input generator reproduces the reference meshes bit-exactly
  (golden fixtures from oracle/_ref) and is deterministic;
* the product P2 numbering equals the oracle's restatement.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "loam_gpu.h")).read()
    return sorted(set(re.findall(r"\b(loam_gpu_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    declared = header_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(L, name), f"{name} declared in loam_gpu.h but not exported"
    assert sorted(capi.EXPORTED) == declared


def test_error_kinds_follow_the_reference_enum():
    txt = open(os.path.join(ROOT, "include", "loam_gpu.h")).read()
    kinds = re.findall(r"LOAM_KIND_(\w+)", txt.split("enum loam_error_kind")[1].split("};")[0])
    assert kinds == capi.ERROR_KINDS  # common.hpp:10-33, same order


@pytest.mark.parametrize("name,ext", [
    ("stiffness_p1_tri", [[3, 3], [3, 2]]),
    ("mass_p2_tri", [[6, 6], [3, 2]]),
    ("helmholtz_p1_tet", [[4, 4], [4, 3]]),
    ("helmholtz_p2_tet", [[10, 10], [4, 3]]),
    ("helmholtz_action_p1_tri", [[3], [3, 2], [3]]),
    ("helmholtz_action_p2_tet", [[10], [4, 3], [10]]),
    ("stiffness_action_p2_tri", [[6], [3, 2], [6]]),
    ("elasticity_p1_tet", [[12, 12], [4, 3]]),
    ("stokes_a_p2_tri", [[12, 12], [3, 2]]),
    ("stokes_b_p2_tri", [[3, 12], [3, 2]]),
    ("stokes_bt_p2_tri", [[12, 3], [3, 2]]),
    ("ones_block", [[3, 3]]),
    ("weighted_scatter", [[3], [1]]),
    ("iincv", [[3, 2], [1]]),
    ("gmm", [[1], [1], [1]]),
])
def test_registry_staged_shapes(name, ext):
    buf = (C.c_int32 * 64)()
    n = capi.lib().loam_gpu_kernel_signature(name.encode(), buf, 64)
    assert n == len(ext)
    out, w = [], 0
    for _ in range(n):
        r = buf[w]
        out.append(list(buf[w + 1:w + 1 + r]))
        w += 1 + r
    assert out == ext


def test_reference_test_kernels_are_opt_in():
    """add_one & co. (the reference test suite's kernels) are not product
    kernels: visible only with LOAM_OPT_TEST_KERNELS (conftest sets it)."""
    L = capi.lib()
    buf = (C.c_int32 * 8)()
    try:
        capi.set_option(capi.OPT_TEST_KERNELS, 0)
        assert L.loam_gpu_kernel_signature(b"add_one", buf, 8) < 0
        assert b"add_one" not in L.loam_gpu_kernel_names()
        assert L.loam_gpu_kernel_signature(b"stiffness_p1_tri", buf, 8) == 2
    finally:
        capi.set_option(capi.OPT_TEST_KERNELS, 1)
    assert L.loam_gpu_kernel_signature(b"add_one", buf, 8) == 1


def test_unregistered_kernel_signature_is_an_error():
    buf = (C.c_int32 * 8)()
    n = capi.lib().loam_gpu_kernel_signature(b"no_such_kernel", buf, 8)
    assert n == -capi.ERROR_KINDS.index("InvalidArgument") - 1


@pytest.mark.skipif(capi.lib().loam_gpu_device_ok() == 1, reason="a device is present")
def test_no_cpu_fallback_without_a_device():
    L = capi.lib()
    kd = capi.KernelDesc(b"stiffness_p1_tri", None, 0)
    rc = L.loam_gpu_execute(C.byref(kd), 0, 0, None, 0, None)
    assert rc == capi.ERR_NO_DEVICE
    assert b"no CPU fallback" in L.loam_gpu_last_error()
    md = capi.MapDesc()
    assert L.loam_gpu_map_check(C.byref(md), None) == capi.ERR_NO_DEVICE


def test_validate_runs_on_the_host():
    """loam_gpu_validate (parloop.hpp:89-146) needs no device: descriptor checks only."""
    L = capi.lib()
    md = capi.MapDesc()
    md.source_size, md.target_size, md.arity, md.source_id, md.target_id, md.id = 2, 4, 3, 1, 2, 3
    sp = capi.SparsityDesc()
    sp.nrows = sp.ncols = 4
    a = (capi.ArgDesc * 1)()
    a[0].kind, a[0].access = capi.ARG_MAT, capi.READ
    a[0].map = a[0].col_map = C.pointer(md)
    a[0].sparsity = C.pointer(sp)
    kd = capi.KernelDesc(b"ones_block", None, 0)
    rc = L.loam_gpu_validate(C.byref(kd), 2, 1, a, 1)
    assert rc == 1 + capi.ERROR_KINDS.index("IllegalAccess")
    assert b"write-only" in L.loam_gpu_last_error()
    a[0].access = capi.INC
    assert L.loam_gpu_validate(C.byref(kd), 2, 1, a, 1) == 0
    assert L.loam_gpu_validate(C.byref(kd), 5, 9, a, 1) == 1 + capi.ERROR_KINDS.index("MapSourceMismatch")


def test_generator_reproduces_reference_meshes():
    g = np.load(os.path.join(ROOT, "tests", "golden", "ref_meshes.npz"))
    sq = configs.mesh(2, 6)
    assert np.array_equal(sq.coords, g["sq_coords"]) and np.array_equal(sq.cv, g["sq_cv"])
    cu = configs.mesh(3, 3)
    assert np.array_equal(cu.coords, g["cube_coords"]) and np.array_equal(cu.cv, g["cube_cv"])


def test_generator_is_deterministic_and_seeded():
    a, b = configs.config_inputs(1, 20), configs.config_inputs(1, 20)
    assert np.array_equal(a.coords, b.coords) and np.array_equal(a.cv, b.cv) and np.array_equal(a.extra["u"], b.extra["u"])
    base = configs.mesh(2, 20)
    # jitter moves interior vertices only, by at most amp*h per coordinate
    d = (a.coords - base.coords).reshape(-1, 2)
    n = 20
    ij = np.array([(v % (n + 1), v // (n + 1)) for v in range(a.nv)])
    boundary = (ij == 0).any(1) | (ij == n).any(1)
    assert np.all(d[boundary] == 0) and np.all(np.abs(d) <= 0.2 / n)
    # permutation moves cell rows only, as a bijection
    assert sorted(map(tuple, a.cv.reshape(-1, 3))) == sorted(map(tuple, base.cv.reshape(-1, 3)))
    assert not np.array_equal(a.cv, base.cv)
    assert np.all((a.extra["u"] >= 0) & (a.extra["u"] < 1))


def test_generator_reproduces_golden_config_inputs():
    for name, cfg, n in (("c1_n8.npz", 1, 8), ("c2_n8.npz", 2, 8), ("p2tri_n4.npz", 5, 4), ("p1tet_n3.npz", 4, 3)):
        g = np.load(os.path.join(ROOT, "tests", "golden", name))
        m = configs.config_inputs(cfg, n)
        assert np.array_equal(m.cv, g["cv"]) and np.array_equal(m.coords, g["coords"])


@pytest.mark.parametrize("gd,n", [(2, 7), (3, 3)])
def test_product_p2_numbering_equals_oracle(gd, n):
    m = configs.mesh(gd, n, 0.1, 1, 2)
    cn, nn = configs.p2_map(m)
    ocn, onn = O.p2_cell_node_map(m.cv, m.nv, gd)
    assert nn == onn and np.array_equal(cn, ocn)


def test_config_sizes_match_baseline():
    """Sizes BASELINE.json states (checked on the generator, full size, cheap ones)."""
    m = configs.config_inputs(1)
    assert m.ncells == 524_288 and m.nv == 263_169
    m = configs.mesh(3, 64)
    assert m.ncells == 1_572_864
    cn, nn = configs.p2_map(m)
    assert nn == 2_146_689
