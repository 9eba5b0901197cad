"""par_loop semantics on the device, mirroring the reference's own tests.

Each test restates a case of /root/reference/proj/tests/test_parloop.cpp (or
acceptance.cpp criterion 3) through the loam mirror, so the device engine is
held to the same known answers: direct loops, indirect INC, Mat INC, validate
errors without mutation, READ version counters, WRITE independence, staging
canary, Global reductions, permutation licence, RW conflict-free updates.
"""
import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi
from paper_1501_01809_b200 import loam as L
from paper_1501_01809_b200.capi import LoamError

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset(gpu_lib):
    yield
    capi.set_strategy("auto")


def two_triangles():  # test_parloop.cpp:13-17
    cells, verts = L.Set(2, "cells"), L.Set(4, "vertices")
    return cells, verts, L.Map(cells, verts, 3, [0, 1, 2, 1, 3, 2], "cell_vertex")


def test_direct_loop_doubles_a_field():  # :46-59
    s = L.Set(3)
    a, b = L.Dat(s, 1, "a"), L.Dat(s, 1, "b")
    b.set_values([1, 2, 3])
    L.execute(L.Parloop(L.kernel("double_direct"), s, [L.arg(a, L.WRITE), L.arg(b, L.READ)]))
    assert list(a.view()) == [2, 4, 6]


@pytest.mark.parametrize("strat", ["auto", "atomic", "color"])
def test_indirect_inc_accumulates_cell_incidence(strat):  # :61-68
    capi.set_strategy(strat)
    cells, verts, m = two_triangles()
    v = L.Dat(verts, 1, "v")
    L.execute(L.Parloop(L.kernel("add_one"), cells, [L.arg(v, L.INC, m)]))
    assert list(v.view()) == [1, 2, 2, 1]


@pytest.mark.parametrize("strat", ["auto", "atomic", "color"])
def test_mat_inc_assembles_both_triangles(strat):  # :70-87
    capi.set_strategy(strat)
    cells, verts, m = two_triangles()
    mat = L.Mat(L.build_sparsity(m, m))
    L.execute(L.Parloop(L.kernel("ones_block"), cells, [L.arg(mat, L.INC, m, m)]))
    assert mat.at(1, 1) == 2.0 and mat.at(2, 2) == 2.0 and mat.at(0, 0) == 1.0 and mat.at(3, 3) == 1.0
    dense = np.zeros((4, 4))
    for e in range(2):
        for i in m.row(e):
            for j in m.row(e):
                dense[i, j] += 1.0
    for r in range(4):
        for c in range(4):
            assert mat.at(r, c) == dense[r, c]


def test_validate_rejects_illegal_descriptors_and_leaves_state_alone():  # :89-149
    cells, verts, m = two_triangles()
    mat = L.Mat(L.build_sparsity(m, m))
    with pytest.raises(LoamError) as e:
        L.validate(L.Parloop(L.kernel("ones_block"), cells, [L.arg(mat, L.READ, m, m)]))
    assert e.value.kind == "IllegalAccess" and "write-only" in str(e.value)
    g = L.Global(1)
    with pytest.raises(LoamError) as e:
        L.validate(L.Parloop(L.kernel("sum"), cells, [L.arg(g, L.INC), L.arg(L.Dat(cells, 1), L.READ)]))
    assert e.value.kind == "IllegalAccess"
    v = L.Dat(verts, 1, "v")
    version = v.version
    L.validate(L.Parloop(L.kernel("add_one"), cells, [L.arg(v, L.INC, m)]))
    assert v.version == version
    other = L.Set(5)
    with pytest.raises(LoamError) as e:
        L.validate(L.Parloop(L.kernel("add_one"), other, [L.arg(v, L.INC, m)]))
    assert e.value.kind == "MapSourceMismatch"
    edge_map = L.Map(cells, verts, 2, [0, 1, 1, 3])
    with pytest.raises(LoamError) as e:
        L.validate(L.Parloop(L.kernel("add_one"), cells, [L.arg(v, L.INC, edge_map)]))
    assert e.value.kind == "ShapeMismatch"
    with pytest.raises(LoamError) as e:
        L.validate(L.Parloop(L.kernel("double_direct"), verts, [L.arg(v, L.WRITE), L.arg(v, L.READ)]))
    assert e.value.kind == "IllegalAccess"
    # execute validates before any mutation (parloop.hpp:193)
    before = v.view().copy()
    with pytest.raises(LoamError):
        L.execute(L.Parloop(L.kernel("add_one"), cells, [L.arg(v, L.INC, edge_map)]))
    assert np.array_equal(v.view(), before)


def test_unregistered_kernel_is_an_error_not_a_fallback():
    cells, verts, m = two_triangles()
    v = L.Dat(verts, 1)
    with pytest.raises(LoamError) as e:
        L.execute(L.Parloop(L.kernel("no_such_kernel"), cells, [L.arg(v, L.INC, m)]))
    assert e.value.kind == "InvalidArgument" and "no CPU fallback" in str(e.value)


def test_read_arguments_keep_their_version_counter():  # :151-160
    s = L.Set(3)
    a, b = L.Dat(s, 1), L.Dat(s, 1)
    version = b.version
    L.execute(L.Parloop(L.kernel("double_direct"), s, [L.arg(a, L.WRITE), L.arg(b, L.READ)]))
    assert b.version == version and a.version > 0


def test_write_results_do_not_depend_on_previous_target_values():  # :162-180
    s = L.Set(4)
    b = L.Dat(s, 1)
    b.set_values([1, 2, 3, 4])

    def run_from(fill):
        a = L.Dat(s, 1)
        a.set_values([fill] * 4)
        L.execute(L.Parloop(L.kernel("double_direct"), s, [L.arg(a, L.WRITE), L.arg(b, L.READ)]))
        return a.view()

    assert np.array_equal(run_from(0.0), run_from(123.456))


def test_kernels_observe_only_staged_slots():  # :182-200
    cells, verts = L.Set(2), L.Set(5)
    m = L.Map(cells, verts, 2, [0, 1, 2, 3])
    v = L.Dat(verts, 1)
    v.set_values([0, 0, 0, 0, -777.0])
    L.execute(L.Parloop(L.kernel("fill"), cells, [L.arg(v, L.WRITE, m)]))
    out = v.view()
    assert out[4] == -777.0 and out[0] == 1.0


def test_global_reductions_match_host_scans():  # :202-237
    s = L.Set(100)
    field = L.Dat(s, 1)
    x = np.random.default_rng(13).uniform(-10, 10, 100)
    field.set_values(x)
    g = L.Global(1)
    L.execute(L.Parloop(L.kernel("sum"), s, [L.arg(g, L.SUM), L.arg(field, L.READ)]))
    assert abs(g.view()[0] - x.sum()) <= 1e-12 * np.abs(x).sum()
    gmax, gmin = L.Global(1), L.Global(1)
    L.execute(L.Parloop(L.kernel("maxval"), s, [L.arg(gmax, L.MAX), L.arg(field, L.READ)]))
    L.execute(L.Parloop(L.kernel("maxval"), s, [L.arg(gmin, L.MIN), L.arg(field, L.READ)]))
    assert gmax.view()[0] == x.max() and gmin.view()[0] == x.min()


def random_mesh(ncells, nverts, seed):  # test_parloop.cpp:242-259 (numpy generator)
    rng = np.random.default_rng(seed)
    cells, verts = L.Set(ncells), L.Set(nverts)
    table = rng.integers(0, nverts, size=3 * ncells).astype(np.int32)
    return cells, verts, L.Map(cells, verts, 3, table), table


def test_colour_strategy_reproduces_the_reference_threaded_order_bitwise():  # :273-315
    """Under colouring each target receives its contributions colour by colour,
    which is exactly the reference's (colour, entity) accumulation order, so the
    device result equals the reference's (any thread count) bit for bit."""
    cells, verts, m, table = random_mesh(400, 97, 17)
    coeff = L.Dat(cells, 1)
    c = np.random.default_rng(18).uniform(-1, 1, 400)
    coeff.set_values(c)
    capi.set_strategy("color")
    v = L.Dat(verts, 1)
    L.execute(L.Parloop(L.kernel("weighted_scatter"), cells, [L.arg(v, L.INC, m), L.arg(coeff, L.READ)]))
    colors, nc = O.color_iteration(400, [table], [3], [97])
    expect = np.zeros(97)
    for col in range(nc):
        for e in np.nonzero(colors == col)[0]:
            for i in range(3):
                expect[table[3 * e + i]] += (i + 1.0) * c[e]
    assert np.array_equal(v.view(), expect)
    # atomics agree within the permutation licence (:317-355)
    capi.set_strategy("atomic")
    w = L.Dat(verts, 1)
    L.execute(L.Parloop(L.kernel("weighted_scatter"), cells, [L.arg(w, L.INC, m), L.arg(coeff, L.READ)]))
    assert np.all(np.abs(w.view() - expect) <= 1e-12 * np.maximum(1.0, np.abs(expect)))


def test_permuted_iteration_order_stays_within_tolerance():  # :317-355
    cells, verts, m, table = random_mesh(200, 61, 23)
    c = np.random.default_rng(24).uniform(-1, 1, 200)
    order = np.random.default_rng(25).permutation(200)

    def run(perm):
        cs = L.Set(200)
        mm = L.Map(cs, verts, 3, table.reshape(200, 3)[perm].reshape(-1))
        cd = L.Dat(cs, 1)
        cd.set_values(c[perm])
        v = L.Dat(verts, 1)
        L.execute(L.Parloop(L.kernel("weighted_scatter"), cs, [L.arg(v, L.INC, mm), L.arg(cd, L.READ)]))
        return v.view()

    a, b = run(np.arange(200)), run(order)
    assert np.all(np.abs(a - b) <= 1e-12 * np.maximum(1.0, np.abs(a)))


def test_rw_indirect_updates_run_conflict_free():  # :357-373
    cells, verts, m = two_triangles()
    v = L.Dat(verts, 1)
    v.set_values([1, 1, 1, 1])
    L.execute(L.Parloop(L.kernel("bump"), cells, [L.arg(v, L.RW, m)]), 4)
    assert list(v.view()) == [2, 3, 3, 2]


def test_acceptance_criterion3_loops_agree_with_numpy():  # acceptance.cpp:102-256
    from paper_1501_01809_b200 import configs
    mesh = configs.mesh(2, 16)
    cells, verts = L.Set(mesh.ncells), L.Set(mesh.nv)
    cv = L.Map(cells, verts, 3, mesh.cv)
    rng = np.random.default_rng(901)
    cf, vf = rng.uniform(-1, 1, mesh.ncells), rng.uniform(-1, 1, mesh.nv)
    cell_field, vertex_field = L.Dat(cells, 1), L.Dat(verts, 1)
    cell_field.set_values(cf)
    vertex_field.set_values(vf)
    t = mesh.cv.reshape(-1, 3)

    out = L.Dat(cells, 1)
    L.execute(L.Parloop(L.kernel("dw"), cells, [L.arg(out, L.WRITE), L.arg(cell_field, L.READ)]))
    assert np.array_equal(out.view(), 3.0 * cf)
    out = L.Dat(cells, 1)
    out.set_values(np.ones(mesh.ncells))
    L.execute(L.Parloop(L.kernel("drw"), cells, [L.arg(out, L.RW), L.arg(cell_field, L.READ)]))
    assert np.array_equal(out.view(), 1.0 + 0.5 * cf)
    out = L.Dat(cells, 1)
    L.execute(L.Parloop(L.kernel("dinc"), cells, [L.arg(out, L.INC), L.arg(cell_field, L.READ)]))
    assert np.array_equal(out.view(), cf * cf)
    out = L.Dat(cells, 1)
    L.execute(L.Parloop(L.kernel("gw"), cells, [L.arg(out, L.WRITE), L.arg(vertex_field, L.READ, cv)]))
    assert np.array_equal(out.view(), vf[t[:, 0]] + vf[t[:, 1]] + vf[t[:, 2]])
    out = L.Dat(verts, 2)
    L.execute(L.Parloop(L.kernel("iincv"), cells, [L.arg(out, L.INC, cv), L.arg(cell_field, L.READ)]))
    exp = np.zeros((mesh.nv, 2))
    for e in range(mesh.ncells):
        for i in range(3):
            exp[t[e, i]] += [cf[e], 2 * cf[e]]
    assert np.allclose(out.view().reshape(-1, 2), exp, rtol=0, atol=1e-12)
    g, scale = L.Global(1), L.Global(init=[1.25])
    L.execute(L.Parloop(L.kernel("gsum"), cells, [L.arg(g, L.SUM), L.arg(cell_field, L.READ), L.arg(scale, L.READ)]))
    assert abs(g.view()[0] - (1.25 * cf).sum()) <= 1e-12 * np.abs(cf).sum() * 1.25
    lo, hi = L.Global(1), L.Global(1)
    L.execute(L.Parloop(L.kernel("gmm"), cells, [L.arg(lo, L.MIN), L.arg(hi, L.MAX), L.arg(cell_field, L.READ)]))
    assert lo.view()[0] == cf.min() and hi.view()[0] == cf.max()


def test_empty_iteration_set_leaves_dats_and_sets_global_identity():
    s = L.Set(0)
    g = L.Global(1)
    g.set_values([5.0])
    L.execute(L.Parloop(L.kernel("sum"), s, [L.arg(g, L.SUM), L.arg(L.Dat(s, 1), L.READ)]))
    assert g.view()[0] == 0.0  # reduction identity written back (parloop.hpp:376-383)
