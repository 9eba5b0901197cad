"""Device build_sparsity / color_iteration / Mat insertion vs the reference.

Restates test_data.cpp:22-150 and test_topology.cpp:55-102 on the device:
sparsity bit-exact (row_ptr/col_idx) including dof expansion, greedy colouring
bit-exact (Jones-Plassmann with ascending priority reproduces the greedy
first-fit order), OutsideSparsity reported with the offending (row, col).
"""
import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L
from paper_1501_01809_b200.capi import LoamError

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _reset(gpu_lib):
    yield
    capi.set_strategy("auto")


def test_sparsity_of_the_two_triangle_mesh():  # test_data.cpp:22-40
    cells, verts = L.Set(2), L.Set(4)
    m = L.Map(cells, verts, 3, [0, 1, 2, 1, 3, 2])
    sp = L.build_sparsity(m, m)
    assert sp.nrows == 4 and sp.ncols == 4 and sp.nnz == 14
    rp, ci = sp.host()
    for r in range(4):
        assert np.all(np.diff(ci[rp[r]:rp[r + 1]]) > 0)


def test_sparsity_trivia():  # test_data.cpp:42-62
    one, verts = L.Set(1), L.Set(3)
    m = L.Map(one, verts, 3, [0, 1, 2])
    assert L.build_sparsity(m, m).nnz == 9
    s5 = L.Set(5)
    ident = L.Map(s5, s5, 1, [0, 1, 2, 3, 4])
    sp = L.build_sparsity(ident, ident)
    assert sp.nnz == 5 and all(sp.find(i, i) == i for i in range(5))
    other = L.Set(4)
    wrong = L.Map(other, verts, 3, [0, 1, 2] * 4)
    with pytest.raises(LoamError) as e:
        L.build_sparsity(m, wrong)
    assert e.value.kind == "SourceMismatch"


@pytest.mark.parametrize("trial", range(10))
def test_sparsity_matches_oracle_on_random_map_pairs(trial):  # test_data.cpp:64-91
    rng = np.random.default_rng(99 + trial)
    ncells, nrt, nct = int(rng.integers(1, 51)), int(rng.integers(2, 14)), int(rng.integers(2, 14))
    rv = rng.integers(0, nrt, 3 * ncells).astype(np.int32)
    cvv = rng.integers(0, nct, 2 * ncells).astype(np.int32)
    rdim, cdim = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    cells = L.Set(ncells)
    rm, cm = L.Map(cells, L.Set(nrt), 3, rv), L.Map(cells, L.Set(nct), 2, cvv)
    sp = L.build_sparsity(rm, cm, rdim, cdim)
    rp, ci = sp.host()
    orp, oci = O.build_sparsity(ncells, rv, 3, nrt, cvv, 2, nct, rdim, cdim)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    dense = np.zeros((nrt * rdim, nct * cdim), dtype=bool)  # oracles.hpp:35-48
    for e in range(ncells):
        for a in rv[3 * e:3 * e + 3]:
            for b in cvv[2 * e:2 * e + 2]:
                dense[a * rdim:(a + 1) * rdim, b * cdim:(b + 1) * cdim] = True
    assert sp.nnz == dense.sum()


@pytest.mark.parametrize("cfg,n", [(1, 64), (2, 128), (3, 6), (4, 8), (5, 32)])
def test_sparsity_of_config_meshes_is_bit_exact(cfg, n):
    m = configs.config_inputs(cfg, n)
    cells = L.Set(m.ncells)
    if cfg in (3, 5):
        cn, nn, ar = m.extra["p2"], m.extra["nn"], (10 if cfg == 3 else 6)
    else:
        cn, nn, ar = m.cv, m.nv, m.gdim + 1
    mp = L.Map(cells, L.Set(nn), ar, cn)
    dim = 3 if cfg == 4 else (2 if cfg == 5 else 1)
    sp = L.build_sparsity(mp, mp, dim, dim)
    rp, ci = sp.host()
    orp, oci = O.build_sparsity(m.ncells, cn, ar, nn, cn, ar, nn, dim, dim)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)


def test_greedy_colouring_kats():  # test_topology.cpp:55-84
    cells, verts = L.Set(2), L.Set(4)
    m = L.Map(cells, verts, 3, [0, 1, 2, 1, 3, 2])
    colors, nc = L.color_iteration(cells, [m])
    assert list(colors) == [0, 1] and nc == 2
    colors, nc = L.color_iteration(cells, [])
    assert list(colors) == [0, 0] and nc == 1
    fc, fv = L.Set(4), L.Set(9)
    fan = L.Map(fc, fv, 3, [0, 1, 2, 0, 3, 4, 0, 5, 6, 0, 7, 8])
    colors, nc = L.color_iteration(fc, [fan])
    assert list(colors) == [0, 1, 2, 3]
    with pytest.raises(LoamError) as e:
        L.color_iteration(fc, [m])
    assert e.value.kind == "SourceMismatch"


@pytest.mark.parametrize("trial", range(20))
def test_colouring_bit_exact_on_random_meshes(trial):  # test_topology.cpp:86-102
    rng = np.random.default_rng(7 + trial)
    ncells, nverts = int(rng.integers(1, 41)), int(rng.integers(3, 33))
    table = rng.integers(0, nverts, 3 * ncells).astype(np.int32)
    cells = L.Set(ncells)
    m = L.Map(cells, L.Set(nverts), 3, table)
    colors, nc = L.color_iteration(cells, [m])
    oc, onc = O.color_iteration(ncells, [table], [3], [nverts])
    assert np.array_equal(colors, oc) and nc == onc


@pytest.mark.parametrize("cfg,n", [(1, 64), (2, 96), (4, 6)])
def test_colouring_bit_exact_on_config_meshes(cfg, n):
    m = configs.config_inputs(cfg, n)
    cells = L.Set(m.ncells)
    mp = L.Map(cells, L.Set(m.nv), m.gdim + 1, m.cv)
    colors, nc = L.color_iteration(cells, [mp])
    oc, onc = O.color_iteration(m.ncells, [m.cv], [m.gdim + 1], [m.nv])
    assert np.array_equal(colors, oc) and nc == onc


def test_two_conflict_maps_union():
    rng = np.random.default_rng(3)
    t1 = rng.integers(0, 20, 3 * 60).astype(np.int32)
    t2 = rng.integers(0, 15, 2 * 60).astype(np.int32)
    cells = L.Set(60)
    m1, m2 = L.Map(cells, L.Set(20), 3, t1), L.Map(cells, L.Set(15), 2, t2)
    colors, nc = L.color_iteration(cells, [m1, m2])
    oc, onc = O.color_iteration(60, [t1, t2], [3, 2], [20, 15])
    assert np.array_equal(colors, oc) and nc == onc


@pytest.mark.parametrize("strat", ["auto", "atomic", "color"])
def test_outside_sparsity_names_the_entry(strat):  # test_data.cpp:93-124
    capi.set_strategy(strat)
    cells, verts = L.Set(1), L.Set(4)
    m = L.Map(cells, verts, 3, [0, 1, 2])
    mat = L.Mat(L.build_sparsity(m, m))
    other = L.Map(cells, verts, 3, [0, 1, 3])  # column 3 is not in the pattern
    with pytest.raises(LoamError) as e:
        L.execute(L.Parloop(L.kernel("ones_block"), cells, [L.arg(mat, L.INC, m, other)]))
    assert e.value.kind == "OutsideSparsity" and "3)" in str(e.value)


def test_map_construction_rejects_out_of_range_entries():  # topology.hpp:45-48
    with pytest.raises(LoamError) as e:
        L.Map(L.Set(1), L.Set(3), 3, [0, 1, 3])
    assert e.value.kind == "IndexOutOfRange"
    with pytest.raises(LoamError) as e:
        L.Map(L.Set(2), L.Set(3), 3, [0, 1, 2])
    assert e.value.kind == "ArityMismatch"
