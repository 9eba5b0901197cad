"""Irregular meshes and degenerate inputs through every auto path.

The config meshes are Kuhn / diagonal-split grids: every edge has 4-6 cells,
every P1 star <= 7 link vertices.  These meshes break those regularities:

* a 3D fan of K tetrahedra around one edge (edge valence K, vertex rows of
  ~K+2 nodes, P2 rows of ~4K entries: the edge-tile plan's wide-record path,
  node-block tiles with long diagonal items);
* a 2D star of K triangles around a vertex plus an outer ring (link of K
  vertices: the vertex-star / ring plans decline, the general owner kernels
  run);
* an empty iteration set.

Every result is compared with the oracle at 1e-12 (relative max norm).
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    den = np.max(np.abs(b)) if np.size(b) else 0.0
    return float(np.max(np.abs(a - b)) / den) if den else float(np.max(np.abs(a))) if np.size(a) else 0.0


def fan3d(K, seed=1):
    rng = np.random.default_rng(seed)
    pts = [(0.0, 0.0, 0.0), (0.0, 0.0, 1.0)]
    for i in range(K):
        t = 2 * math.pi * i / K
        pts.append((math.cos(t), math.sin(t), 0.5 + 0.2 * (rng.random() - 0.5)))
    cv = []
    for i in range(K):
        cv += [0, 1, 2 + i, 2 + (i + 1) % K]
    return configs.MeshInputs(3, 0, np.array(pts, dtype=np.float64).ravel(), np.array(cv, dtype=np.int32))


def star2d(K, seed=2):
    rng = np.random.default_rng(seed)
    pts = [(0.0, 0.0)]
    for i in range(K):  # inner ring 1..K, outer ring K+1..2K
        t = 2 * math.pi * (i + 0.1 * rng.random()) / K
        pts.append((math.cos(t), math.sin(t)))
    for i in range(K):
        t = 2 * math.pi * (i + 0.5) / K
        pts.append((2 * math.cos(t), 2 * math.sin(t)))
    cv = []
    for i in range(K):
        r0, r1, o0, o1 = 1 + i, 1 + (i + 1) % K, 1 + K + i, 1 + K + (i + 1) % K
        cv += [0, r0, r1, r0, o0, r1, r1, o0, o1]
    return configs.MeshInputs(2, 0, np.array(pts, dtype=np.float64).ravel(), np.array(cv, dtype=np.int32))


def build(m, degree):
    from paper_1501_01809_b200 import loam as L
    nv1 = m.gdim + 1
    cells, verts = L.Set(m.ncells, "cells"), L.Set(m.nv, "vertices")
    cvm = L.Map(cells, verts, nv1, m.cv, "cell_vertex")
    X = L.Dat(verts, m.gdim, "coordinates")
    X.set_values(m.coords)
    if degree == 1:
        return L, cells, cvm, cvm, m.nv, X, m.cv, nv1
    cn, nn = configs.p2_map(m)
    ar = 6 if m.gdim == 2 else 10
    nodes = L.Set(nn, "p2_nodes")
    return L, cells, cvm, L.Map(cells, nodes, ar, cn, "cell_node"), nn, X, cn, ar


def matrix_case(m, form, degree, params=()):
    L, cells, cvm, rm, nn, X, rmap, ar = build(m, degree)
    sfx = ("_p%d" % degree) + ("_tri" if m.gdim == 2 else "_tet")
    sp = L.build_sparsity(rm, rm)
    A = L.Mat(sp, form)
    lp = L.Parloop(L.kernel(form + sfx, *params), cells, [L.arg(A, L.INC, rm, rm), L.arg(X, L.READ, cvm)])
    A.zero()
    L.execute(lp)
    rp, ci = sp.host()
    code = {"mass": O.MASS, "stiffness": O.STIFFNESS, "helmholtz": O.HELMHOLTZ}[form]
    ref = O.assemble_matrix(code, degree, m.gdim, m.ncells, rmap, ar, rmap, ar, m.cv, m.coords, rp, ci,
                            params=params)
    return A.host_values(), ref


def action_case(m, degree):
    L, cells, cvm, rm, nn, X, rmap, ar = build(m, degree)
    sfx = ("_p%d" % degree) + ("_tri" if m.gdim == 2 else "_tet")
    u = L.Dat(rm.target, 1, "u")
    uv = np.sin(np.arange(nn) * 0.37)
    u.set_values(uv)
    b = L.Dat(rm.target, 1, "b")
    lp = L.Parloop(L.kernel("helmholtz_action" + sfx, configs.KAPPA), cells,
                   [L.arg(b, L.INC, rm), L.arg(X, L.READ, cvm), L.arg(u, L.READ, rm)])
    b.zero()
    L.execute(lp)
    ref = O.assemble_vector(O.HELMHOLTZ_ACTION, degree, m.gdim, m.ncells, rmap, ar, m.cv, m.coords, rmap, ar,
                            uv, nn, params=(configs.KAPPA,))
    return b.view(), ref


@pytest.fixture(autouse=True)
def _auto(gpu_lib):
    capi.set_strategy("auto")
    yield
    capi.set_strategy("auto")


@pytest.mark.parametrize("K", [3, 12, 40])
@pytest.mark.parametrize("degree", [1, 2])
def test_fan3d_helmholtz_matrix(K, degree):
    got, ref = matrix_case(fan3d(K), "helmholtz", degree, (configs.KAPPA,))
    assert rel(got, ref) <= TOL


@pytest.mark.parametrize("K", [3, 12, 40])
@pytest.mark.parametrize("degree", [1, 2])
def test_fan3d_helmholtz_action(K, degree):
    got, ref = action_case(fan3d(K), degree)
    assert rel(got, ref) <= TOL


@pytest.mark.parametrize("K", [3, 12, 40])
def test_fan3d_elasticity(K):
    from paper_1501_01809_b200 import loam as L
    m = fan3d(K)
    cells, verts = L.Set(m.ncells, "cells"), L.Set(m.nv, "vertices")
    cvm = L.Map(cells, verts, 4, m.cv, "cell_vertex")
    X = L.Dat(verts, 3, "coordinates")
    X.set_values(m.coords)
    dm = L.expanded_map(cvm, 3)
    sp = L.build_sparsity(cvm, cvm, 3, 3)
    A = L.Mat(sp, "elasticity")
    lp = L.Parloop(L.kernel("elasticity_p1_tet", *configs.LAME), cells, [L.arg(A, L.INC, dm, dm), L.arg(X, L.READ, cvm)])
    A.zero()
    L.execute(lp)
    rp, ci = sp.host()
    ref = O.assemble_matrix(O.ELASTICITY, 1, 3, m.ncells, dm.values, 12, dm.values, 12, m.cv, m.coords, rp, ci,
                            params=configs.LAME)
    assert rel(A.host_values(), ref) <= TOL


@pytest.mark.parametrize("K", [5, 9, 20])
@pytest.mark.parametrize("degree", [1, 2])
@pytest.mark.parametrize("form", ["stiffness", "helmholtz"])
def test_star2d_matrix(K, degree, form):
    params = (configs.KAPPA,) if form == "helmholtz" else ()
    got, ref = matrix_case(star2d(K), form, degree, params)
    assert rel(got, ref) <= TOL


@pytest.mark.parametrize("K", [5, 9, 20])
@pytest.mark.parametrize("degree", [1, 2])
def test_star2d_action(K, degree):
    got, ref = action_case(star2d(K), degree)
    assert rel(got, ref) <= TOL


def test_empty_iteration_set_leaves_outputs():
    """par_loop over an empty set (parloop.hpp:191: nothing to do): INC Dat and
    Mat outputs keep their values."""
    from paper_1501_01809_b200 import loam as L
    verts = L.Set(5, "vertices")
    cells = L.Set(0, "cells")
    cvm = L.Map(cells, verts, 3, np.zeros(0, dtype=np.int32), "cell_vertex")
    X = L.Dat(verts, 2, "coordinates")
    X.set_values(np.arange(10, dtype=np.float64))
    b = L.Dat(verts, 1, "b")
    b.set_values(np.full(5, 7.0))
    u = L.Dat(verts, 1, "u")
    u.set_values(np.ones(5))
    L.execute(L.Parloop(L.kernel("helmholtz_action_p1_tri", 1.0), cells,
                        [L.arg(b, L.INC, cvm), L.arg(X, L.READ, cvm), L.arg(u, L.READ, cvm)]))
    assert np.array_equal(b.view(), np.full(5, 7.0))
    sp = L.build_sparsity(cvm, cvm)
    assert sp.nnz == 0
    A = L.Mat(sp, "empty")
    A.zero()
    L.execute(L.Parloop(L.kernel("stiffness_p1_tri"), cells, [L.arg(A, L.INC, cvm, cvm), L.arg(X, L.READ, cvm)]))
    assert A.host_values().size in (0, 1)


@pytest.mark.parametrize("K", [12, 20])
def test_fan3d_takes_the_tile_paths(K):
    """The fan's P2 matrix runs on the edge tiles (its hub edge row has 4K + 3
    entries: the wide-record path) and its elasticity on the node-block tiles.
    (At K = 40 the hub row's lane-interleaved segment exceeds the tile budget
    and the pair tiles run instead -- test_fan3d_helmholtz_matrix covers it.)"""
    from paper_1501_01809_b200 import loam as L
    m = fan3d(K)
    L_, cells, cvm, rm, nn, X, rmap, ar = build(m, 2)
    sp = L.build_sparsity(rm, rm)
    A = L.Mat(sp, "helmholtz")
    lp = L.Parloop(L.kernel("helmholtz_p2_tet", configs.KAPPA), cells, [L.arg(A, L.INC, rm, rm), L.arg(X, L.READ, cvm)])
    A.zero()
    L.execute(lp)
    A.zero()
    l0 = capi.launch_count()
    L.execute(lp)
    assert capi.launch_count() - l0 == 2  # diagonal zeroing + edge tiles
    rp, ci = sp.host()
    ref = O.assemble_matrix(O.HELMHOLTZ, 2, 3, m.ncells, rmap, ar, rmap, ar, m.cv, m.coords, rp, ci,
                            params=(configs.KAPPA,))
    assert rel(A.host_values(), ref) <= TOL
    dm = L.expanded_map(cvm, 3)
    spe = L.build_sparsity(cvm, cvm, 3, 3)
    E = L.Mat(spe, "elasticity")
    le = L.Parloop(L.kernel("elasticity_p1_tet", *configs.LAME), cells, [L.arg(E, L.INC, dm, dm), L.arg(X, L.READ, cvm)])
    E.zero()
    L.execute(le)
    E.zero()
    l0 = capi.launch_count()
    L.execute(le)
    assert capi.launch_count() - l0 == 1  # node-block tiles
    rp, ci = spe.host()
    ref = O.assemble_matrix(O.ELASTICITY, 1, 3, m.ncells, dm.values, 12, dm.values, 12, m.cv, m.coords, rp, ci,
                            params=configs.LAME)
    assert rel(E.host_values(), ref) <= TOL
