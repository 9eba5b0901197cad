"""Link-walk tiles for scalar P2 matrices on tetrahedra (csrc/wtile.cu).

assemble_matrix(mass / stiffness / helmholtz) on a P2 tetrahedral space
(fem/assemble.hpp:85-104): every edge row walks the link of its mesh edge and
carries the vertex rows by symmetry.  Parity: the oracle's par_loop (relative
max norm 1e-12, the north star's tolerance), the edge-tile path, accumulation
into existing values, and meshes the plan must decline (a duplicated cell:
edge links that are no ring or fan) falling back with the same results.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L

pytestmark = pytest.mark.gpu
TOL = 1e-12
KINDS = {"mass": O.MASS, "stiffness": O.STIFFNESS, "helmholtz": O.HELMHOLTZ}


def rel(a, b):
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den else 1.0)


@pytest.fixture(autouse=True)
def _reset(gpu_lib):
    capi.set_strategy("auto")
    for k in ("LOAM_GPU_NO_WTILE", "LOAM_GPU_WT_REQUIRE"):
        os.environ.pop(k, None)
    yield
    for k in ("LOAM_GPU_NO_WTILE", "LOAM_GPU_WT_REQUIRE"):
        os.environ.pop(k, None)


def setup(n, form, cv=None, cn=None, seed=None):
    m = configs.config_inputs(3, n)
    cv = m.cv if cv is None else cv
    cn = m.extra["p2"] if cn is None else cn
    nc = len(cv) // 4
    cells, verts, nodes = L.Set(nc), L.Set(m.nv), L.Set(m.extra["nn"])
    cvm, cnm = L.Map(cells, verts, 4, cv), L.Map(cells, nodes, 10, cn)
    X = L.Dat(verts, 3)
    X.set_values(m.coords)
    A = L.Mat(L.build_sparsity(cnm, cnm))
    params = (1.7,) if form == "helmholtz" else ()
    loop = L.Parloop(L.kernel(f"{form}_p2_tet", *params), cells, [L.arg(A, L.INC, cnm, cnm), L.arg(X, L.READ, cvm)])
    rp, ci = A.sparsity.host()
    ref = O.assemble_matrix(KINDS[form], 2, 3, nc, cn, 10, cn, 10, cv, m.coords, rp, ci, params=params)
    return loop, A, ref


@pytest.mark.parametrize("form", ["mass", "stiffness", "helmholtz"])
@pytest.mark.parametrize("n", [1, 2, 3, 6])
def test_walk_tiles_match_oracle_and_edge_tiles(form, n):
    os.environ["LOAM_GPU_WT_REQUIRE"] = "1"  # the walk-tile plan must be the one that runs
    loop, A, ref = setup(n, form)
    L.execute(loop)
    got = A.host_values().copy()
    assert rel(got, ref) <= TOL
    L.execute(loop)  # INC adds to what is there (parloop.hpp:301-305)
    assert rel(A.host_values(), 2 * ref) <= TOL
    A.zero()
    L.execute(loop)  # a fresh Mat again: the diagonals start from zero
    assert rel(A.host_values(), ref) <= TOL
    os.environ.pop("LOAM_GPU_WT_REQUIRE")
    os.environ["LOAM_GPU_NO_WTILE"] = "1"
    loop2, A2, _ = setup(n, form)
    L.execute(loop2)
    assert rel(A2.host_values(), got) <= TOL


def test_duplicated_cell_declines_the_walk_plan():
    m = configs.config_inputs(3, 3)
    cv = np.concatenate([m.cv, m.cv[: 4 * 3]])
    cn = np.concatenate([m.extra["p2"], m.extra["p2"][: 10 * 3]])
    loop, A, ref = setup(3, "helmholtz", cv, cn)
    L.execute(loop)
    assert rel(A.host_values(), ref) <= TOL
    os.environ["LOAM_GPU_WT_REQUIRE"] = "1"
    loop2, A2, _ = setup(3, "helmholtz", cv, cn)
    with pytest.raises(capi.LoamError):
        L.execute(loop2)


def test_config3_matrix_takes_the_walk_tiles():
    os.environ["LOAM_GPU_WT_REQUIRE"] = "1"
    w = configs.Workload(3, 8, "matrix")
    w.reset()
    w.run()
    m = w.inputs
    A = w.outputs[0]
    rp, ci = A.sparsity.host()
    cn = m.extra["p2"]
    ref = O.assemble_matrix(O.HELMHOLTZ, 2, 3, m.ncells, cn, 10, cn, 10, m.cv, m.coords, rp, ci, params=(configs.KAPPA,))
    assert rel(A.host_values(), ref) <= TOL


@pytest.mark.parametrize("K", [3, 5, 12, 13, 40])
@pytest.mark.parametrize("form", ["mass", "helmholtz"])
def test_fans_around_one_edge(K, form):
    """K tetrahedra around one edge (the meshes of test_irregular_gpu): the
    centre edge's link is a ring of K vertices, every other edge has a fan of
    one or two cells.  Up to 12 cells per link the walk tiles run; beyond, the
    plan declines and the edge tiles take over.  All against the oracle."""
    from tests.test_irregular_gpu import fan3d
    m = fan3d(K)
    cn, nn = configs.p2_map(m)
    cells, verts, nodes = L.Set(m.ncells), L.Set(m.nv), L.Set(nn)
    cvm, cnm = L.Map(cells, verts, 4, m.cv), L.Map(cells, nodes, 10, cn)
    X = L.Dat(verts, 3)
    X.set_values(m.coords)
    A = L.Mat(L.build_sparsity(cnm, cnm))
    params = (1.7,) if form == "helmholtz" else ()
    loop = L.Parloop(L.kernel(f"{form}_p2_tet", *params), cells, [L.arg(A, L.INC, cnm, cnm), L.arg(X, L.READ, cvm)])
    if K <= 12:
        os.environ["LOAM_GPU_WT_REQUIRE"] = "1"
    L.execute(loop)
    rp, ci = A.sparsity.host()
    ref = O.assemble_matrix(KINDS[form], 2, 3, m.ncells, cn, 10, cn, 10, m.cv, m.coords, rp, ci, params=params)
    assert rel(A.host_values(), ref) <= TOL
    L.execute(loop)
    assert rel(A.host_values(), 2 * ref) <= TOL
