"""Edge-tile assembly of scalar P2 matrices (csrc/etile.cu) against the oracle.

The edge-tile path writes every vertex-row entry through the symmetric
edge rows (transposed entries, vertex pairs) and RED-adds the vertex
diagonals, so these tests cover: all three catalogue forms on tetrahedra and
triangles, fresh and accumulating Mats (Mat INC into non-zero values), the
path actually being taken (two launches: diagonal zeroing + edge tiles), and
the fallback when the P2 numbering does not put vertex nodes first.
Tolerance: relative max-norm 1e-12 (north_star); sparsity bit-exact.
"""
import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs

pytestmark = pytest.mark.gpu
TOL = 1e-12
FORMS = {"mass": O.MASS, "stiffness": O.STIFFNESS, "helmholtz": O.HELMHOLTZ}


def rel(a, b):
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den else 1.0)


def setup(gdim, n, form, node_perm_seed=None):
    from paper_1501_01809_b200 import loam as L
    m = configs.mesh(gdim, n, 0.15, 11, 12)
    cn, nn = configs.p2_map(m)
    if node_perm_seed is not None:  # renumber nodes: vertex nodes no longer come first
        perm = np.random.default_rng(node_perm_seed).permutation(nn).astype(np.int32)
        cn = perm[cn]
    cells = L.Set(m.ncells, "cells")
    verts = L.Set(m.nv, "vertices")
    nodes = L.Set(nn, "p2_nodes")
    cvm = L.Map(cells, verts, gdim + 1, m.cv, "cell_vertex")
    cnm = L.Map(cells, nodes, 6 if gdim == 2 else 10, cn, "cell_node")
    X = L.Dat(verts, gdim, "coordinates")
    X.set_values(m.coords)
    sp = L.build_sparsity(cnm, cnm)
    A = L.Mat(sp, form)
    sfx = "_p2_tri" if gdim == 2 else "_p2_tet"
    params = (configs.KAPPA,) if form == "helmholtz" else ()
    loop = L.Parloop(L.kernel(form + sfx, *params), cells, [L.arg(A, L.INC, cnm, cnm), L.arg(X, L.READ, cvm)])
    rp, ci = sp.host()
    ar = 6 if gdim == 2 else 10
    ref = O.assemble_matrix(FORMS[form], 2, gdim, m.ncells, cn, ar, cn, ar, m.cv, m.coords, rp, ci, params=params)
    return L, loop, A, ref


def launches(L, loop):
    l0 = capi.launch_count()
    L.execute(loop)
    return capi.launch_count() - l0


@pytest.mark.parametrize("form", list(FORMS))
@pytest.mark.parametrize("gdim,n", [(3, 1), (3, 3), (3, 6), (2, 2), (2, 9)])
def test_edge_tiles_match_oracle(gpu_lib, form, gdim, n):
    capi.set_strategy("auto")
    L, loop, A, ref = setup(gdim, n, form)
    A.zero()
    L.execute(loop)  # builds and caches the plan
    assert rel(A.host_values(), ref) <= TOL
    A.zero()
    assert launches(L, loop) == 2, "edge-tile path not taken (diagonal zeroing + edge-tile kernel)"
    assert rel(A.host_values(), ref) <= TOL


@pytest.mark.parametrize("gdim,n", [(3, 4), (2, 7)])
def test_edge_tiles_accumulate(gpu_lib, gdim, n):
    """Mat INC into a non-zero Mat adds (data.hpp:219-220): two executes give twice the values."""
    capi.set_strategy("auto")
    L, loop, A, ref = setup(gdim, n, "helmholtz")
    A.zero()
    L.execute(loop)
    L.execute(loop)
    assert rel(A.host_values(), 2 * ref) <= TOL


@pytest.mark.parametrize("gdim,n", [(3, 3), (2, 6)])
def test_renumbered_nodes_fall_back(gpu_lib, gdim, n):
    """Vertex nodes not numbered first: the edge-tile plan declines, the pair-tile path runs."""
    capi.set_strategy("auto")
    L, loop, A, ref = setup(gdim, n, "helmholtz", node_perm_seed=5)
    A.zero()
    L.execute(loop)
    A.zero()
    assert launches(L, loop) == 1
    assert rel(A.host_values(), ref) <= TOL


@pytest.mark.parametrize("n", [1, 3, 8])
def test_stokes_velocity_block_edge_tiles(gpu_lib, n):
    """Config 5's A block (nu grad u : grad v on vector P2, 2x2 component-diagonal
    blocks) through the edge tiles: values and the explicit structural zeros."""
    capi.set_strategy("auto")
    w = configs.Workload(5, n)
    w.reset()
    w.L.execute(w.loops[0])  # (the loop on its own: Workload.run issues the three blocks fused, thtile.cu)
    w.reset()
    l0 = capi.launch_count()
    w.L.execute(w.loops[0])
    assert capi.launch_count() - l0 == 2, "edge-tile path not taken for the Stokes A block"
    m = w.inputs
    dm = w.vdm.values
    A = w.outputs[0]
    rp, ci = A.sparsity.host()
    ref = O.assemble_matrix(O.STOKES_A, 2, 2, m.ncells, dm, 12, dm, 12, m.cv, m.coords, rp, ci, params=(configs.NU,))
    assert rel(A.host_values(), ref) <= TOL
    w.L.execute(w.loops[0])  # accumulate
    assert rel(A.host_values(), 2 * ref) <= TOL


@pytest.mark.parametrize("n", [1, 3, 6])
def test_elasticity_node_block_tiles(gpu_lib, n):
    """Config 4 (vector P1 elasticity, 3x3-blocked CSR) through the node-block
    tiles (csrc/ntile.cu): one launch, values vs the oracle, accumulation."""
    capi.set_strategy("auto")
    w = configs.Workload(4, n)
    w.reset()
    w.run()
    w.reset()
    l0 = capi.launch_count()
    w.run()
    assert capi.launch_count() - l0 == 1, "node-block tile path not taken"
    m = w.inputs
    dm = w.dof_map.values
    A = w.outputs[0]
    rp, ci = A.sparsity.host()
    ref = O.assemble_matrix(O.ELASTICITY, 1, 3, m.ncells, dm, 12, dm, 12, m.cv, m.coords, rp, ci, params=configs.LAME)
    assert rel(A.host_values(), ref) <= TOL
    w.run()  # accumulate
    assert rel(A.host_values(), 2 * ref) <= TOL


@pytest.mark.parametrize("n", [1, 4, 9])
def test_stokes_coupling_blocks_row_tiles(gpu_lib, n):
    """Config 5's B (pressure rows) and B^T (velocity rows) blocks through the
    row tiles with shared cell geometry (csrc/rtile.cu): one launch each,
    values vs the oracle, accumulation."""
    capi.set_strategy("auto")
    w = configs.Workload(5, n)
    w.reset()
    for lp in w.loops:  # (the loops one by one: Workload.run issues the three blocks fused, thtile.cu)
        w.L.execute(lp)
    m = w.inputs
    dm = w.vdm.values
    A, BT, B = w.outputs
    for lp, out, form, rmap, ar, cmap, ac in ((w.loops[1], B, O.STOKES_B, m.cv, 3, dm, 12),
                                              (w.loops[2], BT, O.STOKES_BT, dm, 12, m.cv, 3)):
        out.zero()
        l0 = capi.launch_count()
        w.L.execute(lp)
        assert capi.launch_count() - l0 == 1
        rp, ci = out.sparsity.host()
        ref = O.assemble_matrix(form, 2, 2, m.ncells, rmap, ar, cmap, ac, m.cv, m.coords, rp, ci)
        assert rel(out.host_values(), ref) <= TOL
        w.L.execute(lp)  # accumulate
        assert rel(out.host_values(), 2 * ref) <= TOL
