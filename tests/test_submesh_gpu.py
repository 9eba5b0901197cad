"""par_loops over a SUB-mesh into outputs sized for the whole mesh.

The reference allows a loop whose (map, map) pattern is narrower than its
Mat's sparsity: `validate` only compares shapes (parloop.hpp:119-121), the
Mat starts as zeros (data.hpp:185-187) and `addto` touches only the entries
the loop's cells reach (data.hpp:205-222).  So a loop over some of the cells
into a Mat whose sparsity was built from ALL the cells must leave every other
entry zero -- and a Dat INC over some cells must leave untouched nodes zero.

Every catalogue form of the five configs (C1 P1 residual, C2 P1 stiffness,
C3 P2-tet residual and matrix, C4 vector-P1 elasticity, C5 Taylor-Hood
A / B / B^T) is run on a region sub-mesh (cells with centroid x < 0.55) and a
scattered random half of the cells, through every INC strategy, into fresh
outputs, and compared with the oracle over the same sub-mesh (relative max
norm 1e-12; zeros outside the touched entries are part of the comparison).
"""
import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L

pytestmark = pytest.mark.gpu
TOL = 1e-12
STRATS = ["auto", "owner", "atomic", "color"]


def rel(a, b):
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den else 1.0)


@pytest.fixture(autouse=True)
def _strategy_reset(gpu_lib):
    yield
    capi.set_strategy("auto")


def pick(m, how):
    cv = m.cv.reshape(m.ncells, m.gdim + 1)
    if how == "region":
        cx = m.coords.reshape(-1, m.gdim)[cv][:, :, 0].mean(axis=1)
        sel = np.nonzero(cx < 0.55)[0]
    else:
        sel = np.sort(np.random.default_rng(17).permutation(m.ncells)[: m.ncells // 2])
    assert 0 < sel.size < m.ncells
    return sel.astype(np.int64)


def rows(a, arity, sel):
    return np.ascontiguousarray(np.asarray(a).reshape(-1, arity)[sel].reshape(-1))


class Sub:
    """Whole-mesh Sets / Maps / coordinates plus the sub-mesh cell Set and its maps."""

    def __init__(self, cfg, n, how):
        m = self.m = configs.config_inputs(cfg, n)
        self.sel = pick(m, how)
        self.ns = self.sel.size
        self.verts = L.Set(m.nv, "vertices")
        self.cells = L.Set(m.ncells, "cells")
        self.sub = L.Set(self.ns, "sub_cells")
        self.cvm = L.Map(self.cells, self.verts, m.gdim + 1, m.cv, "cell_vertex")
        self.cv_s = rows(m.cv, m.gdim + 1, self.sel)
        self.svm = L.Map(self.sub, self.verts, m.gdim + 1, self.cv_s, "sub_vertex")
        self.X = L.Dat(self.verts, m.gdim, "coordinates")
        self.X.set_values(m.coords)
        if "p2" in m.extra:
            ar = 6 if m.gdim == 2 else 10
            self.ar = ar
            self.nodes = L.Set(m.extra["nn"], "p2_nodes")
            self.cnm = L.Map(self.cells, self.nodes, ar, m.extra["p2"], "cell_node")
            self.cn_s = rows(m.extra["p2"], ar, self.sel)
            self.snm = L.Map(self.sub, self.nodes, ar, self.cn_s, "sub_node")


@pytest.mark.parametrize("strat", STRATS)
@pytest.mark.parametrize("how", ["region", "random"])
def test_c1_residual_on_sub_mesh(strat, how):
    capi.set_strategy(strat)
    s = Sub(1, 12, how)
    m = s.m
    u = L.Dat(s.verts, 1, "u")
    u.set_values(m.extra["u"])
    b = L.Dat(s.verts, 1, "residual")
    L.execute(L.Parloop(L.kernel("helmholtz_action_p1_tri", configs.KAPPA), s.sub,
                        [L.arg(b, L.INC, s.svm), L.arg(s.X, L.READ, s.svm), L.arg(u, L.READ, s.svm)]))
    ref = O.assemble_vector(O.HELMHOLTZ_ACTION, 1, 2, s.ns, s.cv_s, 3, s.cv_s, m.coords, s.cv_s, 3,
                            m.extra["u"], m.nv, params=(configs.KAPPA,))
    assert np.all(ref[np.setdiff1d(np.arange(m.nv), s.cv_s)] == 0.0)
    assert rel(b.view(), ref) <= TOL


@pytest.mark.parametrize("strat", STRATS)
@pytest.mark.parametrize("how", ["region", "random"])
@pytest.mark.parametrize("form,kind", [("stiffness_p1_tri", O.STIFFNESS), ("helmholtz_p1_tri", O.HELMHOLTZ),
                                       ("mass_p1_tri", O.MASS)])
def test_c2_matrix_on_sub_mesh_into_full_pattern(strat, how, form, kind):
    capi.set_strategy(strat)
    s = Sub(2, 14, how)
    m = s.m
    A = L.Mat(L.build_sparsity(s.cvm, s.cvm), "A")  # the WHOLE mesh's pattern
    A.values.fill_(np.nan)  # stale memory: a fresh Mat must not read it
    A.zero()
    L.execute(L.Parloop(L.kernel(form, 1.0), s.sub, [L.arg(A, L.INC, s.svm, s.svm), L.arg(s.X, L.READ, s.svm)]))
    rp, ci = A.sparsity.host()
    ref = O.assemble_matrix(kind, 1, 2, s.ns, s.cv_s, 3, s.cv_s, 3, s.cv_s, m.coords, rp, ci, params=(1.0,))
    got = A.host_values()
    assert np.count_nonzero(ref == 0.0) > 0  # entries outside the sub-mesh pattern
    assert not np.any(np.isnan(got))
    assert rel(got, ref) <= TOL
    # a second INC adds onto those values (untouched entries stay zero)
    L.execute(L.Parloop(L.kernel(form, 1.0), s.sub, [L.arg(A, L.INC, s.svm, s.svm), L.arg(s.X, L.READ, s.svm)]))
    assert rel(A.host_values(), 2 * ref) <= TOL


@pytest.mark.parametrize("strat", STRATS)
@pytest.mark.parametrize("how", ["region", "random"])
def test_c3_p2_residual_and_matrix_on_sub_mesh(strat, how):
    capi.set_strategy(strat)
    s = Sub(3, 3, how)
    m = s.m
    nn = m.extra["nn"]
    u = L.Dat(s.nodes, 1, "u")
    u.set_values(m.extra["u"])
    b = L.Dat(s.nodes, 1, "residual")
    L.execute(L.Parloop(L.kernel("helmholtz_action_p2_tet", configs.KAPPA), s.sub,
                        [L.arg(b, L.INC, s.snm), L.arg(s.X, L.READ, s.svm), L.arg(u, L.READ, s.snm)]))
    ref_b = O.assemble_vector(O.HELMHOLTZ_ACTION, 2, 3, s.ns, s.cn_s, 10, s.cv_s, m.coords, s.cn_s, 10,
                              m.extra["u"], nn, params=(configs.KAPPA,))
    assert rel(b.view(), ref_b) <= TOL
    A = L.Mat(L.build_sparsity(s.cnm, s.cnm), "A")
    A.values.fill_(np.nan)
    A.zero()
    L.execute(L.Parloop(L.kernel("helmholtz_p2_tet", configs.KAPPA), s.sub,
                        [L.arg(A, L.INC, s.snm, s.snm), L.arg(s.X, L.READ, s.svm)]))
    rp, ci = A.sparsity.host()
    ref_A = O.assemble_matrix(O.HELMHOLTZ, 2, 3, s.ns, s.cn_s, 10, s.cn_s, 10, s.cv_s, m.coords, rp, ci,
                              params=(configs.KAPPA,))
    assert np.count_nonzero(ref_A == 0.0) > 0
    assert rel(A.host_values(), ref_A) <= TOL


@pytest.mark.parametrize("strat", STRATS)
@pytest.mark.parametrize("how", ["region", "random"])
def test_c4_elasticity_on_sub_mesh(strat, how):
    capi.set_strategy(strat)
    s = Sub(4, 3, how)
    m = s.m
    dofs = L.Set(3 * m.nv, "dofs")
    dm_s = L.expanded_map(s.svm, 3, dofs)
    A = L.Mat(L.build_sparsity(s.cvm, s.cvm, 3, 3), "A")
    A.values.fill_(np.nan)
    A.zero()
    L.execute(L.Parloop(L.kernel("elasticity_p1_tet", *configs.LAME), s.sub,
                        [L.arg(A, L.INC, dm_s, dm_s), L.arg(s.X, L.READ, s.svm)]))
    rp, ci = A.sparsity.host()
    ref = O.assemble_matrix(O.ELASTICITY, 1, 3, s.ns, dm_s.values, 12, dm_s.values, 12, s.cv_s, m.coords,
                            rp, ci, params=configs.LAME)
    assert np.count_nonzero(ref == 0.0) > 0
    assert rel(A.host_values(), ref) <= TOL


@pytest.mark.parametrize("strat", STRATS)
@pytest.mark.parametrize("how", ["region", "random"])
def test_c5_taylor_hood_blocks_on_sub_mesh(strat, how):
    capi.set_strategy(strat)
    s = Sub(5, 6, how)
    m = s.m
    nn = m.extra["nn"]
    vdofs = L.Set(2 * nn, "velocity_dofs")
    vdm_s = L.expanded_map(s.snm, 2, vdofs)
    A = L.Mat(L.build_sparsity(s.cnm, s.cnm, 2, 2), "A")
    B = L.Mat(L.build_sparsity(s.cvm, s.cnm, 1, 2), "B")
    BT = L.Mat(L.build_sparsity(s.cnm, s.cvm, 2, 1), "BT")
    for M in (A, B, BT):
        M.values.fill_(np.nan)
        M.zero()
    L.execute(L.Parloop(L.kernel("stokes_a_p2_tri", configs.NU), s.sub,
                        [L.arg(A, L.INC, vdm_s, vdm_s), L.arg(s.X, L.READ, s.svm)]))
    L.execute(L.Parloop(L.kernel("stokes_b_p2_tri"), s.sub, [L.arg(B, L.INC, s.svm, vdm_s), L.arg(s.X, L.READ, s.svm)]))
    L.execute(L.Parloop(L.kernel("stokes_bt_p2_tri"), s.sub, [L.arg(BT, L.INC, vdm_s, s.svm), L.arg(s.X, L.READ, s.svm)]))
    vd = vdm_s.values
    for M, kind, rm, ar_r, cm, ar_c, prm in ((A, O.STOKES_A, vd, 12, vd, 12, (configs.NU,)),
                                             (B, O.STOKES_B, s.cv_s, 3, vd, 12, ()),
                                             (BT, O.STOKES_BT, vd, 12, s.cv_s, 3, ())):
        rp, ci = M.sparsity.host()
        ref = O.assemble_matrix(kind, 2, 2, s.ns, rm, ar_r, cm, ar_c, s.cv_s, m.coords, rp, ci, params=prm)
        assert np.count_nonzero(ref == 0.0) > 0
        assert rel(M.host_values(), ref) <= TOL, M.name
