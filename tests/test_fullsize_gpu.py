"""BASELINE full sizes (configs C1-C5 exactly as bench.py runs them, `auto`
path): every output against the C restatement at full size -- sparsity
row_ptr / col_idx bit-exact against orc_build_sparsity (data.hpp:149-179),
values within relative max norm 1e-12 (north_star tolerance) of
orc_assemble_matrix / orc_assemble_vector (the reference's par_loop + addto,
data.hpp:205-222) -- plus size-independent properties of the assembled
operators (which would also catch an error shared by kernel and oracle):

* C3 matrix (60.9 M nnz): A u = b(u) -- the matrix (edge tiles) and the
  residual (cell kernel) are the same bilinear form through two unrelated
  kernels, and b(u) is itself checked against the oracle above; A = A^T;
  1^T A 1 = kappa |Omega| = kappa (the stiffness part annihilates constants).
* C4 96^3 elasticity (121 M nnz): A r = 0 for the six rigid-body motions
  (three translations, three rotations: the linear strain of a rigid motion
  is zero, so the element matrix annihilates it to rounding); A = A^T.
* C5 768^2 Taylor-Hood blocks: A c = 0 for constant velocity fields (viscous
  block), B c = 0 and sum_p (B u)_p = -|Omega| = -1 for u = (x, 0) and
  (0, y) (B = -int q div u; the P2 interpolant of a linear field is exact),
  B^T = transpose(B), and the nnz counts SURVEY 8(a) a10 states.

Residual tolerances are relative to the magnitudes the products sum
(|A| |x|), 1e-12.
"""
import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs

sp = pytest.importorskip("scipy.sparse")

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den else 1.0)


def csr(mat, ncols):
    rp, ci = mat.sparsity.host()
    return sp.csr_matrix((mat.host_values(), ci, rp), shape=(rp.size - 1, ncols))


def small_against(A, x, y):
    """|A x - y| <= TOL * |A| |x| row by row (the scale of the terms summed)."""
    scale = abs(A) @ np.abs(x)
    return float(np.max(np.abs(A @ x - y) / np.maximum(scale, 1e-300) * (scale > 0)))


def symmetric(A):
    D = (A - A.T).tocsr()
    return (float(np.max(np.abs(D.data))) if D.nnz else 0.0) / float(np.max(np.abs(A.data)))


@pytest.fixture(autouse=True)
def _auto(gpu_lib):
    capi.set_strategy("auto")
    yield


def run(cfg, part=None):
    w = configs.Workload(cfg, None, part)
    w.reset()
    w.run()
    return w


def test_c1_full_residual_equals_oracle():
    w = run(1)
    m = w.inputs
    assert m.ncells == 524288
    ref = O.assemble_vector(O.HELMHOLTZ_ACTION, 1, 2, m.ncells, m.cv, 3, m.cv, m.coords, m.cv, 3,
                            m.extra["u"], m.nv, params=(configs.KAPPA,))
    assert rel(w.outputs[0].view(), ref) <= TOL


def test_c2_full_csr_equals_oracle():
    w = run(2)
    m = w.inputs
    assert m.ncells == 2097152
    A = w.outputs[0]
    rp, ci = A.sparsity.host()
    orp, oci = O.build_sparsity(m.ncells, m.cv, 3, m.nv, m.cv, 3, m.nv)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci) and ci.size == 7346177
    ref = O.assemble_matrix(O.STIFFNESS, 1, 2, m.ncells, m.cv, 3, m.cv, 3, m.cv, m.coords, rp, ci)
    assert rel(A.host_values(), ref) <= TOL
    K = csr(A, m.nv)
    assert small_against(K, np.ones(m.nv), np.zeros(m.nv)) <= TOL  # K 1 = 0
    assert symmetric(K) <= TOL


def oracle_csr(mat, ncells, rmap, ar_r, nrt, cmap, ar_c, nct, rd, cd):
    """row_ptr / col_idx of the Mat, checked bit-exact against the restatement."""
    rp, ci = mat.sparsity.host()
    orp, oci = O.build_sparsity(ncells, rmap, ar_r, nrt, cmap, ar_c, nct, rd, cd)
    assert np.array_equal(rp, orp), "row_ptr differs from orc_build_sparsity"
    assert np.array_equal(ci, oci), "col_idx differs from orc_build_sparsity"
    del orp, oci
    return rp, ci


def dof_map(nodes, arity, dim):
    v = np.asarray(nodes, np.int64).reshape(-1, arity)
    return (v[:, :, None] * dim + np.arange(dim)).reshape(-1).astype(np.int32)


def test_c3_full_residual_equals_oracle_and_matrix_action():
    w = run(3)
    m = w.inputs
    cn, nn = m.extra["p2"], m.extra["nn"]
    assert m.ncells == 1572864 and nn == 2146689
    b = w.outputs[0].view()
    ref = O.assemble_vector(O.HELMHOLTZ_ACTION, 2, 3, m.ncells, cn, 10, m.cv, m.coords, cn, 10,
                            m.extra["u"], nn, params=(configs.KAPPA,))
    assert rel(b, ref) <= TOL
    # the matrix value for value: sparsity bit-exact, values 1e-12
    rp, ci = oracle_csr(w.outputs[1], m.ncells, cn, 10, nn, cn, 10, nn, 1, 1)
    refA = O.assemble_matrix(O.HELMHOLTZ, 2, 3, m.ncells, cn, 10, cn, 10, m.cv, m.coords, rp, ci,
                             params=(configs.KAPPA,))
    assert rel(w.outputs[1].host_values(), refA) <= TOL
    del refA
    A = csr(w.outputs[1], nn)
    assert A.nnz == 60859905
    assert small_against(A, m.extra["u"], b) <= TOL  # A u = b(u): two kernels, one form
    assert symmetric(A) <= TOL
    one = np.ones(nn)
    scale = float(np.sum(abs(A) @ one))  # the magnitude the double sum cancels from
    assert abs(one @ (A @ one) - configs.KAPPA) <= TOL * scale  # kappa |unit cube|


def rigid_modes(X):
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    o, zr = np.ones_like(x), np.zeros_like(x)
    fields = [(o, zr, zr), (zr, o, zr), (zr, zr, o), (-y, x, zr), (zr, -z, y), (z, zr, -x)]
    return [np.stack(f, axis=1).ravel() for f in fields]  # dof = 3 * vertex + component


def test_c4_full_elasticity_equals_oracle_and_annihilates_rigid_motions():
    w = run(4)
    m = w.inputs
    assert m.ncells == 5308416
    rp, ci = oracle_csr(w.outputs[0], m.ncells, m.cv, 4, m.nv, m.cv, 4, m.nv, 3, 3)
    dm = dof_map(m.cv, 4, 3)
    ref = O.assemble_matrix(O.ELASTICITY, 1, 3, m.ncells, dm, 12, dm, 12, m.cv, m.coords, rp, ci,
                            params=configs.LAME)
    assert rel(w.outputs[0].host_values(), ref) <= TOL
    del ref, dm
    A = csr(w.outputs[0], 3 * m.nv)
    assert A.nnz == 121188969
    X = m.coords.reshape(-1, 3)
    for r in rigid_modes(X):
        assert small_against(A, r, np.zeros(3 * m.nv)) <= TOL
    assert symmetric(A) <= TOL


def p2_node_coords(m):
    """Vertex nodes keep the vertex coordinates; edge nodes sit at midpoints
    (cell row = vertices, then edges (1,2), (0,2), (0,1): space.hpp:66-71)."""
    cn, nn = m.extra["p2"].reshape(-1, 6), m.extra["nn"]
    X = m.coords.reshape(-1, 2)
    cv = m.cv.reshape(-1, 3)
    P = np.zeros((nn, 2))
    P[: m.nv] = X
    for k, (a, b) in enumerate(((1, 2), (0, 2), (0, 1))):
        P[cn[:, 3 + k]] = 0.5 * (X[cv[:, a]] + X[cv[:, b]])
    return P


def test_c5_full_blocks_equal_oracle_and_properties():
    w = run(5)
    m = w.inputs
    nn = m.extra["nn"]
    assert m.ncells == 1179648 and nn == 2362369
    Am, BTm, Bm = w.outputs
    cn = m.extra["p2"]
    vd = dof_map(cn, 6, 2)
    for M, form, rmap, ar_r, cmap, ar_c, prm, rsp, csp in (
            (Am, O.STOKES_A, vd, 12, vd, 12, (configs.NU,), (cn, 6, nn, 2), (cn, 6, nn, 2)),
            (Bm, O.STOKES_B, m.cv, 3, vd, 12, (), (m.cv, 3, m.nv, 1), (cn, 6, nn, 2)),
            (BTm, O.STOKES_BT, vd, 12, m.cv, 3, (), (cn, 6, nn, 2), (m.cv, 3, m.nv, 1))):
        rp, ci = oracle_csr(M, m.ncells, rsp[0], rsp[1], rsp[2], csp[0], csp[1], csp[2], rsp[3], csp[3])
        ref = O.assemble_matrix(form, 2, 2, m.ncells, rmap, ar_r, cmap, ar_c, m.cv, m.coords, rp, ci, params=prm)
        assert rel(M.host_values(), ref) <= TOL, M.name
        del ref
    A, B, BT = csr(Am, 2 * nn), csr(Bm, 2 * nn), csr(BTm, m.nv)
    assert (A.nnz, B.nnz, BT.nnz) == (108576772, 22428674, 22428674)
    P = p2_node_coords(m)
    zero_v, zero_p = np.zeros(2 * nn), np.zeros(m.nv)
    for c in ((1.0, 0.0), (0.0, 1.0)):
        cst = np.tile(np.array(c), nn)  # dof = 2 * node + component
        assert small_against(A, cst, zero_v) <= TOL
        assert small_against(B, cst, zero_p) <= TOL
    for comp in (0, 1):
        u = np.zeros((nn, 2))
        u[:, comp] = P[:, comp]  # div u = 1
        Bu = B @ u.ravel()
        assert abs(Bu.sum() + 1.0) <= TOL * float(np.sum(abs(B) @ np.abs(u.ravel())))
    assert symmetric(A) <= TOL
    D = (BT - B.T.tocsr())
    assert (float(np.max(np.abs(D.data))) if D.nnz else 0.0) <= TOL * float(np.max(np.abs(B.data)))
