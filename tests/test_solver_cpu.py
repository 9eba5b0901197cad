"""CPU: pins the oracle's restatement of the matrix consumers
against the compiled reference.

* the reference's own known answers: test_data.cpp:175-205 (spmv),
  test_solver.cpp:24-123 (cg) and :171-206 (block spmv);
* restatement == compiled reference BITWISE (same operation order) for spmv,
  block spmv and CG iterates on random sparse matrices and on assembled
  P1 matrices.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def dense(A):
    A = np.asarray(A, float)
    n, m = A.shape
    rp = np.arange(0, n * m + 1, m, dtype=np.int64)
    ci = np.tile(np.arange(m, dtype=np.int32), n)
    return (n, m, rp, ci, A.ravel().copy())


def random_csr(rng, n, m, density):
    rows, cols = [], []
    rp = [0]
    for r in range(n):
        c = np.sort(rng.choice(m, size=max(1, int(rng.binomial(m, density))), replace=False)).astype(np.int32)
        cols.append(c)
        rp.append(rp[-1] + len(c))
    ci = np.concatenate(cols)
    return (n, m, np.array(rp, np.int64), ci, rng.uniform(-1, 1, len(ci)))


def spd(rng, n, shift):
    B = rng.uniform(0, 1, (n, n))
    return B.T @ B + shift * np.eye(n)


# ---- reference known answers (the restatement must reproduce them) ----------
def test_spmv_known_answers():
    for f in (O.spmv, O.ref_spmv):
        assert list(f(dense([[2, 0], [0, 3]]), [1, 1])) == [2.0, 3.0]
        assert list(f(dense([[4, 1], [1, 3]]), [1, 2])) == [6.0, 7.0]
        assert list(f(dense([[0, 0], [0, 0]]), [1, 2])) == [0.0, 0.0]
    with pytest.raises(O.KindError) as e:
        O.ref_spmv(dense([[4, 1], [1, 3]]), [1, 2, 3])
    assert e.value.kind == "DimensionMismatch"


def test_block_spmv_known_answers():
    A, B, C = dense([[2, 1], [1, 2]]), dense([[0, 1], [2, 0]]), dense([[1, 1], [0, 1]])
    x = np.array([1.0, 2, 3, 4])
    for f in (O.block_spmv, O.ref_block_spmv):
        y = f([[A, None], [None, A]], (2, 2), (2, 2), x)
        assert np.array_equal(y, np.concatenate([O.ref_spmv(A, x[:2]), O.ref_spmv(A, x[2:])]))
        z = f([[None, B], [C, None]], (2, 2), (2, 2), x)
        assert np.array_equal(z, np.concatenate([O.ref_spmv(B, x[2:]), O.ref_spmv(C, x[:2])]))
    with pytest.raises(O.KindError) as e:
        O.ref_block_spmv([[A, None], [None, A]], (2, 2), (2, 2), x[:3])
    assert e.value.kind == "DimensionMismatch"


@pytest.mark.parametrize("solve", [O.cg, O.ref_cg])
def test_cg_known_answers(solve):
    rng = np.random.default_rng(3)
    b = rng.uniform(0, 1, 5)
    x, rep = solve(dense(np.eye(5)), b)
    assert rep["converged"] and rep["iterations"] == 1 and np.max(np.abs(x - b)) <= 1e-14
    x, rep = solve(dense([[4, 1], [1, 3]]), [1, 2], rtol=1e-12, atol=1e-16, maxit=10)
    assert rep["converged"] and abs(x[0] - 1 / 11) <= 1e-12 and abs(x[1] - 7 / 11) <= 1e-12
    with pytest.raises(O.KindError) as e:
        solve(dense([[0, 1], [1, 3]]), [1, 2], rtol=1e-10, atol=1e-15, maxit=10, jacobi=True)
    assert e.value.kind == "IndefiniteBreakdown"
    with pytest.raises(O.KindError) as e:
        solve(dense([[1, 0], [0, -1]]), [1, 1], rtol=1e-10, atol=1e-15, maxit=10)
    assert e.value.kind == "IndefiniteBreakdown"
    n = 30
    x, rep = solve(dense(spd(rng, n, 1.0)), rng.uniform(0, 1, n), rtol=1e-14, atol=0.0, maxit=2)
    assert not rep["converged"] and rep["reason"] == "maxit" and rep["iterations"] == 2


def test_cg_random_spd_converges_within_n():
    rng = np.random.default_rng(31)
    for _ in range(8):
        n = 5 + int(rng.integers(0, 46))
        A = spd(rng, n, n)
        b = rng.uniform(0, 1, n)
        x, rep = O.cg(dense(A), b, rtol=1e-10, atol=1e-16, maxit=n + 2)
        assert rep["converged"] and rep["iterations"] <= n + 2
        assert np.linalg.norm(b - A @ x) <= 1e-10 * np.linalg.norm(b) + 1e-12


# ---- restatement == compiled reference, bitwise -------------------------------
@pytest.mark.parametrize("seed", range(4))
def test_spmv_bitwise_random(seed):
    rng = np.random.default_rng(100 + seed)
    A = random_csr(rng, 57, 43, 0.2)
    x = rng.uniform(-1, 1, 43)
    assert np.array_equal(O.spmv(A, x), O.ref_spmv(A, x))
    B, C = random_csr(rng, 57, 20, 0.3), random_csr(rng, 20, 43, 0.3)
    blocks = [[A, B], [C, None]]
    xx = rng.uniform(-1, 1, 63)
    assert np.array_equal(O.block_spmv(blocks, (57, 20), (43, 20), xx), O.ref_block_spmv(blocks, (57, 20), (43, 20), xx))


def p1_matrix(form, n):
    from paper_1501_01809_b200 import configs
    m = configs.config_inputs(2, n)
    rp, ci = O.build_sparsity(m.ncells, m.cv, 3, m.nv, m.cv, 3, m.nv)
    vals = O.assemble_matrix(form, 1, 2, m.ncells, m.cv, 3, m.cv, 3, m.cv, m.coords, rp, ci, params=(1.0,))
    return (m.nv, m.nv, rp, ci, vals)


@pytest.mark.parametrize("jacobi", [False, True])
def test_cg_bitwise_on_assembled_helmholtz(jacobi):
    A = p1_matrix(O.HELMHOLTZ, 12)
    rng = np.random.default_rng(7)
    b = rng.uniform(-1, 1, A[0])
    x1, r1 = O.cg(A, b, rtol=1e-10, atol=1e-15, maxit=500, jacobi=jacobi)
    x2, r2 = O.ref_cg(A, b, rtol=1e-10, atol=1e-15, maxit=500, jacobi=jacobi)
    assert r1 == r2 and r1["converged"]
    assert np.array_equal(x1, x2)
    blocks = ([[A, None], [None, A]], (A[0], A[0]), (A[0], A[0]))
    bb = np.concatenate([b, -b])
    y1, s1 = O.cg(blocks, bb, rtol=1e-10, atol=1e-15, maxit=500, jacobi=jacobi)
    y2, s2 = O.ref_cg(blocks, bb, rtol=1e-10, atol=1e-15, maxit=500, jacobi=jacobi)
    assert s1 == s2 and np.array_equal(y1, y2)
