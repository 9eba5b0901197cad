"""GPU: the consumers of the assembled matrix through the C ABI.

* loam_gpu_spmv / loam_gpu_block_spmv are BITWISE equal to the reference's
  mat_spmv / block_spmv (data.hpp:236-250, solver.hpp:33-58) on random
  matrices and on matrices the device assembled (C2 Laplace, C4 elasticity,
  the C5 Taylor-Hood BlockMat);
* loam_gpu_cg_solve(_block) reproduces the reference's cg_solve
  (solver.hpp:80-207): its known answers (test_solver.cpp), the iteration
  count (dot products are reordered, so +-1 is allowed) and the iterate to
  the solver tolerance, Jacobi, maxit, and the error contract
  (DimensionMismatch, IndefiniteBreakdown with the reference's messages).
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def dev_mat(csr):
    n, m, rp, ci, v = csr
    sp = L.Sparsity(n, m, torch.as_tensor(np.asarray(rp, np.int64)).cuda(),
                    torch.as_tensor(np.asarray(ci, np.int32)).cuda())
    A = L.Mat(sp)
    A.values[: len(v)] = torch.as_tensor(np.asarray(v, np.float64)).cuda()
    A._zero = False
    return A


def host_csr(A: L.Mat):
    rp, ci = A.sparsity.host()
    return (A.nrows, A.ncols, rp, ci, A.host_values())


def dense(A):
    A = np.asarray(A, float)
    n, m = A.shape
    return (n, m, np.arange(0, n * m + 1, m, dtype=np.int64), np.tile(np.arange(m, dtype=np.int32), n),
            A.ravel().copy())


def random_csr(rng, n, m, density):
    cols, rp = [], [0]
    for _ in range(n):
        c = np.sort(rng.choice(m, size=max(1, int(rng.binomial(m, density))), replace=False)).astype(np.int32)
        cols.append(c)
        rp.append(rp[-1] + len(c))
    ci = np.concatenate(cols)
    return (n, m, np.array(rp, np.int64), ci, rng.uniform(-1, 1, len(ci)))


@needs_ref
@pytest.mark.parametrize("seed", range(3))
def test_spmv_bitwise_random(gpu_lib, seed):
    rng = np.random.default_rng(200 + seed)
    A = random_csr(rng, 301, 257, 0.05)
    x = rng.uniform(-1, 1, 257)
    y = L.mat_spmv(dev_mat(A), x).cpu().numpy()
    assert np.array_equal(y, O.ref_spmv(A, x))


@needs_ref
@pytest.mark.parametrize("cfg,n", [(2, 32), (4, 4)])
def test_spmv_bitwise_on_assembled_matrices(gpu_lib, cfg, n):
    w = configs.Workload(cfg, n)
    w.reset()
    w.run()
    A = w.outputs[0]
    rng = np.random.default_rng(cfg)
    x = rng.uniform(-1, 1, A.ncols)
    assert np.array_equal(L.mat_spmv(A, x).cpu().numpy(), O.ref_spmv(host_csr(A), x))


@needs_ref
def test_block_spmv_bitwise_taylor_hood(gpu_lib):
    w = configs.Workload(5, 8)
    w.reset()
    w.run()
    Am, BTm, Bm = w.outputs  # [[A, B^T], [B, 0]] (solver.hpp:21-28)
    op = L.BlockMat([[Am, BTm], [Bm, None]], (Am.nrows, Bm.nrows), (Am.ncols, BTm.ncols))
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, op.ncols)
    y = L.block_spmv(op, x).cpu().numpy()
    ref = O.ref_block_spmv([[host_csr(Am), host_csr(BTm)], [host_csr(Bm), None]], op.row_sizes, op.col_sizes, x)
    assert np.array_equal(y, ref)


def test_block_spmv_known_answers(gpu_lib):
    A, B, C = dev_mat(dense([[2, 1], [1, 2]])), dev_mat(dense([[0, 1], [2, 0]])), dev_mat(dense([[1, 1], [0, 1]]))
    x = np.array([1.0, 2, 3, 4])
    y = L.block_spmv(L.BlockMat([[A, None], [None, A]], (2, 2), (2, 2)), x).cpu().numpy()
    assert list(y) == [4.0, 5.0, 10.0, 11.0]
    z = L.block_spmv(L.BlockMat([[None, B], [C, None]], (2, 2), (2, 2)), x).cpu().numpy()
    assert list(z) == [4.0, 6.0, 3.0, 2.0]
    with pytest.raises(capi.LoamError) as e:
        L.block_spmv(L.BlockMat([[A, None], [None, A]], (2, 2), (2, 2)), x[:3])
    assert e.value.kind == "DimensionMismatch"


def test_spmv_known_answers_and_errors(gpu_lib):
    assert list(L.mat_spmv(dev_mat(dense([[2, 0], [0, 3]])), [1.0, 1.0]).cpu().numpy()) == [2.0, 3.0]
    assert list(L.mat_spmv(dev_mat(dense([[4, 1], [1, 3]])), [1.0, 2.0]).cpu().numpy()) == [6.0, 7.0]
    with pytest.raises(capi.LoamError) as e:
        L.mat_spmv(dev_mat(dense([[4, 1], [1, 3]])), [1.0, 2.0, 3.0])
    assert e.value.kind == "DimensionMismatch"
    assert "spmv operand length" in str(e.value)


def test_cg_known_answers(gpu_lib):
    rng = np.random.default_rng(3)
    b = rng.uniform(0, 1, 5)
    x, rep = L.cg_solve(dev_mat(dense(np.eye(5))), b)
    assert rep.converged and rep.iterations == 1 and np.max(np.abs(x.cpu().numpy() - b)) <= 1e-14
    x, rep = L.cg_solve(dev_mat(dense([[4, 1], [1, 3]])), [1.0, 2.0], rtol=1e-12, atol=1e-16, maxit=10)
    x = x.cpu().numpy()
    assert rep.converged and abs(x[0] - 1 / 11) <= 1e-12 and abs(x[1] - 7 / 11) <= 1e-12
    with pytest.raises(capi.LoamError) as e:
        L.cg_solve(dev_mat(dense([[0, 1], [1, 3]])), [1.0, 2.0], rtol=1e-10, atol=1e-15, maxit=10,
                   precond=L.Preconditioner.JACOBI)
    assert e.value.kind == "IndefiniteBreakdown" and "row 0" in str(e.value)
    with pytest.raises(capi.LoamError) as e:
        L.cg_solve(dev_mat(dense([[1, 0], [0, -1]])), [1.0, 1.0], rtol=1e-10, atol=1e-15, maxit=10)
    assert e.value.kind == "IndefiniteBreakdown" and "after 1 iterations" in str(e.value)
    n = 30
    B = rng.uniform(0, 1, (n, n))
    x, rep = L.cg_solve(dev_mat(dense(B.T @ B + np.eye(n))), rng.uniform(0, 1, n), rtol=1e-14, atol=0.0, maxit=2)
    assert not rep.converged and rep.reason == "maxit" and rep.iterations == 2
    with pytest.raises(capi.LoamError) as e:
        L.cg_solve(dev_mat(dense(np.eye(3))), [1.0, 2.0])
    assert e.value.kind == "DimensionMismatch"


@needs_ref
@pytest.mark.parametrize("jacobi", [False, True])
def test_cg_matches_reference_on_assembled_helmholtz(gpu_lib, jacobi):
    m = configs.config_inputs(2, 48)
    cells, verts = L.Set(m.ncells), L.Set(m.nv)
    cv = L.Map(cells, verts, 3, m.cv)
    X = L.Dat(verts, 2)
    X.set_values(m.coords)
    A = L.Mat(L.build_sparsity(cv, cv))
    L.execute(L.Parloop(L.kernel("helmholtz_p1_tri", 1.0), cells, [L.arg(A, L.INC, cv, cv), L.arg(X, L.READ, cv)]))
    rng = np.random.default_rng(11)
    b = rng.uniform(-1, 1, m.nv)
    pc = L.Preconditioner.JACOBI if jacobi else L.Preconditioner.NONE
    x, rep = L.cg_solve(A, b, rtol=1e-10, atol=1e-15, maxit=2000, precond=pc)
    xr, rr = O.ref_cg(host_csr(A), b, rtol=1e-10, atol=1e-15, maxit=2000, jacobi=jacobi)
    assert rep.converged and rr["converged"] and rep.reason == rr["reason"]
    assert abs(rep.iterations - rr["iterations"]) <= 1
    x = x.cpu().numpy()
    assert np.max(np.abs(x - xr)) <= 1e-8 * np.max(np.abs(xr))
    # the true residual meets the reference's target
    r = b - L.mat_spmv(A, x).cpu().numpy()
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(b)


@needs_ref
def test_block_cg_matches_reference(gpu_lib):
    m = configs.config_inputs(2, 24)
    cells, verts = L.Set(m.ncells), L.Set(m.nv)
    cv = L.Map(cells, verts, 3, m.cv)
    X = L.Dat(verts, 2)
    X.set_values(m.coords)
    M = L.Mat(L.build_sparsity(cv, cv))
    L.execute(L.Parloop(L.kernel("mass_p1_tri"), cells, [L.arg(M, L.INC, cv, cv), L.arg(X, L.READ, cv)]))
    op = L.BlockMat([[M, None], [None, M]], (m.nv, m.nv), (m.nv, m.nv))
    rng = np.random.default_rng(13)
    b = rng.uniform(-1, 1, 2 * m.nv)
    for jac in (False, True):
        x, rep = L.cg_solve(op, b, rtol=1e-10, atol=1e-15, maxit=500,
                            precond=L.Preconditioner.JACOBI if jac else L.Preconditioner.NONE)
        Mh = host_csr(M)
        xr, rr = O.ref_cg(([[Mh, None], [None, Mh]], (m.nv, m.nv), (m.nv, m.nv)), b, rtol=1e-10, atol=1e-15,
                          maxit=500, jacobi=jac)
        assert rep.converged and abs(rep.iterations - rr["iterations"]) <= 1
        assert np.max(np.abs(x.cpu().numpy() - xr)) <= 1e-8 * np.max(np.abs(xr))
    with pytest.raises(capi.LoamError) as e:
        L.cg_solve(L.BlockMat([[M, None], [None, None]], (m.nv, m.nv), (m.nv, m.nv)), b,
                   precond=L.Preconditioner.JACOBI)
    assert e.value.kind == "IndefiniteBreakdown" and "diagonal blocks" in str(e.value)
