"""CPU: the oracle (C restatement, oracle/liborc.so) pinned to the reference.

Pins, in order of strength:
  1. known-answer tests copied (as numbers) from the reference's own tests:
     test_topology.cpp:55-84, test_data.cpp:22-62, test_fem.cpp:141-161,226-250;
  2. golden vectors produced by the UNMODIFIED reference (oracle/_ref, see
     tools/make_golden.py) -- bit-exact for integer outputs, <= 1e-13 for values;
  3. the reference's property checks (colouring validity by brute force,
     sparsity vs a dense boolean pattern, oracles.hpp:17-48);
  4. exact symbolic integration (tests/exact_fem.py) for what the reference
     lacks: P2 tets, the 14-point rule, elasticity, Stokes -- "parity unpinned"
     by reference tests, pinned here only against exact integrals.
"""
import os

import numpy as np
import pytest

import oracle as O
from tests import exact_fem as EX

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


def rel(a, b):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300)


# ------------------------------------------------------------------ 1. KATs
def test_colouring_kats():  # test_topology.cpp:55-84
    c, n = O.color_iteration(2, [np.array([0, 1, 2, 1, 3, 2])], [3], [4])
    assert list(c) == [0, 1] and n == 2
    c, n = O.color_iteration(2, [], [], [])
    assert list(c) == [0, 0] and n == 1
    c, n = O.color_iteration(4, [np.array([0, 1, 2, 0, 3, 4, 0, 5, 6, 0, 7, 8])], [3], [9])
    assert list(c) == [0, 1, 2, 3] and n == 4


def test_sparsity_kats():  # test_data.cpp:22-62
    rp, ci = O.build_sparsity(2, [0, 1, 2, 1, 3, 2], 3, 4, [0, 1, 2, 1, 3, 2], 3, 4)
    assert rp[-1] == 14 and list(np.diff(rp)) == [3, 4, 4, 3]
    rp, ci = O.build_sparsity(1, [0, 1, 2], 3, 3, [0, 1, 2], 3, 3)
    assert rp[-1] == 9
    rp, ci = O.build_sparsity(5, [0, 1, 2, 3, 4], 1, 5, [0, 1, 2, 3, 4], 1, 5)
    assert rp[-1] == 5 and list(ci) == [0, 1, 2, 3, 4]


def test_p2_numbering_kat():  # test_fem.cpp:226-250 on unit_square_mesh(1)
    cv = np.array([0, 1, 3, 0, 3, 2], dtype=np.int32)  # mesh.hpp:119-124, n=1
    cn, nn = O.p2_cell_node_map(cv, 4, 2)
    assert nn == 9
    edge = {(0, 1): 4, (0, 2): 5, (0, 3): 6, (1, 3): 7, (2, 3): 8}
    assert list(cn[:6]) == [0, 1, 3, edge[(1, 3)], edge[(0, 3)], edge[(0, 1)]]


def test_reference_triangle_kernels_kat():  # test_fem.cpp:141-161
    X = np.array([0.0, 0.0, 1.0, 0.0, 0.0, 1.0])
    K = O.element(O.STIFFNESS, 1, 2, X)
    assert np.allclose(K, [[1.0, -0.5, -0.5], [-0.5, 0.5, 0.0], [-0.5, 0.0, 0.5]], atol=1e-15)
    M = O.element(O.MASS, 1, 2, X)
    assert np.allclose(M, (np.ones((3, 3)) + np.eye(3)) / 24.0, atol=1e-15)
    b = O.element(O.MASS_ACTION, 1, 2, X, np.ones(3))  # source(V, 1.0) == mass action on ones
    assert np.allclose(b.ravel(), 1.0 / 6, atol=1e-15)
    H = O.element(O.HELMHOLTZ, 1, 2, X, params=(2.5,))
    assert np.allclose(H, K + 2.5 * M, atol=1e-15)


# ------------------------------------------------------------------ 2. golden vectors of the reference
def test_golden_colourings_bit_exact():
    g = gold("c1_n8.npz")
    c, n = O.color_iteration(g["cv"].size // 3, [g["cv"]], [3], [g["coords"].size // 2])
    assert np.array_equal(c, g["colors"]) and n == int(g["ncolors"])
    g = gold("p1tet_n3.npz")
    c, n = O.color_iteration(g["cv"].size // 4, [g["cv"]], [4], [g["coords"].size // 3])
    assert np.array_equal(c, g["colors"]) and n == int(g["ncolors"])


def test_golden_sparsities_bit_exact():
    for name, ar, gd in (("c2_n8.npz", 3, 2), ("p1tet_n3.npz", 4, 3)):
        g = gold(name)
        nc, nv = g["cv"].size // ar, g["coords"].size // gd
        rp, ci = O.build_sparsity(nc, g["cv"], ar, nv, g["cv"], ar, nv)
        assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])
    g = gold("sparsity_dims.npz")
    rp, ci = O.build_sparsity(20, g["rv"], 3, 9, g["cv"], 2, 7, 2, 3)
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(ci, g["col_idx"])


def test_golden_p2_triangle_numbering_bit_exact():
    g = gold("p2tri_n4.npz")
    cn, nn = O.p2_cell_node_map(g["cv"], g["coords"].size // 2, 2)
    assert nn == int(g["nn"]) and np.array_equal(cn, g["cn"])


def test_golden_assembled_values():
    g = gold("c1_n8.npz")
    nc, nv = g["cv"].size // 3, g["coords"].size // 2
    b = O.assemble_vector(O.HELMHOLTZ_ACTION, 1, 2, nc, g["cv"], 3, g["cv"], g["coords"], g["cv"], 3, g["u"], nv,
                          params=(1.0,))
    assert rel(b, g["residual"]) <= 1e-13
    g = gold("c2_n8.npz")
    nc = g["cv"].size // 3
    v = O.assemble_matrix(O.STIFFNESS, 1, 2, nc, g["cv"], 3, g["cv"], 3, g["cv"], g["coords"], g["row_ptr"], g["col_idx"])
    assert rel(v, g["values"]) <= 1e-13
    g = gold("p2tri_n4.npz")
    nc = g["cv"].size // 3
    v = O.assemble_matrix(O.HELMHOLTZ, 2, 2, nc, g["cn"], 6, g["cn"], 6, g["cv"], g["coords"], g["row_ptr"],
                          g["col_idx"], params=(1.5,))
    assert rel(v, g["values"]) <= 1e-13
    g = gold("p1tet_n3.npz")
    nc = g["cv"].size // 4
    v = O.assemble_matrix(O.MASS, 1, 3, nc, g["cv"], 4, g["cv"], 4, g["cv"], g["coords"], g["row_ptr"], g["col_idx"])
    assert rel(v, g["values"]) <= 1e-13


def test_golden_local_kernels():
    g = gold("local_kernels.npz")
    for kind in (O.MASS, O.STIFFNESS, O.HELMHOLTZ, O.MASS_ACTION, O.STIFFNESS_ACTION):
        for tag, deg, gd, X, C in (("tri_p1", 1, 2, g["X2"], g["C3"]), ("tri_p2", 2, 2, g["X2"], g["C6"]),
                                   ("tet_p1", 1, 3, g["X3"], np.append(g["C3"], 0.4))):
            out = O.element(kind, deg, gd, X, C if kind >= O.MASS_ACTION else None, params=(2.5,))
            assert rel(out.ravel(), g[f"{tag}_{kind}"].ravel()) <= 1e-13, (tag, kind)


# ------------------------------------------------------------------ 3. property checks (oracles.hpp)
@pytest.mark.parametrize("trial", range(12))
def test_colouring_valid_by_brute_force(trial):  # oracles.hpp:17-32
    rng = np.random.default_rng(trial)
    n, nv = int(rng.integers(1, 60)), int(rng.integers(3, 40))
    t = rng.integers(0, nv, 3 * n).astype(np.int32)
    c, nc = O.color_iteration(n, [t], [3], [nv])
    T = t.reshape(n, 3)
    for a in range(n):
        for b in range(a + 1, n):
            if c[a] == c[b]:
                assert not set(T[a]) & set(T[b])
    # greedy first-fit: every entity's colour is the smallest not used by earlier conflicting entities
    for e in range(n):
        used = {c[f] for f in range(e) if set(T[f]) & set(T[e])}
        assert c[e] == min(set(range(nc + 1)) - used)


@pytest.mark.parametrize("trial", range(8))
def test_sparsity_matches_dense_pattern(trial):  # oracles.hpp:35-48
    rng = np.random.default_rng(100 + trial)
    n, nrt, nct = int(rng.integers(1, 40)), int(rng.integers(2, 12)), int(rng.integers(2, 12))
    rd, cd = int(rng.integers(1, 3)), int(rng.integers(1, 4))
    rv = rng.integers(0, nrt, 3 * n).astype(np.int32)
    cv = rng.integers(0, nct, 2 * n).astype(np.int32)
    rp, ci = O.build_sparsity(n, rv, 3, nrt, cv, 2, nct, rd, cd)
    dense = np.zeros((nrt * rd, nct * cd), dtype=bool)
    for e in range(n):
        for a in rv[3 * e:3 * e + 3]:
            for b in cv[2 * e:2 * e + 2]:
                dense[a * rd:(a + 1) * rd, b * cd:(b + 1) * cd] = True
    for r in range(nrt * rd):
        assert list(ci[rp[r]:rp[r + 1]]) == list(np.nonzero(dense[r])[0])


# ------------------------------------------------------------------ 4. exact integration (unpinned forms)
@pytest.mark.parametrize("d,p", [(2, 1), (2, 2), (3, 1), (3, 2)])
def test_lagrange_kernels_match_exact_integration(d, p):  # test_fem.cpp:163-202 extended to P2 tets
    rng = np.random.default_rng(2024 + 10 * d + p)
    for _ in range(5):
        X = EX.random_simplex(d, rng)
        M, K = EX.mass(X, d, p), EX.stiffness(X, d, p)
        assert rel(O.element(O.MASS, p, d, X), M) <= 1e-12
        assert rel(O.element(O.STIFFNESS, p, d, X), K) <= 1e-12
        assert rel(O.element(O.HELMHOLTZ, p, d, X, params=(1.7,)), K + 1.7 * M) <= 1e-12
        c = rng.uniform(-1, 1, M.shape[0])
        assert rel(O.element(O.MASS_ACTION, p, d, X, c).ravel(), M @ c) <= 1e-12
        assert rel(O.element(O.STIFFNESS_ACTION, p, d, X, c).ravel(), K @ c) <= 1e-12
        assert rel(O.element(O.HELMHOLTZ_ACTION, p, d, X, c, params=(1.7,)).ravel(), (K + 1.7 * M) @ c) <= 1e-12


def test_vector_forms_match_exact_integration():
    rng = np.random.default_rng(77)
    for _ in range(5):
        X3 = EX.random_simplex(3, rng)
        assert rel(O.element(O.ELASTICITY, 1, 3, X3, params=(1.0, 0.5)), EX.elasticity(X3, 1.0, 0.5)) <= 1e-12
        X2 = EX.random_simplex(2, rng)
        A, B = EX.stokes(X2, 1.0)
        assert rel(O.element(O.STOKES_A, 2, 2, X2, params=(1.0,)), A) <= 1e-12
        assert rel(O.element(O.STOKES_B, 2, 2, X2), B) <= 1e-12
        assert rel(O.element(O.STOKES_BT, 2, 2, X2), B.T) <= 1e-12


def test_elasticity_kernel_properties():
    """Rigid motions are in the kernel; the matrix is symmetric."""
    rng = np.random.default_rng(5)
    X = EX.random_simplex(3, rng)
    K = O.element(O.ELASTICITY, 1, 3, X, params=(1.0, 0.5))
    assert rel(K, K.T) <= 1e-14
    pts = X.reshape(4, 3)
    for t in np.eye(3):  # translations
        assert np.max(np.abs(K @ np.tile(t, 4))) <= 1e-12 * np.max(np.abs(K))
    w = np.array([0.3, -0.2, 0.7])  # infinitesimal rotation u = w x x
    u = np.concatenate([np.cross(w, x) for x in pts])
    assert np.max(np.abs(K @ u)) <= 1e-11 * np.max(np.abs(K)) * np.max(np.abs(u))


# ------------------------------------------------------------------ 5. compiled reference directly (build container only)
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
def test_reference_engine_agrees_with_restatement_on_p2_tets():
    from paper_1501_01809_b200 import configs
    m = configs.config_inputs(3, 3)
    cn, nn = m.extra["p2"], m.extra["nn"]
    rp, ci, rv = O.ref_engine_matrix(O.HELMHOLTZ, 2, 3, m.ncells, cn, 10, nn, cn, 10, nn, m.cv, m.coords, params=(1.0,))
    ov = O.assemble_matrix(O.HELMHOLTZ, 2, 3, m.ncells, cn, 10, cn, 10, m.cv, m.coords, rp, ci, params=(1.0,))
    assert rel(ov, rv) <= 1e-13
    rb = O.ref_engine_vector(O.HELMHOLTZ_ACTION, 2, 3, m.ncells, cn, 10, nn, m.cv, m.coords, m.extra["u"], params=(1.0,))
    ob = O.assemble_vector(O.HELMHOLTZ_ACTION, 2, 3, m.ncells, cn, 10, m.cv, m.coords, cn, 10, m.extra["u"], nn,
                           params=(1.0,))
    assert rel(ob, rb) <= 1e-13


@needs_ref
def test_reference_threads_bitwise_identical():  # test_parloop.cpp:273-315 on the compiled reference
    from paper_1501_01809_b200 import configs
    m = configs.config_inputs(2, 12)
    a = O.ref_assemble_matrix(O.STIFFNESS, 1, 2, m.cv, m.coords, threads=1)[2]
    b = O.ref_assemble_matrix(O.STIFFNESS, 1, 2, m.cv, m.coords, threads=4)[2]
    assert np.array_equal(a, b)


def _dof_map(nodes, arity, dim):
    v = np.asarray(nodes, np.int64).reshape(-1, arity)
    return (v[:, :, None] * dim + np.arange(dim)).reshape(-1).astype(np.int32)


@needs_ref
def test_reference_engine_agrees_with_restatement_on_elasticity():
    """C4 through the compiled reference ENGINE (build_sparsity + execute + Mat::addto,
    data.hpp:149-222, parloop.hpp:191-384) with dof-expanded maps:
    sparsity bit-exact and values equal to the restatement's assembly."""
    from paper_1501_01809_b200 import configs
    m = configs.config_inputs(4, 8)
    dm = _dof_map(m.cv, 4, 3)
    rp, ci, rv = O.ref_engine_matrix(O.ELASTICITY, 1, 3, m.ncells, dm, 12, 3 * m.nv, dm, 12, 3 * m.nv, m.cv,
                                     m.coords, params=configs.LAME)
    orp, oci = O.build_sparsity(m.ncells, m.cv, 4, m.nv, m.cv, 4, m.nv, 3, 3)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    ov = O.assemble_matrix(O.ELASTICITY, 1, 3, m.ncells, dm, 12, dm, 12, m.cv, m.coords, rp, ci, params=configs.LAME)
    assert rel(ov, rv) <= 1e-13


@needs_ref
def test_reference_engine_agrees_with_restatement_on_taylor_hood_blocks():
    """C5's A, B and B^T through the compiled reference engine with separate
    velocity (dof-expanded P2) and pressure (P1) maps."""
    from paper_1501_01809_b200 import configs
    m = configs.config_inputs(5, 8)
    cn, nn = m.extra["p2"], m.extra["nn"]
    vd = _dof_map(cn, 6, 2)
    for form, rmap, ar_r, nrt, cmap, ar_c, nct, prm, rdim, cdim in (
            (O.STOKES_A, vd, 12, 2 * nn, vd, 12, 2 * nn, (configs.NU,), (cn, 6, nn, 2), (cn, 6, nn, 2)),
            (O.STOKES_B, m.cv, 3, m.nv, vd, 12, 2 * nn, (), (m.cv, 3, m.nv, 1), (cn, 6, nn, 2)),
            (O.STOKES_BT, vd, 12, 2 * nn, m.cv, 3, m.nv, (), (cn, 6, nn, 2), (m.cv, 3, m.nv, 1))):
        rp, ci, rv = O.ref_engine_matrix(form, 2, 2, m.ncells, rmap, ar_r, nrt, cmap, ar_c, nct, m.cv, m.coords,
                                         params=prm)
        orp, oci = O.build_sparsity(m.ncells, rdim[0], rdim[1], rdim[2], cdim[0], cdim[1], cdim[2], rdim[3], cdim[3])
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
        ov = O.assemble_matrix(form, 2, 2, m.ncells, rmap, ar_r, cmap, ar_c, m.cv, m.coords, rp, ci, params=prm)
        assert rel(ov, rv) <= 1e-13


# ------------------------------------------------------------------ 6. the oracle-side input generator
@pytest.mark.parametrize("cfg,n", [(1, 7), (2, 16), (3, 3), (4, 4), (5, 6), (2, 1024)])
def test_oracle_generator_equals_product_generator(cfg, n):
    """bench --impl reference builds its inputs with the restatement (no product
    library in that process): they must be the very bits the GPU arm assembles."""
    from paper_1501_01809_b200 import configs
    a, b = O.inputs(cfg, n), configs.config_inputs(cfg, n)
    assert np.array_equal(a.cv, b.cv)
    assert np.array_equal(a.coords.view(np.uint64), b.coords.view(np.uint64))
    for k in b.extra:
        va, vb = np.asarray(a.extra[k]), np.asarray(b.extra[k])
        assert np.array_equal(va.view(np.uint64) if va.dtype == np.float64 else va,
                              vb.view(np.uint64) if vb.dtype == np.float64 else vb), k
    assert (O.FULL, O.JITTER, O.PERM_SEED) == (configs.FULL, configs.JITTER, configs.PERM_SEED)


@needs_ref
@pytest.mark.parametrize("gdim,n", [(2, 5), (3, 3)])
def test_oracle_meshes_equal_reference_generators(gdim, n):
    coords, cv = O.ref_unit_mesh(gdim, n)
    m = O.mesh(gdim, n)
    assert np.array_equal(m.cv, cv) and np.array_equal(m.coords, coords)


@needs_ref
def test_timed_reference_engine_runs():
    m = O.inputs(4, 3)
    dm = O.dof_map(m.cv, 4, 3)
    t, sp = O.ref_time_engine(O.ELASTICITY, 1, 3, m.ncells, dm, 12, 3 * m.nv, dm, 12, 3 * m.nv, m.cv, m.coords,
                              params=(1.0, 0.5), threads=2, warmup=1, steps=2)
    assert t.size == 2 and np.all(t > 0) and sp > 0
    m = O.inputs(3, 2)
    t, sp = O.ref_time_engine(O.HELMHOLTZ_ACTION, 2, 3, m.ncells, m.extra["p2"], 10, m.extra["nn"], None, 0, 0,
                              m.cv, m.coords, coeff=m.extra["u"], params=(1.0,), threads=1, warmup=0, steps=1)
    assert t[0] > 0 and sp == 0.0
