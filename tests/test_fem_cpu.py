"""SURVEY 8f-2 / 8f-3 oracle pins (CPU): the C restatements of pointwise
(fem/assemble.hpp:150-319) and apply_dirichlet (fem/assemble.hpp:54-79) are
bitwise equal to the compiled reference on random programs, fields and
patterns, including the MissingDiagonal failure."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="compiled reference (oracle/_ref) not built")

CONST, FIELD, ADD, SUB, MUL, DIV, NEG = range(7)


def random_program(rng, nfields, depth=4, use_out=True):
    """Random expression tree as a postfix program (left subtree first)."""
    def node(d):
        if d == 0 or rng.random() < 0.25:
            if rng.random() < 0.4:
                return [(CONST, 0, float(rng.uniform(-2, 2)))]
            f = int(rng.integers(-1 if use_out else 0, nfields))
            return [(FIELD, f, 0.0)]
        if rng.random() < 0.15:
            return node(d - 1) + [(NEG, 0, 0.0)]
        op = int(rng.choice([ADD, SUB, MUL, DIV]))
        return node(d - 1) + node(d - 1) + [(op, 0, 0.0)]
    return node(depth)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("assign", [0, 1, 2])
def test_pointwise_restatement_is_bitwise_reference(seed, assign):
    rng = np.random.default_rng(seed)
    size, dim = 97, 1 + seed % 3
    fields = [rng.standard_normal(size * dim) + 3.0 for _ in range(3)]  # away from zero (division)
    out = rng.standard_normal((size, dim)) + 3.0
    prog = random_program(rng, 3, use_out=seed % 2 == 0)
    got = O.pointwise(prog, assign, out.reshape(-1), fields)
    ref = O.pointwise(prog, assign, out, fields, lib="ref").reshape(-1)
    assert np.array_equal(got, ref)


def test_pointwise_wave_updates():  # bench.hpp wave loop: phi -= dt/2 p ; p += b * pc
    rng = np.random.default_rng(7)
    n = 50
    phi, p, b, pc = (rng.standard_normal(n) for _ in range(4))
    prog1 = [(CONST, 0, 0.005), (FIELD, 0, 0.0), (MUL, 0, 0.0)]
    prog2 = [(FIELD, 0, 0.0), (FIELD, 1, 0.0), (MUL, 0, 0.0)]
    assert np.array_equal(O.pointwise(prog1, 2, phi, [p]), O.pointwise(prog1, 2, phi, [p], lib="ref"))
    assert np.array_equal(O.pointwise(prog2, 1, p, [b, pc]), O.pointwise(prog2, 1, p, [b, pc], lib="ref"))


def csr_of(ncells, cmap, arity, nn, rng):
    rp, ci = O.build_sparsity(ncells, cmap, arity, nn, cmap, arity, nn)
    return (nn, nn, rp, ci, rng.standard_normal(ci.size))


@pytest.mark.parametrize("with_rhs", [True, False])
@pytest.mark.parametrize("function", [False, True])
def test_apply_dirichlet_restatement_is_bitwise_reference(with_rhs, function):
    rng = np.random.default_rng(3)
    nn, ncells = 60, 90
    cmap = np.array([rng.choice(nn, 3, replace=False) for _ in range(ncells)], np.int32).reshape(-1)
    csr = csr_of(ncells, cmap, 3, nn, rng)
    nodes = np.unique(rng.choice(np.unique(cmap), 12, replace=False)).astype(np.int32)
    rhs = rng.standard_normal(nn) if with_rhs else None
    nv = rng.standard_normal(nn) if function else None
    v1, b1 = O.apply_dirichlet(csr, rhs, nodes, nv, 1.75)
    v2, b2 = O.apply_dirichlet(csr, rhs, nodes, nv, 1.75, lib="ref")
    assert np.array_equal(v1, v2)
    if with_rhs:
        assert np.array_equal(b1, b2)
    rp, ci = csr[2], csr[3]
    for r in nodes:  # zero row, unit diagonal (assemble.hpp:60-63)
        row = slice(rp[r], rp[r + 1])
        assert np.all(v1[row][ci[row] != r] == 0.0) and v1[row][ci[row] == r][0] == 1.0


def test_missing_diagonal_is_reported_like_the_reference():  # assemble.hpp:61-62
    rp = np.array([0, 1, 2, 3], np.int64)
    ci = np.array([1, 1, 2], np.int32)  # row 0 has no (0, 0)
    csr = (3, 3, rp, ci, np.ones(3))
    with pytest.raises(O.KindError) as e1:
        O.apply_dirichlet(csr, np.zeros(3), [0])
    with pytest.raises(O.KindError) as e2:
        O.apply_dirichlet(csr, np.zeros(3), [0], lib="ref")
    assert e1.value.kind == e2.value.kind == "MissingDiagonal"
    assert "diagonal (0, 0) outside sparsity" in str(e2.value)
