"""SURVEY 8f-4 (vertex renumbering): pins the RCM restatement
(oracle orc_rcm_order) before it checks the device.

1. the reference's known answers (test_topology.cpp: path, singleton, star,
   asymmetric adjacency; a bijection on a random graph, two components);
2. the golden fixture tests/golden/rcm.npz (reference rcm_order / reorder,
   tools/make_golden.py rcm_fixture);
3. the compiled reference itself on seeded random graphs (when oracle/_ref is
   built, i.e. in the build container).
"""
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "rcm.npz")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="compiled reference (oracle/_ref) not built")


def random_graph(n, m, seed, self_loops=False, dups=False):
    rng = np.random.default_rng(seed)
    adj = [[] for _ in range(n)]
    for _ in range(m):
        a, b = (int(x) for x in rng.integers(0, n, 2))
        if a == b and not self_loops:
            continue
        if b in adj[a] and not dups:
            continue
        adj[a].append(b)
        if a != b:
            adj[b].append(a)
    for a in adj:
        rng.shuffle(a)
    return adj


def test_rcm_kats():  # test_topology.cpp rcm cases
    assert O.rcm_order([[1], [0, 2], [1]]).tolist() == [2, 1, 0]
    assert O.rcm_order([[]]).tolist() == [0]
    assert O.rcm_order([[1, 2, 3], [0], [0], [0]]).tolist() == [3, 2, 0, 1]
    assert O.rcm_order([]).tolist() == []


def test_rcm_errors():
    with pytest.raises(O.KindError) as e:
        O.rcm_order([[1], []])
    assert e.value.kind == "AsymmetricAdjacency"
    with pytest.raises(O.KindError) as e:
        O.rcm_order([[3], [0]])
    assert e.value.kind == "IndexOutOfRange"


def test_rcm_bijection_and_components():
    adj = random_graph(300, 400, 11)
    r = O.rcm_order(adj)
    assert sorted(r.tolist()) == list(range(300))
    # two components: 0-1-2 and 3-4; the second seed is the min-degree vertex left
    r = O.rcm_order([[1], [0, 2], [1], [4], [3]])
    assert sorted(r.tolist()) == [0, 1, 2, 3, 4]
    assert r.tolist()[::-1][:3] == [0, 1, 2]


def test_rcm_golden_fixture():
    d = np.load(GOLD)
    for k in range(3):
        got = O.rcm_order((d[f"g{k}_row_ptr"], d[f"g{k}_col_idx"]))
        assert np.array_equal(got, d[f"g{k}_order"])
    for tag, gdim in (("sq", 2), ("cube", 3)):
        cv = d[f"{tag}_cv"]
        nv = d[f"{tag}_coords"].size // gdim
        perm = O.rcm_order(O.vertex_adjacency(cv, nv, gdim))
        assert np.array_equal(perm, d[f"{tag}_perm"])
        new_of = np.empty(nv, np.int32)
        new_of[perm] = np.arange(nv, dtype=np.int32)
        assert np.array_equal(new_of[cv], d[f"{tag}_cv_out"])
        assert np.array_equal(d[f"{tag}_coords"].reshape(nv, gdim)[perm].ravel(), d[f"{tag}_coords_out"])


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_rcm_restatement_equals_reference(seed):
    adj = random_graph(120 + 40 * seed, 150 + 60 * seed, seed, self_loops=seed % 2 == 1, dups=seed % 3 == 2)
    assert np.array_equal(O.rcm_order(adj), O.rcm_order(adj, lib="ref"))
