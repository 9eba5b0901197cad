"""vertex renumbering on the device (order.cu), bit-exact.

* rcm_order (topology.hpp:131-178): the reference's known answers, its error
  kinds at the first offending entry, seeded random graphs (self entries,
  duplicates, isolated vertices, many components) against the restatement;
* vertex_adjacency (mesh.hpp:350-362) against the host restatement;
* reorder (mesh.hpp:364-396): the golden fixture of the reference, the strip
  of test_mesh.cpp:171-215 (bandwidth <= 3, coordinates follow perm), and
  the config-sized meshes against the restatement.
"""
import os

import numpy as np
import pytest
import torch

import oracle as O
from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L

from .test_rcm_cpu import random_graph

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "rcm.npz")


def dev_rcm(adj):
    rp, ci = adj if isinstance(adj, tuple) else O._csr_of_lists(adj)
    return L.rcm_order(rp.size - 1, rp, ci).cpu().numpy()


def test_rcm_kats(gpu_lib):  # test_topology.cpp
    assert dev_rcm([[1], [0, 2], [1]]).tolist() == [2, 1, 0]
    assert dev_rcm([[]]).tolist() == [0]
    assert dev_rcm([[1, 2, 3], [0], [0], [0]]).tolist() == [3, 2, 0, 1]
    assert dev_rcm([]).tolist() == []


@pytest.mark.parametrize("adj,kind", [
    ([[1], []], "AsymmetricAdjacency"),
    ([[3], [0]], "IndexOutOfRange"),
    ([[1], [], [7]], "AsymmetricAdjacency"),   # the asymmetric entry comes first
    ([[5], [2], [0]], "IndexOutOfRange"),      # the out-of-range entry comes first
])
def test_rcm_errors_first_entry(gpu_lib, adj, kind):
    with pytest.raises(O.KindError) as r:
        O.rcm_order(adj)
    assert r.value.kind == kind
    with pytest.raises(capi.LoamError) as e:
        dev_rcm(adj)
    assert e.value.kind == kind


@pytest.mark.parametrize("seed", range(8))
def test_rcm_random_graphs_equal_restatement(gpu_lib, seed):
    n = [50, 300, 1000, 5000, 64, 2000, 777, 20000][seed]
    m = [60, 500, 900, 20000, 10, 1500, 3000, 60000][seed]
    adj = random_graph(n, m, 100 + seed, self_loops=seed % 2 == 1, dups=seed % 3 == 2)
    assert np.array_equal(dev_rcm(adj), O.rcm_order(adj))


def test_rcm_many_components_and_isolated(gpu_lib):
    adj = [[] for _ in range(30)]
    for a in range(0, 24, 3):  # 8 paths of 3, 6 isolated vertices
        adj[a] += [a + 1]
        adj[a + 1] += [a, a + 2]
        adj[a + 2] += [a + 1]
    assert np.array_equal(dev_rcm(adj), O.rcm_order(adj))


def test_rcm_golden_graphs(gpu_lib):
    d = np.load(GOLD)
    for k in range(3):
        assert np.array_equal(dev_rcm((d[f"g{k}_row_ptr"], d[f"g{k}_col_idx"])), d[f"g{k}_order"])


@pytest.mark.parametrize("gdim,n", [(2, 1), (2, 9), (3, 2), (3, 5)])
def test_vertex_adjacency_equals_restatement(gpu_lib, gdim, n):
    m = configs.mesh(gdim, n, 0.1, 3, 4)
    cm = L.Map(L.Set(m.ncells), L.Set(m.nv), gdim + 1, m.cv)
    rp, ci = L.vertex_adjacency(cm, gdim)
    hrp, hci = O.vertex_adjacency(m.cv, m.nv, gdim)
    assert np.array_equal(rp.cpu().numpy(), hrp) and np.array_equal(ci.cpu().numpy(), hci)


def reorder_dev(gdim, cv, coords):
    nv = coords.size // gdim
    cm = L.Map(L.Set(cv.size // (gdim + 1)), L.Set(nv, "vertices"), gdim + 1, cv, "cell_vertex")
    X = L.Dat(cm.target, gdim, "coordinates")
    X.set_values(coords)
    m2, X2, perm = L.reorder(cm, X)
    return perm, X2.view(), m2.values


@pytest.mark.parametrize("tag,gdim", [("sq", 2), ("cube", 3)])
def test_reorder_equals_reference_fixture(gpu_lib, tag, gdim):
    d = np.load(GOLD)
    perm, x, cv = reorder_dev(gdim, d[f"{tag}_cv"], d[f"{tag}_coords"])
    assert np.array_equal(perm, d[f"{tag}_perm"])
    assert np.array_equal(x, d[f"{tag}_coords_out"]) and np.array_equal(cv, d[f"{tag}_cv_out"])


def bandwidth(cv, gdim):
    c = cv.reshape(-1, gdim + 1)
    return int(max(np.max(c, axis=1) - np.min(c, axis=1)))


def test_reorder_strip_bandwidth(gpu_lib):  # test_mesh.cpp:171-215
    n = 12
    coords = np.array([(i, 0) for i in range(n + 1)] + [(i, 1) for i in range(n + 1)], np.float64).ravel()
    cv = []
    for i in range(n):
        a, b, c, d = i, i + 1, n + 2 + i, n + 1 + i
        cv += [a, b, c, a, c, d]
    cv = np.array(cv, np.int32)
    perm, x, cv2 = reorder_dev(2, cv, coords)
    assert bandwidth(cv2, 2) <= min(3, bandwidth(cv, 2))
    assert sorted(perm.tolist()) == list(range(2 * (n + 1)))
    assert np.array_equal(x.reshape(-1, 2), coords.reshape(-1, 2)[perm])
    fv, fc = L.exterior_facets(L.Map(L.Set(2 * n), L.Set(2 * (n + 1)), 3, cv2), 2)
    fv0, fc0 = L.exterior_facets(L.Map(L.Set(2 * n), L.Set(2 * (n + 1)), 3, cv), 2)
    assert np.array_equal(fc, fc0)  # facet order survives the renumbering (mesh.hpp:388-393)


@pytest.mark.parametrize("gdim,n", [(2, 256), (3, 24)])
def test_reorder_config_meshes_equal_restatement(gpu_lib, gdim, n):
    m = configs.mesh(gdim, n, 0.1, 5, 6)  # cell order permuted: a badly numbered mesh
    perm, x, cv = reorder_dev(gdim, m.cv, m.coords)
    ref = O.rcm_order(O.vertex_adjacency(m.cv, m.nv, gdim))
    assert np.array_equal(perm, ref)
    new_of = np.empty(m.nv, np.int32)
    new_of[ref] = np.arange(m.nv, dtype=np.int32)
    assert np.array_equal(cv, new_of[m.cv])
    assert np.array_equal(x, m.coords.reshape(-1, gdim)[ref].ravel())


@pytest.mark.parametrize("rp,ci", [
    ([0, 1], [0, 0]),            # n + 1 offsets expected, n = 2
    ([0, 2, 1], [1, 0]),         # decreasing offsets
    ([1, 1, 2], [1, 0]),         # offsets do not start at 0
    ([0, 1, 5], [1, 0]),         # offsets past the column array
])
def test_rcm_rejects_malformed_lists(gpu_lib, rp, ci):
    """A malformed CSR is InvalidArgument ('adjacency list count != n' in the
    reference), never an out-of-bounds read."""
    with pytest.raises(capi.LoamError) as e:
        L.rcm_order(2, np.asarray(rp, np.int64), np.asarray(ci, np.int32))
    assert e.value.kind == "InvalidArgument"
    # the context is still usable
    assert np.array_equal(dev_rcm([[1], [0]]), O.rcm_order([[1], [0]]))
