"""mesh-side builders on the device, bit-exact with the reference.

* P2 numbering (fem/space.hpp:48-72): triangles equal the compiled
  reference's make_function_space(mesh, 2) cell_node_map; tetrahedra equal
  the host restatement (the reference throws UnsupportedForm for P2 tets,
  element.hpp:179-180);
* exterior facets (mesh.hpp:48-89): equal to the reference's
  derive_exterior_facets -- order, sorted vertices, (cell, local facet)."""
import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="compiled reference (oracle/_ref) not built")


def mesh_maps(gdim, n, seed):
    m = configs.mesh(gdim, n, 0.1, seed, seed + 1)
    cells, verts = L.Set(m.ncells), L.Set(m.nv)
    return m, L.Map(cells, verts, gdim + 1, m.cv)


@needs_ref
@pytest.mark.parametrize("n", [1, 5, 24])
def test_p2_triangle_numbering_equals_reference(gpu_lib, n):
    m, cm = mesh_maps(2, n, 3)
    nodes, cn = L.p2_cell_node_map(cm, 2)
    ref, nn = O.ref_p2_tri_map(m.cv, m.coords)
    assert nodes.size == nn and np.array_equal(cn.values, ref)


@pytest.mark.parametrize("n", [1, 3, 9])
def test_p2_tet_numbering_equals_host_restatement(gpu_lib, n):
    m, cm = mesh_maps(3, n, 4)
    nodes, cn = L.p2_cell_node_map(cm, 3)
    host, nn = configs.p2_map(m)
    assert nodes.size == nn == (2 * n + 1) ** 3 and np.array_equal(cn.values, host)


@needs_ref
@pytest.mark.parametrize("gdim,n", [(2, 1), (2, 7), (3, 1), (3, 4)])
def test_exterior_facets_equal_reference(gpu_lib, gdim, n):
    m, cm = mesh_maps(gdim, n, 5)
    fv, fc = L.exterior_facets(cm, gdim)
    rv, rc = O.ref_exterior_facets(gdim, m.cv, m.nv)
    assert np.array_equal(fv, rv) and np.array_equal(fc, rc)
    assert len(fv) == (4 * n if gdim == 2 else 12 * n * n)  # boundary facet count of the unit square / cube


def test_non_manifold_facet_is_an_error(gpu_lib):  # mesh.hpp:59-60
    cv = np.array([0, 1, 2, 0, 1, 3, 0, 1, 4], np.int32)  # edge (0,1) in three triangles
    cm = L.Map(L.Set(3), L.Set(5), 3, cv)
    with pytest.raises(capi.LoamError) as e:
        L.exterior_facets(cm, 2)
    assert e.value.kind == "NonManifold"
