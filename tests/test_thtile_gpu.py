"""The fused Taylor-Hood launch (loam_gpu_execute_blocks, csrc/thtile.cu).

fem::assemble_blocks (fem/assemble.hpp:439-448) assembles A, B and B^T with
one par_loop each; loam_gpu_execute_blocks takes the three loops together and
runs them as one launch.  Parity: every block equals the oracle's par_loop
(relative max norm 1e-12, the tolerance of the north star) and the three
separate loops; one kernel launch per call; accumulation into existing values
(per block); bitwise repeatability; meshes and patterns the fused plan must
decline (a duplicated cell, a sub-mesh loop into whole-mesh patterns, a
renumbered pressure space) fall back to the separate loops with the same
results; validation errors of any loop surface before anything is written.
"""
import os

import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den else 1.0)


@pytest.fixture(autouse=True)
def _reset(gpu_lib):
    capi.set_strategy("auto")
    os.environ.pop("LOAM_GPU_NO_THTILE", None)
    yield
    os.environ.pop("LOAM_GPU_NO_THTILE", None)
    capi.set_strategy("auto")


def oracle_blocks(m, cv=None, cn=None, ncells=None):
    """(A, B^T, B) values of the oracle on the patterns of the oracle."""
    cv = m.cv if cv is None else cv
    cn = m.extra["p2"] if cn is None else cn
    nc = m.ncells if ncells is None else ncells
    nn = m.extra["nn"]
    vd = np.empty(nc * 12, dtype=np.int32)
    vd[0::2] = 2 * np.asarray(cn)
    vd[1::2] = 2 * np.asarray(cn) + 1
    rpA, ciA = O.build_sparsity(nc, cn, 6, nn, cn, 6, nn, 2, 2)
    rpB, ciB = O.build_sparsity(nc, cv, 3, m.nv, cn, 6, nn, 1, 2)
    rpT, ciT = O.build_sparsity(nc, cn, 6, nn, cv, 3, m.nv, 2, 1)
    A = O.assemble_matrix(O.STOKES_A, 2, 2, nc, vd, 12, vd, 12, cv, m.coords, rpA, ciA, params=(configs.NU,))
    B = O.assemble_matrix(O.STOKES_B, 2, 2, nc, cv, 3, vd, 12, cv, m.coords, rpB, ciB)
    T = O.assemble_matrix(O.STOKES_BT, 2, 2, nc, vd, 12, cv, 3, cv, m.coords, rpT, ciT)
    return A, T, B


@pytest.mark.parametrize("n", [1, 2, 5, 17, 48])
def test_fused_blocks_match_oracle_and_separate_loops(n):
    w = configs.Workload(5, n)
    w.reset()
    before = capi.launch_count()
    w.run()  # first call: plan + launch
    w.reset()
    before = capi.launch_count()
    w.run()
    assert capi.launch_count() - before == 1, "the three blocks must be one launch"
    fused = [o.host_values().copy() for o in w.outputs]
    for got, ref in zip(fused, oracle_blocks(w.inputs)):
        assert rel(got, ref) <= TOL
    os.environ["LOAM_GPU_NO_THTILE"] = "1"
    w.reset()
    before = capi.launch_count()
    w.run()
    assert capi.launch_count() - before >= 3
    for got, sep in zip(fused, [o.host_values() for o in w.outputs]):
        assert rel(got, sep) <= TOL


def test_fused_blocks_are_bitwise_repeatable():
    w = configs.Workload(5, 24)
    runs = []
    for _ in range(3):
        w.reset()
        w.run()
        runs.append([o.host_values().copy() for o in w.outputs])
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert np.array_equal(a, b)


def test_fused_blocks_accumulate_per_block():
    """INC adds to what is there (parloop.hpp:301-305): all three blocks, and a
    mix of fresh and used blocks in one call."""
    w = configs.Workload(5, 9)
    w.reset()
    w.run()
    once = [o.host_values().copy() for o in w.outputs]
    w.run()
    for o, ref in zip(w.outputs, once):
        assert rel(o.host_values(), 2 * ref) <= TOL
    w.outputs[2].zero()  # B fresh again, A and B^T keep 2x
    w.run()
    for o, ref, f in zip(w.outputs, once, (3, 3, 1)):
        assert rel(o.host_values(), f * ref) <= TOL


def test_loops_in_any_order_and_other_lists_run_in_sequence():
    w = configs.Workload(5, 7)
    ref = oracle_blocks(w.inputs)
    w.reset()
    L.execute_blocks([w.loops[2], w.loops[0], w.loops[1]])
    for o, r in zip(w.outputs, ref):
        assert rel(o.host_values(), r) <= TOL
    # a pair of loops is not the triple: the loops run one by one
    w.reset()
    L.execute_blocks(w.loops[:2])
    assert rel(w.outputs[0].host_values(), ref[0]) <= TOL
    assert rel(w.outputs[2].host_values(), ref[2]) <= TOL
    assert not np.any(w.outputs[1].host_values())
    L.execute_blocks([])


def _blocks(m, cv, cn, nc, full=None):
    """Taylor-Hood loops over `nc` cells; patterns from `full` = (cv, cn, ncells) when given."""
    cells = L.Set(nc)
    verts, nodes = L.Set(m.nv), L.Set(m.extra["nn"])
    cvm = L.Map(cells, verts, 3, cv)
    vnm = L.Map(cells, nodes, 6, cn)
    vdm = L.expanded_map(vnm, 2)
    if full is None:
        pv, pn = cvm, vnm
    else:
        fcells = L.Set(full[2])
        pv, pn = L.Map(fcells, verts, 3, full[0]), L.Map(fcells, nodes, 6, full[1])
    X = L.Dat(verts, 2)
    X.set_values(m.coords)
    A = L.Mat(L.build_sparsity(pn, pn, 2, 2))
    B = L.Mat(L.build_sparsity(pv, pn, 1, 2))
    T = L.Mat(L.build_sparsity(pn, pv, 2, 1))
    loops = [L.Parloop(L.kernel("stokes_a_p2_tri", configs.NU), cells, [L.arg(A, L.INC, vdm, vdm), L.arg(X, L.READ, cvm)]),
             L.Parloop(L.kernel("stokes_b_p2_tri"), cells, [L.arg(B, L.INC, cvm, vdm), L.arg(X, L.READ, cvm)]),
             L.Parloop(L.kernel("stokes_bt_p2_tri"), cells, [L.arg(T, L.INC, vdm, cvm), L.arg(X, L.READ, cvm)])]
    return loops, (A, T, B)


def test_duplicated_cell_declines_the_fused_plan():
    """A cell listed twice: edges with three cells, stars that are no ring --
    the fused plan must decline and the separate loops still match the oracle."""
    m = configs.config_inputs(5, 8)
    cv = np.concatenate([m.cv, m.cv[: 3 * 4]])
    cn = np.concatenate([m.extra["p2"], m.extra["p2"][: 6 * 4]])
    nc = m.ncells + 4
    loops, outs = _blocks(m, cv, cn, nc)
    before = capi.launch_count()
    L.execute_blocks(loops)
    for o, r in zip(outs, oracle_blocks(m, cv, cn, nc)):
        assert rel(o.host_values(), r) <= TOL
    for o in outs:
        o.zero()
    before = capi.launch_count()
    L.execute_blocks(loops)
    assert capi.launch_count() - before >= 3


def test_submesh_loops_into_whole_mesh_patterns():
    """A sub-mesh triple into whole-mesh patterns (legal: parloop.hpp:119-121):
    entries outside the sub-mesh stay zero (data.hpp:185-187)."""
    m = configs.config_inputs(5, 10)
    sel = np.sort(np.random.default_rng(5).permutation(m.ncells)[: m.ncells // 2])
    cv = np.ascontiguousarray(m.cv.reshape(-1, 3)[sel].reshape(-1))
    cn = np.ascontiguousarray(m.extra["p2"].reshape(-1, 6)[sel].reshape(-1))
    loops, outs = _blocks(m, cv, cn, sel.size, full=(m.cv, m.extra["p2"], m.ncells))
    L.execute_blocks(loops)
    nn = m.extra["nn"]
    vd = np.empty(sel.size * 12, dtype=np.int32)
    vd[0::2], vd[1::2] = 2 * cn, 2 * cn + 1
    rpA, ciA = outs[0].sparsity.host()
    rpT, ciT = outs[1].sparsity.host()
    rpB, ciB = outs[2].sparsity.host()
    refA = O.assemble_matrix(O.STOKES_A, 2, 2, sel.size, vd, 12, vd, 12, cv, m.coords, rpA, ciA, params=(configs.NU,))
    refB = O.assemble_matrix(O.STOKES_B, 2, 2, sel.size, cv, 3, vd, 12, cv, m.coords, rpB, ciB)
    refT = O.assemble_matrix(O.STOKES_BT, 2, 2, sel.size, vd, 12, cv, 3, cv, m.coords, rpT, ciT)
    for o, r in zip(outs, (refA, refT, refB)):
        assert rel(o.host_values(), r) <= TOL


def test_submesh_with_its_own_patterns_runs_fused():
    """An L-shaped region with holes in its boundary stars: fans, not rings."""
    m = configs.config_inputs(5, 12)
    cx = m.coords.reshape(-1, 2)[m.cv.reshape(-1, 3)].mean(axis=1)
    sel = np.nonzero((cx[:, 0] < 0.5) | (cx[:, 1] < 0.4))[0]
    cv = np.ascontiguousarray(m.cv.reshape(-1, 3)[sel].reshape(-1))
    cn = np.ascontiguousarray(m.extra["p2"].reshape(-1, 6)[sel].reshape(-1))
    loops, outs = _blocks(m, cv, cn, sel.size)
    L.execute_blocks(loops)
    for o in outs:
        o.zero()
    before = capi.launch_count()
    L.execute_blocks(loops)
    launches = capi.launch_count() - before
    nn = m.extra["nn"]
    vd = np.empty(sel.size * 12, dtype=np.int32)
    vd[0::2], vd[1::2] = 2 * cn, 2 * cn + 1
    refs = []
    for o, (kind, rm, ra, cm, ca) in zip(outs, ((O.STOKES_A, vd, 12, vd, 12), (O.STOKES_BT, vd, 12, cv, 3),
                                                   (O.STOKES_B, cv, 3, vd, 12))):
        rp, ci = o.sparsity.host()
        prm = (configs.NU,) if kind == O.STOKES_A else ()
        refs.append(O.assemble_matrix(kind, 2, 2, sel.size, rm, ra, cm, ca, cv, m.coords, rp, ci, params=prm))
    for o, r in zip(outs, refs):
        assert rel(o.host_values(), r) <= TOL
    # unused vertices / nodes of the whole mesh have empty rows: still one launch
    assert launches == 1


def test_validation_errors_come_before_any_write():
    w = configs.Workload(5, 4)
    w.reset()
    w.run()
    keep = [o.host_values().copy() for o in w.outputs]
    bad = L.Parloop(L.kernel("stokes_bt_p2_tri"), w.cells,
                    [L.arg(w.outputs[1], L.INC, w.vdm, w.vdm), L.arg(w.X, L.READ, w.cvm)])  # wrong column map
    with pytest.raises(capi.LoamError):
        L.execute_blocks([w.loops[0], w.loops[1], bad])
    for o, k in zip(w.outputs, keep):
        assert np.array_equal(o.host_values(), k)


def test_host_convention_blocks_run_fused_and_match():
    """loam_gpu_execute_blocks_host: host buffers in, host buffers out, the
    triple still one launch (the loops share the coordinates' host array)."""
    w = configs.Workload(5, 11)
    refs = dict(zip(map(id, w.outputs), oracle_blocks(w.inputs)))
    w.reset()
    shared = {}
    hls = [L.HostLoop(lp, mirrors=shared) for lp in w.loops]
    L.run_host_blocks(hls)  # plan
    before = capi.launch_count()
    L.run_host_blocks(hls)
    assert capi.launch_count() - before == 1
    for h in hls:
        ref = refs[id(h.loop.args[0].mat)]
        assert rel(h.outputs[0].numpy()[: len(ref)], ref) <= TOL
    # separate mirrors: the loops no longer share the coordinate array -> loop by loop, same values
    hl2 = [L.HostLoop(lp) for lp in w.loops]
    L.run_host_blocks(hl2)
    for h in hl2:
        ref = refs[id(h.loop.args[0].mat)]
        assert rel(h.outputs[0].numpy()[: len(ref)], ref) <= TOL


@pytest.mark.parametrize("K", [3, 7, 40, 70])
def test_high_valence_star_meshes(K):
    """A star of K triangles around one vertex plus an outer ring (the meshes of
    test_irregular_gpu): the centre vertex has K spokes -- one vertex fills a
    tile at K = 40, and at K = 70 the star exceeds the walk's capacity, the
    plan declines and the separate loops run.  All against the oracle."""
    from tests.test_irregular_gpu import star2d
    m = star2d(K)
    cn, nn = configs.p2_map(m)
    m.extra["p2"], m.extra["nn"] = cn, nn
    loops, outs = _blocks(m, m.cv, cn, m.ncells)
    L.execute_blocks(loops)
    for o in outs:
        o.zero()
    before = capi.launch_count()
    L.execute_blocks(loops)
    launches = capi.launch_count() - before
    assert launches == 1 if K <= 40 else launches >= 3
    for o, r in zip(outs, oracle_blocks(m, m.cv, cn, m.ncells)):
        assert rel(o.host_values(), r) <= TOL
