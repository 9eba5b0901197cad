"""GPU: loam_gpu_execute_host -- the reference's host-memory calling
convention (parloop.hpp:191: execute reads and writes host buffers), which
the bench's e2e number goes through.

* host-convention results equal the device-convention results and the oracle;
* repeated calls reuse the resident Map / Sparsity copies (immutable objects,
  topology.hpp:68, data.hpp:116-179) and give identical results;
* after loam_gpu_plan_cache_clear the objects are re-uploaded;
* anonymous objects (id 0) are copied per call.
"""
import ctypes as C

import numpy as np
import pytest

from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def device_outputs(w):
    w.reset()
    w.run()
    return [o.host_values() if isinstance(o, L.Mat) else o.view().copy() for o in w.outputs]


def loop_output(lp):
    a = lp.args[0]
    return a.mat if a.mat is not None else a.dat


@pytest.mark.parametrize("cfg,n", [(1, 24), (2, 24), (3, 4), (4, 4), (5, 6)])
def test_host_convention_equals_device_convention(gpu_lib, cfg, n):
    w = configs.Workload(cfg, n)
    dev = dict(zip(map(id, w.outputs), device_outputs(w)))
    w.reset()
    hls = [L.HostLoop(lp) for lp in w.loops]
    for h in hls:
        h.run()
    assert len(hls) == len(dev)
    for h in hls:
        d = dev[id(loop_output(h.loop))]
        assert rel(h.outputs[0].numpy()[: len(d)], d) <= TOL


def test_resident_objects_are_reused_and_refreshed(gpu_lib):
    w = configs.Workload(2, 20)
    ref = device_outputs(w)[0]
    w.reset()
    h = L.HostLoop(w.loops[0])
    h.run()
    first = h.outputs[0].numpy().copy()
    assert rel(first[: len(ref)], ref) <= TOL
    h.outputs[0].zero_()
    h.run()  # resident maps / sparsity
    assert np.array_equal(h.outputs[0].numpy(), first)
    capi.check(capi.lib().loam_gpu_plan_cache_clear())
    h.outputs[0].zero_()
    h.run()  # re-uploaded
    assert np.array_equal(h.outputs[0].numpy(), first)


def test_anonymous_objects_are_copied_per_call(gpu_lib):
    w = configs.Workload(1, 16)
    ref = device_outputs(w)[0]
    w.reset()
    h = L.HostLoop(w.loops[0])
    for k in range(len(w.loops[0].args)):
        d = h.descs[k]
        if d.map:
            d.map.contents.id = 0  # no identity: never cached
    h.run()
    assert rel(h.outputs[0].numpy()[: len(ref)], ref) <= TOL


def test_host_byte_accounting_is_per_step_dats_only(gpu_lib):
    w = configs.Workload(2, 16)
    w.reset()
    h = L.HostLoop(w.loops[0])
    m = configs.config_inputs(2, 16)
    assert h.h2d_bytes == m.coords.size * 8                       # coordinates (READ Dat)
    assert h.d2h_bytes == w.outputs[0].sparsity.nnz * 8          # the assembled values


@pytest.mark.parametrize("cfg,n", [(1, 24), (2, 24), (3, 4), (4, 4), (5, 6)])
def test_batched_host_convention(gpu_lib, cfg, n):
    """loam_gpu_execute_host_batch: K steps over two alternating host buffer
    sets, copies pipelined across steps; both sets end with the
    device-convention result."""
    w = configs.Workload(cfg, n)
    dev = dict(zip(map(id, w.outputs), device_outputs(w)))
    w.reset()
    hls = [L.HostLoop(lp) for lp in w.loops]
    for h in hls:
        alt, outs = h.step_buffers()
        h.run_batch([h.descs, alt, h.descs, alt, h.descs])
        d = dev[id(loop_output(h.loop))]
        assert rel(h.outputs[0].numpy()[: len(d)], d) <= TOL
        assert rel(outs[0].numpy()[: len(d)], d) <= TOL


def test_batched_steps_upload_their_own_inputs(gpu_lib):
    w = configs.Workload(1, 20)  # P1 Helmholtz residual: linear in the coefficient u
    ref = device_outputs(w)[0]
    w.reset()
    h = L.HostLoop(w.loops[0])
    alt, outs = h.step_buffers()
    # the alternate set's coefficient is 3u: its residual is 3x (the action is linear in u)
    u_idx = 2
    k = w.loops[0].args[u_idx].dat
    nbytes = k.set.size * 8
    host_u = np.ctypeslib.as_array(C.cast(alt[u_idx].data, C.POINTER(C.c_double)), shape=(k.set.size,))
    host_u *= 3.0
    h.run_batch([h.descs, alt, h.descs, alt])
    assert rel(h.outputs[0].numpy()[: len(ref)], ref) <= TOL
    assert rel(outs[0].numpy()[: len(ref)], 3.0 * ref) <= TOL
    assert nbytes > 0
