"""GPU: the ring plan built on the device (plan.cu:build_ring_dev) against the
host builder (build_nbr's ring mode, LOAM_GPU_HOST_RING=1): the same chain
order, window slots and tiles, so the assembled CSR values are bitwise equal
-- and equal to the oracle."""
import os

import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs

pytestmark = pytest.mark.gpu


def assemble(cfg, n, host):
    if host:
        os.environ["LOAM_GPU_HOST_RING"] = "1"
    try:
        capi.lib().loam_gpu_plan_cache_clear()
        w = configs.Workload(cfg, n)
        w.reset()
        w.run()
        return w, w.outputs[0].host_values().copy()
    finally:
        os.environ.pop("LOAM_GPU_HOST_RING", None)
        capi.lib().loam_gpu_plan_cache_clear()


@pytest.mark.parametrize("n", [7, 40, 300])
def test_device_ring_plan_equals_host_ring_plan(gpu_lib, n):
    capi.set_strategy("auto")
    w, dev = assemble(2, n, host=False)
    _, host = assemble(2, n, host=True)
    assert dev.tobytes() == host.tobytes()
    m = w.inputs
    rp, ci = w.outputs[0].sparsity.host()
    ref = O.assemble_matrix(O.STIFFNESS, 1, 2, m.ncells, m.cv, 3, m.cv, 3, m.cv, m.coords, rp, ci)
    assert np.max(np.abs(dev - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("n", [5, 64])
def test_device_star_plan_equals_host_star_plan(gpu_lib, n):
    """C1 shape: the vertex-star records (build_stars_dev vs the host loop)."""
    capi.set_strategy("auto")

    def residual(host):
        if host:
            os.environ["LOAM_GPU_HOST_RING"] = "1"
        try:
            capi.lib().loam_gpu_plan_cache_clear()
            w = configs.Workload(1, n)
            w.reset()
            w.run()
            return w, w.outputs[0].view().copy()
        finally:
            os.environ.pop("LOAM_GPU_HOST_RING", None)
            capi.lib().loam_gpu_plan_cache_clear()

    w, dev = residual(False)
    _, host = residual(True)
    assert dev.tobytes() == host.tobytes()
    m = w.inputs
    ref = O.assemble_vector(O.HELMHOLTZ_ACTION, 1, 2, m.ncells, m.cv, 3, m.cv, m.coords, m.cv, 3, m.extra["u"], m.nv,
                            params=(configs.KAPPA,))
    assert np.max(np.abs(dev - ref)) <= 1e-12 * np.max(np.abs(ref))
