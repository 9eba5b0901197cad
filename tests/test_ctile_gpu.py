"""GPU: the opt-in cell-tile kernel for P2 actions (csrc/ctile.cu,
LOAM_GPU_CTILE=1) against the oracle -- kept as a measured alternative to the
cell-centric kernel (DESIGN 15), so it must stay correct."""
import os

import numpy as np
import pytest

import oracle as O
from paper_1501_01809_b200 import capi, configs

pytestmark = pytest.mark.gpu


@pytest.fixture
def ctile():
    os.environ["LOAM_GPU_CTILE"] = "1"
    capi.set_strategy("auto")
    capi.lib().loam_gpu_plan_cache_clear()
    yield
    del os.environ["LOAM_GPU_CTILE"]
    capi.lib().loam_gpu_plan_cache_clear()


@pytest.mark.parametrize("n", [3, 9])
def test_ctile_p2_tet_residual_equals_oracle(gpu_lib, ctile, n):
    w = configs.Workload(3, n, "residual")
    w.reset()
    w.run()
    m = w.inputs
    cn, nn = m.extra["p2"], m.extra["nn"]
    ref = O.assemble_vector(O.HELMHOLTZ_ACTION, 2, 3, m.ncells, cn, 10, m.cv, m.coords, cn, 10, m.extra["u"], nn,
                            params=(configs.KAPPA,))
    got = w.outputs[0].view()
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    # accumulate: a second INC adds the same values
    from paper_1501_01809_b200 import loam as L
    L.execute(w.loops[0])
    assert np.max(np.abs(w.outputs[0].view() - 2 * ref)) <= 2e-12 * np.max(np.abs(ref))
