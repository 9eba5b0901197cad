"""CUDA-graph capture of assembly loops: a captured execute replayed any
number of times recomputes the same values (the persistent tile kernels'
tile counters are reset by the last CTA of each launch, so a replay with
frozen arguments starts from tile 0).  The output is poisoned with NaN
before each replay, so a replay that skipped work would fail."""
import numpy as np
import pytest
import torch

from paper_1501_01809_b200 import capi, configs
from paper_1501_01809_b200 import loam as L

pytestmark = pytest.mark.gpu


def values(o):
    return o.host_values() if isinstance(o, L.Mat) else o.view().copy()


def raw(o):
    return o.values if isinstance(o, L.Mat) else o.data


@pytest.mark.parametrize("cfg,n,part", [(1, 40, None), (2, 40, None), (3, 5, "matrix"), (3, 5, "residual"),
                                        (4, 5, None), (5, 12, None)])
def test_replayed_assembly_recomputes(gpu_lib, cfg, n, part):
    capi.set_strategy("auto")
    w = configs.Workload(cfg, n, part)
    w.reset()
    w.run()
    torch.cuda.synchronize()
    ref = [values(o) for o in w.outputs]
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    w.reset()
    with torch.cuda.graph(g, stream=side):
        w.run()
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(3):
        for o in w.outputs:
            raw(o).fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        for o, r in zip(w.outputs, ref):
            got = values(o)
            assert np.all(np.isfinite(got)), "a replay skipped work"
            assert np.max(np.abs(got - r)) <= 1e-12 * np.max(np.abs(r))
