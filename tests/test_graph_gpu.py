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


@pytest.mark.parametrize("cfg,n,part", [(2, 64, None), (3, 6, "matrix"), (4, 6, None), (5, 16, None)])
def test_concurrent_launches_of_one_plan(gpu_lib, cfg, n, part):
    """Two executes of ONE cached plan in flight together (two streams, and a
    graph replay beside a direct execute) must each get their own tile
    counters: both outputs complete and equal (a shared counter
    split one tile sequence between two launches)."""
    capi.set_strategy("auto")
    w = configs.Workload(cfg, n, part)
    w.reset()
    w.run()
    torch.cuda.synchronize()
    firsts = [lp.args[0].mat if lp.args[0].mat is not None else lp.args[0].dat for lp in w.loops]
    ref = [values(o) for o in firsts]  # in loop order (C5 lists its outputs as BlockMat slots)
    # a second set of outputs over the same maps / sparsities -> same cached plans
    outs2 = [L.Mat(lp.args[0].mat.sparsity) if lp.args[0].mat is not None
             else L.Dat(lp.args[0].dat.set, lp.args[0].dat.dim) for lp in w.loops]
    loops2 = []
    for lp, out in zip(w.loops, outs2):
        a0 = lp.args[0]
        new0 = L.arg(out, a0.access, *a0.maps)
        loops2.append(L.Parloop(lp.kernel, lp.iterset, [new0] + list(lp.args[1:])))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for _ in range(8):
        for o in w.outputs + outs2:
            raw(o).fill_(float("nan"))
            o.zero()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            w.run()
        with torch.cuda.stream(s2):
            for lp in loops2:
                L.execute(lp)
        torch.cuda.synchronize()
        for o, r in zip(firsts + outs2, ref + ref):
            got = values(o)
            assert np.all(np.isfinite(got)), "a launch lost tiles to a concurrent one"
            assert np.max(np.abs(got - r)) <= 1e-12 * np.max(np.abs(r))
    # a captured replay on one stream beside direct executes on another
    g = torch.cuda.CUDAGraph()
    w.reset()
    with torch.cuda.graph(g, stream=s1):
        w.run()
    for _ in range(4):
        for o in w.outputs + outs2:
            raw(o).fill_(float("nan"))
        for o in outs2:
            o.zero()
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            g.replay()
        with torch.cuda.stream(s2):
            for lp in loops2:
                L.execute(lp)
        torch.cuda.synchronize()
        for o, r in zip(firsts + outs2, ref + ref):
            got = values(o)
            assert np.all(np.isfinite(got))
            assert np.max(np.abs(got - r)) <= 1e-12 * np.max(np.abs(r))
