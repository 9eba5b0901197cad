"""Developer: the flushed single-step protocol for a direct launch vs a CUDA
graph replay of the same captured step (C1, C2) and an empty kernel."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1501_01809_b200 import configs
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
flush = bench.Flusher(torch)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n=20):
    ts = []
    for _ in range(n):
        flush()
        e0.record(st); fn(); e1.record(st); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts[3:]))


o = torch.zeros(1, dtype=torch.float64, device="cuda")
g0 = torch.cuda.CUDAGraph()
s = torch.cuda.Stream(); s.wait_stream(st)
with torch.cuda.graph(g0, stream=s):
    o.fill_(1.0)
st.wait_stream(s)
print("empty: direct", timed(lambda: o.fill_(1.0)), "graph", timed(g0.replay))
for cfg in (1, 2):
    w = configs.Workload(cfg, None)
    w.reset(); w.run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(); s.wait_stream(st)
    w.reset()
    with torch.cuda.graph(g, stream=s):
        w.run()
    st.wait_stream(s)
    torch.cuda.synchronize()

    def direct():
        w.reset(); w.run()
    print(f"C{cfg}: direct us", timed(direct), "graph us", timed(g.replay), flush=True)
    # parity of the graph-replayed result with the direct one
    g.replay(); torch.cuda.synchronize()
    a = w.outputs[0].host_values() if hasattr(w.outputs[0], "host_values") else w.outputs[0].view().copy()
    direct(); torch.cuda.synchronize()
    b = w.outputs[0].host_values() if hasattr(w.outputs[0], "host_values") else w.outputs[0].view().copy()
    print("  replay == direct:", bool(np.array_equal(a, b)))
