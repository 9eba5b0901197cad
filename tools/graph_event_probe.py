"""Developer: C2 rotation protocol with the event pair outside the graph launch
(bench.Rotation.time) and as the first / last node of the graph, for several K."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1501_01809_b200 import configs
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
w = configs.Workload(2)
w.reset(); w.run(); torch.cuda.synchronize()
rot = bench.Rotation(torch, w)
for K in (10, 20, 40, 80):
    out = [rot.time(K, st, warmup=K) for _ in range(5)]
    print("outside K", K, [round(1e3 * x, 2) for x in out], flush=True)
try:
    for K in (10, 20, 40, 80):
        e0 = torch.cuda.Event(enable_timing=True, external=True)
        e1 = torch.cuda.Event(enable_timing=True, external=True)
        g, side = torch.cuda.CUDAGraph(), torch.cuda.Stream()
        side.wait_stream(st)
        with torch.cuda.graph(g, stream=side):
            e0.record(side)
            for k in range(K):
                ww = rot.ws[k % rot.R]
                ww.reset(); ww.run()
            e1.record(side)
        st.wait_stream(side)
        torch.cuda.synchronize()
        ts = []
        for _ in range(6):
            g.replay(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / K)
        print("inside  K", K, [round(1e3 * x, 2) for x in ts[1:]], flush=True)
except Exception as exc:  # noqa: BLE001
    print("in-graph events unavailable:", repr(exc))
