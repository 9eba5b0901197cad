"""Developer probe: per-step assembly time under two protocols.
  flushed: L2 flushed before every step, events around ONE launch;
  b2b:     R independent replicas (every object distinct: maps, plans,
           coordinates, outputs), one CUDA graph per replica, K graph replays
           back to back cycling the replicas (aggregate working set >> L2, so
           every step starts from its own cold data), events around all K."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1501_01809_b200 import capi, configs  # noqa: E402

capi.set_strategy("auto")
flush = bench.Flusher(torch)
stream = torch.cuda.current_stream()
want = sys.argv[1:] or ["1", "2", "3r", "3m", "4", "5"]
for c in want:
    cfg = int(c[0])
    part = {"r": "residual", "m": "matrix"}.get(c[1:], None)
    m = configs.config_inputs(cfg)
    w0 = configs.Workload(cfg, None, part, inputs=m)
    w0.reset(); w0.run(); torch.cuda.synchronize()
    ab = bench.algorithmic_bytes(w0)
    R = max(2, min(24, int(np.ceil(3 * 126e6 / ab)) + 1))
    ws = [w0] + [configs.Workload(cfg, None, part, inputs=m) for _ in range(R - 1)]
    for w in ws:
        w.reset(); w.run()
    torch.cuda.synchronize()
    fl = bench.time_steps(torch, w0, 10, flush, stream)
    graphs, side = [], torch.cuda.Stream()
    for w in ws:
        g = torch.cuda.CUDAGraph()
        side.wait_stream(stream)
        w.reset()
        with torch.cuda.graph(g, stream=side):
            w.run()
        stream.wait_stream(side)
        graphs.append(g)
    K = max(40, 4 * R)
    for k in range(2 * R):
        graphs[k % R].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = []
    for rep in range(3):
        e0.record(stream)
        for k in range(K):
            graphs[k % R].replay()
        e1.record(stream)
        e1.synchronize()
        res.append(e0.elapsed_time(e1) / K)
    # same buffers back to back (L2-warm; NOT a valid protocol, for scale only)
    e0.record(stream)
    for k in range(K):
        graphs[0].replay()
    e1.record(stream)
    e1.synchronize()
    warm = e0.elapsed_time(e1) / K
    peak = 6551.7
    f = lambda ms: ab / (ms * 1e-3) / 1e9 / peak
    print(f"config {c}: bytes {ab/1e6:.1f} MB R={R}  flushed {np.median(fl)*1e3:.1f} us ({f(np.median(fl)):.3f})  "
          f"b2b {min(res)*1e3:.1f} us ({f(min(res)):.3f}) [{', '.join(f'{x*1e3:.1f}' for x in res)}]  "
          f"warm-same {warm*1e3:.1f} us", flush=True)
    del ws, graphs, w0
    torch.cuda.empty_cache()
