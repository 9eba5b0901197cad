"""Developer: per-loop device time of config 5 (A, B, B^T) with a cold L2."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1501_01809_b200 import configs

torch.cuda.set_device(0)
w = configs.Workload(5, None)
w.reset(); w.run(); torch.cuda.synchronize()
flush = bench.Flusher(torch)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, lp, out in zip(["A", "B", "BT"], w.loops, [w.outputs[0], w.outputs[2], w.outputs[1]]):
    ts = []
    for _ in range(8):
        out.zero(); flush()
        e0.record(st); w.L.execute(lp); e1.record(st); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    nnz = out.sparsity.nnz if hasattr(out.sparsity, "nnz") else 0
    print(f"C5 {name}: {np.median(ts[2:]):.3f} ms  nnz={nnz}", flush=True)
