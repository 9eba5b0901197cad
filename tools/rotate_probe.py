"""Developer: per-step time of back-to-back assemblies over R rotating replicas
(aggregate working set > L2) vs the flushed single-step protocol."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1501_01809_b200 import configs
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for cfg, R in ((2, 4), (1, 12), (3, 3)):
    part = "matrix" if cfg == 3 else None
    ws = [configs.Workload(cfg, None, part) for _ in range(R)]
    for w in ws:
        w.reset(); w.run()
    torch.cuda.synchronize()
    K = 48
    res = []
    for rep in range(3):
        for k in range(2 * R):
            ws[k % R].reset(); ws[k % R].run()
        torch.cuda.synchronize()
        e0.record(st)
        for k in range(K):
            ws[k % R].reset(); ws[k % R].run()
        e1.record(st); e1.synchronize()
        res.append(e0.elapsed_time(e1) / K * 1e3)
    print(f"C{cfg}{'m' if part else ''} rotating R={R}: us/step", [round(x, 2) for x in res], flush=True)
    del ws
    torch.cuda.empty_cache()
