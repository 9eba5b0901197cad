"""Developer: C3 residual (cell-centric fp64 REDs) with and without the cell locality order."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1501_01809_b200 import capi, configs
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
flush = bench.Flusher(torch)
for loc in (1, 0):
    capi.set_option(capi.OPT_LOCALITY if hasattr(capi, "OPT_LOCALITY") else 2, loc)
    w = configs.Workload(3, None, "residual")
    w.reset(); w.run(); torch.cuda.synchronize()
    ts = bench.time_steps(torch, w, 10, flush, st)
    print("locality", loc, "ms", round(float(np.median(ts)), 4), flush=True)
    del w
