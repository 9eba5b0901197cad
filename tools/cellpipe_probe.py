"""Developer: C3 residual with the pipelined cell kernel (LOAM_GPU_CELL_PIPE
given in the environment per process) -- median ms of 20 flushed steps and
the max-norm relative difference to the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1501_01809_b200 import configs
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
flush = bench.Flusher(torch)
w = configs.Workload(3, None, "residual")
w.reset(); w.run(); torch.cuda.synchronize()
ts = bench.time_steps(torch, w, 20, flush, st)
print("pipe", os.environ.get("LOAM_GPU_CELL_PIPE", "default"), "ms", round(float(np.median(ts)), 4), flush=True)
