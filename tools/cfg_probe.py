"""Developer: median ms of 20 flushed steps of one config (bench protocol),
knobs from the environment.  usage: cfg_probe.py CFG [PART] [TAG]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1501_01809_b200 import configs
cfg = int(sys.argv[1]); part = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "-" else None
tag = sys.argv[3] if len(sys.argv) > 3 else ""
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
flush = bench.Flusher(torch)
w = configs.Workload(cfg, None, part)
w.reset(); w.run(); torch.cuda.synchronize()
ts = bench.time_steps(torch, w, 20, flush, st)
print("cfg", cfg, part, tag, "ms", round(float(np.median(ts)), 4), flush=True)
