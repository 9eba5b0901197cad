"""Developer probe: k_ring phase timing (LOAM_GPU_PHASE_TIMING) on the C2
workload, plus per-CTA start/end and per-tile records (LOAM_GPU_PHASE_DUMP)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LOAM_GPU_PHASE_TIMING"] = "1"
os.environ.setdefault("LOAM_GPU_PHASE_DUMP", "gpurun_out/ring_phase.txt")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1501_01809_b200 import capi, configs  # noqa: E402

capi.set_strategy("auto")
w = configs.Workload(2, None)
flush = bench.Flusher(torch)
for _ in range(4):
    w.reset()
    flush()
    w.run()
    torch.cuda.synchronize()
