"""Developer probe: first-execute (plan construction) cost per config, with
the per-phase breakdown printed by LOAM_GPU_PLAN_TIMING=1 (stderr)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LOAM_GPU_PLAN_TIMING", "1")
import torch  # noqa: E402

from paper_1501_01809_b200 import capi, configs  # noqa: E402

capi.set_strategy("auto")
want = sys.argv[1:] or ["1", "2", "3r", "3m", "4", "5"]
for c in want:
    cfg = int(c[0])
    part = {"r": "residual", "m": "matrix"}.get(c[1:], None)
    w = configs.Workload(cfg, None, part)
    torch.cuda.synchronize()
    print(f"== config {c}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    w.reset()
    w.run()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    w.reset()
    w.run()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"config {c}: first execute {1e3 * (t1 - t0):.1f} ms, second {1e3 * (t2 - t1):.2f} ms", flush=True)
    del w
    torch.cuda.empty_cache()
