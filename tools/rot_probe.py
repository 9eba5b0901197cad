"""Developer probe: per-config ms/step under bench.Rotation (K back-to-back
steps in one graph over rotated replicas) and the flushed single-step
protocol.  LOAM_GPU_NO_PDL=1 turns programmatic dependent launch off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1501_01809_b200 import capi, configs  # noqa: E402

capi.set_strategy("auto")
if os.environ.get("DET"):
    capi.set_option(capi.OPT_DETERMINISTIC, 1)
flush = bench.Flusher(torch)
stream = torch.cuda.current_stream()
peak, _ = bench.peaks()
for c in sys.argv[1:] or ["1", "2", "3r", "3m", "4", "5"]:
    cfg = int(c[0])
    part = {"r": "residual", "m": "matrix"}.get(c[1:], None)
    w = configs.Workload(cfg, None, part)
    w.reset(); w.run(); torch.cuda.synchronize()
    ab = bench.algorithmic_bytes(w)
    fl = float(np.median(bench.time_steps(torch, w, 10, flush, stream)))
    rot = bench.Rotation(torch, w)
    K = max(40, 4 * rot.R)
    ts = [rot.time(K, stream, warmup=K) for _ in range(3)]
    f = lambda ms: ab / (ms * 1e-3) / 1e9 / peak
    print(f"config {c} pdl={'off' if os.environ.get('LOAM_GPU_NO_PDL') else 'on'}{' det' if os.environ.get('DET') else ''}: R={rot.R} K={K} "
          f"rotation {min(ts)*1e3:.1f} us ({f(min(ts)):.3f}) [{', '.join(f'{x*1e3:.1f}' for x in ts)}]  "
          f"flushed {fl*1e3:.1f} us ({f(fl):.3f}); launches/step {rot.launches_per_step:.1f}", flush=True)
    del rot, w
    torch.cuda.empty_cache()
