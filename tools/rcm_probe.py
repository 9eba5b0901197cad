"""Times device RCM / reorder against the compiled reference's rcm_order on
the config meshes (cell-permuted C2 / C3 vertex meshes).  Prints one JSON
line per mesh.  Device times: CUDA events around L.rcm_order / L.reorder
(includes the per-level host syncs); reference: wall clock of ref_rcm_order on
the same adjacency (one host thread, as the reference runs it)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from paper_1501_01809_b200 import configs  # noqa: E402
from paper_1501_01809_b200 import loam as L  # noqa: E402


def ev_time(fn, reps=3):
    best, out = 1e30, None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best, out


for gdim, n in ((2, 1024), (3, 64)):
    m = configs.mesh(gdim, n, 0.1, 5, 6)
    cm = L.Map(L.Set(m.ncells), L.Set(m.nv, "vertices"), gdim + 1, m.cv, "cell_vertex")
    X = L.Dat(cm.target, gdim, "coordinates")
    X.set_values(m.coords)
    rp, ci = L.vertex_adjacency(cm, gdim)
    t_adj, _ = ev_time(lambda: L.vertex_adjacency(cm, gdim))
    t_rcm, perm = ev_time(lambda: L.rcm_order(m.nv, rp, ci))
    t_reo, _ = ev_time(lambda: L.reorder(cm, X))
    hrp, hci = rp.cpu().numpy(), ci.cpu().numpy()
    t0 = time.perf_counter()
    ref = O.rcm_order((hrp, hci), lib="ref") if O.ref_available() else O.rcm_order((hrp, hci))
    t_ref = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"mesh": f"{'C2' if gdim == 2 else 'C3'} vertices {n}^{gdim}", "nverts": m.nv,
                      "adj_entries": int(hci.size), "device_adjacency_ms": round(t_adj, 3),
                      "device_rcm_ms": round(t_rcm, 3), "device_reorder_ms": round(t_reo, 3),
                      "cpu_rcm_ms": round(t_ref, 2), "cpu_kind": "reference" if O.ref_available() else "port",
                      "equal": bool(np.array_equal(perm.cpu().numpy(), ref))}), flush=True)
