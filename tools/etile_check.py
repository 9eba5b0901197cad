"""Developer check of the edge-tile path (etile.cu): parity vs oracle at small
sizes (fresh and accumulating), full-size agreement with the pair-tile path."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_1501_01809_b200 import capi, configs


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


for n in (1, 2, 5, 9):
    w = configs.Workload(3, n, "matrix")
    w.reset(); l0 = capi.launch_count(); w.run(); l1 = capi.launch_count()
    m = w.inputs
    cn, nn = m.extra["p2"], m.extra["nn"]
    A = w.outputs[0]
    rp, ci = A.sparsity.host()
    ref = O.assemble_matrix(O.HELMHOLTZ, 2, 3, m.ncells, cn, 10, cn, 10, m.cv, m.coords, rp, ci, params=(configs.KAPPA,))
    got = A.host_values()
    e1 = rel(got, ref)
    w.run()
    e2 = rel(A.host_values(), 2 * ref)
    print(f"n={n} cells={m.ncells} launches={l1 - l0} fresh rel={e1:.2e} accumulate rel={e2:.2e}", flush=True)
for n in (2, 6):
    for cfg_part, form in ((("p2tri", None), None),):
        pass
if len(sys.argv) > 1:
    n = int(sys.argv[1])
    w = configs.Workload(3, n, "matrix")
    w.reset(); t0 = time.time(); w.run(); a = w.outputs[0].host_values().copy(); t1 = time.time()
    os.environ["LOAM_GPU_NO_ETILE"] = "1"
    capi.lib().loam_gpu_plan_cache_clear() if hasattr(capi.lib(), "loam_gpu_plan_cache_clear") else None
    w2 = configs.Workload(3, n, "matrix")
    w2.reset(); w2.run(); b = w2.outputs[0].host_values()
    print(f"full n={n}: etile vs ptile rel={rel(a, b):.2e} (etile first call {t1 - t0:.2f}s)")
