"""Developer: wall clock of loam_gpu_build_sparsity per config pattern (second call of each)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1501_01809_b200 import configs, loam as L
torch.cuda.set_device(0)
tag = "radix" if os.environ.get("LOAM_GPU_SPARSITY_SORT") else "rows"
def t(f):
    out = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); sp = f(); torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3); nnz = sp.nnz; del sp
    return min(out), nnz
for cfg in (2, 3, 4, 5):
    m = configs.config_inputs(cfg)
    cells, verts = L.Set(m.ncells), L.Set(m.nv)
    cv = L.Map(cells, verts, m.gdim + 1, m.cv)
    if cfg == 2:
        print(tag, "C2 (cv, cv)", "%.3f ms nnz %d" % t(lambda: L.build_sparsity(cv, cv)), flush=True)
    elif cfg == 4:
        print(tag, "C4 (cv, cv, 3, 3)", "%.3f ms nnz %d" % t(lambda: L.build_sparsity(cv, cv, 3, 3)), flush=True)
    else:
        nodes = L.Set(m.extra["nn"])
        cn = L.Map(cells, nodes, 10 if cfg == 3 else 6, m.extra["p2"])
        if cfg == 3:
            print(tag, "C3 (cn, cn)", "%.3f ms nnz %d" % t(lambda: L.build_sparsity(cn, cn)), flush=True)
        else:
            print(tag, "C5 A (cn, cn, 2, 2)", "%.3f ms nnz %d" % t(lambda: L.build_sparsity(cn, cn, 2, 2)), flush=True)
            print(tag, "C5 B (cv, cn, 1, 2)", "%.3f ms nnz %d" % t(lambda: L.build_sparsity(cv, cn, 1, 2)), flush=True)
            print(tag, "C5 BT (cn, cv, 2, 1)", "%.3f ms nnz %d" % t(lambda: L.build_sparsity(cn, cv, 2, 1)), flush=True)
