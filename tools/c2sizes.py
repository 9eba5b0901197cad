import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1501_01809_b200 import capi, configs
import oracle as O
capi.set_strategy("auto")
for n in [int(x) for x in sys.argv[1:]]:
    w = configs.Workload(2, n); w.reset(); w.run(); torch.cuda.synchronize()
    m = w.inputs; A = w.outputs[0]; rp, ci = A.sparsity.host()
    ref = O.assemble_matrix(O.STIFFNESS, 1, 2, m.ncells, m.cv, 3, m.cv, 3, m.cv, m.coords, rp, ci)
    got = A.host_values(); print(n, np.max(np.abs(got-ref))/np.max(np.abs(ref)), flush=True)
