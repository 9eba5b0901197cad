"""Developer probe: where the e2e (host calling convention) step time goes."""
import time, sys
import torch
sys.path.insert(0, ".")
from paper_1501_01809_b200 import configs, capi
from paper_1501_01809_b200 import loam as L

w = configs.Workload(2)
w.reset()
h = L.HostLoop(w.loops[0])
for _ in range(3):
    h.run()
torch.cuda.synchronize()
t = []
for _ in range(10):
    t0 = time.perf_counter(); h.run(); t.append(time.perf_counter() - t0)
print("HostLoop.run ms", [round(x * 1e3, 3) for x in t])
# raw transfers of the same sizes (pinned)
a = torch.empty(16810000 // 8, dtype=torch.float64).pin_memory()
b = torch.empty(58769416 // 8, dtype=torch.float64).pin_memory()
da = torch.empty_like(a, device="cuda"); db = torch.empty_like(b, device="cuda")
for _ in range(3):
    da.copy_(a, non_blocking=True); b.copy_(db, non_blocking=True)
torch.cuda.synchronize()
t = []
for _ in range(10):
    t0 = time.perf_counter(); da.copy_(a, non_blocking=True); b.copy_(db, non_blocking=True); torch.cuda.synchronize(); t.append(time.perf_counter() - t0)
print("raw H2D 16.8MB + D2H 58.8MB ms", [round(x * 1e3, 3) for x in t])
t = []
for _ in range(10):
    t0 = time.perf_counter(); b.copy_(db, non_blocking=True); torch.cuda.synchronize(); t.append(time.perf_counter() - t0)
print("raw D2H 58.8MB ms", [round(x * 1e3, 3) for x in t])
# device-resident execute
t = []
for _ in range(10):
    w.reset(); torch.cuda.synchronize()
    t0 = time.perf_counter(); w.run(); torch.cuda.synchronize(); t.append(time.perf_counter() - t0)
print("device execute + sync ms", [round(x * 1e3, 3) for x in t])
