"""Developer: what the bench's cold-L2 event timing charges a trivial kernel
and a 15 MB / 100 MB streaming read (floor for C1 / C2)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
torch.cuda.set_device(0)
flush = bench.Flusher(torch)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a15 = torch.ones(15_000_000 // 8, dtype=torch.float64, device="cuda")
a100 = torch.ones(100_000_000 // 8, dtype=torch.float64, device="cuda")
o = torch.zeros(1, dtype=torch.float64, device="cuda")
b15 = torch.empty_like(a15)
def t(fn, n=20):
    ts = []
    for _ in range(n):
        flush()
        e0.record(st); fn(); e1.record(st); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts[3:])
print("empty fill(1 elem) us", t(lambda: o.fill_(1.0)))
print("sum 15MB us", t(lambda: torch.sum(a15, dim=0, out=o[0])))
print("copy 15MB->15MB us", t(lambda: b15.copy_(a15)))
print("sum 100MB us", t(lambda: torch.sum(a100, dim=0, out=o[0])))
# variants: no flush; flush + settle (a tiny kernel + stream sync before the timed region)
def t2(fn, n=20, mode="noflush"):
    ts = []
    for _ in range(n):
        if mode != "noflush":
            flush()
        if mode == "settle":
            o.fill_(0.0)
            torch.cuda.synchronize()
        e0.record(st); fn(); e1.record(st); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts[3:])
for mode in ("noflush", "settle"):
    print(mode, "empty", t2(lambda: o.fill_(1.0), mode=mode), "copy15", t2(lambda: b15.copy_(a15), mode=mode),
          "sum100", t2(lambda: torch.sum(a100, dim=0, out=o[0]), mode=mode))
# flush, then a GPU-side spin (torch.cuda._sleep) so the timed launches are queued
# before the stream reaches e0: no host launch latency inside the interval
def t3(fn, n=20, spin=200000):
    ts = []
    for _ in range(n):
        flush()
        torch.cuda._sleep(spin)
        e0.record(st); fn(); e1.record(st); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts[3:])
print("flush+spin empty", t3(lambda: o.fill_(1.0)), "copy15", t3(lambda: b15.copy_(a15)),
      "sum100", t3(lambda: torch.sum(a100, dim=0, out=o[0])))
from paper_1501_01809_b200 import configs
w = configs.Workload(2, None)
w.reset(); w.run(); torch.cuda.synchronize()
def step():
    w.run()
for mode in ("flush", "flush+spin"):
    ts = []
    for _ in range(20):
        w.reset(); flush()
        if mode == "flush+spin":
            torch.cuda._sleep(200000)
        e0.record(st); step(); e1.record(st); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print("C2 step", mode, np.median(ts[3:]))

# back to back from one CUDA graph over rotated buffers (bench.Rotation's
# protocol): what a 15 MB / 100 MB streaming read and copy cost per step when
# every step's data is cold but launches are not the gap
def b2b(nbytes, kind, K=40):
    R = max(2, int(np.ceil(3 * 126 * 2**20 / nbytes)) + 1)
    n = nbytes // 8 // (2 if kind == "copy" else 1)
    src = [torch.ones(n, dtype=torch.float64, device="cuda") for _ in range(R)]
    dst = [torch.empty_like(x) for x in src] if kind == "copy" else None
    outs = torch.zeros(R, dtype=torch.float64, device="cuda")
    g, side = torch.cuda.CUDAGraph(), torch.cuda.Stream()
    side.wait_stream(st)
    with torch.cuda.graph(g, stream=side):
        for k in range(K):
            if kind == "copy":
                dst[k % R].copy_(src[k % R])
            else:
                torch.sum(src[k % R], dim=0, out=outs[k % R])
    st.wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    e0.record(st); g.replay(); e1.record(st); e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / K, R
for nb in (15_000_000, 100_000_000):
    for kind in ("read", "copy"):
        us, R = b2b(nb, kind)
        print(f"back-to-back {kind} {nb/1e6:.0f} MB (R={R}): {us:.2f} us/step = {nb/us/1e3:.0f} GB/s")
