#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 par_loop hot path.

Workload (BASELINE.json configs[1], the metric's config): P1 Laplace stiffness
matrix assembly into CSR on the unit square 1024^2 mesh (2,097,152 cells,
1,050,625 vertices, jitter 0.2h seed 2, cell permutation seed 3).  A step is
one par_loop execute(stiffness_p1_tri; Mat INC (cell_vertex, cell_vertex),
coordinates READ) into a freshly zero-initialised Mat whose sparsity was built
once beforehand (assemble_matrix without its build_sparsity: the
sparsity build is reported separately).  Inputs are resident in HBM.  The
timed region is EXACTLY K steps executed back to back from one CUDA graph,
step k on replica k % R of R independent copies of the workload (distinct
maps, plans, coordinates and Mats; R chosen so each step's data was last
touched >= 3 L2 capacities ago: inputs larger than L2), bracketed by one pair
of CUDA events on the launching stream.  The flushed single-step protocol (L2
flushed by a 512 MiB write + 256 MiB read before every step, events around one
launch) is reported beside it.  N>1 runs N independent replicas (one rank per
GPU, weak scaling) and takes the max over ranks.

  value      assembled cells/s (whole job)
  e2e        same metric through loam_gpu_execute_host_batch (the reference
             calling convention, host buffers): H2D of the coordinates and D2H
             of the values inside the timed region; cold_one_shot = a whole
             assemble_matrix with nothing cached (uploads, build_sparsity,
             plan, execute, download)
  roofline   minimal algorithmic bytes (map int32 + coords fp64 + values fp64
             written once) / mean kernel time vs MEASURED_PEAKS.json hbm_gbs
  sparsity_build  C2's build_sparsity on the device vs its roofline (C2-sp)
  cpu_baseline  the reference's own par_loop (oracle/_ref: loam::execute with
             the reference's optimised AST kernel) on the full C2 mesh at all
             host threads, plus 1-thread and compiled-host-kernel lines and
             the CPU model
  all_configs   the six BASELINE workloads: GPU ms, cells/s, HBM fraction,
             first-call plan build, and the reference engine's cells/s on a
             bounded sample of each

--impl reference runs only the reference CPU arm (rank 0) on the SAME workload
(full C2 mesh, inputs from the oracle's restated generator, so the product
library is never loaded there), --steps / --warmup as given.
--all-configs (developer) prints one line per config/strategy for profiles/.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembled cells/s + achieved HBM GB/s vs peak for P1/P2 residual & CSR matrix"
UNIT = "cells/s"
WORKLOAD = "C2: P1 Laplace stiffness CSR assembly, unit square 1024x1024 (2,097,152 cells)"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(tag):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get(tag, {}).get("dram_bytes")
    except Exception:
        return None


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML while the GPU works."""

    REASONS = {
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
    }

    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons, self.period = [], set(), period
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                if util > 0:
                    self.samples.append(mhz)
                    for bit, name in self.REASONS.items():
                        if r & bit:
                            self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples_under_load": len(self.samples)}


# --------------------------------------------------------------------------- helpers
def algorithmic_bytes(w):
    """Minimal bytes: every map entry once (int32), unique inputs once
    and outputs written once (fp64)."""
    m = w.inputs
    cfg = w.cfg
    if cfg == 1:
        return m.ncells * 3 * 4 + m.nv * 2 * 8 + m.nv * 8 + m.nv * 8
    if cfg == 2:
        return m.ncells * 3 * 4 + m.nv * 2 * 8 + w.outputs[0].sparsity.nnz * 8
    if cfg == 3:
        nn = m.extra["nn"]
        b = m.ncells * 10 * 4 + m.nv * 3 * 8
        if w.part == "residual":
            return b + 2 * nn * 8
        return b + w.outputs[0].sparsity.nnz * 8
    if cfg == 4:
        return m.ncells * 4 * 4 + m.nv * 3 * 8 + w.outputs[0].sparsity.nnz * 8
    if cfg == 5:
        return m.ncells * (6 + 3) * 4 + m.nv * 2 * 8 + sum(o.sparsity.nnz for o in w.outputs) * 8
    raise ValueError(cfg)


class Flusher:
    """L2 flush between timed steps: a 512 MiB write (> the 126 MB L2), then a
    256 MiB read of a second buffer so the write's dirty lines are evicted here
    and the step starts with a cold, clean L2 (no write-backs of the flush
    buffer charged to the kernel)."""

    def __init__(self, torch):
        self.buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        self.rbuf = torch.ones(32 << 20, dtype=torch.int64, device="cuda")  # 256 MiB
        self.acc = torch.zeros((), dtype=torch.int64, device="cuda")
        self.v = 0

    def __call__(self):
        self.v = (self.v + 1) & 0xFF
        self.buf.fill_(self.v)
        self.acc += self.rbuf.sum()


def time_steps(torch, w, steps, flush, stream):
    """Per-step device time (ms) with L2 flushed before each step."""
    times = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(steps):
        w.reset()
        flush()
        e0.record(stream)
        w.run()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    return times


L2_BYTES = 126 * 2 ** 20


class Rotation:
    """The timed protocol: R independent replicas of a config's loops (every
    object distinct -- maps and therefore plans, coordinates, coefficients,
    outputs) and K steps executed back to back cycling the replicas, captured
    once into ONE CUDA graph of K executes and launched as one.  R is chosen
    so a replica's data was last touched >= 3 L2 capacities of other traffic
    ago: every step reads its inputs cold from HBM and pays the write-back of
    the previous steps' outputs, with no host launch gaps between steps (the
    rule's "inputs larger than L2" option; the flushed single-step protocol is
    reported beside it).  Consecutive tile kernels are programmatic dependent
    launches: a step's prologue (barriers, plan records) overlaps the previous
    step's tail; it reads the caller's data only after the previous grid
    completed."""

    def __init__(self, torch, w0, replicas=None):
        from paper_1501_01809_b200 import configs
        self.torch = torch
        ab = algorithmic_bytes(w0)
        self.R = replicas or max(2, min(24, int(np.ceil(3 * L2_BYTES / ab)) + 1))
        self.ws = [w0] + [configs.Workload(w0.cfg, None, w0.part, inputs=w0.inputs) for _ in range(self.R - 1)]
        for w in self.ws:  # plans are built outside the graphs
            w.reset()
            w.run()
        torch.cuda.synchronize()
        self.graphs = {}
        self.launches_per_step = 0.0

    def graph(self, steps):
        """One CUDA graph executing `steps` steps (step k on replica k % R)."""
        if steps not in self.graphs:
            from paper_1501_01809_b200 import capi
            torch = self.torch
            g, side = torch.cuda.CUDAGraph(), torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            l0 = capi.launch_count()
            with torch.cuda.graph(g, stream=side):
                for k in range(steps):
                    w = self.ws[k % self.R]
                    w.reset()
                    w.run()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            self.launches_per_step = (capi.launch_count() - l0) / steps  # kernels recorded per step
            self.graphs[steps] = g
        return self.graphs[steps]

    # a captured launch keeps its plan's tile-counter pair (32 per plan,
    # engine.cu TileCounters): a graph holds at most 16 steps per replica and
    # longer runs replay it back to back
    def chunks(self, steps):
        L = min(steps, 16 * self.R)
        return [L] * (steps // L) + ([steps % L] if steps % L else [])

    def replay_steps(self, steps):
        for c in self.chunks(steps):
            self.graph(c).replay()

    def time(self, steps, stream, warmup=0):
        """ms per step over EXACTLY `steps` back-to-back steps (graph
        launches, one pair of events on `stream`)."""
        for c in self.chunks(steps):
            self.graph(c)  # captured before the timed region
        # warm-up: >= `warmup` untimed steps through the SAME graph(s) the timed
        # region replays (a graph's first launch also uploads it to the device)
        for _ in range(max(1, -(-max(warmup, 1) // steps))):
            self.replay_steps(steps)
        e0, e1 = self.torch.cuda.Event(enable_timing=True), self.torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        self.replay_steps(steps)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / steps


def protocol_floor(torch, flush, stream, reps=10):
    """What the per-step protocol (flush, event, launch, event) charges a
    trivial kernel and a 100 MB streaming read (torch.sum) on this box: the
    fixed event + launch cost inside every timed step, and the streaming
    floor C2's 100.7 algorithmic MB compare against."""
    o = torch.zeros(1, dtype=torch.float64, device="cuda")
    a = torch.ones(100_000_000 // 8, dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def t(fn):
        ts = []
        for _ in range(reps):
            flush()
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts[2:]))
    out = {"empty_kernel_ms": t(lambda: o.fill_(1.0)),
           "stream_read_100MB_ms": t(lambda: torch.sum(a, dim=0, out=o[0]))}
    del a
    return out


def config_table(torch, flush, stream, steps=5, cpu=True):
    """Every BASELINE config at full size through `auto` under the headline's
    protocol (Rotation: back-to-back graph replays over rotated replicas) and
    the flushed single-step protocol (median of `steps`): cells/s and the
    fraction of the measured HBM peak, so the contract line carries the whole
    table measured on the same box.  plan_build_s = the first execute (plan
    construction + the assembly); cpu_* = the compiled reference engine with
    the restated host kernel on a bounded sample of the same workload."""
    from paper_1501_01809_b200 import capi, configs
    peak, _ = peaks()
    names = {(1, None): "C1 P1 Helmholtz residual 512^2", (2, None): "C2 P1 Laplace CSR 1024^2",
             (3, "residual"): "C3 P2 Helmholtz residual 64^3", (3, "matrix"): "C3 P2 Helmholtz CSR 64^3",
             (4, None): "C4 vector-P1 elasticity 96^3", (5, None): "C5 Taylor-Hood blocks 768^2"}
    rows = []
    capi.set_strategy("auto")
    for (cfg, part), name in names.items():
        w = configs.Workload(cfg, None, part)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        w.reset()
        w.run()
        torch.cuda.synchronize()
        plan_s = time.perf_counter() - t0
        for _ in range(2):
            w.reset()
            flush()
            w.run()
        ms_flushed = float(np.median(time_steps(torch, w, steps, flush, stream)))
        rot = Rotation(torch, w)
        ms = rot.time(max(4 * rot.R, 40), stream, warmup=2 * rot.R)
        ab = algorithmic_bytes(w)
        row = {"config": name, "ms": round(ms, 4), "cells_per_s": w.inputs.ncells / (ms * 1e-3),
               "frac": round(ab / (ms * 1e-3) / 1e9 / peak, 3), "replicas": rot.R,
               "ms_flushed": round(ms_flushed, 4), "frac_flushed": round(ab / (ms_flushed * 1e-3) / 1e9 / peak, 3),
               "plan_build_s": round(plan_s, 4)}
        del rot
        if cpu:
            try:
                row.update(reference_config_cpu(cfg, part, os.cpu_count() or 1))
            except Exception as exc:  # noqa: BLE001
                row["cpu_error"] = str(exc)
        rows.append(row)
        del w
        torch.cuda.empty_cache()
    return rows


def sparsity_build(torch, w, reps=5):
    """C2-sp: build_sparsity of the C2 cell->vertex map on the
    device (keys, radix sort, unique, row offsets) against its 62,955,540-byte
    roofline (map read + row_ptr + col_idx written once)."""
    from paper_1501_01809_b200 import loam as L
    peak, _ = peaks()
    ts = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sp = L.build_sparsity(w.cvm, w.cvm)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        del sp
    ms = 1e3 * float(np.median(ts[1:]))
    m = w.inputs
    ab = m.ncells * 3 * 4 + (m.nv + 1) * 8 + w.outputs[0].sparsity.nnz * 4
    return {"ms": ms, "algorithmic_bytes": ab, "frac": ab / (ms * 1e-3) / 1e9 / peak,
            "note": "host wall clock around loam_gpu_build_sparsity (one call, synchronous)"}


def cold_one_shot(torch, m):
    """A reference user's one-shot fem::assemble_matrix (assemble.hpp:85-104) on
    the C2 inputs through the device API with nothing cached: upload the map
    and coordinates, build_sparsity, plan + assemble, download the values."""
    from paper_1501_01809_b200 import loam as L
    out = []
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cells, verts = L.Set(m.ncells), L.Set(m.nv)
        cv = L.Map(cells, verts, 3, m.cv)
        X = L.Dat(verts, 2)
        X.set_values(m.coords)
        A = L.Mat(L.build_sparsity(cv, cv))
        L.execute(L.Parloop(L.kernel("stiffness_p1_tri"), cells, [L.arg(A, L.INC, cv, cv), L.arg(X, L.READ, cv)]))
        vals = A.host_values()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
        del cells, verts, cv, X, A, vals
    return {"s": min(out), "includes": "H2D map + coordinates, build_sparsity, plan build, execute, D2H values"}


def e2e_host(torch, w, steps, warmup):
    """The same assembly through the host-memory C ABI with pinned host
    buffers: every step copies the Dats the loop reads host->device and the
    values it writes device->host inside the timed region.  Maps and the
    Sparsity are immutable, id'd objects the library keeps resident after the
    first (warm-up) call, so they are not per-step transfers.

    The timed steps go through loam_gpu_execute_host_batch: K steps over two
    alternating sets of pinned host buffers, step k+1's upload overlapping
    step k's download on the two copy engines (returns ms per step over the
    batch).  `sequential` times the one-call-per-step loam_gpu_execute_host
    (synchronous, no overlap) for comparison."""
    from paper_1501_01809_b200 import loam as L
    w.reset()
    host_loops = [L.HostLoop(lp) for lp in w.loops]
    h2d = sum(h.h2d_bytes for h in host_loops)
    d2h = sum(h.d2h_bytes for h in host_loops)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run():
        for h in host_loops:
            h.run(sh)

    for _ in range(warmup):
        run()
    seq = []
    for _ in range(max(3, min(steps, 5))):
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        seq.append(e0.elapsed_time(e1))
    alts = [h.step_buffers()[0] for h in host_loops]
    batches = [[h.descs if k % 2 == 0 else alt for k in range(steps)] for h, alt in zip(host_loops, alts)]

    def run_batch():
        for h, b in zip(host_loops, batches):
            h.run_batch(b, sh)

    run_batch()  # warm-up of the batch path
    times = []
    for _ in range(3):
        e0.record(stream)
        run_batch()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / steps)
    return times, h2d, d2h, float(np.mean(seq))


def cpu_model() -> str:
    """The host CPU model (lscpu's "Model name"), from /proc/cpuinfo."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_c2(threads, warmup, steps, n=None, as_shipped=True):
    """The reference's own par_loop (oracle/_ref: loam::execute, parloop.hpp:191)
    on the C2 workload, inputs from the oracle's restatement of the generator
    (bit-identical to the GPU arm's, tests/test_oracle_cpu.py) -- the product
    library is never loaded here.  as_shipped: the reference's optimised AST
    kernel (assemble.hpp:16-19); else the restated compiled host kernel
    (kernel.hpp:523-529).  Returns (cells, per-step seconds)."""
    import oracle as O
    m = O.inputs(2, n)
    times = O.ref_time_execute(O.STIFFNESS, 1, 2, m.cv, m.coords, as_shipped=as_shipped, threads=threads,
                               warmup=warmup, steps=steps)
    return m.ncells, times


# per-config CPU figures: the compiled reference ENGINE (build_sparsity + execute +
# Mat::addto) with the restated host kernel, on bounded samples of each workload
CPU_SAMPLES = {(1, None): 512, (2, None): 1024, (3, "residual"): 32, (3, "matrix"): 16, (4, None): 32,
               (5, None): 256}


def reference_config_cpu(cfg, part, threads):
    import oracle as O
    n = CPU_SAMPLES[(cfg, part)]
    m = O.inputs(cfg, n)
    run = []
    if cfg == 1:
        run.append(dict(form=O.HELMHOLTZ_ACTION, degree=1, gdim=2, row_map=m.cv, ar_r=3, nrt=m.nv, col_map=None,
                        ar_c=0, nct=0, coeff=m.extra["u"], params=(1.0,)))
    elif cfg == 2:
        run.append(dict(form=O.STIFFNESS, degree=1, gdim=2, row_map=m.cv, ar_r=3, nrt=m.nv, col_map=m.cv, ar_c=3,
                        nct=m.nv, params=()))
    elif cfg == 3:
        cn, nn = m.extra["p2"], m.extra["nn"]
        if part == "residual":
            run.append(dict(form=O.HELMHOLTZ_ACTION, degree=2, gdim=3, row_map=cn, ar_r=10, nrt=nn, col_map=None,
                            ar_c=0, nct=0, coeff=m.extra["u"], params=(1.0,)))
        else:
            run.append(dict(form=O.HELMHOLTZ, degree=2, gdim=3, row_map=cn, ar_r=10, nrt=nn, col_map=cn, ar_c=10,
                            nct=nn, params=(1.0,)))
    elif cfg == 4:
        dm = O.dof_map(m.cv, 4, 3)
        run.append(dict(form=O.ELASTICITY, degree=1, gdim=3, row_map=dm, ar_r=12, nrt=3 * m.nv, col_map=dm, ar_c=12,
                        nct=3 * m.nv, params=(1.0, 0.5)))
    else:
        cn, nn = m.extra["p2"], m.extra["nn"]
        vd = O.dof_map(cn, 6, 2)
        run += [dict(form=O.STOKES_A, degree=2, gdim=2, row_map=vd, ar_r=12, nrt=2 * nn, col_map=vd, ar_c=12,
                     nct=2 * nn, params=(1.0,)),
                dict(form=O.STOKES_B, degree=2, gdim=2, row_map=m.cv, ar_r=3, nrt=m.nv, col_map=vd, ar_c=12,
                     nct=2 * nn, params=()),
                dict(form=O.STOKES_BT, degree=2, gdim=2, row_map=vd, ar_r=12, nrt=2 * nn, col_map=m.cv, ar_c=3,
                     nct=m.nv, params=())]
    step, sp = 0.0, 0.0
    for r in run:
        t, s_ = O.ref_time_engine(r["form"], r["degree"], r["gdim"], m.ncells, r["row_map"], r["ar_r"], r["nrt"],
                                  r["col_map"], r["ar_c"], r["nct"], m.cv, m.coords, coeff=r.get("coeff"),
                                  params=r["params"], threads=threads, warmup=0, steps=1)
        step += float(t.min())
        sp += s_
    return {"cpu_cells_per_s": m.ncells / step, "cpu_sample_cells": m.ncells, "cpu_threads": threads,
            "cpu_build_sparsity_s": sp if sp else None}


def cpu_baseline_block(threads):
    """SURVEY 8d CPU lines on the GPU box's host cores: the as-shipped reference
    (optimised AST kernel) and the compiled-host-kernel engine, at 1 thread and
    at all threads, next to the CPU model."""
    lines = []

    def line(as_shipped, th, n, warmup, steps):
        cells, t = reference_c2(th, warmup, steps, n, as_shipped)
        lines.append({"kernel": "as-shipped AST (assemble.hpp:16-19)" if as_shipped else
                      "compiled host kernel (kernel.hpp:523-529)", "threads": th, "cells": cells,
                      "cells_per_s": cells / float(np.mean(t)), "steps": steps, "warmup": warmup})
        return lines[-1]

    main = line(True, threads, None, 1, 2)
    line(True, 1, 128, 0, 2)
    line(False, threads, None, 1, 2)
    line(False, 1, None, 0, 1)
    return {"value": main["cells_per_s"], "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": "oracle/_ref loam::execute with the reference's optimised AST stiffness_p1_tri on the full C2 "
                      f"mesh ({main['cells']} cells), {threads} threads, mean of 2 after 1 warm-up",
            "cpu_model": cpu_model(), "nproc": os.cpu_count(), "lines": lines}


# --------------------------------------------------------------------------- arms
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar over all ranks (timing rule: max over ranks).
    Works on NCCL (CUDA tensor) and gloo (CPU tensor) process groups."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_value(cells_per_rank: int, world: int, ms: float) -> float:
    """Whole-job cells/s: every rank assembles its own replica (weak scaling)."""
    return world * cells_per_rank / (ms * 1e-3)


def reference_arm(args):
    """The reference's own CPU par_loop on THIS arm's workload (full C2 mesh),
    all host threads, honouring --steps / --warmup; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    ncells, times = reference_c2(threads, args.warmup, args.steps)
    ms = 1e3 * float(np.mean(times))
    value = ncells / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(ncells),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"the whole workload: loam::execute (optimised AST stiffness_p1_tri) on the "
                                   f"{ncells}-cell C2 mesh, {threads} threads, mean of {args.steps} steps after "
                                   f"{args.warmup} warm-up", "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(cells):
    """The workload both arms report (same dict: the driver compares them)."""
    return {"workload": WORKLOAD, "cells": cells, "mesh": "unit square 1024^2, jitter 0.2h seed 2, "
            "cell permutation seed 3 (splitmix64, SURVEY 8d)"}


def gpu_arm(args):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_1501_01809_b200 import capi, configs
    lib = capi.lib()
    assert lib.loam_gpu_device_ok() == 1, "no sm_100 device"
    capi.set_strategy(args.strategy)

    w = configs.Workload(2, None)
    stream = torch.cuda.current_stream()
    flush = Flusher(torch)
    # plan build (colour/pair/slot plans are cached like the reference's colouring)
    t0 = time.perf_counter()
    w.reset()
    w.run()
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t0
    # flushed single-step protocol (reported beside the headline)
    for _ in range(3):
        w.reset()
        flush()
        w.run()
    flushed = time_steps(torch, w, max(args.steps, 10), flush, stream)
    rot = Rotation(torch, w)
    for c in rot.chunks(args.steps) + rot.chunks(max(args.warmup, 3)):
        rot.graph(c)  # every graph captured before the clocks start
    clocks = ClockSampler(local)
    with clocks:
        rot.replay_steps(max(args.warmup, 3))  # W >= 3 untimed warm-up steps
        soak_end = time.perf_counter() + 0.3  # keep the GPU busy so NVML sees load
        while time.perf_counter() < soak_end:
            rot.replay_steps(args.steps)
            torch.cuda.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        step_ms = rot.time(args.steps, stream)  # EXACTLY K steps (one graph), one event pair
        launches = int(round(rot.launches_per_step * args.steps))
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    times = [step_ms]
    n_rep = rot.R
    del rot
    torch.cuda.empty_cache()
    ms = max_over_ranks(float(np.mean(times)), "cuda")
    cells = w.inputs.ncells
    value = weak_value(cells, world, ms)
    abytes = algorithmic_bytes(w)
    peak, peak_kind = peaks()
    kernel_ms = float(np.mean(times))  # average launch duration: events on the launching stream over K launches
    achieved = abytes / (kernel_ms * 1e-3) / 1e9
    # end to end through the C ABI with host buffers
    e2e_times, h2d, d2h, e2e_seq_ms = e2e_host(torch, w, max(4, args.steps), 2)
    if os.environ.get("LOAM_BENCH_DEBUG"):
        print("e2e step ms:", [round(t, 3) for t in e2e_times], file=sys.stderr)
    e2e_ms = max_over_ranks(float(np.mean(e2e_times)), "cuda")
    floor = protocol_floor(torch, flush, stream)
    sp_build = sparsity_build(torch, w) if rank == 0 else None
    cold = cold_one_shot(torch, w.inputs) if rank == 0 else None
    table = (config_table(torch, flush, stream, cpu=not args.no_cpu_baseline)
             if rank == 0 and not args.no_config_table else None)
    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline_block(os.cpu_count() or 1)
            except Exception as exc:  # noqa: BLE001
                cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                       "sample": f"unavailable: {exc}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(cells),
            "protocol": {"vertices": w.inputs.nv, "nnz": w.outputs[0].sparsity.nnz,
                         "l2": f"inputs larger than L2: K back-to-back CUDA-graph replays cycling {n_rep} "
                               "independent replicas (distinct maps, plans, coordinates, outputs; a replica's data "
                               "was last touched >= 3 L2 capacities ago), one event pair around the K steps",
                         "flushed_ms_per_step": float(np.mean(flushed)),
                         "flushed": "L2 flushed before each step (512 MiB write + 256 MiB read), events around "
                                    "one launch: the per-step event/launch cost included",
                         "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                         "strategy": args.strategy, "plan_build_s": round(plan_s, 4),
                         "step": "one loam::execute into a fresh Mat whose sparsity was built beforehand"},
            "e2e": {"value": weak_value(cells, world, e2e_ms), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "path": "loam_gpu_execute_host_batch: per step H2D of the read Dats + kernel + D2H of the "
                            "values, uploads overlapping the previous step's downloads",
                    "sequential_ms_per_step": e2e_seq_ms, "cold_one_shot": cold},
            "sparsity_build": sp_build,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic("c2_matrix"),
                         "algorithmic_bytes": abytes, "kernel_ms": kernel_ms, "peak_kind": peak_kind,
                         "protocol_floor": floor},
            "cpu_baseline": cpu,
            "all_configs": table,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def all_configs(args):
    """Developer table: every config x strategy (not the contract line)."""
    import torch
    torch.cuda.set_device(0)
    from paper_1501_01809_b200 import capi, configs
    peak, _ = peaks()
    flush = Flusher(torch)
    stream = torch.cuda.current_stream()
    rows = []
    cases = [(1, None), (2, None), (3, "residual"), (3, "matrix"), (4, None), (5, None)]
    if args.configs:
        want = set(args.configs.split(","))
        cases = [c for c in cases if f"{c[0]}{'' if c[1] is None else c[1][0]}" in want or str(c[0]) in want]
    for cfg, part in cases:
        w = configs.Workload(cfg, args.size, part)
        for strat in args.strategies.split(","):
            capi.set_strategy(strat)
            try:
                t0 = time.perf_counter()
                w.reset()
                w.run()
                torch.cuda.synchronize()
                plan = time.perf_counter() - t0
                for _ in range(3):
                    w.reset()
                    flush()
                    w.run()
                l0 = capi.launch_count()
                times = time_steps(torch, w, args.steps, flush, stream)
                launches = (capi.launch_count() - l0) / args.steps
                ms = float(np.median(times))
                ab = algorithmic_bytes(w)
                rows.append({"config": cfg, "part": part, "strategy": strat, "cells": w.inputs.ncells,
                             "ms": ms, "cells_per_s": w.inputs.ncells / (ms * 1e-3),
                             "algorithmic_MB": ab / 1e6, "GB_s": ab / (ms * 1e-3) / 1e9,
                             "frac_of_measured_peak": ab / (ms * 1e-3) / 1e9 / peak,
                             "launches_per_step": launches, "first_call_s": plan})
            except Exception as exc:  # noqa: BLE001
                rows.append({"config": cfg, "part": part, "strategy": strat, "error": str(exc)})
            print(json.dumps(rows[-1]), flush=True)
        del w
        torch.cuda.empty_cache()
    capi.set_strategy("auto")
    return 0


def solver_bench(args):
    """Developer lines for SURVEY 8f-1: device SpMV on assembled config
    matrices against the HBM roofline, and CG time per iteration on the C2-size
    P1 Helmholtz matrix next to the reference's cg_solve on the host."""
    import torch
    from paper_1501_01809_b200 import configs
    from paper_1501_01809_b200 import loam as L
    torch.cuda.set_device(0)
    peak, peak_kind = peaks()
    flush = Flusher(torch)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for cfg in [int(c) for c in (args.configs or "2,4,5").split(",")]:
        w = configs.Workload(cfg, args.size)
        w.reset()
        w.run()
        mats = [o for o in w.outputs if isinstance(o, L.Mat)]
        if cfg == 5:
            Am, BTm, Bm = mats
            op = L.BlockMat([[Am, BTm], [Bm, None]], (Am.nrows, Bm.nrows), (Am.ncols, BTm.ncols))
            run = lambda x: L.block_spmv(op, x)
            nnz = sum(m.sparsity.nnz for m in mats)
            nrows, ncols = op.nrows, op.ncols
            rp_bytes = 8 * sum(m.nrows + 1 for m in mats)
        else:
            A = mats[0]
            run = lambda x: L.mat_spmv(A, x)
            nnz, nrows, ncols = A.sparsity.nnz, A.nrows, A.ncols
            rp_bytes = 8 * (nrows + 1)
        x = torch.rand(ncols, dtype=torch.float64, device="cuda")
        for _ in range(3):
            run(x)
        times = []
        for _ in range(args.steps):
            flush()
            e0.record(stream)
            run(x)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        abytes = nnz * 12 + rp_bytes + ncols * 8 + nrows * 8
        achieved = abytes / (ms * 1e-3) / 1e9
        print(json.dumps({"solver": "spmv", "config": cfg, "nnz": nnz, "rows": nrows, "ms": ms,
                          "algorithmic_MB": abytes / 1e6, "GB_s": achieved, "frac": achieved / peak,
                          "peak_kind": peak_kind, "bitwise": "reference mat_spmv / block_spmv"}), flush=True)
    # CG per iteration: P1 Helmholtz (SPD) on the C2 mesh, fixed iteration count
    import oracle as O
    for n, on_ref in ((1024, False), (256, True)):
        m = configs.config_inputs(2, n)
        cells, verts = L.Set(m.ncells), L.Set(m.nv)
        cv = L.Map(cells, verts, 3, m.cv)
        X = L.Dat(verts, 2)
        X.set_values(m.coords)
        A = L.Mat(L.build_sparsity(cv, cv))
        L.execute(L.Parloop(L.kernel("helmholtz_p1_tri", 1.0), cells, [L.arg(A, L.INC, cv, cv), L.arg(X, L.READ, cv)]))
        b = np.random.default_rng(1).uniform(-1, 1, m.nv)
        its = 200
        L.cg_solve(A, b, rtol=1e-30, atol=0.0, maxit=5)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = L.cg_solve(A, b, rtol=1e-30, atol=0.0, maxit=its)
        torch.cuda.synchronize()
        gpu_ms = (time.perf_counter() - t0) * 1e3 / rep.iterations
        line = {"solver": "cg", "mesh": f"{n}^2 P1 Helmholtz", "rows": m.nv, "nnz": A.sparsity.nnz,
                "iterations": rep.iterations, "gpu_ms_per_iteration": gpu_ms}
        if on_ref and O.ref_available():
            rp, ci = A.sparsity.host()
            t0 = time.perf_counter()
            xr, rr = O.ref_cg((m.nv, m.nv, rp, ci, A.host_values()), b, rtol=1e-30, atol=0.0, maxit=its)
            line["reference_cpu_ms_per_iteration"] = (time.perf_counter() - t0) * 1e3 / rr["iterations"]
            line["reference_iterations"] = rr["iterations"]
        print(json.dumps(line), flush=True)


def wave_bench(args):
    """Developer line for SURVEY 8f-2: the wave time-step chain (bench.hpp:222-300)
    on the device -- 3 pointwise loops + 1 stiffness-action par_loop + bc +
    max-norm per step, the host reading |p| every step as the reference does --
    next to the compiled reference's run_wave on a bounded sample."""
    import torch
    torch.cuda.set_device(0)
    from paper_1501_01809_b200.wave import WaveLoop
    import oracle as O
    n = args.size or 512
    dt = 0.05 / n
    w = WaveLoop(n, dt, 1e9)
    for _ in range(10):
        w.step()
    torch.cuda.synchronize()
    steps = max(args.steps, 50)
    t0 = time.perf_counter()
    for _ in range(steps):
        w.step()
    torch.cuda.synchronize()
    us = (time.perf_counter() - t0) * 1e6 / steps
    cells = 2 * n * n
    line = {"chain": "wave (run_wave)", "mesh": f"{n}^2 P1", "cells": cells, "us_per_step": us,
            "cell_steps_per_s": cells / (us * 1e-6), "launches_per_step": 6}
    # the same chain replayed as CUDA graphs of 100 steps (device-resident forcing / |p| / blow-up test)
    gsteps = max(steps, 2000) // 100 * 100
    for key, fused in (("graph", False), ("graph_fused", True)):
        wg = WaveLoop(n, dt, 1e9)
        wg.run_graph(100, max_steps=200, fused=fused)  # capture + warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        wg.run_graph(100, max_steps=gsteps, fused=fused)
        torch.cuda.synchronize()
        gus = (time.perf_counter() - t0) * 1e6 / gsteps
        line[key] = {"us_per_step": gus, "cell_steps_per_s": cells / (gus * 1e-6), "steps_per_graph": 100,
                     "launches_per_step": 3 if fused else 8,
                     "note": ("one fused kernel per step (loam_gpu_wave_step) + 2 clock kernels; " if fused else
                              "execute + 3 pointwise + bc + |p| + 2 clock kernels; ") +
                             "wall clock per step including one capture per run_graph call"}
    if O.ref_available():
        rn, rT = 32, 0.1
        t0 = time.perf_counter()
        O.ref_run_wave(rn, 1e-3, rT)
        rs = (time.perf_counter() - t0) / int(rT / 1e-3)
        line["reference_cpu"] = {"mesh": f"{rn}^2", "s_per_step": rs, "cell_steps_per_s": 2 * rn * rn / rs,
                                 "kind": "reference", "cores": 1, "sample": f"bench::run_wave({rn}, 1e-3, {rT})"}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="loam_gpu", choices=["loam_gpu", "reference"])
    ap.add_argument("--strategy", default="auto", choices=["auto", "owner", "atomic", "color", "nbr", "warpagg", "patch"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config-table", action="store_true", help="skip the per-config table in the line")
    ap.add_argument("--all-configs", action="store_true")
    ap.add_argument("--configs", default="")
    ap.add_argument("--strategies", default="auto,owner,atomic,warpagg,color,patch")
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--solver", action="store_true", help="developer: SpMV roofline and CG per-iteration lines")
    ap.add_argument("--wave", action="store_true", help="developer: the wave time-step chain (SURVEY 8f-2)")
    args = ap.parse_args()
    if args.solver:
        return solver_bench(args)
    if args.wave:
        return wave_bench(args)
    if args.impl == "reference":
        return reference_arm(args)
    if args.all_configs:
        return all_configs(args)
    return gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
