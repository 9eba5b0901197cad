"""The explicit wave time-step chain on the device.

Mirrors bench::run_wave (reference bench.hpp:222-300): unit square P1, marker-1
Dirichlet forcing p = sin(10 pi t) on x = 0 (mesh.hpp:132-134), lumped mass
(fem/assemble.hpp:145-148 lumped_mass = assemble_vector(source(V, 1))), and the
kick-drift-kick step

    phi -= dt/2 p ;  b = assemble_vector(stiffness_action(V, phi)) ;
    p += b * p_constant ;  bc.apply(p) ;  phi -= dt/2 p ;  |p|_inf

with p_constant = dt / lumped.  Every step is device work through the engine:
three pointwise loops (fem.cu, bitwise equal to the reference), one indirect
INC par_loop (the hot path: the P1 vertex-star kernel), the bc kernel and a
max-norm reduction; the host reads one scalar per step for the instability
check, as the reference does.  Diagnostics every 100 steps (|p|, |phi|,
energy = sum 0.5 m p^2 + sum 0.5 phi (K phi), K the assembled stiffness,
sequential sums as in the reference in run(), device tree sums in
run_graph()) match bench::run_wave's samples.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import capi, configs
from . import loam as L


class WaveLoop:
    def __init__(self, n: int, dt: float, T: float):
        L._require(dt > 0 and T >= dt, "InvalidArgument", "need dt > 0 and T >= dt")
        self.n, self.dt, self.T = n, dt, T
        m = configs.mesh(2, n)  # unit_square_mesh(n): no jitter, no permutation (bench.hpp:228)
        self.cells, self.verts = L.Set(m.ncells, "cells"), L.Set(m.nv, "vertices")
        cm = L.Map(self.cells, self.verts, 3, m.cv, "cell_vertex")
        X = L.Dat(self.verts, 2, "coordinates")
        X.set_values(m.coords)
        self.p, self.phi = L.Dat(self.verts, 1, "p"), L.Dat(self.verts, 1, "phi")
        marker1 = np.nonzero(np.arange(m.nv) % (n + 1) == 0)[0]  # facets with gi == 0
        self.bc = L.DirichletBC(self.verts, marker1, 0.0)
        ones = L.Dat(self.verts, 1, "one")
        ones.set_values(np.ones(m.nv))
        self.lumped = L.Dat(self.verts, 1, "lumped")
        L.execute(L.Parloop(L.kernel("source_p1_tri"), self.cells,
                            [L.arg(self.lumped, L.INC, cm), L.arg(X, L.READ, cm), L.arg(ones, L.READ, cm)]))
        self.p_constant = L.Dat(self.verts, 1, "p_constant")
        L.pointwise(self.p_constant, L.PwOp.ASSIGN, L.pw(dt) / L.pw(self.lumped))
        self.K = L.Mat(L.build_sparsity(cm, cm), "K")  # energy diagnostic
        L.execute(L.Parloop(L.kernel("stiffness_p1_tri"), self.cells,
                            [L.arg(self.K, L.INC, cm, cm), L.arg(X, L.READ, cm)]))
        self.b = L.Dat(self.verts, 1, "b")
        self.action = L.Parloop(L.kernel("stiffness_action_p1_tri"), self.cells,
                                [L.arg(self.b, L.INC, cm), L.arg(X, L.READ, cm), L.arg(self.phi, L.READ, cm)])
        self.half = L.pw(dt / 2) * L.pw(self.p)
        self.kick = L.pw(self.b) * L.pw(self.p_constant)
        self.t, self.steps = 0.0, 0
        self.first_period_max = 0.0
        self.samples = []  # (t, |p|_inf, |phi|_inf, energy)

    def energy(self) -> float:
        pv, phiv, mv = self.p.view(), self.phi.view(), self.lumped.view()
        kphi = L.mat_spmv(self.K, self.phi.data[: self.verts.size]).cpu().numpy()
        # sequential sums in the reference's order (bench.hpp:252-259)
        e = np.cumsum(np.concatenate([[0.0], 0.5 * mv * pv * pv]))[-1]
        return float(np.cumsum(np.concatenate([[e], 0.5 * phiv * kphi]))[-1])

    def energy_dev(self) -> float:
        """energy() reduced on the device (fixed-order tree sums instead of the
        reference's sequential ones: within ~1e-15 relative of them), one read
        back instead of four 2 MB copies and two host scans per sample."""
        nv = self.verts.size
        pv, phiv, mv = self.p.data[:nv], self.phi.data[:nv], self.lumped.data[:nv]
        kphi = L.mat_spmv(self.K, phiv)
        e = torch.stack([(0.5 * mv * pv * pv).sum(), (0.5 * phiv * kphi).sum()])
        h = e.cpu().numpy()
        return float(h[0] + h[1])

    def step(self) -> float:
        self.bc.constant = math.sin(10.0 * math.pi * self.t)
        L.pointwise(self.phi, L.PwOp.SUB, self.half)
        self.b.zero()
        L.execute(self.action)
        L.pointwise(self.p, L.PwOp.ADD, self.kick)
        self.bc.apply(self.p)
        L.pointwise(self.phi, L.PwOp.SUB, self.half)
        self.t += self.dt
        self.steps += 1
        pnorm = L.inf_norm(self.p)
        if self.t <= 0.2:
            self.first_period_max = max(self.first_period_max, pnorm)
        if self.first_period_max > 0 and pnorm > 1e3 * self.first_period_max:
            raise capi.LoamError(1 + capi.ERROR_KINDS.index("InstabilityDetected"),
                                 f"wave field blew up at t = {self.t}")
        if self.steps % 100 == 0:
            self.samples.append((self.t, pnorm, L.inf_norm(self.phi), self.energy()))
        return pnorm

    def run(self):
        while self.t <= self.T:
            self.step()
        torch.cuda.synchronize()
        return self.samples

    # ---- the same chain as one CUDA graph per batch of steps -----------------
    # The per-step host work (|p| read-back, the forcing value, ctypes calls)
    # dominates a 512^2 step; with the forcing, |p|, the first-period maximum
    # and the blow-up test kept in device state (loam_gpu_wave_clock) a batch
    # of steps is captured once and replayed, and the host reads the state
    # once per batch.  Blow-up is reported at the first failing step of the
    # batch (the fields of the later steps of that batch are then discarded
    # with the error, as the reference discards them when it throws).

    def _device_step(self, state):
        lib, sh = capi.lib(), torch.cuda.current_stream().cuda_stream
        sp = state.data_ptr()
        capi.check(lib.loam_gpu_wave_clock(sp, self.dt, 0.2, 0, sh))
        L.pointwise(self.phi, L.PwOp.SUB, self.half)
        self.b.zero()
        L.execute(self.action)
        L.pointwise(self.p, L.PwOp.ADD, self.kick)
        capi.check(lib.loam_gpu_bc_apply_dev(self.p.data.data_ptr(), self.p.set.size, self.bc._dev.data_ptr(),
                                             len(self.bc.nodes), sp + 8, sh))
        L.pointwise(self.phi, L.PwOp.SUB, self.half)
        capi.check(lib.loam_gpu_reduce_dev(self.p.data.data_ptr(), self.p.set.size, capi.REDUCE_MAX_ABS, sp + 16, sh))
        capi.check(lib.loam_gpu_wave_clock(sp, self.dt, 0.2, 1, sh))

    # ---- the step fused into the vertex-star action (loam_gpu_wave_step) ----
    # One kernel per step instead of six (pointwise x3, action, bc, |p|): the
    # half-kick of every gathered neighbour is formed on the fly and the owner
    # of each vertex applies kick, forcing and half-kick; p and phi ping-pong
    # between the Dats and a second buffer pair.  Bitwise equal to the
    # unfused chain (tests/test_fem_gpu.py).

    def _fused_setup(self) -> bool:
        if getattr(self, "_fz", None) is not None:
            return self._fz is not False
        nv = self.verts.size
        mask = torch.zeros(max(nv, 1), dtype=torch.uint8, device="cuda")
        mask[self.bc._dev.long()] = 1
        pb, phib = torch.empty_like(self.p.data), torch.empty_like(self.phi.data)
        kd, descs, keep = L._build(self.action)
        probe = torch.zeros(6, dtype=torch.float64, device="cuda")
        try:  # also builds the loop's plan outside any capture
            self._fused_call(kd, descs, self.p.data, self.phi.data, pb, phib, mask, probe)
        except capi.LoamError as e:
            if e.kind != "UnsupportedForm":
                raise
            self._fz = False
            return False
        self._fz = (kd, descs, keep, mask, pb, phib)
        for d in (self.p, self.phi):  # written behind the Dat's back from here on
            d._materialize()
            d._zero = d._stale = False
        return True

    def _fused_call(self, kd, descs, p_in, phi_in, p_out, phi_out, mask, state):
        capi.check(capi.lib().loam_gpu_wave_step(
            C.byref(kd), self.cells.size, self.cells.id, descs, len(self.action.args), p_in.data_ptr(),
            phi_in.data_ptr(), p_out.data_ptr(), phi_out.data_ptr(), self.p_constant.data.data_ptr(),
            mask.data_ptr(), self.dt / 2, state.data_ptr(), torch.cuda.current_stream().cuda_stream))

    def _fused_step(self, state, parity: int):
        kd, descs, keep, mask, pb, phib = self._fz
        lib, sh = capi.lib(), torch.cuda.current_stream().cuda_stream
        A, B = (self.p.data, self.phi.data), (pb, phib)
        src, dst = (A, B) if parity == 0 else (B, A)
        capi.check(lib.loam_gpu_wave_clock(state.data_ptr(), self.dt, 0.2, 0, sh))
        self._fused_call(kd, descs, src[0], src[1], dst[0], dst[1], mask, state)
        capi.check(lib.loam_gpu_wave_clock(state.data_ptr(), self.dt, 0.2, 1, sh))

    def run_graph(self, batch: int = 100, max_steps: int | None = None, fused: bool = True):
        """run() through CUDA graphs of `batch` steps (`batch` divides 100, so the
        every-100-steps diagnostics fall on batch boundaries); the steps after
        the last full batch run one by one as in run().  `fused`: one kernel per
        step (loam_gpu_wave_step) when the action runs on vertex stars."""
        assert batch >= 1 and 100 % batch == 0
        t, remaining = self.t, 0  # the step count run() would take (same double arithmetic)
        while t <= self.T and (max_steps is None or remaining < max_steps):
            t += self.dt
            remaining += 1
        self.b.zero()
        L.execute(self.action)  # the par_loop's plan is built and cached outside the capture
        state = torch.tensor([self.t, 0.0, 0.0, self.first_period_max, 0.0, float(self.steps)],
                             dtype=torch.float64, device="cuda")
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        fused = fused and self._fused_setup()
        with torch.cuda.graph(g, stream=side):
            for i in range(batch):
                if fused:
                    self._fused_step(state, i & 1)
                else:
                    self._device_step(state)
            if fused and batch & 1:  # the fields end in the second buffers
                self.p.data.copy_(self._fz[4])
                self.phi.data.copy_(self._fz[5])
        torch.cuda.current_stream().wait_stream(side)
        while remaining >= batch and self.steps % batch == 0:
            g.replay()
            remaining -= batch
            h = state.cpu().numpy()
            self.t, pnorm, self.first_period_max, self.steps = float(h[0]), float(h[2]), float(h[3]), int(h[5])
            if h[4] != 0.0:
                raise capi.LoamError(1 + capi.ERROR_KINDS.index("InstabilityDetected"),
                                     f"wave field blew up at step {int(h[4])}")
            if self.steps % 100 == 0:
                self.samples.append((self.t, pnorm, L.inf_norm(self.phi), self.energy_dev()))
        for _ in range(remaining):
            self.step()
        torch.cuda.synchronize()
        return self.samples
