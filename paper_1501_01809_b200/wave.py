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
sequential sums as in the reference) match bench::run_wave's samples.
"""
from __future__ import annotations

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
