"""BASELINE.json configurations: seeded synthetic inputs and their par_loops.

Inputs follow SURVEY 8d: reference mesh generators (mesh.hpp:96-214) plus
splitmix64-driven interior jitter, Fisher-Yates cell permutation and
coefficient fields (generator in csrc/meshgen.cpp, exposed through the C ABI).
Coefficient seeds, which BASELINE.json leaves open, are 1000 + config index.

  C1  P1 Helmholtz residual, unit square 512^2, jitter 0.2h seed 0, perm seed 1, u~U[0,1]
  C2  P1 Laplace CSR matrix, unit square 1024^2, jitter 0.2h seed 2, perm seed 3
  C3  P2 Helmholtz residual + matrix, unit cube 64^3 (6 tets/hex), jitter 0.15h seed 4,
      perm seed 5, u~U[-1,1] per P2 node
  C4  vector-P1 elasticity 3x3-blocked CSR, cube 96^3, jitter 0.1h seed 6, lambda=1, mu=0.5
  C5  Taylor-Hood P2-P1 Stokes 2x2 nested block CSR, square 768^2, jitter 0.2h seed 7, perm seed 8
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi

FULL = {1: 512, 2: 1024, 3: 64, 4: 96, 5: 768}
JITTER = {1: (0.2, 0), 2: (0.2, 2), 3: (0.15, 4), 4: (0.1, 6), 5: (0.2, 7)}
PERM_SEED = {1: 1, 2: 3, 3: 5, 4: None, 5: 8}
KAPPA = 1.0
LAME = (1.0, 0.5)
NU = 1.0


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


@dataclass
class MeshInputs:
    gdim: int
    n: int
    coords: np.ndarray   # [nv * gdim] fp64
    cv: np.ndarray       # [ncells * (gdim+1)] int32 (cell order possibly permuted)
    extra: dict = field(default_factory=dict)

    @property
    def nv(self):
        return self.coords.size // self.gdim

    @property
    def ncells(self):
        return self.cv.size // (self.gdim + 1)


def mesh(gdim: int, n: int, amp: float = 0.0, jitter_seed: int | None = None,
         perm_seed: int | None = None) -> MeshInputs:
    L = capi.lib()
    if gdim == 2:
        nv, nc = (n + 1) ** 2, 2 * n * n
        coords, cv = np.empty(nv * 2), np.empty(nc * 3, dtype=np.int32)
        capi.check(L.loam_gpu_unit_square_mesh(n, _dp(coords), _ip(cv)))
    else:
        nv, nc = (n + 1) ** 3, 6 * n ** 3
        coords, cv = np.empty(nv * 3), np.empty(nc * 4, dtype=np.int32)
        capi.check(L.loam_gpu_unit_cube_mesh(n, _dp(coords), _ip(cv)))
    if jitter_seed is not None and amp:
        capi.check(L.loam_gpu_jitter(gdim, n, amp, jitter_seed, _dp(coords)))
    if perm_seed is not None:
        capi.check(L.loam_gpu_permute_cells(nc, gdim + 1, perm_seed, _ip(cv)))
    return MeshInputs(gdim, n, coords, cv)


def p2_map(m: MeshInputs):
    row = 6 if m.gdim == 2 else 10
    cn = np.empty(m.ncells * row, dtype=np.int32)
    nn = capi.lib().loam_gpu_p2_cell_node_map(m.ncells, m.nv, m.gdim, _ip(m.cv), _ip(cn))
    if nn < 0:
        capi.check(-nn)
    return cn, int(nn)


def uniform(count: int, seed: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(count)
    capi.check(capi.lib().loam_gpu_uniform(count, seed, lo, hi, _dp(out)))
    return out


def config_inputs(cfg: int, n: int | None = None) -> MeshInputs:
    """Inputs of BASELINE config `cfg` (1..5) at size n (default: the full size)."""
    n = FULL[cfg] if n is None else n
    gdim = 3 if cfg in (3, 4) else 2
    amp, js = JITTER[cfg]
    m = mesh(gdim, n, amp, js, PERM_SEED[cfg])
    if cfg == 1:
        m.extra["u"] = uniform(m.nv, 1000, 0.0, 1.0)
    if cfg in (3, 5):
        cn, nn = p2_map(m)
        m.extra["p2"], m.extra["nn"] = cn, nn
    if cfg == 3:
        m.extra["u"] = uniform(m.extra["nn"], 1002, -1.0, 1.0)
    return m


# --------------------------------------------------------------------------- par_loops
class Workload:
    """One config's par_loop(s) built on the loam mirror (device-resident)."""

    def __init__(self, cfg: int, n: int | None = None, part: str | None = None, inputs: MeshInputs | None = None):
        from . import loam as L  # torch import deferred
        self.cfg, self.part = cfg, part
        m = self.inputs = config_inputs(cfg, n) if inputs is None else inputs
        self.L = L
        cells = L.Set(m.ncells, "cells")
        verts = L.Set(m.nv, "vertices")
        cvm = L.Map(cells, verts, m.gdim + 1, m.cv, "cell_vertex")
        X = L.Dat(verts, m.gdim, "coordinates")
        X.set_values(m.coords)
        self.cells, self.verts, self.cvm, self.X = cells, verts, cvm, X
        self.loops, self.outputs = [], []
        if cfg == 1:
            u = L.Dat(verts, 1, "u")
            u.set_values(m.extra["u"])
            b = L.Dat(verts, 1, "residual")
            k = L.kernel("helmholtz_action_p1_tri", KAPPA)
            self.loops.append(L.Parloop(k, cells, [L.arg(b, L.INC, cvm), L.arg(X, L.READ, cvm), L.arg(u, L.READ, cvm)]))
            self.outputs.append(b)
        elif cfg == 2:
            sp = L.build_sparsity(cvm, cvm)
            A = L.Mat(sp, "stiffness")
            k = L.kernel("stiffness_p1_tri")
            self.loops.append(L.Parloop(k, cells, [L.arg(A, L.INC, cvm, cvm), L.arg(X, L.READ, cvm)]))
            self.outputs.append(A)
        elif cfg == 3:
            nodes = L.Set(m.extra["nn"], "p2_nodes")
            cnm = L.Map(cells, nodes, 10, m.extra["p2"], "cell_node")
            self.nodes, self.cnm = nodes, cnm
            if part in (None, "residual"):
                u = L.Dat(nodes, 1, "u")
                u.set_values(m.extra["u"])
                b = L.Dat(nodes, 1, "residual")
                k = L.kernel("helmholtz_action_p2_tet", KAPPA)
                self.loops.append(L.Parloop(k, cells, [L.arg(b, L.INC, cnm), L.arg(X, L.READ, cvm), L.arg(u, L.READ, cnm)]))
                self.outputs.append(b)
            if part in (None, "matrix"):
                sp = L.build_sparsity(cnm, cnm)
                A = L.Mat(sp, "helmholtz")
                k = L.kernel("helmholtz_p2_tet", KAPPA)
                self.loops.append(L.Parloop(k, cells, [L.arg(A, L.INC, cnm, cnm), L.arg(X, L.READ, cvm)]))
                self.outputs.append(A)
        elif cfg == 4:
            dm = L.expanded_map(cvm, 3)
            sp = L.build_sparsity(cvm, cvm, 3, 3)
            A = L.Mat(sp, "elasticity")
            k = L.kernel("elasticity_p1_tet", *LAME)
            self.loops.append(L.Parloop(k, cells, [L.arg(A, L.INC, dm, dm), L.arg(X, L.READ, cvm)]))
            self.outputs.append(A)
            self.dof_map = dm
        elif cfg == 5:
            vnodes = L.Set(m.extra["nn"], "p2_nodes")
            vnm = L.Map(cells, vnodes, 6, m.extra["p2"], "velocity_node")
            vdm = L.expanded_map(vnm, 2)
            pm = cvm  # pressure P1 nodes = vertices
            spA = L.build_sparsity(vnm, vnm, 2, 2)
            spB = L.build_sparsity(pm, vnm, 1, 2)
            spBT = L.build_sparsity(vnm, pm, 2, 1)
            A, B, BT = L.Mat(spA, "A"), L.Mat(spB, "B"), L.Mat(spBT, "BT")
            self.loops.append(L.Parloop(L.kernel("stokes_a_p2_tri", NU), cells,
                                        [L.arg(A, L.INC, vdm, vdm), L.arg(X, L.READ, cvm)]))
            self.loops.append(L.Parloop(L.kernel("stokes_b_p2_tri"), cells,
                                        [L.arg(B, L.INC, pm, vdm), L.arg(X, L.READ, cvm)]))
            self.loops.append(L.Parloop(L.kernel("stokes_bt_p2_tri"), cells,
                                        [L.arg(BT, L.INC, vdm, pm), L.arg(X, L.READ, cvm)]))
            self.outputs += [A, BT, B]  # BlockMat [0][0]=A, [0][1]=B^T, [1][0]=B (solver.hpp:21-28)
            self.vnm, self.vdm = vnm, vdm

    def reset(self):
        """Fresh zero outputs, as assemble_* allocates them (assemble.hpp:89,111)."""
        for o in self.outputs:
            o.zero()

    def run(self):
        if self.cfg == 5:  # fem::assemble_blocks (fem/assemble.hpp:439-448): the three blocks in one call
            self.L.execute_blocks(self.loops)
            return
        for lp in self.loops:
            self.L.execute(lp)
