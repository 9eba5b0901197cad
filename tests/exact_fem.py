"""Exact symbolic integration of Lagrange basis products on affine simplices.

Independent checker for the element kernels (test-only).  Restates the
approach of the reference's tests/exact_fem.hpp:20-205 (barycentric
polynomials integrated with the factorial formula) and extends it to what
the reference lacks: P2 on tetrahedra (edge order (2,3),(1,3),(1,2),(0,3),
(0,2),(0,1)), linear elasticity and the Taylor-Hood Stokes blocks.
"""
from fractions import Fraction
from math import factorial

import numpy as np

TRI_EDGES = [(1, 2), (0, 2), (0, 1)]
TET_EDGES = [(2, 3), (1, 3), (1, 2), (0, 3), (0, 2), (0, 1)]


class Poly:
    def __init__(self, terms=None):
        self.t = dict(terms or {})

    @staticmethod
    def lam(i):
        e = [0, 0, 0, 0]
        e[i] = 1
        return Poly({tuple(e): 1.0})

    @staticmethod
    def const(c):
        return Poly({(0, 0, 0, 0): c} if c else {})

    def __add__(self, o):
        r = dict(self.t)
        for k, v in o.t.items():
            r[k] = r.get(k, 0.0) + v
        return Poly(r)

    def __mul__(self, o):
        if not isinstance(o, Poly):
            return Poly({k: v * o for k, v in self.t.items()})
        r = {}
        for a, ca in self.t.items():
            for b, cb in o.t.items():
                k = tuple(x + y for x, y in zip(a, b))
                r[k] = r.get(k, 0.0) + ca * cb
        return Poly(r)

    __rmul__ = __mul__

    def integrate(self, d, vol):
        tot = 0.0
        for e, c in self.t.items():
            num = 1
            for k in e:
                num *= factorial(k)
            tot += c * num / factorial(sum(e) + d) * factorial(d) * vol
        return tot


def geometry(X, d):
    X = np.asarray(X, dtype=float).reshape(d + 1, d)
    E = (X[1:] - X[0]).T  # J
    vol = abs(np.linalg.det(E)) / factorial(d)
    Jinv = np.linalg.inv(E)
    g = np.zeros((d + 1, d))
    g[1:] = Jinv  # grad lambda_k = row k-1 of J^{-1}
    g[0] = -g[1:].sum(axis=0)
    return g, vol


def basis(d, p):
    nv = d + 1
    if p == 1:
        return [Poly.lam(i) for i in range(nv)]
    out = [Poly.lam(i) * (Poly.lam(i) * 2.0 + Poly.const(-1.0)) for i in range(nv)]
    for a, b in (TRI_EDGES if d == 2 else TET_EDGES):
        out.append(Poly.lam(a) * Poly.lam(b) * 4.0)
    return out


def grads(d, p, g):
    """grad phi_i as d polynomials each."""
    nv = d + 1
    out = []
    if p == 1:
        for i in range(nv):
            out.append([Poly.const(g[i][c]) for c in range(d)])
        return out
    for i in range(nv):
        f = Poly.lam(i) * 4.0 + Poly.const(-1.0)
        out.append([f * g[i][c] for c in range(d)])
    for a, b in (TRI_EDGES if d == 2 else TET_EDGES):
        out.append([(Poly.lam(b) * g[a][c] + Poly.lam(a) * g[b][c]) * 4.0 for c in range(d)])
    return out


def mass(X, d, p):
    g, vol = geometry(X, d)
    B = basis(d, p)
    return np.array([[(bi * bj).integrate(d, vol) for bj in B] for bi in B])


def stiffness(X, d, p):
    g, vol = geometry(X, d)
    G = grads(d, p, g)
    n = len(G)
    K = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            K[i, j] = sum((G[i][c] * G[j][c]).integrate(d, vol) for c in range(d))
    return K


def elasticity(X, lam, mu):
    g, vol = geometry(X, 3)
    K = np.zeros((12, 12))
    for a in range(4):
        for dd in range(3):
            for b in range(4):
                for e in range(3):
                    v = mu * g[a][e] * g[b][dd] + lam * g[a][dd] * g[b][e]
                    if dd == e:
                        v += mu * g[a] @ g[b]
                    K[a * 3 + dd, b * 3 + e] = vol * v
    return K


def stokes(X, nu):
    """(A 12x12, B 3x12) for vector-P2 velocity / P1 pressure on a triangle."""
    K = stiffness(X, 2, 2)
    A = np.zeros((12, 12))
    for a in range(6):
        for b in range(6):
            for dd in range(2):
                A[a * 2 + dd, b * 2 + dd] = nu * K[a, b]
    g, vol = geometry(X, 2)
    G = grads(2, 2, g)
    B = np.zeros((3, 12))
    for q in range(3):
        for b in range(6):
            for e in range(2):
                B[q, b * 2 + e] = -(Poly.lam(q) * G[b][e]).integrate(2, vol)
    return A, B


def random_simplex(d, rng):
    while True:
        X = rng.uniform(-2.0, 2.0, size=(d + 1, d))
        E = X[1:] - X[0]
        v = np.linalg.det(E) / factorial(d)
        if v < 0:
            X[[d - 1, d]] = X[[d, d - 1]]
            v = -v
        if v > 0.05:
            return X.reshape(-1)
