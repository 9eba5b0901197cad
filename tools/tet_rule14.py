"""Solve the symmetric 14-point tetrahedron quadrature rule (exact to degree 5).

The reference (`loam/fem/element.hpp:113-129`) tabulates tet rules only up to
degree 3, but config 3 asks for a degree-4, 14-point rule.  This script solves
the classical orbit structure -- two (a,b,b,b) orbits and one (c,c,d,d) orbit,
weights summing to the reference volume 1/6 -- by Newton/least squares on the
monomial moment equations, starting from the well-known published values, and
prints the constants at full double precision.  The output is pasted into
`oracle/loam_oracle.c` and `paper_1501_01809_b200/csrc/elements.cuh`.

Exactness is verified against the factorial formula
  int_T x^i y^j z^k = i! j! k! / (i+j+k+3)!
on the reference tetrahedron for every monomial of degree <= 5.
"""
from fractions import Fraction
from itertools import permutations
from math import factorial

import numpy as np
from scipy.optimize import least_squares


def points(p):
    b1, b2, c, w1, w2, w3 = p
    pts, wts = [], []
    for b, w in ((b1, w1), (b2, w2)):
        a = 1.0 - 3.0 * b
        for k in range(4):
            bary = [b] * 4
            bary[k] = a
            pts.append(bary[1:])
            wts.append(w)
    d = 0.5 - c
    seen = set()
    for perm in permutations([c, c, d, d]):
        if perm in seen:
            continue
        seen.add(perm)
        pts.append(list(perm[1:]))
        wts.append(w3)
    return np.array(pts), np.array(wts)


MONOS = [(i, j, k) for i in range(6) for j in range(6) for k in range(6) if i + j + k <= 5]


def exact(i, j, k):
    return factorial(i) * factorial(j) * factorial(k) / factorial(i + j + k + 3)


def residual(p):
    pts, wts = points(p)
    return np.array([np.sum(wts * pts[:, 0] ** i * pts[:, 1] ** j * pts[:, 2] ** k) - exact(i, j, k)
                     for (i, j, k) in MONOS])


def main():
    p0 = [0.0927352503108912, 0.3108859192633006, 0.4544962958743504,
          0.01224884051939366, 0.01878132095300264, 0.007091003462846911]
    sol = least_squares(residual, p0, xtol=1e-15, ftol=1e-15, gtol=1e-15)
    p = sol.x
    err = np.max(np.abs(residual(p)))
    assert err < 1e-16, err
    pts, wts = points(p)
    assert abs(wts.sum() - 1.0 / 6.0) < 1e-16
    names = ["b1", "b2", "c", "w1", "w2", "w3"]
    for n, v in zip(names, p):
        print(f"{n} = {v!r}")
    print("max moment error", err)


if __name__ == "__main__":
    main()
