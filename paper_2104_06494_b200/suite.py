"""The fixed-parameter test suite (integrands.hpp:26-34, integrands.cpp:83-255).

Support code for true-error reporting (bench / CLI), not part of the hot path.
Reference values are evaluated in Python double precision from the same closed
forms the reference evaluates in long double (agreement ~1e-15 relative).

`reference_value(id, dim)` reproduces the reference, including its f6 defect
(integrands.cpp:129-136 does not clamp the cut-off (3+i)/10 to the unit cube,
so for dim >= 7 it returns the integral over a larger box); pass
`corrected=True` for the true integral over [0,1]^dim.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

from .api import Integrand, integrand_by_id


def _ref_f1(n):
    phase, p = 0.0, 1.0
    for i in range(1, n + 1):
        h = 0.5 * i
        phase += h
        p *= math.sin(h) / h
    return math.cos(phase) * p


def _ref_f2(n):
    return (100.0 * math.atan(25.0)) ** n


def _ref_f3(n):
    s = 0.0
    for mask in range(1 << n):
        denom, bits = 1.0, 0
        for i in range(n):
            if mask & (1 << i):
                denom += i + 1
                bits += 1
        s += (-1.0 if bits % 2 else 1.0) / denom
    scale = 1.0
    for i in range(1, n + 1):
        scale *= float(i) * i
    return s / scale


def _ref_f4(n):
    return (math.sqrt(math.pi) / 25.0 * math.erf(12.5)) ** n


def _ref_f5(n):
    return ((1.0 - math.exp(-5.0)) / 5.0) ** n


def _ref_f6(n, corrected=False):
    p = 1.0
    for i in range(1, n + 1):
        c = (3.0 + i) / 10.0
        if corrected:
            c = min(c, 1.0)
        p *= (math.exp((i + 4) * c) - 1.0) / (i + 4)
    return p


def _sum_sq_moment(d, k):
    binom = [[0.0] * (k + 1) for _ in range(k + 1)]
    for i in range(k + 1):
        binom[i][0] = 1.0
        for j in range(1, i + 1):
            binom[i][j] = binom[i - 1][j - 1] + (binom[i - 1][j] if j <= i - 1 else 0.0)
    g = [1.0 / (2 * j + 1) for j in range(k + 1)]
    for _ in range(2, d + 1):
        g = [sum(binom[kk][j] * (1.0 / (2 * j + 1)) * g[kk - j] for j in range(kk + 1))
             for kk in range(k + 1)]
    return g[k]


_F8 = {2: 2.9285329205389220, 3: 27.531960573226068, 8: 8879.8511754142763}


def reference_value(name: str, dim: int, corrected: bool = False) -> float:
    if dim < 1 or dim > 16:
        raise ValueError("reference_value: dimension out of range")
    if name == "f1":
        return _ref_f1(dim)
    if name == "f2":
        return _ref_f2(dim)
    if name == "f3":
        return _ref_f3(dim)
    if name == "f4":
        return _ref_f4(dim)
    if name == "f5":
        return _ref_f5(dim)
    if name == "f6":
        return _ref_f6(dim, corrected)
    if name == "f7":
        return _sum_sq_moment(dim, 11)
    if name == "f8":
        if dim not in _F8:
            raise ValueError("f8 reference available for n in {2,3,8}")
        return _F8[dim]
    raise ValueError("unknown integrand id: " + name)


@dataclass
class IntegrandSpec:
    id: str
    dim: int
    callable: Integrand
    reference_value: float
    oscillatory: bool
    headline: bool


def suite():
    """integrands.cpp:228-255: the nine headline configurations, f2 at 6, and
    every integrand at n in {2, 3}."""
    specs = []

    def add(i, d, headline):
        specs.append(IntegrandSpec(i, d, integrand_by_id(i), reference_value(i, d), i == "f1",
                                   headline))

    for i, d in (("f1", 8), ("f3", 8), ("f4", 8), ("f5", 8), ("f7", 8), ("f8", 8), ("f4", 5),
                 ("f6", 6), ("f3", 3)):
        add(i, d, True)
    add("f2", 6, False)
    for d in (2, 3):
        for k in range(1, 9):
            i = f"f{k}"
            if not any(s.id == i and s.dim == d for s in specs):
                add(i, d, False)
    return specs
