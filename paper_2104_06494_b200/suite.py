"""The fixed-parameter test suite (integrands.hpp:26-34, integrands.cpp:83-255).

Support code for true-error reporting (bench / CLI), not part of the hot path.
Reference values come from the library (csrc/suite.cpp): the reference's
long-double closed forms with the same glibc functions, bit-identical.

`reference_value(id, dim)` reproduces the reference, including its f6 defect
(integrands.cpp:129-136 does not clamp the cut-off (3+i)/10 to the unit cube,
so for dim >= 7 it returns the integral over a larger box); pass
`corrected=True` for the true integral over [0,1]^dim.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native as N
from .api import Integrand, integrand_by_id


def reference_value(name: str, dim: int, corrected: bool = False,
                    extended: bool = False) -> float:
    """integrands.cpp:178-188 reference_for: the reference's long-double closed
    forms, bit-identical (csrc/suite.cpp via pagani_reference_value).
    corrected: f6 over the unit cube (the reference's ref_f6 is not, n >= 7).
    extended: f8 beyond n in {2, 3, 8} (the reference's generator tool)."""
    if not isinstance(name, str):
        raise ValueError("unknown integrand id")
    out = C.c_double()
    flags = (N.PAGANI_REFVAL_CORRECTED if corrected else 0) | (
        N.PAGANI_REFVAL_EXTENDED if extended else 0)
    N.check(N.load().pagani_reference_value(name.encode(), dim, flags, C.byref(out)))
    return out.value


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
