"""Algorithmic work per unit for the roofline.

k_evaluate is FP64 CUDA-core bound.  Its algorithmic FLOPs per region
evaluation are the REFERENCE's arithmetic (rule.cpp:351-430 with
integrands.cpp:24-79), independent of how many instructions the kernel
actually executes (the kernel executes fewer: it never recomputes a value the
reference computes identically, see evaluate.cuh):

    F(f, n) = N(n) * (2n [map c + g*h] + 10 [5 x (mul+add)] + C_f(n)) + 11n + 2

with C_f the integrand's own flops (+,-,*,/ count 1; the libm routines count
their FP64 instructions with DFMA = 2, for the glibc restatement the device
actually runs, glibc_math.cuh):
    C_exp = 20   (e_exp.c main path: 8 DFMA + 4 DMUL/DADD/DSUB)
    C_cos = 41   (s_sin.c reduce_sincos 18 + avg(do_sin 24, do_cos 22))
    C_sqrt = 12  (__dsqrt_rn sequence, estimated)
f6 is counted as if every point were inside its box (upper bound).

The HBM-bound kernels' algorithmic bytes per region are in `bytes_*`.
"""
from __future__ import annotations

C_EXP = 20
C_COS = 41
C_SQRT = 12


def rule_points(n: int) -> int:
    return (1 << n) + 2 * n * (n - 1) + 4 * n + 1


def ipow_muls(e: int) -> int:
    muls = 0
    while e > 0:
        if e & 1:
            muls += 1
        muls += 1
        e >>= 1
    return muls


def integrand_flops(fid: int, n: int) -> int:
    """C_f(n) of SURVEY.md 8(d)."""
    if fid == 1:
        return 2 * n + C_COS
    if fid == 2:
        return 5 * n
    if fid == 3:
        return 2 * n + ipow_muls(n + 1) + 1
    if fid == 4:
        return 3 * n + 1 + C_EXP
    if fid == 5:
        return 2 * n + 1 + C_EXP
    if fid == 6:
        return 2 * n + C_EXP
    if fid == 7:
        return 2 * n + ipow_muls(11)
    if fid == 8:
        return 2 * n + ipow_muls(7) + 1 + C_SQRT
    raise ValueError(f"no flop model for integrand {fid}")


def region_flops(fid: int, n: int) -> int:
    """F(f, n): algorithmic FP64 FLOPs per region evaluation."""
    return rule_points(n) * (2 * n + 10 + integrand_flops(fid, n)) + 11 * n + 2


def bytes_evaluate(n: int) -> int:
    """k_evaluate HBM bytes per region: read low/len (16n) + parent est (8);
    write est, err (16) + axis, flag (2)."""
    return 16 * n + 8 + 18


def bytes_fold() -> int:
    """k_fold_eval: est + err + flag read (17 B; each read by two of the four folds,
    the second from L1/L2)."""
    return 17


def bytes_split(n: int, kept_fraction: float) -> float:
    """k_split: flag (1) for every region; kept ones read low/len/axis/est
    (16n + 9) and write two children low/len + parent est (2 * (16n + 8))."""
    return 1 + kept_fraction * (16 * n + 9 + 2 * (16 * n + 8))
