"""Python mirror of the reference's public API (`bfcub`, /root/reference/proj/include/bfcub).

Same names, argument meanings and error behaviour, so code written against the
reference reads the same:

    from paper_2104_06494_b200 import integrate, integrand_by_id, Bounds, Config
    res = integrate(integrand_by_id("f4"), Bounds.unit_cube(5), Config(tau_rel=1e-3))

Every call goes through the C ABI (include/pagani.h) into hand-written sm_100a
kernels; there is no CPU fallback.  Exceptions follow the reference's classes:
std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError,
std::logic_error -> AssertionError (see _native.check).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N

kMaxDim = 16  # geometry.hpp:8
kTwoLevelFloor = 0.125  # errorest.hpp:12


def _lib():
    return N.load()


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- types ----
class Status(enum.IntEnum):
    """driver.hpp:14"""
    Converged = 0
    MaxIterations = 1
    MemoryExhausted = 2

    def __str__(self):  # driver.cpp:19-26
        return {0: "converged", 1: "max_iterations", 2: "memory_exhausted"}[int(self)]


def to_string(s: Status) -> str:
    return str(Status(s))


class Bounds:
    """geometry.hpp:11-23; validated like geometry.cpp:9-23."""

    def __init__(self, lower: Sequence[float], upper: Sequence[float]):
        lower = [float(x) for x in lower]
        upper = [float(x) for x in upper]
        if len(lower) != len(upper):
            raise ValueError("Bounds: lower/upper size mismatch")
        n = len(lower)
        if n < 1 or n > kMaxDim:
            raise ValueError(f"Bounds: dimension must be in [1, {kMaxDim}]")
        for lo, hi in zip(lower, upper):
            if not lo < hi:
                raise ValueError("Bounds: lower must be < upper on every axis")
            if not (math.isfinite(lo) and math.isfinite(hi)):
                raise ValueError("Bounds: entries must be finite")
        self.lower, self.upper = lower, upper

    @staticmethod
    def unit_cube(n: int) -> "Bounds":
        return Bounds([0.0] * n, [1.0] * n)

    def dim(self) -> int:
        return len(self.lower)

    def volume(self) -> float:
        v = 1.0
        for lo, hi in zip(self.lower, self.upper):
            v *= hi - lo
        return v

    def is_unit_cube(self) -> bool:
        return all(lo == 0.0 and hi == 1.0 for lo, hi in zip(self.lower, self.upper))


@dataclass
class ThresholdLimits:
    """classify.hpp:23-29"""
    direction_change_limit: int = 4
    attempt_limit: int = 40
    p_max_start: float = 0.25
    p_max_step: float = 0.10
    p_max_cap: float = 0.95


@dataclass
class Config:
    """driver.hpp:30-45 (+ B200 knobs: mode, device, profile)."""
    tau_rel: float = 1e-3
    tau_abs: float = 1e-20
    it_max: int = 100
    max_regions: int = 1 << 22
    init_target: int = 1 << 14
    init_subdiv: int = 0
    rel_filtering_enabled: bool = True
    threads: int = 0
    validate_invariants: bool = False
    refiner: str = "two_level"  # Config::refiner fn pointer -> "two_level" | "identity"
    threshold_limits: ThresholdLimits = field(default_factory=ThresholdLimits)
    mode: str = "parity"  # "parity" (bit-exact) | "fast"
    device: int = 0
    profile: int = 0  # 1 (or True): every kernel class timed; 2: k_evaluate only (cheap)
    comm: object = None  # dist.Communicator for multi-GPU runs (one process per GPU)

    def convergence_digits(self) -> int:  # driver.cpp:28-33
        return _lib().pagani_convergence_digits(self.tau_rel)

    def validate(self) -> None:  # driver.cpp:35-41
        if not self.tau_rel > 0.0:
            raise ValueError("Config: tau_rel must be > 0")
        if not self.tau_abs >= 0.0:
            raise ValueError("Config: tau_abs must be >= 0")
        if self.it_max < 1:
            raise ValueError("Config: it_max must be >= 1")
        if self.init_subdiv == 0 and self.max_regions < 2 * self.init_target:
            raise ValueError("Config: max_regions must be >= 2 * init_target")

    def to_c(self) -> N.Config:
        c = N.Config()
        _lib().pagani_config_default(C.byref(c))
        c.tau_rel, c.tau_abs = self.tau_rel, self.tau_abs
        c.it_max, c.init_subdiv = self.it_max, self.init_subdiv
        c.max_regions, c.init_target = self.max_regions, self.init_target
        c.rel_filtering_enabled = int(bool(self.rel_filtering_enabled))
        c.threads = self.threads
        c.validate_invariants = int(bool(self.validate_invariants))
        c.refiner = {"two_level": N.REFINER_TWO_LEVEL, "identity": N.REFINER_IDENTITY}[self.refiner]
        L = self.threshold_limits
        c.direction_change_limit, c.attempt_limit = L.direction_change_limit, L.attempt_limit
        c.p_max_start, c.p_max_step, c.p_max_cap = L.p_max_start, L.p_max_step, L.p_max_cap
        c.mode = {"parity": N.MODE_PARITY, "fast": N.MODE_FAST}[self.mode]
        c.device = self.device
        c.profile = int(self.profile) if not isinstance(self.profile, bool) else int(self.profile)
        c.comm = self.comm.handle if self.comm is not None else None
        return c


@dataclass
class ThresholdEvent:
    """driver.hpp:47-58"""
    iteration: int = 0
    success: bool = False
    batch_size: int = 0
    finished_count: int = 0
    discarded_error: float = 0.0
    budget_limit: float = 0.0

    def retained_fraction(self) -> float:
        return 1.0 - self.finished_count / self.batch_size if self.batch_size else 1.0


@dataclass
class IntegrationResult:
    """driver.hpp:60-68 (+ device timing)."""
    estimate: float = 0.0
    errorest: float = 0.0
    status: Status = Status.MaxIterations
    iterations: int = 0
    regions_generated: int = 0
    eval_count: int = 0
    threshold_events: List[ThresholdEvent] = field(default_factory=list)
    wall_ms: float = 0.0
    kernel_ms: dict = field(default_factory=dict)
    kernel_launches: dict = field(default_factory=dict)
    kernel_bytes: dict = field(default_factory=dict)  # algorithmic HBM bytes per kernel kind
    region_evals: int = 0
    peak_regions: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    device_ms: float = 0.0
    probe_fallbacks: int = 0  # streamed threshold passes re-run exactly
    trace: Optional[list] = None
    spec_probe_passes: int = 0  # first passes queued behind k_finalize
    spec_probe_wasted: int = 0  # ... of which no search used


# ----------------------------------------------------------- integrands ----
class Integrand:
    """Replaces bfcub::Integrand (integrand.hpp:8-13).

    The device cannot call a host function pointer, so an Integrand names a
    device implementation: the reference suite f1..f8 (integrand_by_id) or one
    of the reference unit-test integrands (constructors below).  Passing a
    Python callable raises NotImplementedError (no CPU fallback).
    """
    IDS = {f"f{i}": i for i in range(1, 9)}

    def __init__(self, builtin_id: int, params: Sequence[float] = ()):
        self.builtin_id = int(builtin_id)
        self.params = [float(p) for p in params]

    def to_c(self) -> N.Integrand:
        f = N.Integrand()
        arr = (C.c_double * N.PAGANI_MAX_PARAMS)(*self.params)
        _lib().pagani_integrand_builtin(C.byref(f), self.builtin_id, arr, len(self.params))
        return f

    def __repr__(self):
        return f"Integrand(id={self.builtin_id}, params={self.params})"

    # reference unit-test lambdas (include/pagani.h PAGANI_TEST_*)
    @staticmethod
    def constant(v: float = 1.0):
        return Integrand(100, [v])

    @staticmethod
    def monomial(exponents: Sequence[int]):
        return Integrand(101, [float(e) for e in exponents])

    @staticmethod
    def rough(freq: float, power: int, offset_per_dim: float):
        return Integrand(102, [freq, float(power), offset_per_dim])

    @staticmethod
    def nan_box(x0: float, x1: float = -1.0):
        return Integrand(103, [x0, x1])

    @staticmethod
    def pocket(p: float = 0.95):
        return Integrand(104, [p])

    @staticmethod
    def cos_sum(scale: float, freqs: Sequence[float]):
        return Integrand(105, [scale] + [float(f) for f in freqs])

    @staticmethod
    def exp_sq():
        return Integrand(106, [])

    def __call__(self, x, n=None):
        """Evaluate at host points (m x n) on the device."""
        x = _f64(np.atleast_2d(x))
        m, n = x.shape
        y = np.empty(m)
        f = self.to_c()
        N.check(_lib().pagani_call_integrand(C.byref(f), n, m, _dp(x), _dp(y)))
        return y if y.size > 1 else float(y[0])


def integrand_by_id(name: str) -> Integrand:
    """integrands.hpp:31 (integrands.cpp:216-220)."""
    if name not in Integrand.IDS:
        raise ValueError("unknown integrand id: " + name)
    return Integrand(Integrand.IDS[name])


def known_integrand(name: str) -> bool:
    return name in Integrand.IDS


def _as_integrand(f) -> Integrand:
    if isinstance(f, Integrand):
        return f
    if isinstance(f, str):
        return integrand_by_id(f)
    raise NotImplementedError(
        "host callables cannot run on the GPU (no CPU fallback); use integrand_by_id() "
        "or an Integrand test constructor")


# --------------------------------------------------------------- driver ----
def integrate(f, bounds: Bounds, config: Optional[Config] = None,
              trace: bool = False) -> IntegrationResult:
    """driver.hpp:77-79 -- breadth-first adaptive integration on the GPU."""
    config = config or Config()
    fi = _as_integrand(f)
    cf = fi.to_c()
    cc = config.to_c()
    rows = []
    if trace:
        def _cb(row_p, _user):
            rows.append(row_p.contents.as_dict())
        cb = N.TRACE_FN(_cb)
        cc.trace = cb
    n = bounds.dim()
    lo = (C.c_double * n)(*bounds.lower)
    hi = (C.c_double * n)(*bounds.upper)
    out = N.Result()
    N.check(_lib().pagani_integrate(C.byref(cf), n, lo, hi, C.byref(cc), C.byref(out)))
    ne = min(out.n_events, N.PAGANI_MAX_EVENTS)
    events = [ThresholdEvent(e.iteration, bool(e.success), e.batch_size, e.finished_count,
                             e.discarded_error, e.budget_limit) for e in out.events[:ne]]
    return IntegrationResult(
        estimate=out.estimate, errorest=out.errorest, status=Status(out.status),
        iterations=out.iterations, regions_generated=out.regions_generated,
        eval_count=out.eval_count, threshold_events=events, wall_ms=out.wall_ms,
        kernel_ms={k: out.kernel_ms[i] for i, k in enumerate(N.KERNEL_SLOTS)},
        kernel_launches={k: out.kernel_launches[i] for i, k in enumerate(N.KERNEL_SLOTS)},
        kernel_bytes={k: out.kernel_bytes[i] for i, k in enumerate(N.KERNEL_SLOTS)},
        region_evals=out.region_evals, peak_regions=out.peak_regions,
        h2d_bytes=out.h2d_bytes, d2h_bytes=out.d2h_bytes, device_ms=out.device_ms,
        probe_fallbacks=out.probe_fallbacks, trace=rows if trace else None,
        spec_probe_passes=out.spec_probe_passes, spec_probe_wasted=out.spec_probe_wasted)


def integrate_sequential(f, bounds: Bounds, tau_rel: float, tau_abs: float = 1e-20,
                         max_evals: int = 10_000_000, validate_invariants: bool = False,
                         device: int = 0, mode: str = "parity") -> IntegrationResult:
    """sequential.hpp:15-18 -- the reference's globally adaptive comparison
    engine (one max-error region per step), each step's two children
    evaluated and refined on the GPU; bit-identical to the reference."""
    fi = _as_integrand(f)
    cf = fi.to_c()
    n = bounds.dim()
    lo = (C.c_double * n)(*bounds.lower)
    hi = (C.c_double * n)(*bounds.upper)
    out = N.Result()
    md = {"parity": N.MODE_PARITY, "fast": N.MODE_FAST}[mode]
    N.check(_lib().pagani_integrate_sequential(C.byref(cf), n, lo, hi, tau_rel, tau_abs,
                                               max_evals, int(validate_invariants), device, md,
                                               C.byref(out)))
    return IntegrationResult(
        estimate=out.estimate, errorest=out.errorest, status=Status(out.status),
        iterations=out.iterations, regions_generated=out.regions_generated,
        eval_count=out.eval_count, threshold_events=[], wall_ms=out.wall_ms,
        kernel_ms={k: out.kernel_ms[i] for i, k in enumerate(N.KERNEL_SLOTS)},
        kernel_launches={k: out.kernel_launches[i] for i, k in enumerate(N.KERNEL_SLOTS)},
        kernel_bytes={k: out.kernel_bytes[i] for i, k in enumerate(N.KERNEL_SLOTS)},
        region_evals=out.region_evals, peak_regions=out.peak_regions,
        h2d_bytes=out.h2d_bytes, d2h_bytes=out.d2h_bytes, device_ms=out.device_ms, trace=None)


def check_termination(v, e, v_f, e_f, tau_rel, tau_abs) -> bool:  # driver.hpp:71-72
    return bool(_lib().pagani_check_termination(v, e, v_f, e_f, tau_rel, tau_abs))


def digits_converged(v_prev: float, v_curr: float, digits: int) -> bool:  # driver.hpp:74-75
    return bool(_lib().pagani_digits_converged(v_prev, v_curr, digits))


# ---------------------------------------------------------------- rule ----
def rule_point_count(n: int) -> int:  # rule.hpp:51
    return int(_lib().pagani_rule_point_count(n))


def build_rule(n: int):
    """rule.hpp:53.  Returns (orbit_weights[5 sets][5 orbits], generators l2..l5,
    points N x n, weight_sets 5 x N)."""
    if n < 1 or n > kMaxDim:
        raise ValueError("build_rule: dimension out of range")
    Np = rule_point_count(n)
    w = np.empty(25)
    g = np.empty(4)
    pts = np.empty((Np, n))
    ws = np.empty((5, Np))
    N.check(_lib().pagani_build_rule(n, _dp(w), _dp(g), _dp(pts), _dp(ws)))
    return w.reshape(5, 5), g, pts, ws


def evaluate_batch(f, lows, lengths, mode: str = "parity"):
    """rule.hpp:67-68.  lows/lengths region-major (m x n).  Returns
    (estimates, raw_errors, split_axes, eval_count)."""
    fi = _as_integrand(f).to_c()
    lows, lengths = _f64(lows), _f64(lengths)
    m, n = lows.shape
    est, raw = np.empty(m), np.empty(m)
    axes = np.empty(m, dtype=np.int32)
    cnt = C.c_int64()
    N.check(_lib().pagani_evaluate_batch(C.byref(fi), n, m, _dp(lows), _dp(lengths), _dp(est),
                                         _dp(raw), _i32p(axes), C.byref(cnt),
                                         {"parity": 0, "fast": 1}[mode]))
    return est, raw, axes, cnt.value


# ----------------------------------------------------------- errorest ----
def two_level_refine(estimates, raw_errors, parent_estimates, parent_errors):
    """errorest.hpp:20-29."""
    a = [_f64(x) for x in (estimates, raw_errors, parent_estimates, parent_errors)]
    if len({len(x) for x in a}) != 1:
        raise ValueError("two_level_refine: array length mismatch")
    out = np.empty(len(a[0]))
    N.check(_lib().pagani_two_level_refine(len(a[0]), *[_dp(x) for x in a], _dp(out)))
    return out


# ----------------------------------------------------------- classify ----
def rel_err_classify(estimates, errors, tau_rel, filtering_enabled=True):
    """classify.hpp:16-18."""
    est, err = _f64(estimates), _f64(errors)
    if len(est) != len(err):
        raise ValueError("rel_err_classify: array length mismatch")
    fl = np.empty(len(est), dtype=np.uint8)
    N.check(_lib().pagani_rel_err_classify(len(est), _dp(est), _dp(err), tau_rel,
                                           int(bool(filtering_enabled)), _u8p(fl)))
    return fl


def apply_threshold(errors, t):
    """classify.hpp:21."""
    err = _f64(errors)
    fl = np.empty(len(err), dtype=np.uint8)
    N.check(_lib().pagani_apply_threshold(len(err), _dp(err), t, _u8p(fl)))
    return fl


@dataclass
class ThresholdResult:
    """classify.hpp:31-40"""
    success: bool
    flags: np.ndarray
    threshold: float
    discarded_error: float
    budget_limit: float
    finished_count: int
    attempts: int
    direction_changes: int


def threshold_classify(active, errors, v_tot, e_tot, e_it, s_it, tau_rel,
                       limits: Optional[ThresholdLimits] = None) -> ThresholdResult:
    """classify.hpp:46-50."""
    act = np.ascontiguousarray(active, dtype=np.uint8)
    err = _f64(errors)
    if len(act) != s_it or len(err) != s_it:
        raise ValueError("threshold_classify: array length mismatch")
    lim = limits or ThresholdLimits()
    cc = Config(threshold_limits=lim).to_c()
    fl = np.empty(len(err), dtype=np.uint8)
    out = N.ThresholdResult()
    N.check(_lib().pagani_threshold_classify(len(err), _u8p(act), _dp(err), v_tot, e_tot, e_it,
                                             s_it, tau_rel, C.byref(cc), _u8p(fl), C.byref(out)))
    return ThresholdResult(bool(out.success), fl, out.threshold, out.discarded_error,
                           out.budget_limit, out.finished_count, out.attempts,
                           out.direction_changes)


@dataclass
class RegionBatch:
    """geometry.hpp:29-47 (host copy; region-major like the reference)."""
    lows: np.ndarray
    lengths: np.ndarray
    estimates: np.ndarray = None
    errors: np.ndarray = None
    split_axis: np.ndarray = None
    parent_estimates: np.ndarray = None
    parent_errors: np.ndarray = None

    def __post_init__(self):
        self.lows, self.lengths = _f64(self.lows), _f64(self.lengths)
        m = self.lows.shape[0]
        for name, dt in (("estimates", np.float64), ("errors", np.float64),
                         ("split_axis", np.int32), ("parent_estimates", np.float64),
                         ("parent_errors", np.float64)):
            v = getattr(self, name)
            setattr(self, name, np.zeros(m, dtype=dt) if v is None
                    else np.ascontiguousarray(v, dtype=dt))

    @property
    def dim(self):
        return self.lows.shape[1]

    @property
    def count(self):
        return self.lows.shape[0]

    def volume(self, j):
        v = 1.0
        for x in self.lengths[j]:
            v *= float(x)
        return v

    def total_volume(self):
        s = 0.0
        for j in range(self.count):
            s += self.volume(j)
        return s


@dataclass
class FilterResult:
    """classify.hpp:52-58"""
    kept: RegionBatch
    finished_estimate: float
    finished_error: float
    finished_volume: float
    finished_count: int


def filter(batch: RegionBatch, flags) -> FilterResult:  # noqa: A001 - reference name
    """classify.hpp:62."""
    fl = np.ascontiguousarray(flags, dtype=np.uint8)
    m, n = batch.count, batch.dim
    if len(fl) != m:
        raise ValueError("filter: flag length mismatch")
    kl, kn = np.empty((m, n)), np.empty((m, n))
    ke, kr, kp, kq = (np.empty(m) for _ in range(4))
    ka = np.empty(m, dtype=np.int32)
    kept = C.c_int64()
    fe, fr, fv = C.c_double(), C.c_double(), C.c_double()
    N.check(_lib().pagani_filter(n, m, _dp(batch.lows), _dp(batch.lengths),
                                 _dp(batch.estimates), _dp(batch.errors),
                                 _i32p(batch.split_axis), _dp(batch.parent_estimates),
                                 _dp(batch.parent_errors), _u8p(fl), _dp(kl), _dp(kn),
                                 _dp(ke), _dp(kr), _i32p(ka), _dp(kp), _dp(kq), C.byref(kept),
                                 C.byref(fe), C.byref(fr), C.byref(fv)))
    k = kept.value
    rb = RegionBatch(kl[:k], kn[:k], ke[:k], kr[:k], ka[:k], kp[:k], kq[:k])
    return FilterResult(rb, fe.value, fr.value, fv.value, m - k)


# ------------------------------------------------------------ geometry ----
def bisect(batch: RegionBatch, max_regions: int) -> RegionBatch:
    """geometry.hpp:50-52."""
    m, n = batch.count, batch.dim
    cl, cn = np.empty((2 * m, n)), np.empty((2 * m, n))
    cp, cq = np.empty(2 * m), np.empty(2 * m)
    N.check(_lib().pagani_bisect(n, m, _dp(batch.lows), _dp(batch.lengths),
                                 _dp(batch.estimates), _dp(batch.errors),
                                 _i32p(batch.split_axis), max_regions, _dp(cl), _dp(cn),
                                 _dp(cp), _dp(cq)))
    return RegionBatch(cl, cn, parent_estimates=cp, parent_errors=cq)


def uniform_split(bounds: Bounds, d: int, max_regions: int = 1 << 22) -> RegionBatch:
    """geometry.hpp:45-48."""
    n = bounds.dim()
    lo = np.array(bounds.lower)
    hi = np.array(bounds.upper)
    cap = 1
    for _ in range(n):
        cap *= max(d, 1)
        if cap > max_regions:
            break
    cap = min(cap, max_regions)
    lows, lens = np.empty((cap, n)), np.empty((cap, n))
    cnt = C.c_int64()
    N.check(_lib().pagani_uniform_split(n, _dp(lo), _dp(hi), d, max_regions, C.byref(cnt),
                                        _dp(lows), _dp(lens), cap))
    return RegionBatch(lows[:cnt.value], lens[:cnt.value])


def initial_subdivisions(n: int, init_target: int) -> int:  # geometry.hpp:55
    return _lib().pagani_initial_subdivisions(n, init_target)


# -------------------------------------------------------------- reduce ----
def block_sum(x) -> float:
    x = _f64(x)
    out = C.c_double()
    N.check(_lib().pagani_block_sum(len(x), _dp(x), C.byref(out)))
    return out.value


def block_sum_where(x, flags, which: int) -> float:
    x = _f64(x)
    fl = np.ascontiguousarray(flags, dtype=np.uint8)
    out = C.c_double()
    N.check(_lib().pagani_block_sum_where(len(x), _dp(x), _u8p(fl), which, C.byref(out)))
    return out.value


def count_flags(flags, which: int) -> int:
    fl = np.ascontiguousarray(flags, dtype=np.uint8)
    out = C.c_int64()
    N.check(_lib().pagani_count_flags(len(fl), _u8p(fl), which, C.byref(out)))
    return out.value


def min_max(x):
    x = _f64(x)
    lo, hi = C.c_double(), C.c_double()
    N.check(_lib().pagani_min_max(len(x), _dp(x), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


# ---------------------------------------------------------- math check ----
def glibc_exp(x, on_device=True, paired=False):
    """glibc exp restatement (host build, or the device variant; paired: the
    two-point form the evaluator uses, x[2i] and x[2i+1] as one pair)."""
    x = _f64(x)
    y = np.empty_like(x)
    code = 2 if (paired and on_device) else int(bool(on_device))
    N.check(_lib().pagani_math_exp(len(x), _dp(x), _dp(y), code))
    return y


def glibc_cos(x, on_device=True, branch_free=False, paired=False):
    """glibc cos restatement.  on_device: the evaluator's device variant;
    paired: its two-point form (f1's hot path); branch_free: the branch-merged
    SIMT variant (kept as an alternative, measured slower on B200)."""
    x = _f64(x)
    y = np.empty_like(x)
    if paired and on_device:
        code = 4
    else:
        code = (2 if on_device else 3) if branch_free else int(bool(on_device))
    N.check(_lib().pagani_math_cos(len(x), _dp(x), _dp(y), code))
    return y


def fp64_peak(device: int = 0, seconds: float = 1.0):
    """Measured FP64 DFMA peak of `device`: (TFLOP/s, SM MHz seen by the kernel)."""
    t, mhz = C.c_double(), C.c_double()
    N.check(_lib().pagani_fp64_peak(device, seconds, C.byref(t), C.byref(mhz)))
    return t.value, mhz.value


def device_count() -> int:
    c = C.c_int(0)
    rc = _lib().pagani_device_count(C.byref(c))
    return c.value if rc == 0 else 0


def release() -> None:
    N.check(_lib().pagani_release())
