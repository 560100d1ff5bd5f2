"""TEST INFRASTRUCTURE ONLY: ctypes bindings to the checkers under oracle/.

* `Ref`    -> oracle/_ref/libbfcub_ref.so, the UNMODIFIED reference library
              (/root/reference/proj/src) behind oracle/ref_shim.cpp.
* `Port`   -> oracle/liboracle.so, the plain-C restatement (pagani_oracle.c).

Both expose the same surface (integrate / trace / evaluate_batch / ...), so
tests can run the same check against either.  Only tests/, smoke() and the
bench CPU-baseline arm may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libbfcub_ref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")

STATUS = {0: "converged", 1: "max_iterations", 2: "memory_exhausted"}


class RefConfig(C.Structure):
    _fields_ = [("tau_rel", C.c_double), ("tau_abs", C.c_double),
                ("it_max", C.c_int32), ("init_subdiv", C.c_int32),
                ("max_regions", C.c_int64), ("init_target", C.c_int64),
                ("rel_filtering_enabled", C.c_int32), ("threads", C.c_int32),
                ("validate_invariants", C.c_int32), ("refiner", C.c_int32),
                ("direction_change_limit", C.c_int32), ("attempt_limit", C.c_int32),
                ("p_max_start", C.c_double), ("p_max_step", C.c_double),
                ("p_max_cap", C.c_double)]


def make_config(tau_rel=1e-3, tau_abs=1e-20, it_max=100, max_regions=1 << 22,
                init_target=1 << 14, init_subdiv=0, rel_filtering_enabled=True,
                threads=0, validate_invariants=False, refiner=0,
                direction_change_limit=4, attempt_limit=40, p_max_start=0.25,
                p_max_step=0.10, p_max_cap=0.95) -> RefConfig:
    """Defaults = bfcub::Config (driver.hpp:30-45) + ThresholdLimits (classify.hpp:23-29)."""
    return RefConfig(tau_rel, tau_abs, it_max, init_subdiv, max_regions, init_target,
                     int(bool(rel_filtering_enabled)), threads, int(bool(validate_invariants)),
                     refiner, direction_change_limit, attempt_limit, p_max_start,
                     p_max_step, p_max_cap)


class RefEvent(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("success", C.c_int32),
                ("batch_size", C.c_int64), ("finished_count", C.c_int64),
                ("discarded_error", C.c_double), ("budget_limit", C.c_double)]


class RefResult(C.Structure):
    _fields_ = [("estimate", C.c_double), ("errorest", C.c_double),
                ("status", C.c_int32), ("iterations", C.c_int32),
                ("regions_generated", C.c_int64), ("eval_count", C.c_int64),
                ("n_events", C.c_int32), ("pad", C.c_int32)]


class TraceRow(C.Structure):
    _fields_ = [("it", C.c_int32), ("trig_digits", C.c_int32), ("trig_memory", C.c_int32),
                ("thr_invoked", C.c_int32),
                ("m", C.c_int64), ("active_rel", C.c_int64), ("active_final", C.c_int64),
                ("kept", C.c_int64),
                ("v", C.c_double), ("e", C.c_double), ("v_f", C.c_double), ("e_f", C.c_double),
                ("fin_v", C.c_double), ("fin_e", C.c_double),
                ("thr_success", C.c_int32), ("thr_accepted", C.c_int32),
                ("thr_attempts", C.c_int32), ("thr_dir_changes", C.c_int32),
                ("thr_threshold", C.c_double), ("thr_discarded", C.c_double),
                ("thr_budget", C.c_double), ("thr_finished", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ThrOut(C.Structure):
    _fields_ = [("success", C.c_int32), ("attempts", C.c_int32),
                ("direction_changes", C.c_int32), ("pad", C.c_int32),
                ("threshold", C.c_double), ("discarded_error", C.c_double),
                ("budget_limit", C.c_double), ("finished_count", C.c_int64)]


@dataclass
class Result:
    estimate: float
    errorest: float
    status: str
    iterations: int
    regions_generated: int
    eval_count: int
    threshold_events: list = field(default_factory=list)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _params(params):
    p = np.zeros(32, dtype=np.float64)
    if params is not None:
        p[:len(params)] = params
    return p, (0 if params is None else len(params))


class _Lib:
    prefix = "ref_"

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (see oracle/Makefile)")
        self.lib = C.CDLL(path)
        self.path = path
        self._sig()

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _sig(self):
        f = self.fn
        f("last_error").restype = C.c_char_p
        f("block_sum").restype = C.c_double
        f("block_sum_where").restype = C.c_double
        f("reference_value").restype = C.c_double
        f("call_integrand").restype = C.c_double
        f("rule_point_count").restype = C.c_int64
        f("rule_point_count").argtypes = [C.c_int]
        for name in ("block_sum", "block_sum_where", "reference_value", "call_integrand",
                     "digits_converged"):
            f(name).argtypes = None
        f("digits_converged").argtypes = [C.c_double, C.c_double, C.c_int]
        f("convergence_digits").argtypes = [C.c_double]
        f("initial_subdivisions").argtypes = [C.c_int, C.c_int64]

    def _check(self, rc):
        if rc < 0:
            msg = self.fn("last_error")().decode()
            exc = {-1: ValueError, -2: RuntimeError, -3: AssertionError}.get(rc, RuntimeError)
            raise exc(msg)
        return rc

    # -- driver --------------------------------------------------------------
    def integrate(self, fid, ndim, cfg=None, lower=None, upper=None, params=None):
        cfg = cfg or make_config()
        lo = np.zeros(ndim) if lower is None else np.asarray(lower, dtype=np.float64)
        hi = np.ones(ndim) if upper is None else np.asarray(upper, dtype=np.float64)
        p, npar = _params(params)
        out = RefResult()
        ev = (RefEvent * 512)()
        rc = self.fn("integrate")(fid, _dp(p), npar, ndim, _dp(lo), _dp(hi), C.byref(cfg),
                                  C.byref(out), ev, 512)
        self._check(rc)
        events = [dict(iteration=e.iteration, success=bool(e.success), batch_size=e.batch_size,
                       finished_count=e.finished_count, discarded_error=e.discarded_error,
                       budget_limit=e.budget_limit) for e in ev[:min(out.n_events, 512)]]
        return Result(out.estimate, out.errorest, STATUS[out.status], out.iterations,
                      out.regions_generated, out.eval_count, events)

    def trace(self, fid, ndim, cfg=None, params=None, max_rows=200):
        cfg = cfg or make_config()
        p, npar = _params(params)
        out = RefResult()
        rows = (TraceRow * max_rows)()
        n = self._check(self.fn("trace")(fid, _dp(p), npar, ndim, C.byref(cfg), C.byref(out),
                                         rows, max_rows))
        res = Result(out.estimate, out.errorest, STATUS[out.status], out.iterations,
                     out.regions_generated, out.eval_count)
        return res, [rows[i].as_dict() for i in range(min(n, max_rows))]

    # -- batch functions -----------------------------------------------------
    def evaluate_batch(self, fid, lows, lengths, params=None):
        lows = np.ascontiguousarray(lows, dtype=np.float64)
        lengths = np.ascontiguousarray(lengths, dtype=np.float64)
        m, n = lows.shape
        p, npar = _params(params)
        est = np.empty(m)
        raw = np.empty(m)
        axes = np.empty(m, dtype=np.int32)
        cnt = C.c_int64()
        self._check(self.fn("evaluate_batch")(fid, _dp(p), npar, n, C.c_int64(m), _dp(lows),
                                              _dp(lengths), _dp(est), _dp(raw), _i32p(axes),
                                              C.byref(cnt)))
        return est, raw, axes, cnt.value

    def build_rule(self, n):
        N = self.fn("rule_point_count")(n)
        pts = np.empty((N, n))
        w = np.empty((5, N))
        probes = np.empty(4 * n, dtype=np.int32)
        self._check(self.fn("build_rule")(n, _dp(pts), _dp(w), _i32p(probes)))
        return pts, w, probes

    def two_level_refine(self, est, raw, pest, perr):
        a = [np.ascontiguousarray(x, dtype=np.float64) for x in (est, raw, pest, perr)]
        out = np.empty(len(a[0]))
        self._check(self.fn("two_level_refine")(C.c_int64(len(a[0])), *[_dp(x) for x in a],
                                                _dp(out)))
        return out

    def rel_err_classify(self, est, err, tau, enabled=True):
        est = np.ascontiguousarray(est, dtype=np.float64)
        err = np.ascontiguousarray(err, dtype=np.float64)
        fl = np.empty(len(est), dtype=np.uint8)
        self._check(self.fn("rel_err_classify")(C.c_int64(len(est)), _dp(est), _dp(err),
                                                C.c_double(tau), int(enabled), _u8p(fl)))
        return fl

    def threshold_classify(self, active, errors, v_tot, e_tot, e_it, s_it, tau, cfg=None):
        active = np.ascontiguousarray(active, dtype=np.uint8)
        errors = np.ascontiguousarray(errors, dtype=np.float64)
        fl = np.empty(len(errors), dtype=np.uint8)
        out = ThrOut()
        self._check(self.fn("threshold_classify")(
            C.c_int64(len(errors)), _u8p(active), _dp(errors), C.c_double(v_tot),
            C.c_double(e_tot), C.c_double(e_it), C.c_int64(s_it), C.c_double(tau),
            C.byref(cfg) if cfg is not None else None, _u8p(fl), C.byref(out)))
        return dict(success=bool(out.success), flags=fl, threshold=out.threshold,
                    discarded_error=out.discarded_error, budget_limit=out.budget_limit,
                    finished_count=out.finished_count, attempts=out.attempts,
                    direction_changes=out.direction_changes)

    def filter(self, lows, lengths, est, err, axis, pest, perr, flags):
        lows = np.ascontiguousarray(lows, dtype=np.float64)
        lengths = np.ascontiguousarray(lengths, dtype=np.float64)
        m, n = lows.shape
        a = [np.ascontiguousarray(x, dtype=np.float64) for x in (est, err)]
        axis = np.ascontiguousarray(axis, dtype=np.int32)
        b = [np.ascontiguousarray(x, dtype=np.float64) for x in (pest, perr)]
        flags = np.ascontiguousarray(flags, dtype=np.uint8)
        kl, kn = np.empty((m, n)), np.empty((m, n))
        ke, kr, kp, kq = (np.empty(m) for _ in range(4))
        ka = np.empty(m, dtype=np.int32)
        kept = C.c_int64()
        fe, fr, fv = C.c_double(), C.c_double(), C.c_double()
        self._check(self.fn("filter")(n, C.c_int64(m), _dp(lows), _dp(lengths), _dp(a[0]),
                                      _dp(a[1]), _i32p(axis), _dp(b[0]), _dp(b[1]),
                                      _u8p(flags), _dp(kl), _dp(kn), _dp(ke), _dp(kr),
                                      _i32p(ka), _dp(kp), _dp(kq), C.byref(kept),
                                      C.byref(fe), C.byref(fr), C.byref(fv)))
        k = kept.value
        return dict(lows=kl[:k], lengths=kn[:k], estimates=ke[:k], errors=kr[:k],
                    split_axis=ka[:k], parent_estimates=kp[:k], parent_errors=kq[:k],
                    finished_estimate=fe.value, finished_error=fr.value,
                    finished_volume=fv.value, kept=k)

    def bisect(self, lows, lengths, est, err, axis, max_regions=1 << 22):
        lows = np.ascontiguousarray(lows, dtype=np.float64)
        lengths = np.ascontiguousarray(lengths, dtype=np.float64)
        m, n = lows.shape
        est = np.ascontiguousarray(est, dtype=np.float64)
        err = np.ascontiguousarray(err, dtype=np.float64)
        axis = np.ascontiguousarray(axis, dtype=np.int32)
        cl, cn = np.empty((2 * m, n)), np.empty((2 * m, n))
        cp, cq = np.empty(2 * m), np.empty(2 * m)
        self._check(self.fn("bisect")(n, C.c_int64(m), _dp(lows), _dp(lengths), _dp(est),
                                      _dp(err), _i32p(axis), C.c_int64(max_regions), _dp(cl),
                                      _dp(cn), _dp(cp), _dp(cq)))
        return cl, cn, cp, cq

    def uniform_split(self, lower, upper, d, max_regions=1 << 22):
        lo = np.asarray(lower, dtype=np.float64)
        hi = np.asarray(upper, dtype=np.float64)
        n = len(lo)
        cap = 1
        for _ in range(n):
            cap *= d
        cnt = C.c_int64()
        cap = min(cap, max_regions, 1 << 24)
        lows, lens = np.empty((cap, n)), np.empty((cap, n))
        self._check(self.fn("uniform_split")(n, _dp(lo), _dp(hi), d, C.c_int64(max_regions),
                                             C.byref(cnt), _dp(lows), _dp(lens),
                                             C.c_int64(cap)))
        return lows[:cnt.value], lens[:cnt.value]

    def initial_subdivisions(self, n, target=1 << 14):
        return self.fn("initial_subdivisions")(n, C.c_int64(target))

    def block_sum(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.fn("block_sum")(C.c_int64(len(x)), _dp(x))

    def block_sum_where(self, x, flags, which):
        x = np.ascontiguousarray(x, dtype=np.float64)
        flags = np.ascontiguousarray(flags, dtype=np.uint8)
        return self.fn("block_sum_where")(C.c_int64(len(x)), _dp(x), _u8p(flags),
                                          C.c_int(which))

    def digits_converged(self, a, b, digits):
        return bool(self.fn("digits_converged")(a, b, digits))

    def convergence_digits(self, tau):
        return self.fn("convergence_digits")(C.c_double(tau))

    def call_integrand(self, fid, x, params=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        p, npar = _params(params)
        return self.fn("call_integrand")(C.c_int(fid), _dp(p), C.c_int(npar), _dp(x),
                                         C.c_int(len(x)))


class Ref(_Lib):
    """The unmodified reference library (oracle/_ref)."""
    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)

    def reference_value(self, fid_name, dim):
        return self.fn("reference_value")(fid_name.encode(), C.c_int(dim))

    def integrate_sequential(self, fid, ndim, tau_rel, tau_abs=1e-20, max_evals=10_000_000,
                             params=None, lower=None, upper=None):
        p, npar = _params(params)
        lo = np.zeros(ndim) if lower is None else np.asarray(lower, dtype=np.float64)
        hi = np.ones(ndim) if upper is None else np.asarray(upper, dtype=np.float64)
        out = RefResult()
        self._check(self.fn("integrate_sequential")(
            fid, _dp(p), npar, ndim, _dp(lo), _dp(hi), C.c_double(tau_rel),
            C.c_double(tau_abs), C.c_int64(max_evals), C.byref(out)))
        return Result(out.estimate, out.errorest, STATUS[out.status], out.iterations,
                      out.regions_generated, out.eval_count)


class Port(_Lib):
    """The plain-C restatement (oracle/pagani_oracle.c)."""
    prefix = "orc_"

    def __init__(self, path=PORT_SO):
        super().__init__(path)


def available(kind="ref"):
    return os.path.exists(REF_SO if kind == "ref" else PORT_SO)
