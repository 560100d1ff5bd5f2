"""GPU parity tests: the sm_100a path (through the C ABI) against the
unmodified reference library (oracle/_ref) and the committed goldens.

Bar: bit-exact for everything (estimates, errors, split axes, counts, traces)
in parity mode; fast mode within 1e-12 relative with identical decisions.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import bits, load_golden, unhex
from ref_ctypes import make_config

pytestmark = pytest.mark.gpu

TOL_FAST = 1e-12  # north_star: final integral within 1e-12 relative


def cfg_pair(pg, tau, relf=True, **extra):
    """The same configuration for the product and the reference shim."""
    refkw = dict(extra)
    pgkw = dict(extra)
    if "refiner" in pgkw:
        pgkw["refiner"] = {0: "two_level", 1: "identity"}[pgkw["refiner"]]
    lim = {k: pgkw.pop(k) for k in ("attempt_limit", "direction_change_limit", "p_max_start",
                                    "p_max_step", "p_max_cap") if k in pgkw}
    if lim:
        pgkw["threshold_limits"] = pg.ThresholdLimits(**lim)
    return (pg.Config(tau_rel=tau, rel_filtering_enabled=relf, **pgkw),
            make_config(tau_rel=tau, rel_filtering_enabled=relf, **refkw))


def integrand(pg, fid, params=None):
    return pg.Integrand(fid, params or [])


def assert_same_result(res, want):
    assert res.estimate == unhex(want["estimate"]) or (
        np.isnan(res.estimate) and np.isnan(unhex(want["estimate"])))
    assert res.errorest == unhex(want["errorest"]) or (
        np.isinf(res.errorest) and np.isinf(unhex(want["errorest"])))
    assert str(res.status) == want["status"]
    assert res.iterations == want["iterations"]
    assert res.regions_generated == want["regions_generated"]
    assert res.eval_count == want["eval_count"]


def assert_same_trace(rows, want_rows, name):
    assert len(rows) == len(want_rows), name
    for got, want in zip(rows, want_rows):
        for k, v in want.items():
            w = unhex(v)
            g = got[k]
            assert g == w or (isinstance(w, float) and w != w and g != g), (name, got["it"], k, g, w)


# ----------------------------------------------------------- libm ----------
def test_device_glibc_exp_cos_bit_exact(pg, gpu, ref):
    rng = np.random.default_rng(5)
    for fn, libm, xs in (
            (pg.glibc_exp, ref.lib.ref_libm_exp,
             np.concatenate([rng.uniform(-1300, 720, 2_000_000), rng.uniform(-45, 45, 2_000_000),
                             rng.uniform(-760, -500, 1_000_000),  # f4's special-case band
                             rng.uniform(500, 720, 200_000), rng.uniform(-1e-15, 1e-15, 100_000),
                             [0.0, -0.0, -745.2, -708.3, -1024.0, -1075.0, 709.8, 710.0, np.inf,
                              -np.inf, np.nan, -512.0, 1e-300, -745.1332191019411,
                              -745.1332191019412, -708.3964185322641, 709.782712893384]])),
            (pg.glibc_cos, ref.lib.ref_libm_cos,
             np.concatenate([rng.uniform(-40, 40, 2_000_000), rng.uniform(0, 140, 2_000_000),
                             # __branred territory (|x| >= 105414350), every binade
                             np.ldexp(rng.uniform(-2.0, 2.0, 400_000),
                                      rng.integers(27, 1024, 400_000)),
                             [0.0, -0.0, 1e-9, 0.855469, 2.426265, np.pi / 2, 36.0, np.inf,
                              np.nan, 105414350.0, 1e22, 1.7976931348623157e308]]))):
        got = fn(xs, on_device=True)
        want = np.empty_like(xs)
        libm(C.c_int64(len(xs)), xs.ctypes.data_as(C.POINTER(C.c_double)),
             want.ctypes.data_as(C.POINTER(C.c_double)))
        assert np.array_equal(bits(got), bits(want))
        # the paired two-point forms the evaluator runs (incl. their fix-ups)
        assert np.array_equal(bits(fn(xs, on_device=True, paired=True)), bits(want))
        if fn is pg.glibc_cos:
            assert np.array_equal(bits(pg.glibc_cos(xs, on_device=True, branch_free=True)),
                                  bits(want))


# ------------------------------------------------------ evaluate ----------
@pytest.mark.parametrize("fid", [1, 2, 3, 4, 5, 6, 7, 8])
def test_evaluate_batch_bit_exact(pg, gpu, ref, fid):
    rng = np.random.default_rng(100 + fid)
    for n in (1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12):
        m = 700 if n <= 10 else 64
        lows = rng.uniform(0.0, 0.6, size=(m, n))
        lens = rng.uniform(0.01, 0.4, size=(m, n))
        lens[:5] = 2.0 ** -rng.integers(1, 30, size=(5, n))  # deep bisection lengths
        est, raw, axes, cnt = pg.evaluate_batch(pg.Integrand(fid), lows, lens)
        e2, r2, a2, c2 = ref.evaluate_batch(fid, lows, lens)
        assert np.array_equal(bits(est), bits(e2)), (fid, n)
        assert np.array_equal(bits(raw), bits(r2)), (fid, n)
        assert np.array_equal(axes, a2), (fid, n)
        assert cnt == c2


def test_evaluate_batch_nonfinite_and_overflow(pg, gpu, ref):
    """The separable evaluator tracks rule.cpp:384's `finite` flag lazily (a
    non-finite S[0] triggers an exact re-walk of the region's points): regions
    with inf/NaN point values AND regions whose finite values overflow the
    weighted sums (finite=true, est=+-inf) must both match the reference."""
    rng = np.random.default_rng(77)
    for fid, n, scale in ((7, 3, 5e13), (7, 2, 1e13), (7, 4, 1e14), (8, 3, 1e20), (3, 2, 1.0),
                         (3, 3, 1.0)):
        m = 600
        if fid == 3:  # 1 + x0 + 2 x1 (+ 3 x2) crosses 0: huge / inf / NaN values
            lows = rng.uniform(-2.0, 0.5, size=(m, n))
            lens = rng.uniform(0.01, 1.5, size=(m, n))
        else:  # point values from ~1e250 to inf: overflowing sums and inf points
            lows = rng.uniform(0.0, scale, size=(m, n))
            lens = rng.uniform(0.01, 1.0, size=(m, n)) * scale
        est, raw, axes, cnt = pg.evaluate_batch(pg.Integrand(fid), lows, lens)
        e2, r2, a2, c2 = ref.evaluate_batch(fid, lows, lens)
        assert np.array_equal(bits(est), bits(e2)), (fid, n)
        assert np.array_equal(bits(raw), bits(r2)), (fid, n)
        assert np.array_equal(axes, a2), (fid, n)
        if fid != 3:  # inf points and overflowing finite sums both occur
            assert (~np.isfinite(r2)).any() and (np.isinf(e2)).any(), (fid, n)


def test_evaluate_batch_n16_and_unit_cube_splits(pg, gpu, ref):
    for fid in (3, 4, 5):
        lows, lens = ref.uniform_split([0.0] * 16, [1.0] * 16, 1)
        a = pg.evaluate_batch(pg.Integrand(fid), lows, lens)
        b = ref.evaluate_batch(fid, lows, lens)
        assert np.array_equal(bits(a[0]), bits(b[0])) and np.array_equal(a[2], b[2])
    for fid in range(1, 9):
        lows, lens = ref.uniform_split([0.0] * 5, [1.0] * 5, 6)  # 5D initial batch
        a = pg.evaluate_batch(pg.Integrand(fid), lows, lens)
        b = ref.evaluate_batch(fid, lows, lens)
        assert np.array_equal(bits(a[0]), bits(b[0])) and np.array_equal(bits(a[1]), bits(b[1]))
        assert np.array_equal(a[2], b[2])


def test_evaluate_matches_golden_batches(pg, gpu):
    for name, b in load_golden("batch.json").items():
        lows = np.array([[unhex(v) for v in r] for r in b["lows"]])
        lens = np.array([[unhex(v) for v in r] for r in b["lengths"]])
        est, raw, axes, cnt = pg.evaluate_batch(pg.Integrand(b["fid"]), lows, lens)
        assert np.array_equal(bits(est), bits([unhex(v) for v in b["est"]])), name
        assert np.array_equal(bits(raw), bits([unhex(v) for v in b["raw"]])), name
        assert axes.tolist() == b["axes"] and cnt == b["eval_count"], name


TEST_INTEGRANDS = [(100, [1.0]), (100, [-2.5]), (101, [1, 2, 0, 3]), (102, [40.0, 1.0, 2.0]),
                   (102, [50.0, 2.0, 2.0]), (103, [0.6, 0.6]), (103, [0.8, -1.0]), (104, [0.95]),
                   (105, [7.25, 0.7, 1.9, 2.6, 1.1]), (106, [])]


@pytest.mark.parametrize("fid,params", TEST_INTEGRANDS)
def test_unit_test_integrands_bit_exact(pg, gpu, ref, fid, params):
    rng = np.random.default_rng(fid)
    for n in (3, 4):
        lows = rng.uniform(0.0, 0.7, size=(300, n))
        lens = rng.uniform(0.01, 0.3, size=(300, n))
        a = pg.evaluate_batch(pg.Integrand(fid, params), lows, lens)
        b = ref.evaluate_batch(fid, lows, lens, params=params)
        assert np.array_equal(bits(a[0]), bits(b[0])) and np.array_equal(bits(a[1]), bits(b[1]))
        assert np.array_equal(a[2], b[2])


def test_rule_known_answers_on_device(pg, gpu):
    """test_rule.cpp:82-254 through the device evaluator."""
    for n in (1, 2, 4, 8):  # constant: exact estimate, ~zero raw error
        b = pg.uniform_split(pg.Bounds.unit_cube(n), 1)
        est, raw, _, cnt = pg.evaluate_batch(pg.Integrand.constant(1.0), b.lows, b.lengths)
        assert abs(est[0] - 1.0) <= 1e-14 and raw[0] < 1e-13 and cnt == pg.rule_point_count(n)
    import itertools
    for n in (1, 2, 3):  # degree-7 exactness
        b = pg.uniform_split(pg.Bounds.unit_cube(n), 1)
        for alpha in itertools.product(range(8), repeat=n):
            if sum(alpha) > 7:
                continue
            est, _, _, _ = pg.evaluate_batch(pg.Integrand.monomial(alpha), b.lows, b.lengths)
            exact = 1.0
            for e in alpha:
                exact /= e + 1
            assert abs(est[0] - exact) <= 1e-12 * exact, alpha
    b = pg.uniform_split(pg.Bounds.unit_cube(1), 1)
    est, raw, _, _ = pg.evaluate_batch(pg.Integrand.monomial([9]), b.lows, b.lengths)
    assert est[0] != 0.1 and raw[0] > 0.0
    # zero axis signal -> widest extent (axis 1)
    lens = np.array([[0.25, 1.0, 0.5]])
    _, _, axes, _ = pg.evaluate_batch(pg.Integrand.pocket(0.95), 1.0 - lens, lens)
    assert axes[0] == 1
    # NaN -> est 0, raw +inf
    b = pg.uniform_split(pg.Bounds.unit_cube(2), 2)
    est, raw, _, _ = pg.evaluate_batch(pg.Integrand.nan_box(0.6, 0.6), b.lows, b.lengths)
    assert np.isinf(raw).sum() >= 1 and (est[np.isinf(raw)] == 0.0).all()
    # split axis invariant under positive scaling (seeded freqs as in test_rule.cpp)
    fr = np.random.default_rng(21).uniform(0.5, 3.0, size=4)
    b = pg.uniform_split(pg.Bounds.unit_cube(4), 2)
    a1 = pg.evaluate_batch(pg.Integrand.cos_sum(1.0, fr), b.lows, b.lengths)[2]
    a2 = pg.evaluate_batch(pg.Integrand.cos_sum(7.25, fr), b.lows, b.lengths)[2]
    assert np.array_equal(a1, a2)


# ------------------------------------------------- batch functions --------
def test_refine_classify_threshold_bit_exact(pg, gpu, ref):
    rng = np.random.default_rng(42)
    m = 200_000
    est = rng.normal(size=m)
    raw = np.abs(rng.normal(size=m)) * 10.0 ** rng.integers(-12, 0, size=m)
    raw[::97] = 0.0
    raw[::1001] = np.inf
    pest = np.repeat(rng.normal(size=m // 2) * 2, 2)
    perr = np.abs(rng.normal(size=m))
    a = pg.two_level_refine(est, raw, pest, perr)
    b = ref.two_level_refine(est, raw, pest, perr)
    assert np.array_equal(bits(a), bits(b))
    for tau, en in ((1e-3, True), (1e-6, True), (1e-3, False)):
        assert np.array_equal(pg.rel_err_classify(est, a, tau, en),
                              ref.rel_err_classify(est, a, tau, en))
    assert np.array_equal(pg.apply_threshold(a, 1e-6), (a >= 1e-6).astype(np.uint8))
    # reference known answers (test_errorest.cpp:10-29, test_classify.cpp:114-146)
    out = pg.two_level_refine([3.0, 1.0], [0.08, 0.02], [4.0, 4.0], [0.5, 0.5])
    assert abs(out[0] - 0.01) < 1e-15 and abs(out[1] - 0.0025) < 1e-15
    with pytest.raises(ValueError):
        pg.two_level_refine([1.0], [1.0], [1.0], [1.0])
    r = pg.threshold_classify([1, 1, 1, 1], [9, 9, 1, 1], 0.0, 100.0, 20.0, 4, 1e-3)
    assert not r.success and r.flags.tolist() == [1, 1, 1, 1]
    r = pg.threshold_classify([1, 1, 1, 1], [9, 1, 1, 1], 0.0, 100.0, 12.0, 4, 1e-3)
    assert r.success and r.finished_count == 3 and r.discarded_error == 3.0
    assert r.flags.tolist() == [1, 0, 0, 0] and r.discarded_error <= r.budget_limit
    assert not pg.threshold_classify([1, 1], [5, 5], 1e6, 10.0, 10.0, 2, 1e-3).success


def test_threshold_trace_oracle_instances(pg, gpu, ref):
    """test_classify.cpp:148-182: 300 random instances (seeded), plus large ones."""
    rng = np.random.default_rng(2024)
    for trial in range(300):
        m = 2 + int(rng.uniform() * 40) if trial < 280 else int(rng.integers(3000, 300_000))
        e = 10.0 ** (-6.0 * rng.uniform(size=m))
        act = (rng.uniform(size=m) < 0.8).astype(np.uint8)
        v_tot = rng.uniform() * 10
        e_it = float(e.sum())
        e_tot = e_it * (1 + rng.uniform())
        tau = 10.0 ** (-1.0 - 3.0 * rng.uniform())
        a = pg.threshold_classify(act, e, v_tot, e_tot, e_it, m, tau)
        b = ref.threshold_classify(act, e, v_tot, e_tot, e_it, m, tau)
        assert a.success == b["success"] and np.array_equal(a.flags, b["flags"]), trial
        assert (a.threshold, a.discarded_error, a.budget_limit, a.finished_count, a.attempts,
                a.direction_changes) == (b["threshold"], b["discarded_error"], b["budget_limit"],
                                         b["finished_count"], b["attempts"],
                                         b["direction_changes"]), trial


def test_filter_bisect_split_sums_bit_exact(pg, gpu, ref):
    rng = np.random.default_rng(11)
    for n, m in ((1, 3), (3, 5000), (8, 70_000)):
        lows = rng.uniform(0, 0.5, size=(m, n))
        lens = 2.0 ** -rng.integers(1, 20, size=(m, n)).astype(float)
        est = rng.normal(size=m)
        err = np.abs(rng.normal(size=m))
        axis = rng.integers(0, n, size=m).astype(np.int32)
        pest, perr = rng.normal(size=m), np.abs(rng.normal(size=m))
        flags = (rng.uniform(size=m) < 0.6).astype(np.uint8)
        batch = pg.RegionBatch(lows, lens, est, err, axis, pest, perr)
        f = pg.filter(batch, flags)
        g = ref.filter(lows, lens, est, err, axis, pest, perr, flags)
        assert f.kept.count == g["kept"]
        assert (f.finished_estimate, f.finished_error, f.finished_volume) == (
            g["finished_estimate"], g["finished_error"], g["finished_volume"])
        for k1, k2 in (("lows", "lows"), ("lengths", "lengths"), ("estimates", "estimates"),
                       ("errors", "errors"), ("parent_estimates", "parent_estimates"),
                       ("parent_errors", "parent_errors")):
            assert np.array_equal(bits(getattr(f.kept, k1)), bits(g[k2])), k1
        assert np.array_equal(f.kept.split_axis, g["split_axis"])
        c = pg.bisect(batch, 1 << 22)
        d = ref.bisect(lows, lens, est, err, axis)
        assert np.array_equal(bits(c.lows), bits(d[0])) and np.array_equal(bits(c.lengths), bits(d[1]))
        assert np.array_equal(bits(c.parent_estimates), bits(d[2]))
        assert np.array_equal(bits(c.parent_errors), bits(d[3]))
    with pytest.raises(AssertionError):  # logic_error: doubling beyond the cap
        pg.bisect(pg.RegionBatch(np.zeros((2, 1)), np.ones((2, 1))), 3)
    for lo, hi, d in (([0, 0], [1, 1], 3), ([0, -1], [2, 1], 2), ([-1.5, 0.25, 3], [2, 0.5, 7], 5)):
        u = pg.uniform_split(pg.Bounds(lo, hi), d)
        v = ref.uniform_split(lo, hi, d)
        assert np.array_equal(bits(u.lows), bits(v[0])) and np.array_equal(bits(u.lengths), bits(v[1]))
    with pytest.raises(RuntimeError):
        pg.uniform_split(pg.Bounds([0, 0, 0], [1, 1, 1]), 100, 1000)
    x = rng.normal(size=5_000_001) * 10.0 ** rng.integers(-5, 5, size=5_000_001)
    fl = (rng.uniform(size=len(x)) < 0.3).astype(np.uint8)
    assert pg.block_sum(x) == ref.block_sum(x)
    assert pg.block_sum_where(x, fl, 0) == ref.block_sum_where(x, fl, 0)
    assert pg.block_sum_where(x, fl, 1) == ref.block_sum_where(x, fl, 1)
    assert pg.count_flags(fl, 1) == int(fl.sum())
    assert pg.min_max(x) == (x.min(), x.max())
    assert pg.block_sum([]) == 0.0


# ------------------------------------------------------ integrate ---------
def test_integrate_matches_golden_traces(pg, gpu):
    """Every per-iteration field of the reference's own trace, bit for bit."""
    for name, case in load_golden("traces.json").items():
        cfg, _ = cfg_pair(pg, case["tau"], case["rel_filter"], **case["extra"])
        res = pg.integrate(integrand(pg, case["fid"], case["params"]),
                           pg.Bounds.unit_cube(case["n"]), cfg, trace=True)
        assert_same_result(res, case["result"])
        assert_same_trace(res.trace, case["trace"], name)
        want_ev = case["result"]["threshold_events"]
        assert len(res.threshold_events) == len(want_ev), name
        for e, w in zip(res.threshold_events, want_ev):
            assert (e.iteration, e.success, e.batch_size, e.finished_count,
                    e.discarded_error, e.budget_limit) == (
                w["iteration"], w["success"], w["batch_size"], w["finished_count"],
                unhex(w["discarded_error"]), unhex(w["budget_limit"])), name


def test_integrate_matches_reference_finals_8d(pg, gpu):
    """BASELINE 8D configs at the reference default cap (2^22): the reference's
    final results (tests/golden/finals.json, minutes of CPU each)."""
    for name, want in load_golden("finals.json").items():
        cfg = pg.Config(tau_rel=want["tau"], rel_filtering_enabled=want["fid"] != 1)
        res = pg.integrate(pg.Integrand(want["fid"]), pg.Bounds.unit_cube(want["n"]), cfg)
        assert_same_result(res, want)
        assert len(res.threshold_events) == want["n_events"], name


def test_integrate_matches_reference_finals_deep(pg, gpu):
    """Every BASELINE config at full size against the reference's own final
    results (tests/golden/finals_deep.json, made by make_deep_finals.py with
    the unmodified reference: tens of CPU-minutes): the whole 8D suite
    f1..f6 x tau 1e-3..1e-6 (bench.py's workload), f2 8D 1e-9, f5 / f6 8D 1e-8.
    Bit-exact estimates and errors, identical status, iterations, region and
    evaluation counts and threshold-event counts."""
    cases = load_golden("finals_deep.json")
    assert len(cases) >= 6
    for name, want in cases.items():
        cfg = pg.Config(tau_rel=want["tau"], rel_filtering_enabled=want["fid"] != 1)
        res = pg.integrate(pg.Integrand(want["fid"]), pg.Bounds.unit_cube(want["n"]), cfg)
        assert_same_result(res, want)
        assert len(res.threshold_events) == min(want["n_events"], 256), name


def test_integrate_matches_reference_finals_bigcap(pg, gpu):
    """A 2^24-region cap (8192 fold blocks): the global-memory tree path of
    the finalize kernels and 8192-block probe passes, against the reference's
    finals at the same cap (tests/golden/finals_bigcap.json)."""
    for name, want in load_golden("finals_bigcap.json").items():
        cfg = pg.Config(tau_rel=want["tau"], rel_filtering_enabled=want["fid"] != 1,
                        max_regions=want["max_regions"])
        res = pg.integrate(pg.Integrand(want["fid"]), pg.Bounds.unit_cube(want["n"]), cfg)
        assert_same_result(res, want)
        assert len(res.threshold_events) == min(want["n_events"], 256), name


def test_integrate_matches_10d_traces(pg, gpu):
    """BASELINE configs[4]'s dimension (f4 Gaussian 10D: N = 1245 rule points,
    its own k_evaluate instance) over full-length runs of the unmodified
    reference (tests/golden/traces_10d.json, make_10d_traces.py): every
    per-iteration field, the threshold events and the final result, bit for
    bit, at the default cap (tau 1e-3 and configs[4]'s 1e-7) and at 2^24."""
    cases = load_golden("traces_10d.json")
    assert cases, "tests/golden/traces_10d.json is empty"
    for name, case in cases.items():
        cfg = pg.Config(tau_rel=case["tau"], rel_filtering_enabled=case["fid"] != 1,
                        max_regions=case["max_regions"])
        res = pg.integrate(pg.Integrand(case["fid"]), pg.Bounds.unit_cube(case["n"]), cfg,
                           trace=True)
        assert_same_result(res, case["result"])
        assert_same_trace(res.trace, case["trace"], name)
        want_ev = case["result"]["threshold_events"]
        assert len(res.threshold_events) == len(want_ev), name
        for e, w in zip(res.threshold_events, want_ev):
            assert (e.iteration, e.success, e.batch_size, e.finished_count,
                    e.discarded_error, e.budget_limit) == (
                w["iteration"], w["success"], w["batch_size"], w["finished_count"],
                unhex(w["discarded_error"]), unhex(w["budget_limit"])), name


MORE_CASES = [
    ("mapped_xy", 101, 2, 1e-6, True, {}, [1, 1], ([0, 1], [2, 3])),
    ("mapped_f4", 4, 3, 1e-4, True, {}, None, ([-1, 0, 0.25], [1, 2, 0.75])),
    ("identity_refiner", 5, 3, 1e-6, True, {"refiner": 1}, None, None),
    ("it_max_1", 3, 4, 1e-9, True, {"it_max": 1}, None, None),
    ("tight_limits", 4, 3, 1e-8, True, {"max_regions": 1 << 11, "init_target": 1 << 8,
                                        "attempt_limit": 3, "direction_change_limit": 1},
     None, None),
    ("init_subdiv", 6, 4, 1e-5, True, {"init_subdiv": 3}, None, None),
]


@pytest.mark.parametrize("name,fid,n,tau,relf,extra,params,bounds", MORE_CASES)
def test_integrate_matches_live_reference(pg, gpu, ref, name, fid, n, tau, relf, extra, params,
                                          bounds):
    cfg, rcfg = cfg_pair(pg, tau, relf, **extra)
    b = pg.Bounds(*bounds) if bounds else pg.Bounds.unit_cube(n)
    res = pg.integrate(integrand(pg, fid, params), b, cfg)
    want = ref.integrate(fid, n, rcfg, lower=b.lower, upper=b.upper, params=params)
    assert (res.estimate, res.errorest, str(res.status), res.iterations, res.regions_generated,
            res.eval_count) == (want.estimate, want.errorest, want.status, want.iterations,
                                want.regions_generated, want.eval_count), name
    if bounds is None:
        _, rows = ref.trace(fid, n, rcfg, params=params)
        res2 = pg.integrate(integrand(pg, fid, params), b, cfg, trace=True)
        assert res2.trace == rows


def test_driver_known_answers(pg, gpu):
    """test_driver.cpp:22-154 through the GPU driver."""
    r = pg.integrate(pg.Integrand.constant(1.0), pg.Bounds.unit_cube(3),
                     pg.Config(tau_rel=1e-3, init_subdiv=2))
    assert r.status == pg.Status.Converged and r.iterations == 1 and r.regions_generated == 8
    assert abs(r.estimate - 1.0) < 1e-13 and r.errorest < 1e-10
    r = pg.integrate(pg.Integrand.rough(40.0, 1, 2.0), pg.Bounds.unit_cube(2),
                     pg.Config(tau_rel=1e-12, rel_filtering_enabled=False, init_subdiv=2, it_max=4))
    assert r.status == pg.Status.MaxIterations and r.regions_generated == 60
    assert r.eval_count == 60 * 17
    r = pg.integrate(pg.Integrand.monomial([1, 1]), pg.Bounds([0, 1], [2, 3]),
                     pg.Config(tau_rel=1e-6))
    assert r.status == pg.Status.Converged and abs(r.estimate - 8.0) <= 1e-10 * 8.0
    r = pg.integrate(pg.integrand_by_id("f4"), pg.Bounds.unit_cube(2),
                     pg.Config(tau_rel=1e-9, max_regions=1 << 10, init_target=1 << 9))
    assert r.threshold_events
    r = pg.integrate(pg.Integrand.nan_box(0.8), pg.Bounds.unit_cube(2),
                     pg.Config(tau_rel=1e-6, max_regions=1 << 10, init_target=1 << 8, it_max=12))
    assert r.status != pg.Status.Converged and np.isinf(r.errorest)
    r = pg.integrate(pg.integrand_by_id("f4"), pg.Bounds.unit_cube(3),
                     pg.Config(tau_rel=5e-7, max_regions=1 << 12, init_target=1 << 10))
    for ev in r.threshold_events:
        if ev.success:
            assert ev.retained_fraction() < 0.5
            assert ev.discarded_error <= ev.budget_limit * (1 + 1e-12)
    with pytest.raises(RuntimeError):  # runtime_error: d^n exceeds max_regions
        pg.integrate(pg.integrand_by_id("f4"), pg.Bounds.unit_cube(3),
                     pg.Config(init_subdiv=100, max_regions=1000))


VALIDATE_CASES = [(3, 3, 1e-3), (4, 3, 1e-6), (2, 4, 1e-4), (5, 5, 1e-4), (6, 3, 1e-5),
                  (4, 5, 1e-3)]  # the last one trips the reference's own volume check


def _outcome(fn):
    try:
        r = fn()
        return ("ok", r.estimate, r.errorest, str(r.status), r.iterations, r.regions_generated)
    except AssertionError as e:  # logic_error: an invariant tripped
        return ("logic_error", str(e))


@pytest.mark.parametrize("fid,n,tau", VALIDATE_CASES)
def test_validate_invariants_mode(pg, gpu, ref, fid, n, tau):
    """validate_invariants (driver.cpp:75-79,148,185-198): volume conservation,
    filter estimate conservation, finished-error checks.  Same outcome as the
    reference: identical results, or the same invariant violation."""
    cfg, rcfg = cfg_pair(pg, tau, True, validate_invariants=True)
    got = _outcome(lambda: pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n), cfg))
    want = _outcome(lambda: ref.integrate(fid, n, rcfg))
    assert got == want


def test_determinism_and_workspace_reuse(pg, gpu):
    cfg = pg.Config(tau_rel=1e-3)
    a = pg.integrate(pg.integrand_by_id("f4"), pg.Bounds.unit_cube(5), cfg)
    b = pg.integrate(pg.integrand_by_id("f6"), pg.Bounds.unit_cube(6), cfg)
    c = pg.integrate(pg.integrand_by_id("f4"), pg.Bounds.unit_cube(5), cfg)
    assert (a.estimate, a.errorest, a.regions_generated) == (c.estimate, c.errorest,
                                                              c.regions_generated)
    assert b.estimate != a.estimate


def test_fast_mode_within_tolerance(pg, gpu):
    for fid, n, tau in ((4, 5, 1e-3), (3, 8, 1e-3), (5, 5, 1e-4), (2, 6, 1e-3), (6, 6, 1e-3)):
        p = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n), pg.Config(tau_rel=tau))
        f = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n),
                         pg.Config(tau_rel=tau, mode="fast"))
        assert (f.status, f.iterations, f.regions_generated) == (p.status, p.iterations,
                                                                  p.regions_generated)
        assert abs(f.estimate - p.estimate) <= TOL_FAST * abs(p.estimate)


def test_large_batch_properties(pg, gpu):
    """At the full default cap: the region count identity and the trace's
    accounting hold exactly (sizes too large for the CPU oracle in a test)."""
    res = pg.integrate(pg.integrand_by_id("f4"), pg.Bounds.unit_cube(8),
                       pg.Config(tau_rel=1e-6), trace=True)
    ms = [r["m"] for r in res.trace]
    assert sum(ms) == res.region_evals == res.eval_count // 401
    assert res.regions_generated == sum(ms)
    for prev, nxt in zip(res.trace, res.trace[1:]):
        assert nxt["m"] == 2 * prev["kept"]
        assert nxt["v_f"] == prev["v_f"] + prev["fin_v"]
        assert nxt["e_f"] == prev["e_f"] + prev["fin_e"]
    assert max(ms) <= 1 << 22


def test_batch_functions_on_empty_and_tiny_inputs(pg, gpu, ref):
    """Empty and one/odd-element inputs through every batch entry point (the
    reference's functions accept them: reduce.cpp:13-82, classify.cpp:11-129,
    geometry.cpp:114-143, rule.cpp:351-430)."""
    for m in (0, 1, 2, 3, 2047, 2049):
        rng = np.random.default_rng(m)
        n = 3
        lows = rng.uniform(0.0, 0.5, size=(m, n))
        lens = rng.uniform(0.01, 0.5, size=(m, n))
        est, raw, axes, cnt = pg.evaluate_batch(pg.Integrand(4), lows, lens)
        e2, r2, a2, c2 = ref.evaluate_batch(4, lows, lens)
        assert len(est) == m and cnt == c2
        assert np.array_equal(bits(est), bits(e2)) and np.array_equal(bits(raw), bits(r2))
        assert np.array_equal(axes, a2)
        x = rng.uniform(-1.0, 1.0, size=m)
        assert np.array_equal(bits([pg.block_sum(x)]), bits([ref.block_sum(x)]))
        fl = (rng.uniform(size=m) < 0.5).astype(np.uint8)
        for which in (0, 1):
            assert np.array_equal(bits([pg.block_sum_where(x, fl, which)]),
                                  bits([ref.block_sum_where(x, fl, which)]))
        err = np.abs(raw)
        assert np.array_equal(pg.rel_err_classify(est, err, 1e-3), ref.rel_err_classify(est, err, 1e-3))
        if m % 2 == 0:  # siblings come in pairs
            pest = rng.uniform(0.0, 1.0, size=m)
            perr = rng.uniform(0.0, 1.0, size=m)
            assert np.array_equal(bits(pg.two_level_refine(est, raw, pest, perr)),
                                  bits(ref.two_level_refine(est, raw, pest, perr)))
        b = pg.RegionBatch(lows, lens, est, err, axes)
        fr = pg.filter(b, fl)
        want = ref.filter(lows, lens, est, err, axes, np.zeros(m), np.zeros(m), fl)
        assert fr.kept.count == want["kept"]
        assert np.array_equal(bits(fr.kept.lows), bits(want["lows"]))
        assert np.array_equal(bits([fr.finished_estimate, fr.finished_error]),
                              bits([want["finished_estimate"], want["finished_error"]]))
        kids = pg.bisect(b, 1 << 22)
        cl, cn, cp, cq = ref.bisect(lows, lens, est, err, axes)
        assert np.array_equal(bits(kids.lows), bits(cl)) and np.array_equal(bits(kids.lengths), bits(cn))
        if m:
            act = np.ones(m, dtype=np.uint8)
            got = pg.threshold_classify(act, err, float(est.sum()), float(err.sum()),
                                        float(err.sum()), m, 1e-3)
            exp = ref.threshold_classify(act, err, float(est.sum()), float(err.sum()),
                                         float(err.sum()), m, 1e-3)
            assert got.success == exp["success"] and got.attempts == exp["attempts"]
            assert np.array_equal(got.flags, exp["flags"])


def test_streamed_threshold_search_equals_exact_folds(pg, gpu, tmp_path):
    """PAGANI_PROBE_STREAM=1 decides the threshold search from streamed passes
    (exact counts, fast sums with a rounding bound) and folds only the accepted
    threshold exactly; the default runs every pass with the strict folds.
    Both must give the same trace bit for bit."""
    import json
    import subprocess
    import sys
    cases = [(1, 8, 1e-3, False, 30), (6, 8, 1e-4, True, 60), (2, 8, 1e-3, True, 40)]
    code = ("import json,sys; sys.path.insert(0, %r); import paper_2104_06494_b200 as pg\n"
            "out=[]\n"
            "for f,n,tau,relf,itm in %r:\n"
            "    r=pg.integrate(pg.Integrand(f), pg.Bounds.unit_cube(n),"
            " pg.Config(tau_rel=tau, rel_filtering_enabled=relf, it_max=itm), trace=True)\n"
            "    out.append([r.estimate.hex(), r.errorest.hex(), r.iterations, r.regions_generated,"
            " [[row[k].hex() if isinstance(row[k], float) else row[k] for k in sorted(row)]"
            " for row in r.trace], r.probe_fallbacks, len(r.threshold_events)])\n"
            "print(json.dumps(out))\n") % (str(pg.__path__[0]).rsplit("/", 1)[0], cases)
    env = dict(__import__("os").environ, PAGANI_PROBE_STREAM="1")
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr
    streamed = json.loads(p.stdout.strip().splitlines()[-1])
    fallbacks = 0
    for (f, n, tau, relf, itm), got in zip(cases, streamed):
        r = pg.integrate(pg.Integrand(f), pg.Bounds.unit_cube(n),
                         pg.Config(tau_rel=tau, rel_filtering_enabled=relf, it_max=itm),
                         trace=True)
        want = [r.estimate.hex(), r.errorest.hex(), r.iterations, r.regions_generated,
                [[row[k].hex() if isinstance(row[k], float) else row[k] for k in sorted(row)]
                 for row in r.trace]]
        assert got[:5] == want, (f, n, tau)
        assert got[6] > 0  # threshold searches happened
        fallbacks += got[5]
    assert fallbacks <= 2  # the streamed passes decide (nearly) always


def test_pipeline_switches_do_not_change_results(pg, gpu):
    """The default launch pipeline -- deferred bisection (k_link + children
    derived in k_evaluate) and programmatic dependent launches -- and the
    opt-in speculative first probe pass queued behind k_finalize
    (PAGANI_SPEC_PROBE=1) against the plain one (PAGANI_DEFER_BISECT=0
    PAGANI_PDL=0: explicit split kernel, ordinary launches, every pass launched
    by the host): the same trace bit for bit, including multi-pass searches
    (f3) and failed ones."""
    import json
    import subprocess
    import sys
    cases = [(3, 8, 1e-3, True, 100), (6, 8, 1e-4, True, 60), (2, 8, 1e-3, True, 40),
             (1, 8, 1e-3, False, 30), (4, 10, 1e-3, True, 10), (5, 5, 1e-4, True, 100)]

    def row_key(r):
        return [r.estimate.hex(), r.errorest.hex(), r.iterations, r.regions_generated,
                str(r.status), [[row[k].hex() if isinstance(row[k], float) else row[k]
                                 for k in sorted(row)] for row in r.trace]]

    code = ("import json,sys; sys.path.insert(0, %r); import paper_2104_06494_b200 as pg\n"
            "out=[]\n"
            "for f,n,tau,relf,itm in %r:\n"
            "    r=pg.integrate(pg.Integrand(f), pg.Bounds.unit_cube(n),"
            " pg.Config(tau_rel=tau, rel_filtering_enabled=relf, it_max=itm), trace=True)\n"
            "    out.append([r.estimate.hex(), r.errorest.hex(), r.iterations, r.regions_generated,"
            " str(r.status), [[row[k].hex() if isinstance(row[k], float) else row[k]"
            " for k in sorted(row)] for row in r.trace], r.spec_probe_passes])\n"
            "print(json.dumps(out))\n") % (str(pg.__path__[0]).rsplit("/", 1)[0], cases)
    def run(**sw):
        env = dict(__import__("os").environ, **sw)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr
        return json.loads(p.stdout.strip().splitlines()[-1])

    plain = run(PAGANI_DEFER_BISECT="0", PAGANI_PDL="0", PAGANI_SPEC_PROBE="0")
    spec = run(PAGANI_SPEC_PROBE="1")  # the opt-in speculative first pass
    spec_passes = 0
    for (f, n, tau, relf, itm), got, sp in zip(cases, plain, spec):
        assert got[6] == 0  # the plain pipeline never speculates
        r = pg.integrate(pg.Integrand(f), pg.Bounds.unit_cube(n),
                         pg.Config(tau_rel=tau, rel_filtering_enabled=relf, it_max=itm),
                         trace=True)
        assert row_key(r) == got[:6], (f, n, tau)
        assert sp[:6] == got[:6], (f, n, tau, "speculative first pass")
        spec_passes += sp[6]
    assert spec_passes > 0  # the speculative pipeline did speculate
