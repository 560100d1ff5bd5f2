"""Pin the oracle (CPU only).

The parity oracle is the unmodified reference library (oracle/_ref), so these
tests check it against (a) the golden values SURVEY.md Appendix A recorded
from the reference, (b) the known answers of the reference's own unit tests
(/root/reference/proj/tests/*.cpp, which cannot be built here: doctest is
absent), and (c) the committed golden fixtures.  The plain-C restatement
(oracle/pagani_oracle.c) is then checked bit-for-bit against the reference.
"""
import numpy as np
import pytest

from conftest import bits, load_golden, unhex
from ref_ctypes import make_config

# f4 5D tau=1e-3 (BASELINE config 1), per-iteration v, e
APPENDIX_A2 = [
    (1, 7776, 5.4388403733303074e-06, 5.4358370412334869e-06),
    (2, 15552, 3.9387960753605537e-06, 1.5000443628544841e-06),
    (3, 31104, 2.8971230593458089e-06, 1.0445672425022762e-06),
    (4, 62208, 2.3143992174881852e-06, 5.8484684762703138e-07),
    (5, 124416, 1.9819480117574552e-06, 3.3424670793643816e-07),
    (6, 248832, 1.8430648736984902e-06, 1.3990663580782258e-07),
    (7, 497664, 1.8134887815878933e-06, 3.020074060455488e-08),
    (8, 995328, 1.7982481612035684e-06, 1.5534311147334534e-08),
    (9, 1990656, 1.7921086239115944e-06, 7.1029340893134449e-09),
    (10, 3981312, 1.7913505380336946e-06, 3.427162475653217e-09),
    (11, 4864, 1.7912720563699448e-06, 1.3292060373241654e-09),
]
# SURVEY.md Appendix A.1 (n=8 row subset): [w7, null1..null4] per orbit
APPENDIX_A1_N8 = [
    [-1.7546105776558532, 3.281054717268705, 0.017939012198401206, -3.784189502422832e-21,
     4.8511247467994986e-05],
    [0.14936747447035581, -0.35474775186709306, 0.0050352690507120528, 0.0051049650621062606,
     4.6406231097148812e-05],
    [-0.070111263526901738, 0.29682975156226166, -0.006540570445199235, 0.0047472580383307698,
     3.3776132872071801e-05],
    [0.0101610526850582, -0.024132500127013141, -0.00027168241170028642, -0.0023269510597505958,
     1.9041018276148613e-05],
    [0.0013612238352893342, 0.0013612238352893342, 0.00014286812587431947, 0.00040227714486357121,
     -1.3531340304313163e-05],
]


def test_reference_reproduces_survey_appendix_a2(ref):
    res, rows = ref.trace(4, 5, make_config(tau_rel=1e-3))
    assert res.status == "converged" and res.iterations == 11
    assert res.estimate == 1.7913125097877638e-06
    assert res.errorest == 1.3298630282412981e-09
    assert res.regions_generated == 7_959_712 and res.eval_count == 740_253_216
    for (it, m, v, e), row in zip(APPENDIX_A2, rows):
        assert (row["it"], row["m"], row["v"], row["e"]) == (it, m, v, e)
    thr = rows[9]
    assert thr["thr_invoked"] and thr["thr_accepted"] and thr["thr_attempts"] == 1
    assert thr["thr_threshold"] == 8.6081233413839887e-16
    assert thr["thr_finished"] == 3_978_880


def test_reference_reproduces_survey_appendix_a1(ref):
    n = 8
    _, w, _ = ref.build_rule(n)
    firsts = [0, 1, 1 + 2 * n, 1 + 4 * n, 1 + 4 * n + 2 * n * (n - 1)]
    for o in range(5):
        for k in range(5):
            assert w[k, firsts[o]] == APPENDIX_A1_N8[o][k], (o, k)


def test_reference_unit_test_known_answers(ref):
    """Known answers of test_errorest.cpp, test_classify.cpp, test_geometry.cpp."""
    out = ref.two_level_refine([3.0, 1.0], [0.08, 0.02], [4.0, 4.0], [0.5, 0.5])
    assert abs(out[0] - 0.01) < 1e-15 and abs(out[1] - 0.0025) < 1e-15
    out = ref.two_level_refine([3.0, 1.0], [0.08, 0.02], [9.0, 9.0], [0.5, 0.5])
    assert out.tolist() == [0.08, 0.02]
    r = ref.threshold_classify([1, 1, 1, 1], [9, 9, 1, 1], 0.0, 100.0, 20.0, 4, 1e-3)
    assert not r["success"] and r["flags"].tolist() == [1, 1, 1, 1]
    r = ref.threshold_classify([1, 1, 1, 1], [9, 1, 1, 1], 0.0, 100.0, 12.0, 4, 1e-3)
    assert r["success"] and r["finished_count"] == 3 and r["discarded_error"] == 3.0
    assert r["flags"].tolist() == [1, 0, 0, 0]
    r = ref.threshold_classify([1, 1], [5, 5], 1e6, 10.0, 10.0, 2, 1e-3)
    assert not r["success"]
    assert ref.rel_err_classify([1.0, 0.5], [1e-4, 1e-2], 1e-3).tolist() == [0, 1]
    assert ref.rel_err_classify([0.0, 0.0], [0.0, 1e-9], 1e-3).tolist() == [0, 1]
    assert ref.initial_subdivisions(8, 1 << 14) == 3
    lows, lens = ref.uniform_split([0, -1], [2, 1], 2)
    assert lows.shape == (4, 2) and (lens == 1.0).all()


def test_golden_traces_are_self_consistent():
    tr = load_golden("traces.json")
    assert "f4_5d_1e-3" in tr
    for name, case in tr.items():
        rows = case["trace"]
        assert len(rows) == case["result"]["iterations"], name
        last = rows[-1]
        assert unhex(last["v"]) is not None


def test_reference_matches_golden_traces(ref):
    """The reference library built here reproduces the committed goldens (the
    same fixtures the GPU tests compare against)."""
    tr = load_golden("traces.json")
    for name in ("f4_5d_1e-3", "f3_8d_1e-3", "f2_6d_1e-3", "f4_2d_1e-9_memtrigger", "nanbox_2d",
                 "rough_2d_doubling"):
        case = tr[name]
        cfg = make_config(tau_rel=case["tau"], rel_filtering_enabled=case["rel_filter"],
                          **case["extra"])
        res, rows = ref.trace(case["fid"], case["n"], cfg, params=case["params"])
        g = case["result"]
        assert res.estimate == unhex(g["estimate"]) and res.errorest == unhex(g["errorest"])
        assert (res.status, res.iterations, res.regions_generated) == (
            g["status"], g["iterations"], g["regions_generated"])
        for got, want in zip(rows, case["trace"]):
            for k, v in want.items():
                w = unhex(v)
                assert got[k] == w or (w != w and got[k] != got[k]), (name, k)


def test_reference_evaluate_matches_golden_batches(ref):
    batch = load_golden("batch.json")
    for name, b in list(batch.items())[::3]:
        lows = np.array([[unhex(v) for v in r] for r in b["lows"]])
        lens = np.array([[unhex(v) for v in r] for r in b["lengths"]])
        est, raw, axes, _ = ref.evaluate_batch(b["fid"], lows, lens)
        assert np.array_equal(bits(est), bits([unhex(v) for v in b["est"]])), name
        assert np.array_equal(bits(raw), bits([unhex(v) for v in b["raw"]])), name
        assert axes.tolist() == b["axes"], name


# --------------------------------------------------- the C restatement ------
PORT_CASES = [(4, 5, 1e-3, True), (3, 8, 1e-3, True), (1, 3, 1e-3, False), (2, 3, 1e-4, True),
              (5, 5, 1e-4, True), (6, 6, 1e-3, True), (7, 3, 1e-5, True), (8, 3, 1e-5, True),
              (4, 2, 1e-9, True), (2, 6, 1e-3, True)]


@pytest.mark.parametrize("fid,n,tau,relf", PORT_CASES)
def test_c_restatement_matches_reference_trace(port, ref, fid, n, tau, relf):
    cfg = make_config(tau_rel=tau, rel_filtering_enabled=relf)
    if (fid, n) == (4, 2):
        cfg = make_config(tau_rel=tau, max_regions=1 << 10, init_target=1 << 9)
    r1, rows1 = ref.trace(fid, n, cfg)
    r2, rows2 = port.trace(fid, n, cfg)
    assert (r1.estimate, r1.errorest, r1.status, r1.iterations, r1.regions_generated,
            r1.eval_count) == (r2.estimate, r2.errorest, r2.status, r2.iterations,
                               r2.regions_generated, r2.eval_count)
    assert rows1 == rows2


def test_c_restatement_batch_functions(port, ref):
    rng = np.random.default_rng(2024)
    for fid in range(1, 9):
        for n in (1, 2, 5, 8):
            lows = rng.uniform(0.0, 0.6, size=(50, n))
            lens = rng.uniform(0.01, 0.4, size=(50, n))
            a = ref.evaluate_batch(fid, lows, lens)
            b = port.evaluate_batch(fid, lows, lens)
            assert np.array_equal(bits(a[0]), bits(b[0])) and np.array_equal(bits(a[1]), bits(b[1]))
            assert np.array_equal(a[2], b[2]) and a[3] == b[3]
    for n in range(1, 17):
        pa, wa, qa = ref.build_rule(n)
        pb, wb, qb = port.build_rule(n)
        assert np.array_equal(bits(pa), bits(pb)) and np.array_equal(bits(wa), bits(wb))
        assert np.array_equal(qa, qb)
    # threshold trace oracle instances (test_classify.cpp:148-182 shape)
    for _ in range(300):
        m = 2 + int(rng.uniform() * 40)
        e = 10.0 ** (-6.0 * rng.uniform(size=m))
        act = (rng.uniform(size=m) < 0.8).astype(np.uint8)
        v_tot = rng.uniform() * 10
        e_it = float(e.sum())
        e_tot = e_it * (1 + rng.uniform())
        tau = 10.0 ** (-1.0 - 3.0 * rng.uniform())
        ra = ref.threshold_classify(act, e, v_tot, e_tot, e_it, m, tau)
        rb = port.threshold_classify(act, e, v_tot, e_tot, e_it, m, tau)
        assert ra["success"] == rb["success"] and np.array_equal(ra["flags"], rb["flags"])
        assert ra["threshold"] == rb["threshold"] and ra["attempts"] == rb["attempts"]
    x = rng.normal(size=10_000)
    f = (rng.uniform(size=10_000) < 0.5).astype(np.uint8)
    assert ref.block_sum(x) == port.block_sum(x)
    assert ref.block_sum_where(x, f, 0) == port.block_sum_where(x, f, 0)
