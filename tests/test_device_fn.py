"""User-defined device integrands (include/pagani_device.cuh, PAGANI_DEVICE_FN):
the device counterpart of the reference's arbitrary {fn, ctx} integrand
(integrand.hpp:8-13).  tests/ext/libuser_integrands.so holds three functors
compiled in a caller's translation unit:
  Gauss(c, a)   exp(-a sum (x-c)^2) via pagani::Math::exp  == reference f4 at (0.5, 625)
  Oscillatory   cos(sum (i+1) x_i)  via pagani::Math::cos  == reference f1
  Product       x_0 x_1 ... (plain (x, n) functor)         == reference PAGANI_TEST_MONOMIAL [1..1]
so their integrations must be bit-identical to the reference's.
"""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import ROOT, bits
from ref_ctypes import make_config

LIB = os.path.join(ROOT, "tests", "ext", "libuser_integrands.so")
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)


@pytest.fixture(scope="module")
def ulib(pg):
    if not os.path.exists(LIB):
        pytest.fail("tests/ext/libuser_integrands.so not built (make -C tests/ext)")
    lib = C.CDLL(LIB)
    lib.user_integrate.argtypes = [C.c_int, _D, C.c_int, C.c_double, C.c_int, C.c_int, _D, _D,
                                   _D, _I64]
    lib.user_evaluate_batch.argtypes = [C.c_int, _D, C.c_int, C.c_int64, _D, _D, _D, _D,
                                        C.POINTER(C.c_int32)]
    return lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(_D)


def user_integrate(lib, which, n, tau, params=(0.0, 0.0), relf=True, mode=0, lower=None,
                   upper=None):
    p = np.array(params, dtype=np.float64)
    od = np.zeros(2)
    oi = np.zeros(4, dtype=np.int64)
    lo = None if lower is None else np.ascontiguousarray(lower, dtype=np.float64)
    hi = None if upper is None else np.ascontiguousarray(upper, dtype=np.float64)
    rc = lib.user_integrate(which, _dp(p), n, tau, int(relf), mode, _dp(lo), _dp(hi), _dp(od),
                            oi.ctypes.data_as(_I64))
    assert rc == 0
    status = ["converged", "max_iterations", "memory_exhausted"][oi[0]]
    return od[0], od[1], status, int(oi[1]), int(oi[2]), int(oi[3])


def test_library_exports_and_rejects_abi_mismatch(ulib):
    # runs on a CPU-only host: the descriptor is validated before any CUDA call
    assert ulib.user_integrate_bad_abi() == -1  # PAGANI_E_INVALID


@pytest.mark.gpu
@pytest.mark.parametrize("which,fid,n,tau,params,relf", [
    (0, 4, 3, 1e-3, (0.5, 625.0), True),
    (0, 4, 5, 1e-3, (0.5, 625.0), True),   # BASELINE config 1 with a user integrand
    (1, 1, 4, 1e-3, (0.0, 0.0), False),    # f1 runs with rel filtering off (bfcub_cli.cpp:77-78)
    (2, 101, 3, 1e-6, (0.0, 0.0), True),
])
def test_user_integrand_matches_reference(pg, gpu, ref, ulib, which, fid, n, tau, params, relf):
    est, err, status, it, regions, evals = user_integrate(ulib, which, n, tau, params, relf)
    rparams = [1.0] * n if fid == 101 else None
    want = ref.integrate(fid, n, make_config(tau_rel=tau, rel_filtering_enabled=relf),
                         params=rparams)
    assert (est, err, status, it, regions, evals) == (
        want.estimate, want.errorest, want.status, want.iterations, want.regions_generated,
        want.eval_count)


@pytest.mark.gpu
def test_user_integrand_batch_bit_exact(pg, gpu, ref, ulib):
    rng = np.random.default_rng(11)
    for which, fid, params in ((0, 4, (0.5, 625.0)), (1, 1, (0.0, 0.0))):
        for n in (2, 5, 8):
            m = 400
            lows = rng.uniform(0.0, 0.6, size=(m, n))
            lens = rng.uniform(0.01, 0.4, size=(m, n))
            est, raw = np.empty(m), np.empty(m)
            axes = np.empty(m, dtype=np.int32)
            p = np.array(params, dtype=np.float64)
            assert ulib.user_evaluate_batch(which, _dp(p), n, m, _dp(np.ascontiguousarray(lows)),
                                            _dp(np.ascontiguousarray(lens)), _dp(est), _dp(raw),
                                            axes.ctypes.data_as(C.POINTER(C.c_int32))) == 0
            e2, r2, a2, _ = ref.evaluate_batch(fid, lows, lens)
            assert np.array_equal(bits(est), bits(e2)) and np.array_equal(bits(raw), bits(r2))
            assert np.array_equal(axes, a2)


@pytest.mark.gpu
def test_user_integrand_state_and_bounds(pg, gpu, ulib):
    # a functor with its own parameters on a non-unit box: the Gaussian centred
    # at 0.25 with a = 50 on [-1, 1.5]^3 against the closed form
    from math import erf, pi, sqrt
    a, c = 50.0, 0.25
    est, err, status, *_ = user_integrate(ulib, 0, 3, 1e-7, params=(c, a),
                                          lower=[-1.0] * 3, upper=[1.5] * 3)
    one = sqrt(pi / a) / 2 * (erf(sqrt(a) * (1.5 - c)) - erf(sqrt(a) * (-1.0 - c)))
    assert status == "converged" and abs(est - one ** 3) <= 1e-6 * one ** 3


@pytest.mark.gpu
def test_user_integrand_fast_mode(pg, gpu, ulib):
    e0 = user_integrate(ulib, 0, 5, 1e-3, (0.5, 625.0), mode=0)
    e1 = user_integrate(ulib, 0, 5, 1e-3, (0.5, 625.0), mode=1)
    assert abs(e1[0] - e0[0]) <= 1e-12 * abs(e0[0])
