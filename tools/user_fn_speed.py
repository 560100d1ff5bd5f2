"""Time a user device functor (tests/ext/libuser_integrands.so, Gauss(0.5, 625)
== f4) against the built-in f4 on the same problem (dev helper)."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2104_06494_b200 as pg  # noqa: E402

lib = C.CDLL(os.environ.get("USER_LIB") or os.path.join(ROOT, "tests", "ext", "libuser_integrands.so"))
D = C.POINTER(C.c_double)
lib.user_integrate.argtypes = [C.c_int, D, C.c_int, C.c_double, C.c_int, C.c_int, D, D, D,
                               C.POINTER(C.c_int64)]
for n, tau in ((5, 1e-3), (8, 1e-3)):
    p = np.array([0.5, 625.0])
    od, oi = np.zeros(2), np.zeros(4, dtype=np.int64)
    for _ in range(2):
        t0 = time.perf_counter()
        lib.user_integrate(0, p.ctypes.data_as(D), n, tau, 1, 0, None, None, od.ctypes.data_as(D),
                           oi.ctypes.data_as(C.POINTER(C.c_int64)))
        tu = time.perf_counter() - t0
    for _ in range(2):
        t0 = time.perf_counter()
        r = pg.integrate(pg.Integrand(4), pg.Bounds.unit_cube(n), pg.Config(tau_rel=tau))
        tb = time.perf_counter() - t0
    print(f"f4 {n}D tau={tau}: user functor {tu*1e3:.1f} ms (est {od[0]!r}), builtin {tb*1e3:.1f} ms "
          f"(est {r.estimate!r}), same bits: {od[0] == r.estimate}")
