"""Quick end-to-end parity check on a GPU box (development helper).

Runs a few integrate() calls on the GPU and the reference library (oracle/_ref)
and prints per-iteration trace diffs.  Usage: python tools/quick_parity.py [cases]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import paper_2104_06494_b200 as pg  # noqa: E402
from ref_ctypes import Ref, make_config  # noqa: E402

CASES = {
    "f4_3d": (4, 3, 1e-3, True),
    "f4_5d": (4, 5, 1e-3, True),
    "f3_8d": (3, 8, 1e-3, True),
    "f1_3d": (1, 3, 1e-3, False),
    "f2_3d": (2, 3, 1e-4, True),
    "f5_5d": (5, 5, 1e-4, True),
    "f6_6d": (6, 6, 1e-3, True),
    "f7_3d": (7, 3, 1e-5, True),
    "f8_3d": (8, 3, 1e-5, True),
}


def main():
    ref = Ref()
    names = sys.argv[1:] or list(CASES)
    ok_all = True
    for name in names:
        fid, n, tau, relf = CASES[name]
        t0 = time.time()
        res = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n),
                           pg.Config(tau_rel=tau, rel_filtering_enabled=relf, profile=True),
                           trace=True)
        t1 = time.time()
        eres, erows = ref.trace(fid, n, make_config(tau_rel=tau, rel_filtering_enabled=relf))
        t2 = time.time()
        same = (res.estimate == eres.estimate and res.errorest == eres.errorest
                and str(res.status) == eres.status and res.iterations == eres.iterations
                and res.regions_generated == eres.regions_generated
                and res.eval_count == eres.eval_count)
        nrow_diff = 0
        for a, b in zip(res.trace, erows):
            for k in b:
                va, vb = a[k], b[k]
                if va != vb and not (isinstance(va, float) and np.isnan(va) and np.isnan(vb)):
                    nrow_diff += 1
                    if nrow_diff <= 5:
                        print(f"   {name} it={b['it']} {k}: gpu={va!r} ref={vb!r}")
        same = same and nrow_diff == 0 and len(res.trace) == len(erows)
        ok_all &= same
        print(f"{name}: {'PARITY' if same else 'DIFF'} gpu est={res.estimate!r} it={res.iterations} "
              f"regions={res.regions_generated} status={res.status} | ref est={eres.estimate!r} "
              f"it={eres.iterations} regions={eres.regions_generated} status={eres.status} | "
              f"gpu {1e3*(t1-t0):.1f} ms (eval {res.kernel_ms['evaluate']:.2f} ms) "
              f"ref {1e3*(t2-t1):.0f} ms", flush=True)
    print("ALL PARITY" if ok_all else "SOME DIFF")


if __name__ == "__main__":
    main()
