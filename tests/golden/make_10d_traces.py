"""Full-length golden traces of the 10D configuration (BASELINE configs[4],
f4 Gaussian 10D) from the UNMODIFIED reference (oracle/_ref/libbfcub_ref.so,
OpenMP on all cores).

The 10D kernels are their own template instance (N = 1245 rule points, a
different launch bound and staging size), so they get their own full-length
pins: every per-iteration field (m, active counts, v, e, finished sums,
threshold events) plus the final result, at

  * cap 2^22 (reference default), tau = 1e-3   -> memory_exhausted, ~38 its
  * cap 2^22,                     tau = 1e-7   -> BASELINE configs[4]'s tau
  * cap 2^24,                     tau = 1e-3   -> 8192 fold blocks at 10D

Tens of CPU-minutes in total.  Output: tests/golden/traces_10d.json (hex
floats), checked by tests/test_gpu_parity.py::test_integrate_matches_10d_traces.

Usage: python tests/golden/make_10d_traces.py
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from ref_ctypes import Ref, make_config  # noqa: E402

CASES = [  # (name, fid, n, tau, max_regions)
    ("f4_10d_1e-3_cap2^22", 4, 10, 1e-3, 1 << 22),
    ("f4_10d_1e-7_cap2^22", 4, 10, 1e-7, 1 << 22),
    ("f4_10d_1e-3_cap2^24", 4, 10, 1e-3, 1 << 24),
]


def hx(x):
    return float(x).hex()


def main():
    ref = Ref()
    path = os.path.join(HERE, "traces_10d.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    only = sys.argv[1:]
    for name, fid, n, tau, cap in CASES:
        if name in out or (only and name not in only):
            continue
        t0 = time.time()
        cfg = make_config(tau_rel=tau, rel_filtering_enabled=fid != 1, max_regions=cap)
        res, rows = ref.trace(fid, n, cfg)
        fin = ref.integrate(fid, n, make_config(tau_rel=tau, rel_filtering_enabled=fid != 1,
                                                max_regions=cap))
        # the trace re-drives the public functions in driver.cpp order; it must
        # end where integrate() ends
        assert (res.estimate, res.errorest, res.status, res.iterations) == (
            fin.estimate, fin.errorest, fin.status, fin.iterations), name
        out[name] = {
            "fid": fid, "n": n, "tau": tau, "max_regions": cap,
            "result": {"estimate": hx(fin.estimate), "errorest": hx(fin.errorest),
                       "status": fin.status, "iterations": fin.iterations,
                       "regions_generated": fin.regions_generated,
                       "eval_count": fin.eval_count,
                       "threshold_events": [
                           {**e, "discarded_error": hx(e["discarded_error"]),
                            "budget_limit": hx(e["budget_limit"])}
                           for e in fin.threshold_events]},
            "trace": [{k: (hx(v) if isinstance(v, float) else v) for k, v in r.items()}
                      for r in rows],
            "cpu_seconds": round(time.time() - t0, 1), "cpu_threads": os.cpu_count()}
        print(f"{name}: {fin.status} it={fin.iterations} est={fin.estimate!r} "
              f"regions={fin.regions_generated} ({time.time() - t0:.1f}s)", flush=True)
        json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
