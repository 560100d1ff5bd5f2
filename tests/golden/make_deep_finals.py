"""Golden final results of the BASELINE configs at full size, from the
UNMODIFIED reference (oracle/_ref/libbfcub_ref.so, OpenMP on all cores).

  configs[1]  f1..f6 8D at tau in {1e-3, 1e-4, 1e-5, 1e-6} (bench.py's workload)
  configs[2]  f2 8D tau=1e-9
  configs[3]  f5 and f6 8D tau=1e-8
all at the reference defaults (max_regions 2^22, it_max 100, tau_abs 1e-20,
rel filtering off for f1 only).  Tens of minutes of CPU in total; the output
(tests/golden/finals_deep.json, hex floats) is committed and checked by
tests/test_gpu_parity.py::test_integrate_matches_reference_finals_deep.

Usage: python tests/golden/make_deep_finals.py
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from ref_ctypes import Ref, make_config  # noqa: E402

CASES = [(fid, 8, tau) for tau in (1e-3, 1e-4, 1e-5, 1e-6) for fid in (1, 2, 3, 4, 5, 6)]
CASES += [(2, 8, 1e-9), (5, 8, 1e-8), (6, 8, 1e-8)]


def main():
    ref = Ref()
    path = os.path.join(HERE, "finals_deep.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for fid, n, tau in CASES:
        name = f"f{fid}_{n}d_{tau:g}"
        if name in out:
            continue
        t0 = time.time()
        r = ref.integrate(fid, n, make_config(tau_rel=tau, rel_filtering_enabled=fid != 1))
        out[name] = {"fid": fid, "n": n, "tau": tau, "estimate": float(r.estimate).hex(),
                     "errorest": float(r.errorest).hex(), "status": r.status,
                     "iterations": r.iterations, "regions_generated": r.regions_generated,
                     "eval_count": r.eval_count, "n_events": len(r.threshold_events),
                     "cpu_seconds": round(time.time() - t0, 1), "cpu_threads": os.cpu_count()}
        print(f"{name}: {r.status} it={r.iterations} est={r.estimate!r} "
              f"({time.time() - t0:.1f}s)", flush=True)
        json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
