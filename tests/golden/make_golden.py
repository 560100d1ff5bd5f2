#!/usr/bin/env python3
"""Generate tests/golden/*.json from the UNMODIFIED reference library.

Runs oracle/_ref/libbfcub_ref.so (built by `make -C oracle ref` from
/root/reference/proj/src) in this container and records:
  * traces.json   full-precision per-iteration traces + final results of small
                  and medium configs (the parity pins for the GPU path)
  * finals.json   final IntegrationResults of the BASELINE 8D configs at the
                  reference default cap 2^22 (minutes of CPU each; GPU tests
                  compare against these without re-running the reference)
  * rule.json     orbit weights (hex) for n = 1..16
  * batch.json    evaluate_batch outputs (hex) on seeded random batches
Floats are stored as hex strings (float.hex) so they round-trip exactly.

Usage: python tests/golden/make_golden.py [--skip-finals]
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from ref_ctypes import Ref, make_config  # noqa: E402

# (name, fid, n, tau, rel_filter, extra config, params)
TRACE_CASES = [
    ("f4_5d_1e-3", 4, 5, 1e-3, True, {}, None),           # BASELINE config 1
    ("f3_8d_1e-3", 3, 8, 1e-3, True, {}, None),
    ("f1_3d_1e-3_nofilter", 1, 3, 1e-3, False, {}, None),
    ("f1_2d_1e-6_nofilter", 1, 2, 1e-6, False, {}, None),
    ("f2_3d_1e-4", 2, 3, 1e-4, True, {}, None),
    ("f2_6d_1e-3", 2, 6, 1e-3, True, {}, None),
    ("f3_3d_1e-6", 3, 3, 1e-6, True, {}, None),
    ("f4_3d_5e-7_small_cap", 4, 3, 5e-7, True, {"max_regions": 1 << 12, "init_target": 1 << 10}, None),
    ("f4_2d_1e-9_memtrigger", 4, 2, 1e-9, True, {"max_regions": 1 << 10, "init_target": 1 << 9}, None),
    ("f5_5d_1e-4", 5, 5, 1e-4, True, {}, None),
    ("f6_6d_1e-3", 6, 6, 1e-3, True, {}, None),
    ("f6_3d_1e-5", 6, 3, 1e-5, True, {}, None),
    ("f7_3d_1e-5", 7, 3, 1e-5, True, {}, None),
    ("f8_2d_1e-7", 8, 2, 1e-7, True, {}, None),
    ("f8_3d_1e-5", 8, 3, 1e-5, True, {}, None),
    ("f4_10d_1e-3_it8", 4, 10, 1e-3, True, {"it_max": 8}, None),
    ("f5_8d_1e-3_it8", 5, 8, 1e-3, True, {"it_max": 8}, None),
    ("f4_1d_1e-9", 4, 1, 1e-9, True, {}, None),
    ("f2_4d_identity_refiner", 2, 4, 1e-3, True, {"refiner": 1}, None),
    ("rough_2d_doubling", 102, 2, 1e-12, False, {"init_subdiv": 2, "it_max": 4}, [40.0, 1.0, 2.0]),
    ("rough_2d_memexhausted", 102, 2, 1e-10, False, {"max_regions": 1 << 8, "init_target": 1 << 7},
     [50.0, 2.0, 2.0]),
    ("nanbox_2d", 103, 2, 1e-6, True, {"max_regions": 1 << 10, "init_target": 1 << 8, "it_max": 12},
     [0.8, -1.0]),
    ("const_3d", 100, 3, 1e-3, True, {"init_subdiv": 2}, [1.0]),
    ("expsq_4d", 106, 4, 1e-6, True, {}, None),
    ("cossum_3d", 105, 3, 1e-5, True, {}, [1.5, 0.7, 1.9, 2.6]),
]

# BASELINE 8D configs (finals only; minutes of CPU each)
FINAL_CASES = [
    ("f3_8d_1e-3", 3, 1e-3), ("f4_8d_1e-3", 4, 1e-3), ("f5_8d_1e-3", 5, 1e-3),
    ("f6_8d_1e-3", 6, 1e-3), ("f2_8d_1e-3", 2, 1e-3), ("f4_5d_1e-7", 4, 1e-7),
]


def hx(x):
    return float(x).hex()


def row_hex(row):
    return {k: (hx(v) if isinstance(v, float) else v) for k, v in row.items()}


def main():
    skip_finals = "--skip-finals" in sys.argv
    ref = Ref()
    out = {}
    for name, fid, n, tau, relf, extra, params in TRACE_CASES:
        cfg = make_config(tau_rel=tau, rel_filtering_enabled=relf, **extra)
        t0 = time.time()
        res, rows = ref.trace(fid, n, cfg, params=params, max_rows=200)
        full = ref.integrate(fid, n, cfg, params=params)
        assert (res.estimate, res.errorest, res.status, res.iterations, res.regions_generated,
                res.eval_count) == (full.estimate, full.errorest, full.status, full.iterations,
                                    full.regions_generated, full.eval_count), name
        out[name] = {"fid": fid, "n": n, "tau": tau, "rel_filter": relf, "extra": extra,
                     "params": params,
                     "result": {"estimate": hx(res.estimate), "errorest": hx(res.errorest),
                                "status": res.status, "iterations": res.iterations,
                                "regions_generated": res.regions_generated,
                                "eval_count": res.eval_count,
                                "threshold_events": [
                                    {k: (hx(v) if isinstance(v, float) else v) for k, v in e.items()}
                                    for e in full.threshold_events]},
                     "trace": [row_hex(r) for r in rows]}
        print(f"trace {name}: {res.status} it={res.iterations} ({time.time() - t0:.1f}s)", flush=True)
    json.dump(out, open(os.path.join(HERE, "traces.json"), "w"), indent=0)

    rule = {}
    for n in range(1, 17):
        pts, w, probes = ref.build_rule(n)
        firsts = [0, 1, 1 + 2 * n, 1 + 4 * n, 1 + 4 * n + 2 * n * (n - 1)]
        rule[str(n)] = {"point_count": int(pts.shape[0]),
                        "orbit_weights": [[hx(w[k, firsts[o]]) if not (o == 3 and n == 1) else None
                                           for o in range(5)] for k in range(5)],
                        "generators": [hx(pts[1, 0]), hx(pts[1 + 2 * n, 0]) if n >= 1 else None,
                                       hx(pts[1 + 4 * n, 0]) if n >= 2 else None,
                                       hx(pts[-1, 0])],
                        "probes": probes.tolist()}
    json.dump(rule, open(os.path.join(HERE, "rule.json"), "w"), indent=0)

    rng = np.random.default_rng(1234)
    batch = {}
    for fid in (1, 2, 3, 4, 5, 6, 7, 8):
        for n in (2, 5, 8):
            m = 64
            lows = rng.uniform(0.0, 0.6, size=(m, n))
            lens = rng.uniform(0.05, 0.4, size=(m, n))
            est, raw, axes, cnt = ref.evaluate_batch(fid, lows, lens)
            batch[f"f{fid}_{n}d"] = {"fid": fid, "n": n,
                                     "lows": [[hx(v) for v in r] for r in lows],
                                     "lengths": [[hx(v) for v in r] for r in lens],
                                     "est": [hx(v) for v in est], "raw": [hx(v) for v in raw],
                                     "axes": axes.tolist(), "eval_count": cnt}
    json.dump(batch, open(os.path.join(HERE, "batch.json"), "w"))

    if not skip_finals:
        finals = {}
        for name, fid, tau in FINAL_CASES:
            n = int(name.split("_")[1][:-1])
            cfg = make_config(tau_rel=tau, rel_filtering_enabled=fid != 1)
            t0 = time.time()
            r = ref.integrate(fid, n, cfg)
            finals[name] = {"fid": fid, "n": n, "tau": tau, "estimate": hx(r.estimate),
                            "errorest": hx(r.errorest), "status": r.status,
                            "iterations": r.iterations, "regions_generated": r.regions_generated,
                            "eval_count": r.eval_count, "n_events": len(r.threshold_events),
                            "cpu_seconds": round(time.time() - t0, 1)}
            print(f"final {name}: {r.status} it={r.iterations} est={r.estimate!r} "
                  f"({time.time() - t0:.1f}s)", flush=True)
            json.dump(finals, open(os.path.join(HERE, "finals.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
