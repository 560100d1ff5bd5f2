"""Fast mode vs parity mode over the 8D suite: decisions and final estimates (dev helper)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_06494_b200 as pg  # noqa: E402

rows = []
for fid in (1, 2, 3, 4, 5, 6):
    for tau in (1e-3, 1e-4, 1e-5, 1e-6):
        res = {}
        for mode in ("parity", "fast"):
            cfg = pg.Config(tau_rel=tau, rel_filtering_enabled=fid != 1, mode=mode, profile=True)
            res[mode] = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(8), cfg, trace=True)
        p, f = res["parity"], res["fast"]
        same = (str(p.status), p.iterations, p.regions_generated) == (str(f.status), f.iterations,
                                                                      f.regions_generated)
        ms_same = [r["m"] for r in p.trace] == [r["m"] for r in f.trace]
        rel = abs(f.estimate - p.estimate) / abs(p.estimate)
        rows.append({"case": f"f{fid}@{tau:g}", "decisions_identical": same and ms_same,
                     "rel_diff": rel, "eval_ms_parity": round(p.kernel_ms["evaluate"], 2),
                     "eval_ms_fast": round(f.kernel_ms["evaluate"], 2),
                     "device_ms_parity": round(p.device_ms, 2), "device_ms_fast": round(f.device_ms, 2)})
        print(json.dumps(rows[-1]), flush=True)
print(json.dumps({"all_identical": all(r["decisions_identical"] for r in rows),
                  "max_rel_diff": max(r["rel_diff"] for r in rows),
                  "eval_ms": [sum(r["eval_ms_parity"] for r in rows), sum(r["eval_ms_fast"] for r in rows)],
                  "device_ms": [sum(r["device_ms_parity"] for r in rows),
                                sum(r["device_ms_fast"] for r in rows)]}))
