"""Time k_evaluate for a library variant (PAGANI_LIB=...) on 8D cases (dev helper)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_06494_b200 as pg  # noqa: E402
from paper_2104_06494_b200 import roofline  # noqa: E402

CASES = [(4, 8, 1e-3, 100), (1, 8, 1e-3, 40), (2, 8, 1e-3, 100), (6, 8, 1e-4, 60), (4, 5, 1e-3, 100),
         (5, 8, 1e-3, 100), (3, 8, 1e-6, 100), (4, 10, 1e-3, 16)]
if os.environ.get("VARIANT_CASES"):  # e.g. "4:8:1e-3:100,1:8:1e-3:40"
    CASES = [tuple(t(v) for t, v in zip((int, int, float, int), c.split(":")))
             for c in os.environ["VARIANT_CASES"].split(",")]
out = {"lib": os.environ.get("PAGANI_LIB", "default")}
for fid, n, tau, itm in CASES:
    cfg = pg.Config(tau_rel=tau, it_max=itm, rel_filtering_enabled=fid != 1, profile=True)
    pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n), cfg)  # warm
    r = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n), cfg)
    ev = r.kernel_ms["evaluate"]
    tf = r.region_evals * roofline.region_flops(fid, n) / (ev / 1e3) / 1e12
    out[f"f{fid}_{n}d_{tau:g}"] = {"eval_ms": round(ev, 2), "device_ms": round(r.device_ms, 2),
                                  "tflops": round(tf, 2), "est": r.estimate.hex(),
                                  "regions": r.regions_generated}
print(json.dumps(out))
