"""Per-iteration fixed cost on small runs (dev helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_06494_b200 as pg  # noqa: E402

for fid, n, tau in ((3, 8, 1e-3), (4, 5, 1e-3), (4, 3, 1e-3), (3, 3, 1e-6)):
    cfg = pg.Config(tau_rel=tau, profile=True)
    pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n), cfg)
    t0 = time.perf_counter()
    r = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n), cfg)
    wall = (time.perf_counter() - t0) * 1e3
    print(f"f{fid} {n}D {tau:g}: it={r.iterations} regions={r.regions_generated} events={len(r.threshold_events)} "
          f"wall={wall:.2f} ms device={r.device_ms:.2f} ms launches={sum(r.kernel_launches.values())} "
          + " ".join(f"{k}={v:.2f}" for k, v in r.kernel_ms.items() if v))
