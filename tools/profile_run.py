"""Single integrate() call for ncu captures (development helper).

  python tools/profile_run.py FID N TAU [IT_MAX] [MODE]
e.g. ncu --set full -k regex:k_evaluate -s 12 -c 1 python tools/profile_run.py 4 8 1e-3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_06494_b200 as pg  # noqa: E402

fid, n, tau = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
it_max = int(sys.argv[4]) if len(sys.argv) > 4 else 100
mode = sys.argv[5] if len(sys.argv) > 5 else "parity"
r = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n),
                 pg.Config(tau_rel=tau, it_max=it_max, rel_filtering_enabled=fid != 1, mode=mode,
                           profile=True))
print(f"f{fid} {n}D tau={tau}: est={r.estimate!r} status={r.status} it={r.iterations} "
      f"regions={r.regions_generated} device_ms={r.device_ms:.2f}")
print({k: round(v, 3) for k, v in r.kernel_ms.items()})
print(r.kernel_launches)
