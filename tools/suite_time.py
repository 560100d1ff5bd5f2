import sys, time
sys.path.insert(0, '/root/repo')
import paper_2104_06494_b200 as pg
prof = sys.argv[1] == '1'
def step():
    ms = 0.0; ev = 0
    for f in range(1, 7):
        for tau in (1e-3, 1e-4, 1e-5, 1e-6):
            r = pg.integrate(pg.Integrand(f), pg.Bounds.unit_cube(8), pg.Config(tau_rel=tau, rel_filtering_enabled=f != 1, profile=prof))
            ms += r.device_ms; ev += r.region_evals
    return ms, ev
for _ in range(2): step()
res = [step() for _ in range(4)]
ms = sorted(r[0] for r in res)
print(f"profile={prof} step_ms median={ms[1]:.1f} min={ms[0]:.1f} rate={res[0][1]/(ms[1]/1e3):.4g}")
