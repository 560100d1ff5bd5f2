"""Executed FP64 FLOPs per region-evaluation of k_evaluate, from the ncu SASS
op counters of tools/exec_flops.sh (2 per DFMA, 1 per DMUL / DADD), next to
the algorithmic (reference-arithmetic) count of roofline.py.

  python tools/exec_flops.py gpurun_out > profiles/r02_executed_flops.json
"""
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_06494_b200 import roofline  # noqa: E402

d = sys.argv[1]
out = {"source": "ncu smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum over "
                 "every k_evaluate launch of f{1..6} 8D tau=1e-3 it_max=12 (tools/exec_flops.sh)",
       "per_integrand": {}}
for f in range(1, 7):
    rows = list(csv.reader(open(os.path.join(d, f"r02_execflops_f{f}.csv"))))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    tot = {"dfma": 0.0, "dmul": 0.0, "dadd": 0.0, "ns": 0.0}
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        name, val = r[h.index("Metric Name")], float(r[h.index("Metric Value")].replace(",", ""))
        for k in ("dfma", "dmul", "dadd"):
            if f"op_{k}_pred_on" in name:
                tot[k] += val
        if name == "gpu__time_duration.sum":
            unit = r[h.index("Metric Unit")]
            tot["ns"] += val * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6,
                                "msecond": 1e6}.get(unit, 1)
    log = open(os.path.join(d, f"r02_execflops_f{f}.log")).read()
    regions = int(re.search(r"regions=(\d+)", log).group(1))
    exec_flops = 2 * tot["dfma"] + tot["dmul"] + tot["dadd"]
    alg = roofline.region_flops(f, 8)
    out["per_integrand"][f"f{f}"] = {
        "region_evals": regions, "executed_fp64_flops_per_region": exec_flops / regions,
        "algorithmic_flops_per_region": alg, "executed_over_algorithmic": exec_flops / regions / alg,
        "executed_tflops_cold_ncu": exec_flops / (tot["ns"] * 1e-9) / 1e12 if tot["ns"] else None}
print(json.dumps(out, indent=1))
