"""Predicted strong scaling of the sharded driver -- a MODEL from
single-GPU measurements, not a multi-GPU measurement (this pod has one GPU).

Inputs
  * a tools/baseline_configs.py JSON (one B200: device time, per-kernel-class
    CUDA-event time, iterations, threshold passes);
  * the sharded runs' exchange log (tests/test_gpu_multirank.py with
    PAGANI_XCHG_LOG; R ranks sharing one GPU): bytes each rank sent per
    iteration, as a fraction of the bytes of the children it produced, and the
    region-evaluation imbalance between ranks.

Model, per integrate() call on R GPUs:
  T(R) = (evaluate + fold + split + probe + init) / R * imbalance   [data-parallel]
       + finalize                                                   [trees over the gathered records, replicated]
       + gaps                                                       [host decisions between launches, replicated]
       + (iterations + probe passes) * alpha                        [one small allgather each]
       + iterations * (exchange bytes per rank / link BW + alpha)   [post-bisection boundary exchange]
with alpha = 20 us (NCCL small-message latency on NVLink/NVSwitch) and an
effective 400 GB/s per-rank point-to-point bandwidth (NVLink 5: 900 GB/s per
direction).

  python tools/scaling_model.py BASELINE_JSON XCHG_JSON > profiles/r02_scaling_model.json
"""
import json
import sys
from collections import defaultdict

ALPHA_S = 20e-6
P2P_BPS = 400e9


def exchange_fraction(xchg):
    """Per R: max over cases of (max per-rank bytes sent per iteration) /
    (per-rank child bytes per iteration), and the region-eval imbalance."""
    agg = defaultdict(list)
    for r in xchg:
        agg[(r["case"], r["ranks"])].append(r)
    frac, imb = defaultdict(float), defaultdict(float)
    for (case, R), rs in agg.items():
        n = int(case.split()[1].rstrip("D"))
        it = rs[0]["iterations"]
        evals = sum(r["local_region_evals"] for r in rs)
        child_bytes_per_rank_it = evals / it / R * (16 * n + 8)
        mx = max(r["exchange_bytes"] for r in rs) / it
        frac[R] = max(frac[R], mx / child_bytes_per_rank_it)
        e = [r["local_region_evals"] for r in rs]
        imb[R] = max(imb[R], max(e) / (sum(e) / len(e)))
    return frac, imb


def predict(row, R, frac, imb):
    km = row["kernel_ms"]
    t1 = row["time_to_result_s"]
    par = sum(km.get(k, 0.0) for k in ("evaluate", "fold", "split", "probe", "init")) / 1e3
    rep = km.get("finalize", 0.0) / 1e3
    gaps = max(0.0, t1 - par - rep - km.get("minmax", 0.0) / 1e3)
    if R == 1:
        return t1
    it = row["iterations"]
    passes = row.get("kernel_launches", {}).get("probe", 0) // 2  # 2 launches per pass (1 GPU)
    n = row["n"]
    child_bytes_rank_it = row["region_evals"] / it / R * (16 * n + 8)
    xbytes = frac.get(R, max(frac.values()) if frac else 0.06) * child_bytes_rank_it
    comm = (it + passes) * ALPHA_S + it * (xbytes / P2P_BPS + ALPHA_S)
    return par / R * imb.get(R, 1.0) + rep + gaps + comm


def main():
    rows = json.load(open(sys.argv[1]))
    frac, imb = exchange_fraction(json.load(open(sys.argv[2])))
    out = {"model": __doc__.split("Model, per integrate() call on R GPUs:")[1].strip(),
           "measured_exchange_fraction": {str(k): round(v, 4) for k, v in sorted(frac.items())},
           "measured_imbalance": {str(k): round(v, 4) for k, v in sorted(imb.items())},
           "cases": []}
    for row in rows:
        t = {R: predict(row, R, frac, imb) for R in (1, 2, 4, 8)}
        out["cases"].append({
            "config": row["config"], "case": f"{row['f']} {row['n']}D tau={row['tau']:g}",
            "max_regions": row["max_regions"], "iterations": row["iterations"],
            "t1_s_measured": round(t[1], 5),
            "predicted_s": {str(R): round(t[R], 5) for R in (2, 4, 8)},
            "predicted_speedup": {str(R): round(t[1] / t[R], 2) for R in (2, 4, 8)}})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
