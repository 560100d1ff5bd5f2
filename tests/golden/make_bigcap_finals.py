"""Golden finals at a region cap above the reference default (2^24 regions,
8192 fold blocks): exercises the device paths that only large stores take
(pairwise trees in global memory instead of shared memory, 8192-block probe
passes).  From the UNMODIFIED reference (oracle/_ref), minutes of CPU.

Usage: python tests/golden/make_bigcap_finals.py  -> tests/golden/finals_bigcap.json
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from ref_ctypes import Ref, make_config  # noqa: E402

CASES = [(4, 8, 1e-6, 1 << 24), (2, 8, 1e-5, 1 << 24)]


def main():
    ref = Ref()
    path = os.path.join(HERE, "finals_bigcap.json")
    out = {}
    for fid, n, tau, cap in CASES:
        t0 = time.time()
        r = ref.integrate(fid, n, make_config(tau_rel=tau, rel_filtering_enabled=fid != 1,
                                              max_regions=cap))
        name = f"f{fid}_{n}d_{tau:g}_cap2^{cap.bit_length() - 1}"
        out[name] = {"fid": fid, "n": n, "tau": tau, "max_regions": cap,
                     "estimate": float(r.estimate).hex(), "errorest": float(r.errorest).hex(),
                     "status": r.status, "iterations": r.iterations,
                     "regions_generated": r.regions_generated, "eval_count": r.eval_count,
                     "n_events": len(r.threshold_events),
                     "cpu_seconds": round(time.time() - t0, 1)}
        print(name, r.status, r.iterations, r.estimate, f"{time.time() - t0:.1f}s", flush=True)
        json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
