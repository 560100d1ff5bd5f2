"""Command-line front-end with the reference CLI's CSV (bfcub_cli.cpp:24-26, 337-493).

    python -m paper_2104_06494_b200.cli integrate f4 5 1e-3
    python -m paper_2104_06494_b200.cli bench --k-max 2 --out bench.csv
    python -m paper_2104_06494_b200.cli compare --tau-rel 1e-3 --out compare.csv

The 13 CSV columns, their order and number formatting (%.17g) are the
reference's, so its CSV pipeline can consume this output unchanged.  Exit
codes mirror the reference: `integrate` returns 0 iff converged with true
relative error <= tau, 1 otherwise; usage errors return 2.  `compare` pits the
GPU's bit-exact parity engine against its fast engine (the reference compared
breadth-first vs its sequential oracle, which is out of scope here); the
agreement column uses the reference's rule |a - b| <= err_a + err_b.
"""
from __future__ import annotations

import argparse
import math
import sys
import time

from . import api as pg
from .suite import reference_value, suite

CSV_HEADER = ("integrand_id,dim,tau_rel,estimate,errorest,reference_value,true_rel_err,"
              "claimed_rel_err,status,iterations,regions_generated,eval_count,wall_ms")


def fmt(v: float) -> str:  # bfcub_cli.cpp:44-48 ("%.17g")
    return "%.17g" % v


def run_one(id_: str, dim: int, tau: float, opt, mode="parity"):
    """bfcub_cli.cpp:69-101 run_breadth_first."""
    ref = reference_value(id_, dim)
    cfg = pg.Config(tau_rel=tau, tau_abs=opt.tau_abs, max_regions=opt.max_regions,
                    it_max=opt.it_max, threads=opt.threads,
                    rel_filtering_enabled=not (opt.no_rel_filter or id_ == "f1"), mode=mode,
                    device=opt.device)
    t0 = time.perf_counter()
    r = pg.integrate(pg.integrand_by_id(id_), pg.Bounds.unit_cube(dim), cfg)
    wall = (time.perf_counter() - t0) * 1e3
    true_rel = abs(r.estimate - ref) / abs(ref)
    claimed = r.errorest / abs(r.estimate) if r.estimate != 0 else math.inf
    row = [id_, str(dim), fmt(tau), fmt(r.estimate), fmt(r.errorest), fmt(ref), fmt(true_rel),
           fmt(claimed), str(r.status), str(r.iterations), str(r.regions_generated),
           str(r.eval_count), fmt(wall)]
    return ",".join(row), r, true_rel


def parse_subset(text: str):
    out = []
    for item in text.split(","):
        if ":" not in item:
            raise ValueError(f"subset entries must look like f4:5, got '{item}'")
        i, d = item.split(":", 1)
        if not pg.known_integrand(i):
            raise ValueError(f"unknown integrand '{i}'")
        d = int(d)
        if d < 1 or d > 16:
            raise ValueError(f"bad dimension in '{item}'")
        reference_value(i, d)  # raises like the reference for f8 at other dims
        out.append((i, d))
    return out


def headline():
    return [(s.id, s.dim) for s in suite() if s.headline]


def _common(p):
    p.add_argument("--tau-abs", type=float, default=1e-20)
    p.add_argument("--max-regions", type=int, default=1 << 22)
    p.add_argument("--it-max", type=int, default=100)
    p.add_argument("--threads", type=int, default=0)
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--mode", choices=["parity", "fast"], default="parity")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="pagani", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    c_int = sub.add_parser("integrate", help="integrate one suite function")
    c_int.add_argument("id")
    c_int.add_argument("dim", type=int)
    c_int.add_argument("tau_rel", type=float)
    c_int.add_argument("--no-rel-filter", action="store_true")
    _common(c_int)
    c_b = sub.add_parser("bench", help="tolerance sweep tau = 1e-3 * 5^-k over the suite")
    c_b.add_argument("--subset", default=None)
    c_b.add_argument("--k-max", type=int, default=0, choices=range(0, 11))
    c_b.add_argument("--out", default="bench.csv")
    c_b.add_argument("--no-rel-filter", action="store_true")
    _common(c_b)
    c_c = sub.add_parser("compare", help="parity vs fast engine at one tolerance")
    c_c.add_argument("--subset", default=None)
    c_c.add_argument("--tau-rel", type=float, default=1e-3)
    c_c.add_argument("--out", default="compare.csv")
    c_c.add_argument("--no-rel-filter", action="store_true")
    _common(c_c)
    args = ap.parse_args(argv)

    try:
        if args.cmd == "integrate":
            if not pg.known_integrand(args.id):
                print(f"unknown integrand '{args.id}'", file=sys.stderr)
                return 2
            if args.dim < 1 or args.dim > 16 or not args.tau_rel > 0:
                print("bad dimension or tolerance", file=sys.stderr)
                return 2
            try:
                parse_subset(f"{args.id}:{args.dim}")
            except ValueError as e:
                print(str(e), file=sys.stderr)
                return 2
            line, r, true_rel = run_one(args.id, args.dim, args.tau_rel, args, args.mode)
            print(CSV_HEADER)
            print(line)
            return 0 if (r.status == pg.Status.Converged and true_rel <= args.tau_rel) else 1
        try:
            specs = parse_subset(args.subset) if args.subset is not None else headline()
        except ValueError as e:
            print(str(e), file=sys.stderr)
            return 2
        if args.cmd == "bench":
            with open(args.out, "w") as os_:
                os_.write(CSV_HEADER + "\n")
                for i, d in specs:
                    for k in range(args.k_max + 1):
                        os_.write(run_one(i, d, 1e-3 * 5.0 ** -k, args, args.mode)[0] + "\n")
            return 0
        with open(args.out, "w") as os_:  # compare
            os_.write("engine," + CSV_HEADER + ",agreement\n")
            for i, d in specs:
                a, ra, _ = run_one(i, d, args.tau_rel, args, "parity")
                b, rb, _ = run_one(i, d, args.tau_rel, args, "fast")
                agree = int(abs(ra.estimate - rb.estimate) <= ra.errorest + rb.errorest)
                os_.write(f"parity,{a},{agree}\nfast,{b},{agree}\n")
        return 0
    except Exception as e:  # noqa: BLE001 - mirrors the reference's catch-all (exit 1)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
