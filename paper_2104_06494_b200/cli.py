"""Command-line front-end with the reference CLI's CSV (bfcub_cli.cpp:24-26, 337-493).

    python -m paper_2104_06494_b200.cli integrate f4 5 1e-3
    python -m paper_2104_06494_b200.cli bench --k-max 2 --out bench.csv
    python -m paper_2104_06494_b200.cli compare --tau-rel 1e-3 --out compare.csv
    python -m paper_2104_06494_b200.cli plot bench.csv --out-dir plots

The 13 CSV columns, their order and number formatting (%.17g) are the
reference's, and the reference_value column is its long-double closed form to
the last bit (csrc/suite.cpp), so a row of this CSV equals the reference's
row except for wall_ms.  Exit codes mirror the reference: `integrate` returns
0 iff converged with true relative error <= tau, 1 otherwise; usage errors
return 2.  `compare` pits the breadth-first engine against the sequential one
(integrate_sequential, both on the GPU), as the reference does
(bfcub_cli.cpp:454-485); `--fast-vs-parity` compares the two breadth-first
numeric modes instead.  The agreement column uses the reference's rule
|a - b| <= err_a + err_b.  `plot` renders a bench CSV to accuracy.svg and
regions.svg like bfcub_cli.cpp:189-333.
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


def fmt(v: float) -> str:  # bfcub_cli.cpp:44-48 ("%.17g", glibc spelling of nan)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.17g" % v


def _div(a: float, b: float) -> float:
    """IEEE a / b (C++ semantics: x/0 = +-inf, 0/0 = nan)."""
    if b == 0.0:
        if a == 0.0 or math.isnan(a):
            return math.nan
        return math.copysign(math.inf, a) * math.copysign(1.0, b)
    return a / b


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
    return _record(id_, dim, tau, ref, r, wall)


def _record(id_, dim, tau, ref, r, wall):
    true_rel = _div(abs(r.estimate - ref), abs(ref))
    claimed = _div(r.errorest, abs(r.estimate))
    row = [id_, str(dim), fmt(tau), fmt(r.estimate), fmt(r.errorest), fmt(ref), fmt(true_rel),
           fmt(claimed), str(r.status), str(r.iterations), str(r.regions_generated),
           str(r.eval_count), fmt(wall)]
    return ",".join(row), r, true_rel


def run_sequential(id_: str, dim: int, tau: float, opt, max_evals: int):
    """bfcub_cli.cpp:103-127 run_sequential (the GPU-evaluated sequential engine)."""
    ref = reference_value(id_, dim)
    t0 = time.perf_counter()
    r = pg.integrate_sequential(pg.integrand_by_id(id_), pg.Bounds.unit_cube(dim), tau,
                                tau_abs=opt.tau_abs, max_evals=max_evals, device=opt.device)
    wall = (time.perf_counter() - t0) * 1e3
    return _record(id_, dim, tau, ref, r, wall)


# ---- SVG plotting (bfcub_cli.cpp:189-333) -----------------------------------
_PALETTE = ["#1f77b4", "#d62728", "#2ca02c", "#9467bd", "#ff7f0e", "#8c564b", "#17becf",
            "#e377c2", "#7f7f7f", "#bcbd22"]


def _g(v) -> str:  # std::ostream << double (defaultfloat, precision 6)
    return str(v) if isinstance(v, int) else "%g" % v


def write_log_scatter(path, title, y_label, pts, tau_line):
    """pts: [(digits, y, converged, series)]."""
    W, H, L, R, T, B = 760.0, 520.0, 70.0, 180.0, 40.0, 50.0
    xmin, xmax, ymin, ymax = 1e300, -1e300, 1e300, -1e300
    for d, y, _, _ in pts:
        xmin, xmax = min(xmin, d), max(xmax, d)
        if y > 0:
            ymin, ymax = min(ymin, y), max(ymax, y)
    if xmin > xmax:
        xmin, xmax = 2.0, 11.0
    xmin = math.floor(xmin) - 0.5
    xmax = math.ceil(xmax) + 0.5
    if ymin > ymax:
        ymin, ymax = 1e-12, 1.0
    if tau_line:
        ymin = min(ymin, math.pow(10.0, -xmax))
        ymax = max(ymax, math.pow(10.0, -xmin))
    ly0 = math.floor(math.log10(ymin)) - 0.5
    ly1 = math.ceil(math.log10(ymax)) + 0.5

    def X(d):
        return L + (d - xmin) / (xmax - xmin) * (W - L - R)

    def Y(v):
        ly = math.log10(max(v, 1e-300))
        return H - B - (ly - ly0) / (ly1 - ly0) * (H - T - B)

    o = [f"<svg xmlns='http://www.w3.org/2000/svg' width='{_g(W)}' height='{_g(H)}'>\n"
         "<rect width='100%' height='100%' fill='white'/>\n",
         f"<text x='{_g(W / 2)}' y='20' text-anchor='middle' font-size='15'>{title}</text>\n",
         f"<line x1='{_g(L)}' y1='{_g(H - B)}' x2='{_g(W - R)}' y2='{_g(H - B)}' "
         "stroke='black'/>\n",
         f"<line x1='{_g(L)}' y1='{_g(T)}' x2='{_g(L)}' y2='{_g(H - B)}' stroke='black'/>\n"]
    d = int(math.ceil(xmin))
    while d <= xmax:
        o.append(f"<line x1='{_g(X(d))}' y1='{_g(H - B)}' x2='{_g(X(d))}' y2='{_g(H - B + 5)}' "
                 f"stroke='black'/>\n<text x='{_g(X(d))}' y='{_g(H - B + 18)}' "
                 f"text-anchor='middle' font-size='11'>{d}</text>\n")
        d += 1
    e = int(math.ceil(ly0))
    while e <= ly1:
        yy = Y(math.pow(10.0, e))
        o.append(f"<line x1='{_g(L - 5)}' y1='{_g(yy)}' x2='{_g(L)}' y2='{_g(yy)}' "
                 f"stroke='black'/>\n<text x='{_g(L - 8)}' y='{_g(yy + 4)}' "
                 f"text-anchor='end' font-size='11'>1e{e}</text>\n")
        e += 1
    o.append(f"<text x='{_g((L + W - R) / 2)}' y='{_g(H - 12)}' text-anchor='middle' "
             "font-size='12'>digits of precision, log10(1/tau_rel)</text>\n")
    o.append(f"<text x='18' y='{_g((T + H - B) / 2)}' text-anchor='middle' font-size='12' "
             f"transform='rotate(-90 18 {_g((T + H - B) / 2)})'>{y_label}</text>\n")
    if tau_line:
        o.append("<polyline fill='none' stroke='black' stroke-dasharray='5,4' points='")
        d = xmin
        while d <= xmax + 1e-9:
            o.append(f"{_g(X(d))},{_g(Y(math.pow(10.0, -d)))} ")
            d += (xmax - xmin) / 64.0
        o.append("'/>\n")
    color = {}
    for p in pts:
        if p[3] not in color:
            color[p[3]] = len(color) % 10
    for dd, y, conv, series in pts:
        c = _PALETTE[color[series]]
        if conv:
            o.append(f"<circle cx='{_g(X(dd))}' cy='{_g(Y(y))}' r='4' fill='{c}'/>\n")
        else:  # non-converged runs are drawn as crosses
            cx, cy = X(dd), Y(y)
            o.append(f"<path d='M{_g(cx - 4)} {_g(cy - 4)} L{_g(cx + 4)} {_g(cy + 4)} "
                     f"M{_g(cx - 4)} {_g(cy + 4)} L{_g(cx + 4)} {_g(cy - 4)}' stroke='{c}' "
                     "stroke-width='2'/>\n")
    for row, name in enumerate(sorted(color, key=lambda k: k.encode())):
        yy = T + 16 + 18 * row
        o.append(f"<circle cx='{_g(W - R + 18)}' cy='{_g(yy)}' r='4' fill='{_PALETTE[color[name]]}'/>"
                 f"\n<text x='{_g(W - R + 30)}' y='{_g(yy + 4)}' font-size='12'>{name}</text>\n")
    o.append("</svg>\n")
    with open(path, "w") as f:
        f.write("".join(o))


def cmd_plot(csv_path: str, out_dir: str) -> int:
    """bfcub_cli.cpp:286-333."""
    try:
        f = open(csv_path)
    except OSError:
        print(f"plot: cannot open {csv_path}", file=sys.stderr)
        return 2
    with f:
        lines = f.read().split("\n")
    if not lines or lines[0] != CSV_HEADER:
        print(f"plot: {csv_path} is not a bench CSV", file=sys.stderr)
        return 2
    acc, reg = [], []
    for line in lines[1:]:
        if not line:
            continue
        cells = line.split(",")
        if len(cells) != 13:
            print(f"plot: malformed row '{line}'", file=sys.stderr)
            return 2
        series = cells[0] + ":" + cells[1]
        try:
            tau, true_err, regions = float(cells[2]), float(cells[6]), float(cells[10])
        except ValueError:
            tau, true_err, regions = 0.0, 0.0, 0.0
        if not tau > 0:
            print(f"plot: bad tau_rel in '{line}'", file=sys.stderr)
            return 2
        conv = cells[8] == "converged"
        digits = math.log10(1.0 / tau)
        acc.append((digits, max(true_err, 1e-17), conv, series))
        reg.append((digits, max(regions, 1.0), conv, series))
    if not acc:
        print(f"plot: no data rows in {csv_path}", file=sys.stderr)
        return 2
    write_log_scatter(f"{out_dir}/accuracy.svg", "true relative error vs requested precision",
                      "true relative error", acc, True)
    write_log_scatter(f"{out_dir}/regions.svg", "generated sub-regions vs requested precision",
                      "sub-regions generated", reg, False)
    print(f"wrote {out_dir}/accuracy.svg and {out_dir}/regions.svg")
    return 0


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
    c_c = sub.add_parser("compare", help="breadth-first vs sequential at one tolerance")
    c_c.add_argument("--subset", default=None)
    c_c.add_argument("--tau-rel", type=float, default=1e-3)
    c_c.add_argument("--out", default="compare.csv")
    c_c.add_argument("--max-evals", type=int, default=10_000_000)
    c_c.add_argument("--no-rel-filter", action="store_true")
    c_c.add_argument("--fast-vs-parity", action="store_true",
                     help="compare the breadth-first parity and fast modes instead")
    _common(c_c)
    c_p = sub.add_parser("plot", help="render a bench CSV to SVG")
    c_p.add_argument("csv")
    c_p.add_argument("--out-dir", default=".")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:  # CLI11 returns 2 on parse errors, 0 for --help
        return 0 if e.code == 0 else 2
    if args.cmd == "plot":
        return cmd_plot(args.csv, args.out_dir)

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
        with open(args.out, "w") as os_:  # compare (bfcub_cli.cpp:454-485)
            os_.write("engine," + CSV_HEADER + ",agreement\n")
            for i, d in specs:
                if args.fast_vs_parity:
                    a, ra, _ = run_one(i, d, args.tau_rel, args, "parity")
                    b, rb, _ = run_one(i, d, args.tau_rel, args, "fast")
                    names = ("parity", "fast")
                else:
                    a, ra, _ = run_one(i, d, args.tau_rel, args, args.mode)
                    b, rb, _ = run_sequential(i, d, args.tau_rel, args, args.max_evals)
                    names = ("breadth_first", "sequential")
                agree = int(abs(ra.estimate - rb.estimate) <= ra.errorest + rb.errorest)
                os_.write(f"{names[0]},{a},{agree}\n{names[1]},{b},{agree}\n")
        return 0
    except Exception as e:  # noqa: BLE001 - mirrors the reference's catch-all (exit 1)
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
