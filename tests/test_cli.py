"""CLI front-end (bfcub_cli.cpp) -- exit codes, CSV schema; the GPU test
checks a row against the reference's own result."""
import subprocess
import sys

import pytest

from conftest import ROOT
from paper_2104_06494_b200 import cli

HEADER = ("integrand_id,dim,tau_rel,estimate,errorest,reference_value,true_rel_err,"
          "claimed_rel_err,status,iterations,regions_generated,eval_count,wall_ms")


def run(*args):
    return subprocess.run([sys.executable, "-m", "paper_2104_06494_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True)


def test_header_matches_reference_schema():
    assert cli.CSV_HEADER == HEADER  # bfcub_cli.cpp:24-26
    assert cli.fmt(0.1) == "0.10000000000000001" and cli.fmt(1e-3) == "0.001"


def test_usage_errors_exit_2():
    assert run().returncode == 2
    assert run("integrate", "f9", "3", "1e-3").returncode == 2
    assert run("integrate", "f4", "17", "1e-3").returncode == 2
    assert run("bench", "--subset", "f4").returncode == 2
    assert run("bench", "--subset", "f8:5").returncode == 2  # no f8 reference at 5D


def test_plot_renders_both_svgs(tmp_path):
    """plot (bfcub_cli.cpp:189-333): accuracy.svg and regions.svg from a bench
    CSV; converged runs are dots, the others crosses; one legend row per series."""
    csv = tmp_path / "bench.csv"
    csv.write_text(HEADER + "\n"
                   "f4,5,0.001,1.79e-06,1.3e-09,1.79e-06,7.6e-06,7.4e-04,converged,11,7959712,"
                   "740253216,3.4\n"
                   "f4,5,0.0002,1.79e-06,2e-10,1.79e-06,1e-07,1e-04,converged,14,9000000,"
                   "840253216,5.1\n"
                   "f1,8,0.001,3.4e-05,4e-05,3.4e-05,0.2,1.2,max_iterations,100,176649775,"
                   "70836559775,99\n")
    p = run("plot", str(csv), "--out-dir", str(tmp_path))
    assert p.returncode == 0, p.stderr
    for name in ("accuracy.svg", "regions.svg"):
        svg = (tmp_path / name).read_text()
        assert svg.startswith("<svg xmlns='http://www.w3.org/2000/svg' width='760' height='520'>")
        assert svg.count("<circle") == 2 + 2 and svg.count("<path") == 1
        assert ">f1:8</text>" in svg and ">f4:5</text>" in svg
    assert "stroke-dasharray" in (tmp_path / "accuracy.svg").read_text()  # the tau line
    assert run("plot", str(tmp_path / "missing.csv")).returncode == 2
    bad = tmp_path / "bad.csv"
    bad.write_text("x,y\n")
    assert run("plot", str(bad)).returncode == 2


def test_reference_values_are_the_references_long_double(ref):
    """The CSV's reference_value column: integrands.cpp:83-188 in long double,
    to the last bit, for every suite id and dimension."""
    for i in ("f1", "f2", "f3", "f4", "f5", "f6", "f7"):
        for d in range(1, 17):
            assert cli.fmt(cli.reference_value(i, d)) == cli.fmt(ref.reference_value(i, d))
    for d in (2, 3, 8):
        assert cli.reference_value("f8", d) == ref.reference_value("f8", d)


def test_headline_specs():
    assert cli.headline() == [("f1", 8), ("f3", 8), ("f4", 8), ("f5", 8), ("f7", 8), ("f8", 8),
                              ("f4", 5), ("f6", 6), ("f3", 3)]


@pytest.mark.gpu
def test_integrate_row_matches_reference(tmp_path, ref):
    from ref_ctypes import make_config
    p = run("integrate", "f4", "5", "1e-3")
    assert p.returncode == 0, p.stderr
    lines = p.stdout.strip().splitlines()
    assert lines[0] == HEADER
    row = lines[1].split(",")
    want = ref.integrate(4, 5, make_config(tau_rel=1e-3))
    assert float(row[3]) == want.estimate and float(row[4]) == want.errorest
    assert row[8] == want.status and int(row[9]) == want.iterations
    assert int(row[10]) == want.regions_generated and int(row[11]) == want.eval_count
    out = tmp_path / "b.csv"
    p = run("bench", "--subset", "f4:3,f3:3", "--k-max", "2", "--out", str(out))
    assert p.returncode == 0, p.stderr
    rows = out.read_text().strip().splitlines()
    assert rows[0] == HEADER and len(rows) == 1 + 2 * 3
    # every column but wall_ms is the reference's own row (bfcub_cli.cpp:51-61,69-101)
    rv = ref.reference_value("f4", 5)
    want_row = ["f4", "5", cli.fmt(1e-3), cli.fmt(want.estimate), cli.fmt(want.errorest),
                cli.fmt(rv), cli.fmt(abs(want.estimate - rv) / abs(rv)),
                cli.fmt(want.errorest / abs(want.estimate)), want.status, str(want.iterations),
                str(want.regions_generated), str(want.eval_count)]
    assert row[:12] == want_row
    out = tmp_path / "c.csv"
    p = run("compare", "--subset", "f4:3,f3:4", "--out", str(out))
    assert p.returncode == 0, p.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "engine," + HEADER + ",agreement"
    assert [ln.split(",")[0] for ln in lines[1:]] == ["breadth_first", "sequential"] * 2
    seq = lines[2].split(",")
    ws = ref.integrate_sequential(4, 3, 1e-3)
    assert (float(seq[4]), float(seq[5]), seq[9], int(seq[10])) == (
        ws.estimate, ws.errorest, ws.status, ws.iterations)


def test_f8_extended_reference_values():
    """f8 beyond the reference's n in {2, 3, 8} (the reference's generator tool,
    csrc/suite.cpp kF8): opt-in, and consistent with the exact moment ordering
    E[S^7.5] between E[S^7] and E[S^8] (S = sum x_i^2)."""
    import pytest as _pt
    with _pt.raises(ValueError):
        cli.reference_value("f8", 5)
    assert cli.reference_value("f8", 1, extended=True) == 1.0 / 16.0
    for n in (1, 2, 3, 4, 5, 6, 7, 8, 9, 10):
        v = cli.reference_value("f8", n, extended=True)
        # Jensen / Lyapunov: E[S^7]^(15/14) <= E[S^7.5] <= E[S^8]^(15/16)
        lo = _moment(n, 7) ** (15 / 14)
        hi = _moment(n, 8) ** (15 / 16)
        assert lo <= v <= hi, (n, lo, v, hi)


def _moment(d, k):  # E[(sum x_i^2)^k] on the unit cube, exact recursion
    from math import comb
    g = [1.0 / (2 * j + 1) for j in range(k + 1)]
    for _ in range(2, d + 1):
        g = [sum(comb(kk, j) / (2 * j + 1) * g[kk - j] for j in range(kk + 1))
             for kk in range(k + 1)]
    return g[k]
