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
    out = tmp_path / "c.csv"
    p = run("compare", "--subset", "f4:5", "--out", str(out))
    assert p.returncode == 0 and out.read_text().splitlines()[0] == "engine," + HEADER + ",agreement"
