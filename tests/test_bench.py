"""bench.py's contract plumbing on the CPU (no GPU needed): the rank-count
check behind --gpus, the host-CPU description of the baseline protocol, and
that both arms print the same workload config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode == 2
    assert "WORLD_SIZE=1" in json.loads(p.stdout.strip().splitlines()[-1])["error"]


def test_gpus_without_enough_devices_fails_loudly():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "8"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 2
    assert "GPU(s) visible" in json.loads(p.stdout.strip().splitlines()[-1])["error"]


def test_host_cpu_description():
    cpu = bench.host_cpu()
    assert cpu["physical"] >= 1 and cpu["logical"] >= cpu["physical"] // 2
    assert cpu["usable"] >= 1
    desc = bench.cpu_desc(cpu, cpu["usable"])
    assert "physical cores" in desc and "OpenMP threads" in desc


def test_both_arms_share_the_config():
    class A:
        max_regions = 1 << 22
        mode = "parity"
    cfg = bench.bench_config(A)
    assert cfg == bench.bench_config(A)
    assert "genz_8d_suite" in cfg["workload"]
    # the CPU sample is a subset of the suite's own cases
    assert set(bench.CPU_SAMPLE) <= set(bench.workload(None))
    assert set(bench.CPU_SAMPLE_1T) <= set(bench.CPU_SAMPLE)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libbfcub_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_sample_runs_suite_calls_to_their_end():
    ref, make_config = bench.load_reference()
    e, s = bench.ref_sample(ref, make_config, os.cpu_count(), ((3, 1e-3),))
    # f3 8D tau=1e-3 (tests/golden/finals_deep.json): 40979 regions evaluated
    assert e == 40979 and s > 0
    # the sample's size as described (finals_deep.json region counts)
    from conftest import load_golden
    fin = load_golden("finals_deep.json")
    tot = sum(fin[f"f{f}_8d_{t:g}"]["regions_generated"] for f, t in bench.CPU_SAMPLE)
    assert f"{tot / 1e6:.1f}M region-evals" in bench.CPU_SAMPLE_DESC
