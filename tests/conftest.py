"""Shared fixtures.

* `ref`  - the UNMODIFIED reference library (oracle/_ref/libbfcub_ref.so),
           the parity oracle.  Built here by `make -C oracle ref`; the .so
           travels to the GPU box with the snapshot.
* `port` - the plain-C restatement (oracle/liboracle.so).
* `pg`   - the product package (libpagani_b200.so through its C ABI).
GPU tests are marked `@pytest.mark.gpu`; everything else runs on a CPU-only
host.  Golden fixtures live in tests/golden/ (made by make_golden.py).
"""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200)")


@pytest.fixture(scope="session")
def ref():
    from ref_ctypes import Ref, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    return Ref()


@pytest.fixture(scope="session")
def port():
    from ref_ctypes import Port, available
    if not available("port"):
        pytest.skip("oracle/liboracle.so not built (make -C oracle)")
    return Port()


@pytest.fixture(scope="session")
def pg():
    import paper_2104_06494_b200 as pg
    pg.api._lib()  # loads libpagani_b200.so or raises (no fallback)
    return pg


@pytest.fixture(scope="session")
def gpu(pg):
    if pg.device_count() < 1:
        pytest.fail("GPU test on a host without a CUDA device")
    return 0


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing (python tests/golden/make_golden.py)")
    return json.load(open(path))


def unhex(v):
    return float.fromhex(v) if isinstance(v, str) else v


def bits(a):
    import numpy as np
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)
