import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from pyoracle import REF_SO, RefLib
    if not REF_SO.exists():
        pytest.skip("oracle/_ref/libblco_ref.so not built")
    return RefLib()


@pytest.fixture(scope="session")
def blco():
    import paper_2201_12523_b200 as b
    return b


@pytest.fixture(scope="session")
def gpu(blco):
    if blco.device_count() < 1:
        pytest.fail("no CUDA device visible: -m gpu tests need a B200")
    return blco


def rel_frobenius(a, b):
    """proj/tests/test_util.hpp:82-90."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    diff = float(np.sum((a - b) ** 2))
    ref = float(np.sum(b * b))
    return (diff / ref) ** 0.5 if ref > 0 else diff ** 0.5
