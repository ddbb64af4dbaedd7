"""The reference's bucket-P cases restated in C++ against the drop-in headers
(tests/cpp/test_api.cpp), linked to libblco_b200.so and run on the GPU."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
EXE = Path(__file__).resolve().parent / "cpp" / "test_api"


def test_cpp_dropin_suite(gpu):
    if not EXE.exists():
        subprocess.run(["make", "-C", str(EXE.parent)], check=True)
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failures" in r.stdout
