"""bench.py --impl reference (CPU only, the unmodified reference from
oracle/_ref): one JSON line with the contract's keys, for the default
config family and for the generator-prefix sampler used by the large
configs (checked here at small sizes through reference_sample_run)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref" / "libblco_ref.so"


@pytest.mark.skipif(not REF.exists(), reason="oracle/_ref/libblco_ref.so not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "cfg1",
                        "--steps", "1", "--warmup", "1", "--ref-step-s", "0.2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "fitted as a + b*nnz" in d["cpu_baseline"]["sample"]


@pytest.mark.skipif(not REF.exists(), reason="oracle/_ref/libblco_ref.so not built")
@pytest.mark.parametrize("sampler,skew,op", [("generator_prefix", None, "mttkrp"), ("generator_prefix", 2, "mttkrp"),
                                             ("generator_prefix", None, "stream"), ("alto_prefix", None, "mttkrp")])
def test_reference_sampler_extrapolates(sampler, skew, op):
    sys.path.insert(0, str(ROOT))
    import bench

    gbps, info = bench.reference_sample_run([300, 200, 100], 400_000, 8, steps=1, warmup=0, target_step_s=0.05,
                                            sampler=sampler, skew=skew, op=op)
    assert gbps > 0 and info["full_step_s"] > 0 and info["per_elem_s"] > 0
    assert info["sample_nnz"] <= 400_000 and info["full_step_s"] >= info["fixed_s"]
