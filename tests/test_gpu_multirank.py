"""The N > 1 code paths of bench.py (span partition + per-rank kernels +
overlapped all-reduce of M; multi-rank e2e; multi-rank all-mode streaming)
run under torchrun with two ranks.  The box has one GPU, so both ranks share
cuda:0 and reduce over gloo (BLCO_B200_ONE_DEVICE, BLCO_B200_DIST_BACKEND):
the plumbing is the one NCCL runs on an 8-GPU node; the timings are
meaningless and not asserted.  --check compares the ranks' summed M_n with a
single-device MTTKRP of the whole tensor (relative Frobenius <= 1e-12)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, timeout=600, world=2):
    env = dict(os.environ, BLCO_B200_ONE_DEVICE="1", BLCO_B200_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", str(world),
           *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("world,combine", [(2, "reducescatter"), (3, "allreduce")])
def test_multi_rank_all_mode_step(gpu, world, combine):
    """G ranks vs G = 1 (SURVEY.md 4 "multi-node without a cluster"), the
    device step and the e2e step, with either combine of the partials."""
    d = _torchrun(["--config", "cfg1", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--check",
                   "--reduce", combine], world=world)
    assert d["n_gpus"] == world and d["value"] > 0
    assert max(d["check"]["rel_frobenius_vs_single_device"]) <= 1e-12
    word = "reduce-scatter" if combine == "reducescatter" else "all-reduce"
    assert d["e2e"]["value"] > 0 and word in d["e2e"]["path"] and word in d["config"]["parallelism"]


def test_two_rank_reference_arm_prints_once(gpu):
    d = _torchrun(["--config", "cfg1", "--impl", "reference", "--steps", "1", "--warmup", "1",
                   "--ref-step-s", "0.2"])
    assert d["impl"] == "reference"


def test_two_rank_all_mode_streaming(gpu):
    """Two ranks stream disjoint ALTO chunk ranges (streaming.cpp:103-309 per
    rank) and all-reduce M_n; --check compares the summed M_n with one device
    streaming the whole tensor (relative Frobenius <= 1e-12)."""
    d = _torchrun(["--config", "reddit_stream_tiny", "--steps", "1", "--check", "--no-cpu-baseline"])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["nnz"] > 19_000_000 and "all-reduce" in d["config"]["step"]
    assert d["check"]["nnz_single_device"] == d["config"]["nnz"]
    assert max(d["check"]["rel_frobenius_vs_single_device"]) <= 1e-12


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_reduce_scatter_step(gpu, world):
    """The default N > 1 combine: reduce-scatter of M_n into row shards
    (SURVEY.md 8e); --check all-gathers the shards and compares them with a
    single-device MTTKRP of the whole tensor."""
    d = _torchrun(["--config", "cfg1", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--check",
                   "--reduce", "reducescatter"], world=world)
    assert "reduce-scatter" in d["config"]["parallelism"]
    assert max(d["check"]["rel_frobenius_vs_single_device"]) <= 1e-12


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_cp_als(gpu, world):
    """cp_als_distributed (reduce-scatter of M_n, row-block solve, all-reduced
    Gram, all-gathered A_n) against single-device cp_als on the whole tensor:
    the fit history within 1e-10 and the factors within 1e-8."""
    d = _torchrun(["--config", "als_tiny", "--check"], world=world)
    c = d["check"]
    assert d["n_gpus"] == world and len(d["fit_history"]) == 10
    assert c["max_abs_fit_diff_vs_single_device"] <= 1e-10
    assert max(c["factor_rel_frobenius"]) <= 1e-8 and c["lambda_rel"] <= 1e-8
