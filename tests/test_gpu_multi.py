"""The library's own multi-GPU partition (multi.cu): span
ranges over G devices, replicated factors, per-mode NCCL all-reduce or
reduce-scatter of the partial M_n, driven inside libblco_b200.so.

The GPU boxes here have one B200, so G = 1 runs everywhere (the reduction is
the identity, no NCCL communicator) and the G >= 2 cases skip below two
devices.  Tolerance: relative Frobenius <= 1e-12 against the single-device
MTTKRP (the reference's fp64 bar, proj/tests/test_mttkrp.cpp:267-290)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_frobenius

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
DIMS, NNZ, RANK = [3000, 2500, 4000], 300_000, 16


@pytest.fixture(scope="module")
def case(gpu):
    dt = gpu.DeviceTensor.synthetic(DIMS, NNZ, 42, 64, 20_000)  # several blocks
    f = gpu.FactorMatrices.random(DIMS, RANK, 7)
    want = [gpu.mttkrp(dt, f, m) for m in range(3)]
    return dt, f, want


def _devices(gpu, g):
    if gpu.device_count() < g:
        pytest.skip(f"needs {g} GPUs")
    return list(range(g))


@pytest.mark.parametrize("reduce", ["allreduce", "reducescatter"])
@pytest.mark.parametrize("g", [1, 2, 4, 8])
def test_multi_device_all_modes(gpu, case, g, reduce):
    dt, f, want = case
    mt = gpu.MultiDeviceTensor(dt, _devices(gpu, g))
    ranges = mt.ranges()
    assert ranges[0][0] == 0 and ranges[-1][1] == NNZ
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    rep = gpu.MultiReport()
    got = mt.mttkrp_all_modes(f, reduce=reduce, report=rep)
    for m in range(3):
        assert rel_frobenius(got[m], want[m]) <= 1e-12, (g, reduce, m)
    assert rep.devices == g and rep.device_ms > 0
    assert rep.h2d_bytes == g * sum(d * RANK * 8 for d in DIMS)
    assert rep.d2h_bytes == sum(d * RANK * 8 for d in DIMS)


@pytest.mark.parametrize("reduce", ["allreduce", "reducescatter"])
def test_single_rank_communicator(gpu, case, reduce):
    """blco_dist_mttkrp_all on a one-rank communicator: the per-rank step of
    the multi-process path, enqueued on a caller stream."""
    import torch
    dt, f, want = case
    comm = gpu.Communicator(None, 1, 0, 0)
    fac = [torch.from_numpy(a).cuda() for a in f.factors]
    outs = [torch.full((d, RANK), 7.0, dtype=torch.float64, device="cuda") for d in DIMS]  # zeroed by the call
    shards = [torch.empty((d, RANK), dtype=torch.float64, device="cuda") for d in DIMS]
    s = torch.cuda.Stream()
    comm.mttkrp_all(dt, [a.data_ptr() for a in fac], RANK, [o.data_ptr() for o in outs],
                    [x.data_ptr() for x in shards], reduce=reduce, stream=s.cuda_stream)
    s.synchronize()
    res = shards if reduce == "reducescatter" else outs
    for m in range(3):
        assert rel_frobenius(res[m].cpu().numpy(), want[m]) <= 1e-12


def test_dist_rejects_bad_arguments(gpu, case):
    dt, f, _ = case
    comm = gpu.Communicator(None, 1, 0, 0)
    with pytest.raises(gpu.FormatError, match="shard"):
        comm.mttkrp_all(dt, [1, 1, 1], RANK, [1, 1, 1], None, reduce="reducescatter")
    with pytest.raises(gpu.FormatError, match="null factor"):
        comm.mttkrp_all(dt, [0, 0, 0], RANK, [1, 1, 1])
    with pytest.raises(gpu.FormatError, match="deterministic"):
        comm.mttkrp_all(dt, [1, 1, 1], RANK, [1, 1, 1], config=gpu.ExecConfig(deterministic=True))


def test_library_reuses_the_process_nccl(gpu):
    """In a torch process the library binds the NCCL torch already loaded
    (no second libnccl.so.2 in the process)."""
    code = ("import torch, torch.distributed, sys; sys.path.insert(0, %r); v = torch.cuda.nccl.version(); "
            "import paper_2201_12523_b200 as b; "
            "want = v[0] * 10000 + v[1] * 100 + v[2] if isinstance(v, tuple) else v; "
            "got = b.nccl_version(); print(got, want); assert got == want, (got, want)") % str(ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ))
    assert r.returncode == 0, r.stderr[-2000:] + r.stdout


@pytest.mark.parametrize("reduce", ["allreduce", "reducescatter"])
def test_nccl_collectives_on_one_rank(gpu, case, monkeypatch, reduce):
    """BLCO_B200_NCCL_SINGLE=1: the one-rank communicator and the one-device
    driver create real NCCL communicators (ncclGetUniqueId +
    ncclCommInitRank, ncclCommInitAll), so each mode's ncclReduceScatter /
    ncclAllReduce is enqueued on the collective stream behind the mode
    kernel's event -- the multi-GPU code path run over NCCL on a one-GPU box
    (a reduction over one rank is a copy)."""
    import torch
    monkeypatch.setenv("BLCO_B200_NCCL_SINGLE", "1")
    dt, f, want = case
    comm = gpu.Communicator(None, 1, 0, 0)
    fac = [torch.from_numpy(a).cuda() for a in f.factors]
    outs = [torch.full((d, RANK), 7.0, dtype=torch.float64, device="cuda") for d in DIMS]
    shards = [torch.full((d, RANK), -1.0, dtype=torch.float64, device="cuda") for d in DIMS]
    s = torch.cuda.Stream()
    for _ in range(2):  # the communicator is reused across steps
        comm.mttkrp_all(dt, [a.data_ptr() for a in fac], RANK, [o.data_ptr() for o in outs],
                        [x.data_ptr() for x in shards], reduce=reduce, stream=s.cuda_stream)
        s.synchronize()
        res = shards if reduce == "reducescatter" else outs
        for m in range(3):
            assert rel_frobenius(res[m].cpu().numpy(), want[m]) <= 1e-12, (reduce, m)
    mt = gpu.MultiDeviceTensor(dt, [0])
    got = mt.mttkrp_all_modes(f, reduce=reduce)
    for m in range(3):
        assert rel_frobenius(got[m], want[m]) <= 1e-12, (reduce, m)
