"""Randomised cross-path parity on the device: many small tensors of random
order, shape, density, rank and block capacity, every MTTKRP path (register,
hierarchical, deterministic, fp32, the all-mode host pipeline, all-mode
streaming) against the oracle.  Targets the edge cases of the kernels' lane
group split, tail batches and packed staging (ranges shorter than a batch,
single-element blocks, order 1, unit-length modes, ranks around the lane
widths)."""
import numpy as np
import pytest

from conftest import rel_frobenius

pytestmark = pytest.mark.gpu

CASES = 150


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    order = int(rng.integers(1, 9))
    hi = {1: 5000, 2: 400, 3: 90}.get(order, 16)
    dims = [int(x) for x in rng.integers(1, hi, size=order)]
    cells = int(np.prod(dims))
    nnz = int(min(cells, rng.integers(1, 6000)))
    rank = int(rng.choice([1, 2, 3, 8, 15, 16, 17, 31, 32, 33, 64, 65]))
    total_bits = sum(int(d - 1).bit_length() for d in dims)
    target = int(rng.integers(max(1, total_bits - 6), 65)) if total_bits > 1 else 64
    cap = int(rng.choice([1, 7, 64, 1000, 1 << 27]))
    return dims, nnz, rank, target, cap


@pytest.mark.parametrize("seed", range(CASES))
def test_random_paths_match_oracle(gpu, oracle, seed):
    dims, nnz, rank, target, cap = _case(seed)
    coo = gpu.synth_uniform_host(dims, nnz, seed)
    f = gpu.FactorMatrices.random(dims, rank, seed + 1)
    t = gpu.build_blco(coo, target, cap)
    want = [oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m) for m in range(len(dims))]
    ctx = (dims, nnz, rank, target, cap)
    for m in range(len(dims)):
        for strat in (gpu.Strategy.Register, gpu.Strategy.Hierarchical):
            assert rel_frobenius(gpu.mttkrp(t, f, m, strategy=strat), want[m]) <= 1e-12, (ctx, m, strat)
        assert rel_frobenius(gpu.mttkrp(t, f, m, gpu.ExecConfig(deterministic=True)), want[m]) <= 1e-12, (ctx, m)
        assert rel_frobenius(gpu.mttkrp_f32(t, f, m), want[m]) <= 1e-5, (ctx, m, "fp32")
    got = gpu.mttkrp_all_modes(t, f, chunk_elems=int(np.random.default_rng(seed).integers(1, 3000)))
    for m in range(len(dims)):
        assert rel_frobenius(got[m], want[m]) <= 1e-12, (ctx, m, "all-modes")
    res = min(cap, nnz) * 16
    b = gpu.DeviceBudget(capacity_bytes=1 << 28, num_queues=2, reservation_bytes=max(res, 16))
    got = gpu.stream_mttkrp_all_modes(t, f, b)
    for m in range(len(dims)):
        assert rel_frobenius(got[m], want[m]) <= 1e-12, (ctx, m, "stream")


@pytest.mark.parametrize("seed", range(60))
def test_random_builds_bit_exact(gpu, oracle, seed):
    """Device build_blco against the C restatement of build_blco on random
    shapes, including layouts wider than 64 bits (two-word sort, multi-key
    blocking) and tiny block capacities: keys, offsets, indices, values and
    the batch table bit-exact."""
    rng = np.random.default_rng(7000 + seed)
    order = int(rng.integers(1, 7))
    wide = seed % 3 == 0
    hi = (1 << 20) if wide else 3000
    dims = [int(x) for x in rng.integers(1, hi, size=order)]
    nnz = int(rng.integers(1, 20_000))
    if np.prod(np.array(dims, dtype=object)) < 2 ** 64:
        nnz = int(min(nnz, int(np.prod(np.array(dims, dtype=object)))))
        coo = gpu.synth_uniform_host(dims, nnz, seed)
    else:  # cell space beyond 2^64: the first nnz distinct uniform draws
        idx0, vals0 = oracle.synth_draws(dims, nnz, seed, 1)
        coo = gpu.SparseTensorCoo(dims, idx0, vals0)
    total_bits = sum(int(d - 1).bit_length() for d in dims)
    lo = max(1, total_bits - 64, min(64, total_bits - 12))  # stripped bits <= 64 (device limit)
    if lo > 64 or total_bits > 128:
        pytest.skip("layout beyond the device's 64-bit block key")
    target = int(rng.integers(lo, 65))
    cap = int(rng.choice([1, 5, 100, 1 << 27]))
    t = gpu.build_blco(coo, target, cap)
    keys, offs, idx, vals = oracle.build(dims, coo.indices, coo.values, target, cap)
    assert np.array_equal(t.keys, keys) and np.array_equal(t.offsets, offs)
    assert np.array_equal(t.idx, idx) and np.array_equal(t.vals, vals)
    assert np.array_equal(t.batch_table, oracle.batch_table(np.diff(offs), 512))


@pytest.mark.parametrize("seed", range(24))
def test_random_multi_and_stream_paths(gpu, oracle, monkeypatch, seed):
    """The remaining entry points on random shapes: the per-mode streaming
    API (stream_mttkrp, 1-3 queues), the library multi-GPU driver at one
    device and the one-rank communicator with real NCCL communicators
    (BLCO_B200_NCCL_SINGLE=1, both reductions), against the oracle."""
    import torch
    monkeypatch.setenv("BLCO_B200_NCCL_SINGLE", "1")
    dims, nnz, rank, target, cap = _case(500 + seed)
    coo = gpu.synth_uniform_host(dims, nnz, seed)
    f = gpu.FactorMatrices.random(dims, rank, seed + 7)
    t = gpu.build_blco(coo, target, cap)
    want = [oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m) for m in range(len(dims))]
    ctx = (dims, nnz, rank, target, cap)
    queues = 1 + seed % 3
    res = min(cap, nnz) * 16
    for m in range(len(dims)):
        b = gpu.DeviceBudget(capacity_bytes=1 << 28, num_queues=queues, reservation_bytes=max(res, 16))
        assert rel_frobenius(gpu.stream_mttkrp(t, f, m, b), want[m]) <= 1e-12, (ctx, m, "stream per mode")
    reduce = "reducescatter" if seed % 2 else "allreduce"
    dt = gpu.DeviceTensor.upload(t)
    got = gpu.MultiDeviceTensor(dt, [0]).mttkrp_all_modes(f, reduce=reduce)
    for m in range(len(dims)):
        assert rel_frobenius(got[m], want[m]) <= 1e-12, (ctx, m, "multi")
    comm = gpu.Communicator(None, 1, 0, 0)
    fac = [torch.from_numpy(a).cuda() for a in f.factors]
    outs = [torch.empty((d, rank), dtype=torch.float64, device="cuda") for d in dims]
    shards = [torch.empty((d, rank), dtype=torch.float64, device="cuda") for d in dims]
    comm.mttkrp_all(dt, [a.data_ptr() for a in fac], rank, [o.data_ptr() for o in outs],
                    [x.data_ptr() for x in shards], reduce=reduce)
    torch.cuda.synchronize()
    res_t = shards if reduce == "reducescatter" else outs
    for m in range(len(dims)):
        assert rel_frobenius(res_t[m].cpu().numpy(), want[m]) <= 1e-12, (ctx, m, "communicator")
