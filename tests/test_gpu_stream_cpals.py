"""Out-of-memory streaming (proj/tests/test_streaming.cpp) and CP-ALS
(proj/src/cpals.cpp) on the device."""
import numpy as np
import pytest

from conftest import rel_frobenius

pytestmark = pytest.mark.gpu


def factor_bytes(f, out_rows):  # test_streaming.cpp:12-16
    return out_rows * f.rank * 8 + sum(a.size * 8 for a in f.factors)


def small_tensor(gpu, dims, nnz, seed, target, cap):
    coo = gpu.synth_uniform_host(dims, nnz, seed)
    return coo, gpu.build_blco(coo, target, cap)


def test_streamed_equals_in_memory(gpu):  # test_streaming.cpp:21-52
    coo, t = small_tensor(gpu, [50, 40, 60], 600, 83, 8, 64)
    assert t.keys.size >= 4
    f = gpu.FactorMatrices.random([50, 40, 60], 4, 1)
    want = gpu.mttkrp(t, f, 0, strategy=gpu.Strategy.Register)
    for queues in (1, 2, 4):
        b = gpu.DeviceBudget(num_queues=queues, reservation_bytes=t.max_nnz_per_block * 16)
        b.capacity_bytes = factor_bytes(f, 50) + queues * b.reservation_bytes
        rep = gpu.StreamReport()
        got = gpu.stream_mttkrp(t, f, 0, b, strategy=gpu.Strategy.Register, report=rep)
        assert rel_frobenius(got, want) <= 1e-12
        assert rep.blocks == t.keys.size and rep.peak_resident_bytes <= b.capacity_bytes
        assert rep.block_queue == [i % queues for i in range(t.keys.size)]
        assert rep.bytes_streamed == t.total_nnz * 16


def test_streamed_all_modes(gpu, oracle):
    """stream_mttkrp_all_modes: blocks cross the link once, every mode's M
    equals the oracle; the resident set counts all N outputs."""
    dims = [50, 40, 60]
    coo, t = small_tensor(gpu, dims, 600, 83, 8, 64)
    f = gpu.FactorMatrices.random(dims, 4, 1)
    want = [oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m) for m in range(3)]
    outs_bytes = sum(d * 4 * 8 for d in dims)
    for queues in (1, 3):
        for strat in (gpu.Strategy.Register, gpu.Strategy.Hierarchical):
            b = gpu.DeviceBudget(num_queues=queues, reservation_bytes=t.max_nnz_per_block * 16)
            b.capacity_bytes = sum(a.size * 8 for a in f.factors) + outs_bytes + queues * b.reservation_bytes
            rep = gpu.StreamReport()
            got = gpu.stream_mttkrp_all_modes(t, f, b, strategy=strat, report=rep)
            for m in range(3):
                assert rel_frobenius(got[m], want[m]) <= 1e-12, (queues, strat, m)
            assert rep.blocks == t.keys.size and rep.bytes_streamed == t.total_nnz * 16
            assert rep.peak_resident_bytes <= b.capacity_bytes
    b.capacity_bytes -= 8  # one output short of the resident set
    with pytest.raises(gpu.FormatError):
        gpu.stream_mttkrp_all_modes(t, f, b, strategy=gpu.Strategy.Register)


def test_streaming_matches_reference_stream(gpu, golden):
    z, meta = golden
    for j, ent in enumerate(meta["streams"]):
        bm = meta["builds"][ent["build"]]
        b = ent["build"]
        dims = bm["dims"]
        t = gpu.BlcoTensor(gpu.make_layout(dims, bm["target"]), bm["max_nnz"], z[f"b{b}_keys"],
                           z[f"b{b}_offsets"], z[f"b{b}_idx"], z[f"b{b}_vals"])
        f = gpu.FactorMatrices(ent["rank"], [z[f"s{j}_f{m}"] for m in range(len(dims))])
        res = bm["max_nnz"] * 16
        # resident set: factors + output x copies (streaming.cpp:117-124)
        budget = gpu.DeviceBudget(factor_bytes(f, dims[0]) + dims[0] * ent["rank"] * 8 + 2 * res, 2, res)
        for strat in (gpu.Strategy.Register, gpu.Strategy.Hierarchical):
            got = gpu.stream_mttkrp(t, f, 0, budget, gpu.ExecConfig(num_factor_copies=2), strat)
            assert rel_frobenius(got, z[f"s{j}_out"]) <= 1e-12


def test_overlap_with_injected_latency(gpu):  # test_streaming.cpp:105-139
    coo, t = small_tensor(gpu, [6, 4000], 3000, 101, 9, 512)
    f = gpu.FactorMatrices.random([6, 4000], 8, 2)
    b = gpu.DeviceBudget(num_queues=2, reservation_bytes=t.max_nnz_per_block * 16,
                         injected_transfer_latency_s=0.02)
    b.capacity_bytes = factor_bytes(f, 6) + 2 * b.reservation_bytes
    rep = gpu.StreamReport()
    gpu.stream_mttkrp(t, f, 0, b, report=rep)
    tr = [e for e in rep.timeline if e.kind == "transfer"]
    cp = [e for e in rep.timeline if e.kind == "compute"]
    assert any(x.begin_s < y.end_s and y.begin_s < x.end_s and x.block != y.block for x in tr for y in cp)
    assert rep.transfer_busy_seconds > 0 and rep.compute_busy_seconds > 0
    assert rep.overall_gbps < rep.compute_gbps  # transfer-dominated (test_streaming.cpp:164-170)


def test_source_refilling_one_pinned_buffer(gpu, oracle):
    """A BlockSource that refills ONE pinned buffer on every pull (the
    synth_alto_chunk pattern): the engine must finish each block's copy
    before pulling the next (a pinned cudaMemcpyAsync returns before its DMA
    reads host memory), with several queues in flight."""
    dims = [300, 200, 250]
    coo, t = small_tensor(gpu, dims, 60_000, 91, 64, 4096)
    assert t.keys.size >= 10
    f = gpu.FactorMatrices.random(dims, 32, 5)
    cap = t.max_nnz_per_block
    pidx = gpu.api.pinned_empty(cap, np.uint64)
    pvals = gpu.api.pinned_empty(cap, np.float64)

    def source():
        for b in range(t.keys.size):
            o0, o1 = int(t.offsets[b]), int(t.offsets[b + 1])
            n = o1 - o0
            pidx[:n] = t.idx[o0:o1]
            pvals[:n] = t.vals[o0:o1]
            yield (int(t.keys[b]), pidx[:n], pvals[:n])

    budget = gpu.DeviceBudget(capacity_bytes=1 << 30, num_queues=4, reservation_bytes=cap * 16)
    got = gpu.stream_mttkrp_all_modes(source(), f, budget, layout=t.layout, max_nnz_per_block=cap,
                                      block_count=int(t.keys.size))
    for m in range(3):
        want = oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m)
        assert rel_frobenius(got[m], want) <= 1e-12, m


def test_budget_errors(gpu):  # test_streaming.cpp:173-199
    coo, t = small_tensor(gpu, [30, 30], 100, 107, 6, 32)
    f = gpu.FactorMatrices.random([30, 30], 4, 1)
    with pytest.raises(gpu.FormatError, match="exceed device capacity"):
        gpu.stream_mttkrp(t, f, 0, gpu.DeviceBudget(capacity_bytes=64))
    b = gpu.DeviceBudget(num_queues=2, reservation_bytes=8)
    b.capacity_bytes = factor_bytes(f, 30) + 16
    with pytest.raises(gpu.FormatError, match="reservation"):
        gpu.stream_mttkrp(t, f, 0, b)


def test_oversized_budget(gpu):  # test_streaming.cpp:201-217
    coo, t = small_tensor(gpu, [25, 25, 25], 250, 109, 64, 1 << 27)
    f = gpu.FactorMatrices.random([25, 25, 25], 4, 3)
    want = gpu.mttkrp(t, f, 0)
    got = gpu.stream_mttkrp(t, f, 0, gpu.DeviceBudget(capacity_bytes=1 << 34, num_queues=4))
    assert rel_frobenius(got, want) <= 1e-12


def test_alto_chunk_generator_is_blco_order(gpu, oracle):
    """Config-5 generator: concatenated chunks are the BLCO element order of
    the tensor they describe (same bytes as building that COO), and streaming
    them equals the in-memory MTTKRP."""
    dims, nchunks, ncand = [300, 200, 250], 5, 4000
    idx = np.zeros(nchunks * ncand, np.uint64)
    vals = np.zeros(nchunks * ncand)
    off = 0
    for c in range(nchunks):
        off += gpu.api.synth_alto_chunk(dims, c, nchunks, ncand, 42, idx[off:], vals[off:])
    idx, vals = idx[:off], vals[:off]
    # valid fraction = prod(dims) / 2^total_bits = 15e6 / 2^25 = 0.447
    assert 0.40 * nchunks * ncand < off < 0.50 * nchunks * ncand
    layout = gpu.make_layout(dims, 64)
    coords = np.array([gpu.delinearize(layout, int(i), 0) for i in idx], np.uint64).T
    assert all((coords[m] < dims[m]).all() for m in range(3))
    t = gpu.build_blco(gpu.SparseTensorCoo(dims, coords, vals), 64, 3000)
    assert np.array_equal(t.idx, idx) and np.array_equal(t.vals, vals)
    f = gpu.FactorMatrices.random(dims, 32, 3)
    blocks = [(0, idx[o:o + 3000], vals[o:o + 3000]) for o in range(0, off, 3000)]
    budget = gpu.DeviceBudget(capacity_bytes=1 << 30, num_queues=3, reservation_bytes=3000 * 16)
    for mode in range(3):
        want = oracle.mttkrp_coo(dims, coords, vals, f.factors, mode)
        got = gpu.stream_mttkrp(iter(blocks), f, mode, budget, layout=layout, max_nnz_per_block=3000,
                                block_count=len(blocks))
        assert rel_frobenius(got, want) <= 1e-12
    # determinism
    idx2 = np.zeros(ncand, np.uint64)
    vals2 = np.zeros(ncand)
    n2 = gpu.api.synth_alto_chunk(dims, 0, nchunks, ncand, 42, idx2, vals2)
    assert np.array_equal(idx2[:n2], idx[:n2])


def test_cp_als_matches_reference(gpu, golden):
    """fit history within 1e-10 absolute, factors within 1e-8 relative."""
    z, meta = golden
    for j, ent in enumerate(meta["cpals"]):
        dims = ent["dims"]
        t = gpu.build_blco(gpu.SparseTensorCoo(dims, z[f"c{j}_in_idx"], z[f"c{j}_in_vals"]))
        model = gpu.cp_als(t, gpu.CpAlsOptions(rank=ent["rank"], max_iters=ent["iters"], tol=ent["tol"],
                                               seed=ent["seed"]))
        want = z[f"c{j}_fit"]
        assert len(model.fit_history) == want.size
        assert np.max(np.abs(np.array(model.fit_history) - want)) <= 1e-10
        for m in range(len(dims)):
            assert rel_frobenius(model.factors.factors[m], z[f"c{j}_f{m}"]) <= 1e-8
        assert np.allclose(model.lambda_, z[f"c{j}_lambda"], rtol=1e-9)
        assert abs(gpu.fit(t, model) - model.final_fit()) <= 1e-10


def test_cp_als_zero_iters_and_errors(gpu):
    coo, t = small_tensor(gpu, [5, 6, 7], 50, 1, 64, 1 << 27)
    m = gpu.cp_als(t, gpu.CpAlsOptions(rank=3, max_iters=0, seed=9))
    ref = gpu.FactorMatrices.random([5, 6, 7], 3, 9)
    assert all(np.array_equal(a, b) for a, b in zip(m.factors.factors, ref.factors))
    with pytest.raises(gpu.FormatError):
        gpu.cp_als(t, gpu.CpAlsOptions(rank=0))


def test_cp_als_deterministic_is_bit_reproducible(gpu, golden):
    """ExecConfig::deterministic: fixed-order MTTKRP (determ.cu) plus the
    epilogue's fixed-order reductions make two CP-ALS runs bit-identical,
    and they stay within the reference tolerance."""
    z, meta = golden
    ent = meta["cpals"][0]
    dims = ent["dims"]
    t = gpu.build_blco(gpu.SparseTensorCoo(dims, z["c0_in_idx"], z["c0_in_vals"]))
    opts = gpu.CpAlsOptions(rank=ent["rank"], max_iters=ent["iters"], tol=ent["tol"], seed=ent["seed"])
    det = gpu.ExecConfig(deterministic=True)
    a = gpu.cp_als(t, opts, det)
    b = gpu.cp_als(t, opts, det)
    assert a.fit_history == b.fit_history
    for m in range(len(dims)):
        assert np.array_equal(a.factors.factors[m], b.factors.factors[m])
    assert np.max(np.abs(np.array(a.fit_history) - z["c0_fit"])) <= 1e-10


@pytest.mark.parametrize("dims,rank", [([30, 40, 50], 1), ([30, 40, 50], 7), ([45, 35, 55], 24),
                                       ([50, 60, 70, 40], 33), ([40, 50, 60, 30, 20], 17), ([80, 90, 70], 64),
                                       ([60, 50, 40], 16), ([40, 50], 5), ([9, 8, 7, 6, 5, 6, 7, 8], 3)])
def test_cp_als_random_shapes_match_oracle(gpu, oracle, dims, rank):
    """Device CP-ALS (the normalisation folded into the solves, every solve
    path: constant-bank L for R = 16, shared-memory L for the other ranks)
    against the C restatement of the reference's cp_als (oracle/blco_oracle.c,
    cpals.cpp:66-111) on random shapes, orders 2 to 8: fit history within
    1e-10, factors within 1e-8, lambda within 1e-9 relative."""
    nnz = min(4000, int(np.prod(dims)) // 2)
    idx, vals = oracle.synth_uniform(dims, nnz, 3 + rank)
    keys, offs, oi, ov = oracle.build(dims, idx, vals)
    fs, lam, fit = oracle.cp_als(dims, keys, offs, oi, ov, rank, 6, -1e300, 11)
    t = gpu.build_blco(gpu.SparseTensorCoo(dims, idx, vals))
    model = gpu.cp_als(t, gpu.CpAlsOptions(rank=rank, max_iters=6, tol=-1e300, seed=11))
    assert len(model.fit_history) == fit.size == 6
    assert np.max(np.abs(np.array(model.fit_history) - fit)) <= 1e-10
    for m in range(len(dims)):
        assert rel_frobenius(model.factors.factors[m], fs[m]) <= 1e-8, m
    assert np.allclose(model.lambda_, lam, rtol=1e-9)
