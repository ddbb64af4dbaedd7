"""MTTKRP on the device vs the oracle (relative Frobenius <= 1e-12 in fp64,
the reference's own bar, proj/tests/test_mttkrp.cpp:267-290)."""
import numpy as np
import pytest

from conftest import rel_frobenius

pytestmark = pytest.mark.gpu

GI = np.array([[0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 3, 3],
               [0, 0, 2, 0, 0, 0, 3, 1, 1, 2, 2, 3],
               [0, 1, 2, 1, 2, 1, 3, 0, 1, 2, 3, 3]], np.uint64)
GV = np.arange(1, 13, dtype=np.float64)
TOL = 1e-12


def test_all_ones_rows(gpu):  # test_mttkrp.cpp:33-47
    t = gpu.build_blco(gpu.SparseTensorCoo([4, 4, 4], GI, GV), 5, 6)
    f = gpu.FactorMatrices.ones([4, 4, 4], 2)
    m1 = gpu.mttkrp(t, f, 0, strategy=gpu.Strategy.Register)
    assert np.allclose(m1[:, 0], [6, 9, 13, 50], rtol=1e-13) and np.allclose(m1[:, 1], [6, 9, 13, 50])
    m3 = gpu.mttkrp(t, f, 2, strategy=gpu.Strategy.Hierarchical)
    assert np.allclose(m3[:, 0], [9, 21, 18, 30], rtol=1e-13)


def test_golden_grid_both_strategies(gpu, golden):
    """Every golden build x rank x mode x strategy x factor copies."""
    z, meta = golden
    for j, ent in enumerate(meta["mttkrps"]):
        b = ent["build"]
        bm = meta["builds"][b]
        dims = bm["dims"]
        t = gpu.BlcoTensor(gpu.make_layout(dims, bm["target"]), bm["max_nnz"], z[f"b{b}_keys"],
                           z[f"b{b}_offsets"], z[f"b{b}_idx"], z[f"b{b}_vals"])
        f = gpu.FactorMatrices(ent["rank"], [z[f"m{j}_f{m}"] for m in range(len(dims))])
        for mode in range(len(dims)):
            want = z[f"m{j}_coo{mode}"]
            for strat in (gpu.Strategy.Register, gpu.Strategy.Hierarchical):
                for copies in (1, 3):
                    cfg = gpu.ExecConfig(num_factor_copies=copies, stash_slots=4)
                    got = gpu.mttkrp(t, f, mode, cfg, strat)
                    assert rel_frobenius(got, want) <= TOL, (j, mode, strat, copies)


@pytest.mark.parametrize("order", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("rank", [1, 3, 8, 16, 32, 33, 64, 100])
def test_orders_and_ranks(gpu, oracle, order, rank):
    rng = np.random.default_rng(order * 131 + rank)
    dims = [int(x) for x in rng.integers(2, 60, size=order)]
    cells = int(np.prod(dims))
    nnz = min(cells, 3000)
    coo = gpu.synth_uniform_host(dims, nnz, order + rank)
    f = gpu.FactorMatrices(rank, [rng.uniform(-1, 1, (d, rank)) for d in dims])
    t = gpu.build_blco(coo, 64)
    for mode in range(order):
        want = oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, mode)
        for strat in (gpu.Strategy.Register, gpu.Strategy.Hierarchical):
            got = gpu.mttkrp(t, f, mode, strategy=strat)
            assert rel_frobenius(got, want) <= TOL, (mode, strat)


@pytest.mark.parametrize("target,cap", [(64, 1 << 27), (12, 64), (9, 1000), (20, 1)])
def test_multiblock_layouts(gpu, oracle, target, cap):
    dims = [700, 90, 1300]
    coo = gpu.synth_uniform_host(dims, 40_000, 17)
    f = gpu.FactorMatrices.random(dims, 16, 7)
    t = gpu.build_blco(coo, target, cap)
    for mode in range(3):
        want = oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, mode)
        for strat in (gpu.Strategy.Register, gpu.Strategy.Hierarchical):
            assert rel_frobenius(gpu.mttkrp(t, f, mode, strategy=strat), want) <= TOL


def test_config1_full_size(gpu, oracle):
    """BASELINE config 1: 1000^3, 1M nnz, R=16, every mode, against the oracle."""
    dims = [1000, 1000, 1000]
    dt = gpu.DeviceTensor.synthetic(dims, 1_000_000, 42)
    idx, vals = oracle.synth_uniform(dims, 1_000_000, 42)
    f = gpu.FactorMatrices.random(dims, 16, 7)
    for mode in range(3):
        want = oracle.mttkrp_coo(dims, idx, vals, f.factors, mode)
        st = gpu.MttkrpStats()
        got = gpu.mttkrp(dt, f, mode, stats=st)
        assert rel_frobenius(got, want) <= TOL
        assert st.strategy == gpu.Strategy.Register and 0 < st.segments <= 1_000_000


def test_high_conflict_short_mode(gpu, oracle):
    """Many elements per row (short target mode).  Auto reports the
    reference's label (Hierarchical: 24 < CUs, mttkrp.cpp:17-21) and runs the
    register kernel, the faster one on B200; the hierarchical stash runs when
    asked for explicitly."""
    dims = [24, 3000, 50]
    coo = gpu.synth_uniform_host(dims, 200_000, 8)
    f = gpu.FactorMatrices.random(dims, 16, 3)
    t = gpu.build_blco(coo)
    want = oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, 0)
    for cfg in (gpu.ExecConfig(), gpu.ExecConfig(num_factor_copies=4), gpu.ExecConfig(num_compute_units=148)):
        st = gpu.MttkrpStats()
        got = gpu.mttkrp(t, f, 0, cfg, stats=st)  # Auto -> label Hierarchical (24 < CUs)
        assert st.strategy == gpu.Strategy.Hierarchical and st.kernel == gpu.Strategy.Register
        assert rel_frobenius(got, want) <= TOL
        st = gpu.MttkrpStats()
        hier = gpu.mttkrp(t, f, 0, cfg, strategy=gpu.Strategy.Hierarchical, stats=st)
        assert st.strategy == st.kernel == gpu.Strategy.Hierarchical and st.stash_flushes > 0
        assert rel_frobenius(hier, want) <= TOL
    reg = gpu.mttkrp(t, f, 0, strategy=gpu.Strategy.Register)
    assert rel_frobenius(reg, want) <= TOL


def test_stats_register_commits(gpu):  # test_mttkrp.cpp:152-188 (GPU meaning)
    coo = gpu.SparseTensorCoo([4, 8], np.array([[1, 1, 2], [0, 4, 1]], np.uint64), [1.0, 2.0, 3.0])
    t = gpu.build_blco(coo)
    f = gpu.FactorMatrices.ones([4, 8], 4)
    st = gpu.MttkrpStats()
    m = gpu.mttkrp(t, f, 0, strategy=gpu.Strategy.Register, stats=st)
    assert st.segments == 2 and st.scalar_adds == 8
    assert m[1, 0] == 3.0 and m[2, 0] == 3.0


def test_validation(gpu):  # test_mttkrp.cpp:319-326
    t = gpu.build_blco(gpu.SparseTensorCoo([4, 4, 4], GI, GV))
    f = gpu.FactorMatrices.ones([4, 4, 4], 2)
    with pytest.raises(gpu.FormatError):
        gpu.mttkrp(t, f, 5)
    bad = gpu.FactorMatrices(2, [f.factors[0], np.zeros((3, 2)), f.factors[2]])
    with pytest.raises(gpu.FormatError):
        gpu.mttkrp(t, bad, 0)


def test_device_pointer_entry(gpu, oracle):
    """blco_mttkrp_device on torch-owned buffers, on torch's current stream."""
    import torch
    dims = [300, 200, 100]
    dt = gpu.DeviceTensor.synthetic(dims, 50_000, 1)
    fs = [torch.empty((d, 32), dtype=torch.float64, device="cuda") for d in dims]
    gpu.factors_random_device(dims, 32, 7, [a.data_ptr() for a in fs],
                              torch.cuda.current_stream().cuda_stream)
    out = torch.empty((dims[1], 32), dtype=torch.float64, device="cuda")
    dt.mttkrp_device([a.data_ptr() for a in fs], 32, 1, out.data_ptr(),
                     stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    idx, vals = oracle.synth_uniform(dims, 50_000, 1)
    hf = oracle.factors_random(dims, 32, 7)
    for a, b in zip(fs, hf):
        assert np.array_equal(a.cpu().numpy(), b)
    want = oracle.mttkrp_coo(dims, idx, vals, hf, 1)
    assert rel_frobenius(out.cpu().numpy(), want) <= TOL
    # accumulate=True adds onto the existing output
    dt.mttkrp_device([a.data_ptr() for a in fs], 32, 1, out.data_ptr(), accumulate=True,
                     stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert rel_frobenius(out.cpu().numpy(), 2 * want) <= TOL


@pytest.mark.parametrize("dims,rank", [([500, 400, 300], 16), ([600_000, 300_000, 300_000], 32)])
def test_slices_sum_to_whole(gpu, oracle, dims, rank):
    """Multi-GPU partition unit: span-aligned slices' partial outputs sum to M
    (the second shape's factors exceed L2, so every slice runs panel-ordered
    with its own tables)."""
    dt = gpu.DeviceTensor.synthetic(dims, 200_000, 4, 20 if dims[0] < 1000 else 48, 30_000)
    f = gpu.FactorMatrices.random(dims, rank, 2)
    idx, vals = oracle.synth_uniform(dims, 200_000, 4)
    for parts in (2, 3, 8):
        ranges = gpu.partition(dt.block_nnz(), 512, parts)
        for mode in range(3):
            acc = sum(gpu.mttkrp(dt.slice(b, e), f, mode) for b, e in ranges)
            want = oracle.mttkrp_coo(dims, idx, vals, f.factors, mode)
            assert rel_frobenius(acc, want) <= TOL


@pytest.mark.parametrize("target,cap,chunk", [(64, 1 << 27, 0), (64, 1 << 27, 5000), (12, 7000, 3000),
                                              (20, 1, 1), (9, 1000, 100_000)])
def test_all_modes_host_pipeline(gpu, oracle, target, cap, chunk):
    """mttkrp_all_modes (blco_mttkrp_all_host): host tensor uploaded in
    chunks (crossing block boundaries) under the per-mode kernels; every M_n
    against the oracle, pageable and pinned host memory, both strategies."""
    dims = [700, 90, 1300]
    coo = gpu.synth_uniform_host(dims, 40_000, 17)
    f = gpu.FactorMatrices.random(dims, 16, 7)
    t = gpu.build_blco(coo, target, cap)
    want = [oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m) for m in range(3)]
    rep = gpu.AllModesReport()
    for strat in (gpu.Strategy.Auto, gpu.Strategy.Hierarchical):
        got = gpu.mttkrp_all_modes(t, f, strategy=strat, chunk_elems=chunk, report=rep)
        for m in range(3):
            assert rel_frobenius(got[m], want[m]) <= TOL, (m, strat)
    assert rep.h2d_bytes >= 40_000 * 16 and rep.d2h_bytes == sum(d * 16 * 8 for d in dims)
    assert rep.launches >= 3 * rep.chunks and rep.device_ms > 0
    # pinned payload / outputs, repeated calls reuse the cached device buffers
    idx = gpu.api.pinned_empty(t.idx.size, np.uint64)
    vals = gpu.api.pinned_empty(t.vals.size, np.float64)
    idx[:], vals[:] = t.idx, t.vals
    tp = gpu.BlcoTensor(t.layout, t.max_nnz_per_block, t.keys, t.offsets, idx, vals)
    outs = [gpu.api.pinned_empty(d * 16, np.float64).reshape(d, 16) for d in dims]
    for _ in range(2):
        got = gpu.mttkrp_all_modes(tp, f, outs=outs, chunk_elems=chunk)
        for m in range(3):
            assert rel_frobenius(got[m], want[m]) <= TOL


def test_all_modes_host_empty_and_errors(gpu):
    dims = [5, 6, 7]
    t = gpu.build_blco(gpu.SparseTensorCoo(dims, np.zeros((3, 0), np.uint64), np.zeros(0)))
    f = gpu.FactorMatrices.random(dims, 4, 1)
    got = gpu.mttkrp_all_modes(t, f)
    assert all(g.shape == (d, 4) and not g.any() for g, d in zip(got, dims))
    with pytest.raises(gpu.FormatError):
        gpu.mttkrp_all_modes(t, gpu.FactorMatrices.random([5, 6, 8], 4, 1))


@pytest.mark.parametrize("dims,nnz,rank", [([700, 90, 1300], 40_000, 16), ([24, 3000, 50], 200_000, 32),
                                           ([40, 50, 30, 20], 30_000, 33), ([300, 200], 20_000, 100),
                                           ([5000], 3000, 8)])
def test_deterministic_mode(gpu, oracle, dims, nnz, rank):
    """ExecConfig::deterministic (exec.hpp:22; exec.cpp:78-86): a fixed
    summation order on the device.  Within 1e-12 of the oracle; bit-identical
    across runs and across block splits / key widths of the same tensor (the
    ALTO element order does not depend on them); rows longer than one chunk
    (2048 elements) go through the ordered partial combine."""
    coo = gpu.synth_uniform_host(dims, nnz, 5)
    f = gpu.FactorMatrices.random(dims, rank, 9)
    det = gpu.ExecConfig(deterministic=True)
    t64 = gpu.build_blco(coo, 64)
    tsplit = gpu.build_blco(coo, max(1, sum(int(d - 1).bit_length() for d in dims) - 3), 1000)
    assert tsplit.keys.size > 1
    for mode in range(len(dims)):
        want = oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, mode)
        a = gpu.mttkrp(t64, f, mode, det)
        assert rel_frobenius(a, want) <= TOL
        assert np.array_equal(a, gpu.mttkrp(t64, f, mode, det))
        assert np.array_equal(a, gpu.mttkrp(tsplit, f, mode, det, gpu.Strategy.Hierarchical))


def test_deterministic_rejected_on_streamed_paths(gpu):
    dims = [50, 40, 60]
    coo = gpu.synth_uniform_host(dims, 600, 3)
    t = gpu.build_blco(coo, 64)
    f = gpu.FactorMatrices.random(dims, 4, 1)
    det = gpu.ExecConfig(deterministic=True)
    with pytest.raises(gpu.FormatError, match="deterministic"):
        gpu.mttkrp_all_modes(t, f, det)
    b = gpu.DeviceBudget(capacity_bytes=1 << 30, num_queues=2, reservation_bytes=1 << 20)
    with pytest.raises(gpu.FormatError, match="deterministic"):
        gpu.stream_mttkrp(t, f, 0, b, det)


@pytest.mark.parametrize("dims,nnz,rank", [([700, 90, 1300], 40_000, 32), ([700, 90, 1300], 40_000, 16),
                                           ([40, 50, 30, 20], 30_000, 64), ([300, 200], 20_000, 8),
                                           ([60, 70, 80], 20_000, 33), ([24, 3000, 50], 100_000, 32)])
def test_fp32_variant(gpu, oracle, dims, nnz, rank):
    """fp32 factors / products / output: relative Frobenius
    <= 1e-5 against the fp64 oracle, every mode, device and host entries."""
    import torch
    coo = gpu.synth_uniform_host(dims, nnz, 13)
    f = gpu.FactorMatrices.random(dims, rank, 7)
    t = gpu.build_blco(coo, 64)
    d = t.device()
    fd = [torch.from_numpy(a.astype(np.float32)).cuda() for a in f.factors]
    for mode in range(len(dims)):
        want = oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, mode)
        got = gpu.mttkrp_f32(t, f, mode)
        assert got.dtype == np.float32 and rel_frobenius(got, want) <= 1e-5, mode
        out = torch.full((dims[mode], rank), 1.0, dtype=torch.float32, device="cuda")
        d.mttkrp_device_f32([a.data_ptr() for a in fd], rank, mode, out.data_ptr(), accumulate=True,
                            stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert rel_frobenius(out.cpu().numpy() - 1.0, want) <= 1e-5


def test_warp_variant_subprocess(gpu):
    """BLCO_B200_VARIANT=warp (the paper's 32-element __match_any_sync tiles,
    read once per process) against the oracle in a fresh process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    code = """
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np
import paper_2201_12523_b200 as b
from pyoracle import Oracle
o = Oracle()
worst = 0.0
for dims, rank in (([700, 90, 1300], 32), ([40, 50, 30, 20], 16), ([300, 200], 33)):
    coo = b.synth_uniform_host(dims, 20000, 3)
    f = b.FactorMatrices.random(dims, rank, 7)
    t = b.build_blco(coo, 64)
    for m in range(len(dims)):
        want = o.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m)
        got = b.mttkrp(t, f, m, strategy=b.Strategy.Register)
        worst = max(worst, float(np.sqrt(((got - want) ** 2).sum() / (want ** 2).sum())))
print(worst)
"""
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, BLCO_B200_VARIANT="warp"))
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL


def test_release_thread_caches(gpu, oracle):
    """blco_release_thread_caches frees the per-thread device buffers; later
    calls re-create them and still match the oracle."""
    dims = [200, 150, 100]
    coo = gpu.synth_uniform_host(dims, 20_000, 4)
    f = gpu.FactorMatrices.random(dims, 16, 2)
    t = gpu.build_blco(coo, 64)
    want = [oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m) for m in range(3)]
    gpu.mttkrp_all_modes(t, f)
    gpu.mttkrp(t, f, 0, gpu.ExecConfig(deterministic=True))
    assert gpu.api.lib.blco_release_thread_caches() == 0
    got = gpu.mttkrp_all_modes(t, f)
    for m in range(3):
        assert rel_frobenius(got[m], want[m]) <= TOL
    assert rel_frobenius(gpu.mttkrp(t, f, 1, gpu.ExecConfig(deterministic=True)), want[1]) <= TOL


_STREAMS_SCRIPT = r"""
import sys, json
import numpy as np
import torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/oracle")
import paper_2201_12523_b200 as b
from pyoracle import Oracle
o = Oracle()
out = {}
cfgs = {"auto": (b.Strategy.Auto, b.ExecConfig()),
        "hier_c3": (b.Strategy.Hierarchical, b.ExecConfig(num_factor_copies=3)),
        "det": (b.Strategy.Auto, b.ExecConfig(deterministic=1))}
for dims, nnz, R in (([300, 200, 500], 400_000, 32), ([64, 3000, 40, 9], 300_000, 16), ([5000, 7], 30_000, 8)):
    dt = b.DeviceTensor.synthetic(dims, nnz, 11)
    idx, vals = o.synth_uniform(dims, nnz, 11)
    f = b.FactorMatrices.random(dims, R, 5)
    fac = [torch.from_numpy(a).cuda() for a in f.factors]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, (strat, cfg) in cfgs.items():
        errs = []
        for m in range(len(dims)):
            want = o.mttkrp_coo(dims, idx, vals, f.factors, m)
            # accumulate=True launches back to back on one stream and
            # concurrently on two (per-stream scratch: hierarchical copies,
            # deterministic partials)
            outs = [torch.zeros((dims[m], R), dtype=torch.float64, device="cuda") for _ in range(4)]
            for k, o_ in enumerate(outs):
                st = (s1, s1, s2, s2)[k]
                dt.mttkrp_device([a.data_ptr() for a in fac], R, m, o_.data_ptr(), strat, cfg, accumulate=True,
                                 stream=st.cuda_stream)
            torch.cuda.synchronize()
            for o_ in outs:
                got = o_.cpu().numpy()
                errs.append(float(np.sqrt(((got - want) ** 2).sum() / (want ** 2).sum())))
        out[f"{dims} {name}"] = max(errs)
print(json.dumps(out))
"""


def test_concurrent_streams_accumulate(gpu):
    """blco_mttkrp_device with accumulate on two streams of one thread at
    once (register, hierarchical with 3 factor copies, deterministic): each
    launch's scratch is per stream, so every result matches the oracle."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", _STREAMS_SCRIPT, root], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert max(res.values()) <= TOL, res


_BIG_TILES_SCRIPT = r"""
import sys, json
import numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/oracle")
import paper_2201_12523_b200 as b
from pyoracle import Oracle
o = Oracle()
out = {}
rng = np.random.default_rng(5)
for dims, nnz, cap in (([300, 200, 500], 200_000, 3000), ([5000, 7], 30_000, 2047), ([90, 80, 70], 100_000, 1 << 27),
                       ([2000, 3000, 10], 150_000, 4097)):
    coo = b.synth_uniform_host(dims, nnz, 3)
    t = b.build_blco(coo, 64, cap)  # many blocks, ragged tile tails at every block end
    for R in (8, 16, 32, 64):
        f = b.FactorMatrices(R, [rng.uniform(-1, 1, (d, R)) for d in dims])
        for m in range(len(dims)):
            want = o.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m)
            got = b.mttkrp(t, f, m, strategy=b.Strategy.Register)
            got32 = b.mttkrp_f32(t, b.FactorMatrices(R, [a.astype(np.float32) for a in f.factors]), m)
            e = float(np.sqrt(((got - want) ** 2).sum() / (want ** 2).sum()))
            e32 = float(np.sqrt(((got32 - want) ** 2).sum() / (want ** 2).sum()))
            out[f"{dims} cap {cap} R {R} mode {m}"] = [e, e32]
print(json.dumps(out))
"""


def test_big_tiles_forced_on_ragged_blocks(gpu):
    """The 2048-element tile path (fp64 and fp32 kernels) forced on
    (BLCO_B200_BIG_TILES=1) for tensors of many small blocks, where every
    block ends in a ragged tile: fp64 within 1e-12, fp32 within 1e-5."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", _BIG_TILES_SCRIPT, root], capture_output=True, text=True,
                       env=dict(os.environ, BLCO_B200_BIG_TILES="1"), timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert max(v[0] for v in res.values()) <= TOL, res
    assert max(v[1] for v in res.values()) <= 1e-5, res


FUSED_CASES = [
    # (dims, nnz, rank, target_bits, cap): narrow staging (non-grouped modes <= 65536 rows), several
    # keyed blocks, R = 16 / 32; a wide case (non-grouped modes > 65536 rows: the general stage)
    ([3000, 2500, 4000], 300_000, 32, 64, 1 << 27),
    ([3000, 2500, 4000], 300_000, 16, 20, 40_000),
    ([70000, 100, 90000], 200_000, 16, 64, 1 << 27),
    ([12092, 9184, 28818], 500_000, 32, 64, 1 << 27),  # NELL-2 dims
]


def _fused_worst(gpu, oracle, dims, nnz, rank, tb, cap):
    import torch
    dt = gpu.DeviceTensor.synthetic(dims, nnz, 5, tb, cap)
    idx, vals = oracle.synth_uniform(dims, nnz, 5)
    f = gpu.FactorMatrices.random(dims, rank, 9)
    fac = [torch.from_numpy(a).cuda() for a in f.factors]
    outs = [torch.full((d, rank), 3.0, dtype=torch.float64, device="cuda") for d in dims]
    fused = dt.mttkrp_all_device([a.data_ptr() for a in fac], rank, [o.data_ptr() for o in outs])
    torch.cuda.synchronize()
    worst = 0.0
    for m in range(3):
        want = oracle.mttkrp_coo(dims, idx, vals, f.factors, m)
        worst = max(worst, rel_frobenius(outs[m].cpu().numpy(), want))
    return fused, worst


@pytest.mark.parametrize("dims,nnz,rank,tb,cap", FUSED_CASES)
def test_all_modes_fused_kernel(gpu, oracle, monkeypatch, dims, nnz, rank, tb, cap):
    """blco_mttkrp_all_device with BLCO_B200_FUSED=1: the fused all-mode
    kernel (k_mttkrp_all3: one staging pass, three rows gathered once per
    element, per-element terms in the oracle's product order) against
    oracle::mttkrp_coo for every mode; without the knob the same entry runs
    the per-mode kernels."""
    monkeypatch.setenv("BLCO_B200_FUSED", "0")
    fused, worst = _fused_worst(gpu, oracle, dims, nnz, rank, tb, cap)
    assert not fused and worst <= TOL
    monkeypatch.setenv("BLCO_B200_FUSED", "1")
    fused, worst = _fused_worst(gpu, oracle, dims, nnz, rank, tb, cap)
    assert fused
    assert worst <= TOL


def test_all_modes_device_falls_back_per_mode(gpu, oracle):
    """Ineligible shapes (order 4, rank 33, or factors beyond the L2 budget)
    run the per-mode kernels through the same entry."""
    import torch
    for dims, rank in (([40, 50, 30, 20], 16), ([300, 200, 100], 33), ([300000, 200000, 100], 32)):
        dt = gpu.DeviceTensor.synthetic(dims, 30_000, 4)
        idx, vals = oracle.synth_uniform(dims, 30_000, 4)
        f = gpu.FactorMatrices.random(dims, rank, 9)
        fac = [torch.from_numpy(a).cuda() for a in f.factors]
        outs = [torch.empty((d, rank), dtype=torch.float64, device="cuda") for d in dims]
        assert not dt.mttkrp_all_device([a.data_ptr() for a in fac], rank, [o.data_ptr() for o in outs])
        torch.cuda.synchronize()
        for m in range(len(dims)):
            want = oracle.mttkrp_coo(dims, idx, vals, f.factors, m)
            assert rel_frobenius(outs[m].cpu().numpy(), want) <= TOL


def test_all_modes_fused_u4_subprocess(gpu):
    """The other register/latency configuration of the fused kernel
    (BLCO_B200_FUSED_CFG=u4m2, read once per process)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    code = """
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import paper_2201_12523_b200 as b
from pyoracle import Oracle
from test_gpu_mttkrp import FUSED_CASES, _fused_worst
o = Oracle()
print(max(_fused_worst(b, o, *c)[1] for c in FUSED_CASES))
"""
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, BLCO_B200_FUSED_CFG="u4m2", BLCO_B200_FUSED="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    assert float(r.stdout.strip().splitlines()[-1]) <= TOL


@pytest.mark.parametrize("dims,panel", [
    ([600_000, 300_000, 300_000], ""), ([600_000, 300_000, 300_000], "10,10"),
    ([600_000, 300_000, 300_000], "3,18"), ([600_000, 300_000, 300_000], "17,2"),
    ([300_000, 200_000, 150_000, 50], ""), ([300_000, 200_000, 150_000, 50], "12,9")])
def test_panel_ordered_dispatch(gpu, oracle, monkeypatch, dims, panel):
    """Factors beyond L2 (here 166-307 MB at R = 32): the register kernel runs
    its tiles in panel order (mttkrp.cu panel_plan: target-mode x
    second-longest non-target-mode panels, ALTO order inside), across keyed
    blocks and with tiles straddling panel edges, against
    oracle::mttkrp_coo for every mode (fp64 within 1e-12, the fp32 variant
    within 1e-5).  The reordered table is built once per (mode, widths): one
    k_tile_panel launch beside the MTTKRP on first use, none after."""
    monkeypatch.setenv("BLCO_B200_PANEL", panel)
    nnz = 400_000
    dt = gpu.DeviceTensor.synthetic(dims, nnz, 11, 48, 90_000)
    idx, vals = oracle.synth_uniform(dims, nnz, 11)
    f = gpu.FactorMatrices.random(dims, 32, 5)
    for mode in range(len(dims)):
        want = oracle.mttkrp_coo(dims, idx, vals, f.factors, mode)
        n0 = gpu.kernel_launch_count()
        got = gpu.mttkrp(dt, f, mode, strategy=gpu.Strategy.Register)
        n1 = gpu.kernel_launch_count()
        again = gpu.mttkrp(dt, f, mode, strategy=gpu.Strategy.Register)
        n2 = gpu.kernel_launch_count()
        assert rel_frobenius(got, want) <= TOL and rel_frobenius(again, want) <= TOL, mode
        assert n2 - n1 == 1 and n1 - n0 == 2, (mode, n1 - n0, n2 - n1)
        # the fp32 variant takes the same panel order (rows of R * 4 bytes)
        assert rel_frobenius(gpu.mttkrp_f32(dt, f, mode).astype(np.float64), want) <= 1e-5, mode


@pytest.mark.parametrize("dims,rank", [([600_000, 300_000, 300_000], 32), ([300_000, 200_000, 150_000, 50], 16),
                                       ([5000, 4000, 3000, 90], 16)])
def test_tile_relative_stage(gpu, oracle, monkeypatch, dims, rank):
    """BLCO_B200_REL_STAGE=1: the opt-in tile-relative 16-byte staging record
    (StageR: every coordinate minus the tile's minimum, packed in 64 bits,
    field widths from the largest per-mode span over the tiles) for wide
    order-3 modes and order 4, across keyed blocks, against the oracle."""
    monkeypatch.setenv("BLCO_B200_REL_STAGE", "1")
    nnz = 300_000
    dt = gpu.DeviceTensor.synthetic(dims, nnz, 13, 48, 70_000)
    idx, vals = oracle.synth_uniform(dims, nnz, 13)
    f = gpu.FactorMatrices.random(dims, rank, 3)
    for mode in range(len(dims)):
        want = oracle.mttkrp_coo(dims, idx, vals, f.factors, mode)
        assert rel_frobenius(gpu.mttkrp(dt, f, mode, strategy=gpu.Strategy.Register), want) <= TOL, mode


@pytest.mark.parametrize("rank", [128, 257, 512])
def test_large_ranks(gpu, oracle, rank):
    """Ranks beyond one lane-group row (several column chunks per launch):
    register and hierarchical fp64 within 1e-12, the fp32 variant within
    1e-5, the deterministic kernel up to its R <= 256 limit."""
    dims = [70, 50, 90]
    coo = gpu.synth_uniform_host(dims, 20_000, rank)
    f = gpu.FactorMatrices.random(dims, rank, 5)
    t = gpu.build_blco(coo, 12, 3000)
    for mode in range(3):
        want = oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, mode)
        for strat in (gpu.Strategy.Register, gpu.Strategy.Hierarchical):
            assert rel_frobenius(gpu.mttkrp(t, f, mode, strategy=strat), want) <= TOL, (mode, strat)
        assert rel_frobenius(gpu.mttkrp_f32(t, f, mode).astype(np.float64), want) <= 1e-5, mode
        if rank <= 256:
            dt = gpu.DeviceTensor.synthetic(dims, 20_000, rank)
            idx, vals = oracle.synth_uniform(dims, 20_000, rank)
            want_d = oracle.mttkrp_coo(dims, idx, vals, f.factors, mode)
            got = gpu.mttkrp(dt, f, mode, gpu.ExecConfig(deterministic=True))
            assert rel_frobenius(got, want_d) <= TOL, mode
