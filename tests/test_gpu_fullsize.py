"""Parity at BASELINE.json's full sizes (SURVEY.md 8c "Large configs").

The oracle cannot hold these tensors' MTTKRPs in seconds, so full-size parity
goes through size-independent checks:
  * row-sampled MTTKRP: S seeded rows per mode of the device M_n against the
    streamed row-sampled oracle (oracle/blco_oracle.c orc_rowsample_uniform),
    whose rows are bit-identical to oracle::mttkrp_coo's on the full tensor;
    tolerance: relative Frobenius <= 1e-12 over the sampled rows (the
    reference's fp64 bar, proj/tests/test_mttkrp.cpp:267-290);
  * the device-built BLCO at full size passes read_blco_block's element checks
    (fields in width, coordinates inside dims, strictly ascending ALTO order;
    blco_format.cpp:201-227) on the device, and (NELL-2) its (cell, value)
    multiset equals the generator's: an order-free 64-bit hash of every
    element, bit-exact.
"""
import numpy as np
import pytest

from conftest import rel_frobenius

pytestmark = pytest.mark.gpu

NELL2 = ([12092, 9184, 28818], 76_879_419, 32)
AMAZON = ([4821207, 1774269, 1805187], 1_741_809_018, 32)
TOL = 1e-12


def _mix64(z):
    z = np.asarray(z, np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _multiset_hash(cells, vals):
    h = _mix64(cells ^ _mix64(np.ascontiguousarray(vals).view(np.uint64)))
    with np.errstate(over="ignore"):
        return int(np.sum(h, dtype=np.uint64))


def _sample_rows(dims, per_mode, seed=11):
    rng = np.random.default_rng(seed)
    return [np.sort(rng.choice(d, size=min(d, per_mode), replace=False)).astype(np.uint64) for d in dims]


def _check_rows(gpu, oracle, dt, dims, nnz, rank, per_mode):
    f = gpu.FactorMatrices.random(dims, rank, 7)
    rows = _sample_rows(dims, per_mode)
    want = oracle.rowsample_uniform(dims, nnz, 42, f.factors, rows)
    for mode in range(len(dims)):
        got = gpu.mttkrp(dt, f, mode)[rows[mode].astype(np.int64)]
        assert rel_frobenius(got, want[mode]) <= TOL, mode
        # every sampled row is non-trivial at these densities
        assert np.count_nonzero(want[mode].any(axis=1)) > 0.9 * rows[mode].size


def test_nell2_full_size_rows(gpu, oracle):
    """BASELINE configs[1] at full size: 76.9M nnz, R=32, every mode."""
    dims, nnz, rank = NELL2
    dt = gpu.DeviceTensor.synthetic(dims, nnz, 42)
    assert dt.nnz == nnz
    _check_rows(gpu, oracle, dt, dims, nnz, rank, 512)


def test_nell2_full_size_build(gpu, oracle):
    """The full-size device build: block checks on the device, and the
    element multiset (cell, value) equals the generator's, bit-exact."""
    dims, nnz, _ = NELL2
    dt = gpu.DeviceTensor.synthetic(dims, nnz, 42)
    dt.validate_device()
    host = dt.to_host()
    lay = host.layout
    cells = np.zeros(nnz, np.uint64)
    stride = 1
    for m in range(3):
        base = np.repeat(np.array([lay.block_base(int(k))[m] for k in host.keys], np.uint64),
                         np.diff(host.offsets).astype(np.int64))
        c = base | ((host.idx >> np.uint64(lay.field_shift[m])) & np.uint64(lay.field_mask[m]))
        assert int(c.max()) < dims[m]
        cells += c * np.uint64(stride)
        stride *= dims[m]
    idx, vals = oracle.synth_uniform(dims, nnz, 42)
    want_cells = idx[0] + idx[1] * np.uint64(dims[0]) + idx[2] * np.uint64(dims[0] * dims[1])
    want = _multiset_hash(want_cells, vals)
    assert _multiset_hash(cells, host.vals) == want
    # the device census and the streamed oracle census agree with it
    assert dt.census() == want == oracle.census_uniform(dims, nnz, 42)[0]


def _reference_chunking(key_counts, max_nnz=1 << 27):
    """Block sizes build_blco produces from per-key element counts: each run
    of equal keys (ascending) is cut every max_nnz elements from its start
    (proj/src/blco_format.cpp:86-111)."""
    sizes = []
    for c in (int(x) for x in key_counts):
        while c > 0:
            sizes.append(min(c, max_nnz))
            c -= sizes[-1]
    return sizes


def test_amazon_full_size_rows(gpu, oracle):
    """BASELINE configs[2] at full size on one B200: 1.74B nnz, 65-bit layout
    (1 stripped bit, 14 blocks), R=32, every mode; device block checks; the
    element multiset (device census vs the generator's streamed census) and
    the per-block nnz against the reference chunking of the per-key counts
    (key 0 = 1,515,318,366 nnz in 12 blocks of <= 2^27, key 1 = 226,490,652
    in 2; blco_format.cpp:86-111)."""
    dims, nnz, rank = AMAZON
    dt = gpu.DeviceTensor.synthetic(dims, nnz, 42)
    assert dt.nnz == nnz and dt.block_nnz().size == 14
    dt.validate_device()
    h, counts = oracle.census_uniform(dims, nnz, 42)
    assert counts.size == 2 and int(counts.sum()) == nnz  # one stripped bit: keys 0 and 1
    assert dt.block_nnz().tolist() == _reference_chunking(counts)  # 12 + 2 blocks
    assert dt.census() == h
    _check_rows(gpu, oracle, dt, dims, nnz, rank, 512)


def test_reddit_stream_chunks_rows(gpu, oracle):
    """BASELINE configs[4] at full scale, two of the 64 ALTO chunks of the
    Reddit-shaped generator (146M elements, 64-bit layout) streamed through a
    capped budget with stream_mttkrp_all_modes (blocks of 2^25); sampled rows
    of every mode against the row-sampled oracle over the decoded COO."""
    dims, nnz_target, nchunks = [8211298, 176962, 8116559], 4_687_474_081, 64
    frac = float(np.prod(np.array(dims, dtype=np.float64))) / 2.0 ** 64
    ncand = int(nnz_target / nchunks / frac) + 1
    idx = gpu.api.pinned_empty(2 * ncand, np.uint64)
    vals = gpu.api.pinned_empty(2 * ncand, np.float64)
    off = 0
    for c in (0, 37):
        off += gpu.api.synth_alto_chunk(dims, c, nchunks, ncand, 42, idx[off:], vals[off:])
    assert off > 2 * 0.95 * nnz_target / nchunks
    layout = gpu.make_layout(dims, 64)
    assert layout.stripped_bits == 0
    coords = np.empty((3, off), np.uint64)
    for m in range(3):
        coords[m] = (idx[:off] >> np.uint64(layout.field_shift[m])) & np.uint64(layout.field_mask[m])
        assert int(coords[m].max()) < dims[m]
    bmax = 1 << 25
    blocks = [(0, idx[o:o + min(bmax, off - o)], vals[o:o + min(bmax, off - o)]) for o in range(0, off, bmax)]
    f = gpu.FactorMatrices.random(dims, 32, 7)
    budget = gpu.DeviceBudget(capacity_bytes=12 << 30, num_queues=3, reservation_bytes=bmax * 16)
    rep = gpu.StreamReport()
    got = gpu.stream_mttkrp_all_modes(iter(blocks), f, budget, report=rep, layout=layout, max_nnz_per_block=bmax,
                                      block_count=len(blocks))
    assert rep.blocks == len(blocks) and rep.bytes_streamed == off * 16
    assert rep.peak_resident_bytes <= budget.capacity_bytes
    rows = _sample_rows(dims, 512)
    want = oracle.rowsample_coo(dims, coords, vals[:off], f.factors, rows)
    for mode in range(3):
        assert rel_frobenius(got[mode][rows[mode].astype(np.int64)], want[mode]) <= TOL, mode


def test_delicious_full_size_rows(gpu, oracle):
    """BASELINE configs[3] at full size: the Delicious-shaped power-law tensor
    (140M distinct draws floor(I*u^4), 78-bit layout, 14 stripped bits, many
    keyed blocks), R=16: device block checks, then sampled rows of every mode
    of the device MTTKRP against the row-sampled oracle over the tensor's
    decoded COO."""
    dims, nnz, rank = [532924, 17262471, 2480308, 1443], 140_126_181, 16
    dt = gpu.DeviceTensor.synthetic_draws(dims, nnz, 42, 4)
    assert dt.nnz == nnz
    dt.validate_device()
    host = dt.to_host()
    lay = host.layout
    assert lay.total_bits == 78 and lay.stripped_bits == 14 and host.keys.size > 1
    counts = np.diff(host.offsets).astype(np.int64)
    coords = np.empty((4, nnz), np.uint64)
    for m in range(4):
        base = np.repeat(np.array([lay.block_base(int(k))[m] for k in host.keys], np.uint64), counts)
        coords[m] = base | ((host.idx >> np.uint64(lay.field_shift[m])) & np.uint64(lay.field_mask[m]))
        assert int(coords[m].max()) < dims[m]
    f = gpu.FactorMatrices.random(dims, rank, 7)
    rows = _sample_rows(dims, 256)
    want = oracle.rowsample_coo(dims, coords, host.vals, f.factors, rows)
    for mode in range(4):
        got = gpu.mttkrp(dt, f, mode)[rows[mode].astype(np.int64)]
        assert rel_frobenius(got, want[mode]) <= TOL, mode


def test_repeated_streaming_three_queues(gpu):
    """Regression: repeated stream_mttkrp_all_modes calls with 3 queues in one
    process.  A queue's tile table used to be uploaded with a plain pageable
    cudaMemcpy, which returns once the data is staged; the queue is a
    non-blocking stream, so its kernels could read the table before the DMA
    landed, and every third call or so one block came out wrong (rel. error
    0.18-0.30).  scripts/stream_repro.py: one Reddit ALTO chunk (73M
    elements), 2^24-element blocks, 4 calls against a device-resident MTTKRP."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "scripts" / "stream_repro.py"), "1", "24", "4", "3"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    errs = [float(ln.split("err ")[1].split()[0]) for ln in r.stdout.splitlines() if ln.startswith("rep ")]
    assert len(errs) == 4 and max(errs) <= 1e-12, r.stdout
