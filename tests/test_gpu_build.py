"""Device BLCO construction (K1 encode, K2 radix sort, K3 runs/chunks/gather)
is bit-exact with the reference build_blco (proj/src/blco_format.cpp:62-134):
same blocks, keys, element order, re-encoded indices, values, batch table."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GI = np.array([[0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 3, 3],
               [0, 0, 2, 0, 0, 0, 3, 1, 1, 2, 2, 3],
               [0, 1, 2, 1, 2, 1, 3, 0, 1, 2, 3, 3]], np.uint64)
GV = np.arange(1, 13, dtype=np.float64)


def build(b, dims, idx, vals, tb=64, cap=1 << 27):
    return b.build_blco(b.SparseTensorCoo(list(dims), idx, vals), tb, cap)


def test_fig5b_blocks(gpu):  # proj/tests/test_blco.cpp:11-24
    t = build(gpu, [4, 4, 4], GI, GV, 5, 6)
    blocks = t.blocks
    assert len(blocks) == 2 and t.total_nnz == 12
    assert blocks[0].key == 0 and blocks[0].linear_indices.tolist() == [0, 16, 17, 7, 18, 23]
    assert blocks[0].values.tolist() == [1, 2, 4, 8, 6, 9]
    assert blocks[1].key == 1 and blocks[1].linear_indices.tolist() == [1, 8, 11, 27, 30, 31]
    assert blocks[1].values.tolist() == [5, 3, 10, 11, 7, 12]


def test_single_block_at_64(gpu):  # test_blco.cpp:26-31
    t = build(gpu, [4, 4, 4], GI, GV, 64)
    assert t.keys.tolist() == [0] and t.total_nnz == 12


def test_capacity_split(gpu):  # test_blco.cpp:33-48
    t = build(gpu, [4, 4, 4], GI, GV, 5, 4)
    assert t.keys.tolist() == [0, 0, 1, 1]
    assert np.diff(t.offsets).tolist() == [4, 2, 4, 2]
    assert t.idx.tolist() == [0, 16, 17, 7, 18, 23, 1, 8, 11, 27, 30, 31]


def test_duplicates_rejected(gpu):  # test_blco.cpp:95-101
    with pytest.raises(gpu.FormatError, match="duplicate"):
        build(gpu, [2, 2], np.array([[0, 0], [1, 1]], np.uint64), [1.0, 2.0])


def test_out_of_range_rejected(gpu):
    with pytest.raises(gpu.FormatError, match="out of range"):
        build(gpu, [2, 2], np.array([[0, 2], [1, 1]], np.uint64), [1.0, 2.0])


def test_empty_tensor(gpu):
    t = build(gpu, [3, 4], np.zeros((2, 0), np.uint64), np.zeros(0))
    assert t.total_nnz == 0 and t.keys.size == 0


def test_golden_builds_bitexact(gpu, golden):
    z, meta = golden
    for k, ent in enumerate(meta["builds"]):
        t = build(gpu, ent["dims"], z[f"b{k}_in_idx"], z[f"b{k}_in_vals"], ent["target"], ent["max_nnz"])
        assert np.array_equal(t.keys, z[f"b{k}_keys"]), k
        assert np.array_equal(t.offsets, z[f"b{k}_offsets"]), k
        assert np.array_equal(t.idx, z[f"b{k}_idx"]), k
        assert np.array_equal(t.vals, z[f"b{k}_vals"]), k
        assert np.array_equal(t.batch_table, z[f"b{k}_batch"]), k


@pytest.mark.parametrize("dims,nnz,tb,cap", [
    ([1000, 1000, 1000], 1_000_000, 64, 1 << 27),            # config 1 shape
    ([4821207, 1774269, 1805187], 300_000, 64, 100_000),     # Amazon: 65 bits, 1 stripped
    ([6066, 5699, 244268, 1176], 300_000, 40, 50_000),       # Enron at a tight budget
    ([8211298, 176962, 8116559], 200_000, 64, 30_000),       # Reddit: 64 bits, chunked
])
def test_synthetic_builds_match_oracle(gpu, oracle, dims, nnz, tb, cap):
    dt = gpu.DeviceTensor.synthetic(dims, nnz, 42, tb, cap)
    t = dt.to_host()
    idx, vals = oracle.synth_uniform(dims, nnz, 42)
    keys, offs, oi, ov = oracle.build(dims, idx, vals, tb, cap)
    assert np.array_equal(t.keys, keys)
    assert np.array_equal(t.offsets, offs)
    assert np.array_equal(t.idx, oi)
    assert np.array_equal(t.vals, ov)
    # host COO path gives the same tensor as the on-device generator
    t2 = build(gpu, dims, idx, vals, tb, cap)
    assert t2.structurally_equal(t)
    # the device census (order-free multiset hash) equals the generator's
    h, counts = oracle.census_uniform(dims, nnz, 42, tb)
    assert dt.census() == h
    per_key = {}
    for k, n in zip(t.keys, np.diff(t.offsets)):
        per_key[int(k)] = per_key.get(int(k), 0) + int(n)
    assert per_key == {k: int(c) for k, c in enumerate(counts) if c}


@pytest.mark.parametrize("dims,nnz,skew,cap", [
    ([532924, 17262471, 2480308, 1443], 200_000, 1, 1 << 27),  # Delicious: 78 bits, 14 stripped
    ([532924, 17262471, 2480308, 1443], 200_000, 4, 40_000),   # skewed power law, chunked
    ([6066, 5699, 244268, 1176], 300_000, 6, 1 << 27),         # Enron-shaped, heavy skew
    ([50, 60, 70], 150_000, 3, 1 << 27),                       # dense-ish: many duplicate draws
])
def test_draws_builds_match_oracle(gpu, oracle, dims, nnz, skew, cap):
    """Config-4 generator: first nnz distinct draws; multi-key wide layouts."""
    dt = gpu.DeviceTensor.synthetic_draws(dims, nnz, 42, skew, 64, cap)
    t = dt.to_host()
    idx, vals = oracle.synth_draws(dims, nnz, 42, skew)
    keys, offs, oi, ov = oracle.build(dims, idx, vals, 64, cap)
    assert t.total_nnz == nnz
    assert np.array_equal(t.keys, keys) and np.array_equal(t.offsets, offs)
    assert np.array_equal(t.idx, oi) and np.array_equal(t.vals, ov)
    # the host candidate stream is the same draw sequence
    hi, hv = gpu.synth_draws_host(dims, 64, 42, skew)
    oi2, ov2 = oracle.synth_draws(dims, 8, 42, skew)
    assert np.array_equal(hi[:, 0], oi2[:, 0]) and hv[0] == ov2[0]


def test_reference_build_live(gpu, reflib):
    """Against the reference library itself (built here from /root/reference)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        order = int(rng.integers(2, 6))
        dims = [int(rng.integers(1, 1 << int(rng.integers(1, 18)))) for _ in range(order)]
        cells = int(np.prod(np.array(dims, dtype=object)))
        nnz = int(min(cells, rng.integers(1, 3000)))
        if cells < 2**62:
            ids = rng.choice(cells, size=nnz, replace=False)
        else:
            ids = np.unique(rng.integers(0, 2**62, size=2 * nnz))[:nnz]
        x = ids.astype(object)
        idx = np.zeros((order, len(ids)), np.uint64)
        for m, d in enumerate(dims):
            idx[m] = [int(v) % d for v in x]
            x = np.array([int(v) // d for v in x], dtype=object)
        vals = rng.uniform(-1, 1, len(ids))
        tb, cap = int(rng.integers(8, 65)), int(rng.integers(1, 4000))
        try:
            r = reflib.build(dims, idx, vals, tb, cap).blocks()
        except Exception:  # noqa: BLE001
            with pytest.raises(gpu.Error):
                build(gpu, dims, idx, vals, tb, cap)
            continue
        if gpu.make_layout(dims, tb).stripped_bits > 64:
            continue
        t = build(gpu, dims, idx, vals, tb, cap)
        assert np.array_equal(t.keys, r[0]) and np.array_equal(t.offsets, r[1])
        assert np.array_equal(t.idx, r[2]) and np.array_equal(t.vals, r[3])


def test_conservation_roundtrip(gpu):  # test_blco.cpp:50-84 (delinearize all blocks)
    dims = [300, 17, 129, 5]
    dt = gpu.DeviceTensor.synthetic(dims, 20_000, 5, 13, 997)
    t = dt.to_host()
    coo = gpu.synth_uniform_host(dims, 20_000, 5)
    got = set()
    for blk in t.blocks:
        assert blk.nnz() <= 997
        for i, v in zip(blk.linear_indices.tolist(), blk.values.tolist()):
            got.add((tuple(gpu.delinearize(t.layout, i, blk.key)), v))
    want = {(tuple(int(x) for x in coo.indices[:, e]), float(coo.values[e])) for e in range(coo.nnz())}
    assert got == want
    assert (np.diff(t.keys.astype(np.int64)) >= 0).all()


@pytest.fixture
def small_passes(monkeypatch):
    """Force the multi-pass host-COO build (the >= 2^31-element / beyond
    device memory path) at test sizes: BLCO_B200_BUILD_PASS_ELEMS is read on
    every build call."""
    def set_cap(n):
        monkeypatch.setenv("BLCO_B200_BUILD_PASS_ELEMS", str(n))
    return set_cap


@pytest.mark.parametrize("dims,nnz,tb,cap,pass_elems,draws", [
    ([300, 200, 250], 50_000, 20, 3000, 7_000, 0),             # several keys, runs spanning passes
    ([8211298, 176962, 8116559], 60_000, 64, 5_000, 9_000, 0),  # Reddit dims: one key over every pass
    ([4821207, 1774269, 1805187], 40_000, 64, 1 << 27, 6_000, 0),  # Amazon: 65-bit, two-word ALTO
    ([532924, 17262471, 2480308, 1443], 40_000, 64, 2_000, 5_000, 4),  # Delicious: 78 bits, 14 stripped
])
def test_multi_pass_build_bit_exact(gpu, oracle, small_passes, dims, nnz, tb, cap, pass_elems, draws):
    """The out-of-core build (ALTO-range passes over the host COO, runs merged
    across passes, global chunking at max_nnz_per_block) equals the in-core
    reference build_blco bit for bit (blco_format.cpp:62-134)."""
    if draws:
        idx, vals = oracle.synth_draws(dims, nnz, 42, draws)
    else:
        idx, vals = oracle.synth_uniform(dims, nnz, 42)
    keys, offs, oi, ov = oracle.build(dims, idx, vals, tb, cap)
    small_passes(pass_elems)
    t = build(gpu, dims, idx, vals, tb, cap)
    assert np.array_equal(t.keys, keys) and np.array_equal(t.offsets, offs)
    assert np.array_equal(t.idx, oi) and np.array_equal(t.vals, ov)


def test_multi_pass_build_errors(gpu, small_passes):
    """Duplicates (in one pass by construction: equal ALTO) and out-of-range
    coordinates are rejected on the multi-pass path too."""
    small_passes(1_000)
    rng = np.random.default_rng(1)
    idx = rng.integers(0, 100, size=(3, 5_000)).astype(np.uint64)
    idx[:, 4_000] = idx[:, 10]  # a duplicate far from its twin in input order
    vals = rng.uniform(size=5_000)
    with pytest.raises(gpu.FormatError, match="duplicate"):
        build(gpu, [100, 100, 100], idx, vals)
    idx = rng.integers(0, 100, size=(3, 5_000)).astype(np.uint64)
    idx[1, 77] = 100
    with pytest.raises(gpu.FormatError, match="out of range"):
        build(gpu, [100, 100, 100], idx, vals)
