"""The C oracle (oracle/blco_oracle.c) pinned against the reference.

Two anchors: (1) the reference's own golden vectors, restated from
proj/tests/*.cpp with the cited lines; (2) tests/golden/golden.npz, produced
by the unmodified reference library (tests/golden/gen_golden.py).  CPU only.
"""
import numpy as np
import pytest

from conftest import rel_frobenius

GI = np.array([[0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 3, 3],
               [0, 0, 2, 0, 0, 0, 3, 1, 1, 2, 2, 3],
               [0, 1, 2, 1, 2, 1, 3, 0, 1, 2, 3, 3]], np.uint64)  # test_util.hpp:31-35
GV = np.arange(1, 13, dtype=np.float64)


def test_layout_444_full_width(oracle):  # test_layout.cpp:8-21
    l = oracle.layout([4, 4, 4], 64)
    assert list(l.mode_bits[:3]) == [2, 2, 2] and l.total_bits == 6 and l.stripped_bits == 0
    assert [(l.imap_mode[p], l.imap_bit[p]) for p in range(6)] == [(0, 0), (1, 0), (2, 0), (0, 1), (1, 1), (2, 1)]


def test_layout_444_5bit(oracle):  # test_layout.cpp:23-30
    l = oracle.layout([4, 4, 4], 5)
    assert l.stripped_bits == 1
    assert list(l.rem_bits[:3]) == [2, 2, 1]
    assert list(l.field_shift[:3]) == [0, 2, 4]
    assert list(l.field_mask[:3]) == [3, 3, 1]


def test_layout_errors(oracle):  # test_layout.cpp:41-46
    from pyoracle import OracleError
    for dims, tb in (([4, 4], 0), ([4, 4], 65), ([0, 4], 32)):
        with pytest.raises(OracleError):
            oracle.layout(dims, tb)


def test_alto_goldens(oracle):  # test_layout.cpp:48-64
    l = oracle.layout([4, 4, 4], 64)
    for c, a in (([0, 0, 0], 0), ([0, 0, 1], 4), ([3, 3, 3], 63), ([1, 0, 1], 5), ([3, 1, 0], 11),
                 ([2, 0, 1], 12), ([3, 1, 1], 15), ([1, 0, 2], 33), ([0, 2, 2], 48), ([3, 2, 2], 57),
                 ([3, 2, 3], 61), ([2, 3, 3], 62)):
        assert oracle.linearize(l, c) == a


def test_split_goldens(oracle):  # test_layout.cpp:66-86 (value-8.0 entry is 7, PAPER.md:469 typo)
    l = oracle.layout([4, 4, 4], 5)
    assert oracle.split(l, 48) == (1, 8)
    assert oracle.split(l, 15) == (0, 23)
    assert oracle.split(l, 0) == (0, 0)
    assert oracle.split(l, 11) == (0, 7)
    assert oracle.delinearize(l, 23, 0) == [3, 1, 1]  # test_layout.cpp:88-95
    assert oracle.delinearize(l, 1, 1) == [1, 0, 2]


def test_fig5b_blocks(oracle):  # test_blco.cpp:11-24
    keys, offs, idx, vals = oracle.build([4, 4, 4], GI, GV, 5, 6)
    assert keys.tolist() == [0, 1] and offs.tolist() == [0, 6, 12]
    assert idx[:6].tolist() == [0, 16, 17, 7, 18, 23] and vals[:6].tolist() == [1, 2, 4, 8, 6, 9]
    assert idx[6:].tolist() == [1, 8, 11, 27, 30, 31] and vals[6:].tolist() == [5, 3, 10, 11, 7, 12]


def test_capacity_split(oracle):  # test_blco.cpp:33-48
    keys, offs, idx, _ = oracle.build([4, 4, 4], GI, GV, 5, 4)
    assert keys.tolist() == [0, 0, 1, 1] and np.diff(offs).tolist() == [4, 2, 4, 2]
    assert idx.tolist() == [0, 16, 17, 7, 18, 23, 1, 8, 11, 27, 30, 31]


def test_batch_table(oracle):  # test_blco.cpp:103-122
    assert oracle.batch_table([6, 6], 6).tolist() == [[0, 0, 6], [1, 0, 6]]
    assert oracle.batch_table([6, 6], 4).tolist() == [[0, 0, 4], [0, 4, 2], [1, 0, 4], [1, 4, 2]]
    assert oracle.batch_table([0], 8).size == 0


def test_duplicates_rejected(oracle):  # test_blco.cpp:95-101
    from pyoracle import OracleError
    with pytest.raises(OracleError, match="duplicate"):
        oracle.build([2, 2], np.array([[0, 0], [1, 1]]), [1.0, 2.0], 64)


def test_all_ones_rows(oracle):  # test_oracle.cpp:8-21 / test_mttkrp.cpp:33-47
    ones = [np.ones((4, 2))] * 3
    m1 = oracle.mttkrp_coo([4, 4, 4], GI, GV, ones, 0)
    assert m1[:, 0].tolist() == [6, 9, 13, 50] and m1[:, 1].tolist() == [6, 9, 13, 50]
    m3 = oracle.mttkrp_coo([4, 4, 4], GI, GV, ones, 2)
    assert m3[:, 0].tolist() == [9, 21, 18, 30]


def test_golden_layouts(oracle, golden):
    z, meta = golden
    from pyoracle import OracleError
    for ent in meta["layouts"]:
        if not ent["ok"]:
            with pytest.raises(OracleError):
                oracle.layout(ent["dims"], ent["target"])
            continue
        l = oracle.layout(ent["dims"], ent["target"])
        n = len(ent["dims"])
        assert l.total_bits == ent["total_bits"] and l.stripped_bits == ent["stripped_bits"]
        assert list(l.mode_bits[:n]) == ent["mode_bits"]
        assert list(l.rem_bits[:n]) == ent["rem_bits"]
        assert list(l.field_shift[:n]) == ent["field_shift"]
        assert [int(x) for x in l.field_mask[:n]] == ent["field_mask"]
        assert list(l.imap_mode[: l.total_bits]) == ent["imap_mode"]
        assert list(l.imap_bit[: l.total_bits]) == ent["imap_bit"]


def test_golden_encodes(oracle, golden):
    z, meta = golden
    for k, ent in enumerate(meta["encodes"]):
        l = oracle.layout(ent["dims"], ent["target"])
        coords, outs = z[f"enc{k}_coords"], z[f"enc{k}_out"]
        for j in range(coords.shape[1]):
            c = coords[:, j]
            alto = oracle.linearize(l, c)
            hi, lo, sk, sr, ek, er = (int(x) for x in outs[j])
            assert alto == (hi << 64) | lo
            assert oracle.split(l, alto) == (sk, sr)
            assert oracle.encode(l, c) == (ek, er)
            assert oracle.delinearize(l, er, ek) == [int(x) for x in c]


def test_golden_builds(oracle, golden):
    z, meta = golden
    for k, ent in enumerate(meta["builds"]):
        keys, offs, idx, vals = oracle.build(ent["dims"], z[f"b{k}_in_idx"], z[f"b{k}_in_vals"],
                                             ent["target"], ent["max_nnz"])
        assert np.array_equal(keys, z[f"b{k}_keys"]), k
        assert np.array_equal(offs, z[f"b{k}_offsets"]), k
        assert np.array_equal(idx, z[f"b{k}_idx"]), k
        assert np.array_equal(vals, z[f"b{k}_vals"]), k
        assert np.array_equal(oracle.batch_table(np.diff(offs), 512), z[f"b{k}_batch"]), k


def test_golden_mttkrp_coo_bitexact(oracle, golden):
    """The oracle is the same sequential loop as oracle::mttkrp_coo: bit-exact."""
    z, meta = golden
    for j, ent in enumerate(meta["mttkrps"]):
        b = ent["build"]
        dims = meta["builds"][b]["dims"]
        fs = [z[f"m{j}_f{m}"] for m in range(len(dims))]
        for mode in range(len(dims)):
            got = oracle.mttkrp_coo(dims, z[f"b{b}_in_idx"], z[f"b{b}_in_vals"], fs, mode)
            assert np.array_equal(got, z[f"m{j}_coo{mode}"])
            assert rel_frobenius(z[f"m{j}_blco{mode}"], got) <= 1e-12


def test_golden_factors_random(oracle, golden):
    z, meta = golden
    for j, ent in enumerate(meta["factors"]):
        fs = oracle.factors_random(ent["dims"], ent["rank"], ent["seed"])
        for m, a in enumerate(fs):
            assert np.array_equal(a, z[f"fr{j}_{m}"])


def test_golden_cp_als(oracle, golden):
    z, meta = golden
    for j, ent in enumerate(meta["cpals"]):
        dims = ent["dims"]
        keys, offs, idx, vals = oracle.build(dims, z[f"c{j}_in_idx"], z[f"c{j}_in_vals"], 64)
        fs, lam, fit = oracle.cp_als(dims, keys, offs, idx, vals, ent["rank"], ent["iters"], ent["tol"],
                                     ent["seed"])
        want = z[f"c{j}_fit"]
        assert fit.size == want.size
        assert np.max(np.abs(fit - want)) <= 1e-10
        for m in range(len(dims)):
            assert rel_frobenius(fs[m], z[f"c{j}_f{m}"]) <= 1e-8


def test_synth_unique_and_in_range(oracle):
    dims = [37, 41, 43]
    idx, vals = oracle.synth_uniform(dims, 20000, 42)
    cell = idx[0] + 37 * (idx[1] + 41 * idx[2])
    assert np.unique(cell).size == 20000
    assert all((idx[m] < dims[m]).all() for m in range(3))
    assert (vals >= 0).all() and (vals < 1).all()
    # the full cell set is a permutation
    idx2, _ = oracle.synth_uniform(dims, 37 * 41 * 43, 1)
    cell2 = idx2[0] + 37 * (idx2[1] + 41 * idx2[2])
    assert np.array_equal(np.sort(cell2), np.arange(37 * 41 * 43))


def test_oracle_matches_reference_live(oracle, reflib):
    """Randomised cross-check against the reference library (when built here)."""
    rng = np.random.default_rng(11)
    for trial in range(25):
        order = int(rng.integers(2, 5))
        dims = [int(rng.integers(1, 200)) for _ in range(order)]
        cells = int(np.prod(dims))
        nnz = min(cells, int(rng.integers(1, 400)))
        ids = rng.choice(cells, size=nnz, replace=False)
        idx = np.array(np.unravel_index(ids, dims[::-1])[::-1], np.uint64)
        vals = rng.uniform(-1, 1, nnz)
        tb, cap = int(rng.integers(3, 65)), int(rng.integers(1, 100))
        try:
            t = reflib.build(dims, idx, vals, tb, cap)
        except Exception:  # noqa: BLE001 - layout errors must agree
            from pyoracle import OracleError
            with pytest.raises(OracleError):
                oracle.build(dims, idx, vals, tb, cap)
            continue
        got = oracle.build(dims, idx, vals, tb, cap)
        for a, b in zip(got, t.blocks()):
            assert np.array_equal(a, b)


def test_rowsample_equals_full_oracle_rows(oracle, reflib):
    """The streamed row-sampled oracle (full-size parity) gives
    bit-identical rows to oracle::mttkrp_coo on the materialised tensor --
    both the C restatement's and the reference's own."""
    dims, nnz, rank = [300, 170, 410], 200_000, 8
    idx, vals = oracle.synth_uniform(dims, nnz, 42)
    f = oracle.factors_random(dims, rank, 7)
    rng = np.random.default_rng(5)
    rows = [np.sort(rng.choice(d, size=min(d, 37), replace=False)) for d in dims]
    got = oracle.rowsample_uniform(dims, nnz, 42, f, rows, threads=3)
    for m in range(3):
        full = oracle.mttkrp_coo(dims, idx, vals, f, m)
        assert np.array_equal(got[m], full[rows[m]])
        assert np.array_equal(got[m], reflib.mttkrp_coo(dims, idx, vals, f, m)[rows[m]])


def test_rowsample_coo_equals_full_oracle_rows(oracle):
    dims, nnz, rank = [120, 90, 60], 40_000, 8
    idx, vals = oracle.synth_uniform(dims, nnz, 9)
    f = oracle.factors_random(dims, rank, 3)
    rng = np.random.default_rng(2)
    rows = [np.sort(rng.choice(d, size=17, replace=False)) for d in dims]
    got = oracle.rowsample_coo(dims, idx, vals, f, rows)
    for m in range(3):
        assert np.array_equal(got[m], oracle.mttkrp_coo(dims, idx, vals, f, m)[rows[m]])


def test_census_uniform_matches_materialised_tensor(oracle):
    """orc_census_uniform streams the generator: its multiset hash equals the
    hash of the materialised COO, and its per-key counts equal the per-key
    totals of the oracle build of a multi-key layout (blco_format.cpp:86-111)."""
    from test_gpu_fullsize import _multiset_hash, _reference_chunking
    dims, nnz, tb = [300, 200, 250], 50_000, 20
    h, counts = oracle.census_uniform(dims, nnz, 42, tb, threads=3)
    idx, vals = oracle.synth_uniform(dims, nnz, 42)
    cells = idx[0] + idx[1] * np.uint64(dims[0]) + idx[2] * np.uint64(dims[0] * dims[1])
    assert h == _multiset_hash(cells, vals)
    keys, offs, _, _ = oracle.build(dims, idx, vals, tb, 1000)
    per_key = np.zeros(counts.size, np.uint64)
    for k, n in zip(keys, np.diff(offs)):
        per_key[int(k)] += n
    assert np.array_equal(per_key, counts)
    assert np.diff(offs).tolist() == _reference_chunking(counts, 1000)


def test_oracle_cp_als_matches_reference_r32(oracle):
    """The C restatement of cp_als (cpals.cpp:66-111) at R = 32 against the
    reference's own run (tests/golden/cpals_exact_rank.npz, n32): the oracle
    is pinned on the exact rank the device epilogue specialises."""
    import json
    from pathlib import Path
    z = np.load(Path(__file__).resolve().parent / "golden" / "cpals_exact_rank.npz")
    c = json.loads(bytes(z["meta"]).decode())["n32"]
    dims = c["dims"]
    idx, vals = oracle.synth_draws(dims, c["nnz"], c["seed"], c["skew"])
    keys, offs, oi, ov = oracle.build(dims, idx, vals)
    fs, lam, fit = oracle.cp_als(dims, keys, offs, oi, ov, c["rank"], c["iters"], c["tol"], c["fseed"])
    assert np.max(np.abs(fit - z["n32_fit"])) <= 1e-10
    assert rel_frobenius(lam, z["n32_lambda"]) <= 1e-9
    for m in range(len(dims)):
        assert rel_frobenius(fs[m], z[f"n32_f{m}"]) <= 1e-9



@pytest.mark.parametrize("dims,rank", [([30, 40, 50], 1), ([30, 40, 50], 7), ([45, 35, 55], 24),
                                       ([50, 60, 70, 40], 33), ([40, 50, 60, 30, 20], 17), ([80, 90, 70], 64),
                                       ([40, 50], 5), ([9, 8, 7, 6, 5, 6, 7, 8], 3)])
def test_oracle_cp_als_matches_reference_live(oracle, reflib, dims, rank):
    """The C restatement of cp_als against the live reference (libblco_ref.so
    cp_als, 1 thread) on the random shapes the GPU CP-ALS is checked on
    (tests/test_gpu_stream_cpals.py): the oracle those GPU tests trust is
    itself pinned over ranks 1-64 and orders 2-8."""
    nnz = min(4000, int(np.prod(dims)) // 2)
    idx, vals = oracle.synth_uniform(dims, nnz, 3 + rank)
    keys, offs, oi, ov = oracle.build(dims, idx, vals)
    fs, lam, fit = oracle.cp_als(dims, keys, offs, oi, ov, rank, 6, -1e300, 11)
    from pyoracle import cfg_array
    t = reflib.build(dims, idx, vals, 64)
    rfs, rlam, rfit = t.cp_als(dims, rank, 6, -1e300, 11, cfg=cfg_array(num_threads=1))
    assert rfit.size == fit.size == 6
    assert np.max(np.abs(fit - rfit)) <= 1e-10
    for m in range(len(dims)):
        assert rel_frobenius(fs[m], rfs[m]) <= 1e-9, m
    assert rel_frobenius(lam, rlam) <= 1e-9
