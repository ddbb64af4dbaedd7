"""libblco_b200.so: loads, exports every declared symbol, and its host-side
logic (layout, encode/decode, batch table, partition, seeded generators,
config) matches the reference.  CPU only -- no compute calls need a GPU."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    hdr = (ROOT / "include" / "blco_b200.h").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(blco_[a-z0-9_]+)\s*\(", hdr)) - {"blco_block_source_fn"})


def test_exports_every_declared_symbol(blco):
    from paper_2201_12523_b200 import _lib
    syms = declared_symbols()
    assert len(syms) > 30
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    """The fat binary carries sm_100a SASS (no PTX fallback to other archs)."""
    import subprocess
    so = ROOT / "paper_2201_12523_b200" / "lib" / "libblco_b200.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_layouts_match_reference(blco, golden):
    z, meta = golden
    for ent in meta["layouts"]:
        if not ent["ok"]:
            with pytest.raises(blco.FormatError):
                blco.make_layout(ent["dims"], ent["target"])
            continue
        l = blco.make_layout(ent["dims"], ent["target"])
        assert l.total_bits == ent["total_bits"] and l.stripped_bits == ent["stripped_bits"]
        assert l.mode_bits == ent["mode_bits"] and l.rem_bits == ent["rem_bits"]
        assert l.field_shift == ent["field_shift"] and l.field_mask == ent["field_mask"]
        assert [m for m, _ in l.interleave_map] == ent["imap_mode"]
        assert [b for _, b in l.interleave_map] == ent["imap_bit"]


def test_encode_decode_match_reference(blco, golden):
    z, meta = golden
    for k, ent in enumerate(meta["encodes"]):
        l = blco.make_layout(ent["dims"], ent["target"])
        coords, outs = z[f"enc{k}_coords"], z[f"enc{k}_out"]
        for j in range(coords.shape[1]):
            c = [int(x) for x in coords[:, j]]
            hi, lo, sk, sr, ek, er = (int(x) for x in outs[j])
            alto = blco.linearize(l, c)
            assert alto == (hi << 64) | lo
            s = blco.split_block_key(l, alto)
            assert (s.block_key, s.reencoded) == (sk, sr)
            e = blco.encode_coords(l, c)
            assert (e.block_key, e.reencoded) == (ek, er)
            assert blco.delinearize(l, er, ek) == c


def test_reference_layout_goldens(blco):  # proj/tests/test_layout.cpp:8-95
    l = blco.make_layout([4, 4, 4], 5)
    assert l.rem_bits == [2, 2, 1] and l.field_shift == [0, 2, 4] and l.field_mask == [3, 3, 1]
    s = blco.split_block_key(l, 11)
    assert (s.block_key, s.reencoded) == (0, 7)
    assert blco.delinearize(l, 1, 1) == [1, 0, 2]
    with pytest.raises(blco.FormatError):
        blco.linearize(blco.make_layout([4, 4, 4]), [4, 0, 0])
    l1 = blco.make_layout([1, 1, 1], 64)
    assert l1.total_bits == 0 and blco.linearize(l1, [0, 0, 0]) == 0


def test_stripped_above_64_is_rejected(blco):
    """the reference silently truncates keys of > 64 stripped bits
    (proj/src/layout.cpp:87); we refuse instead of reproducing UB."""
    l = blco.make_layout([1 << 20] * 5, 4)  # 100 bits, 96 stripped
    assert l.stripped_bits > 64
    with pytest.raises(blco.FormatError, match="stripped"):
        blco.encode_coords(l, [1, 2, 3, 4, 5])


def test_batch_table_and_partition(blco, golden):
    z, meta = golden
    for k, ent in enumerate(meta["builds"]):
        bn = np.diff(z[f"b{k}_offsets"])
        layout = blco.make_layout(ent["dims"], ent["target"])
        t = blco.BlcoTensor(layout, ent["max_nnz"], z[f"b{k}_keys"], z[f"b{k}_offsets"], z[f"b{k}_idx"],
                            z[f"b{k}_vals"])
        assert np.array_equal(t.batch_table, z[f"b{k}_batch"])
        for parts in (1, 2, 3, 8):
            rng_ = blco.partition(bn, 512, parts)
            assert rng_[0][0] == 0 and rng_[-1][1] == int(bn.sum())
            assert all(rng_[i][1] == rng_[i + 1][0] for i in range(parts - 1))


def test_partition_balance(blco):
    bn = [1 << 27] * 12 + [7_000_000, 123]
    total = sum(bn)
    for parts in (2, 4, 8):
        r = blco.partition(bn, 512, parts)
        sizes = [e - b for b, e in r]
        assert sum(sizes) == total
        assert max(sizes) - min(sizes) <= 2 * 512


def test_factors_random_matches_reference(blco, golden):
    z, meta = golden
    for j, ent in enumerate(meta["factors"]):
        f = blco.FactorMatrices.random(ent["dims"], ent["rank"], ent["seed"])
        for m, a in enumerate(f.factors):
            assert np.array_equal(a, z[f"fr{j}_{m}"])


def test_synth_host_matches_oracle(blco, oracle):
    for dims, nnz, seed in (([1000, 1000, 1000], 5000, 42), ([12092, 9184, 28818], 3000, 42),
                            ([4821207, 1774269, 1805187], 2000, 3), ([8211298, 176962, 8116559], 1000, 9),
                            ([5, 7], 35, 1)):
        coo = blco.synth_uniform_host(dims, nnz, seed)
        idx, vals = oracle.synth_uniform(dims, nnz, seed)
        assert np.array_equal(coo.indices, idx)
        assert np.array_equal(coo.values, vals)


def test_exec_config(blco):  # proj/tests/test_exec.cpp:12-25, test_mttkrp.cpp:24-31
    blco.ExecConfig().validate()
    for bad in (dict(workgroup_size=0), dict(tile_size=64, workgroup_size=32), dict(tile_size=3),
                dict(num_threads=-1)):
        with pytest.raises(blco.FormatError):
            blco.ExecConfig(**bad).validate()
    cfg = blco.ExecConfig(num_compute_units=108)
    S = blco.Strategy
    assert blco.choose_strategy(24, cfg) == S.Hierarchical
    assert blco.choose_strategy(23_800_000, cfg) == S.Register
    assert blco.choose_strategy(108, cfg) == S.Register
    assert blco.choose_strategy(107, cfg) == S.Hierarchical


def test_merge_copies(blco):  # proj/tests/test_mttkrp.cpp:246-265
    rng = np.random.default_rng(71)
    a = rng.uniform(-1, 1, (3, 2))
    assert (blco.merge_copies([a, -a]) == 0).all()
    cs = [rng.uniform(-1, 1, (3, 2)) for _ in range(4)]
    assert np.array_equal(blco.merge_copies(cs), cs[0] + cs[1] + cs[2] + cs[3])
    assert np.array_equal(blco.merge_copies([a]), a)
    with pytest.raises(blco.FormatError):
        blco.merge_copies([a, np.zeros((2, 2))])


def test_container_stream_hooks_match_reference_bytes(blco, reflib):
    """blco_container_write_header/_block (the C++ serialize_blco path) write
    the reference's serialize_blco bytes (blco_format.cpp:149-166), and
    blco_container_read_header / _checked_layout parse them back
    (:173-199); header-level errors keep the reference's messages.  No GPU:
    the per-element block checks are not reached."""
    import ctypes as C
    from paper_2201_12523_b200 import _lib as L
    dims = [40, 35, 30, 12]
    rng = np.random.default_rng(3)
    cells = rng.choice(40 * 35 * 30 * 12, size=500, replace=False)
    idx = np.array(np.unravel_index(cells, dims[::-1])[::-1], np.uint64)
    vals = rng.uniform(-1, 1, 500)
    rt = reflib.build(dims, idx, vals, 14, 64)
    want = rt.serialize()
    out = bytearray()
    wfn = L.WRITE_FN(lambda ctx, src, n: (out.extend(C.string_at(src, n)), n)[1])
    lay = blco.make_layout(dims, 14)
    keys, offs, bi, bv = rt.blocks()
    blocks = list(zip(keys, offs[:-1], offs[1:]))
    assert L.lib.blco_container_write_header(wfn, None, C.byref(lay._c), 64, len(blocks)) == 0
    for key, lo, hi in blocks:
        bidx, bvals = np.ascontiguousarray(bi[lo:hi]), np.ascontiguousarray(bv[lo:hi])
        assert L.lib.blco_container_write_block(wfn, None, int(key), bidx.size, bidx.ctypes.data,
                                                bvals.ctypes.data) == 0
    assert bytes(out) == want
    pos = [0]

    def reader(data):
        def fn(ctx, dst, n):
            k = min(n, len(data) - pos[0])
            C.memmove(dst, data[pos[0]:pos[0] + k], k)
            pos[0] += k
            return k
        return L.READ_FN(fn)

    h = L.ContainerHeader()
    rfn = reader(want)
    assert L.lib.blco_container_read_header(rfn, None, C.byref(h)) == 0
    assert (h.version, h.order, h.target_bits, h.max_nnz_per_block, h.block_count) == (1, 4, 14, 64, len(blocks))
    assert list(h.dims[:4]) == dims and list(h.mode_bits[:4]) == list(lay.mode_bits)
    c = L.Layout()
    assert L.lib.blco_container_checked_layout(C.byref(h), C.byref(c)) == 0
    assert c.total_bits == lay.total_bits and c.stripped_bits == lay.stripped_bits
    h.mode_bits[1] += 1
    assert L.lib.blco_container_checked_layout(C.byref(h), C.byref(c)) == L.EFORMAT
    assert b"mode bit widths" in L.lib.blco_last_error()
    for bad, msg in ((b"XLCO" + want[4:], b"bad magic"), (want[:4] + b"\x02\x00" + want[6:], b"version 2"),
                     (want[:9], b"truncated payload")):
        pos[0] = 0
        st = L.lib.blco_container_read_header(reader(bad), None, C.byref(h))
        assert st != 0 and msg in L.lib.blco_last_error(), (msg, L.lib.blco_last_error())



def test_panel_plan(blco, monkeypatch):
    """The register kernel's dispatch order (mttkrp.cu panel_plan, host
    logic): ALTO order while the factors fit in L2; beyond it, panels of the
    target mode x the second-longest non-target mode (the longest streams),
    2 * 2^b rows within BLCO_B200_PANEL_MB (32 MB) of L2; the knob's
    overrides and the fallbacks."""
    amazon = blco.make_layout([4821207, 1774269, 1805187])
    monkeypatch.delenv("BLCO_B200_PANEL", raising=False)
    monkeypatch.delenv("BLCO_B200_PANEL_MB", raising=False)
    assert blco.panel_plan(amazon, 0, 32) == (1, 16, 16)  # Z = mode 2 (1805187 > 1774269)
    assert blco.panel_plan(amazon, 2, 32) == (1, 16, 16)  # Z = mode 0
    assert blco.panel_plan(amazon, 1, 32) == (2, 16, 16)
    assert blco.panel_plan(amazon, 0, 16) == (1, 17, 17)  # 128-byte rows
    assert blco.panel_plan(amazon, 0, 32, 4) == (1, 17, 17)  # fp32 rows
    assert blco.panel_plan(blco.make_layout([12092, 9184, 28818]), 0, 32) is None  # NELL-2: L2-resident
    delicious = blco.make_layout([532924, 17262471, 2480308, 1443])
    assert blco.panel_plan(delicious, 1, 16) == (0, 17, 17)  # Z = mode 2, mode 3 stays in L2
    assert blco.panel_plan(delicious, 3, 16) == (2, 17, 17)  # Z = mode 1, Y = mode 2
    assert blco.panel_plan(blco.make_layout([5000, 6000]), 0, 32) is None  # order 2
    monkeypatch.setenv("BLCO_B200_PANEL_MB", "64")
    assert blco.panel_plan(amazon, 0, 32) == (1, 17, 17)
    monkeypatch.setenv("BLCO_B200_PANEL", "12,9")
    assert blco.panel_plan(amazon, 0, 32) == (1, 12, 9)
    monkeypatch.setenv("BLCO_B200_PANEL", "2,2")  # 2^36 panels: keep ALTO order
    assert blco.panel_plan(amazon, 0, 32) is None
    monkeypatch.setenv("BLCO_B200_PANEL", "0")
    assert blco.panel_plan(amazon, 0, 32) is None
    with pytest.raises(blco.FormatError):
        blco.panel_plan(amazon, 3, 32)
