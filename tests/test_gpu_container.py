"""`.blco` container: byte-compatible with the reference (serialize_blco,
proj/src/blco_format.cpp:149-255), element validation on the device,
corruption handling (proj/tests/test_blco.cpp:124-182) and the streaming
file source (proj/tests/test_streaming.cpp:81-103)."""
import struct

import numpy as np
import pytest

from conftest import rel_frobenius

pytestmark = pytest.mark.gpu

GI = np.array([[0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 3, 3],
               [0, 0, 2, 0, 0, 0, 3, 1, 1, 2, 2, 3],
               [0, 1, 2, 1, 2, 1, 3, 0, 1, 2, 3, 3]], np.uint64)
GV = np.arange(1, 13, dtype=np.float64)


def golden_tensor(gpu, z, meta, k):
    bm = meta["builds"][k]
    return gpu.BlcoTensor(gpu.make_layout(bm["dims"], bm["target"]), bm["max_nnz"], z[f"b{k}_keys"],
                          z[f"b{k}_offsets"], z[f"b{k}_idx"], z[f"b{k}_vals"])


def test_save_is_byte_identical_to_reference(gpu, golden, tmp_path):
    z, meta = golden
    for key in [k for k in z.files if k.endswith("_blco")]:
        k = int(key[1:-5])
        p = tmp_path / f"t{k}.blco"
        gpu.save_blco(golden_tensor(gpu, z, meta, k), p)
        assert p.read_bytes() == z[key].tobytes(), k


def test_load_reference_bytes(gpu, golden, tmp_path):
    z, meta = golden
    for key in [k for k in z.files if k.endswith("_blco")]:
        k = int(key[1:-5])
        p = tmp_path / f"r{k}.blco"
        p.write_bytes(z[key].tobytes())
        t = gpu.load_blco(p)
        assert t.structurally_equal(golden_tensor(gpu, z, meta, k))
        assert np.array_equal(t.batch_table, z[f"b{k}_batch"])
        h = gpu.read_blco_header(p)
        assert h.version == 1 and h.dims == meta["builds"][k]["dims"]
        assert h.block_count == z[f"b{k}_keys"].size


def test_roundtrip_and_resave(gpu, tmp_path):  # test_blco.cpp:124-135
    t = gpu.build_blco(gpu.SparseTensorCoo([4, 4, 4], GI, GV), 5, 6)
    p1, p2 = tmp_path / "a.blco", tmp_path / "b.blco"
    gpu.save_blco(t, p1)
    t2 = gpu.load_blco(p1)
    assert t.structurally_equal(t2)
    gpu.save_blco(t2, p2)
    assert p1.read_bytes() == p2.read_bytes()


@pytest.mark.parametrize("case", ["magic", "version", "truncated", "field_width", "order", "outside"])
def test_corruption_rejected(gpu, tmp_path, case):  # test_blco.cpp:137-162
    t = gpu.build_blco(gpu.SparseTensorCoo([4, 4, 4], GI, GV), 5, 6)
    p = tmp_path / "c.blco"
    gpu.save_blco(t, p)
    b = bytearray(p.read_bytes())
    header = 4 + 2 + 2 + 3 * 8 + 2 + 3 * 2 + 8 + 8
    first = header + 16  # first index of block 0
    if case == "magic":
        b[0] = ord("X")
        err, msg = gpu.FormatError, "blco: bad magic"
    elif case == "version":
        b[4] = 9
        err, msg = gpu.FormatError, "unsupported format version"
    elif case == "truncated":
        b = b[:-5]
        err, msg = gpu.IoError, "truncated"
    elif case == "field_width":
        b[first] = 0xFF
        err, msg = gpu.FormatError, "field width"
    elif case == "order":  # swap the first two indices of block 0
        i0, i1 = struct.unpack_from("<QQ", b, first)
        struct.pack_into("<QQ", b, first, i1, i0)
        err, msg = gpu.FormatError, "ascending ALTO order"
    else:  # index inside the 5-bit field whose mode-0 field decodes outside dims
        # dims (4,4,4) cannot decode outside; use a (3,4,4) tensor instead
        t3 = gpu.build_blco(gpu.SparseTensorCoo([3, 4, 4], np.array([[0, 2], [1, 3], [2, 3]], np.uint64),
                                                [1.0, 2.0]), 64)
        gpu.save_blco(t3, p)
        b = bytearray(p.read_bytes())
        first3 = 4 + 2 + 2 + 3 * 8 + 2 + 3 * 2 + 8 + 8 + 16
        struct.pack_into("<Q", b, first3 + 8, 3)  # mode-0 field 3 >= dim 3 (keeps ALTO order)
        err, msg = gpu.FormatError, "outside dims"
    p.write_bytes(bytes(b))
    with pytest.raises(err, match=msg):
        gpu.load_blco(p)


def test_header_of_huge_descriptor(gpu, tmp_path):  # test_blco.cpp:166-182
    p = tmp_path / "h.blco"
    dims = [1 << 20] * 3
    hdr = b"BLCO" + struct.pack("<HH", 1, 3) + struct.pack("<3Q", *dims) + struct.pack("<H", 64)
    hdr += struct.pack("<3H", 20, 20, 20) + struct.pack("<QQ", 1 << 27, 13)
    p.write_bytes(hdr)  # no payload at all
    h = gpu.read_blco_header(p)
    assert h.block_count == 13 and h.max_nnz_per_block == 1 << 27
    assert h.block_count * h.max_nnz_per_block > 1_700_000_000 and h.dims == dims


def test_file_source_streams(gpu, tmp_path):  # test_streaming.cpp:81-103
    coo = gpu.synth_uniform_host([40, 30, 20], 300, 97)
    t = gpu.build_blco(coo, 8, 40)
    p = tmp_path / "s.blco"
    gpu.save_blco(t, p)
    f = gpu.FactorMatrices.random([40, 30, 20], 4, 5)
    want = gpu.mttkrp(t, f, 2, strategy=gpu.Strategy.Register)
    fb = sum(a.size * 8 for a in f.factors) + 20 * 4 * 8
    budget = gpu.DeviceBudget(capacity_bytes=fb + 2 * 40 * 16, num_queues=2, reservation_bytes=40 * 16)
    got = gpu.stream_mttkrp(gpu.FileBlockSource(p), f, 2, budget, strategy=gpu.Strategy.Register)
    assert rel_frobenius(got, want) <= 1e-12


def test_cpp_file_source_matches(gpu):
    """FileBlockSource / save_blco / load_blco are also exercised through the
    C++ drop-in suite (tests/cpp/test_api.cpp, test_gpu_cxx.py)."""
    assert hasattr(gpu, "FileBlockSource")


@pytest.mark.parametrize("queues", [1, 3])
def test_native_file_stream_all_modes(gpu, oracle, tmp_path, queues):
    """blco_stream_mttkrp_file: the .blco blocks are read into pinned ring
    slots by a reader thread and cross the link once; every mode against
    the oracle, and a per-mode call through the same path."""
    dims = [60, 45, 70]
    coo = gpu.synth_uniform_host(dims, 5000, 11)
    t = gpu.build_blco(coo, 12, 300)
    assert t.keys.size > 4
    p = tmp_path / "n.blco"
    gpu.save_blco(t, p)
    f = gpu.FactorMatrices.random(dims, 8, 3)
    budget = gpu.DeviceBudget(capacity_bytes=1 << 26, num_queues=queues, reservation_bytes=300 * 16)
    rep = gpu.StreamReport()
    got = gpu.stream_mttkrp_all_modes(gpu.FileBlockSource(p), f, budget, report=rep)
    for m in range(3):
        assert rel_frobenius(got[m], oracle.mttkrp_coo(dims, coo.indices, coo.values, f.factors, m)) <= 1e-12
    assert rep.blocks == t.keys.size and rep.bytes_streamed == t.total_nnz * 16
    assert rep.block_queue == [i % queues for i in range(t.keys.size)]
    one = gpu.stream_mttkrp(gpu.FileBlockSource(p), f, 1, budget)
    assert rel_frobenius(one, got[1]) <= 1e-12


@pytest.mark.parametrize("case", ["truncated", "field_width", "order", "outside", "key_order"])
def test_native_file_stream_rejects_corruption(gpu, tmp_path, case):
    """read_blco_block's checks on the streamed path: record checks on the
    host reader, element checks on the device copy (same messages)."""
    dims = [3, 4, 4] if case == "outside" else [4, 4, 4]
    if case == "outside":
        t = gpu.build_blco(gpu.SparseTensorCoo(dims, np.array([[0, 2], [1, 3], [2, 3]], np.uint64), [1.0, 2.0]), 64)
    else:
        t = gpu.build_blco(gpu.SparseTensorCoo(dims, GI, GV), 5, 6)
    p = tmp_path / "c.blco"
    gpu.save_blco(t, p)
    b = bytearray(p.read_bytes())
    first = 4 + 2 + 2 + 3 * 8 + 2 + 3 * 2 + 8 + 8 + 16
    if case == "truncated":
        b = b[:-5]
        err, msg = gpu.IoError, "truncated"
    elif case == "field_width":
        b[first] = 0xFF
        err, msg = gpu.FormatError, "field width"
    elif case == "order":
        i0, i1 = struct.unpack_from("<QQ", b, first)
        struct.pack_into("<QQ", b, first, i1, i0)
        err, msg = gpu.FormatError, "ascending ALTO order"
    elif case == "outside":
        struct.pack_into("<Q", b, first + 8, 3)
        err, msg = gpu.FormatError, "outside dims"
    else:  # second block's key below the first's
        n0 = struct.unpack_from("<Q", b, first - 8)[0]
        second = first + 16 * n0
        struct.pack_into("<Q", b, first - 16, 1)  # block 0 key 1
        struct.pack_into("<Q", b, second, 0)      # block 1 key 0
        err, msg = gpu.FormatError, "ascending key order"
    p.write_bytes(bytes(b))
    f = gpu.FactorMatrices.random(dims, 2, 1)
    budget = gpu.DeviceBudget(capacity_bytes=1 << 24, num_queues=2, reservation_bytes=1 << 16)
    with pytest.raises(err, match=msg):
        gpu.stream_mttkrp(gpu.FileBlockSource(p), f, 0, budget)
