"""Python mirror of the reference's BLCO API over the C ABI.

Names, argument meaning and error behaviour follow proj/include/blco/*.hpp
(BitLayout / make_layout / build_blco / compute_batch_table / mttkrp /
stream_mttkrp / cp_als / fit, exceptions FormatError / IoError / Error) so the
parity tests read like the reference's own doctest cases.  All compute runs in
libblco_b200.so on the GPU; nothing here computes MTTKRP or builds BLCO.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Iterable, Sequence

import numpy as np

from . import _lib as L

lib = L.lib

# --------------------------------------------------------------------- errors


class Error(RuntimeError):
    """blco::Error (proj/include/blco/common.hpp:26-29)."""


class FormatError(Error):
    """blco::FormatError."""


class IoError(Error):
    """blco::IoError."""


class VerifyError(Error):
    """blco::VerifyError."""


class CudaError(Error):
    """A CUDA runtime failure inside libblco_b200."""


_ERRORS = {L.EFORMAT: FormatError, L.EIO: IoError, L.EVERIFY: VerifyError, L.ECUDA: CudaError}


def _check(status: int) -> None:
    if status != L.OK:
        msg = (lib.blco_last_error() or b"").decode()
        raise _ERRORS.get(status, Error)(msg)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _pu64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _pd(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ptr_array(arrays) -> C.Array:
    return (C.c_void_p * max(1, len(arrays)))(*[a.ctypes.data for a in arrays])


# --------------------------------------------------------------------- config


class Strategy(IntEnum):
    """blco::Strategy (proj/include/blco/mttkrp.hpp:9)."""
    Auto = 0
    Register = 1
    Hierarchical = 2


@dataclass
class ExecConfig:
    """blco::ExecConfig (proj/include/blco/exec.hpp:15-30), same defaults."""
    workgroup_size: int = 128
    tile_size: int = 32
    coarsening: int = 4
    num_compute_units: int = 108
    num_factor_copies: int = 1
    stash_slots: int = 32
    deterministic: bool = False
    num_threads: int = 0

    def _c(self) -> L.ExecCfg:
        return L.ExecCfg(self.workgroup_size, self.tile_size, self.coarsening,
                         self.num_compute_units, self.num_factor_copies, self.stash_slots,
                         int(self.deterministic), self.num_threads)

    def validate(self) -> None:
        c = self._c()
        _check(lib.blco_exec_config_validate(C.byref(c)))

    def workgroup_quota(self) -> int:
        return self.workgroup_size * self.coarsening


def choose_strategy(target_mode_length: int, config: ExecConfig | None = None) -> Strategy:
    c = (config or ExecConfig())._c()
    return Strategy(lib.blco_choose_strategy(int(target_mode_length), C.byref(c)))


@dataclass
class MttkrpStats:
    """blco::MttkrpStats (proj/include/blco/mttkrp.hpp:18-25) + device time."""
    strategy: Strategy = Strategy.Register
    workgroups: int = 0
    segments: int = 0
    stash_flushes: int = 0
    commit_events: int = 0
    scalar_adds: int = 0
    kernel_ms: float = 0.0
    processing_cycles: int = 0  # sorted register kernel: SM cycles, summed over CTAs
    computing_cycles: int = 0   # ... and over warps
    kernel: Strategy = Strategy.Register  # the kernel family that ran (Auto: register; `strategy` = reference label)


@dataclass
class BuildStats:
    sort_seconds: float = 0.0
    block_seconds: float = 0.0
    reencode_seconds: float = 0.0
    batch_seconds: float = 0.0


# --------------------------------------------------------------------- layout


class BitLayout:
    """blco::BitLayout (proj/include/blco/layout.hpp:19-51)."""

    def __init__(self, c: L.Layout):
        self._c = c

    @property
    def dims(self) -> list[int]:
        return list(self._c.dims[: self._c.order])

    def order(self) -> int:
        return self._c.order

    @property
    def mode_bits(self) -> list[int]:
        return list(self._c.mode_bits[: self._c.order])

    @property
    def total_bits(self) -> int:
        return self._c.total_bits

    @property
    def target_bits(self) -> int:
        return self._c.target_bits

    @property
    def stripped_bits(self) -> int:
        return self._c.stripped_bits

    @property
    def interleave_map(self) -> list[tuple[int, int]]:
        return [(self._c.imap_mode[p], self._c.imap_bit[p]) for p in range(self.total_bits)]

    @property
    def rem_bits(self) -> list[int]:
        return list(self._c.rem_bits[: self._c.order])

    @property
    def field_shift(self) -> list[int]:
        return list(self._c.field_shift[: self._c.order])

    @property
    def field_mask(self) -> list[int]:
        return list(self._c.field_mask[: self._c.order])

    def key_upper(self, mode: int, key: int) -> int:
        return lib.blco_key_upper(C.byref(self._c), mode, key)

    def block_base(self, key: int) -> list[int]:
        return [self.key_upper(m, key) << self.rem_bits[m] for m in range(self.order())]


def make_layout(dims: Sequence[int], target_bits: int = 64) -> BitLayout:
    d = _u64(dims)
    c = L.Layout()
    _check(lib.blco_make_layout(_pu64(d), len(d), target_bits, C.byref(c)))
    return BitLayout(c)


def panel_plan(layout: BitLayout, mode: int, rank: int, elem_bytes: int = 8) -> tuple[int, int, int] | None:
    """The register kernel's CTA dispatch order for `mode` (blco_panel_plan,
    B200 extension): (y_mode, bx, by) -- panels of 2^bx target rows x 2^by
    rows of y_mode, ALTO order inside -- or None for plain ALTO order."""
    y, bx, by = C.c_int(), C.c_int(), C.c_int()
    _check(lib.blco_panel_plan(C.byref(layout._c), mode, rank, elem_bytes, C.byref(y), C.byref(bx), C.byref(by)))
    return None if y.value < 0 else (y.value, bx.value, by.value)


def linearize(layout: BitLayout, coords: Sequence[int]) -> int:
    if len(coords) != layout.order():
        raise FormatError("linearize: coordinate count does not match order")
    c = _u64(coords)
    hi, lo = C.c_uint64(), C.c_uint64()
    _check(lib.blco_linearize(C.byref(layout._c), _pu64(c), C.byref(hi), C.byref(lo)))
    return (hi.value << 64) | lo.value


@dataclass
class SplitIndex:
    block_key: int = 0
    reencoded: int = 0


def split_block_key(layout: BitLayout, alto: int) -> SplitIndex:
    k, r = C.c_uint64(), C.c_uint64()
    _check(lib.blco_split_block_key(C.byref(layout._c), (alto >> 64) & (2**64 - 1),
                                    alto & (2**64 - 1), C.byref(k), C.byref(r)))
    return SplitIndex(k.value, r.value)


def encode_coords(layout: BitLayout, coords: Sequence[int]) -> SplitIndex:
    c = _u64(coords)
    k, r = C.c_uint64(), C.c_uint64()
    _check(lib.blco_encode_coords(C.byref(layout._c), _pu64(c), C.byref(k), C.byref(r)))
    return SplitIndex(k.value, r.value)


def delinearize(layout: BitLayout, reencoded: int, block_key: int) -> list[int]:
    out = np.zeros(layout.order(), dtype=np.uint64)
    _check(lib.blco_delinearize(C.byref(layout._c), reencoded, block_key, _pu64(out)))
    return [int(x) for x in out]


def interleaved_remainder(layout: BitLayout, reencoded: int) -> int:
    hi, lo = C.c_uint64(), C.c_uint64()
    _check(lib.blco_interleaved_remainder(C.byref(layout._c), reencoded, C.byref(hi), C.byref(lo)))
    return (hi.value << 64) | lo.value


# ---------------------------------------------------------------------- types


@dataclass
class SparseTensorCoo:
    """blco::SparseTensorCoo: dims, indices[mode][element] (uint64), values."""
    dims: list[int]
    indices: np.ndarray  # (order, nnz) uint64
    values: np.ndarray   # (nnz,) float64

    def __post_init__(self):
        self.indices = np.ascontiguousarray(np.asarray(self.indices, dtype=np.uint64).reshape(len(self.dims), -1))
        self.values = _f64(self.values)

    def order(self) -> int:
        return len(self.dims)

    def nnz(self) -> int:
        return int(self.values.size)


@dataclass
class FactorMatrices:
    """blco::FactorMatrices: one I_n x R row-major float64 matrix per mode."""
    rank: int
    factors: list[np.ndarray]

    @staticmethod
    def random(dims: Sequence[int], rank: int, seed: int) -> "FactorMatrices":
        """FactorMatrices::random (proj/src/types.cpp:118-130), SplitMix64."""
        fs = [np.empty((int(d), rank), dtype=np.float64) for d in dims]
        _check(lib.blco_factors_random(_pu64(_u64(dims)), len(dims), rank, seed, _ptr_array(fs)))
        return FactorMatrices(rank, fs)

    @staticmethod
    def ones(dims: Sequence[int], rank: int) -> "FactorMatrices":
        return FactorMatrices(rank, [np.ones((int(d), rank)) for d in dims])

    def order(self) -> int:
        return len(self.factors)

    def validate(self, dims: Sequence[int]) -> None:
        if len(self.factors) != len(dims):
            raise FormatError("factors: mode count does not match tensor order")
        for m, (a, d) in enumerate(zip(self.factors, dims)):
            if a.shape != (int(d), self.rank):
                raise FormatError(
                    f"factors: mode {m + 1} has shape {a.shape[0]}x{a.shape[1] if a.ndim > 1 else 0},"
                    f" expected {d}x{self.rank}")


# ---------------------------------------------------------------------- BLCO


@dataclass
class BlcoBlock:
    key: int
    linear_indices: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return int(self.values.size)


@dataclass
class BlcoTensor:
    """blco::BlcoTensor with the block payload kept block-concatenated."""
    layout: BitLayout
    max_nnz_per_block: int
    keys: np.ndarray      # (nblocks,) uint64
    offsets: np.ndarray   # (nblocks + 1,) uint64
    idx: np.ndarray       # (nnz,) uint64 re-encoded, ALTO order
    vals: np.ndarray      # (nnz,) float64
    batch_quota: int = 512
    batch_table: np.ndarray = field(default=None)  # (spans, 3) uint64
    _device: "DeviceTensor | None" = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.batch_table is None:
            self.batch_table = compute_batch_table(self, self.batch_quota)

    @property
    def total_nnz(self) -> int:
        return int(self.vals.size)

    def dims(self) -> list[int]:
        return self.layout.dims

    def order(self) -> int:
        return self.layout.order()

    @property
    def blocks(self) -> list[BlcoBlock]:
        o = self.offsets
        return [BlcoBlock(int(self.keys[b]), self.idx[o[b]:o[b + 1]], self.vals[o[b]:o[b + 1]])
                for b in range(self.keys.size)]

    def block_nnz(self) -> np.ndarray:
        return np.diff(self.offsets).astype(np.uint64)

    def structurally_equal(self, o: "BlcoTensor") -> bool:
        return (self.layout.dims == o.layout.dims and self.layout.target_bits == o.layout.target_bits
                and self.max_nnz_per_block == o.max_nnz_per_block
                and np.array_equal(self.keys, o.keys) and np.array_equal(self.offsets, o.offsets)
                and np.array_equal(self.idx, o.idx) and np.array_equal(self.vals, o.vals))

    def device(self, device: int = 0) -> "DeviceTensor":
        """The cached device copy of this tensor (uploaded on first use)."""
        if self._device is None or self._device.device_id != device:
            self._device = DeviceTensor.upload(self, device)
        return self._device

    @staticmethod
    def from_blocks(layout: BitLayout, blocks: Iterable[tuple[int, np.ndarray, np.ndarray]],
                    max_nnz_per_block: int = 1 << 27) -> "BlcoTensor":
        keys, idx, vals, offs = [], [], [], [0]
        for k, i, v in blocks:
            keys.append(k)
            idx.append(_u64(i))
            vals.append(_f64(v))
            offs.append(offs[-1] + len(v))
        return BlcoTensor(layout, max_nnz_per_block, _u64(keys), _u64(offs),
                          np.concatenate(idx) if idx else np.zeros(0, np.uint64),
                          np.concatenate(vals) if vals else np.zeros(0))


def compute_batch_table(t: BlcoTensor, elements_per_workgroup: int) -> np.ndarray:
    """compute_batch_table (proj/src/blco_format.cpp:136-147): (block, offset, count)."""
    if elements_per_workgroup < 1:
        raise FormatError("blco: elements_per_workgroup must be >= 1")
    bn = _u64(np.diff(t.offsets))
    n = lib.blco_batch_table(_pu64(bn), bn.size, elements_per_workgroup, None)
    out = np.zeros((n, 3), dtype=np.uint64)
    if n:
        lib.blco_batch_table(_pu64(bn), bn.size, elements_per_workgroup, _pu64(out))
    return out


class DeviceTensor:
    """A BLCO tensor resident in HBM (opaque blco_tensor handle)."""

    def __init__(self, handle: int, device: int):
        self._h = C.c_void_p(handle)
        self.device_id = device
        c = L.Layout()
        nb, nnz, mx = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib.blco_tensor_info(self._h, C.byref(c), C.byref(nb), C.byref(nnz), C.byref(mx)))
        self.layout = BitLayout(c)
        self.nblocks, self.nnz, self.max_nnz_per_block = nb.value, nnz.value, mx.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.blco_tensor_free(h)
            self._h = C.c_void_p(0)

    free = __del__

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @staticmethod
    def build(coo: SparseTensorCoo, target_bits: int = 64, max_nnz_per_block: int = 1 << 27,
              device: int = 0, stats: BuildStats | None = None) -> "DeviceTensor":
        h = C.c_void_p()
        bs = L.BuildStats()
        d = _u64(coo.dims)
        _check(lib.blco_build(_pu64(d), len(d), coo.nnz(), _pu64(coo.indices), _pd(coo.values),
                              target_bits, max_nnz_per_block, device, C.byref(h), C.byref(bs)))
        if stats is not None:
            stats.__dict__.update({k: getattr(bs, k) for k, _ in L.BuildStats._fields_})
        return DeviceTensor(h.value, device)

    @staticmethod
    def synthetic(dims: Sequence[int], nnz: int, seed: int, target_bits: int = 64,
                  max_nnz_per_block: int = 1 << 27, device: int = 0,
                  stats: BuildStats | None = None) -> "DeviceTensor":
        h = C.c_void_p()
        bs = L.BuildStats()
        d = _u64(dims)
        _check(lib.blco_build_synthetic(_pu64(d), len(d), nnz, seed, target_bits, max_nnz_per_block,
                                        device, C.byref(h), C.byref(bs)))
        if stats is not None:
            stats.__dict__.update({k: getattr(bs, k) for k, _ in L.BuildStats._fields_})
        return DeviceTensor(h.value, device)

    @staticmethod
    def synthetic_draws(dims: Sequence[int], nnz: int, seed: int, skew: int = 1, target_bits: int = 64,
                        max_nnz_per_block: int = 1 << 27, device: int = 0,
                        stats: BuildStats | None = None) -> "DeviceTensor":
        """Independent per-mode draws floor(I*u^skew), first nnz distinct tuples."""
        h = C.c_void_p()
        bs = L.BuildStats()
        d = _u64(dims)
        _check(lib.blco_build_synthetic_draws(_pu64(d), len(d), nnz, seed, skew, target_bits,
                                              max_nnz_per_block, device, C.byref(h), C.byref(bs)))
        if stats is not None:
            stats.__dict__.update({k: getattr(bs, k) for k, _ in L.BuildStats._fields_})
        return DeviceTensor(h.value, device)

    @staticmethod
    def upload(t: BlcoTensor, device: int = 0) -> "DeviceTensor":
        h = C.c_void_p()
        bn = _u64(np.diff(t.offsets))
        nb = int(bn.size)
        idx_ptrs = (C.c_void_p * max(1, nb))(*[t.idx.ctypes.data + 8 * int(t.offsets[b]) for b in range(nb)])
        val_ptrs = (C.c_void_p * max(1, nb))(*[t.vals.ctypes.data + 8 * int(t.offsets[b]) for b in range(nb)])
        keys = _u64(t.keys)
        _check(lib.blco_tensor_upload(C.byref(t.layout._c), t.max_nnz_per_block, nb, _pu64(keys),
                                      _pu64(bn), idx_ptrs, val_ptrs, device, C.byref(h)))
        return DeviceTensor(h.value, device)

    def slice(self, begin: int, end: int, device: int | None = None) -> "DeviceTensor":
        h = C.c_void_p()
        dev = self.device_id if device is None else device
        _check(lib.blco_tensor_slice(self._h, begin, end, dev, C.byref(h)))
        return DeviceTensor(h.value, dev)

    def block_nnz(self) -> np.ndarray:
        keys = np.zeros(max(1, self.nblocks), np.uint64)
        bn = np.zeros(max(1, self.nblocks), np.uint64)
        _check(lib.blco_tensor_blocks(self._h, _pu64(keys), _pu64(bn)))
        return bn[: self.nblocks]

    def validate_device(self) -> None:
        """read_blco_block's per-element checks (blco_format.cpp:201-227:
        fields within width, coordinates inside dims, strictly ascending ALTO
        order) on every block, run on the device; raises FormatError."""
        keys = np.zeros(max(1, self.nblocks), np.uint64)
        bn = np.zeros(max(1, self.nblocks), np.uint64)
        _check(lib.blco_tensor_blocks(self._h, _pu64(keys), _pu64(bn)))
        ip, vp = C.c_void_p(), C.c_void_p()
        _check(lib.blco_tensor_device_ptrs(self._h, C.byref(ip), C.byref(vp)))
        off = 0
        for b in range(self.nblocks):
            _check(lib.blco_validate_block_device(C.byref(self.layout._c), int(keys[b]), int(bn[b]),
                                                  C.c_void_p((ip.value or 0) + 8 * off)))
            off += int(bn[b])

    def census(self) -> int:
        """Order-free checksum of the (coordinates, value) multiset
        (blco_tensor_census), computed on the device."""
        h = C.c_uint64()
        _check(lib.blco_tensor_census(self._h, C.byref(h)))
        return int(h.value)

    def to_host(self) -> BlcoTensor:
        keys = np.zeros(max(1, self.nblocks), np.uint64)
        bn = np.zeros(max(1, self.nblocks), np.uint64)
        _check(lib.blco_tensor_blocks(self._h, _pu64(keys), _pu64(bn)))
        idx = np.zeros(self.nnz, np.uint64)
        vals = np.zeros(self.nnz, np.float64)
        _check(lib.blco_tensor_download(self._h, _pu64(idx), _pd(vals)))
        offs = np.zeros(self.nblocks + 1, np.uint64)
        offs[1:] = np.cumsum(bn[: self.nblocks])
        return BlcoTensor(self.layout, self.max_nnz_per_block, keys[: self.nblocks].copy(), offs,
                          idx, vals)

    def mttkrp_device_f32(self, d_factors: Sequence[int], rank: int, mode: int, d_out: int,
                          config: ExecConfig | None = None, accumulate: bool = False, stream: int = 0) -> None:
        """fp32 variant on device pointers (blco_mttkrp_device_f32), enqueued on `stream`."""
        c = (config or ExecConfig())._c()
        fp = (C.c_void_p * len(d_factors))(*d_factors)
        _check(lib.blco_mttkrp_device_f32(self._h, fp, rank, mode, C.byref(c), C.c_void_p(d_out),
                                          int(accumulate), C.c_void_p(stream)))

    def mttkrp_device(self, d_factors: Sequence[int], rank: int, mode: int, d_out: int,
                      strategy: Strategy = Strategy.Auto, config: ExecConfig | None = None,
                      accumulate: bool = False, stream: int = 0,
                      stats: MttkrpStats | None = None) -> None:
        """Enqueue MTTKRP on device pointers (no synchronisation unless stats)."""
        c = (config or ExecConfig())._c()
        fp = (C.c_void_p * len(d_factors))(*d_factors)
        st = L.MttkrpStats()
        _check(lib.blco_mttkrp_device(self._h, fp, rank, mode, int(strategy), C.byref(c),
                                      C.c_void_p(d_out), int(accumulate), C.c_void_p(stream),
                                      C.byref(st) if stats is not None else None))
        if stats is not None:
            _fill_stats(stats, st)

    def mttkrp_all_device(self, d_factors: Sequence[int], rank: int, d_outs: Sequence[int],
                          strategy: Strategy = Strategy.Auto, config: ExecConfig | None = None,
                          accumulate: bool = False, stream: int = 0) -> bool:
        """Every mode in one call on device pointers (blco_mttkrp_all_device);
        returns True when the fused all-mode kernel ran."""
        c = (config or ExecConfig())._c()
        fp = (C.c_void_p * len(d_factors))(*d_factors)
        op = (C.c_void_p * len(d_outs))(*d_outs)
        fused = C.c_int()
        _check(lib.blco_mttkrp_all_device(self._h, fp, rank, int(strategy), C.byref(c), op, int(accumulate),
                                          C.c_void_p(stream), C.byref(fused)))
        return bool(fused.value)


def mttkrp_f32(t, f, mode: int, config: ExecConfig | None = None) -> np.ndarray:
    """fp32 variant (blco_mttkrp_f32): factors as float32 (a FactorMatrices is
    converted), output dims[mode] x rank float32; 1e-5 relative Frobenius
    against the fp64 oracle."""
    config = config or ExecConfig()
    config.validate()
    dims = t.layout.dims
    fs = [np.ascontiguousarray(a, dtype=np.float32) for a in (f.factors if isinstance(f, FactorMatrices) else f)]
    rank = fs[0].shape[1]
    if len(fs) != len(dims) or any(a.shape != (d, rank) for a, d in zip(fs, dims)):
        raise FormatError("factors: shapes do not match the tensor")
    if mode < 0 or mode >= len(dims):
        raise FormatError(f"mttkrp: mode {mode + 1} out of range for order {len(dims)}")
    d = _as_device(t)
    out = np.zeros((dims[mode], rank), dtype=np.float32)
    c = config._c()
    _check(lib.blco_mttkrp_f32(d.handle, _ptr_array(fs), rank, mode, C.byref(c), C.c_void_p(out.ctypes.data)))
    return out


def _fill_stats(stats: MttkrpStats, st: L.MttkrpStats) -> None:
    stats.strategy = Strategy(st.strategy)
    stats.workgroups = st.workgroups
    stats.segments = st.segments
    stats.stash_flushes = st.stash_flushes
    stats.commit_events = st.commit_events
    stats.scalar_adds = st.scalar_adds
    stats.kernel_ms = st.kernel_ms
    stats.processing_cycles = st.processing_cycles
    stats.computing_cycles = st.computing_cycles
    stats.kernel = Strategy(st.kernel) if st.kernel else stats.strategy


def build_blco(coo: SparseTensorCoo, target_bits: int = 64, max_nnz_per_block: int = 1 << 27,
               stats: BuildStats | None = None, device: int = 0) -> BlcoTensor:
    """build_blco (proj/include/blco/blco_format.hpp:59-61), on the device."""
    dt = DeviceTensor.build(coo, target_bits, max_nnz_per_block, device, stats)
    t = dt.to_host()
    t._device = dt
    return t


# ----------------------------------------------------------------- container


@dataclass
class BlcoHeader:
    """blco::BlcoHeader (proj/include/blco/blco_format.hpp:77-87)."""
    version: int
    layout: BitLayout
    max_nnz_per_block: int
    block_count: int

    @property
    def dims(self) -> list[int]:
        return self.layout.dims


def save_blco(t, path) -> None:
    """save_blco (blco_format.hpp:72): the reference's byte format."""
    _check(lib.blco_save(_as_device(t).handle, str(path).encode()))


def load_blco(path, device: int = 0) -> BlcoTensor:
    """load_blco (blco_format.hpp:74): every element validated on the device."""
    h = C.c_void_p()
    _check(lib.blco_load(str(path).encode(), device, C.byref(h)))
    dt = DeviceTensor(h.value, device)
    t = dt.to_host()
    t._device = dt
    return t


def read_blco_header(path) -> BlcoHeader:
    """read_blco_header (blco_format.hpp:91): header only, payload untouched."""
    c = L.Layout()
    mx, nb, ver = C.c_uint64(), C.c_uint64(), C.c_uint16()
    _check(lib.blco_read_header(str(path).encode(), C.byref(c), C.byref(mx), C.byref(nb), C.byref(ver)))
    return BlcoHeader(ver.value, BitLayout(c), mx.value, nb.value)


class FileBlockSource:
    """blco::FileBlockSource (proj/include/blco/streaming.hpp:45-58): header up
    front, one block record per iteration, each validated on the device."""

    def __init__(self, path, device: int = 0):
        self.path = str(path)
        self.header = read_blco_header(path)
        self.layout = self.header.layout
        self.max_nnz_per_block = self.header.max_nnz_per_block
        self.device = device
        self._f = open(path, "rb")
        order = self.layout.order()
        self._f.seek(4 + 2 + 2 + 8 * order + 2 + 2 * order + 8 + 8)
        self._left = self.header.block_count

    def block_count(self) -> int:
        return self.header.block_count

    def __iter__(self):
        return self

    def __next__(self):
        if self._left == 0:
            self._f.close()
            raise StopIteration
        raw = self._f.read(16)
        if len(raw) < 16:
            raise IoError("blco: truncated payload")
        key, n = np.frombuffer(raw, np.uint64)
        key, n = int(key), int(n)
        if self.layout.stripped_bits < 64 and key >= (1 << self.layout.stripped_bits):
            raise FormatError("blco: block key out of range")
        idx = np.frombuffer(self._f.read(8 * n), np.uint64)
        vals = np.frombuffer(self._f.read(8 * n), np.float64)
        if idx.size < n or vals.size < n:
            raise IoError("blco: truncated payload")
        idx = np.ascontiguousarray(idx)
        _check(lib.blco_validate_block(C.byref(self.layout._c), key, n, _pu64(idx), self.device))
        self._left -= 1
        return key, idx, np.ascontiguousarray(vals)


# -------------------------------------------------------------------- MTTKRP


def _as_device(t) -> DeviceTensor:
    return t if isinstance(t, DeviceTensor) else t.device()


def mttkrp(t, f: FactorMatrices, mode: int, config: ExecConfig | None = None,
           strategy: Strategy = Strategy.Auto, stats: MttkrpStats | None = None) -> np.ndarray:
    """mttkrp (proj/include/blco/mttkrp.hpp:110-112): returns dims[mode] x rank."""
    config = config or ExecConfig()
    config.validate()
    dims = t.layout.dims
    f.validate(dims)
    if mode < 0 or mode >= len(dims):
        raise FormatError(f"mttkrp: mode {mode + 1} out of range for order {len(dims)}")
    d = _as_device(t)
    fs = [_f64(a) for a in f.factors]
    out = np.zeros((dims[mode], f.rank), dtype=np.float64)
    c = config._c()
    st = L.MttkrpStats()
    _check(lib.blco_mttkrp(d.handle, _ptr_array(fs), f.rank, mode, int(strategy), C.byref(c),
                           _pd(out), C.byref(st) if stats is not None else None))
    if stats is not None:
        _fill_stats(stats, st)
    return out


@dataclass
class AllModesReport:
    """blco_all_modes_report: device time and bytes of one mttkrp_all_modes call."""
    device_ms: float = 0.0
    chunks: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    launches: int = 0


def mttkrp_all_modes(t: BlcoTensor, f: FactorMatrices, config: ExecConfig | None = None,
                     strategy: Strategy = Strategy.Auto, outs: Sequence[np.ndarray] | None = None,
                     chunk_elems: int = 0, device: int = 0,
                     report: AllModesReport | None = None,
                     device_outs: Sequence[int] | None = None) -> list[np.ndarray] | None:
    """mttkrp(t, f, n) for every mode n of a HOST BlcoTensor in one call
    (blco_mttkrp_all_host): the payload is uploaded in chunks under the
    compute, every call.  `outs` (dims[n] x rank float64, C-contiguous; pinned
    memory makes the read-back asynchronous) are overwritten and returned."""
    config = config or ExecConfig()
    config.validate()
    dims = t.layout.dims
    f.validate(dims)
    if device_outs is not None:  # device pointers (dims[n] x rank doubles on `device`)
        if len(device_outs) != len(dims):
            raise FormatError("mttkrp: one output pointer per mode required")
        optr = (C.c_void_p * len(dims))(*[int(x) for x in device_outs])
    else:
        if outs is None:
            outs = [np.empty((d, f.rank), dtype=np.float64) for d in dims]
        for d, o in zip(dims, outs):
            if o.dtype != np.float64 or o.shape != (d, f.rank) or not o.flags.c_contiguous:
                raise FormatError("mttkrp: output arrays must be C-contiguous float64 dims[n] x rank")
        optr = _ptr_array(outs)
    bn = _u64(np.diff(t.offsets))
    nb = int(bn.size)
    idx_ptrs = (C.c_void_p * max(1, nb))(*[t.idx.ctypes.data + 8 * int(t.offsets[b]) for b in range(nb)])
    val_ptrs = (C.c_void_p * max(1, nb))(*[t.vals.ctypes.data + 8 * int(t.offsets[b]) for b in range(nb)])
    keys = _u64(t.keys)
    fs = [a if a.dtype == np.float64 and a.flags.c_contiguous else _f64(a) for a in f.factors]
    rep = L.AllModesReport()
    c = config._c()
    _check(lib.blco_mttkrp_all_host(C.byref(t.layout._c), nb, _pu64(keys), _pu64(bn), idx_ptrs, val_ptrs,
                                    _ptr_array(fs), f.rank, int(strategy), C.byref(c), chunk_elems, device,
                                    optr, int(device_outs is not None), C.byref(rep)))
    if report is not None:
        report.device_ms, report.chunks = rep.device_ms, rep.chunks
        report.h2d_bytes, report.d2h_bytes, report.launches = rep.h2d_bytes, rep.d2h_bytes, rep.launches
    return None if device_outs is not None else list(outs)


def merge_copies(copies: Sequence[np.ndarray]) -> np.ndarray:
    if not copies:
        raise FormatError("merge_copies: no copies")
    cs = [_f64(c) for c in copies]
    if any(c.shape != cs[0].shape for c in cs):
        raise FormatError("merge_copies: shape mismatch")
    out = np.empty_like(cs[0])
    _check(lib.blco_merge_copies(_ptr_array(cs), len(cs), cs[0].size, _pd(out)))
    return out


# ----------------------------------------------------------------- streaming


@dataclass
class DeviceBudget:
    """blco::DeviceBudget (proj/include/blco/streaming.hpp:12-17)."""
    capacity_bytes: int = 0
    num_queues: int = 4
    reservation_bytes: int = 0
    injected_transfer_latency_s: float = 0.0


@dataclass
class StreamEventRec:
    kind: str  # "transfer" | "compute"
    queue: int
    block: int
    begin_s: float
    end_s: float


@dataclass
class StreamReport:
    blocks: int = 0
    bytes_streamed: int = 0
    total_seconds: float = 0.0
    transfer_busy_seconds: float = 0.0
    compute_busy_seconds: float = 0.0
    overall_gbps: float = 0.0
    compute_gbps: float = 0.0
    peak_resident_bytes: int = 0
    timeline: list = field(default_factory=list)
    block_queue: list = field(default_factory=list)


def throughput_report(r: StreamReport) -> tuple[float, float]:
    return r.overall_gbps, r.compute_gbps


def stream_mttkrp(source, f: FactorMatrices, mode: int, budget: DeviceBudget,
                  config: ExecConfig | None = None, strategy: Strategy = Strategy.Auto,
                  report: StreamReport | None = None, device: int = 0,
                  layout: BitLayout | None = None, max_nnz_per_block: int | None = None,
                  block_count: int | None = None) -> np.ndarray:
    """stream_mttkrp (proj/include/blco/streaming.hpp:92-94).

    ``source`` is a host BlcoTensor (MemoryBlockSource) or an iterator of
    (key, idx, vals) blocks together with ``layout`` / ``max_nnz_per_block``.
    """
    return _stream(source, f, mode, budget, config, strategy, report, device, layout, max_nnz_per_block,
                   block_count)


def stream_mttkrp_all_modes(source, f: FactorMatrices, budget: DeviceBudget,
                            config: ExecConfig | None = None, strategy: Strategy = Strategy.Auto,
                            report: StreamReport | None = None, device: int = 0,
                            layout: BitLayout | None = None, max_nnz_per_block: int | None = None,
                            block_count: int | None = None,
                            device_outs: Sequence[int] | None = None) -> list[np.ndarray] | None:
    """B200 extension of stream_mttkrp: the blocks cross the host link once and
    every mode's MTTKRP runs on each resident block (blco_stream_mttkrp_all).
    Returns [M_0, ..., M_{N-1}], or writes them to `device_outs` (device
    pointers on `device`, for an NCCL reduction across ranks) and returns None."""
    return _stream(source, f, None, budget, config, strategy, report, device, layout, max_nnz_per_block,
                   block_count, device_outs)


def _fill_report(report, r, bq, tl, cap):
    for k in ("blocks", "bytes_streamed", "total_seconds", "transfer_busy_seconds",
              "compute_busy_seconds", "overall_gbps", "compute_gbps", "peak_resident_bytes"):
        setattr(report, k, getattr(r, k))
    n = min(r.blocks, cap)
    report.block_queue = [bq[i] for i in range(n)]
    report.timeline = [StreamEventRec("transfer" if tl[i].kind == 0 else "compute", tl[i].queue,
                                      tl[i].block, tl[i].begin_s, tl[i].end_s)
                       for i in range(min(r.timeline_count, 2 * cap))]


def _stream_file(source, f, mode, budget, config, strategy, report, device):
    """Unconsumed FileBlockSource: the native pinned-ring file reader with
    device-side element checks (blco_stream_mttkrp_file)."""
    layout = source.layout
    f.validate(layout.dims)
    if mode is not None and (mode < 0 or mode >= layout.order()):
        raise FormatError("stream: mode out of range")
    fs = [_f64(a) for a in f.factors]
    modes = range(layout.order()) if mode is None else [mode]
    outs = [np.zeros((layout.dims[m], f.rank)) for m in modes]
    cap = max(1, source.block_count())
    bq = (C.c_int32 * cap)()
    tl = (L.StreamEvent * (2 * cap))()
    r = L.StreamReport()
    r.block_queue, r.block_queue_capacity = C.cast(bq, C.POINTER(C.c_int32)), cap
    r.timeline, r.timeline_capacity = C.cast(tl, C.POINTER(L.StreamEvent)), 2 * cap
    b = L.Budget(budget.capacity_bytes, budget.num_queues, budget.reservation_bytes,
                 budget.injected_transfer_latency_s)
    c = config._c()
    _check(lib.blco_stream_mttkrp_file(source.path.encode(), _ptr_array(fs), f.rank, -1 if mode is None else mode,
                                       C.byref(b), C.byref(c), int(strategy), device, _ptr_array(outs), C.byref(r)))
    source._left = 0
    if report is not None:
        _fill_report(report, r, bq, tl, cap)
    return outs[0] if mode is not None else outs


def _stream(source, f, mode, budget, config, strategy, report, device, layout, max_nnz_per_block, block_count,
            device_outs=None):
    config = config or ExecConfig()
    config.validate()
    stable = isinstance(source, BlcoTensor)  # MemoryBlockSource: views outlive the call
    if stable:
        layout = source.layout
        max_nnz_per_block = source.max_nnz_per_block
        block_count = int(source.keys.size)
        it = iter(source.blocks)
    elif isinstance(source, FileBlockSource):
        if source._left == source.header.block_count and device_outs is None:
            return _stream_file(source, f, mode, budget, config, strategy, report, device)
        layout = source.layout
        max_nnz_per_block = source.max_nnz_per_block
        block_count = source.block_count()
        it = iter(source)
    else:
        it = iter(source)
    f.validate(layout.dims)
    if mode is not None and (mode < 0 or mode >= layout.order()):
        raise FormatError("stream: mode out of range")
    keep: list = []
    err: list = []

    def pull(_ctx, out):
        try:
            blk = next(it)
        except StopIteration:
            return 0
        except Exception as e:  # noqa: BLE001 - surfaced after the call
            err.append(e)
            lib.blco_set_error(L.ERROR, b"stream: block source failed")
            return -L.ERROR
        key, idx, vals = (blk.key, blk.linear_indices, blk.values) if isinstance(blk, BlcoBlock) else blk
        idx, vals = _u64(idx), _f64(vals)
        keep[:] = [idx, vals]
        out[0].key, out[0].nnz = int(key), int(vals.size)
        out[0].idx, out[0].vals = idx.ctypes.data, vals.ctypes.data
        out[0].flags = L.BLOCK_STABLE if stable else 0
        return 1

    cb = L.SOURCE_FN(pull)
    fs = [_f64(a) for a in f.factors]
    modes = range(layout.order()) if mode is None else [mode]
    outs = [] if device_outs is not None else [np.zeros((layout.dims[m], f.rank)) for m in modes]
    cap = max(1, block_count or 4096)
    bq = (C.c_int32 * cap)()
    tl = (L.StreamEvent * (2 * cap))()
    r = L.StreamReport()
    r.block_queue, r.block_queue_capacity = C.cast(bq, C.POINTER(C.c_int32)), cap
    r.timeline, r.timeline_capacity = C.cast(tl, C.POINTER(L.StreamEvent)), 2 * cap
    b = L.Budget(budget.capacity_bytes, budget.num_queues, budget.reservation_bytes,
                 budget.injected_transfer_latency_s)
    c = config._c()
    if mode is None:
        optr = ((C.c_void_p * len(modes))(*[int(x) for x in device_outs]) if device_outs is not None
                else _ptr_array(outs))
        status = lib.blco_stream_mttkrp_all(C.byref(layout._c), max_nnz_per_block or 0, cb, None,
                                            _ptr_array(fs), f.rank, C.byref(b), C.byref(c),
                                            int(strategy), device, optr, int(device_outs is not None),
                                            C.byref(r))
    else:
        status = lib.blco_stream_mttkrp(C.byref(layout._c), max_nnz_per_block or 0, cb, None,
                                        _ptr_array(fs), f.rank, mode, C.byref(b), C.byref(c),
                                        int(strategy), device, _pd(outs[0]), C.byref(r))
    if err:
        raise err[0]
    _check(status)
    if report is not None:
        for k in ("blocks", "bytes_streamed", "total_seconds", "transfer_busy_seconds",
                  "compute_busy_seconds", "overall_gbps", "compute_gbps", "peak_resident_bytes"):
            setattr(report, k, getattr(r, k))
        n = min(r.blocks, cap)
        report.block_queue = [bq[i] for i in range(n)]
        report.timeline = [StreamEventRec("transfer" if tl[i].kind == 0 else "compute", tl[i].queue,
                                          tl[i].block, tl[i].begin_s, tl[i].end_s)
                           for i in range(min(r.timeline_count, 2 * cap))]
    if device_outs is not None:
        return None
    return outs[0] if mode is not None else outs


# -------------------------------------------------------------------- CP-ALS


@dataclass
class CpAlsOptions:
    """blco::CpAlsOptions (proj/include/blco/cpals.hpp:9-15)."""
    rank: int = 32
    max_iters: int = 50
    tol: float = 1e-5
    seed: int = 0
    strategy: Strategy = Strategy.Auto


@dataclass
class CpModel:
    factors: FactorMatrices
    lambda_: np.ndarray
    fit_history: list[float]
    seed: int = 0

    def final_fit(self) -> float:
        return self.fit_history[-1] if self.fit_history else 0.0


class CpAlsError(Error):
    def __init__(self, msg: str, history: list[float]):
        super().__init__(msg)
        self.fit_history = history


def cp_als(t, opts: CpAlsOptions, config: ExecConfig | None = None) -> CpModel:
    """cp_als (proj/include/blco/cpals.hpp:38) with MTTKRP and dense steps on the GPU."""
    if opts.rank < 1:
        raise FormatError("cp_als: rank must be >= 1")
    if opts.max_iters < 0:
        raise FormatError("cp_als: max_iters must be >= 0")
    config = config or ExecConfig()
    config.validate()
    d = _as_device(t)
    dims = d.layout.dims
    fs = [np.empty((int(n), opts.rank)) for n in dims]
    lam = np.ones(opts.rank)
    fits = np.zeros(max(1, opts.max_iters))
    iters = C.c_int(0)
    c = config._c()
    st = L.CpAlsStats()
    status = lib.blco_cp_als_timed(d.handle, opts.rank, opts.max_iters, opts.tol, opts.seed,
                                   int(opts.strategy), C.byref(c), _ptr_array(fs), _pd(lam), _pd(fits),
                                   C.byref(iters), C.byref(st))
    hist = [float(x) for x in fits[: iters.value]]
    if status == L.ERROR and (lib.blco_last_error() or b"").startswith(b"cp_als: non-finite"):
        raise CpAlsError(lib.blco_last_error().decode(), hist)
    _check(status)
    model = CpModel(FactorMatrices(opts.rank, fs), lam, hist, opts.seed)
    model.device_ms = {"iterations": st.iterations, "iterations_ms": st.iterations_ms,
                       "mttkrp_ms": st.mttkrp_ms}
    return model


def fit(t, model: CpModel, config: ExecConfig | None = None) -> float:
    d = _as_device(t)
    model.factors.validate(d.layout.dims)
    if model.lambda_.size != model.factors.rank:
        raise FormatError("fit: lambda length does not match rank")
    fs = [_f64(a) for a in model.factors.factors]
    lam = _f64(model.lambda_)
    out = C.c_double()
    c = (config or ExecConfig())._c()
    _check(lib.blco_fit(d.handle, _ptr_array(fs), _pd(lam), model.factors.rank, C.byref(c),
                        C.byref(out)))
    return out.value


# -------------------------------------------------------------------- misc


def synth_uniform_host(dims: Sequence[int], nnz: int, seed: int) -> SparseTensorCoo:
    """Host restatement of the device generator (small sizes)."""
    d = _u64(dims)
    idx = np.zeros((len(d), nnz), np.uint64)
    vals = np.zeros(nnz, np.float64)
    _check(lib.blco_synth_uniform_host(len(d), _pu64(d), nnz, seed, _pu64(idx), _pd(vals)))
    return SparseTensorCoo(list(dims), idx, vals)


def synth_draws_host(dims: Sequence[int], ncand: int, seed: int, skew: int = 1):
    """The candidate stream of DeviceTensor.synthetic_draws (duplicates kept)."""
    d = _u64(dims)
    idx = np.zeros((len(d), ncand), np.uint64)
    vals = np.zeros(ncand, np.float64)
    _check(lib.blco_synth_draws_host(len(d), _pu64(d), ncand, seed, skew, _pu64(idx), _pd(vals)))
    return idx, vals


def synth_alto_chunk(dims: Sequence[int], chunk: int, nchunks: int, ncand: int, seed: int,
                     idx_out: np.ndarray, vals_out: np.ndarray, device: int = 0) -> int:
    """Chunk of an out-of-core uniform tensor, in BLCO order, into host arrays
    (ideally pinned, see pinned_empty).  Returns the element count."""
    n = C.c_uint64()
    _check(lib.blco_synth_alto_chunk(_pu64(_u64(dims)), len(dims), chunk, nchunks, ncand, seed, device,
                                     idx_out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     vals_out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n)))
    return n.value


def partition(block_nnz: Sequence[int], quota: int, nparts: int) -> list[tuple[int, int]]:
    """Contiguous nnz-balanced span ranges, one per GPU."""
    bn = _u64(block_nnz)
    b = np.zeros(nparts, np.uint64)
    e = np.zeros(nparts, np.uint64)
    _check(lib.blco_partition(_pu64(bn), bn.size, quota, nparts, _pu64(b), _pu64(e)))
    return [(int(x), int(y)) for x, y in zip(b, e)]


# ------------------------------------------------------------- multi-GPU
# The library's own multi-GPU partition (include/blco_b200.h "multi-GPU"):
# NCCL is driven inside libblco_b200.so, torch only moves the unique id.

REDUCE = {"allreduce": L.REDUCE_ALL, "reducescatter": L.REDUCE_SCATTER}


def nccl_version() -> int:
    """NCCL's version code as the library resolved it (raises when absent)."""
    v = C.c_int()
    _check(lib.blco_nccl_version(C.byref(v)))
    return int(v.value)


class Communicator:
    """One rank of a G-rank communicator (blco_comm): one process per GPU.
    Rank 0 calls `unique_id()`, the caller moves the bytes to every rank
    (e.g. torch.distributed.broadcast_object_list), each rank constructs
    Communicator(uid, nranks, rank, device)."""

    def __init__(self, uid: bytes | None, nranks: int, rank: int, device: int):
        self._h = C.c_void_p()
        buf = (C.c_uint8 * L.COMM_ID_BYTES).from_buffer_copy(uid or bytes(L.COMM_ID_BYTES))
        _check(lib.blco_comm_init_rank(buf, nranks, rank, device, C.byref(self._h)))
        self.nranks, self.rank, self.device = nranks, rank, device

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * L.COMM_ID_BYTES)()
        _check(lib.blco_comm_unique_id(buf))
        return bytes(buf)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.blco_comm_free(h)
            self._h = C.c_void_p(0)

    def mttkrp_all(self, local: "DeviceTensor", d_factors: Sequence[int], rank: int, d_outs: Sequence[int],
                   d_shards: Sequence[int] | None = None, reduce: str = "allreduce",
                   strategy: "Strategy" = None, config: "ExecConfig | None" = None, stream: int = 0) -> None:
        """blco_dist_mttkrp_all: this rank's partial M_n of every mode, reduced
        across the communicator per mode (enqueued on `stream`)."""
        c = (config or ExecConfig())._c()
        fp = (C.c_void_p * len(d_factors))(*d_factors)
        op = (C.c_void_p * len(d_outs))(*d_outs)
        sp = (C.c_void_p * len(d_outs))(*(d_shards or [0] * len(d_outs)))
        st = int(strategy if strategy is not None else Strategy.Auto)
        _check(lib.blco_dist_mttkrp_all(local.handle, fp, rank, self._h, REDUCE[reduce], st, C.byref(c), op, sp,
                                        C.c_void_p(stream)))


@dataclass
class MultiReport:
    devices: int = 0
    device_ms: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


class MultiDeviceTensor:
    """A tensor partitioned over several GPUs of this process, driven by one
    host thread (blco_multi): contiguous nnz-balanced span ranges, replicated
    factors, per-mode NCCL all-reduce or reduce-scatter of the partial M_n."""

    def __init__(self, t: "DeviceTensor", devices: Sequence[int]):
        self._h = C.c_void_p()
        devs = (C.c_int * len(devices))(*devices)
        _check(lib.blco_multi_create(t.handle, devs, len(devices), C.byref(self._h)))
        self.devices = list(devices)
        self.dims = list(t.layout.dims)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.blco_multi_free(h)
            self._h = C.c_void_p(0)

    def ranges(self) -> list[tuple[int, int]]:
        n = C.c_int()
        b = np.zeros(len(self.devices), np.uint64)
        e = np.zeros(len(self.devices), np.uint64)
        _check(lib.blco_multi_info(self._h, C.byref(n), _pu64(b), _pu64(e)))
        return [(int(x), int(y)) for x, y in zip(b, e)]

    def mttkrp_all_modes(self, f: "FactorMatrices", reduce: str = "allreduce", strategy: "Strategy" = None,
                         config: "ExecConfig | None" = None, report: MultiReport | None = None) -> list[np.ndarray]:
        f.validate(self.dims)
        fs = [_f64(a) for a in f.factors]
        outs = [np.zeros((d, f.rank)) for d in self.dims]
        c = (config or ExecConfig())._c()
        r = L.MultiReport()
        st = int(strategy if strategy is not None else Strategy.Auto)
        _check(lib.blco_multi_mttkrp_all(self._h, (C.c_void_p * len(fs))(*[a.ctypes.data for a in fs]), f.rank,
                                         REDUCE[reduce], st, C.byref(c),
                                         (C.c_void_p * len(outs))(*[o.ctypes.data for o in outs]), C.byref(r)))
        if report is not None:
            report.devices, report.device_ms = r.devices, r.device_ms
            report.h2d_bytes, report.d2h_bytes = r.h2d_bytes, r.d2h_bytes
        return outs


def factors_random_device(dims: Sequence[int], rank: int, seed: int, d_ptrs: Sequence[int],
                          stream: int = 0) -> None:
    ptrs = (C.c_void_p * len(d_ptrs))(*d_ptrs)
    _check(lib.blco_factors_random_device(_pu64(_u64(dims)), len(dims), rank, seed, ptrs,
                                          C.c_void_p(stream)))


class _Pinned:
    def __init__(self, nbytes: int):
        self.ptr = lib.blco_host_alloc_pinned(nbytes)
        if not self.ptr:
            _check(L.ECUDA)

    def __del__(self):
        if getattr(self, "ptr", None):
            lib.blco_host_free_pinned(C.c_void_p(self.ptr))
            self.ptr = None


def pinned_empty(n: int, dtype) -> np.ndarray:
    """A numpy array in page-locked host memory (full-speed async H2D)."""
    dtype = np.dtype(dtype)
    buf = _Pinned(max(1, n) * dtype.itemsize)
    raw = (C.c_char * (max(1, n) * dtype.itemsize)).from_address(buf.ptr)
    raw.owner = buf  # the ctypes view (arr.base) keeps the allocation alive
    return np.frombuffer(raw, dtype=dtype, count=n)


def device_count() -> int:
    return lib.blco_device_count()


def kernel_launch_count() -> int:
    return int(lib.blco_kernel_launch_count())


def release_thread_caches() -> None:
    """Frees this thread's cached device buffers (host pipeline, streaming,
    deterministic-mode and MTTKRP workspaces; blco_release_thread_caches)."""
    _check(lib.blco_release_thread_caches())
