"""ctypes access to the CPU checkers -- TEST INFRASTRUCTURE ONLY.

  Oracle  : oracle/liboracle.so, the plain-C restatement (blco_oracle.c).
  RefLib  : oracle/_ref/libblco_ref.so, the unmodified reference library
            compiled from /root/reference/proj/src by oracle/Makefile.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
--impl reference arm) import this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libblco_ref.so"

MAXO, MAXB = 32, 128


class OrcLayout(C.Structure):
    _fields_ = [
        ("order", C.c_int), ("total_bits", C.c_int), ("target_bits", C.c_int),
        ("stripped_bits", C.c_int), ("dims", C.c_uint64 * MAXO), ("mode_bits", C.c_int * MAXO),
        ("rem_bits", C.c_int * MAXO), ("field_shift", C.c_int * MAXO),
        ("field_mask", C.c_uint64 * MAXO), ("imap_mode", C.c_int * MAXB),
        ("imap_bit", C.c_int * MAXB), ("mode_pos", (C.c_int * 64) * MAXO),
    ]


class OrcBlco(C.Structure):
    _fields_ = [("nblocks", C.c_uint64), ("keys", C.POINTER(C.c_uint64)),
                ("offsets", C.POINTER(C.c_uint64)), ("idx", C.POINTER(C.c_uint64)),
                ("vals", C.POINTER(C.c_double)), ("nnz", C.c_uint64)]


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _pu(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pp(arrs):
    return (C.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])


class OracleError(RuntimeError):
    pass


class Oracle:
    """The C restatement (oracle/blco_oracle.c)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(str(path))
        self.lib.orc_last_error.restype = C.c_char_p

    def _ck(self, st):
        if st != 0:
            raise OracleError(self.lib.orc_last_error().decode())

    def layout(self, dims, target_bits=64) -> OrcLayout:
        l = OrcLayout()
        d = _u64(dims)
        self._ck(self.lib.orc_make_layout(_pu(d), len(d), target_bits, C.byref(l)))
        return l

    def linearize(self, l, coords) -> int:
        c = _u64(coords)
        hi, lo = C.c_uint64(), C.c_uint64()
        self._ck(self.lib.orc_linearize(C.byref(l), _pu(c), C.byref(hi), C.byref(lo)))
        return (hi.value << 64) | lo.value

    def split(self, l, alto) -> tuple[int, int]:
        k, r = C.c_uint64(), C.c_uint64()
        self.lib.orc_split_block_key(C.byref(l), C.c_uint64(alto >> 64), C.c_uint64(alto & (2**64 - 1)),
                                     C.byref(k), C.byref(r))
        return k.value, r.value

    def encode(self, l, coords) -> tuple[int, int]:
        c = _u64(coords)
        k, r = C.c_uint64(), C.c_uint64()
        self._ck(self.lib.orc_encode_coords(C.byref(l), _pu(c), C.byref(k), C.byref(r)))
        return k.value, r.value

    def delinearize(self, l, reenc, key) -> list[int]:
        out = np.zeros(l.order, np.uint64)
        self.lib.orc_delinearize(C.byref(l), C.c_uint64(reenc), C.c_uint64(key), _pu(out))
        return [int(x) for x in out]

    def build(self, dims, idx, vals, target_bits=64, max_nnz=1 << 27):
        """-> (keys, offsets, idx, vals) numpy arrays."""
        l = self.layout(dims, target_bits)
        idx = _u64(idx).reshape(len(dims), -1)
        vals = _f64(vals)
        b = OrcBlco()
        self._ck(self.lib.orc_build_blco(C.byref(l), C.c_uint64(vals.size), _pu(idx), _pd(vals),
                                         C.c_uint64(max_nnz), C.byref(b)))
        try:
            nb, n = b.nblocks, b.nnz
            keys = np.ctypeslib.as_array(b.keys, (max(nb, 1),))[:nb].copy()
            offs = np.ctypeslib.as_array(b.offsets, (nb + 1,)).copy()
            ii = np.ctypeslib.as_array(b.idx, (max(n, 1),))[:n].copy()
            vv = np.ctypeslib.as_array(b.vals, (max(n, 1),))[:n].copy()
        finally:
            self.lib.orc_free_blco(C.byref(b))
        return keys, offs, ii, vv

    def batch_table(self, block_nnz, quota) -> np.ndarray:
        bn = _u64(block_nnz)
        n = self.lib.orc_batch_table(_pu(bn), C.c_uint64(bn.size), C.c_uint64(quota), None)
        out = np.zeros((n, 3), np.uint64)
        if n:
            self.lib.orc_batch_table(_pu(bn), C.c_uint64(bn.size), C.c_uint64(quota), _pu(out))
        return out

    def mttkrp_coo(self, dims, idx, vals, factors, mode) -> np.ndarray:
        idx = _u64(idx).reshape(len(dims), -1)
        vals = _f64(vals)
        fs = [_f64(a) for a in factors]
        rank = fs[0].shape[1]
        out = np.zeros((dims[mode], rank))
        self._ck(self.lib.orc_mttkrp_coo(len(dims), _pu(_u64(dims)), C.c_uint64(vals.size), _pu(idx),
                                         _pd(vals), _pp(fs), C.c_uint64(rank), mode, _pd(out)))
        return out

    def factors_random(self, dims, rank, seed) -> list[np.ndarray]:
        fs = [np.zeros((int(d), rank)) for d in dims]
        self.lib.orc_factors_random(_pu(_u64(dims)), len(dims), C.c_uint64(rank), C.c_uint64(seed), _pp(fs))
        return fs

    def synth_uniform(self, dims, nnz, seed):
        idx = np.zeros((len(dims), nnz), np.uint64)
        vals = np.zeros(nnz)
        self._ck(self.lib.orc_synth_uniform(len(dims), _pu(_u64(dims)), C.c_uint64(nnz),
                                            C.c_uint64(seed), _pu(idx), _pd(vals)))
        return idx, vals

    def rowsample_coo(self, dims, idx, vals, factors, rows):
        """Rows rows[m] of mttkrp_coo(COO, factors, m), every mode (one pass,
        bit-identical to mttkrp_coo's rows)."""
        idx = _u64(idx).reshape(len(dims), -1)
        vals = _f64(vals)
        fs = [_f64(a) for a in factors]
        rank = fs[0].shape[1]
        rows = [_u64(r) for r in rows]
        outs = [np.zeros((r.size, rank)) for r in rows]
        rp = (C.c_void_p * len(rows))(*[r.ctypes.data for r in rows])
        self._ck(self.lib.orc_rowsample_coo(len(dims), _pu(_u64(dims)), C.c_uint64(vals.size), _pu(idx), _pd(vals),
                                            _pp(fs), C.c_uint64(rank), _pu(_u64([r.size for r in rows])), rp,
                                            _pp(outs)))
        return outs

    def rowsample_uniform(self, dims, nnz, seed, factors, rows, threads=None):
        """Rows rows[m] of mttkrp_coo(T, factors, m), every mode m, of the
        uniform synthetic tensor T (streamed, never stored); bit-identical to
        the full oracle's rows.  Returns one (len(rows[m]), rank) array per mode."""
        import os
        fs = [_f64(a) for a in factors]
        rank = fs[0].shape[1]
        rows = [_u64(r) for r in rows]
        outs = [np.zeros((r.size, rank)) for r in rows]
        nrows = _u64([r.size for r in rows])
        rp = (C.c_void_p * len(rows))(*[r.ctypes.data for r in rows])
        self._ck(self.lib.orc_rowsample_uniform(len(dims), _pu(_u64(dims)), C.c_uint64(nnz), C.c_uint64(seed),
                                                _pp(fs), C.c_uint64(rank), _pu(nrows), rp, _pp(outs),
                                                int(threads or os.cpu_count() or 1)))
        return outs

    def census_uniform(self, dims, nnz, seed, target_bits=64, threads=None):
        """(multiset hash, per-key element counts) of the uniform synthetic
        tensor, streamed from the generator on all host threads."""
        import os
        l = self.layout(dims, target_bits)
        counts = np.zeros(1 << l.stripped_bits, np.uint64)
        h = C.c_uint64()
        self._ck(self.lib.orc_census_uniform(len(dims), _pu(_u64(dims)), C.c_uint64(nnz), C.c_uint64(seed),
                                             target_bits, threads or os.cpu_count() or 1, C.byref(h), _pu(counts)))
        return int(h.value), counts

    def solve_normal(self, m, v):
        """dense_kernels.cpp:68-92 (Tikhonov escalation included); raises
        OracleError when V stays singular after the maximal shift."""
        a = np.array(m, np.float64, copy=True, order="C")
        v = np.ascontiguousarray(v, np.float64)
        self._ck(self.lib.orc_solve_normal(_pd(a), C.c_uint64(a.shape[0]), _pd(v), C.c_uint64(v.shape[0])))
        return a

    def synth_draws(self, dims, nnz, seed, skew=1):
        idx = np.zeros((len(dims), nnz), np.uint64)
        vals = np.zeros(nnz)
        self._ck(self.lib.orc_synth_draws(len(dims), _pu(_u64(dims)), C.c_uint64(nnz), C.c_uint64(seed),
                                          skew, _pu(idx), _pd(vals)))
        return idx, vals

    def alto_lo(self, dims, idx) -> np.ndarray:
        """Low ALTO word of every element (layouts of <= 64 bits)."""
        l = self.layout(dims, 64)
        idx = _u64(idx).reshape(len(dims), -1)
        out = np.zeros(idx.shape[1], np.uint64)
        self._ck(self.lib.orc_alto_lo_batch(C.byref(l), C.c_uint64(out.size), _pu(idx), _pu(out)))
        return out

    def cp_als(self, dims, keys, offsets, idx, vals, rank, max_iters, tol, seed, target_bits=64):
        l = self.layout(dims, target_bits)
        keys, offsets, idx, vals = _u64(keys), _u64(offsets), _u64(idx), _f64(vals)
        b = OrcBlco(keys.size, _pu(keys), _pu(offsets), _pu(idx), _pd(vals), idx.size)
        fs = [np.zeros((int(d), rank)) for d in dims]
        lam = np.zeros(rank)
        fit = np.zeros(max(1, max_iters))
        it = self.lib.orc_cp_als(C.byref(l), C.byref(b), C.c_uint64(rank), max_iters, C.c_double(tol),
                                 C.c_uint64(seed), _pp(fs), _pd(lam), _pd(fit))
        if it < 0:
            raise OracleError(self.lib.orc_last_error().decode())
        return fs, lam, fit[:it].copy()


class RefLib:
    """The unmodified reference library (oracle/_ref/libblco_ref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = C.CDLL(str(path))
        self.lib.ref_last_error.restype = C.c_char_p
        self.lib.ref_blco_nblocks.restype = C.c_uint64
        self.lib.ref_blco_batch.restype = C.c_uint64
        self.lib.ref_blco_free.argtypes = [C.c_void_p]
        self.lib.ref_blco_nblocks.argtypes = [C.c_void_p]
        self.lib.ref_blco_batch.argtypes = [C.c_void_p, C.c_void_p]
        self.lib.ref_blco_block.argtypes = [C.c_void_p, C.c_uint64] + [C.c_void_p] * 4

    def _ck(self, st):
        if st != 0:
            raise OracleError(f"[{st}] " + self.lib.ref_last_error().decode())

    def layout(self, dims, target_bits=64) -> dict:
        d = _u64(dims)
        n = len(d)
        out = np.zeros(2 + 3 * n + 2 * 128, np.int32)
        mask = np.zeros(n, np.uint64)
        self._ck(self.lib.ref_layout(_pu(d), n, target_bits, out.ctypes.data_as(C.POINTER(C.c_int)), _pu(mask)))
        total, stripped = int(out[0]), int(out[1])
        o = out[2:]
        return dict(total_bits=total, stripped_bits=stripped, mode_bits=o[:n].tolist(),
                    rem_bits=o[n:2 * n].tolist(), field_shift=o[2 * n:3 * n].tolist(),
                    imap_mode=o[3 * n:3 * n + total].tolist(),
                    imap_bit=o[3 * n + total:3 * n + 2 * total].tolist(),
                    field_mask=[int(x) for x in mask])

    def encode(self, dims, target_bits, coords) -> list[int]:
        out = np.zeros(6, np.uint64)
        self._ck(self.lib.ref_encode(_pu(_u64(dims)), len(dims), target_bits, _pu(_u64(coords)), _pu(out)))
        return [int(x) for x in out]

    def build(self, dims, idx, vals, target_bits=64, max_nnz=1 << 27, stage_seconds=None):
        idx = _u64(idx).reshape(len(dims), -1)
        vals = _f64(vals)
        h = C.c_void_p()
        st = np.zeros(4)
        self._ck(self.lib.ref_build_blco(len(dims), _pu(_u64(dims)), C.c_uint64(vals.size), _pu(idx),
                                         _pd(vals), target_bits, C.c_uint64(max_nnz), C.byref(h), _pd(st)))
        if stage_seconds is not None:
            stage_seconds[:] = st
        return RefTensor(self, h)

    def from_blocks(self, dims, target_bits, max_nnz, keys, offsets, idx, vals):
        keys, offsets, idx, vals = _u64(keys), _u64(offsets), _u64(idx), _f64(vals)
        h = C.c_void_p()
        self._ck(self.lib.ref_blco_from_blocks(len(dims), _pu(_u64(dims)), target_bits, C.c_uint64(max_nnz),
                                               C.c_uint64(keys.size), _pu(keys), _pu(offsets), _pu(idx),
                                               _pd(vals), C.byref(h)))
        return RefTensor(self, h)

    def mttkrp_coo(self, dims, idx, vals, factors, mode):
        idx = _u64(idx).reshape(len(dims), -1)
        vals = _f64(vals)
        fs = [_f64(a) for a in factors]
        out = np.zeros((dims[mode], fs[0].shape[1]))
        self._ck(self.lib.ref_mttkrp_coo(len(dims), _pu(_u64(dims)), C.c_uint64(vals.size), _pu(idx),
                                         _pd(vals), _pp(fs), C.c_uint64(fs[0].shape[1]), mode, _pd(out)))
        return out

    def factors_random(self, dims, rank, seed):
        fs = [np.zeros((int(d), rank)) for d in dims]
        self._ck(self.lib.ref_factors_random(_pu(_u64(dims)), len(dims), C.c_uint64(rank),
                                             C.c_uint64(seed), _pp(fs)))
        return fs


def cfg_array(workgroup_size=128, tile_size=32, coarsening=4, num_compute_units=108,
              num_factor_copies=1, stash_slots=32, deterministic=False, num_threads=0):
    return np.array([workgroup_size, tile_size, coarsening, num_compute_units, num_factor_copies,
                     stash_slots, int(deterministic), num_threads], np.int32)


class RefTensor:
    def __init__(self, ref: RefLib, h: C.c_void_p):
        self.ref, self.h = ref, h

    def __del__(self):
        if self.h:
            self.ref.lib.ref_blco_free(self.h)
            self.h = None

    def blocks(self):
        """-> (keys, offsets, idx, vals) block-concatenated numpy arrays."""
        lib = self.ref.lib
        nb = lib.ref_blco_nblocks(self.h)
        keys, offs, ii, vv = [], [0], [], []
        for b in range(nb):
            k, n = C.c_uint64(), C.c_uint64()
            pi, pv = C.c_void_p(), C.c_void_p()
            lib.ref_blco_block(self.h, b, C.byref(k), C.byref(n), C.byref(pi), C.byref(pv))
            keys.append(k.value)
            offs.append(offs[-1] + n.value)
            if n.value:
                ii.append(np.ctypeslib.as_array(C.cast(pi, C.POINTER(C.c_uint64)), (n.value,)).copy())
                vv.append(np.ctypeslib.as_array(C.cast(pv, C.POINTER(C.c_double)), (n.value,)).copy())
        cat = lambda xs, dt: np.concatenate(xs) if xs else np.zeros(0, dt)  # noqa: E731
        return _u64(keys), _u64(offs), cat(ii, np.uint64), cat(vv, np.float64)

    def serialize(self) -> bytes:
        """serialize_blco of the reference tensor."""
        lib = self.ref.lib
        lib.ref_serialize.restype = C.c_uint64
        lib.ref_serialize.argtypes = [C.c_void_p, C.c_char_p, C.c_uint64]
        cap = 64 + 16 * (1 << 20)
        while True:
            buf = C.create_string_buffer(cap)
            n = lib.ref_serialize(self.h, buf, cap)
            if n:
                return buf.raw[:n]
            cap *= 4

    def batch_table(self) -> np.ndarray:
        n = self.ref.lib.ref_blco_batch(self.h, None)
        out = np.zeros((n, 3), np.uint64)
        if n:
            self.ref.lib.ref_blco_batch(self.h, out.ctypes.data)
        return out

    def mttkrp(self, factors, mode, cfg=None, strategy=0):
        fs = [_f64(a) for a in factors]
        rows = fs[mode].shape[0]
        out = np.zeros((rows, fs[0].shape[1]))
        stats = np.zeros(6, np.uint64)
        c = cfg if cfg is not None else cfg_array()
        self.ref._ck(self.ref.lib.ref_mttkrp(self.h, _pp(fs), C.c_uint64(fs[0].shape[1]), mode,
                                             c.ctypes.data_as(C.POINTER(C.c_int)), strategy, _pd(out),
                                             _pu(stats)))
        return out, stats

    def stream_mttkrp(self, factors, mode, capacity, queues, reservation, cfg=None, strategy=0):
        fs = [_f64(a) for a in factors]
        out = np.zeros((fs[mode].shape[0], fs[0].shape[1]))
        rep = np.zeros(6)
        b = _u64([capacity, queues, reservation])
        c = cfg if cfg is not None else cfg_array()
        self.ref._ck(self.ref.lib.ref_stream_mttkrp(self.h, _pp(fs), C.c_uint64(fs[0].shape[1]), mode,
                                                    _pu(b), c.ctypes.data_as(C.POINTER(C.c_int)),
                                                    strategy, _pd(out), _pd(rep)))
        return out, rep

    def cp_als(self, dims, rank, max_iters, tol, seed, strategy=0, cfg=None):
        fs = [np.zeros((int(d), rank)) for d in dims]
        lam = np.zeros(rank)
        fit = np.zeros(max(1, max_iters))
        it = C.c_int()
        c = cfg if cfg is not None else cfg_array()
        self.ref._ck(self.ref.lib.ref_cp_als(self.h, C.c_uint64(rank), max_iters, C.c_double(tol),
                                             C.c_uint64(seed), strategy,
                                             c.ctypes.data_as(C.POINTER(C.c_int)), _pp(fs), _pd(lam),
                                             _pd(fit), C.byref(it)))
        return fs, lam, fit[: it.value].copy()
