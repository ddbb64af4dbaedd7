"""ctypes binding of libblco_b200.so (the C ABI in include/blco_b200.h).

The library is built in-tree (``paper_2201_12523_b200/lib``) by
``__graft_entry__.build()`` / ``make -C paper_2201_12523_b200/csrc``.  There is
no fallback: if the shared object is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("BLCO_B200_LIB") or Path(__file__).resolve().parent / "lib" / "libblco_b200.so")

MAX_ORDER = 32
MAX_DEV_ORDER = 8
MAX_BITS = 128

OK, ERROR, EFORMAT, EIO, EVERIFY, ECUDA, ENCCL = 0, 1, 2, 3, 4, 5, 6


class Layout(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("total_bits", C.c_int32),
        ("target_bits", C.c_int32),
        ("stripped_bits", C.c_int32),
        ("dims", C.c_uint64 * MAX_ORDER),
        ("mode_bits", C.c_int32 * MAX_ORDER),
        ("rem_bits", C.c_int32 * MAX_ORDER),
        ("field_shift", C.c_int32 * MAX_ORDER),
        ("field_mask", C.c_uint64 * MAX_ORDER),
        ("imap_mode", C.c_uint8 * MAX_BITS),
        ("imap_bit", C.c_uint8 * MAX_BITS),
    ]


class ExecCfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "workgroup_size", "tile_size", "coarsening", "num_compute_units",
        "num_factor_copies", "stash_slots", "deterministic", "num_threads")]


class MttkrpStats(C.Structure):
    _fields_ = [
        ("strategy", C.c_int32),
        ("workgroups", C.c_uint64),
        ("segments", C.c_uint64),
        ("stash_flushes", C.c_uint64),
        ("commit_events", C.c_uint64),
        ("scalar_adds", C.c_uint64),
        ("kernel_ms", C.c_float),
        ("processing_cycles", C.c_uint64),
        ("computing_cycles", C.c_uint64),
        ("kernel", C.c_int32),
    ]


class BuildStats(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "sort_seconds", "block_seconds", "reencode_seconds", "batch_seconds")]


class BlockView(C.Structure):
    _fields_ = [("key", C.c_uint64), ("nnz", C.c_uint64),
                ("idx", C.c_void_p), ("vals", C.c_void_p), ("flags", C.c_uint32)]


BLOCK_STABLE = 1


class Budget(C.Structure):
    _fields_ = [("capacity_bytes", C.c_uint64), ("num_queues", C.c_int32),
                ("reservation_bytes", C.c_uint64),
                ("injected_transfer_latency_s", C.c_double)]


class StreamEvent(C.Structure):
    _fields_ = [("kind", C.c_int32), ("queue", C.c_int32), ("block", C.c_uint64),
                ("begin_s", C.c_double), ("end_s", C.c_double)]


class StreamReport(C.Structure):
    _fields_ = [
        ("blocks", C.c_uint64),
        ("bytes_streamed", C.c_uint64),
        ("total_seconds", C.c_double),
        ("transfer_busy_seconds", C.c_double),
        ("compute_busy_seconds", C.c_double),
        ("overall_gbps", C.c_double),
        ("compute_gbps", C.c_double),
        ("peak_resident_bytes", C.c_uint64),
        ("block_queue", C.POINTER(C.c_int32)),
        ("block_queue_capacity", C.c_uint64),
        ("timeline", C.POINTER(StreamEvent)),
        ("timeline_capacity", C.c_uint64),
        ("timeline_count", C.c_uint64),
    ]


class AllModesReport(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("chunks", C.c_uint64), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("launches", C.c_uint64)]


class CpAlsStats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("iterations_ms", C.c_double), ("mttkrp_ms", C.c_double)]


SOURCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(BlockView))

_P = C.c_void_p
_U64 = C.c_uint64
_I = C.c_int
_PU64 = C.POINTER(C.c_uint64)
_PD = C.POINTER(C.c_double)

# name -> (restype, argtypes); every symbol declared in include/blco_b200.h

class MultiReport(C.Structure):
    _fields_ = [("devices", C.c_int), ("device_ms", C.c_double), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64)]


REDUCE_ALL, REDUCE_SCATTER, COMM_ID_BYTES = 0, 1, 128


class ContainerHeader(C.Structure):
    _fields_ = [("version", C.c_uint16), ("order", C.c_uint16), ("target_bits", C.c_uint16),
                ("dims", C.c_uint64 * MAX_ORDER), ("mode_bits", C.c_uint16 * MAX_ORDER),
                ("max_nnz_per_block", C.c_uint64), ("block_count", C.c_uint64)]

# container stream hooks (blco_read_fn / blco_write_fn / blco_alloc_fn)
READ_FN = C.CFUNCTYPE(C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64)
WRITE_FN = C.CFUNCTYPE(C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint64)
ALLOC_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.POINTER(C.c_uint64)),
                       C.POINTER(C.POINTER(C.c_double)))

SIGNATURES = {
    "blco_last_error": (C.c_char_p, []),
    "blco_abi_version": (_I, []),
    "blco_make_layout": (_I, [_PU64, _I, _I, C.POINTER(Layout)]),
    "blco_linearize": (_I, [C.POINTER(Layout), _PU64, _PU64, _PU64]),
    "blco_split_block_key": (_I, [C.POINTER(Layout), _U64, _U64, _PU64, _PU64]),
    "blco_encode_coords": (_I, [C.POINTER(Layout), _PU64, _PU64, _PU64]),
    "blco_delinearize": (_I, [C.POINTER(Layout), _U64, _U64, _PU64]),
    "blco_interleaved_remainder": (_I, [C.POINTER(Layout), _U64, _PU64, _PU64]),
    "blco_key_upper": (_U64, [C.POINTER(Layout), _I, _U64]),
    "blco_batch_table": (_U64, [_PU64, _U64, _U64, _PU64]),
    "blco_exec_config_default": (None, [C.POINTER(ExecCfg)]),
    "blco_exec_config_validate": (_I, [C.POINTER(ExecCfg)]),
    "blco_choose_strategy": (_I, [_U64, C.POINTER(ExecCfg)]),
    "blco_panel_plan": (_I, [C.POINTER(Layout), _I, _U64, _U64, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "blco_build": (_I, [_PU64, _I, _U64, _PU64, _PD, _I, _U64, _I, C.POINTER(_P),
                        C.POINTER(BuildStats)]),
    "blco_build_synthetic": (_I, [_PU64, _I, _U64, _U64, _I, _U64, _I, C.POINTER(_P),
                                  C.POINTER(BuildStats)]),
    "blco_build_synthetic_draws": (_I, [_PU64, _I, _U64, _U64, _I, _I, _U64, _I, C.POINTER(_P),
                                        C.POINTER(BuildStats)]),
    "blco_synth_draws_host": (_I, [_I, _PU64, _U64, _U64, _I, _PU64, _PD]),
    "blco_synth_alto_chunk": (_I, [_PU64, _I, _U64, _U64, _U64, _U64, _I, _PU64, _PD, _PU64]),
    "blco_tensor_upload": (_I, [C.POINTER(Layout), _U64, _U64, _PU64, _PU64,
                                C.POINTER(_P), C.POINTER(_P), _I, C.POINTER(_P)]),
    "blco_tensor_slice": (_I, [_P, _U64, _U64, _I, C.POINTER(_P)]),
    "blco_tensor_info": (_I, [_P, C.POINTER(Layout), _PU64, _PU64, _PU64]),
    "blco_tensor_blocks": (_I, [_P, _PU64, _PU64]),
    "blco_tensor_download": (_I, [_P, _PU64, _PD]),
    "blco_tensor_device_ptrs": (_I, [_P, C.POINTER(_P), C.POINTER(_P)]),
    "blco_tensor_census": (_I, [_P, C.POINTER(C.c_uint64)]),
    "blco_tensor_free": (None, [_P]),
    "blco_save": (_I, [_P, C.c_char_p]),
    "blco_load": (_I, [C.c_char_p, _I, C.POINTER(_P)]),
    "blco_read_header": (_I, [C.c_char_p, C.POINTER(Layout), _PU64, _PU64, C.POINTER(C.c_uint16)]),
    "blco_validate_block": (_I, [C.POINTER(Layout), _U64, _U64, _PU64, _I]),
    "blco_validate_block_device": (_I, [C.POINTER(Layout), _U64, _U64, _P]),
    "blco_mttkrp": (_I, [_P, C.POINTER(_P), _U64, _I, _I, C.POINTER(ExecCfg), _PD,
                         C.POINTER(MttkrpStats)]),
    "blco_mttkrp_device": (_I, [_P, C.POINTER(_P), _U64, _I, _I, C.POINTER(ExecCfg), _P, _I,
                                _P, C.POINTER(MttkrpStats)]),
    "blco_mttkrp_all_host": (_I, [C.POINTER(Layout), _U64, _PU64, _PU64, C.POINTER(_P), C.POINTER(_P),
                                  C.POINTER(_P), _U64, _I, C.POINTER(ExecCfg), _U64, _I, C.POINTER(_P), _I,
                                  C.POINTER(AllModesReport)]),
    "blco_mttkrp_device_f32": (_I, [_P, C.POINTER(_P), _U64, _I, C.POINTER(ExecCfg), _P, _I, _P]),
    "blco_mttkrp_f32": (_I, [_P, C.POINTER(_P), _U64, _I, C.POINTER(ExecCfg), _P]),
    "blco_merge_copies": (_I, [C.POINTER(_P), _U64, _U64, _PD]),
    "blco_stream_mttkrp": (_I, [C.POINTER(Layout), _U64, SOURCE_FN, _P, C.POINTER(_P), _U64,
                                _I, C.POINTER(Budget), C.POINTER(ExecCfg), _I, _I, _PD,
                                C.POINTER(StreamReport)]),
    "blco_stream_mttkrp_all": (_I, [C.POINTER(Layout), _U64, SOURCE_FN, _P, C.POINTER(_P), _U64,
                                    C.POINTER(Budget), C.POINTER(ExecCfg), _I, _I, C.POINTER(_P), _I,
                                    C.POINTER(StreamReport)]),
    "blco_stream_mttkrp_file": (_I, [C.c_char_p, C.POINTER(_P), _U64, _I, C.POINTER(Budget), C.POINTER(ExecCfg),
                                     _I, _I, C.POINTER(_P), C.POINTER(StreamReport)]),
    "blco_set_error": (None, [_I, C.c_char_p]),
    "blco_host_alloc_pinned": (_P, [_U64]),
    "blco_host_free_pinned": (None, [_P]),
    "blco_host_register": (_I, [_P, _U64]),
    "blco_host_unregister": (_I, [_P]),
    "blco_cp_als": (_I, [_P, _U64, _I, C.c_double, _U64, _I, C.POINTER(ExecCfg),
                         C.POINTER(_P), _PD, _PD, C.POINTER(_I)]),
    "blco_cp_als_timed": (_I, [_P, _U64, _I, C.c_double, _U64, _I, C.POINTER(ExecCfg),
                               C.POINTER(_P), _PD, _PD, C.POINTER(_I), C.POINTER(CpAlsStats)]),
    "blco_fit": (_I, [_P, C.POINTER(_P), _PD, _U64, C.POINTER(ExecCfg), _PD]),
    "blco_tensor_norm_sq": (_I, [_P, _P, _P]),
    "blco_als_gram": (_I, [_P, _U64, _U64, _P, _P]),
    "blco_als_solve": (_I, [_P, _I, _I, _U64, _P, _U64, _P, _P, _P, _P]),
    "blco_als_normalize": (_I, [_P, _U64, _P, _U64, _P, _P, _P, _P, _P]),
    "blco_als_fit": (_I, [_P, _I, _U64, _P, _P, C.c_double, _P, _P]),
    "blco_factors_random": (_I, [_PU64, _I, _U64, _U64, C.POINTER(_P)]),
    "blco_factors_random_device": (_I, [_PU64, _I, _U64, _U64, C.POINTER(_P), _P]),
    "blco_synth_uniform_host": (_I, [_I, _PU64, _U64, _U64, _PU64, _PD]),
    "blco_partition": (_I, [_PU64, _U64, _U64, _I, _PU64, _PU64]),
    "blco_nccl_version": (_I, [C.POINTER(_I)]),
    "blco_comm_unique_id": (_I, [_P]),
    "blco_comm_init_rank": (_I, [_P, _I, _I, _I, C.POINTER(_P)]),
    "blco_comm_init_all": (_I, [C.POINTER(_I), _I, C.POINTER(_P)]),
    "blco_comm_free": (None, [_P]),
    "blco_dist_mttkrp_all": (_I, [_P, C.POINTER(_P), _U64, _P, _I, _I, C.POINTER(ExecCfg), C.POINTER(_P),
                                  C.POINTER(_P), _P]),
    "blco_multi_create": (_I, [_P, C.POINTER(_I), _I, C.POINTER(_P)]),
    "blco_multi_info": (_I, [_P, C.POINTER(_I), _PU64, _PU64]),
    "blco_multi_mttkrp_all": (_I, [_P, C.POINTER(_P), _U64, _I, _I, C.POINTER(ExecCfg), C.POINTER(_P),
                                   C.POINTER(MultiReport)]),
    "blco_multi_free": (None, [_P]),
    "blco_container_read_header": (_I, [READ_FN, _P, _P]),
    "blco_container_checked_layout": (_I, [_P, C.POINTER(Layout)]),
    "blco_container_read_block": (_I, [READ_FN, _P, C.POINTER(Layout), C.POINTER(_U64), C.POINTER(_U64), ALLOC_FN,
                                       _P, _I]),
    "blco_container_write_header": (_I, [WRITE_FN, _P, C.POINTER(Layout), _U64, _U64]),
    "blco_container_write_block": (_I, [WRITE_FN, _P, _U64, _U64, _P, _P]),
    "blco_mttkrp_all_device": (_I, [_P, C.POINTER(_P), _U64, _I, C.POINTER(ExecCfg), C.POINTER(_P), _I, _P,
                                    C.POINTER(_I)]),
    "blco_device_count": (_I, []),
    "blco_kernel_launch_count": (_U64, []),
    "blco_release_thread_caches": (_I, []),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback for the BLCO path)")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
