"""B200-native BLCO sparse MTTKRP (arXiv 2201.12523).

Host mirror of the reference API (proj/include/blco) over libblco_b200.so,
whose CUDA kernels (sm_100a) do all the work.  See DESIGN.md.
"""
from .api import (  # noqa: F401
    BitLayout, BlcoBlock, BlcoHeader, BlcoTensor, BuildStats, CpAlsError, CpAlsOptions, CpModel, CudaError,
    DeviceBudget, DeviceTensor, Error, ExecConfig, FactorMatrices, FileBlockSource, FormatError, IoError,
    AllModesReport, MttkrpStats, SparseTensorCoo, SplitIndex, Strategy, StreamReport, VerifyError, build_blco,
    choose_strategy, compute_batch_table, cp_als, delinearize, device_count, encode_coords,
    factors_random_device, fit, interleaved_remainder, kernel_launch_count, linearize, release_thread_caches,
    load_blco, make_layout, merge_copies, mttkrp, mttkrp_all_modes, mttkrp_f32, panel_plan, partition, read_blco_header,
    save_blco,
    split_block_key, stream_mttkrp, stream_mttkrp_all_modes,
    synth_draws_host, synth_uniform_host, throughput_report, Communicator, MultiDeviceTensor, MultiReport,
    nccl_version)
