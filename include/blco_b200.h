/*
 * blco_b200.h -- C ABI of libblco_b200.so, the B200-native BLCO MTTKRP path.
 *
 * The reference (proj/, a CPU C++20 library) has no C ABI: its boundary is the
 * link-level C++ API in the proj/include/blco headers.  This header is the plain-C
 * layer underneath our re-declaration of that C++ API (include/blco/,
 * implemented in paper_2201_12523_b200/csrc/cxx_api.cpp); every entry point
 * names the reference declaration it replaces.  Plain pointers and sizes only.
 *
 * Conventions
 *   - Every function returning int returns a blco_status; on failure
 *     blco_last_error() holds a thread-local message whose prefix matches the
 *     reference exception text (e.g. "blco: duplicate coordinate tuple").
 *   - Modes are 0-based (proj/include/blco/mttkrp.hpp:107-109).
 *   - Sparse coordinates are passed mode-major: idx[m * nnz + e].
 *   - Dense matrices are row-major doubles (proj/include/blco/types.hpp:12-28).
 *   - Device-side limits: dims[m] < 2^32 and order <= 8 for tensors that are
 *     built or multiplied on the GPU (a mode of 2^32 rows would need a factor
 *     matrix of >= 32 GiB per rank column); layouts stripped_bits <= 64.
 */
#ifndef BLCO_B200_H
#define BLCO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BLCO_MAX_ORDER 32     /* host-side layouts */
#define BLCO_MAX_DEV_ORDER 8  /* device kernels */
#define BLCO_MAX_BITS 128

typedef enum blco_status {
  BLCO_OK = 0,
  BLCO_ERROR = 1,   /* blco::Error */
  BLCO_EFORMAT = 2, /* blco::FormatError (proj/include/blco/common.hpp:31-34) */
  BLCO_EIO = 3,     /* blco::IoError */
  BLCO_EVERIFY = 4, /* blco::VerifyError */
  BLCO_ECUDA = 5,
  BLCO_ENCCL = 6
} blco_status;

typedef enum blco_strategy {
  BLCO_STRATEGY_AUTO = 0, /* proj/include/blco/mttkrp.hpp:9 (enum class Strategy) */
  BLCO_STRATEGY_REGISTER = 1,
  BLCO_STRATEGY_HIERARCHICAL = 2
} blco_strategy;

const char* blco_last_error(void);
int blco_abi_version(void);

/* ---------------------------------------------------------------- layout
 * Replaces blco::BitLayout / make_layout (proj/include/blco/layout.hpp:19-55,
 * proj/src/layout.cpp:15-69).  key_slices are implied: stripped position p
 * (p >= total - stripped) carries bit imap_bit[p] of mode imap_mode[p]. */
typedef struct blco_layout {
  int32_t order;
  int32_t total_bits;
  int32_t target_bits;
  int32_t stripped_bits;
  uint64_t dims[BLCO_MAX_ORDER];
  int32_t mode_bits[BLCO_MAX_ORDER];
  int32_t rem_bits[BLCO_MAX_ORDER];
  int32_t field_shift[BLCO_MAX_ORDER];
  uint64_t field_mask[BLCO_MAX_ORDER];
  uint8_t imap_mode[BLCO_MAX_BITS]; /* interleaved position -> mode */
  uint8_t imap_bit[BLCO_MAX_BITS];  /* interleaved position -> bit within mode */
} blco_layout;

/* make_layout (layout.hpp:55) */
int blco_make_layout(const uint64_t* dims, int order, int target_bits, blco_layout* out);
/* linearize (layout.hpp:58): 128-bit ALTO index as (hi, lo) */
int blco_linearize(const blco_layout* l, const uint64_t* coords, uint64_t* alto_hi,
                   uint64_t* alto_lo);
/* split_block_key (layout.hpp:66) */
int blco_split_block_key(const blco_layout* l, uint64_t alto_hi, uint64_t alto_lo,
                         uint64_t* key, uint64_t* reencoded);
/* encode_coords (layout.hpp:70) */
int blco_encode_coords(const blco_layout* l, const uint64_t* coords, uint64_t* key,
                       uint64_t* reencoded);
/* delinearize (layout.hpp:73-74) */
int blco_delinearize(const blco_layout* l, uint64_t reencoded, uint64_t key, uint64_t* coords);
/* interleaved_remainder (layout.hpp:78) */
int blco_interleaved_remainder(const blco_layout* l, uint64_t reencoded, uint64_t* hi,
                               uint64_t* lo);
/* BitLayout::key_upper / block_base (layout.hpp:42-50) */
uint64_t blco_key_upper(const blco_layout* l, int mode, uint64_t key);

/* compute_batch_table (proj/include/blco/blco_format.hpp:64-65): writes
 * (block, offset, count) triples into spans (NULL = count only). */
uint64_t blco_batch_table(const uint64_t* block_nnz, uint64_t nblocks, uint64_t quota,
                          uint64_t* spans);

/* -------------------------------------------------------------- config
 * Replaces blco::ExecConfig (proj/include/blco/exec.hpp:15-30); same fields in
 * the same order.  On the GPU, workgroup_size/tile_size/coarsening are hints
 * (DESIGN.md), num_compute_units feeds choose_strategy exactly as in
 * proj/src/mttkrp.cpp:17-21, num_factor_copies is honoured by the
 * hierarchical kernel, stash_slots is a lower bound on the shared-memory
 * stash, num_threads has no device meaning.  deterministic != 0 selects the
 * fixed-order kernels of determ.cu (bit-identical results run to run, and
 * across block splits of the same tensor; device-resident tensors only, the
 * streamed paths reject it, nnz < 2^32, rank <= 256). */
typedef struct blco_exec_config {
  int32_t workgroup_size;
  int32_t tile_size;
  int32_t coarsening;
  int32_t num_compute_units;
  int32_t num_factor_copies;
  int32_t stash_slots;
  int32_t deterministic;
  int32_t num_threads;
} blco_exec_config;

void blco_exec_config_default(blco_exec_config* cfg);
/* ExecConfig::validate (proj/src/exec.cpp:11-20) */
int blco_exec_config_validate(const blco_exec_config* cfg);
/* choose_strategy (proj/src/mttkrp.cpp:17-21) */
int blco_choose_strategy(uint64_t target_mode_length, const blco_exec_config* cfg);

/* MttkrpStats (proj/include/blco/mttkrp.hpp:18-25).  On the GPU a segment is
 * one run of equal target rows inside a 32-element warp tile;
 * commit_events counts per-lane RED.ADD.F64 commit lanes (segments x
 * committing lanes), scalar_adds counts committed scalars. */
typedef struct blco_mttkrp_stats {
  int32_t strategy;
  uint64_t workgroups;
  uint64_t segments;
  uint64_t stash_flushes;
  uint64_t commit_events;
  uint64_t scalar_adds;
  float kernel_ms; /* device time of the MTTKRP kernel(s), CUDA events */
  /* sorted register kernel only: SM cycles summed over CTAs in the
   * processing phase (load, decode, group by row) and over warps in the
   * computing phase (gather, multiply, commit) */
  uint64_t processing_cycles;
  uint64_t computing_cycles;
  /* the kernel family that ran (REGISTER / HIERARCHICAL).  Under AUTO,
   * `strategy` is the reference's choose_strategy label (mttkrp.cpp:17-21)
   * while the B200 runs the register kernel for every mode length (measured
   * faster everywhere) */
  int32_t kernel;
} blco_mttkrp_stats;

/* BuildStats (proj/include/blco/blco_format.hpp:49-54), device stage times */
typedef struct blco_build_stats {
  double sort_seconds;
  double block_seconds;
  double reencode_seconds;
  double batch_seconds;
} blco_build_stats;

/* ------------------------------------------------------- device tensor
 * A BLCO tensor resident in HBM: block-concatenated re-encoded indices (u64)
 * and values (f64) in ALTO order, per-block keys / offsets / decoded base
 * coordinates, and the CTA tile table the kernels consume. */
typedef struct blco_tensor blco_tensor;

/* build_blco (blco_format.hpp:59-61) on the device from a host COO.
 * Bit-exact with the reference: same blocks, keys, order, indices, values. */
int blco_build(const uint64_t* dims, int order, uint64_t nnz, const uint64_t* idx,
               const double* vals, int target_bits, uint64_t max_nnz_per_block, int device,
               blco_tensor** out, blco_build_stats* stats);

/* Same, from a seeded synthetic uniform COO generated on the device
 * (identical to blco_synth_uniform_host). */
int blco_build_synthetic(const uint64_t* dims, int order, uint64_t nnz, uint64_t seed,
                         int target_bits, uint64_t max_nnz_per_block, int device,
                         blco_tensor** out, blco_build_stats* stats);

/* Same, from independent per-mode draws (config 4, "skewed power-law"):
 * coordinate m of candidate j is floor(I_m * u^skew) (skew = 1: uniform), the
 * tensor keeps the first nnz distinct tuples in draw order.  Works for any
 * prod(dims) (Delicious-shaped layouts of 78 bits included). */
int blco_build_synthetic_draws(const uint64_t* dims, int order, uint64_t nnz, uint64_t seed,
                               int skew, int target_bits, uint64_t max_nnz_per_block, int device,
                               blco_tensor** out, blco_build_stats* stats);
/* The candidate stream of blco_build_synthetic_draws on the host: ncand
 * draws (duplicates included), idx mode-major, for oracle parity. */
int blco_synth_draws_host(int order, const uint64_t* dims, uint64_t ncand, uint64_t seed, int skew,
                          uint64_t* idx, double* vals);

/* Out-of-core generator (config 5): chunk `chunk` of `nchunks` equal ALTO
 * ranges of a layout with no stripped bits.  ncand uniform ALTO candidates in
 * the range; those decoding inside dims, deduplicated, are written in ALTO
 * order to host_idx (re-encoded) / host_vals (capacity >= ncand); *count gets
 * their number.  Concatenating chunks 0..nchunks-1 yields the BLCO element
 * order of one uniform random tensor (a single key run). */
int blco_synth_alto_chunk(const uint64_t* dims, int order, uint64_t chunk, uint64_t nchunks,
                          uint64_t ncand, uint64_t seed, int device, uint64_t* host_idx,
                          double* host_vals, uint64_t* count);

/* Upload host-resident blocks (a reference BlcoTensor's payload). */
int blco_tensor_upload(const blco_layout* layout, uint64_t max_nnz_per_block, uint64_t nblocks,
                       const uint64_t* keys, const uint64_t* block_nnz,
                       const uint64_t* const* idx, const double* const* vals, int device,
                       blco_tensor** out);

/* A new device tensor holding elements [elem_begin, elem_end) of t (block
 * boundaries and keys kept); the multi-GPU partition unit. */
int blco_tensor_slice(const blco_tensor* t, uint64_t elem_begin, uint64_t elem_end, int device,
                      blco_tensor** out);

int blco_tensor_info(const blco_tensor* t, blco_layout* layout, uint64_t* nblocks,
                     uint64_t* nnz, uint64_t* max_nnz_per_block);
int blco_tensor_blocks(const blco_tensor* t, uint64_t* keys, uint64_t* block_nnz);
int blco_tensor_download(const blco_tensor* t, uint64_t* idx, double* vals);
/* Order-free checksum of the element multiset (a checksum of checksums):
 * sum over elements of mix64(cell ^ mix64(bits(value))) mod 2^64, with
 * cell = sum_m c_m * prod_{k<m} dims[k] mod 2^64 and mix64 the SplitMix64
 * finaliser.  Equal for any two tensors holding the same (coordinates,
 * value) pairs, whatever their blocking; used to pin full-size device builds
 * against the generator's stream (oracle orc_census_*). */
int blco_tensor_census(const blco_tensor* t, uint64_t* hash);
/* Device pointers (idx, vals) of the resident payload. */
int blco_tensor_device_ptrs(const blco_tensor* t, const uint64_t** idx, const double** vals);
void blco_tensor_free(blco_tensor* t);

/* ------------------------------------------------------ .blco container
 * Byte-compatible with the reference container (blco_format.hpp:67-93,
 * blco_format.cpp:149-255).  Per-element validation of read_blco_block
 * (field width, coordinates inside dims, ascending ALTO order; :201-227) runs
 * on the device.  Messages match the reference ("blco: bad magic", ...). */
int blco_save(const blco_tensor* t, const char* path);                   /* save_blco */
int blco_load(const char* path, int device, blco_tensor** out);          /* load_blco */
int blco_read_header(const char* path, blco_layout* layout, uint64_t* max_nnz_per_block,
                     uint64_t* block_count, uint16_t* version);            /* read_blco_header */
/* The container on a caller-supplied byte stream (the C++ API's
 * std::istream / std::ostream overloads: serialize_blco, read_blco_header,
 * read_blco_block, deserialize_blco; blco_format.hpp:67-93).  A read hook
 * returns the bytes produced (fewer only at end of stream), a write hook the
 * bytes consumed; a short count raises "blco: truncated payload" /
 * "blco: write failed" (BLCO_EIO). */
typedef uint64_t (*blco_read_fn)(void* ctx, void* dst, uint64_t bytes);
typedef uint64_t (*blco_write_fn)(void* ctx, const void* src, uint64_t bytes);
/* caller storage for one block's payload: *idx and *vals must hold nnz
 * elements each on return (return 0; non-zero = allocation failed) */
typedef int (*blco_alloc_fn)(void* ctx, uint64_t nnz, uint64_t** idx, double** vals);

typedef struct blco_container_header {
  uint16_t version;
  uint16_t order;
  uint16_t target_bits;
  uint64_t dims[BLCO_MAX_ORDER];
  uint16_t mode_bits[BLCO_MAX_ORDER];
  uint64_t max_nnz_per_block;
  uint64_t block_count;
} blco_container_header;

/* read_blco_header (blco_format.cpp:173-191): magic, version, raw fields */
int blco_container_read_header(blco_read_fn fn, void* ctx, blco_container_header* out);
/* BlcoHeader::make_layout_checked (blco_format.cpp:193-199) */
int blco_container_checked_layout(const blco_container_header* h, blco_layout* out);
/* read_blco_block (blco_format.cpp:201-227): the record head (key range
 * check), the payload into storage from `alloc`, then the per-element checks
 * on `device` */
int blco_container_read_block(blco_read_fn fn, void* ctx, const blco_layout* layout, uint64_t* key,
                              uint64_t* nnz, blco_alloc_fn alloc, void* alloc_ctx, int device);
/* serialize_blco (blco_format.cpp:149-166), header then one call per block */
int blco_container_write_header(blco_write_fn fn, void* ctx, const blco_layout* layout,
                                uint64_t max_nnz_per_block, uint64_t block_count);
int blco_container_write_block(blco_write_fn fn, void* ctx, uint64_t key, uint64_t nnz, const uint64_t* idx,
                               const double* vals);

/* read_blco_block's element checks for one block (host or device indices) */
int blco_validate_block(const blco_layout* layout, uint64_t key, uint64_t nnz, const uint64_t* idx,
                        int device);
int blco_validate_block_device(const blco_layout* layout, uint64_t key, uint64_t nnz,
                               const uint64_t* d_idx);

/* -------------------------------------------------------------- MTTKRP
 * mttkrp (proj/include/blco/mttkrp.hpp:110-112): host factors in, host M out
 * (dims[mode] x rank, overwritten). */
int blco_mttkrp(const blco_tensor* t, const double* const* factors, uint64_t rank, int mode,
                int strategy, const blco_exec_config* cfg, double* out,
                blco_mttkrp_stats* stats);

/* Device-resident variant: factors[m] and out are device pointers, work is
 * enqueued on `stream` (cudaStream_t; NULL = legacy default stream) and not
 * synchronised.  out is zeroed first unless accumulate != 0. */
int blco_mttkrp_device(const blco_tensor* t, const double* const* d_factors, uint64_t rank,
                       int mode, int strategy, const blco_exec_config* cfg, double* d_out,
                       int accumulate, void* stream, blco_mttkrp_stats* stats);

/* fp32 variant: fp32 factors, products and output over
 * the same fp64-valued BLCO tensor (values rounded to fp32 per element);
 * register strategy only, no deterministic mode.  Tolerance 1e-5 relative
 * Frobenius against the fp64 oracle.  Device (d_*, stream, accumulate as in
 * blco_mttkrp_device) and host (factors in, out overwritten) entries. */
/* Every mode of a device-resident tensor in one call (B200 extension: the
 * all-mode step with fixed factors, BASELINE's "MTTKRP time/iter (all
 * modes)").  d_outs[n] (I_n x R, device) receive M_n: the per-mode
 * kernels run back to back on `stream`.  With BLCO_B200_FUSED=1 (opt-in,
 * measured slower on B200: L2-atomic bound), order 3, R = 16 / 32 and
 * factors + outputs within 64 MB, one fused kernel stages each element once
 * and gathers its three rows once for all three modes (k_mttkrp_all3;
 * per-element terms in the oracle's order).  *fused (optional) says which. */
/* CTA dispatch order of the register kernel for `mode` (B200 extension,
 * mttkrp.cu panel_plan): when the factors exceed L2 the tiles run in panels
 * of 2^bx target rows x 2^by rows of mode *y_mode, ALTO order inside a panel;
 * *y_mode = -1 when they run in plain ALTO order.  elem_bytes = 8 (fp64) or
 * 4 (the fp32 variant).  Reads BLCO_B200_PANEL / BLCO_B200_PANEL_MB. */
int blco_panel_plan(const blco_layout* layout, int mode, uint64_t rank, uint64_t elem_bytes, int* y_mode, int* bx,
                    int* by);
int blco_mttkrp_all_device(const blco_tensor* t, const double* const* d_factors, uint64_t rank, int strategy,
                           const blco_exec_config* cfg, double* const* d_outs, int accumulate, void* stream,
                           int* fused);
int blco_mttkrp_device_f32(const blco_tensor* t, const float* const* d_factors, uint64_t rank, int mode,
                           const blco_exec_config* cfg, float* d_out, int accumulate, void* stream);
int blco_mttkrp_f32(const blco_tensor* t, const float* const* factors, uint64_t rank, int mode,
                    const blco_exec_config* cfg, float* out);

/* All-mode MTTKRP of a HOST-resident BLCO tensor: outs[n] = mttkrp(t, f, n)
 * for every mode n (mttkrp.hpp:110-112 applied to modes 0..N-1, the
 * BASELINE "time/iter (all modes)" step).  The block payload (keys,
 * block_nnz, idx[b], vals[b] as in blco_tensor_upload; pinned host memory
 * gives asynchronous copies) is uploaded in tile-aligned chunks on one stream
 * while every mode's kernel runs on the chunks already resident on another;
 * factors[m] are host dims[m] x rank, outs[m] host dims[m] x rank
 * (overwritten), or device pointers on `device` when outs_on_device != 0
 * (multi-GPU callers reduce them with NCCL).  chunk_elems = 0 picks
 * max(2^20, nnz/32), shrinking geometrically over the last chunks.
 * Device buffers are cached per calling thread and reused by later calls.
 * Returns after the outputs are written. */
typedef struct blco_all_modes_report {
  double device_ms;   /* CUDA events: first copy enqueued .. last D2H done */
  uint64_t chunks;
  uint64_t h2d_bytes; /* payload + factors + tile table + block bases */
  uint64_t d2h_bytes; /* every M_n */
  uint64_t launches;  /* kernels this call launched */
} blco_all_modes_report;

int blco_mttkrp_all_host(const blco_layout* layout, uint64_t nblocks, const uint64_t* keys,
                         const uint64_t* block_nnz, const uint64_t* const* idx,
                         const double* const* vals, const double* const* factors, uint64_t rank,
                         int strategy, const blco_exec_config* cfg, uint64_t chunk_elems,
                         int device, double* const* outs, int outs_on_device,
                         blco_all_modes_report* report);

/* merge_copies (mttkrp.hpp:103): out = sum_c copies[c], copy 0 first. */
int blco_merge_copies(const double* const* copies, uint64_t ncopies, uint64_t elems,
                      double* out);

/* ----------------------------------------------------------- streaming
 * DeviceBudget / BlockSource / StreamReport / stream_mttkrp
 * (proj/include/blco/streaming.hpp:12-94).  Blocks arrive through a pull
 * callback called from the calling thread in order (BlockSource::next). */
typedef struct blco_block_view {
  uint64_t key;
  uint64_t nnz;
  const uint64_t* idx;
  const double* vals;
  /* BLCO_BLOCK_STABLE: idx/vals stay valid until blco_stream_mttkrp returns
   * (e.g. MemoryBlockSource), so the copy need not finish before the next
   * pull.  Without it the library waits for each block's host-to-device copy
   * (pinned or pageable) before pulling the next block, so a source may
   * refill one buffer per pull. */
  uint32_t flags;
} blco_block_view;

#define BLCO_BLOCK_STABLE 1u

/* returns 1 = block produced, 0 = end of stream, < 0 = error (message via
 * blco_set_error from the callback, status = -return) */
typedef int (*blco_block_source_fn)(void* ctx, blco_block_view* out);

typedef struct blco_device_budget {
  uint64_t capacity_bytes;
  int32_t num_queues;
  uint64_t reservation_bytes;
  double injected_transfer_latency_s;
} blco_device_budget;

typedef struct blco_stream_event {
  int32_t kind; /* 0 = transfer, 1 = compute */
  int32_t queue;
  uint64_t block;
  double begin_s, end_s;
} blco_stream_event;

typedef struct blco_stream_report {
  uint64_t blocks;
  uint64_t bytes_streamed;
  double total_seconds;
  double transfer_busy_seconds;
  double compute_busy_seconds;
  double overall_gbps;
  double compute_gbps;
  uint64_t peak_resident_bytes;
  /* caller-provided arrays (may be NULL); filled up to the capacities */
  int32_t* block_queue;
  uint64_t block_queue_capacity;
  blco_stream_event* timeline;
  uint64_t timeline_capacity;
  uint64_t timeline_count;
} blco_stream_report;

int blco_stream_mttkrp(const blco_layout* layout, uint64_t max_nnz_per_block,
                       blco_block_source_fn next, void* ctx, const double* const* factors,
                       uint64_t rank, int mode, const blco_device_budget* budget,
                       const blco_exec_config* cfg, int strategy, int device, double* out,
                       blco_stream_report* report);

/* B200 extension: the blocks stream once and every mode's MTTKRP runs on each
 * resident block (outs[m] = dims[m] x rank, host).  The resident set adds all
 * N outputs to the factors; same budget rules and report as above, with
 * compute intervals covering the N kernels of a block.  outs_on_device != 0:
 * outs[m] are device pointers on `device` (multi-GPU streaming: each rank
 * streams its own blocks, then the partial M_m are summed with NCCL). */
int blco_stream_mttkrp_all(const blco_layout* layout, uint64_t max_nnz_per_block,
                           blco_block_source_fn next, void* ctx, const double* const* factors,
                           uint64_t rank, const blco_device_budget* budget,
                           const blco_exec_config* cfg, int strategy, int device, double* const* outs,
                           int outs_on_device, blco_stream_report* report);

/* stream_mttkrp over a FileBlockSource (streaming.hpp:45-58) without a host
 * round trip through pageable memory: a reader thread reads each block of the
 * .blco container at `path` into a ring of pinned host slots (num_queues + 2)
 * while earlier blocks are copied and multiplied; read_blco_block's record
 * checks run on the host, its per-element checks on the device on the copy
 * that is multiplied (reference messages: "blco: bad magic",
 * "blco: truncated payload", ...).  mode >= 0: outs[0] = M_mode; mode < 0:
 * every mode, outs[m] (host, dims[m] x rank). */
int blco_stream_mttkrp_file(const char* path, const double* const* factors, uint64_t rank, int mode,
                            const blco_device_budget* budget, const blco_exec_config* cfg, int strategy,
                            int device, double* const* outs, blco_stream_report* report);

void blco_set_error(int status, const char* msg);

/* Pinned host memory for stream sources (true async H2D); pageable source
 * memory is accepted but each of its transfers completes before next(). */
void* blco_host_alloc_pinned(uint64_t bytes);
void blco_host_free_pinned(void* p);
int blco_host_register(void* p, uint64_t bytes);
int blco_host_unregister(void* p);

/* -------------------------------------------------------------- CP-ALS
 * cp_als / fit (proj/include/blco/cpals.hpp:38-43).  MTTKRP, Gram, normal
 * solve and normalisation run on the device; factors_out[m] (host) receives
 * dims[m] x rank, fit_out[max_iters] the fit history. */
int blco_cp_als(const blco_tensor* t, uint64_t rank, int max_iters, double tol, uint64_t seed,
                int strategy, const blco_exec_config* cfg, double* const* factors_out,
                double* lambda_out, double* fit_out, int* iters_out);
/* Same, plus device time of the iteration loop (CUDA events): iterations_ms
 * covers every mode's MTTKRP + solve + normalise + Gram and the fit;
 * mttkrp_ms the MTTKRP kernels alone. */
typedef struct blco_cp_als_stats {
  int32_t iterations;
  double iterations_ms;
  double mttkrp_ms;
} blco_cp_als_stats;
int blco_cp_als_timed(const blco_tensor* t, uint64_t rank, int max_iters, double tol, uint64_t seed,
                      int strategy, const blco_exec_config* cfg, double* const* factors_out,
                      double* lambda_out, double* fit_out, int* iters_out, blco_cp_als_stats* stats);
int blco_fit(const blco_tensor* t, const double* const* factors, const double* lambda,
             uint64_t rank, const blco_exec_config* cfg, double* fit_out);

/* ------------------------------------------------------------ multi-GPU
 * The partition of SURVEY.md 8e inside the library: the tensor's element
 * spans are cut into G contiguous nnz-balanced ranges (blco_partition), the
 * factor matrices are replicated, every device runs each mode's kernel on its
 * range into a full partial M_n, and the partials are summed by NCCL over
 * NVLink/NVSwitch -- per mode an all-reduce (BLCO_REDUCE_ALL: every device
 * holds M_n) or a reduce-scatter (BLCO_REDUCE_SCATTER: device g holds rows
 * [g*P, (g+1)*P) of M_n, P = ceil(I_n / G), from partials padded to G*P rows).
 * The collective of mode n runs on the communicator's stream, ordered after
 * that mode's kernel by an event, so it overlaps the kernel of mode n+1.
 * NCCL is loaded at run time (libnccl.so.2, reusing a copy already in the
 * process; BLCO_B200_NCCL overrides the path); G = 1 needs no NCCL.  Errors
 * from NCCL return BLCO_ENCCL.  The reference has no multi-device path
 * (SPEC.md:489): this is the north_star's multi-GPU subsystem. */
#define BLCO_REDUCE_ALL 0
#define BLCO_REDUCE_SCATTER 1
#define BLCO_COMM_ID_BYTES 128

/* NCCL's version code (e.g. 22809), or BLCO_ENCCL when NCCL is absent */
int blco_nccl_version(int* version);

/* One member of a G-rank communicator: its device, NCCL communicator and
 * collective stream.  Multi-process use (one process per GPU): rank 0 calls
 * blco_comm_unique_id, the caller moves the BLCO_COMM_ID_BYTES bytes to every
 * rank (any channel), each rank calls blco_comm_init_rank on its device. */
typedef struct blco_comm blco_comm;
int blco_comm_unique_id(uint8_t* id);
int blco_comm_init_rank(const uint8_t* id, int nranks, int rank, int device, blco_comm** out);
/* single-process: comms_out[g] for devices[g], g < ndev (ncclCommInitAll) */
int blco_comm_init_all(const int* devices, int ndev, blco_comm** comms_out);
void blco_comm_free(blco_comm* comm);

/* One rank's all-mode step: d_outs[n] (device, I_n x R rows; G*P rows for
 * BLCO_REDUCE_SCATTER) are zeroed, receive this rank's partial M_n from the
 * kernel of mode n on `stream`, and are reduced across the communicator on
 * its stream; BLCO_REDUCE_SCATTER leaves this rank's P x R shard in
 * d_shards[n].  `local` must live on the communicator's device (e.g. a
 * blco_tensor_slice of the rank's blco_partition range).  Enqueued only:
 * `stream` is made to wait for the collectives before the call returns. */
int blco_dist_mttkrp_all(const blco_tensor* local, const double* const* d_factors, uint64_t rank,
                         blco_comm* comm, int reduce, int strategy, const blco_exec_config* cfg,
                         double* const* d_outs, double* const* d_shards, void* stream);

/* One host thread driving G devices of this process (SURVEY.md 8b
 * "Threading"): blco_multi_create partitions `t` (any device) into G span
 * ranges copied peer-to-peer onto devices[g]; blco_multi_mttkrp_all uploads
 * the host factors to every device, runs the all-mode step with the chosen
 * reduction (group calls around each mode's G collectives) and writes every
 * M_n to the host outs[n] (I_n x R): from device 0 after an all-reduce, or
 * each device's row shard after a reduce-scatter. */
typedef struct blco_multi blco_multi;
typedef struct blco_multi_report {
  int devices;
  double device_ms;   /* kernels + collectives, max over devices (CUDA events) */
  uint64_t h2d_bytes; /* factor replicas uploaded */
  uint64_t d2h_bytes; /* M_n read back */
} blco_multi_report;
int blco_multi_create(const blco_tensor* t, const int* devices, int ndev, blco_multi** out);
int blco_multi_info(const blco_multi* m, int* ndev, uint64_t* elem_begin, uint64_t* elem_end);
int blco_multi_mttkrp_all(blco_multi* m, const double* const* factors, uint64_t rank, int reduce, int strategy,
                          const blco_exec_config* cfg, double* const* outs, blco_multi_report* report);
void blco_multi_free(blco_multi* m);

/* ------------------------------------------------ distributed CP-ALS pieces
 * The dense steps of one cp_als mode (proj/src/cpals.cpp:84-96) split where a
 * multi-GPU run reduces across ranks: after a reduce-scatter
 * of M_n, rank g holds `rows` rows of it; it solves them locally, the ranks
 * all-reduce the R x R partial Gram (whose diagonal carries the column
 * norms), normalise their rows and all-gather A_n.  The collectives are the
 * caller's (torch.distributed / NCCL); paper_2201_12523_b200/dist.py is the
 * driver.  Device pointers, enqueued on `stream`, never synchronised.
 * Matrices are row-major R x R (full, symmetric) or rows x R.  Ranks up to
 * 64.  The solve reads L from its own device buffer (the constant-bank
 * variant is reserved to blco_cp_als, which serialises its runs), so
 * concurrent calls on different streams are safe. */
/* *d_out = sum of squared values of t (tensor_norm_squared, cpals.cpp:15-20) */
int blco_tensor_norm_sq(const blco_tensor* t, double* d_out, void* stream);
/* d_gram = A^T A over `rows` rows of d_a (gram, dense_kernels.cpp:8-21) */
int blco_als_gram(const double* d_a, uint64_t rows, uint64_t rank, double* d_gram, void* stream);
/* V = hadamard_{m != mode} d_grams[m] (d_grams: order x R x R), its Cholesky
 * factor with solve_normal's Tikhonov escalation (dense_kernels.cpp:68-92),
 * d_a = d_m V^-1 over `rows` rows, d_gram = A^T A over those rows;
 * d_status[0] = 1 when V stays singular after the maximal shift. */
int blco_als_solve(const double* d_grams, int order, int mode, uint64_t rank, const double* d_m, uint64_t rows,
                   double* d_a, double* d_gram, int* d_status, void* stream);
/* normalize_columns (cpals.cpp:51-61) from the summed Gram G of every rank's
 * rows: d_lambda = sqrt(diag G) (0 -> 1), d_gram_n = G / (l l^T) (the Gram of
 * the normalised factor), d_a /= lambda over `rows` rows; with d_m != NULL
 * also *d_inner = sum_{i,r} m[i,r] lambda[r] A[i,r] over those rows (the
 * fit's <X, Xhat>, cpals.cpp:36-44). */
int blco_als_normalize(const double* d_gram_sum, uint64_t rank, double* d_a, uint64_t rows, double* d_gram_n,
                       double* d_lambda, const double* d_m, double* d_inner, void* stream);
/* *d_fit = fit_value(xnormsq, *d_inner, |Xhat|^2 from d_grams and d_lambda)
 * (cpals.cpp:23-49) */
int blco_als_fit(const double* d_grams, int order, uint64_t rank, const double* d_lambda, const double* d_inner,
                 double xnormsq, double* d_fit, void* stream);

/* ----------------------------------------------------------- factories
 * FactorMatrices::random (proj/src/types.cpp:118-130), SplitMix64; host and
 * device (d_out[m] device pointers) produce identical bits. */
int blco_factors_random(const uint64_t* dims, int order, uint64_t rank, uint64_t seed,
                        double* const* out);
int blco_factors_random_device(const uint64_t* dims, int order, uint64_t rank, uint64_t seed,
                               double* const* d_out, void* stream);
/* Host restatement of the device synthetic generator (small sizes). */
int blco_synth_uniform_host(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed,
                            uint64_t* idx, double* vals);

/* ---------------------------------------------------------- multi-GPU
 * Contiguous, nnz-balanced partition of the batch-table spans (quota
 * elements each, never straddling blocks) into nparts ranges; part p gets
 * global elements [begin[p], end[p]). */
int blco_partition(const uint64_t* block_nnz, uint64_t nblocks, uint64_t quota, int nparts,
                   uint64_t* begin, uint64_t* end);

/* --------------------------------------------------------- diagnostics */
int blco_device_count(void);
/* Number of kernels this library launched since load (tests/bench audit). */
uint64_t blco_kernel_launch_count(void);
/* Frees the calling thread's cached device buffers (the all-mode host
 * pipeline's payload/factor/output buffers, hierarchical copies, the
 * deterministic partials); later calls re-create them. */
int blco_release_thread_caches(void);

#ifdef __cplusplus
}
#endif
#endif
