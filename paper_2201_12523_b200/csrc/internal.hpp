// internal.hpp -- shared internals of libblco_b200 (not installed).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "blco_b200.h"

namespace b200 {

// NVTX range for the stages of the path (build, MTTKRP launches, streamed
// blocks, ALS iterations), visible to nsys / ncu --nvtx.  Header-only NVTX3:
// a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ------------------------------------------------------------------ errors
// Internal code throws Status; the C ABI converts to (code, message).
struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void throw_format(const std::string& m) { throw Status(BLCO_EFORMAT, m); }
[[noreturn]] inline void throw_error(const std::string& m) { throw Status(BLCO_ERROR, m); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define B200_CUDA(expr) ::b200::cuda_check((expr), #expr, __FILE__, __LINE__)

void set_error(int code, const std::string& msg);

template <class F>
int guarded(F&& f) {
  try {
    f();
    return BLCO_OK;
  } catch (const Status& s) {
    set_error(s.code, s.what());
    return s.code;
  } catch (const std::exception& e) {
    set_error(BLCO_ERROR, e.what());
    return BLCO_ERROR;
  }
}

// Kernel attribute helpers, cached per (device, kernel): cudaFuncSetAttribute
// is only called when a kernel needs more dynamic shared memory than it was
// last granted, and occupancy queries are answered from the cache, so the
// hot enqueue paths make no attribute calls in steady state.
void ensure_dyn_smem(const void* kernel, size_t bytes);
int blocks_per_sm(const void* kernel, int threads, size_t dyn_smem);
// SMs of the current device (queried once per device; 148 on B200)
int sm_count();
// the kernel family Strategy::Auto runs for a mode of `len` rows (host.cpp)
int auto_kernel(uint64_t len, const blco_exec_config& c);

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void check_launch(const char* what);

// ----------------------------------------------------------------- layout
int bits_for_extent(uint64_t extent);
blco_layout make_layout(const uint64_t* dims, int order, int target_bits);
uint64_t key_upper(const blco_layout& l, int mode, uint64_t key);

// --------------------------------------------------------- device buffers
// BLCO_B200_POISON=1 (debug): fill every new device buffer with 0xFF bytes
// (NaN doubles, all-ones indices), so a read before the first write shows.
bool poison_allocations();

// Build-scoped scratch: while a ScratchScope is live on this thread, DevBuf
// allocations are stream-ordered (cudaMallocAsync / cudaFreeAsync on the
// legacy stream, the device's default pool keeping up to 4 GiB cached), so
// the temporaries of a BLCO build no longer pay a device-synchronising
// cudaMalloc / cudaFree per stage, and a repeated build reuses the pool.
// Buffers that outlive the build (the tensor's payload) are allocated under
// ScratchScope(false).  All users of scratch buffers run on the legacy stream.
struct ScratchScope {
  bool prev;
  explicit ScratchScope(bool on = true);
  ~ScratchScope();
  ScratchScope(const ScratchScope&) = delete;
  ScratchScope& operator=(const ScratchScope&) = delete;
};
bool scratch_active();
void* scratch_alloc(size_t bytes);
void scratch_trim();  // blco_release_thread_caches: return the pool's cached memory

template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  bool scratch = false;  // stream-ordered (ScratchScope) allocation
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), n(o.n), scratch(o.scratch) { o.ptr = nullptr, o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      ptr = o.ptr, n = o.n, scratch = o.scratch;
      o.ptr = nullptr, o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void alloc(size_t count) {
    reset();
    if (count) {
      scratch = scratch_active();
      if (scratch) ptr = static_cast<T*>(scratch_alloc(count * sizeof(T)));
      else B200_CUDA(cudaMalloc(&ptr, count * sizeof(T)));
      if (poison_allocations()) B200_CUDA(cudaMemset(ptr, 0xFF, count * sizeof(T)));
    }
    n = count;
  }
  void reset() {
    if (ptr) {
      if (scratch) cudaFreeAsync(ptr, nullptr);
      else cudaFree(ptr);
    }
    ptr = nullptr, n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Scoped device selection (restores the caller's device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    B200_CUDA(cudaGetDevice(&prev));
    if (dev != prev) B200_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// CTA work unit of the MTTKRP kernels: contiguous elements of one block.
struct TileDesc {
  uint64_t start;  // global element offset
  uint32_t count;  // <= tile elements
  uint32_t block;  // block ordinal
};
static_assert(sizeof(TileDesc) == 16, "TileDesc must stay 16 bytes");

// Deterministic-mode index of one mode (determ.cu): element ids sorted
// stably by target row, rows split into chunks, long rows' partial slots.
struct DetIndex {
  DevBuf<uint32_t> perm;
  DevBuf<uint64_t> chunk_begin, block_off;
  DevBuf<uint32_t> chunk_count, chunk_row, chunk_part;
  DevBuf<uint32_t> multi_row, multi_first, multi_nparts;
  uint64_t nparts = 0;
};

}  // namespace b200

// ------------------------------------------------------- the opaque tensor
struct blco_tensor {
  blco_layout layout{};
  int device = 0;
  uint64_t nnz = 0;
  uint64_t max_nnz_per_block = 0;
  std::vector<uint64_t> keys;     // per block
  std::vector<uint64_t> offsets;  // nblocks + 1 element offsets
  b200::DevBuf<uint64_t> idx;     // re-encoded indices, ALTO order
  b200::DevBuf<double> vals;
  b200::DevBuf<uint32_t> block_base;  // [nblocks * order] decoded base coords
  // tile tables keyed by tile size, built lazily
  mutable std::mutex mu;
  mutable std::map<uint32_t, b200::DevBuf<b200::TileDesc>> tiles;
  // panel-ordered tile tables (mttkrp.cu panel_tile_table), keyed by
  // tile size, mode and panel widths
  mutable std::map<uint64_t, b200::DevBuf<b200::TileDesc>> panel_tiles;
  // per tile size: the largest coordinate span (bits) of each mode over the
  // tiles (mttkrp.cu tile_span_bits, sizes the StageR record fields)
  mutable std::map<uint32_t, std::vector<uint32_t>> span_bits;
  // deterministic-mode indices keyed by mode, built lazily
  mutable std::map<int, b200::DetIndex> det;

  uint64_t nblocks() const { return keys.size(); }
};

namespace b200 {
// What one MTTKRP launch reads: the payload, its tile table and block bases.
struct KernelView {
  const blco_layout* layout;
  const blco_tensor* tensor;  // device-resident tensor (null for the streamed / pipelined views)
  const TileDesc* tiles;
  uint64_t ntiles;
  uint64_t elem_end;
  const uint64_t* idx;
  const double* vals;
  const uint32_t* block_base;
};

struct MttkrpLaunch {
  KernelView view;
  const double* const* factors;  // device pointers, one per mode
  uint64_t rank;
  int mode;
  int strategy;  // resolved (not AUTO) when enqueued
  blco_exec_config cfg;
  double* out;  // device, dims[mode] x rank
  int accumulate;
  cudaStream_t stream;
  const blco_tensor* tensor = nullptr;     // set for device-resident tensors (deterministic mode)
  double* hier_copies = nullptr;           // persistent copies (caller merges)
  unsigned long long* counters = nullptr;  // stats counters or null
  uint64_t workgroups = 0;                 // out
  int stash_slots = 0;                     // out
};

// primitives.cu: hand-written sort / scan / compaction (construction path)
void scan_exclusive_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s);
// Stable LSD sort on bits [begin_bit, end_bit); the result lands in the
// *_alt buffers iff *result_in_alt.
template <class K>
void radix_sort_pairs(K* keys, K* keys_alt, uint32_t* vals, uint32_t* vals_alt, uint64_t n, int begin_bit,
                      int end_bit, cudaStream_t s, bool* result_in_alt);
// Stable compaction; in == nullptr writes the element indices.  Returns count.
template <class T>
uint64_t select_flagged(const T* in, const uint8_t* flags, uint64_t n, T* out, cudaStream_t s);

KernelView view_of(const blco_tensor& t);
void mttkrp_enqueue(MttkrpLaunch& a);
void det_mttkrp_enqueue(const blco_tensor& t, MttkrpLaunch& a);
// container.cu: .blco header and the device-side element checks of
// read_blco_block (blco_format.cpp:201-227), asynchronous: bits are ORed
// into *d_bad (1 field width, 2 outside dims, 4 ALTO order).
struct BlcoFileHeader {
  uint16_t version;
  blco_layout layout;
  uint64_t max_nnz, nblocks;
};
BlcoFileHeader read_blco_file_header(FILE* f);
void enqueue_block_check(const blco_layout& l, uint64_t key, const uint64_t* d_idx, uint64_t n, unsigned* d_bad,
                         cudaStream_t s);
void throw_block_check(unsigned bad);
// per-thread device caches (blco_release_thread_caches)
void release_allmode_cache();
void release_det_cache();
void release_mttkrp_workspace();
void merge_copies_enqueue(const double* copies, uint64_t elems, int ncopies, double* out,
                          int accumulate, cudaStream_t s);
uint32_t mttkrp_tile_elems();

// Builds per-block base coordinates on the device and finalises a tensor
// whose idx/vals/keys/offsets are populated.
void finalize_tensor(blco_tensor& t);
const TileDesc* tile_table(const blco_tensor& t, uint32_t tile_elems, uint64_t* ntiles);
void check_device_layout(const blco_layout& l);
}  // namespace b200
