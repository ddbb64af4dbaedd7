// blco/b200.hpp -- the reference's public C++ API, re-declared for the
// B200 implementation (libblco_b200.so).  A program written against the
// reference headers (proj/include/blco/) recompiles against this tree
// unchanged for the hot path; the per-name headers next to this file
// (blco/mttkrp.hpp, ...) forward here.
//
// Declared here: every type and function on the BLCO MTTKRP path (SURVEY
// §8a rows a1-a25).  Not declared: the CPU execution-simulator internals
// (Scratch, WgCommit, run_workgroups, processing_phase, Stash, tile
// primitives -- proj/include/blco/exec.hpp:33-137, mttkrp.hpp:27-101), which
// have no meaning once the work runs as CUDA kernels, and FROSTT text I/O /
// model export (out of scope).
#pragma once

#include <bit>
#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <filesystem>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

struct blco_multi;  // include/blco_b200.h (the multi-GPU handle)

namespace blco {

// ---------------------------------------------------------------- common.hpp
using index_t = std::uint64_t;
using alto_t = unsigned __int128;
inline constexpr index_t kMaxModeBits = 64;

inline int bits_for_extent(index_t extent) {
  return extent > 1 ? static_cast<int>(std::bit_width(extent - 1)) : 0;
}

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct FormatError : Error {
  using Error::Error;
};
struct IoError : Error {
  using Error::Error;
};
struct VerifyError : Error {
  using Error::Error;
};

// ----------------------------------------------------------------- types.hpp
struct DenseMatrix {
  std::size_t rows = 0, cols = 0;
  std::vector<double> data;  // row-major

  DenseMatrix() = default;
  DenseMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
  double& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
  double operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
  std::span<double> row(std::size_t i) { return {data.data() + i * cols, cols}; }
  std::span<const double> row(std::size_t i) const { return {data.data() + i * cols, cols}; }
  bool same_shape(const DenseMatrix& o) const { return rows == o.rows && cols == o.cols; }
  bool all_finite() const;
};

struct SparseTensorCoo {
  std::vector<index_t> dims;
  std::vector<std::vector<index_t>> indices;  // [mode][element]
  std::vector<double> values;

  int order() const { return static_cast<int>(dims.size()); }
  std::size_t nnz() const { return values.size(); }
  void validate(bool check_duplicates = false) const;
  static SparseTensorCoo from_arrays(std::vector<index_t> dims,
                                     std::vector<std::vector<index_t>> indices,
                                     std::vector<double> values);
  double norm_squared() const;
};

struct FactorMatrices {
  std::size_t rank = 0;
  std::vector<DenseMatrix> factors;

  int order() const { return static_cast<int>(factors.size()); }
  void validate(std::span<const index_t> dims) const;
  static FactorMatrices random(std::span<const index_t> dims, std::size_t rank, std::uint64_t seed);
  static FactorMatrices ones(std::span<const index_t> dims, std::size_t rank);
};

// ---------------------------------------------------------------- layout.hpp
struct BitLayout {
  std::vector<index_t> dims;
  std::vector<int> mode_bits;
  int total_bits = 0;
  int target_bits = 64;
  int stripped_bits = 0;
  std::vector<std::pair<int, int>> interleave_map;  // LSB first: (mode, bit)
  std::vector<int> rem_bits;
  std::vector<int> field_shift;
  std::vector<index_t> field_mask;
  std::vector<std::vector<int>> mode_positions;
  std::vector<std::vector<std::pair<int, int>>> key_slices;  // (key bit, coord bit)

  int order() const { return static_cast<int>(dims.size()); }
  index_t key_upper(int mode, index_t packed_key) const {
    index_t up = 0;
    for (const auto& [kbit, cbit] : key_slices[mode]) up |= ((packed_key >> kbit) & 1u) << cbit;
    return up;
  }
  std::vector<index_t> block_base(index_t packed_key) const;
};

BitLayout make_layout(std::span<const index_t> dims, int target_bits = 64);
alto_t linearize(const BitLayout& layout, std::span<const index_t> coords);

struct SplitIndex {
  index_t block_key = 0;
  index_t reencoded = 0;
};

SplitIndex split_block_key(const BitLayout& layout, alto_t alto);
SplitIndex encode_coords(const BitLayout& layout, std::span<const index_t> coords);
void delinearize(const BitLayout& layout, index_t reencoded, index_t block_key,
                 std::span<index_t> coords_out);
alto_t interleaved_remainder(const BitLayout& layout, index_t reencoded);

// ----------------------------------------------------------- blco_format.hpp
inline constexpr std::uint64_t kDefaultMaxNnzPerBlock = std::uint64_t{1} << 27;
inline constexpr std::uint64_t kDefaultBatchQuota = 512;

struct BlcoBlock {
  index_t key = 0;
  std::vector<index_t> linear_indices;
  std::vector<double> values;
  std::size_t nnz() const { return values.size(); }
};

struct BatchSpan {
  std::uint64_t block = 0, offset = 0, count = 0;
  bool operator==(const BatchSpan&) const = default;
};

struct BlcoTensor {
  BitLayout layout;
  std::uint64_t max_nnz_per_block = kDefaultMaxNnzPerBlock;
  std::vector<BlcoBlock> blocks;
  std::uint64_t total_nnz = 0;
  std::uint64_t batch_quota = kDefaultBatchQuota;
  std::vector<BatchSpan> batch_table;

  int order() const { return layout.order(); }
  const std::vector<index_t>& dims() const { return layout.dims; }
  bool structurally_equal(const BlcoTensor& o) const;
};

struct BuildStats {
  double sort_seconds = 0, block_seconds = 0, reencode_seconds = 0, batch_seconds = 0;
};

// Device construction (K1-K3); the blocks come back to host vectors bit-exact
// with the reference's build.
BlcoTensor build_blco(const SparseTensorCoo& coo, int target_bits = 64,
                      std::uint64_t max_nnz_per_block = kDefaultMaxNnzPerBlock,
                      BuildStats* stats = nullptr);
std::vector<BatchSpan> compute_batch_table(const BlcoTensor& t,
                                           std::uint64_t elements_per_workgroup);
SparseTensorCoo delinearize_all(const BlcoTensor& t);

// .blco container, byte-compatible with the reference; element validation of
// read_blco_block runs on the device.
void serialize_blco(const BlcoTensor& t, std::ostream& out);
void save_blco(const BlcoTensor& t, const std::filesystem::path& path);
BlcoTensor deserialize_blco(std::istream& in);
BlcoTensor load_blco(const std::filesystem::path& path);

struct BlcoHeader {
  std::uint16_t version = 0;
  std::vector<index_t> dims;
  int target_bits = 0;
  std::vector<int> mode_bits;
  std::uint64_t max_nnz_per_block = 0;
  std::uint64_t block_count = 0;

  BitLayout make_layout_checked() const;
};

BlcoHeader read_blco_header(std::istream& in);
BlcoBlock read_blco_block(std::istream& in, const BitLayout& layout);

// ------------------------------------------------------------------ exec.hpp
struct ExecConfig {
  int workgroup_size = 128;
  int tile_size = 32;
  int coarsening = 4;
  int num_compute_units = 108;
  int num_factor_copies = 1;
  int stash_slots = 32;
  bool deterministic = false;
  int num_threads = 0;

  void validate() const;
  std::uint64_t workgroup_quota() const {
    return static_cast<std::uint64_t>(workgroup_size) * coarsening;
  }
  int host_threads() const;
};

// ---------------------------------------------------------------- mttkrp.hpp
enum class Strategy { Auto, Register, Hierarchical };

const char* strategy_name(Strategy s);
Strategy choose_strategy(index_t target_mode_length, const ExecConfig& config);

struct MttkrpStats {
  Strategy strategy = Strategy::Register;
  std::uint64_t workgroups = 0;
  std::uint64_t segments = 0;
  std::uint64_t stash_flushes = 0;
  std::uint64_t commit_events = 0;
  std::uint64_t scalar_adds = 0;
};

DenseMatrix merge_copies(std::span<const DenseMatrix> copies);
DenseMatrix mttkrp(const BlcoTensor& t, const FactorMatrices& f, int mode,
                   const ExecConfig& config = {}, Strategy strategy = Strategy::Auto,
                   MttkrpStats* stats = nullptr);

// B200 extension: mttkrp(t, f, n) for every mode n in one call, the host
// payload uploaded (every call, no device cache) in chunks under the compute
// (blco_mttkrp_all_host).  Result n is dims[n] x rank.
std::vector<DenseMatrix> mttkrp_all_modes(const BlcoTensor& t, const FactorMatrices& f,
                                          const ExecConfig& config = {},
                                          Strategy strategy = Strategy::Auto);

// B200 extension, multi-GPU (the reference has no multi-device
// path): one host thread drives G GPUs.  The tensor's element
// spans are cut into G contiguous nnz-balanced ranges, device g holds range g
// and a replica of the factors, every device runs each mode's kernel on its
// range, and the partial M_n are summed by NCCL over NVLink/NVSwitch (an
// all-reduce, or a reduce-scatter into row shards), the reduction of mode n
// overlapping the kernel of mode n+1.  Results equal mttkrp(t, f, n) within
// the fp64 summation-order tolerance.
enum class Reduction { AllReduce, ReduceScatter };

struct MultiReport {
  int devices = 0;
  double device_ms = 0.0;  // kernels + collectives, max over devices
  std::uint64_t h2d_bytes = 0, d2h_bytes = 0;
};

class MultiDeviceTensor {
 public:
  MultiDeviceTensor(const BlcoTensor& t, std::vector<int> devices);
  ~MultiDeviceTensor();
  MultiDeviceTensor(const MultiDeviceTensor&) = delete;
  MultiDeviceTensor& operator=(const MultiDeviceTensor&) = delete;

  std::vector<DenseMatrix> mttkrp_all_modes(const FactorMatrices& f, Reduction how = Reduction::AllReduce,
                                            const ExecConfig& config = {}, Strategy strategy = Strategy::Auto,
                                            MultiReport* report = nullptr);
  const std::vector<int>& devices() const { return devices_; }
  // element range [first, second) of the ALTO-ordered tensor held by each device
  std::vector<std::pair<std::uint64_t, std::uint64_t>> ranges() const;

 private:
  std::vector<int> devices_;
  std::vector<index_t> dims_;
  ::blco_multi* handle_ = nullptr;
};

// ------------------------------------------------------------- streaming.hpp
struct DeviceBudget {
  std::uint64_t capacity_bytes = 0;
  int num_queues = 4;
  std::uint64_t reservation_bytes = 0;
  double injected_transfer_latency_s = 0.0;
};

class BlockSource {
 public:
  virtual ~BlockSource() = default;
  virtual const BitLayout& layout() const = 0;
  virtual std::uint64_t block_count() const = 0;
  virtual std::uint64_t max_nnz_per_block() const = 0;
  virtual bool next(BlcoBlock& out) = 0;
};

class MemoryBlockSource final : public BlockSource {
 public:
  explicit MemoryBlockSource(const BlcoTensor& t) : t_(&t) {}
  const BitLayout& layout() const override { return t_->layout; }
  std::uint64_t block_count() const override { return t_->blocks.size(); }
  std::uint64_t max_nnz_per_block() const override { return t_->max_nnz_per_block; }
  bool next(BlcoBlock& out) override;
  // Zero-copy access for the device pipeline (no BlcoBlock copy).
  const BlcoBlock* next_view();

 private:
  const BlcoTensor* t_;
  std::uint64_t cursor_ = 0;
};

// Incremental `.blco` reader: header up front, one validated block per next().
class FileBlockSource final : public BlockSource {
 public:
  explicit FileBlockSource(const std::filesystem::path& path);
  ~FileBlockSource() override;
  const BitLayout& layout() const override { return layout_; }
  std::uint64_t block_count() const override { return header_.block_count; }
  std::uint64_t max_nnz_per_block() const override { return header_.max_nnz_per_block; }
  bool next(BlcoBlock& out) override;
  // B200: stream_mttkrp on an unconsumed FileBlockSource reads the file
  // through the native pinned-ring reader (blco_stream_mttkrp_file)
  const std::filesystem::path& path() const { return path_; }
  bool consumed() const { return cursor_ != 0; }

 private:
  std::filesystem::path path_;
  std::unique_ptr<std::istream> in_;
  BlcoHeader header_;
  BitLayout layout_;
  std::uint64_t cursor_ = 0;
};

struct StreamEvent {
  enum class Kind { Transfer, Compute };
  Kind kind;
  int queue;
  std::uint64_t block;
  double begin_s, end_s;
};

struct StreamReport {
  std::uint64_t blocks = 0;
  std::uint64_t bytes_streamed = 0;
  double total_seconds = 0;
  double transfer_busy_seconds = 0;
  double compute_busy_seconds = 0;
  double overall_gbps = 0;
  double compute_gbps = 0;
  std::uint64_t peak_resident_bytes = 0;
  std::vector<StreamEvent> timeline;
  std::vector<int> block_queue;
};

struct ThroughputSummary {
  double overall_gbps = 0;
  double compute_only_gbps = 0;
};

ThroughputSummary throughput_report(const StreamReport& report);

DenseMatrix stream_mttkrp(BlockSource& source, const FactorMatrices& f, int mode,
                          const DeviceBudget& budget, const ExecConfig& config = {},
                          Strategy strategy = Strategy::Auto, StreamReport* report = nullptr);

// B200 extension: every block crosses the host link once and all N modes are
// computed on it (blco_stream_mttkrp_all).  Result n is dims[n] x rank; the
// resident set adds all N outputs to the factors.
std::vector<DenseMatrix> stream_mttkrp_all_modes(BlockSource& source, const FactorMatrices& f,
                                                 const DeviceBudget& budget, const ExecConfig& config = {},
                                                 Strategy strategy = Strategy::Auto,
                                                 StreamReport* report = nullptr);

// ----------------------------------------------------------------- cpals.hpp
struct CpAlsOptions {
  std::size_t rank = 32;
  int max_iters = 50;
  double tol = 1e-5;
  std::uint64_t seed = 0;
  Strategy strategy = Strategy::Auto;
};

struct CpModel {
  FactorMatrices factors;
  std::vector<double> lambda;
  std::vector<double> fit_history;
  std::uint64_t seed = 0;
  double final_fit() const { return fit_history.empty() ? 0.0 : fit_history.back(); }
};

class CpAlsError : public Error {
 public:
  CpAlsError(const std::string& msg, std::vector<double> history)
      : Error(msg), fit_history(std::move(history)) {}
  std::vector<double> fit_history;
};

CpModel cp_als(const BlcoTensor& t, const CpAlsOptions& opts, const ExecConfig& config = {});
double fit(const BlcoTensor& t, const CpModel& model, const ExecConfig& config = {});

// ------------------------------------------------- B200 additions (no ref.)
// The device copy of a host BlcoTensor is cached per object (keyed by its
// address and payload pointers/sizes); call this after mutating a tensor in
// place, or to free HBM.
void release_device_cache(const BlcoTensor* t = nullptr);

}  // namespace blco
