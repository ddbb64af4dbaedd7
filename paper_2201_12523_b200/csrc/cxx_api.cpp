// cxx_api.cpp -- the reference's C++ API (include/blco/b200.hpp) implemented
// over the C ABI (include/blco_b200.h).  Host-side data stays in the
// reference's std::vector containers; every compute call goes to the device.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <istream>
#include <map>
#include <ostream>
#include <mutex>
#include <numeric>
#include <optional>
#include <thread>

#include <cuda_runtime.h>

#include "blco/b200.hpp"
#include "blco_b200.h"

namespace blco {

namespace {

[[noreturn]] void rethrow(int status) {
  const std::string msg = blco_last_error();
  switch (status) {
    case BLCO_EFORMAT: throw FormatError(msg);
    case BLCO_EIO: throw IoError(msg);
    case BLCO_EVERIFY: throw VerifyError(msg);
    default: throw Error(msg);
  }
}

inline void ck(int status) {
  if (status != BLCO_OK) rethrow(status);
}

int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) throw Error("cuda: no device available");
  return d;
}

blco_layout to_c(const BitLayout& l) {
  blco_layout c;
  ck(blco_make_layout(l.dims.data(), l.order(), l.target_bits, &c));
  return c;
}

BitLayout from_c(const blco_layout& c) {
  BitLayout l;
  l.dims.assign(c.dims, c.dims + c.order);
  l.mode_bits.assign(c.mode_bits, c.mode_bits + c.order);
  l.total_bits = c.total_bits;
  l.target_bits = c.target_bits;
  l.stripped_bits = c.stripped_bits;
  l.rem_bits.assign(c.rem_bits, c.rem_bits + c.order);
  l.field_shift.assign(c.field_shift, c.field_shift + c.order);
  l.field_mask.assign(c.field_mask, c.field_mask + c.order);
  l.mode_positions.assign(c.order, {});
  for (int m = 0; m < c.order; ++m) l.mode_positions[m].resize(c.mode_bits[m]);
  l.key_slices.assign(c.order, {});
  const int kept = c.total_bits - c.stripped_bits;
  for (int p = 0; p < c.total_bits; ++p) {
    const int m = c.imap_mode[p], k = c.imap_bit[p];
    l.interleave_map.emplace_back(m, k);
    l.mode_positions[m][k] = p;
    if (p >= kept) l.key_slices[m].emplace_back(p - kept, k - c.rem_bits[m]);
  }
  return l;
}

blco_exec_config to_c(const ExecConfig& e) {
  return blco_exec_config{e.workgroup_size,    e.tile_size,        e.coarsening,
                          e.num_compute_units, e.num_factor_copies, e.stash_slots,
                          e.deterministic ? 1 : 0, e.num_threads};
}

std::vector<const double*> factor_ptrs(const FactorMatrices& f) {
  std::vector<const double*> p;
  for (const auto& a : f.factors) p.push_back(a.data.data());
  return p;
}

// ---- device cache for host BlcoTensors
struct Fingerprint {
  const void* first = nullptr;
  const void* last = nullptr;
  std::uint64_t nnz = 0, nblocks = 0;
  int device = -1;
  bool operator==(const Fingerprint&) const = default;
};

struct CacheEntry {
  Fingerprint fp;
  blco_tensor* dev = nullptr;
};

std::mutex g_cache_mu;
std::map<const BlcoTensor*, CacheEntry> g_cache;

Fingerprint fingerprint(const BlcoTensor& t, int device) {
  Fingerprint f;
  f.nnz = t.total_nnz;
  f.nblocks = t.blocks.size();
  f.device = device;
  if (!t.blocks.empty()) {
    f.first = t.blocks.front().linear_indices.data();
    f.last = t.blocks.back().values.data();
  }
  return f;
}

const blco_tensor* device_tensor(const BlcoTensor& t) {
  const int dev = current_device();
  const Fingerprint fp = fingerprint(t, dev);
  std::lock_guard<std::mutex> g(g_cache_mu);
  auto it = g_cache.find(&t);
  if (it != g_cache.end() && it->second.fp == fp) return it->second.dev;
  if (it != g_cache.end()) {
    blco_tensor_free(it->second.dev);
    g_cache.erase(it);
  }
  const blco_layout l = to_c(t.layout);
  std::vector<std::uint64_t> keys, nnz;
  std::vector<const std::uint64_t*> idx;
  std::vector<const double*> vals;
  for (const auto& b : t.blocks) {
    if (b.linear_indices.size() != b.values.size())
      throw FormatError("blco: block index/value arrays have mismatched lengths");
    keys.push_back(b.key);
    nnz.push_back(b.nnz());
    idx.push_back(b.linear_indices.data());
    vals.push_back(b.values.data());
  }
  blco_tensor* d = nullptr;
  ck(blco_tensor_upload(&l, t.max_nnz_per_block, keys.size(), keys.data(), nnz.data(), idx.data(),
                        vals.data(), dev, &d));
  g_cache[&t] = CacheEntry{fp, d};
  return d;
}

}  // namespace

void release_device_cache(const BlcoTensor* t) {
  std::lock_guard<std::mutex> g(g_cache_mu);
  for (auto it = g_cache.begin(); it != g_cache.end();) {
    if (!t || it->first == t) {
      blco_tensor_free(it->second.dev);
      it = g_cache.erase(it);
    } else {
      ++it;
    }
  }
}

// ------------------------------------------------------------------- types
bool DenseMatrix::all_finite() const {
  for (double v : data)
    if (!std::isfinite(v)) return false;
  return true;
}

namespace {

// Tuples packed into one 128-bit word in lexicographic order (mode 0 most
// significant, each mode in bits_for_extent(dims[m]) bits), so tuple order
// and duplicates become integer order and equality.  nullopt when the modes
// need more than 128 bits together.
std::optional<std::vector<alto_t>> packed_tuples(std::span<const index_t> dims,
                                                 const std::vector<std::vector<index_t>>& idx, std::size_t n) {
  if (dims.size() != idx.size()) return std::nullopt;
  int total = 0;
  for (index_t d : dims) total += bits_for_extent(d);
  if (total > 128) return std::nullopt;
  std::vector<alto_t> key(n, 0);
  for (std::size_t m = 0; m < dims.size(); ++m) {
    const int w = bits_for_extent(dims[m]);
    for (std::size_t e = 0; e < n; ++e) key[e] = w ? ((key[e] << w) | idx[m][e]) : key[e];
  }
  return key;
}

// Element ids in lexicographic tuple order, ties in input order.
std::vector<std::uint32_t> tuple_order(std::span<const index_t> dims, const std::vector<std::vector<index_t>>& idx,
                                       std::size_t n) {
  std::vector<std::uint32_t> ids(n);
  for (std::size_t e = 0; e < n; ++e) ids[e] = static_cast<std::uint32_t>(e);
  if (auto key = packed_tuples(dims, idx, n)) {
    const auto& k = *key;
    std::stable_sort(ids.begin(), ids.end(), [&](std::uint32_t a, std::uint32_t b) { return k[a] < k[b]; });
  } else {
    std::stable_sort(ids.begin(), ids.end(), [&](std::uint32_t a, std::uint32_t b) {
      for (const auto& mode : idx)
        if (mode[a] != mode[b]) return mode[a] < mode[b];
      return false;
    });
  }
  return ids;
}

bool same_tuple(const std::vector<std::vector<index_t>>& idx, std::uint32_t a, std::uint32_t b) {
  for (const auto& mode : idx)
    if (mode[a] != mode[b]) return false;
  return true;
}

}  // namespace

void SparseTensorCoo::validate(bool check_duplicates) const {
  if (indices.size() != dims.size()) throw FormatError("coo: index array count does not match order");
  for (std::size_t m = 0; m < dims.size(); ++m) {
    if (dims[m] == 0) throw FormatError("coo: mode length must be >= 1");
    if (indices[m].size() != values.size()) throw FormatError("coo: index/value arrays have mismatched lengths");
    const auto hi = std::max_element(indices[m].begin(), indices[m].end());
    if (hi != indices[m].end() && *hi >= dims[m]) throw FormatError("coo: coordinate out of range");
  }
  if (!check_duplicates || values.size() < 2) return;
  if (values.size() > UINT32_MAX) throw FormatError("coo: too many elements for the duplicate check");
  const std::vector<std::uint32_t> ids = tuple_order(dims, indices, values.size());
  for (std::size_t k = 1; k < ids.size(); ++k)
    if (same_tuple(indices, ids[k - 1], ids[k])) throw FormatError("coo: duplicate coordinate tuple");
}

SparseTensorCoo SparseTensorCoo::from_arrays(std::vector<index_t> dims,
                                             std::vector<std::vector<index_t>> indices,
                                             std::vector<double> values) {
  if (indices.empty()) throw FormatError("coo: at least one mode required");
  const std::size_t n = values.size();
  if (std::any_of(indices.begin(), indices.end(), [&](const auto& v) { return v.size() != n; }))
    throw FormatError("coo: index/value arrays have mismatched lengths");
  if (n > UINT32_MAX) throw FormatError("coo: too many elements");
  if (dims.empty())  // inferred: one past the largest coordinate of each mode
    for (const auto& mode : indices)
      dims.push_back(mode.empty() ? 1 : *std::max_element(mode.begin(), mode.end()) + 1);
  // canonical form: tuples in lexicographic order, each distinct tuple once,
  // its values summed in input order
  const std::vector<std::uint32_t> ids = tuple_order(dims, indices, n);
  SparseTensorCoo out;
  out.dims = std::move(dims);
  out.indices.assign(indices.size(), {});
  std::size_t k = 0;
  while (k < ids.size()) {
    const std::uint32_t head = ids[k];
    double sum = values[head];
    for (++k; k < ids.size() && same_tuple(indices, head, ids[k]); ++k) sum += values[ids[k]];
    for (std::size_t m = 0; m < indices.size(); ++m) out.indices[m].push_back(indices[m][head]);
    out.values.push_back(sum);
  }
  out.validate();
  return out;
}

double SparseTensorCoo::norm_squared() const {
  return std::accumulate(values.begin(), values.end(), 0.0, [](double acc, double v) { return acc + v * v; });
}

void FactorMatrices::validate(std::span<const index_t> dims) const {
  if (factors.size() != dims.size()) throw FormatError("factors: mode count does not match tensor order");
  auto shape = [](std::size_t r, std::size_t c) { return std::to_string(r) + "x" + std::to_string(c); };
  for (std::size_t m = 0; m < dims.size(); ++m) {
    const DenseMatrix& a = factors[m];
    const bool ok = a.rows == dims[m] && a.cols == rank;
    if (!ok)
      throw FormatError("factors: mode " + std::to_string(m + 1) + " has shape " + shape(a.rows, a.cols) +
                        ", expected " + shape(dims[m], rank));
    if (a.data.size() != a.rows * a.cols) throw FormatError("factors: malformed matrix storage");
  }
}

FactorMatrices FactorMatrices::random(std::span<const index_t> dims, std::size_t rank,
                                      std::uint64_t seed) {
  if (rank < 1) throw FormatError("factors: rank must be >= 1");
  FactorMatrices f;
  f.rank = rank;
  std::vector<double*> p;
  for (index_t d : dims) f.factors.emplace_back(d, rank);
  for (auto& a : f.factors) p.push_back(a.data.data());
  ck(blco_factors_random(dims.data(), static_cast<int>(dims.size()), rank, seed, p.data()));
  return f;
}

FactorMatrices FactorMatrices::ones(std::span<const index_t> dims, std::size_t rank) {
  FactorMatrices f;
  f.rank = rank;
  f.factors.reserve(dims.size());
  for (index_t d : dims) {
    f.factors.emplace_back(d, rank);
    f.factors.back().data.assign(d * rank, 1.0);
  }
  return f;
}

// ------------------------------------------------------------------ layout
std::vector<index_t> BitLayout::block_base(index_t packed_key) const {
  std::vector<index_t> base(dims.size());
  for (int m = 0; m < order(); ++m) base[m] = key_upper(m, packed_key) << rem_bits[m];
  return base;
}

BitLayout make_layout(std::span<const index_t> dims, int target_bits) {
  blco_layout c;
  ck(blco_make_layout(dims.data(), static_cast<int>(dims.size()), target_bits, &c));
  return from_c(c);
}

alto_t linearize(const BitLayout& layout, std::span<const index_t> coords) {
  if (coords.size() != layout.dims.size())
    throw FormatError("linearize: coordinate count does not match order");
  const blco_layout c = to_c(layout);
  std::uint64_t hi = 0, lo = 0;
  ck(blco_linearize(&c, coords.data(), &hi, &lo));
  return (static_cast<alto_t>(hi) << 64) | lo;
}

SplitIndex split_block_key(const BitLayout& layout, alto_t alto) {
  const blco_layout c = to_c(layout);
  SplitIndex s;
  ck(blco_split_block_key(&c, static_cast<std::uint64_t>(alto >> 64), static_cast<std::uint64_t>(alto),
                          &s.block_key, &s.reencoded));
  return s;
}

SplitIndex encode_coords(const BitLayout& layout, std::span<const index_t> coords) {
  const blco_layout c = to_c(layout);
  SplitIndex s;
  ck(blco_encode_coords(&c, coords.data(), &s.block_key, &s.reencoded));
  return s;
}

void delinearize(const BitLayout& layout, index_t reencoded, index_t block_key,
                 std::span<index_t> coords_out) {
  const blco_layout c = to_c(layout);
  ck(blco_delinearize(&c, reencoded, block_key, coords_out.data()));
}

alto_t interleaved_remainder(const BitLayout& layout, index_t reencoded) {
  const blco_layout c = to_c(layout);
  std::uint64_t hi = 0, lo = 0;
  ck(blco_interleaved_remainder(&c, reencoded, &hi, &lo));
  return (static_cast<alto_t>(hi) << 64) | lo;
}

// ------------------------------------------------------------------- build
bool BlcoTensor::structurally_equal(const BlcoTensor& o) const {
  const bool same_frame = layout.dims == o.layout.dims && layout.target_bits == o.layout.target_bits &&
                          max_nnz_per_block == o.max_nnz_per_block && total_nnz == o.total_nnz;
  return same_frame && std::equal(blocks.begin(), blocks.end(), o.blocks.begin(), o.blocks.end(),
                                  [](const BlcoBlock& x, const BlcoBlock& y) {
                                    return x.key == y.key && x.values == y.values &&
                                           x.linear_indices == y.linear_indices;
                                  });
}

std::vector<BatchSpan> compute_batch_table(const BlcoTensor& t, std::uint64_t quota) {
  if (quota < 1) throw FormatError("blco: elements_per_workgroup must be >= 1");
  std::vector<std::uint64_t> nnz;
  for (const auto& b : t.blocks) nnz.push_back(b.nnz());
  const std::uint64_t n = blco_batch_table(nnz.data(), nnz.size(), quota, nullptr);
  std::vector<std::uint64_t> raw(3 * n);
  blco_batch_table(nnz.data(), nnz.size(), quota, raw.data());
  std::vector<BatchSpan> spans(n);
  for (std::uint64_t i = 0; i < n; ++i) spans[i] = BatchSpan{raw[3 * i], raw[3 * i + 1], raw[3 * i + 2]};
  return spans;
}

BlcoTensor build_blco(const SparseTensorCoo& coo, int target_bits, std::uint64_t max_nnz,
                      BuildStats* stats) {
  coo.validate();
  if (max_nnz < 1) throw FormatError("blco: max_nnz_per_block must be >= 1");
  const std::size_t nnz = coo.nnz();
  std::vector<std::uint64_t> flat(static_cast<std::size_t>(coo.order()) * nnz);
  for (int m = 0; m < coo.order(); ++m)
    std::copy(coo.indices[m].begin(), coo.indices[m].end(), flat.begin() + m * nnz);
  blco_tensor* d = nullptr;
  blco_build_stats bs{};
  ck(blco_build(coo.dims.data(), coo.order(), nnz, flat.data(), coo.values.data(), target_bits,
                max_nnz, current_device(), &d, &bs));
  std::unique_ptr<blco_tensor, void (*)(blco_tensor*)> guard(d, blco_tensor_free);
  blco_layout c;
  std::uint64_t nb = 0, total = 0, mx = 0;
  ck(blco_tensor_info(d, &c, &nb, &total, &mx));
  std::vector<std::uint64_t> keys(nb), bn(nb), idx(total);
  std::vector<double> vals(total);
  ck(blco_tensor_blocks(d, keys.data(), bn.data()));
  ck(blco_tensor_download(d, idx.data(), vals.data()));
  BlcoTensor t;
  t.layout = from_c(c);
  t.max_nnz_per_block = max_nnz;
  t.total_nnz = total;
  std::uint64_t off = 0;
  for (std::uint64_t b = 0; b < nb; ++b) {
    BlcoBlock blk;
    blk.key = keys[b];
    blk.linear_indices.assign(idx.begin() + off, idx.begin() + off + bn[b]);
    blk.values.assign(vals.begin() + off, vals.begin() + off + bn[b]);
    off += bn[b];
    t.blocks.push_back(std::move(blk));
  }
  t.batch_quota = kDefaultBatchQuota;
  t.batch_table = compute_batch_table(t, t.batch_quota);
  if (stats) *stats = BuildStats{bs.sort_seconds, bs.block_seconds, bs.reencode_seconds, bs.batch_seconds};
  return t;
}

SparseTensorCoo delinearize_all(const BlcoTensor& t) {
  SparseTensorCoo coo;
  coo.dims = t.dims();
  coo.indices.assign(t.order(), {});
  std::vector<index_t> c(t.order());
  for (const auto& b : t.blocks)
    for (std::size_t e = 0; e < b.nnz(); ++e) {
      delinearize(t.layout, b.linear_indices[e], b.key, c);
      for (int m = 0; m < t.order(); ++m) coo.indices[m].push_back(c[m]);
      coo.values.push_back(b.values[e]);
    }
  return coo;
}

// --------------------------------------------------------------- container
// The byte format and every check live in the library (container.cu); these
// overloads only adapt std::istream / std::ostream to its stream hooks.
namespace {
std::uint64_t istream_read(void* ctx, void* dst, std::uint64_t n) {
  auto& in = *static_cast<std::istream*>(ctx);
  in.read(static_cast<char*>(dst), static_cast<std::streamsize>(n));
  return static_cast<std::uint64_t>(in.gcount());
}

std::uint64_t ostream_write(void* ctx, const void* src, std::uint64_t n) {
  auto& out = *static_cast<std::ostream*>(ctx);
  out.write(static_cast<const char*>(src), static_cast<std::streamsize>(n));
  return out ? n : 0;
}

int block_storage(void* ctx, std::uint64_t n, std::uint64_t** idx, double** vals) {
  auto& blk = *static_cast<BlcoBlock*>(ctx);
  blk.linear_indices.resize(n);
  blk.values.resize(n);
  *idx = blk.linear_indices.data();
  *vals = blk.values.data();
  return 0;
}

// the std::ostream overloads report a failed stream as the reference does
void throw_if_failed(const std::ostream& out) {
  if (!out) throw IoError("blco: write failed");
}
}  // namespace

void serialize_blco(const BlcoTensor& t, std::ostream& out) {
  const blco_layout c = to_c(t.layout);
  ck(blco_container_write_header(ostream_write, &out, &c, t.max_nnz_per_block, t.blocks.size()));
  for (const BlcoBlock& b : t.blocks)
    ck(blco_container_write_block(ostream_write, &out, b.key, b.nnz(), b.linear_indices.data(), b.values.data()));
  throw_if_failed(out);
}

void save_blco(const BlcoTensor& t, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open " + path.string() + " for writing");
  serialize_blco(t, out);
}

BlcoHeader read_blco_header(std::istream& in) {
  blco_container_header raw{};
  ck(blco_container_read_header(istream_read, &in, &raw));
  BlcoHeader h;
  h.version = raw.version;
  h.dims.assign(raw.dims, raw.dims + raw.order);
  h.target_bits = raw.target_bits;
  h.mode_bits.assign(raw.mode_bits, raw.mode_bits + raw.order);
  h.max_nnz_per_block = raw.max_nnz_per_block;
  h.block_count = raw.block_count;
  return h;
}

BitLayout BlcoHeader::make_layout_checked() const {
  blco_container_header raw{};
  if (dims.size() > BLCO_MAX_ORDER || mode_bits.size() != dims.size())
    throw FormatError("blco: stored mode bit widths do not match dims");
  raw.version = version;
  raw.order = static_cast<std::uint16_t>(dims.size());
  raw.target_bits = static_cast<std::uint16_t>(target_bits);
  std::copy(dims.begin(), dims.end(), raw.dims);
  std::transform(mode_bits.begin(), mode_bits.end(), raw.mode_bits,
                 [](int b) { return static_cast<std::uint16_t>(b); });
  raw.max_nnz_per_block = max_nnz_per_block;
  raw.block_count = block_count;
  blco_layout c{};
  ck(blco_container_checked_layout(&raw, &c));
  return from_c(c);
}

BlcoBlock read_blco_block(std::istream& in, const BitLayout& layout) {
  const blco_layout c = to_c(layout);
  BlcoBlock blk;
  std::uint64_t n = 0;
  ck(blco_container_read_block(istream_read, &in, &c, &blk.key, &n, block_storage, &blk, current_device()));
  return blk;
}

BlcoTensor deserialize_blco(std::istream& in) {
  const BlcoHeader h = read_blco_header(in);
  BlcoTensor t;
  t.layout = h.make_layout_checked();
  t.max_nnz_per_block = h.max_nnz_per_block;
  t.blocks.reserve(h.block_count);
  for (std::uint64_t b = 0; b < h.block_count; ++b) {
    t.blocks.push_back(read_blco_block(in, t.layout));
    const BlcoBlock& blk = t.blocks.back();
    // record-level rules of deserialize_blco (blco_format.cpp:236-242)
    const char* bad = blk.nnz() == 0                    ? "blco: empty block record"
                      : blk.nnz() > t.max_nnz_per_block ? "blco: block exceeds max_nnz_per_block"
                      : b > 0 && blk.key < t.blocks[b - 1].key ? "blco: blocks not in ascending key order"
                                                               : nullptr;
    if (bad) throw FormatError(bad);
    t.total_nnz += blk.nnz();
  }
  t.batch_quota = kDefaultBatchQuota;
  t.batch_table = compute_batch_table(t, t.batch_quota);
  return t;
}

BlcoTensor load_blco(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path.string());
  return deserialize_blco(in);
}

FileBlockSource::FileBlockSource(const std::filesystem::path& path)
    : path_(path), in_(std::make_unique<std::ifstream>(path, std::ios::binary)) {
  if (!*in_) throw IoError("cannot open " + path.string());
  header_ = read_blco_header(*in_);
  layout_ = header_.make_layout_checked();
}

FileBlockSource::~FileBlockSource() = default;

bool FileBlockSource::next(BlcoBlock& out) {
  if (cursor_ == header_.block_count) return false;
  out = read_blco_block(*in_, layout_);
  ++cursor_;
  return true;
}

// ------------------------------------------------------------------ config
void ExecConfig::validate() const {
  const blco_exec_config c = to_c(*this);
  ck(blco_exec_config_validate(&c));
}

int ExecConfig::host_threads() const {
  if (num_threads > 0) return num_threads;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? static_cast<int>(hw) : 1;
}

const char* strategy_name(Strategy s) {
  switch (s) {
    case Strategy::Auto: return "auto";
    case Strategy::Register: return "register";
    case Strategy::Hierarchical: return "hierarchical";
  }
  return "?";
}

Strategy choose_strategy(index_t len, const ExecConfig& config) {
  const blco_exec_config c = to_c(config);
  return blco_choose_strategy(len, &c) == BLCO_STRATEGY_HIERARCHICAL ? Strategy::Hierarchical
                                                                     : Strategy::Register;
}

// ------------------------------------------------------------------ mttkrp
DenseMatrix merge_copies(std::span<const DenseMatrix> copies) {
  if (copies.empty()) throw FormatError("merge_copies: no copies");
  std::vector<const double*> p;
  for (const auto& c : copies) {
    if (!c.same_shape(copies[0])) throw FormatError("merge_copies: shape mismatch");
    p.push_back(c.data.data());
  }
  DenseMatrix m(copies[0].rows, copies[0].cols);
  ck(blco_merge_copies(p.data(), p.size(), m.data.size(), m.data.data()));
  return m;
}

DenseMatrix mttkrp(const BlcoTensor& t, const FactorMatrices& f, int mode, const ExecConfig& config,
                   Strategy strategy, MttkrpStats* stats) {
  config.validate();
  f.validate(t.dims());
  if (mode < 0 || mode >= t.order())
    throw FormatError("mttkrp: mode " + std::to_string(mode + 1) + " out of range for order " +
                      std::to_string(t.order()));
  const blco_tensor* d = device_tensor(t);
  const auto ptrs = factor_ptrs(f);
  const blco_exec_config c = to_c(config);
  DenseMatrix m(t.dims()[mode], f.rank);
  blco_mttkrp_stats s{};
  ck(blco_mttkrp(d, ptrs.data(), f.rank, mode, static_cast<int>(strategy), &c, m.data.data(),
                 stats ? &s : nullptr));
  if (stats) {
    stats->strategy = s.strategy == BLCO_STRATEGY_HIERARCHICAL ? Strategy::Hierarchical : Strategy::Register;
    stats->workgroups = s.workgroups;
    stats->segments = s.segments;
    stats->stash_flushes = s.stash_flushes;
    stats->commit_events = s.commit_events;
    stats->scalar_adds = s.scalar_adds;
  }
  return m;
}

std::vector<DenseMatrix> mttkrp_all_modes(const BlcoTensor& t, const FactorMatrices& f,
                                          const ExecConfig& config, Strategy strategy) {
  config.validate();
  f.validate(t.dims());
  const blco_layout l = to_c(t.layout);
  std::vector<std::uint64_t> keys, nnz;
  std::vector<const std::uint64_t*> idx;
  std::vector<const double*> vals;
  for (const auto& b : t.blocks) {
    if (b.linear_indices.size() != b.values.size())
      throw FormatError("blco: block index/value arrays have mismatched lengths");
    keys.push_back(b.key);
    nnz.push_back(b.nnz());
    idx.push_back(b.linear_indices.data());
    vals.push_back(b.values.data());
  }
  std::vector<DenseMatrix> out;
  std::vector<double*> optr;
  for (int m = 0; m < t.order(); ++m) out.emplace_back(t.dims()[m], f.rank);
  for (auto& o : out) optr.push_back(o.data.data());
  const auto ptrs = factor_ptrs(f);
  const blco_exec_config c = to_c(config);
  ck(blco_mttkrp_all_host(&l, keys.size(), keys.data(), nnz.data(), idx.data(), vals.data(), ptrs.data(),
                          f.rank, static_cast<int>(strategy), &c, 0, current_device(), optr.data(), 0, nullptr));
  return out;
}

// --------------------------------------------------------------- multi-GPU
MultiDeviceTensor::MultiDeviceTensor(const BlcoTensor& t, std::vector<int> devices)
    : devices_(std::move(devices)), dims_(t.dims()) {
  if (devices_.empty()) throw FormatError("multi: need at least one device");
  // staged on the first device, then cut into span ranges copied peer to peer
  const blco_layout l = to_c(t.layout);
  std::vector<std::uint64_t> keys, nnz;
  std::vector<const std::uint64_t*> idx;
  std::vector<const double*> vals;
  for (const auto& b : t.blocks) {
    if (b.linear_indices.size() != b.values.size())
      throw FormatError("blco: block index/value arrays have mismatched lengths");
    keys.push_back(b.key);
    nnz.push_back(b.nnz());
    idx.push_back(b.linear_indices.data());
    vals.push_back(b.values.data());
  }
  blco_tensor* staged = nullptr;
  ck(blco_tensor_upload(&l, t.max_nnz_per_block, keys.size(), keys.data(), nnz.data(), idx.data(), vals.data(),
                        devices_[0], &staged));
  std::unique_ptr<blco_tensor, void (*)(blco_tensor*)> guard(staged, blco_tensor_free);
  ck(blco_multi_create(staged, devices_.data(), static_cast<int>(devices_.size()), &handle_));
}

MultiDeviceTensor::~MultiDeviceTensor() { blco_multi_free(handle_); }

std::vector<std::pair<std::uint64_t, std::uint64_t>> MultiDeviceTensor::ranges() const {
  int n = 0;
  std::vector<std::uint64_t> b(devices_.size()), e(devices_.size());
  ck(blco_multi_info(handle_, &n, b.data(), e.data()));
  std::vector<std::pair<std::uint64_t, std::uint64_t>> r;
  for (int g = 0; g < n; ++g) r.emplace_back(b[g], e[g]);
  return r;
}

std::vector<DenseMatrix> MultiDeviceTensor::mttkrp_all_modes(const FactorMatrices& f, Reduction how,
                                                             const ExecConfig& config, Strategy strategy,
                                                             MultiReport* report) {
  config.validate();
  f.validate(dims_);
  std::vector<DenseMatrix> out;
  std::vector<double*> optr;
  for (index_t d : dims_) out.emplace_back(d, f.rank);
  for (auto& o : out) optr.push_back(o.data.data());
  const auto ptrs = factor_ptrs(f);
  const blco_exec_config c = to_c(config);
  blco_multi_report r{};
  ck(blco_multi_mttkrp_all(handle_, ptrs.data(), f.rank,
                           how == Reduction::ReduceScatter ? BLCO_REDUCE_SCATTER : BLCO_REDUCE_ALL,
                           static_cast<int>(strategy), &c, optr.data(), &r));
  if (report) *report = MultiReport{r.devices, r.device_ms, r.h2d_bytes, r.d2h_bytes};
  return out;
}

// --------------------------------------------------------------- streaming
bool MemoryBlockSource::next(BlcoBlock& out) {
  if (cursor_ >= t_->blocks.size()) return false;
  out = t_->blocks[cursor_++];
  return true;
}

const BlcoBlock* MemoryBlockSource::next_view() {
  if (cursor_ >= t_->blocks.size()) return nullptr;
  return &t_->blocks[cursor_++];
}

ThroughputSummary throughput_report(const StreamReport& r) { return {r.overall_gbps, r.compute_gbps}; }

namespace {
struct SourceCtx {
  BlockSource* src;
  MemoryBlockSource* mem;
  BlcoBlock scratch;
  std::exception_ptr error;
};

int pull(void* ctx, blco_block_view* out) {
  auto* c = static_cast<SourceCtx*>(ctx);
  try {
    const BlcoBlock* b = nullptr;
    if (c->mem) {
      b = c->mem->next_view();
    } else if (c->src->next(c->scratch)) {
      b = &c->scratch;
    }
    if (!b) return 0;
    if (b->linear_indices.size() != b->values.size()) throw FormatError("stream: malformed block");
    // MemoryBlockSource blocks live in the caller's tensor for the whole call
    *out = blco_block_view{b->key, b->nnz(), b->linear_indices.data(), b->values.data(),
                           c->mem ? BLCO_BLOCK_STABLE : 0u};
    return 1;
  } catch (...) {
    c->error = std::current_exception();
    blco_set_error(BLCO_ERROR, "stream: block source failed");
    return -BLCO_ERROR;
  }
}
}  // namespace

namespace {
// Shared by stream_mttkrp (mode >= 0) and stream_mttkrp_all_modes (mode < 0).
std::vector<DenseMatrix> stream_impl(BlockSource& source, const FactorMatrices& f, int mode,
                                     const DeviceBudget& budget, const ExecConfig& config, Strategy strategy,
                                     StreamReport* report) {
  config.validate();
  const BitLayout& layout = source.layout();
  f.validate(layout.dims);
  if (mode >= layout.order()) throw FormatError("stream: mode out of range");
  const blco_layout l = to_c(layout);
  const blco_exec_config c = to_c(config);
  const blco_device_budget b{budget.capacity_bytes, budget.num_queues, budget.reservation_bytes,
                             budget.injected_transfer_latency_s};
  SourceCtx ctx{&source, dynamic_cast<MemoryBlockSource*>(&source), {}, nullptr};
  const auto ptrs = factor_ptrs(f);
  std::vector<DenseMatrix> outs;
  std::vector<double*> optr;
  if (mode >= 0) {
    outs.emplace_back(layout.dims[mode], f.rank);
  } else {
    for (int m = 0; m < layout.order(); ++m) outs.emplace_back(layout.dims[m], f.rank);
  }
  for (auto& o : outs) optr.push_back(o.data.data());
  const std::uint64_t nb = source.block_count();
  std::vector<int32_t> bq(nb);
  std::vector<blco_stream_event> tl(2 * nb);
  blco_stream_report r{};
  r.block_queue = bq.data();
  r.block_queue_capacity = nb;
  r.timeline = tl.data();
  r.timeline_capacity = tl.size();
  auto* file = dynamic_cast<FileBlockSource*>(&source);
  int status;
  if (file && !file->consumed()) {
    // pinned-ring reader and device-side element checks (blco_stream_mttkrp_file)
    status = blco_stream_mttkrp_file(file->path().c_str(), ptrs.data(), f.rank, mode, &b, &c,
                                     static_cast<int>(strategy), current_device(), optr.data(), &r);
  } else {
    status = mode >= 0
                 ? blco_stream_mttkrp(&l, source.max_nnz_per_block(), pull, &ctx, ptrs.data(), f.rank, mode, &b, &c,
                                      static_cast<int>(strategy), current_device(), optr[0], &r)
                 : blco_stream_mttkrp_all(&l, source.max_nnz_per_block(), pull, &ctx, ptrs.data(), f.rank, &b, &c,
                                          static_cast<int>(strategy), current_device(), optr.data(), 0, &r);
  }
  if (ctx.error) std::rethrow_exception(ctx.error);
  ck(status);
  if (report) {
    report->blocks = r.blocks;
    report->bytes_streamed = r.bytes_streamed;
    report->total_seconds = r.total_seconds;
    report->transfer_busy_seconds = r.transfer_busy_seconds;
    report->compute_busy_seconds = r.compute_busy_seconds;
    report->overall_gbps = r.overall_gbps;
    report->compute_gbps = r.compute_gbps;
    report->peak_resident_bytes = r.peak_resident_bytes;
    report->block_queue.assign(bq.begin(), bq.begin() + std::min<std::uint64_t>(nb, r.blocks));
    report->timeline.clear();
    for (std::uint64_t i = 0; i < std::min<std::uint64_t>(r.timeline_count, tl.size()); ++i)
      report->timeline.push_back(StreamEvent{tl[i].kind == 0 ? StreamEvent::Kind::Transfer
                                                              : StreamEvent::Kind::Compute,
                                             tl[i].queue, tl[i].block, tl[i].begin_s, tl[i].end_s});
  }
  return outs;
}
}  // namespace

DenseMatrix stream_mttkrp(BlockSource& source, const FactorMatrices& f, int mode, const DeviceBudget& budget,
                          const ExecConfig& config, Strategy strategy, StreamReport* report) {
  if (mode < 0) throw FormatError("stream: mode out of range");
  return std::move(stream_impl(source, f, mode, budget, config, strategy, report)[0]);
}

std::vector<DenseMatrix> stream_mttkrp_all_modes(BlockSource& source, const FactorMatrices& f,
                                                 const DeviceBudget& budget, const ExecConfig& config,
                                                 Strategy strategy, StreamReport* report) {
  return stream_impl(source, f, -1, budget, config, strategy, report);
}

// ------------------------------------------------------------------- cp-als
CpModel cp_als(const BlcoTensor& t, const CpAlsOptions& opts, const ExecConfig& config) {
  if (opts.rank < 1) throw FormatError("cp_als: rank must be >= 1");
  if (opts.max_iters < 0) throw FormatError("cp_als: max_iters must be >= 0");
  config.validate();
  const blco_tensor* d = device_tensor(t);
  const blco_exec_config c = to_c(config);
  CpModel model;
  model.seed = opts.seed;
  model.factors.rank = opts.rank;
  std::vector<double*> out;
  for (index_t dim : t.dims()) model.factors.factors.emplace_back(dim, opts.rank);
  for (auto& a : model.factors.factors) out.push_back(a.data.data());
  model.lambda.assign(opts.rank, 1.0);
  std::vector<double> fits(std::max(1, opts.max_iters));
  int iters = 0;
  const int status = blco_cp_als(d, opts.rank, opts.max_iters, opts.tol, opts.seed,
                                 static_cast<int>(opts.strategy), &c, out.data(),
                                 model.lambda.data(), fits.data(), &iters);
  model.fit_history.assign(fits.begin(), fits.begin() + iters);
  if (status == BLCO_ERROR && std::string(blco_last_error()).rfind("cp_als: non-finite", 0) == 0)
    throw CpAlsError(blco_last_error(), model.fit_history);
  ck(status);
  return model;
}

double fit(const BlcoTensor& t, const CpModel& model, const ExecConfig& config) {
  model.factors.validate(t.dims());
  if (model.lambda.size() != model.factors.rank)
    throw FormatError("fit: lambda length does not match rank");
  const blco_tensor* d = device_tensor(t);
  const blco_exec_config c = to_c(config);
  const auto ptrs = factor_ptrs(model.factors);
  double f = 0;
  ck(blco_fit(d, ptrs.data(), model.lambda.data(), model.factors.rank, &c, &f));
  return f;
}

}  // namespace blco
