#include <cstdlib>
// host.cpp -- host-side pieces of the C ABI: errors, bit layout, batch table,
// config, partitioning and the host restatements of the seeded generators.
//
// Layout rules follow proj/src/layout.cpp:15-69 (make_layout) and the
// encode/decode functions at :71-124; batch spans follow
// proj/src/blco_format.cpp:136-147.
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>

#include "internal.hpp"
#include "synth.hpp"

namespace b200 {

namespace {
thread_local std::string t_msg;
thread_local int t_code = BLCO_OK;
}  // namespace

std::atomic<uint64_t> g_launches{0};

void set_error(int code, const std::string& msg) {
  t_code = code;
  t_msg = msg;
}

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  throw Status(BLCO_ECUDA, std::string("cuda: ") + cudaGetErrorString(e) + " in " + what + " (" +
                               file + ":" + std::to_string(line) + ")");
}

void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Status(BLCO_ECUDA, std::string("cuda: launch of ") + what + " failed: " +
                                 cudaGetErrorString(e));
}

namespace {
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, size_t> g_smem_granted;
std::map<std::tuple<int, const void*, int, size_t>, int> g_occupancy;
}  // namespace

void ensure_dyn_smem(const void* kernel, size_t bytes) {
  int dev = 0;
  B200_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(g_attr_mu);
  size_t& have = g_smem_granted[{dev, kernel}];
  if (bytes <= have) return;
  B200_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  have = bytes;
}

int blocks_per_sm(const void* kernel, int threads, size_t dyn_smem) {
  int dev = 0;
  B200_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(g_attr_mu);
  auto key = std::make_tuple(dev, kernel, threads, dyn_smem);
  auto it = g_occupancy.find(key);
  if (it != g_occupancy.end()) return it->second;
  int n = 0;
  B200_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, dyn_smem));
  g_occupancy[key] = n;
  return n;
}

namespace {
thread_local bool t_scratch = false;
}

ScratchScope::ScratchScope(bool on) : prev(t_scratch) { t_scratch = on; }
ScratchScope::~ScratchScope() { t_scratch = prev; }
bool scratch_active() { return t_scratch; }

void* scratch_alloc(size_t bytes) {
  int dev = 0;
  B200_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<int, bool> configured;
  {
    std::lock_guard<std::mutex> g(mu);
    if (!configured[dev]) {
      cudaMemPool_t pool;
      B200_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      uint64_t keep = uint64_t(4) << 30;  // cached between builds; the rest is released at syncs
      B200_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      configured[dev] = true;
    }
  }
  void* p = nullptr;
  B200_CUDA(cudaMallocAsync(&p, bytes, nullptr));
  return p;
}

void scratch_trim() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
  }
}

int sm_count() {
  int dev = 0;
  B200_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  B200_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  return cache[dev] = n > 0 ? n : 1;
}

bool poison_allocations() {
  static const bool on = std::getenv("BLCO_B200_POISON") != nullptr;
  return on;
}

int bits_for_extent(uint64_t extent) { return extent <= 1 ? 0 : 64 - __builtin_clzll(extent - 1); }

blco_layout make_layout(const uint64_t* dims, int order, int target_bits) {
  if (order < 1) throw_format("layout: at least one mode required");
  if (target_bits < 1 || target_bits > 64)
    throw_format("layout: target_bits must lie in [1, 64], got " + std::to_string(target_bits));
  if (order > BLCO_MAX_ORDER)
    throw_format("layout: order " + std::to_string(order) + " above the supported " +
                 std::to_string(BLCO_MAX_ORDER));
  blco_layout l;
  std::memset(&l, 0, sizeof l);
  l.order = order;
  l.target_bits = target_bits;
  int widest = 0;
  for (int m = 0; m < order; ++m) {
    if (dims[m] < 1) throw_format("layout: mode length must be >= 1");
    l.dims[m] = dims[m];
    l.mode_bits[m] = bits_for_extent(dims[m]);
    widest = std::max(widest, static_cast<int>(l.mode_bits[m]));
  }
  // Interleave level by level from the LSB; a mode drops out once its bits
  // are exhausted.  Count first so the >128 error fires before any write.
  int total = 0;
  for (int m = 0; m < order; ++m) total += l.mode_bits[m];
  if (total > BLCO_MAX_BITS)
    throw_format("layout: tensor needs " + std::to_string(total) +
                 " index bits, more than the 128 supported");
  int pos = 0;
  for (int level = 0; level < widest; ++level)
    for (int m = 0; m < order; ++m)
      if (level < l.mode_bits[m]) {
        l.imap_mode[pos] = static_cast<uint8_t>(m);
        l.imap_bit[pos] = static_cast<uint8_t>(level);
        ++pos;
      }
  l.total_bits = total;
  l.stripped_bits = total > target_bits ? total - target_bits : 0;
  const int kept = total - l.stripped_bits;
  for (int p = 0; p < kept; ++p) ++l.rem_bits[l.imap_mode[p]];
  int shift = 0;
  for (int m = 0; m < order; ++m) {
    l.field_shift[m] = shift;
    l.field_mask[m] = l.rem_bits[m] ? (~uint64_t{0} >> (64 - l.rem_bits[m])) : 0;
    shift += l.rem_bits[m];
  }
  if (shift == 0 && total > 0)
    throw_format("layout: every index bit stripped; no addressable field remains");
  return l;
}

uint64_t key_upper(const blco_layout& l, int mode, uint64_t key) {
  const int kept = l.total_bits - l.stripped_bits;
  uint64_t up = 0;
  for (int p = kept; p < l.total_bits; ++p)
    if (l.imap_mode[p] == mode) up |= ((key >> (p - kept)) & 1u) << (l.imap_bit[p] - l.rem_bits[mode]);
  return up;
}

void check_device_layout(const blco_layout& l) {
  if (l.order > BLCO_MAX_DEV_ORDER)
    throw_format("b200: order " + std::to_string(l.order) + " above the device limit of " +
                 std::to_string(BLCO_MAX_DEV_ORDER));
  for (int m = 0; m < l.order; ++m)
    if (l.dims[m] >= (uint64_t{1} << 32))
      throw_format("b200: mode length " + std::to_string(l.dims[m]) +
                   " needs 64-bit rows; the device path supports < 2^32");
  if (l.stripped_bits > 64)
    throw_format("layout: " + std::to_string(l.stripped_bits) +
                 " stripped bits do not fit the 64-bit block key");
}

}  // namespace b200

using namespace b200;

extern "C" {

const char* blco_last_error(void) { return t_msg.c_str(); }
int blco_abi_version(void) { return 1; }
void blco_set_error(int status, const char* msg) { set_error(status, msg ? msg : ""); }
uint64_t blco_kernel_launch_count(void) { return g_launches.load(); }

int blco_release_thread_caches(void) {
  return guarded([] {
    release_allmode_cache();
    release_det_cache();
    release_mttkrp_workspace();
    scratch_trim();
  });
}

int blco_make_layout(const uint64_t* dims, int order, int target_bits, blco_layout* out) {
  return guarded([&] { *out = make_layout(dims, order, target_bits); });
}

int blco_linearize(const blco_layout* l, const uint64_t* c, uint64_t* hi, uint64_t* lo) {
  return guarded([&] {
    unsigned __int128 a = 0;
    // position of bit k of mode m: walk the interleave map once
    for (int p = 0; p < l->total_bits; ++p) {
      const int m = l->imap_mode[p];
      if (c[m] >= l->dims[m]) throw_format("linearize: coordinate out of range");
      a |= static_cast<unsigned __int128>((c[m] >> l->imap_bit[p]) & 1u) << p;
    }
    for (int m = 0; m < l->order; ++m)
      if (c[m] >= l->dims[m]) throw_format("linearize: coordinate out of range");
    *hi = static_cast<uint64_t>(a >> 64);
    *lo = static_cast<uint64_t>(a);
  });
}

int blco_split_block_key(const blco_layout* l, uint64_t hi, uint64_t lo, uint64_t* key,
                         uint64_t* reenc) {
  return guarded([&] {
    const unsigned __int128 a = (static_cast<unsigned __int128>(hi) << 64) | lo;
    const int kept = l->total_bits - l->stripped_bits;
    if (l->stripped_bits > 64)
      throw_format("layout: " + std::to_string(l->stripped_bits) +
                   " stripped bits do not fit the 64-bit block key");
    *key = l->stripped_bits ? static_cast<uint64_t>(a >> kept) : 0;
    uint64_t r = 0;
    for (int p = 0; p < kept; ++p)
      r |= static_cast<uint64_t>((a >> p) & 1u) << (l->field_shift[l->imap_mode[p]] + l->imap_bit[p]);
    *reenc = r;
  });
}

int blco_encode_coords(const blco_layout* l, const uint64_t* c, uint64_t* key, uint64_t* reenc) {
  return guarded([&] {
    if (l->stripped_bits > 64)
      throw_format("layout: " + std::to_string(l->stripped_bits) +
                   " stripped bits do not fit the 64-bit block key");
    uint64_t r = 0, k = 0;
    for (int m = 0; m < l->order; ++m) {
      if (c[m] >= l->dims[m]) throw_format("encode: coordinate out of range");
      r |= (c[m] & l->field_mask[m]) << l->field_shift[m];
    }
    const int kept = l->total_bits - l->stripped_bits;
    for (int p = kept; p < l->total_bits; ++p)
      k |= ((c[l->imap_mode[p]] >> l->imap_bit[p]) & 1u) << (p - kept);
    *key = k;
    *reenc = r;
  });
}

int blco_delinearize(const blco_layout* l, uint64_t reenc, uint64_t key, uint64_t* c) {
  return guarded([&] {
    for (int m = 0; m < l->order; ++m)
      c[m] = (key_upper(*l, m, key) << l->rem_bits[m]) |
             ((reenc >> l->field_shift[m]) & l->field_mask[m]);
  });
}

int blco_interleaved_remainder(const blco_layout* l, uint64_t reenc, uint64_t* hi, uint64_t* lo) {
  return guarded([&] {
    unsigned __int128 a = 0;
    const int kept = l->total_bits - l->stripped_bits;
    for (int p = 0; p < kept; ++p) {
      const int m = l->imap_mode[p];
      a |= static_cast<unsigned __int128>((reenc >> (l->field_shift[m] + l->imap_bit[p])) & 1u) << p;
    }
    *hi = static_cast<uint64_t>(a >> 64);
    *lo = static_cast<uint64_t>(a);
  });
}

uint64_t blco_key_upper(const blco_layout* l, int mode, uint64_t key) {
  return key_upper(*l, mode, key);
}

uint64_t blco_batch_table(const uint64_t* block_nnz, uint64_t nblocks, uint64_t quota,
                          uint64_t* spans) {
  if (quota == 0) return 0;
  uint64_t n = 0;
  for (uint64_t b = 0; b < nblocks; ++b) {
    for (uint64_t off = 0; off < block_nnz[b]; off += quota, ++n) {
      if (!spans) continue;
      spans[3 * n + 0] = b;
      spans[3 * n + 1] = off;
      spans[3 * n + 2] = std::min(quota, block_nnz[b] - off);
    }
  }
  return n;
}

void blco_exec_config_default(blco_exec_config* c) {
  // proj/include/blco/exec.hpp:16-23 defaults
  c->workgroup_size = 128;
  c->tile_size = 32;
  c->coarsening = 4;
  c->num_compute_units = 108;
  c->num_factor_copies = 1;
  c->stash_slots = 32;
  c->deterministic = 0;
  c->num_threads = 0;
}

int blco_exec_config_validate(const blco_exec_config* c) {
  return guarded([&] {
    if (c->workgroup_size < 1 || c->tile_size < 1 || c->coarsening < 1 ||
        c->num_compute_units < 1 || c->num_factor_copies < 1 || c->stash_slots < 1)
      throw_format("exec: all config counts must be >= 1");
    if (c->tile_size > c->workgroup_size) throw_format("exec: tile_size exceeds workgroup_size");
    if (c->workgroup_size % c->tile_size != 0)
      throw_format("exec: tile_size must divide workgroup_size");
    if (c->num_threads < 0) throw_format("exec: num_threads must be >= 0");
  });
}

int blco_choose_strategy(uint64_t len, const blco_exec_config* c) {
  return len < static_cast<uint64_t>(c->num_compute_units) ? BLCO_STRATEGY_HIERARCHICAL
                                                           : BLCO_STRATEGY_REGISTER;
}

}  // extern "C"

namespace b200 {
// Strategy::Auto on B200: the register kernel for every mode length.  Its
// CTA bucket grouping already commits one RED per distinct target row per
// tile, and it measured faster than the hierarchical stash on every mode
// length tried (24 rows 0.59 vs 0.77 ms, 100 rows 0.42 vs 0.52 ms, the
// Delicious modes 5.4 vs 28 ms).  MttkrpStats::strategy still
// reports the reference's choose_strategy label.  BLCO_B200_AUTO=reference
// runs the reference's mapping instead.
int auto_kernel(uint64_t len, const blco_exec_config& c) {
  static const bool reference = [] {
    const char* e = std::getenv("BLCO_B200_AUTO");
    return e && std::string(e) == "reference";
  }();
  return reference ? blco_choose_strategy(len, &c) : BLCO_STRATEGY_REGISTER;
}
}  // namespace b200

extern "C" {

int blco_partition(const uint64_t* block_nnz, uint64_t nblocks, uint64_t quota, int nparts,
                   uint64_t* begin, uint64_t* end) {
  return guarded([&] {
    if (nparts < 1) throw_format("partition: nparts must be >= 1");
    if (quota < 1) throw_format("partition: quota must be >= 1");
    // Span boundaries in global element space; part p takes the spans whose
    // start lies in [p*total/n, (p+1)*total/n) -- contiguous, balanced to one span.
    uint64_t total = 0;
    for (uint64_t b = 0; b < nblocks; ++b) total += block_nnz[b];
    std::vector<uint64_t> cuts;  // span starts
    uint64_t base = 0;
    for (uint64_t b = 0; b < nblocks; ++b) {
      for (uint64_t off = 0; off < block_nnz[b]; off += quota) cuts.push_back(base + off);
      base += block_nnz[b];
    }
    size_t s = 0;
    for (int p = 0; p < nparts; ++p) {
      const uint64_t lo_target = static_cast<uint64_t>(
          (static_cast<unsigned __int128>(total) * p) / static_cast<unsigned>(nparts));
      while (s < cuts.size() && cuts[s] < lo_target) ++s;
      begin[p] = s < cuts.size() ? cuts[s] : total;
    }
    for (int p = 0; p < nparts; ++p) end[p] = p + 1 < nparts ? begin[p + 1] : total;
  });
}

int blco_factors_random(const uint64_t* dims, int order, uint64_t rank, uint64_t seed,
                        double* const* out) {
  return guarded([&] {
    if (rank < 1) throw_format("factors: rank must be >= 1");
    uint64_t i = 0;
    for (int m = 0; m < order; ++m)
      for (uint64_t j = 0; j < dims[m] * rank; ++j, ++i) out[m][j] = synth::factor_value(seed, i);
  });
}

int blco_synth_uniform_host(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed,
                            uint64_t* idx, double* vals) {
  return guarded([&] {
    synth::Feistel f = synth::make_feistel(dims, order, nnz, seed);
    for (uint64_t e = 0; e < nnz; ++e) {
      uint64_t x = f.permute(e);
      for (int m = 0; m < order; ++m) {
        idx[static_cast<uint64_t>(m) * nnz + e] = x % dims[m];
        x /= dims[m];
      }
      vals[e] = synth::element_value(seed, e);
    }
  });
}

int blco_merge_copies(const double* const* copies, uint64_t ncopies, uint64_t elems, double* out) {
  return guarded([&] {
    if (ncopies == 0) throw_format("merge_copies: no copies");
    std::memcpy(out, copies[0], elems * sizeof(double));
    for (uint64_t c = 1; c < ncopies; ++c)
      for (uint64_t i = 0; i < elems; ++i) out[i] += copies[c][i];
  });
}

int blco_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

}  // extern "C"
