// container.cu -- the `.blco` container, byte-compatible with the reference
// (proj/include/blco/blco_format.hpp:67-70; proj/src/blco_format.cpp:149-255):
//
//   "BLCO" | u16 version=1 | u16 order | u64 dims[order] | u16 target_bits |
//   u16 mode_bits[order] | u64 max_nnz_per_block | u64 block_count |
//   block_count x { u64 key | u64 nnz | u64 idx[nnz] | f64 vals[nnz] }
//
// little-endian.  Header and record I/O are host code; the per-element checks
// the reference runs on the host for every element of every block
// (read_blco_block, blco_format.cpp:201-227: field width, coordinates inside
// dims, strictly ascending ALTO order) run as one device kernel per block --
// at 4.7B elements the host loop would dominate a streamed run.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.hpp"

namespace b200 {
namespace {

struct CheckParams {
  int order;
  int kept;  // total - stripped
  uint64_t limit;  // 2^kept, or 0 when kept >= 64 (no width check)
  uint32_t dims[BLCO_MAX_DEV_ORDER];
  uint32_t base[BLCO_MAX_DEV_ORDER];
  uint32_t shift[BLCO_MAX_DEV_ORDER];
  uint64_t mask[BLCO_MAX_DEV_ORDER];
  uint8_t src_bit[64];  // interleaved position p -> bit position in the re-encoded index
};

// interleaved_remainder (layout.cpp:116-124): bit p of the remainder is bit
// src_bit[p] of the re-encoded index (kept <= 64, so it fits one word).
__device__ __forceinline__ uint64_t remainder(const CheckParams& c, uint64_t idx) {
  uint64_t r = 0;
  for (int p = 0; p < c.kept; ++p) r |= ((idx >> c.src_bit[p]) & 1ull) << p;
  return r;
}

// bit 0: index beyond the field width, bit 1: coordinate outside dims,
// bit 2: not strictly ascending in ALTO order
__global__ void k_check_block(CheckParams c, const uint64_t* __restrict__ idx, uint64_t n,
                              unsigned* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = idx[i];
    unsigned b = 0;
    if (c.limit && x >= c.limit) b |= 1u;
    for (int m = 0; m < c.order; ++m) {
      const uint64_t coord = c.base[m] | ((x >> c.shift[m]) & c.mask[m]);
      if (coord >= c.dims[m]) b |= 2u;
    }
    if (i > 0 && remainder(c, x) <= remainder(c, idx[i - 1])) b |= 4u;
    if (b) atomicOr(bad, b);
  }
}

CheckParams check_params(const blco_layout& l, uint64_t key) {
  CheckParams c{};
  c.order = l.order;
  c.kept = l.total_bits - l.stripped_bits;
  c.limit = c.kept >= 64 ? 0 : (uint64_t{1} << c.kept);
  for (int m = 0; m < l.order; ++m) {
    c.dims[m] = static_cast<uint32_t>(l.dims[m]);
    c.base[m] = static_cast<uint32_t>(key_upper(l, m, key) << l.rem_bits[m]);
    c.shift[m] = static_cast<uint32_t>(l.field_shift[m]);
    c.mask[m] = l.field_mask[m];
  }
  for (int p = 0; p < c.kept && p < 64; ++p)
    c.src_bit[p] = static_cast<uint8_t>(l.field_shift[l.imap_mode[p]] + l.imap_bit[p]);
  return c;
}

void validate_device(const blco_layout& l, uint64_t key, const uint64_t* d_idx, uint64_t n) {
  if (l.stripped_bits < 64 && key >= (uint64_t{1} << l.stripped_bits))
    throw_format("blco: block key out of range");
  if (!n) return;
  DevBuf<unsigned> bad(1);
  B200_CUDA(cudaMemset(bad.ptr, 0, sizeof(unsigned)));
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, sm_count() * 16));
  k_check_block<<<grid, 256>>>(check_params(l, key), d_idx, n, bad.ptr);
  count_launch();
  check_launch("k_check_block");
  unsigned h = 0;
  B200_CUDA(cudaMemcpy(&h, bad.ptr, sizeof h, cudaMemcpyDeviceToHost));
  if (h & 1u) throw_format("blco: re-encoded index exceeds field width");
  if (h & 2u) throw_format("blco: element de-linearizes outside dims");
  if (h & 4u) throw_format("blco: elements not in ascending ALTO order");
}

// ---- order-free element census (a checksum of checksums over a tensor):
// sum over elements of mix64(cell ^ mix64(value bits)) mod 2^64, where cell =
// sum_m c_m * prod_{k<m} dims[k] (mod 2^64) -- the mixed-radix cell id the
// synthetic generators draw, so the oracle can hash the generator's stream
// without storing it (oracle/blco_oracle.c orc_census_*).
__device__ __forceinline__ uint64_t census_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_census_block(CheckParams c, const uint64_t* __restrict__ idx, const double* __restrict__ vals,
                               uint64_t n, unsigned long long* __restrict__ sum) {
  uint64_t h = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = idx[i];
    uint64_t cell = 0, st = 1;
    for (int m = 0; m < c.order; ++m) {
      const uint64_t coord = c.base[m] | ((x >> c.shift[m]) & c.mask[m]);
      cell += coord * st;
      st *= c.dims[m];
    }
    h += census_mix(cell ^ census_mix(__double_as_longlong(vals[i])));
  }
  for (int d = 16; d > 0; d >>= 1) h += __shfl_down_sync(0xffffffffu, h, d);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(sum, static_cast<unsigned long long>(h));
}

// ---- raw little-endian I/O over a byte stream: a FILE* (blco_save/load,
// the file block source) or a caller's stream through the blco_read_fn /
// blco_write_fn hooks (the C++ API's std::istream / std::ostream).
struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

uint64_t file_read(void* ctx, void* dst, uint64_t n) { return std::fread(dst, 1, n, static_cast<FILE*>(ctx)); }
uint64_t file_write(void* ctx, const void* src, uint64_t n) {
  return std::fwrite(src, 1, n, static_cast<FILE*>(ctx));
}

struct ByteIn {
  blco_read_fn fn;
  void* ctx;
  void bytes(void* dst, uint64_t n) const {
    if (n && fn(ctx, dst, n) != n) throw Status(BLCO_EIO, "blco: truncated payload");
  }
  template <class T>
  T word() const {
    T v{};
    bytes(&v, sizeof(T));
    return v;
  }
};

struct ByteOut {
  blco_write_fn fn;
  void* ctx;
  void bytes(const void* src, uint64_t n) const {
    if (n && fn(ctx, src, n) != n) throw Status(BLCO_EIO, "blco: write failed");
  }
  template <class T>
  void word(T v) const {
    bytes(&v, sizeof(T));
  }
};

ByteIn in_of(FILE* f) { return ByteIn{file_read, f}; }
ByteOut out_of(FILE* f) { return ByteOut{file_write, f}; }

// read_blco_header (blco_format.cpp:173-191): the raw fields, unchecked
blco_container_header parse_header(const ByteIn& in) {
  char magic[4] = {};
  if (in.fn(in.ctx, magic, 4) != 4 || std::memcmp(magic, "BLCO", 4) != 0) throw_format("blco: bad magic");
  blco_container_header h{};
  h.version = in.word<uint16_t>();
  if (h.version != 1) throw_format("blco: unsupported format version " + std::to_string(h.version));
  h.order = in.word<uint16_t>();
  if (h.order < 1) throw_format("blco: order must be >= 1");
  if (h.order > BLCO_MAX_ORDER) throw_format("blco: order exceeds " + std::to_string(BLCO_MAX_ORDER));
  in.bytes(h.dims, h.order * sizeof(uint64_t));
  h.target_bits = in.word<uint16_t>();
  in.bytes(h.mode_bits, h.order * sizeof(uint16_t));
  h.max_nnz_per_block = in.word<uint64_t>();
  h.block_count = in.word<uint64_t>();
  return h;
}

// BlcoHeader::make_layout_checked (blco_format.cpp:193-199)
blco_layout checked_layout(const blco_container_header& h) {
  blco_layout l = make_layout(h.dims, h.order, h.target_bits);
  for (int m = 0; m < h.order; ++m)
    if (l.mode_bits[m] != h.mode_bits[m]) throw_format("blco: stored mode bit widths do not match dims");
  if (h.max_nnz_per_block < 1) throw_format("blco: max_nnz_per_block must be >= 1");
  return l;
}

struct Header {
  uint16_t version = 0;
  blco_layout layout{};
  uint64_t max_nnz = 0, nblocks = 0;
};

Header read_header(const ByteIn& in) {
  const blco_container_header raw = parse_header(in);
  return Header{raw.version, checked_layout(raw), raw.max_nnz_per_block, raw.block_count};
}

void write_header(const ByteOut& out, const blco_layout& l, uint64_t max_nnz, uint64_t nblocks) {
  out.bytes("BLCO", 4);
  out.word<uint16_t>(1);
  out.word<uint16_t>(static_cast<uint16_t>(l.order));
  out.bytes(l.dims, l.order * sizeof(uint64_t));
  out.word<uint16_t>(static_cast<uint16_t>(l.target_bits));
  for (int m = 0; m < l.order; ++m) out.word<uint16_t>(static_cast<uint16_t>(l.mode_bits[m]));
  out.word<uint64_t>(max_nnz);
  out.word<uint64_t>(nblocks);
}

void write_record(const ByteOut& out, uint64_t key, uint64_t n, const uint64_t* idx, const double* vals) {
  out.word<uint64_t>(key);
  out.word<uint64_t>(n);
  out.bytes(idx, n * sizeof(uint64_t));
  out.bytes(vals, n * sizeof(double));
}

// read_blco_block's record head (blco_format.cpp:201-207): key range, nnz
void read_record_head(const ByteIn& in, const blco_layout& l, uint64_t* key, uint64_t* n) {
  *key = in.word<uint64_t>();
  if (l.stripped_bits < 64 && *key >= (uint64_t{1} << l.stripped_bits)) throw_format("blco: block key out of range");
  *n = in.word<uint64_t>();
}

}  // namespace

void enqueue_block_check(const blco_layout& l, uint64_t key, const uint64_t* d_idx, uint64_t n, unsigned* d_bad,
                         cudaStream_t s) {
  if (!n) return;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, sm_count() * 16));
  k_check_block<<<grid, 256, 0, s>>>(check_params(l, key), d_idx, n, d_bad);
  count_launch();
  check_launch("k_check_block");
}

void throw_block_check(unsigned bad) {
  if (bad & 1u) throw_format("blco: re-encoded index exceeds field width");
  if (bad & 2u) throw_format("blco: element de-linearizes outside dims");
  if (bad & 4u) throw_format("blco: elements not in ascending ALTO order");
}

BlcoFileHeader read_blco_file_header(FILE* f) {
  const Header h = read_header(in_of(f));
  return BlcoFileHeader{h.version, h.layout, h.max_nnz, h.nblocks};
}

}  // namespace b200

using namespace b200;

extern "C" {

int blco_validate_block(const blco_layout* l, uint64_t key, uint64_t nnz, const uint64_t* idx, int device) {
  return guarded([&] {
    check_device_layout(*l);
    DeviceGuard dg(device);
    DevBuf<uint64_t> d(nnz);
    if (nnz) B200_CUDA(cudaMemcpy(d.ptr, idx, nnz * 8, cudaMemcpyHostToDevice));
    validate_device(*l, key, d.ptr, nnz);
  });
}

int blco_validate_block_device(const blco_layout* l, uint64_t key, uint64_t nnz, const uint64_t* d_idx) {
  return guarded([&] {
    check_device_layout(*l);
    validate_device(*l, key, d_idx, nnz);
  });
}

int blco_save(const blco_tensor* t, const char* path) {
  return guarded([&] {
    File f;
    f.f = std::fopen(path, "wb");
    if (!f.f) throw Status(BLCO_EIO, std::string("cannot open ") + path + " for writing");
    DeviceGuard dg(t->device);
    const ByteOut out = out_of(f.f);
    write_header(out, t->layout, t->max_nnz_per_block, t->nblocks());
    std::vector<uint64_t> idx;
    std::vector<double> vals;
    for (uint64_t b = 0; b < t->nblocks(); ++b) {
      const uint64_t o = t->offsets[b], n = t->offsets[b + 1] - o;
      idx.resize(n);
      vals.resize(n);
      if (n) {
        B200_CUDA(cudaMemcpy(idx.data(), t->idx.ptr + o, n * 8, cudaMemcpyDeviceToHost));
        B200_CUDA(cudaMemcpy(vals.data(), t->vals.ptr + o, n * 8, cudaMemcpyDeviceToHost));
      }
      write_record(out, t->keys[b], n, idx.data(), vals.data());
    }
    if (std::fflush(f.f) != 0) throw Status(BLCO_EIO, "blco: write failed");
  });
}

int blco_read_header(const char* path, blco_layout* layout, uint64_t* max_nnz, uint64_t* nblocks,
                     uint16_t* version) {
  return guarded([&] {
    File f;
    f.f = std::fopen(path, "rb");
    if (!f.f) throw Status(BLCO_EIO, std::string("cannot open ") + path);
    const Header h = read_header(in_of(f.f));
    if (layout) *layout = h.layout;
    if (max_nnz) *max_nnz = h.max_nnz;
    if (nblocks) *nblocks = h.nblocks;
    if (version) *version = h.version;
  });
}

// load_blco / deserialize_blco (blco_format.cpp:229-255): every block is
// validated on the device as it is read, then kept resident.
int blco_load(const char* path, int device, blco_tensor** out) {
  *out = nullptr;
  return guarded([&] {
    File f;
    f.f = std::fopen(path, "rb");
    if (!f.f) throw Status(BLCO_EIO, std::string("cannot open ") + path);
    const ByteIn in = in_of(f.f);
    const Header h = read_header(in);
    check_device_layout(h.layout);
    DeviceGuard dg(device);
    auto* t = new blco_tensor;
    try {
      t->layout = h.layout;
      t->device = device;
      t->max_nnz_per_block = h.max_nnz;
      std::vector<uint64_t> all_idx;
      std::vector<double> all_vals;
      uint64_t prev_key = 0;
      for (uint64_t b = 0; b < h.nblocks; ++b) {
        uint64_t key = 0, n = 0;
        read_record_head(in, h.layout, &key, &n);
        const size_t o = all_idx.size();
        all_idx.resize(o + n);
        all_vals.resize(o + n);
        in.bytes(all_idx.data() + o, n * 8);
        in.bytes(all_vals.data() + o, n * 8);
        DevBuf<uint64_t> d(n);
        if (n) B200_CUDA(cudaMemcpy(d.ptr, all_idx.data() + o, n * 8, cudaMemcpyHostToDevice));
        validate_device(h.layout, key, d.ptr, n);
        if (n == 0) throw_format("blco: empty block record");
        if (n > h.max_nnz) throw_format("blco: block exceeds max_nnz_per_block");
        if (b > 0 && key < prev_key) throw_format("blco: blocks not in ascending key order");
        prev_key = key;
        t->keys.push_back(key);
        t->offsets.push_back(o);
      }
      t->nnz = all_idx.size();
      t->offsets.push_back(t->nnz);
      t->idx.alloc(t->nnz);
      t->vals.alloc(t->nnz);
      if (t->nnz) {
        B200_CUDA(cudaMemcpy(t->idx.ptr, all_idx.data(), t->nnz * 8, cudaMemcpyHostToDevice));
        B200_CUDA(cudaMemcpy(t->vals.ptr, all_vals.data(), t->nnz * 8, cudaMemcpyHostToDevice));
      }
      finalize_tensor(*t);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

// ---- the container on a caller's byte stream (the C++ API's istream /
// ostream entry points: serialize_blco, read_blco_header, read_blco_block,
// deserialize_blco, FileBlockSource)
int blco_container_read_header(blco_read_fn fn, void* ctx, blco_container_header* out) {
  return guarded([&] { *out = parse_header(ByteIn{fn, ctx}); });
}

int blco_container_checked_layout(const blco_container_header* h, blco_layout* out) {
  return guarded([&] { *out = checked_layout(*h); });
}

int blco_container_read_block(blco_read_fn fn, void* ctx, const blco_layout* layout, uint64_t* key,
                              uint64_t* nnz, blco_alloc_fn alloc, void* alloc_ctx, int device) {
  return guarded([&] {
    const ByteIn in{fn, ctx};
    read_record_head(in, *layout, key, nnz);
    uint64_t* idx = nullptr;
    double* vals = nullptr;
    if (alloc(alloc_ctx, *nnz, &idx, &vals) != 0 || (*nnz && (!idx || !vals)))
      throw_error("blco: block allocation failed");
    in.bytes(idx, *nnz * sizeof(uint64_t));
    in.bytes(vals, *nnz * sizeof(double));
    check_device_layout(*layout);
    DeviceGuard dg(device);
    DevBuf<uint64_t> d(*nnz);
    if (*nnz) B200_CUDA(cudaMemcpy(d.ptr, idx, *nnz * 8, cudaMemcpyHostToDevice));
    validate_device(*layout, *key, d.ptr, *nnz);
  });
}

int blco_container_write_header(blco_write_fn fn, void* ctx, const blco_layout* layout,
                                uint64_t max_nnz_per_block, uint64_t block_count) {
  return guarded([&] { write_header(ByteOut{fn, ctx}, *layout, max_nnz_per_block, block_count); });
}

int blco_container_write_block(blco_write_fn fn, void* ctx, uint64_t key, uint64_t nnz, const uint64_t* idx,
                               const double* vals) {
  return guarded([&] { write_record(ByteOut{fn, ctx}, key, nnz, idx, vals); });
}

}  // extern "C"

extern "C" int blco_tensor_census(const blco_tensor* t, uint64_t* hash) {
  return guarded([&] {
    if (!t || !hash) throw_format("census: null argument");
    DeviceGuard dg(t->device);
    const blco_layout& l = t->layout;
    DevBuf<unsigned long long> sum(1);
    B200_CUDA(cudaMemset(sum.ptr, 0, sizeof(unsigned long long)));
    for (uint64_t b = 0; b < t->nblocks(); ++b) {
      const uint64_t n = t->offsets[b + 1] - t->offsets[b];
      if (!n) continue;
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, sm_count() * 16));
      k_census_block<<<grid, 256>>>(check_params(l, t->keys[b]), t->idx.ptr + t->offsets[b],
                                    t->vals.ptr + t->offsets[b], n, sum.ptr);
      count_launch();
      check_launch("k_census_block");
    }
    unsigned long long h = 0;
    B200_CUDA(cudaMemcpy(&h, sum.ptr, sizeof h, cudaMemcpyDeviceToHost));
    *hash = h;
  });
}
