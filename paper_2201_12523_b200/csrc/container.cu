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
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148 * 16));
  k_check_block<<<grid, 256>>>(check_params(l, key), d_idx, n, bad.ptr);
  count_launch();
  check_launch("k_check_block");
  unsigned h = 0;
  B200_CUDA(cudaMemcpy(&h, bad.ptr, sizeof h, cudaMemcpyDeviceToHost));
  if (h & 1u) throw_format("blco: re-encoded index exceeds field width");
  if (h & 2u) throw_format("blco: element de-linearizes outside dims");
  if (h & 4u) throw_format("blco: elements not in ascending ALTO order");
}

// ---- raw little-endian I/O
struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

template <class T>
void put(FILE* f, const T& v) {
  if (std::fwrite(&v, sizeof(T), 1, f) != 1) throw Status(BLCO_EIO, "blco: write failed");
}

template <class T>
T get(FILE* f) {
  T v{};
  if (std::fread(&v, sizeof(T), 1, f) != 1) throw Status(BLCO_EIO, "blco: truncated payload");
  return v;
}

void get_n(FILE* f, void* dst, size_t bytes) {
  if (bytes && std::fread(dst, 1, bytes, f) != bytes) throw Status(BLCO_EIO, "blco: truncated payload");
}

struct Header {
  uint16_t version = 0;
  blco_layout layout{};
  uint64_t max_nnz = 0, nblocks = 0;
};

// read_blco_header + make_layout_checked (blco_format.cpp:173-199)
Header read_header(FILE* f) {
  char magic[4] = {};
  if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "BLCO", 4) != 0)
    throw_format("blco: bad magic");
  Header h;
  h.version = get<uint16_t>(f);
  if (h.version != 1) throw_format("blco: unsupported format version " + std::to_string(h.version));
  const uint16_t order = get<uint16_t>(f);
  if (order < 1) throw_format("blco: order must be >= 1");
  std::vector<uint64_t> dims(order);
  get_n(f, dims.data(), order * 8);
  const uint16_t target = get<uint16_t>(f);
  std::vector<uint16_t> mb(order);
  get_n(f, mb.data(), order * 2);
  h.max_nnz = get<uint64_t>(f);
  h.nblocks = get<uint64_t>(f);
  h.layout = make_layout(dims.data(), order, target);
  for (int m = 0; m < order; ++m)
    if (h.layout.mode_bits[m] != mb[m]) throw_format("blco: stored mode bit widths do not match dims");
  if (h.max_nnz < 1) throw_format("blco: max_nnz_per_block must be >= 1");
  return h;
}

void write_header(FILE* f, const blco_layout& l, uint64_t max_nnz, uint64_t nblocks) {
  if (std::fwrite("BLCO", 1, 4, f) != 4) throw Status(BLCO_EIO, "blco: write failed");
  put<uint16_t>(f, 1);
  put<uint16_t>(f, static_cast<uint16_t>(l.order));
  for (int m = 0; m < l.order; ++m) put<uint64_t>(f, l.dims[m]);
  put<uint16_t>(f, static_cast<uint16_t>(l.target_bits));
  for (int m = 0; m < l.order; ++m) put<uint16_t>(f, static_cast<uint16_t>(l.mode_bits[m]));
  put<uint64_t>(f, max_nnz);
  put<uint64_t>(f, nblocks);
}

}  // namespace

void enqueue_block_check(const blco_layout& l, uint64_t key, const uint64_t* d_idx, uint64_t n, unsigned* d_bad,
                         cudaStream_t s) {
  if (!n) return;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148 * 16));
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
  const Header h = read_header(f);
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
    write_header(f.f, t->layout, t->max_nnz_per_block, t->nblocks());
    std::vector<uint64_t> idx;
    std::vector<double> vals;
    for (uint64_t b = 0; b < t->nblocks(); ++b) {
      const uint64_t o = t->offsets[b], n = t->offsets[b + 1] - o;
      put<uint64_t>(f.f, t->keys[b]);
      put<uint64_t>(f.f, n);
      idx.resize(n);
      vals.resize(n);
      if (n) {
        B200_CUDA(cudaMemcpy(idx.data(), t->idx.ptr + o, n * 8, cudaMemcpyDeviceToHost));
        B200_CUDA(cudaMemcpy(vals.data(), t->vals.ptr + o, n * 8, cudaMemcpyDeviceToHost));
        if (std::fwrite(idx.data(), 8, n, f.f) != n || std::fwrite(vals.data(), 8, n, f.f) != n)
          throw Status(BLCO_EIO, "blco: write failed");
      }
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
    const Header h = read_header(f.f);
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
    const Header h = read_header(f.f);
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
        const uint64_t key = get<uint64_t>(f.f);
        const uint64_t n = get<uint64_t>(f.f);
        if (h.layout.stripped_bits < 64 && key >= (uint64_t{1} << h.layout.stripped_bits))
          throw_format("blco: block key out of range");
        const size_t o = all_idx.size();
        all_idx.resize(o + n);
        all_vals.resize(o + n);
        get_n(f.f, all_idx.data() + o, n * 8);
        get_n(f.f, all_vals.data() + o, n * 8);
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

}  // extern "C"
