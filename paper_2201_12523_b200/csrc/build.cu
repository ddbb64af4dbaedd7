// build.cu -- BLCO construction on the device (K1 encode, K2 radix sort,
// K3 segment/chunk/gather) plus device-tensor management.
//
// Reference: build_blco, proj/src/blco_format.cpp:62-134.  The reference
// linearizes every non-zero to a <=128-bit ALTO index (layout.cpp:71-82),
// stable-sorts by it (:80-83), groups runs of equal block key rejecting
// duplicate tuples (:86-106), chunks every run into <= max_nnz_per_block
// pieces restarting at the run start (:107-110), stores the re-encoded
// index of each element (:115-126) and builds the batch table (:129-131).
//
// Device design:
//   K1 k_encode   : one thread per element; ALTO (lo, hi) via a constant-memory
//                   interleave map, re-encoded index via shift/mask.
//   K2 sort       : hand-written stable LSD radix sort (primitives.cu) of the
//                   64-bit low ALTO word carrying a 32-bit element id, then
//                   (total_bits > 64 only) a stable sort of the high word --
//                   LSD stability makes the pair sort equal to a 128-bit
//                   sort.  Keys are unique unless the input has duplicates, so
//                   any correct sort reproduces std::stable_sort's order.
//   K3 k_runs     : adjacent compare on the sorted ALTO words -> duplicate
//                   flag + key-run starts (stable compaction, primitives.cu);
//                   the host chunks the (few) runs; k_gather places idx/values.

#include <algorithm>
#include <chrono>
#include <functional>
#include <cstring>

#include "internal.hpp"
#include "synth.hpp"

namespace b200 {

namespace synth {
Feistel make_feistel(const uint64_t* dims, int order, uint64_t nnz, uint64_t seed) {
  unsigned __int128 cells = 1;
  for (int m = 0; m < order; ++m) cells *= dims[m];
  if (cells > static_cast<unsigned __int128>(UINT64_MAX))
    throw_format("synth: cell count exceeds 2^64-1");
  Feistel f{};
  f.cells = static_cast<uint64_t>(cells);
  if (nnz > f.cells) throw_format("synth: more non-zeros than cells");
  int kb = bits_for_extent(f.cells);
  if (kb & 1) ++kb;
  if (kb < 2) kb = 2;
  f.half = kb / 2;
  f.mask = (uint64_t{1} << f.half) - 1;
  for (int r = 0; r < 4; ++r) f.key[r] = mix64(seed + static_cast<uint64_t>(r + 1) * kGolden);
  return f;
}
}  // namespace synth

namespace {

struct EncodeParams {
  int order;
  int total_bits;
  int kept_bits;  // total - stripped
  uint32_t dims[BLCO_MAX_DEV_ORDER];
  uint32_t shift[BLCO_MAX_DEV_ORDER];
  uint64_t mask[BLCO_MAX_DEV_ORDER];
  uint8_t imap_mode[BLCO_MAX_BITS];
  uint8_t imap_bit[BLCO_MAX_BITS];
  // per-mode scatter table: bit k of coordinate m lands at
  // interleaved position pos[m][k] (k < mode_bits[m], layout.cpp:34-36)
  uint8_t mode_bits[BLCO_MAX_DEV_ORDER];
  uint8_t pos[BLCO_MAX_DEV_ORDER][32];
};

EncodeParams encode_params(const blco_layout& l) {
  EncodeParams p{};
  p.order = l.order;
  p.total_bits = l.total_bits;
  p.kept_bits = l.total_bits - l.stripped_bits;
  for (int m = 0; m < l.order; ++m) {
    p.dims[m] = static_cast<uint32_t>(l.dims[m]);
    p.shift[m] = static_cast<uint32_t>(l.field_shift[m]);
    p.mask[m] = l.field_mask[m];
  }
  std::memcpy(p.imap_mode, l.imap_mode, sizeof p.imap_mode);
  std::memcpy(p.imap_bit, l.imap_bit, sizeof p.imap_bit);
  for (int q = 0; q < l.total_bits && q < BLCO_MAX_BITS; ++q) {
    const int m = l.imap_mode[q], k = l.imap_bit[q];
    if (m < BLCO_MAX_DEV_ORDER && k < 32) p.pos[m][k] = static_cast<uint8_t>(q);
  }
  for (int m = 0; m < l.order && m < BLCO_MAX_DEV_ORDER; ++m)
    p.mode_bits[m] = static_cast<uint8_t>(std::min(32, l.mode_bits[m]));
  return p;
}

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t n, int per_thread = 1) {
  uint64_t g = (n + static_cast<uint64_t>(kThreads) * per_thread - 1) /
               (static_cast<uint64_t>(kThreads) * per_thread);
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(g, 1u << 30)));
}

// Host COO (u64, validated here) -> u32 device coordinates.
__global__ void k_narrow_coords(const uint64_t* __restrict__ in, uint32_t* __restrict__ out,
                                uint64_t n, uint64_t dim, unsigned* __restrict__ bad) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t c = in[i];
    if (c >= dim) atomicOr(bad, 1u);
    out[i] = static_cast<uint32_t>(c);
  }
}

__global__ void k_synth(synth::Feistel f, uint64_t seed, int order, uint64_t nnz,
                        const uint64_t* __restrict__ dims, uint32_t* __restrict__ coords,
                        double* __restrict__ vals) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t x = f.permute(e);
    for (int m = 0; m < order; ++m) {
      const uint64_t d = dims[m];
      coords[m * nnz + e] = static_cast<uint32_t>(x % d);
      x /= d;
    }
    vals[e] = synth::element_value(seed, e);
  }
}

// K1: ALTO words + re-encoded index; perm = element id.  Templated on the
// order so every coordinate stays in a register: mode m's bits are scattered
// to their interleaved positions through the per-mode table (linearize,
// layout.cpp:71-82, one shift/or per bit, no dynamically indexed arrays);
// the re-encoded index is sum_m (c_m & mask_m) << shift_m (encode_coords,
// layout.cpp:97-107).
template <int N>
__global__ void k_encode(EncodeParams p, uint64_t nnz, const uint32_t* __restrict__ coords,
                         uint64_t* __restrict__ alto_lo, uint64_t* __restrict__ alto_hi,
                         uint64_t* __restrict__ reenc, uint32_t* __restrict__ perm) {
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t r = 0, lo = 0, hi = 0;
#pragma unroll
    for (int m = 0; m < N; ++m) {
      const uint32_t c = __ldcs(coords + m * nnz + e);
      r |= (static_cast<uint64_t>(c) & p.mask[m]) << p.shift[m];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k >= p.mode_bits[m]) break;
        const uint64_t bit = (c >> k) & 1u;
        const int q = p.pos[m][k];
        if (q < 64) lo |= bit << q;
        else hi |= bit << (q - 64);
      }
    }
    alto_lo[e] = lo;
    if (alto_hi) alto_hi[e] = hi;
    reenc[e] = r;
    perm[e] = static_cast<uint32_t>(e);
  }
}

// K1 for orders <= 4: the bit scatter through byte tables in shared memory.
// tab[(m * 4 + j) * 256 + v] holds, as {lo.x, lo.y, hi.x, hi.y}, the ALTO
// bits that byte j = v of coordinate m deposits (bit 8j + i of mode m lands
// at pos[m][8j + i]), so an element costs ceil(b_m / 8) table loads per mode
// instead of one shift/or chain per bit (ncu on NELL-2: the bit loop issued
// ~735 instructions per 32 elements and ran at 0.75 TB/s).  Persistent grid:
// each CTA stages the N x 16 KB tables once.  Same bits as k_encode.
template <int N>
__global__ void __launch_bounds__(256) k_encode_lut(EncodeParams p, const uint4* __restrict__ lut, uint64_t nnz,
                                                    const uint32_t* __restrict__ coords,
                                                    uint64_t* __restrict__ alto_lo, uint64_t* __restrict__ alto_hi,
                                                    uint64_t* __restrict__ reenc, uint32_t* __restrict__ perm) {
  extern __shared__ uint4 tab[];  // [N][4][256]
  for (int i = threadIdx.x; i < N * 1024; i += blockDim.x) tab[i] = lut[i];
  __syncthreads();
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < nnz;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t c[N];
#pragma unroll
    for (int m = 0; m < N; ++m) c[m] = __ldcs(coords + m * nnz + e);
    uint64_t r = 0, lo = 0, hi = 0;
#pragma unroll
    for (int m = 0; m < N; ++m) {
      r |= (static_cast<uint64_t>(c[m]) & p.mask[m]) << p.shift[m];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (8 * j < p.mode_bits[m]) {
          const uint4 t = tab[(m * 4 + j) * 256 + ((c[m] >> (8 * j)) & 255u)];
          lo |= (static_cast<uint64_t>(t.y) << 32) | t.x;
          hi |= (static_cast<uint64_t>(t.w) << 32) | t.z;
        }
    }
    alto_lo[e] = lo;
    if (alto_hi) alto_hi[e] = hi;
    reenc[e] = r;
    perm[e] = static_cast<uint32_t>(e);
  }
}

// The byte tables of k_encode_lut for a layout (host, from pos / mode_bits).
std::vector<uint4> encode_lut(const EncodeParams& p) {
  std::vector<uint4> t(static_cast<size_t>(p.order) * 1024, make_uint4(0, 0, 0, 0));
  for (int m = 0; m < p.order; ++m)
    for (int j = 0; j < 4; ++j)
      for (int v = 0; v < 256; ++v) {
        uint64_t lo = 0, hi = 0;
        for (int i = 0; i < 8; ++i) {
          const int k = 8 * j + i;
          if (k >= p.mode_bits[m] || !((v >> i) & 1)) continue;
          const int q = p.pos[m][k];
          if (q < 64) lo |= uint64_t(1) << q;
          else hi |= uint64_t(1) << (q - 64);
        }
        t[(static_cast<size_t>(m) * 4 + j) * 256 + v] =
            make_uint4(static_cast<uint32_t>(lo), static_cast<uint32_t>(lo >> 32), static_cast<uint32_t>(hi),
                       static_cast<uint32_t>(hi >> 32));
      }
  return t;
}

using EncodeKernel = void (*)(EncodeParams, uint64_t, const uint32_t*, uint64_t*, uint64_t*, uint64_t*, uint32_t*);
EncodeKernel encode_kernel(int order) {
  switch (order) {
    case 1: return k_encode<1>;
    case 2: return k_encode<2>;
    case 3: return k_encode<3>;
    case 4: return k_encode<4>;
    case 5: return k_encode<5>;
    case 6: return k_encode<6>;
    case 7: return k_encode<7>;
    default: return k_encode<8>;
  }
}

// K1 launch: byte tables for orders <= 4 (lut: the device copy of
// encode_lut(ep), or null), the bit loop otherwise.
void launch_encode(const EncodeParams& ep, const uint4* lut, uint64_t n, const uint32_t* coords, uint64_t* lo,
                   uint64_t* hi, uint64_t* reenc, uint32_t* perm, cudaStream_t s) {
  if (lut && ep.order <= 4) {
    using LutKernel = void (*)(EncodeParams, const uint4*, uint64_t, const uint32_t*, uint64_t*, uint64_t*,
                               uint64_t*, uint32_t*);
    const LutKernel k = ep.order == 1   ? k_encode_lut<1>
                        : ep.order == 2 ? k_encode_lut<2>
                        : ep.order == 3 ? k_encode_lut<3>
                                        : k_encode_lut<4>;
    const size_t smem = static_cast<size_t>(ep.order) * 1024 * sizeof(uint4);
    ensure_dyn_smem(reinterpret_cast<const void*>(k), smem);
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>(grid_for(n), static_cast<uint64_t>(sm_count()) * 4)));
    k<<<grid, kThreads, smem, s>>>(ep, lut, n, coords, lo, hi, reenc, perm);
  } else {
    encode_kernel(ep.order)<<<grid_for(n, 4), kThreads, 0, s>>>(ep, n, coords, lo, hi, reenc, perm);
  }
  count_launch();
  check_launch("k_encode");
}

DevBuf<uint4> upload_encode_lut(const EncodeParams& ep) {
  DevBuf<uint4> d;
  if (ep.order > 4) return d;
  const std::vector<uint4> h = encode_lut(ep);
  d.alloc(h.size());
  B200_CUDA(cudaMemcpy(d.ptr, h.data(), h.size() * sizeof(uint4), cudaMemcpyHostToDevice));
  return d;
}

__global__ void k_iota(uint32_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(i);
}

template <class T>
__global__ void k_gather(const T* __restrict__ src, const uint32_t* __restrict__ perm,
                         T* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = src[perm[i]];
}

// K3: sorted ALTO (lo[], hi[] in sorted order) -> run-start flags + dup flag.
__global__ void k_runs(const uint64_t* __restrict__ lo, const uint64_t* __restrict__ hi,
                       uint64_t n, int kept_bits, int stripped, uint8_t* __restrict__ flag,
                       unsigned* __restrict__ dup) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    if (i == 0) {
      flag[0] = 1;
      continue;
    }
    const uint64_t l0 = lo[i - 1], l1 = lo[i];
    const uint64_t h0 = hi ? hi[i - 1] : 0, h1 = hi ? hi[i] : 0;
    if (l0 == l1 && h0 == h1) atomicOr(dup, 1u);
    uint8_t f = 0;
    if (stripped > 0) {
      const unsigned __int128 a0 = (static_cast<unsigned __int128>(h0) << 64) | l0;
      const unsigned __int128 a1 = (static_cast<unsigned __int128>(h1) << 64) | l1;
      f = static_cast<uint64_t>(a0 >> kept_bits) != static_cast<uint64_t>(a1 >> kept_bits);
    }
    flag[i] = f;
  }
}

__global__ void k_run_keys(const uint64_t* __restrict__ starts, uint64_t nruns,
                           const uint64_t* __restrict__ lo, const uint64_t* __restrict__ hi,
                           int kept_bits, uint64_t* __restrict__ keys) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (r >= nruns) return;
  const uint64_t i = starts[r];
  const unsigned __int128 a = (static_cast<unsigned __int128>(hi ? hi[i] : 0) << 64) | lo[i];
  keys[r] = static_cast<uint64_t>(a >> kept_bits);
}

__global__ void k_block_base(const uint64_t* __restrict__ keys, uint64_t nblocks, int order,
                             int kept, int total, const uint8_t* __restrict__ imap_mode,
                             const uint8_t* __restrict__ imap_bit, const int32_t* __restrict__ rem,
                             uint32_t* __restrict__ base) {
  const uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (b >= nblocks) return;
  uint64_t up[BLCO_MAX_DEV_ORDER] = {};
  const uint64_t key = keys[b];
  for (int p = kept; p < total; ++p) {
    const int m = imap_mode[p];
    up[m] |= ((key >> (p - kept)) & 1u) << (imap_bit[p] - rem[m]);
  }
  for (int m = 0; m < order; ++m) base[b * order + m] = static_cast<uint32_t>(up[m] << rem[m]);
}

__global__ void k_fill_factors(double* __restrict__ out, uint64_t n, uint64_t first,
                               uint64_t seed) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = synth::factor_value(seed, first + i);
}

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Core pipeline: device u32 coords (mode-major) + values -> tensor payload.
// Consumes (frees) coords/vals.
constexpr int kRetryDraws = -77;

// f[i] = 1 iff element i starts a run of equal ALTO words and its candidate
// id is <= max_id.
__global__ void k_first_of_run(const uint64_t* __restrict__ lo, const uint64_t* __restrict__ hi,
                               uint64_t n, uint8_t* __restrict__ f, const uint32_t* __restrict__ ids,
                               uint32_t max_id) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const bool first = i == 0 || lo[i] != lo[i - 1] || (hi && hi[i] != hi[i - 1]);
    f[i] = first && ids[i] <= max_id;
  }
}

// Candidate draws for the skewed generator: coordinate m of candidate j is
// floor(I_m * u^k) with u = unit(mix64(salted seed + (j*order + m + 1)*golden))
// (k = 1 uniform; larger k concentrates mass on low indices, a power law with
// density ~ x^(1/k - 1)); value = element_value(seed, j).
__global__ void k_draws(uint64_t seed, int order, int skew, uint64_t ncand,
                        const uint64_t* __restrict__ dims, uint32_t* __restrict__ coords,
                        double* __restrict__ vals) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < ncand;
       j += uint64_t(gridDim.x) * blockDim.x) {
    for (int m = 0; m < order; ++m) {
      const double u = synth::unit(synth::mix64((seed ^ synth::kDrawSalt) +
                                                 (j * order + m + 1) * synth::kGolden));
      coords[m * ncand + j] = synth::skewed_coord(u, dims[m], skew);
    }
    vals[j] = synth::element_value(seed, j);
  }
}

// ALTO-chunked generator (config 5): candidate j of a chunk is a uniform ALTO
// value in [lo, lo + width); it is a cell of the tensor iff every decoded
// coordinate lies inside dims.
constexpr uint64_t kAltoSalt = 0x8cb92ba72f3d8dd7ull;

__device__ __forceinline__ void alto_decode(const EncodeParams& p, uint64_t a, uint32_t (&c)[BLCO_MAX_DEV_ORDER]) {
  for (int m = 0; m < BLCO_MAX_DEV_ORDER; ++m) c[m] = 0;
  for (int q = 0; q < p.total_bits; ++q) c[p.imap_mode[q]] |= static_cast<uint32_t>((a >> q) & 1u) << p.imap_bit[q];
}

__global__ void k_alto_cand(EncodeParams p, uint64_t seed, uint64_t id0, uint64_t lo, uint64_t width,
                            uint64_t ncand, uint64_t* __restrict__ alto, uint32_t* __restrict__ ids,
                            uint8_t* __restrict__ flag) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < ncand;
       j += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = synth::mix64((seed ^ kAltoSalt) + (id0 + j + 1) * synth::kGolden);
    const uint64_t a = lo + (width ? r % width : r);
    bool ok = p.total_bits >= 64 || (a >> p.total_bits) == 0;
    uint32_t c[BLCO_MAX_DEV_ORDER];
    alto_decode(p, a, c);
    for (int m = 0; m < p.order; ++m) ok = ok && c[m] < p.dims[m];
    alto[j] = a;
    ids[j] = static_cast<uint32_t>(j);
    flag[j] = ok;
  }
}

__global__ void k_alto_finish(EncodeParams p, uint64_t seed, uint64_t id0, uint64_t n,
                              const uint64_t* __restrict__ alto, const uint32_t* __restrict__ ids,
                              uint64_t* __restrict__ out_idx, double* __restrict__ out_val) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t c[BLCO_MAX_DEV_ORDER];
    alto_decode(p, alto[i], c);
    uint64_t r = 0;
    for (int m = 0; m < p.order; ++m) r |= (static_cast<uint64_t>(c[m]) & p.mask[m]) << p.shift[m];
    out_idx[i] = r;
    out_val[i] = synth::element_value(seed, id0 + ids[i]);
  }
}

void build_from_device_coo(blco_tensor& t, DevBuf<uint32_t>& coords, DevBuf<double>& vals,
                           uint64_t nnz, blco_build_stats* stats, uint64_t dedup_target = 0) {
  const blco_layout& l = t.layout;
  if (nnz >= (uint64_t{1} << 32))
    throw_format("b200: device build handles < 2^32 elements per call (got " +
                 std::to_string(nnz) + ")");
  t.nnz = nnz;
  cudaStream_t s = 0;
  auto t0 = std::chrono::steady_clock::now();
  if (nnz == 0) {
    t.keys.clear();
    t.offsets.assign(1, 0);
    finalize_tensor(t);
    if (stats) *stats = blco_build_stats{};
    return;
  }
  const bool wide = l.total_bits > 64;
  NvtxRange nv_sort("blco build: encode + sort");
  DevBuf<uint64_t> lo(nnz), hi(wide ? nnz : 0), reenc(nnz);
  DevBuf<uint32_t> perm(nnz);
  const EncodeParams ep = encode_params(l);
  {
    const DevBuf<uint4> lut = upload_encode_lut(ep);
    launch_encode(ep, lut.ptr, nnz, coords.ptr, lo.ptr, hi.ptr, reenc.ptr, perm.ptr, s);
  }
  coords.reset();

  // K2: stable LSD radix sort (low word, then high word), payload = element id
  // (primitives.cu).  keys_out / perm_out receive the sorted low word and the
  // final order.
  DevBuf<uint64_t> keys_out(nnz);
  DevBuf<uint32_t> perm_out(nnz);
  const int lo_bits = std::max(1, std::min(64, l.total_bits));
  {
    bool alt = false;
    radix_sort_pairs<uint64_t>(lo.ptr, keys_out.ptr, perm.ptr, perm_out.ptr, nnz, 0, lo_bits, s, &alt);
    if (!alt) {  // result still in (lo, perm): move it into (keys_out, perm_out)
      std::swap(lo.ptr, keys_out.ptr);
      std::swap(perm.ptr, perm_out.ptr);
    }
  }
  DevBuf<uint64_t> sorted_hi;
  if (wide) {
    // high words in the low-word order, then a stable sort on them
    sorted_hi.alloc(nnz);
    k_gather<uint64_t><<<grid_for(nnz, 4), kThreads, 0, s>>>(hi.ptr, perm_out.ptr, sorted_hi.ptr, nnz);
    count_launch();
    check_launch("k_gather(hi)");
    // keep the sorted low word alongside: sort (hi, position) pairs, then
    // gather both the element ids and the low words through the positions
    DevBuf<uint32_t> pos(nnz), pos_alt(nnz);
    k_iota<<<grid_for(nnz, 4), kThreads, 0, s>>>(pos.ptr, nnz);
    count_launch();
    bool alt = false;
    radix_sort_pairs<uint64_t>(sorted_hi.ptr, hi.ptr, pos.ptr, pos_alt.ptr, nnz, 0, l.total_bits - 64, s, &alt);
    if (alt) {
      std::swap(sorted_hi.ptr, hi.ptr);
      std::swap(pos.ptr, pos_alt.ptr);
    }
    k_gather<uint32_t><<<grid_for(nnz, 4), kThreads, 0, s>>>(perm_out.ptr, pos.ptr, perm.ptr, nnz);
    k_gather<uint64_t><<<grid_for(nnz, 4), kThreads, 0, s>>>(keys_out.ptr, pos.ptr, lo.ptr, nnz);
    count_launch(2);
    check_launch("k_gather(order)");
    std::swap(perm.ptr, perm_out.ptr);
    std::swap(lo.ptr, keys_out.ptr);
  }
  lo.reset();
  hi.reset();
  perm.reset();
  B200_CUDA(cudaStreamSynchronize(s));
  if (stats) stats->sort_seconds = secs(t0);

  if (dedup_target) {
    // Candidates are sorted by (ALTO, candidate id): the first of each equal
    // run is the earliest draw.  Keep the dedup_target earliest unique draws.
    DevBuf<uint8_t> f(nnz);
    k_first_of_run<<<grid_for(nnz, 4), kThreads, 0, s>>>(keys_out.ptr, wide ? sorted_hi.ptr : nullptr,
                                                         nnz, f.ptr, perm_out.ptr, UINT32_MAX);
    count_launch();
    check_launch("k_first_of_run");
    DevBuf<uint32_t> ids(nnz), ids_alt(nnz), dummy(nnz), dummy_alt(nnz);
    const uint64_t uniq = select_flagged<uint32_t>(perm_out.ptr, f.ptr, nnz, ids.ptr, s);
    if (uniq < dedup_target) throw Status(kRetryDraws, "synth: not enough unique draws");
    bool alt = false;
    radix_sort_pairs<uint32_t>(ids.ptr, ids_alt.ptr, dummy.ptr, dummy_alt.ptr, uniq, 0, 32, s, &alt);
    uint32_t last = 0;
    B200_CUDA(cudaMemcpy(&last, (alt ? ids_alt.ptr : ids.ptr) + (dedup_target - 1), 4, cudaMemcpyDeviceToHost));
    k_first_of_run<<<grid_for(nnz, 4), kThreads, 0, s>>>(keys_out.ptr, wide ? sorted_hi.ptr : nullptr,
                                                         nnz, f.ptr, perm_out.ptr, last);
    count_launch();
    check_launch("k_first_of_run");
    // compact (lo, hi, perm) through the selection, preserving ALTO order
    DevBuf<uint64_t> lo2(dedup_target), hi2(wide ? dedup_target : 0);
    DevBuf<uint32_t> perm2(dedup_target);
    select_flagged<uint64_t>(keys_out.ptr, f.ptr, nnz, lo2.ptr, s);
    select_flagged<uint32_t>(perm_out.ptr, f.ptr, nnz, perm2.ptr, s);
    if (wide) select_flagged<uint64_t>(sorted_hi.ptr, f.ptr, nnz, hi2.ptr, s);
    keys_out = std::move(lo2);
    sorted_hi = std::move(hi2);
    perm_out = std::move(perm2);
    nnz = dedup_target;
    t.nnz = nnz;
  }

  // K3: key runs, duplicate check.
  NvtxRange nv_blocks("blco build: key runs + blocks");
  t0 = std::chrono::steady_clock::now();
  DevBuf<uint8_t> flags(nnz);
  DevBuf<unsigned> dflag(1);
  B200_CUDA(cudaMemsetAsync(dflag.ptr, 0, sizeof(unsigned), s));
  k_runs<<<grid_for(nnz, 4), kThreads, 0, s>>>(keys_out.ptr, wide ? sorted_hi.ptr : nullptr, nnz,
                                                l.total_bits - l.stripped_bits, l.stripped_bits,
                                                flags.ptr, dflag.ptr);
  count_launch();
  check_launch("k_runs");
  unsigned dup = 0;
  B200_CUDA(cudaMemcpyAsync(&dup, dflag.ptr, sizeof dup, cudaMemcpyDeviceToHost, s));
  B200_CUDA(cudaStreamSynchronize(s));
  if (dup) throw_format("blco: duplicate coordinate tuple in input");

  DevBuf<uint64_t> run_starts(nnz);
  const uint64_t nruns = select_flagged<uint64_t>(nullptr, flags.ptr, nnz, run_starts.ptr, s);
  std::vector<uint64_t> starts(nruns);
  B200_CUDA(cudaMemcpy(starts.data(), run_starts.ptr, nruns * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  // block key of each run, read off the sorted ALTO words at the run start
  std::vector<uint64_t> run_keys(nruns, 0);
  if (l.stripped_bits > 0 && nruns) {
    DevBuf<uint64_t> dkeys(nruns);
    k_run_keys<<<grid_for(nruns), kThreads, 0, s>>>(run_starts.ptr, nruns, keys_out.ptr,
                                                     wide ? sorted_hi.ptr : nullptr,
                                                     l.total_bits - l.stripped_bits, dkeys.ptr);
    count_launch();
    check_launch("k_run_keys");
    B200_CUDA(cudaMemcpy(run_keys.data(), dkeys.ptr, nruns * 8, cudaMemcpyDeviceToHost));
  }
  t.keys.clear();
  t.offsets.clear();
  for (uint64_t r = 0; r < nruns; ++r) {
    const uint64_t b = starts[r], e = r + 1 < nruns ? starts[r + 1] : nnz;
    // blocks of max_nnz_per_block from the run start (no overflow for huge caps)
    for (uint64_t c = b;; c += t.max_nnz_per_block) {
      t.keys.push_back(run_keys[r]);
      t.offsets.push_back(c);
      if (e - c <= t.max_nnz_per_block) break;
    }
  }
  t.offsets.push_back(nnz);
  if (stats) stats->block_seconds = secs(t0);

  // Re-encoded indices and values in ALTO order.
  NvtxRange nv_gather("blco build: gather payload");
  t0 = std::chrono::steady_clock::now();
  flags.reset();
  keys_out.reset();
  sorted_hi.reset();
  {
    ScratchScope keep(false);  // the payload outlives the build
    t.idx.alloc(nnz);
    t.vals.alloc(nnz);
  }
  k_gather<uint64_t><<<grid_for(nnz, 4), kThreads, 0, s>>>(reenc.ptr, perm_out.ptr, t.idx.ptr, nnz);
  k_gather<double><<<grid_for(nnz, 4), kThreads, 0, s>>>(vals.ptr, perm_out.ptr, t.vals.ptr, nnz);
  count_launch(2);
  check_launch("k_gather(payload)");
  B200_CUDA(cudaStreamSynchronize(s));
  if (stats) stats->reencode_seconds = secs(t0);

  t0 = std::chrono::steady_clock::now();
  finalize_tensor(t);
  if (stats) stats->batch_seconds = secs(t0);
}

// ---- multi-pass build of a host COO (>= 2^32 elements, or more than one
// device pass holds).  The element ids of the in-core sort are u32 and its
// temporaries cost ~60-80 B per element, so a large COO is built in ALTO-range
// passes: (1) the COO streams through the device in chunks once to histogram
// the top H bits of every element's ALTO index; (2) consecutive buckets are
// grouped into passes of at most `cap` elements; (3) per pass, the COO
// streams through again, the elements whose bucket falls in the pass are
// compacted on the device and built in core (sorted, duplicates rejected,
// re-encoded) with unbounded blocks, so its blocks are exactly its key runs;
// the pass's payload is appended to the tensor in ALTO order.  ALTO ranges
// are disjoint and ascending, so the concatenation is the global ALTO order
// and a duplicate can only meet its twin inside one pass.  Runs of one key
// that continue across a pass boundary are merged, then every run is cut
// every max_nnz_per_block elements from its start -- build_blco's chunking
// (blco_format.cpp:86-111), so the result is bit-identical to the in-core
// build and to the reference.
// ALTO range [lo, lo + 2^width) split into 2^hb buckets of 2^(width - hb):
// bucket(i) = (alto_i - lo) >> shift, or 0xffffffff outside the range
using u128 = unsigned __int128;
struct AltoRange {
  uint64_t lo_lo, lo_hi;  // lo as two words (kernel parameters stay POD)
  int width;              // log2 of the range size (<= 128)
  int shift;              // bucket width in bits
};

__device__ __forceinline__ u128 alto_of(const uint64_t* lo, const uint64_t* hi, uint64_t i) {
  return (static_cast<u128>(hi ? hi[i] : 0) << 64) | lo[i];
}

__global__ void k_bucket_of(const uint64_t* __restrict__ lo, const uint64_t* __restrict__ hi, uint64_t n,
                            AltoRange r, uint32_t* __restrict__ bucket) {
  const u128 base = (static_cast<u128>(r.lo_hi) << 64) | r.lo_lo;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const u128 a = alto_of(lo, hi, i);
    const u128 d = a - base;  // wraps above 2^128 when a < base: caught by the width test
    const bool in = a >= base && (r.width >= 128 || (d >> r.width) == 0);
    bucket[i] = in ? static_cast<uint32_t>(d >> r.shift) : 0xffffffffu;
  }
}

__global__ void k_bucket_hist(const uint32_t* __restrict__ bucket, uint64_t n,
                              unsigned long long* __restrict__ hist) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (bucket[i] != 0xffffffffu) atomicAdd(&hist[bucket[i]], 1ull);
}

// flag = ALTO in [plo, phi)
__global__ void k_range_flag(const uint64_t* __restrict__ lo, const uint64_t* __restrict__ hi, uint64_t n,
                             uint64_t plo_lo, uint64_t plo_hi, uint64_t phi_lo, uint64_t phi_hi,
                             uint8_t* __restrict__ flag) {
  const u128 plo = (static_cast<u128>(plo_hi) << 64) | plo_lo, phi = (static_cast<u128>(phi_hi) << 64) | phi_lo;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const u128 a = alto_of(lo, hi, i);
    flag[i] = a >= plo && a < phi;
  }
}

// append the selected chunk elements (ids sel[0..k)) at offset `off` of the
// pass buffers (coordinates mode-major with stride `cnt`)
__global__ void k_pass_append(const uint64_t* __restrict__ sel, uint64_t k, int order,
                              const uint32_t* __restrict__ cc, uint64_t cn, const double* __restrict__ cv,
                              uint32_t* __restrict__ pc, uint64_t cnt, double* __restrict__ pv, uint64_t off) {
  for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < k;
       j += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t e = sel[j];
    for (int m = 0; m < order; ++m) pc[m * cnt + off + j] = cc[m * cn + e];
    pv[off + j] = cv[e];
  }
}

// elements per device pass: BLCO_B200_BUILD_PASS_ELEMS overrides (tests);
// otherwise what the free memory holds at ~96 B per element, below 2^31
uint64_t build_pass_cap(uint64_t payload_bytes) {
  if (const char* e = std::getenv("BLCO_B200_BUILD_PASS_ELEMS")) {
    const uint64_t v = std::strtoull(e, nullptr, 10);
    if (v > 0) return v;
  }
  size_t free_b = 0, total_b = 0;
  B200_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const uint64_t room = free_b > payload_bytes + (uint64_t(4) << 30) ? free_b - payload_bytes - (uint64_t(4) << 30) : 0;
  return std::max<uint64_t>(1, std::min<uint64_t>((uint64_t{1} << 31) - 1, room / 96));
}

void build_host_passes(blco_tensor& t, const uint64_t* dims, int order, uint64_t nnz, const uint64_t* idx,
                       const double* vals, uint64_t cap, blco_build_stats* stats) {
  const blco_layout& l = t.layout;
  const uint64_t chunk = std::min<uint64_t>(cap, uint64_t{1} << 27);
  const EncodeParams ep = encode_params(l);
  const bool wide = l.total_bits > 64;
  cudaStream_t s = 0;
  auto t0 = std::chrono::steady_clock::now();
  DevBuf<uint64_t> stage(chunk), lo(chunk), hi(wide ? chunk : 0), reenc(chunk), sel(chunk);
  DevBuf<uint32_t> cc(chunk * order), perm(chunk), bucket(chunk);
  DevBuf<double> cv(chunk);
  DevBuf<uint8_t> flag(chunk);
  DevBuf<unsigned> bad(1);
  B200_CUDA(cudaMemset(bad.ptr, 0, sizeof(unsigned)));
  const DevBuf<uint4> lut = upload_encode_lut(ep);
  // one chunk of the host COO -> device coordinates, values and ALTO words
  auto load_chunk = [&](uint64_t c0, uint64_t n) {
    for (int m = 0; m < order; ++m) {
      B200_CUDA(cudaMemcpy(stage.ptr, idx + static_cast<uint64_t>(m) * nnz + c0, n * 8, cudaMemcpyHostToDevice));
      k_narrow_coords<<<grid_for(n, 4), kThreads>>>(stage.ptr, cc.ptr + static_cast<uint64_t>(m) * n, n, dims[m],
                                                    bad.ptr);
      count_launch();
    }
    B200_CUDA(cudaMemcpy(cv.ptr, vals + c0, n * 8, cudaMemcpyHostToDevice));
    launch_encode(ep, lut.ptr, n, cc.ptr, lo.ptr, hi.ptr, reenc.ptr, perm.ptr, s);
  };
  // (1)+(2) passes: histogram a range's ALTO sub-ranges (one stream of the
  // COO), group consecutive sub-ranges into passes of <= cap elements, and
  // refine any sub-range that alone holds more than cap (skewed tensors:
  // power-law coordinates share their high ALTO bits)
  struct Pass {
    u128 lo, hi;
    uint64_t cnt;
  };
  std::vector<Pass> passes;
  Pass cur{0, 0, 0};
  auto close = [&] {
    if (cur.cnt) passes.push_back(cur);
    cur = Pass{0, 0, 0};
  };
  std::function<void(u128, int)> split = [&](u128 base, int width) {
    const int hb = std::min(20, width);
    const int shift = width - hb;
    const uint64_t nb = uint64_t{1} << hb;
    DevBuf<unsigned long long> hist(nb);
    B200_CUDA(cudaMemset(hist.ptr, 0, nb * sizeof(unsigned long long)));
    const AltoRange r{static_cast<uint64_t>(base), static_cast<uint64_t>(base >> 64), width, shift};
    for (uint64_t c0 = 0; c0 < nnz; c0 += chunk) {
      const uint64_t n = std::min(chunk, nnz - c0);
      load_chunk(c0, n);
      k_bucket_of<<<grid_for(n, 4), kThreads, 0, s>>>(lo.ptr, wide ? hi.ptr : nullptr, n, r, bucket.ptr);
      k_bucket_hist<<<grid_for(n, 4), kThreads, 0, s>>>(bucket.ptr, n, hist.ptr);
      count_launch(2);
    }
    unsigned b = 0;
    B200_CUDA(cudaMemcpy(&b, bad.ptr, sizeof b, cudaMemcpyDeviceToHost));
    if (b) throw_format("coo: coordinate out of range");
    std::vector<uint64_t> h(nb);
    B200_CUDA(cudaMemcpy(h.data(), hist.ptr, nb * 8, cudaMemcpyDeviceToHost));
    for (uint64_t q = 0; q < nb; ++q) {
      if (!h[q]) continue;
      const u128 qlo = base + (static_cast<u128>(q) << shift), qhi = qlo + (static_cast<u128>(1) << shift);
      if (h[q] > cap) {  // one ALTO value holds one element, so refining terminates
        close();
        split(qlo, shift);
        continue;
      }
      if (cur.cnt + h[q] > cap) close();
      if (!cur.cnt) cur.lo = qlo;
      cur.hi = qhi;
      cur.cnt += h[q];
    }
  };
  split(0, l.total_bits);
  close();
  // (3) each pass built in core; payload appended in ALTO order
  {
    ScratchScope keep(false);  // the payload outlives the build
    t.idx.alloc(nnz);
    t.vals.alloc(nnz);
  }
  std::vector<uint64_t> run_keys, run_starts;  // global runs of equal key
  uint64_t out_off = 0;
  blco_build_stats acc{};
  for (const Pass& ps : passes) {
    const uint64_t cnt = ps.cnt;
    DevBuf<uint32_t> pc(cnt * order);
    DevBuf<double> pv(cnt);
    uint64_t off = 0;
    for (uint64_t c0 = 0; c0 < nnz; c0 += chunk) {
      const uint64_t n = std::min(chunk, nnz - c0);
      load_chunk(c0, n);
      k_range_flag<<<grid_for(n, 4), kThreads, 0, s>>>(lo.ptr, wide ? hi.ptr : nullptr, n,
                                                       static_cast<uint64_t>(ps.lo), static_cast<uint64_t>(ps.lo >> 64),
                                                       static_cast<uint64_t>(ps.hi), static_cast<uint64_t>(ps.hi >> 64),
                                                       flag.ptr);
      count_launch();
      const uint64_t k = select_flagged<uint64_t>(nullptr, flag.ptr, n, sel.ptr, s);
      if (off + k > cnt) throw_error("b200: multi-pass build: pass overflow");
      if (k) {
        k_pass_append<<<grid_for(k, 2), kThreads, 0, s>>>(sel.ptr, k, order, cc.ptr, n, cv.ptr, pc.ptr, cnt, pv.ptr,
                                                           off);
        count_launch();
        check_launch("k_pass_append");
      }
      off += k;
    }
    if (off != cnt) throw_error("b200: multi-pass build: pass count mismatch");
    blco_tensor tp;
    tp.layout = l;
    tp.device = t.device;
    tp.max_nnz_per_block = ~uint64_t{0};  // blocks = key runs
    blco_build_stats st{};
    build_from_device_coo(tp, pc, pv, cnt, &st);
    acc.sort_seconds += st.sort_seconds;
    acc.block_seconds += st.block_seconds;
    acc.reencode_seconds += st.reencode_seconds;
    B200_CUDA(cudaMemcpy(t.idx.ptr + out_off, tp.idx.ptr, cnt * 8, cudaMemcpyDeviceToDevice));
    B200_CUDA(cudaMemcpy(t.vals.ptr + out_off, tp.vals.ptr, cnt * 8, cudaMemcpyDeviceToDevice));
    for (uint64_t r = 0; r < tp.keys.size(); ++r) {
      if (r == 0 && !run_keys.empty() && run_keys.back() == tp.keys[0]) continue;  // run continues across passes
      run_keys.push_back(tp.keys[r]);
      run_starts.push_back(out_off + tp.offsets[r]);
    }
    out_off += cnt;
  }
  if (out_off != nnz) throw_error("b200: multi-pass build: element count mismatch");
  // global chunking of the runs (blco_format.cpp:86-111)
  t.nnz = nnz;
  t.keys.clear();
  t.offsets.clear();
  for (size_t r = 0; r < run_keys.size(); ++r) {
    const uint64_t b0 = run_starts[r], e = r + 1 < run_keys.size() ? run_starts[r + 1] : nnz;
    for (uint64_t c = b0;; c += t.max_nnz_per_block) {
      t.keys.push_back(run_keys[r]);
      t.offsets.push_back(c);
      if (e - c <= t.max_nnz_per_block) break;
    }
  }
  t.offsets.push_back(nnz);
  finalize_tensor(t);
  if (stats) {
    *stats = acc;
    stats->batch_seconds = secs(t0) - acc.sort_seconds - acc.block_seconds - acc.reencode_seconds;
  }
}

// Build temporaries come from the stream-ordered pool (ScratchScope) for
// builds up to 2^27 elements (a few GB of temporaries, kept cached between
// builds: NELL-2 26 -> 17 ms).  Larger builds allocate directly: their
// temporaries exceed the pool's cached 4 GiB, and the tensor's own payload
// allocation then waits while the driver trims tens of GB out of the pool
// (Amazon 0.65 -> 6.7 s measured with the pool).
bool scratch_build(uint64_t elems) { return elems <= (uint64_t{1} << 27); }

blco_tensor* new_tensor(const uint64_t* dims, int order, int target_bits, uint64_t max_nnz,
                        int device) {
  if (max_nnz < 1) throw_format("blco: max_nnz_per_block must be >= 1");
  auto* t = new blco_tensor;
  t->layout = make_layout(dims, order, target_bits);
  t->device = device;
  t->max_nnz_per_block = max_nnz;
  try {
    check_device_layout(t->layout);
  } catch (...) {
    delete t;
    throw;
  }
  return t;
}

}  // namespace

void finalize_tensor(blco_tensor& t) {
  const blco_layout& l = t.layout;
  const uint64_t nb = t.nblocks();
  {
    ScratchScope keep(false);  // lives with the tensor
    t.block_base.alloc(std::max<uint64_t>(1, nb * l.order));
  }
  if (nb) {
    DevBuf<uint64_t> dkeys(nb);
    DevBuf<uint8_t> dmode(BLCO_MAX_BITS), dbit(BLCO_MAX_BITS);
    DevBuf<int32_t> drem(BLCO_MAX_ORDER);
    B200_CUDA(cudaMemcpy(dkeys.ptr, t.keys.data(), nb * 8, cudaMemcpyHostToDevice));
    B200_CUDA(cudaMemcpy(dmode.ptr, l.imap_mode, BLCO_MAX_BITS, cudaMemcpyHostToDevice));
    B200_CUDA(cudaMemcpy(dbit.ptr, l.imap_bit, BLCO_MAX_BITS, cudaMemcpyHostToDevice));
    B200_CUDA(cudaMemcpy(drem.ptr, l.rem_bits, sizeof(int32_t) * BLCO_MAX_ORDER, cudaMemcpyHostToDevice));
    k_block_base<<<static_cast<unsigned>((nb + 127) / 128), 128>>>(
        dkeys.ptr, nb, l.order, l.total_bits - l.stripped_bits, l.total_bits, dmode.ptr, dbit.ptr,
        drem.ptr, t.block_base.ptr);
    count_launch();
    check_launch("k_block_base");
    B200_CUDA(cudaDeviceSynchronize());
  }
  std::lock_guard<std::mutex> g(t.mu);
  t.tiles.clear();
  t.panel_tiles.clear();
  t.span_bits.clear();
  t.det.clear();
}

const TileDesc* tile_table(const blco_tensor& t, uint32_t tile_elems, uint64_t* ntiles) {
  std::lock_guard<std::mutex> g(t.mu);
  auto it = t.tiles.find(tile_elems);
  if (it == t.tiles.end()) {
    std::vector<TileDesc> h;
    for (uint64_t b = 0; b < t.nblocks(); ++b)
      for (uint64_t off = t.offsets[b]; off < t.offsets[b + 1]; off += tile_elems)
        h.push_back(TileDesc{off, static_cast<uint32_t>(std::min<uint64_t>(tile_elems, t.offsets[b + 1] - off)),
                             static_cast<uint32_t>(b)});
    ScratchScope keep(false);  // cached with the tensor
    DevBuf<TileDesc> d(h.size());
    if (!h.empty()) {
      B200_CUDA(cudaMemcpy(d.ptr, h.data(), h.size() * sizeof(TileDesc), cudaMemcpyHostToDevice));
      // the table is read by kernels on any stream, non-blocking ones
      // included: wait until the staged pageable copy has landed
      B200_CUDA(cudaDeviceSynchronize());
    }
    it = t.tiles.emplace(tile_elems, std::move(d)).first;
  }
  *ntiles = it->second.n;
  return it->second.ptr;
}

}  // namespace b200

using namespace b200;

extern "C" {

int blco_build(const uint64_t* dims, int order, uint64_t nnz, const uint64_t* idx,
               const double* vals, int target_bits, uint64_t max_nnz, int device,
               blco_tensor** out, blco_build_stats* stats) {
  *out = nullptr;
  return guarded([&] {
    DeviceGuard dg(device);
    ScratchScope scratch(scratch_build(nnz));
    blco_tensor* t = new_tensor(dims, order, target_bits, max_nnz, device);
    try {
      const uint64_t cap = build_pass_cap(nnz * 16);
      if (nnz > cap) {  // beyond one device pass (>= 2^31 elements, or device memory)
        build_host_passes(*t, dims, order, nnz, idx, vals, cap, stats);
        *out = t;
        return;
      }
      DevBuf<uint32_t> coords(static_cast<size_t>(nnz) * order);
      DevBuf<double> dv(nnz);
      DevBuf<unsigned> bad(1);
      B200_CUDA(cudaMemset(bad.ptr, 0, sizeof(unsigned)));
      if (nnz) {
        // stage one mode at a time through a u64 buffer
        DevBuf<uint64_t> stage(nnz);
        for (int m = 0; m < order; ++m) {
          B200_CUDA(cudaMemcpy(stage.ptr, idx + static_cast<uint64_t>(m) * nnz, nnz * 8,
                               cudaMemcpyHostToDevice));
          k_narrow_coords<<<grid_for(nnz, 4), kThreads>>>(stage.ptr, coords.ptr + static_cast<uint64_t>(m) * nnz,
                                                          nnz, dims[m], bad.ptr);
          count_launch();
          check_launch("k_narrow_coords");
        }
        B200_CUDA(cudaMemcpy(dv.ptr, vals, nnz * 8, cudaMemcpyHostToDevice));
      }
      unsigned b = 0;
      B200_CUDA(cudaMemcpy(&b, bad.ptr, sizeof b, cudaMemcpyDeviceToHost));
      if (b) throw_format("coo: coordinate out of range");
      build_from_device_coo(*t, coords, dv, nnz, stats);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

int blco_build_synthetic(const uint64_t* dims, int order, uint64_t nnz, uint64_t seed,
                         int target_bits, uint64_t max_nnz, int device, blco_tensor** out,
                         blco_build_stats* stats) {
  *out = nullptr;
  return guarded([&] {
    DeviceGuard dg(device);
    ScratchScope scratch(scratch_build(nnz));
    blco_tensor* t = new_tensor(dims, order, target_bits, max_nnz, device);
    try {
      const synth::Feistel f = synth::make_feistel(dims, order, nnz, seed);
      DevBuf<uint32_t> coords(static_cast<size_t>(nnz) * order);
      DevBuf<double> dv(nnz);
      DevBuf<uint64_t> ddims(order);
      B200_CUDA(cudaMemcpy(ddims.ptr, dims, order * 8, cudaMemcpyHostToDevice));
      if (nnz) {
        k_synth<<<grid_for(nnz, 2), kThreads>>>(f, seed, order, nnz, ddims.ptr, coords.ptr, dv.ptr);
        count_launch();
        check_launch("k_synth");
      }
      build_from_device_coo(*t, coords, dv, nnz, stats);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

int blco_build_synthetic_draws(const uint64_t* dims, int order, uint64_t nnz, uint64_t seed,
                               int skew, int target_bits, uint64_t max_nnz, int device,
                               blco_tensor** out, blco_build_stats* stats) {
  *out = nullptr;
  return guarded([&] {
    if (skew < 1 || skew > 64) throw_format("synth: skew exponent must lie in [1, 64]");
    DeviceGuard dg(device);
    ScratchScope scratch(scratch_build(nnz + nnz / 2));
    DevBuf<uint64_t> ddims(order);
    B200_CUDA(cudaMemcpy(ddims.ptr, dims, order * 8, cudaMemcpyHostToDevice));
    uint64_t ncand = nnz + nnz / 8 + 1024;
    for (int attempt = 0;; ++attempt) {
      if (ncand >= (uint64_t{1} << 32) || attempt > 12)
        throw_format("synth: cannot draw " + std::to_string(nnz) + " unique coordinates");
      blco_tensor* t = new_tensor(dims, order, target_bits, max_nnz, device);
      try {
        DevBuf<uint32_t> coords(static_cast<size_t>(ncand) * order);
        DevBuf<double> dv(ncand);
        k_draws<<<grid_for(ncand, 2), kThreads>>>(seed, order, skew, ncand, ddims.ptr, coords.ptr, dv.ptr);
        count_launch();
        check_launch("k_draws");
        build_from_device_coo(*t, coords, dv, ncand, stats, nnz);
      } catch (const Status& st) {
        delete t;
        if (st.code != kRetryDraws) throw;
        ncand = ncand * 3 / 2 + 1024;
        continue;
      } catch (...) {
        delete t;
        throw;
      }
      *out = t;
      return;
    }
  });
}

int blco_synth_alto_chunk(const uint64_t* dims, int order, uint64_t chunk, uint64_t nchunks,
                          uint64_t ncand, uint64_t seed, int device, uint64_t* host_idx,
                          double* host_vals, uint64_t* count) {
  return guarded([&] {
    const blco_layout l = make_layout(dims, order, 64);
    check_device_layout(l);
    if (l.stripped_bits != 0 || l.total_bits < 1)
      throw_format("synth: ALTO-chunked generation needs a layout with no stripped bits");
    if (nchunks < 1 || chunk >= nchunks) throw_format("synth: chunk out of range");
    if (ncand >= (uint64_t{1} << 32)) throw_format("synth: too many candidates per chunk");
    const unsigned __int128 space = static_cast<unsigned __int128>(1) << l.total_bits;
    const uint64_t width = static_cast<uint64_t>((space + nchunks - 1) / nchunks);
    const uint64_t lo = static_cast<uint64_t>(space * chunk / nchunks);
    DeviceGuard dg(device);
    ScratchScope scratch(scratch_build(ncand));
    cudaStream_t s = 0;
    DevBuf<uint64_t> alto(ncand), alto_s(ncand), out_idx(ncand);
    DevBuf<uint32_t> ids(ncand), ids_s(ncand), ids_sel(ncand);
    DevBuf<uint8_t> flag(ncand);
    DevBuf<double> out_val(ncand);
    const EncodeParams ep = encode_params(l);
    // 1. candidates uniform in the chunk's ALTO range, valid iff every
    //    decoded coordinate lies inside dims
    k_alto_cand<<<grid_for(ncand, 2), kThreads, 0, s>>>(ep, seed, chunk * ncand, lo, width, ncand, alto.ptr,
                                                        ids.ptr, flag.ptr);
    count_launch();
    check_launch("k_alto_cand");
    const uint64_t nv = select_flagged<uint64_t>(alto.ptr, flag.ptr, ncand, alto_s.ptr, s);
    select_flagged<uint32_t>(ids.ptr, flag.ptr, ncand, ids_s.ptr, s);
    // 2. ALTO order (stable: equal keys keep candidate order)
    bool alt = false;
    radix_sort_pairs<uint64_t>(alto_s.ptr, alto.ptr, ids_s.ptr, ids.ptr, nv, 0, l.total_bits, s, &alt);
    if (!alt) {
      std::swap(alto_s.ptr, alto.ptr);
      std::swap(ids_s.ptr, ids.ptr);
    }
    // 3. duplicates: keep the first (earliest) candidate of each equal run
    k_first_of_run<<<grid_for(nv, 4), kThreads, 0, s>>>(alto.ptr, nullptr, nv, flag.ptr, ids.ptr, UINT32_MAX);
    count_launch();
    check_launch("k_first_of_run");
    const uint64_t n = select_flagged<uint64_t>(alto.ptr, flag.ptr, nv, alto_s.ptr, s);
    select_flagged<uint32_t>(ids.ptr, flag.ptr, nv, ids_sel.ptr, s);
    alto = std::move(alto_s);
    if (n) {
      k_alto_finish<<<grid_for(n, 2), kThreads, 0, s>>>(ep, seed, chunk * ncand, n, alto.ptr, ids_sel.ptr,
                                                         out_idx.ptr, out_val.ptr);
      count_launch();
      check_launch("k_alto_finish");
      B200_CUDA(cudaMemcpy(host_idx, out_idx.ptr, n * 8, cudaMemcpyDeviceToHost));
      B200_CUDA(cudaMemcpy(host_vals, out_val.ptr, n * 8, cudaMemcpyDeviceToHost));
    }
    *count = n;
  });
}

int blco_synth_draws_host(int order, const uint64_t* dims, uint64_t ncand, uint64_t seed, int skew,
                          uint64_t* idx, double* vals) {
  return guarded([&] {
    for (uint64_t j = 0; j < ncand; ++j) {
      for (int m = 0; m < order; ++m) {
        const double u = synth::unit(synth::mix64((seed ^ synth::kDrawSalt) +
                                                   (j * order + m + 1) * synth::kGolden));
        idx[static_cast<uint64_t>(m) * ncand + j] = synth::skewed_coord(u, dims[m], skew);
      }
      vals[j] = synth::element_value(seed, j);
    }
  });
}

int blco_tensor_upload(const blco_layout* layout, uint64_t max_nnz, uint64_t nblocks,
                       const uint64_t* keys, const uint64_t* block_nnz, const uint64_t* const* idx,
                       const double* const* vals, int device, blco_tensor** out) {
  *out = nullptr;
  return guarded([&] {
    DeviceGuard dg(device);
    blco_tensor* t = new_tensor(layout->dims, layout->order, layout->target_bits,
                                std::max<uint64_t>(1, max_nnz), device);
    try {
      uint64_t total = 0;
      for (uint64_t b = 0; b < nblocks; ++b) {
        t->keys.push_back(keys[b]);
        t->offsets.push_back(total);
        total += block_nnz[b];
      }
      t->offsets.push_back(total);
      t->nnz = total;
      t->idx.alloc(total);
      t->vals.alloc(total);
      for (uint64_t b = 0; b < nblocks; ++b) {
        if (!block_nnz[b]) continue;
        B200_CUDA(cudaMemcpy(t->idx.ptr + t->offsets[b], idx[b], block_nnz[b] * 8, cudaMemcpyHostToDevice));
        B200_CUDA(cudaMemcpy(t->vals.ptr + t->offsets[b], vals[b], block_nnz[b] * 8, cudaMemcpyHostToDevice));
      }
      finalize_tensor(*t);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

int blco_tensor_slice(const blco_tensor* src, uint64_t begin, uint64_t end, int device,
                      blco_tensor** out) {
  *out = nullptr;
  return guarded([&] {
    if (begin > end || end > src->nnz) throw_format("slice: element range out of bounds");
    DeviceGuard dg(device);
    blco_tensor* t = new_tensor(src->layout.dims, src->layout.order, src->layout.target_bits,
                                src->max_nnz_per_block, device);
    try {
      for (uint64_t b = 0; b < src->nblocks(); ++b) {
        const uint64_t lo = std::max(begin, src->offsets[b]), hi = std::min(end, src->offsets[b + 1]);
        if (lo >= hi) continue;
        t->keys.push_back(src->keys[b]);
        t->offsets.push_back(lo - begin);
      }
      t->offsets.push_back(end - begin);
      t->nnz = end - begin;
      t->idx.alloc(t->nnz);
      t->vals.alloc(t->nnz);
      if (t->nnz) {
        B200_CUDA(cudaMemcpyPeer(t->idx.ptr, device, src->idx.ptr + begin, src->device, t->nnz * 8));
        B200_CUDA(cudaMemcpyPeer(t->vals.ptr, device, src->vals.ptr + begin, src->device, t->nnz * 8));
      }
      finalize_tensor(*t);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

int blco_tensor_info(const blco_tensor* t, blco_layout* layout, uint64_t* nblocks, uint64_t* nnz,
                     uint64_t* max_nnz) {
  return guarded([&] {
    if (layout) *layout = t->layout;
    if (nblocks) *nblocks = t->nblocks();
    if (nnz) *nnz = t->nnz;
    if (max_nnz) *max_nnz = t->max_nnz_per_block;
  });
}

int blco_tensor_blocks(const blco_tensor* t, uint64_t* keys, uint64_t* block_nnz) {
  return guarded([&] {
    for (uint64_t b = 0; b < t->nblocks(); ++b) {
      if (keys) keys[b] = t->keys[b];
      if (block_nnz) block_nnz[b] = t->offsets[b + 1] - t->offsets[b];
    }
  });
}

int blco_tensor_download(const blco_tensor* t, uint64_t* idx, double* vals) {
  return guarded([&] {
    DeviceGuard dg(t->device);
    if (!t->nnz) return;
    if (idx) B200_CUDA(cudaMemcpy(idx, t->idx.ptr, t->nnz * 8, cudaMemcpyDeviceToHost));
    if (vals) B200_CUDA(cudaMemcpy(vals, t->vals.ptr, t->nnz * 8, cudaMemcpyDeviceToHost));
  });
}

int blco_tensor_device_ptrs(const blco_tensor* t, const uint64_t** idx, const double** vals) {
  return guarded([&] {
    *idx = t->idx.ptr;
    *vals = t->vals.ptr;
  });
}

void blco_tensor_free(blco_tensor* t) {
  if (!t) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(t->device);
  delete t;
  cudaSetDevice(prev);
}

int blco_factors_random_device(const uint64_t* dims, int order, uint64_t rank, uint64_t seed,
                               double* const* d_out, void* stream) {
  return guarded([&] {
    if (rank < 1) throw_format("factors: rank must be >= 1");
    uint64_t first = 0;
    for (int m = 0; m < order; ++m) {
      const uint64_t n = dims[m] * rank;
      if (n) {
        k_fill_factors<<<grid_for(n, 4), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(d_out[m], n, first, seed);
        count_launch();
        check_launch("k_fill_factors");
      }
      first += n;
    }
  });
}

}  // extern "C"
