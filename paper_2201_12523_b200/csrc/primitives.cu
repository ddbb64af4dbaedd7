// primitives.cu -- hand-written device primitives for BLCO construction:
// a stable LSD radix sort of (key, u32 payload) pairs, an exclusive scan and a
// flagged compaction.  They replace CUB on the construction path (K2/K3);
// CUB's DeviceRadixSort stays only as the cross-check in the GPU tests.
//
// Radix sort, per 8-bit digit pass over tiles of 2048 elements (256 threads x
// 8 items):
//   k_digit_hist : per-tile 256-bin histogram -> hist[digit * ntiles + tile]
//   scan         : exclusive scan of hist (digit-major) -> global offsets
//   k_digit_scatter : stable in-tile ranks (warp __match_any_sync against
//                  per-warp digit histograms), one block scan, the tile
//                  sorted by digit in shared memory, then written out as
//                  coalesced digit runs at offset[digit][tile].
// HBM traffic per pass: keys read twice, payload once, both written once.
#include <algorithm>

#include "internal.hpp"

namespace b200 {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;
constexpr int kSortTile = kSortThreads * kSortItems;  // 2048
constexpr int kDigits = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = 256 * kScanItems;

template <class K>
__global__ void __launch_bounds__(kSortThreads) k_digit_hist(const K* __restrict__ keys, uint64_t n, int shift,
                                                           uint32_t dmask, uint64_t ntiles,
                                                           uint64_t* __restrict__ hist) {
  __shared__ uint32_t h[kDigits];
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t base = tile * kSortTile;
#pragma unroll
    for (int s = 0; s < kSortItems; ++s) {
      const uint64_t e = base + s * kSortThreads + threadIdx.x;
      if (e < n) atomicAdd(&h[static_cast<uint32_t>(keys[e] >> shift) & dmask], 1u);
    }
    __syncthreads();
    hist[static_cast<uint64_t>(threadIdx.x) * ntiles + tile] = h[threadIdx.x];
    __syncthreads();
  }
}

// Stable scatter of one tile, staged through shared memory so the global
// writes are digit runs (coalesced) instead of one random store per element:
//   1. warp w ranks its 256 elements (w*256 + i*32 + lane, i = 0..7, i.e.
//      in element order) with __match_any_sync against a per-warp digit
//      histogram in shared memory -- no block barrier per item;
//   2. one block scan over (digit, warp) gives each element's position in
//      the tile sorted by digit (stable: digit, then warp, then item, lane);
//   3. keys and payloads are scattered into shared memory at those
//      positions, then written out in position order: position p of digit d
//      goes to offsets[d][tile] + (p - tile_start[d]), so neighbouring
//      threads write neighbouring addresses.
template <class K>
__global__ void __launch_bounds__(kSortThreads) k_digit_scatter(const K* __restrict__ keys_in,
                                                              const uint32_t* __restrict__ vals_in, uint64_t n,
                                                              int shift, uint32_t dmask, uint64_t ntiles,
                                                              const uint64_t* __restrict__ offsets,
                                                              K* __restrict__ keys_out,
                                                              uint32_t* __restrict__ vals_out) {
  constexpr int W = kSortThreads / 32;
  __shared__ uint32_t whist[W][kDigits];   // per-warp digit counts -> tile positions
  __shared__ uint32_t dstart[kDigits];     // first tile position of each digit
  __shared__ uint64_t gbase[kDigits];      // global offset of the digit's run for this tile
  __shared__ uint32_t wsum[W];
  extern __shared__ __align__(16) unsigned char stage_raw[];  // the tile, sorted by digit
  K* skeys = reinterpret_cast<K*>(stage_raw);
  uint32_t* svals = reinterpret_cast<uint32_t*>(stage_raw + sizeof(K) * kSortTile);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t base = tile * kSortTile;
    const int cnt = static_cast<int>(n - base < uint64_t(kSortTile) ? n - base : kSortTile);
    for (int w = 0; w < W; ++w) whist[w][threadIdx.x] = 0;
    gbase[threadIdx.x] = offsets[static_cast<uint64_t>(threadIdx.x) * ntiles + tile];
    __syncthreads();
    K key[kSortItems];
    uint32_t val[kSortItems], rank[kSortItems];
    uint32_t dig[kSortItems];
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const int e = warp * (32 * kSortItems) + i * 32 + lane;
      const bool ok = e < cnt;
      key[i] = ok ? keys_in[base + e] : K{};
      val[i] = ok ? vals_in[base + e] : 0u;
      dig[i] = ok ? static_cast<uint32_t>(key[i] >> shift) & dmask : kDigits;
    }
#pragma unroll
    for (int i = 0; i < kSortItems; ++i) {
      const unsigned peers = __match_any_sync(0xffffffffu, dig[i]);
      const uint32_t before = __popc(peers & ((1u << lane) - 1u));
      uint32_t prior = 0;
      if (dig[i] < kDigits) prior = whist[warp][dig[i]];
      __syncwarp();
      rank[i] = prior + before;
      if (dig[i] < kDigits && before == 0) whist[warp][dig[i]] = prior + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // exclusive scan over (digit, warp) in digit-major order: thread t owns digit t
    uint32_t tot = 0;
    uint32_t mine[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      mine[w] = tot;
      tot += whist[w][threadIdx.x];
    }
    uint32_t x = tot;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t woff = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) woff += w < warp ? wsum[w] : 0;
    const uint32_t start = woff + x - tot;
    dstart[threadIdx.x] = start;
#pragma unroll
    for (int w = 0; w < W; ++w) whist[w][threadIdx.x] = start + mine[w];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortItems; ++i)
      if (dig[i] < kDigits) {
        const uint32_t pos = whist[warp][dig[i]] + rank[i];
        skeys[pos] = key[i];
        svals[pos] = val[i];
      }
    __syncthreads();
#pragma unroll 4
    for (int i = 0; i < kSortItems; ++i) {
      const int p = i * kSortThreads + threadIdx.x;
      if (p < cnt) {
        const K k = skeys[p];
        const uint32_t d = static_cast<uint32_t>(k >> shift) & dmask;
        const uint64_t g = gbase[d] + (p - dstart[d]);
        keys_out[g] = k;
        vals_out[g] = svals[p];
      }
    }
    __syncthreads();
  }
}

// Exclusive scan of u64 values, chunk by chunk; chunk totals to sums.
__global__ void __launch_bounds__(256) k_scan_chunks(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                   uint64_t n, uint64_t* __restrict__ sums) {
  __shared__ uint64_t warp_tot[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = blockIdx.x * uint64_t(kScanTile) + threadIdx.x * uint64_t(kScanItems);
  uint64_t v[kScanItems], run = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    const uint64_t x = v[i];
    v[i] = run;
    run += x;
  }
  uint64_t x = run;
#pragma unroll
  for (int dd = 1; dd < 32; dd <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, dd);
    if (lane >= dd) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  uint64_t woff = 0;
  for (int w = 0; w < warp; ++w) woff += warp_tot[w];
  const uint64_t toff = woff + x - run;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) out[base + i] = toff + v[i];
  if (threadIdx.x == 255) sums[blockIdx.x] = woff + x;
}

__global__ void k_add_chunk_offsets(uint64_t* __restrict__ out, uint64_t n, const uint64_t* __restrict__ offs) {
  const uint64_t add = offs[blockIdx.x];
  const uint64_t base = blockIdx.x * uint64_t(kScanTile);
  for (int i = threadIdx.x; i < kScanTile; i += blockDim.x)
    if (base + i < n) out[base + i] += add;
}

// Per-tile flag counts for compaction.
__global__ void __launch_bounds__(256) k_flag_counts(const uint8_t* __restrict__ flags, uint64_t n,
                                                   uint64_t* __restrict__ counts) {
  __shared__ uint32_t c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  const uint64_t base = blockIdx.x * uint64_t(kScanTile);
  uint32_t mine = 0;
  for (int i = threadIdx.x; i < kScanTile; i += blockDim.x)
    if (base + i < n) mine += flags[base + i] != 0;
  for (int dd = 16; dd > 0; dd >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, dd);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&c, mine);
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

// Stable compaction of a tile: warp ballots give in-warp order, warps are
// visited in order, 16 position-ordered steps per tile.
template <class T>
__global__ void __launch_bounds__(256) k_compact(const T* __restrict__ in, const uint8_t* __restrict__ flags,
                                               uint64_t n, const uint64_t* __restrict__ offs,
                                               T* __restrict__ out) {
  __shared__ uint32_t wtot[8];
  __shared__ uint64_t run;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) run = offs[blockIdx.x];
  const uint64_t base = blockIdx.x * uint64_t(kScanTile);
  for (int s = 0; s < kScanTile / 256; ++s) {
    const uint64_t e = base + s * 256 + threadIdx.x;
    const bool f = e < n && flags[e];
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wtot[warp] = __popc(b);
    __syncthreads();
    uint64_t pos = run + __popc(b & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) pos += wtot[w];
    if (f) out[pos] = in ? in[e] : static_cast<T>(e);  // in == nullptr: write the index
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < 8; ++w) t += wtot[w];
      run += t;
    }
    __syncthreads();
  }
}

unsigned grid_cap(uint64_t n) { return static_cast<unsigned>(std::min<uint64_t>(std::max<uint64_t>(n, 1), 1u << 30)); }

}  // namespace

// exclusive scan (u64) of n values, in -> out (may alias)
void scan_exclusive_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  const uint64_t chunks = (n + kScanTile - 1) / kScanTile;
  DevBuf<uint64_t> sums(chunks), sums_scan(chunks);
  k_scan_chunks<<<grid_cap(chunks), 256, 0, s>>>(in, out, n, sums.ptr);
  count_launch();
  check_launch("k_scan_chunks");
  if (chunks > 1) {
    scan_exclusive_u64(sums.ptr, sums_scan.ptr, chunks, s);
    k_add_chunk_offsets<<<grid_cap(chunks), 256, 0, s>>>(out, n, sums_scan.ptr);
    count_launch();
    check_launch("k_add_chunk_offsets");
  }
}

template <class K>
void radix_sort_pairs(K* keys, K* keys_alt, uint32_t* vals, uint32_t* vals_alt, uint64_t n, int begin_bit,
                      int end_bit, cudaStream_t s, bool* result_in_alt) {
  *result_in_alt = false;
  if (n <= 1 || end_bit <= begin_bit) return;
  const uint64_t ntiles = (n + kSortTile - 1) / kSortTile;
  DevBuf<uint64_t> hist(ntiles * kDigits);
  const int nsm = sm_count();
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(nsm) * 8));
  K *kin = keys, *kout = keys_alt;
  uint32_t *vin = vals, *vout = vals_alt;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    const int bits = std::min(8, end_bit - shift);
    const uint32_t dmask = (1u << bits) - 1u;
    k_digit_hist<K><<<grid, kSortThreads, 0, s>>>(kin, n, shift, dmask, ntiles, hist.ptr);
    count_launch();
    check_launch("k_digit_hist");
    scan_exclusive_u64(hist.ptr, hist.ptr, ntiles * kDigits, s);
    constexpr size_t stage = (sizeof(K) + sizeof(uint32_t)) * kSortTile;
    ensure_dyn_smem(reinterpret_cast<const void*>(k_digit_scatter<K>), stage);
    k_digit_scatter<K><<<grid, kSortThreads, stage, s>>>(kin, vin, n, shift, dmask, ntiles, hist.ptr, kout, vout);
    count_launch();
    check_launch("k_digit_scatter");
    std::swap(kin, kout);
    std::swap(vin, vout);
    *result_in_alt = !*result_in_alt;
  }
}

template void radix_sort_pairs<uint64_t>(uint64_t*, uint64_t*, uint32_t*, uint32_t*, uint64_t, int, int,
                                         cudaStream_t, bool*);
template void radix_sort_pairs<uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, uint64_t, int, int,
                                         cudaStream_t, bool*);

template <class T>
uint64_t select_flagged(const T* in, const uint8_t* flags, uint64_t n, T* out, cudaStream_t s) {
  if (!n) return 0;
  const uint64_t chunks = (n + kScanTile - 1) / kScanTile;
  DevBuf<uint64_t> counts(chunks), offs(chunks + 1);
  k_flag_counts<<<grid_cap(chunks), 256, 0, s>>>(flags, n, counts.ptr);
  count_launch();
  check_launch("k_flag_counts");
  scan_exclusive_u64(counts.ptr, offs.ptr, chunks, s);
  k_compact<T><<<grid_cap(chunks), 256, 0, s>>>(in, flags, n, offs.ptr, out);
  count_launch();
  check_launch("k_compact");
  uint64_t last_off = 0, last_cnt = 0;
  B200_CUDA(cudaMemcpyAsync(&last_off, offs.ptr + chunks - 1, 8, cudaMemcpyDeviceToHost, s));
  B200_CUDA(cudaMemcpyAsync(&last_cnt, counts.ptr + chunks - 1, 8, cudaMemcpyDeviceToHost, s));
  B200_CUDA(cudaStreamSynchronize(s));
  return last_off + last_cnt;
}

template uint64_t select_flagged<uint64_t>(const uint64_t*, const uint8_t*, uint64_t, uint64_t*, cudaStream_t);
template uint64_t select_flagged<uint32_t>(const uint32_t*, const uint8_t*, uint64_t, uint32_t*, cudaStream_t);

}  // namespace b200
