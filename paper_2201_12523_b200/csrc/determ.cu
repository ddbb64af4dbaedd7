// determ.cu -- deterministic (run-to-run bit-stable) MTTKRP.
//
// Reference: ExecConfig::deterministic (proj/include/blco/exec.hpp:22) makes
// the simulator log every commit and apply the log in work-group order
// (proj/src/exec.cpp:78-86, :130-136), so a CPU run is reproducible bit for
// bit.  The device kernels of mttkrp.cu commit with RED.E.ADD.F64 from many
// CTAs, whose arrival order varies between runs.  This path fixes the order:
//
//   index (once per tensor and mode, cached on the tensor):
//     k_det_rows   decodes every element's target row and counts per row;
//     radix sort   of (row, element id) -- stable, so each row's elements
//                  stay in ALTO order (the BLCO element order);
//     host         splits every row into chunks of <= kChunk elements.
//   multiply:
//     k_mttkrp_det one warp per chunk; lane q owns columns q + 32c; the
//                  chunk's elements are summed in ALTO order, each term
//                  formed in the oracle's product order (oracle.cpp:15-24);
//                  a single-chunk row is written to M directly, the chunks
//                  of a longer row go to a partial buffer;
//     k_det_combine sums a long row's partials in chunk order.
//
// Every floating-point operation therefore happens in an order fixed by the
// tensor alone, so results are identical across runs, streams and block
// splits of the same tensor (ALTO order does not depend on the split).  It
// cannot equal the CPU's deterministic bits: the CPU adds in work-group /
// COO order, this in ALTO order per row.
#include <algorithm>

#include "internal.hpp"

namespace b200 {
namespace {

constexpr uint32_t kChunk = 2048;
constexpr uint32_t kDirect = 0xffffffffu;
constexpr int kDetWarps = 8;

template <int N>
struct DetParams {
  const uint32_t* __restrict__ perm;
  const uint64_t* __restrict__ idx;
  const double* __restrict__ val;
  const uint32_t* __restrict__ block_base;
  const uint64_t* __restrict__ block_off;  // nblocks + 1
  uint32_t nblocks;
  const uint64_t* __restrict__ chunk_begin;
  const uint32_t* __restrict__ chunk_count;
  const uint32_t* __restrict__ chunk_row;
  const uint32_t* __restrict__ chunk_part;
  uint64_t nchunks;
  // per non-target mode k (ascending): its factor, mode index, field shift
  // and mask -- indexed by the compile-time k only (a param array indexed by
  // a runtime value would be copied to local memory)
  const double* factors[N];
  int other[N];
  uint32_t oshift[N];
  uint64_t omask[N];
  int mode;
  int rank;
  double* out;
  double* partial;
  int accumulate;
};

__global__ void k_det_rows(const TileDesc* __restrict__ tiles, const uint64_t* __restrict__ idx,
                           const uint32_t* __restrict__ block_base, int order, int mode, uint32_t shift,
                           uint64_t mask, uint32_t* __restrict__ rows, uint32_t* __restrict__ counts) {
  const TileDesc td = tiles[blockIdx.x];
  const uint32_t base = block_base[static_cast<uint64_t>(td.block) * order + mode];
  for (uint32_t i = threadIdx.x; i < td.count; i += blockDim.x) {
    const uint32_t r = base | static_cast<uint32_t>((idx[td.start + i] >> shift) & mask);
    rows[td.start + i] = r;
    atomicAdd(&counts[r], 1u);
  }
}

__global__ void k_det_iota(uint32_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint32_t>(i);
}

__device__ __forceinline__ uint32_t block_of(const uint64_t* off, uint32_t nb, uint64_t e) {
  uint32_t lo = 0, hi = nb;  // largest b with off[b] <= e
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) / 2;
    if (off[mid] <= e) lo = mid;
    else hi = mid;
  }
  return lo;
}

template <int N, int CPL>
__global__ void __launch_bounds__(32 * kDetWarps) k_mttkrp_det(DetParams<N> p) {
  const uint64_t chunk = blockIdx.x * uint64_t(kDetWarps) + (threadIdx.x >> 5);
  if (chunk >= p.nchunks) return;
  const int lane = threadIdx.x & 31, R = p.rank;
  const uint64_t b0 = p.chunk_begin[chunk];
  const uint32_t cnt = p.chunk_count[chunk];
  double acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
  constexpr int U = 4;
  for (uint32_t j0 = 0; j0 < cnt; j0 += U) {
    double prod[U][CPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = j0 + u < cnt ? j0 + u : cnt - 1;  // tail: recompute the last element, unused
      const uint32_t e = p.perm[b0 + j];
      const uint64_t ix = p.idx[e];
      const double v = p.val[e];
      const uint32_t blk = block_of(p.block_off, p.nblocks, e);
#pragma unroll
      for (int c = 0; c < CPL; ++c) prod[u][c] = v;
#pragma unroll
      for (int k = 0; k + 1 < N; ++k) {  // the oracle's order: value, then the modes ascending
        const uint32_t coord = p.block_base[static_cast<uint64_t>(blk) * N + p.other[k]] |
                               static_cast<uint32_t>((ix >> p.oshift[k]) & p.omask[k]);
        const double* rp = p.factors[k] + static_cast<uint64_t>(coord) * R;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int col = lane + 32 * c;
          if (col < R) prod[u][c] = __dmul_rn(prod[u][c], __ldg(rp + col));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (j0 + u < cnt)
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = __dadd_rn(acc[c], prod[u][c]);
  }
  const uint32_t part = p.chunk_part[chunk];
  const uint32_t row = p.chunk_row[chunk];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int col = lane + 32 * c;
    if (col >= R) continue;
    if (part == kDirect) {
      double* o = p.out + static_cast<uint64_t>(row) * R + col;
      *o = p.accumulate ? __dadd_rn(*o, acc[c]) : acc[c];
    } else {
      p.partial[static_cast<uint64_t>(part) * R + col] = acc[c];
    }
  }
}

// rows split into several chunks: sum the partials in chunk order
__global__ void k_det_combine(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ first,
                              const uint32_t* __restrict__ nparts, uint64_t n, const double* __restrict__ partial,
                              int R, int accumulate, double* __restrict__ out) {
  const uint64_t w = blockIdx.x * uint64_t(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= n) return;
  const int lane = threadIdx.x & 31;
  for (int col = lane; col < R; col += 32) {
    double s = 0.0;
    for (uint32_t q = 0; q < nparts[w]; ++q) s = __dadd_rn(s, partial[static_cast<uint64_t>(first[w] + q) * R + col]);
    double* o = out + static_cast<uint64_t>(rows[w]) * R + col;
    *o = accumulate ? __dadd_rn(*o, s) : s;
  }
}

template <int N, int CPL>
void launch_det(const DetIndex& d, const blco_tensor& t, const MttkrpLaunch& a, double* partial) {
  DetParams<N> p{};
  p.perm = d.perm.ptr;
  p.idx = t.idx.ptr;
  p.val = t.vals.ptr;
  p.block_base = t.block_base.ptr;
  p.block_off = d.block_off.ptr;
  p.nblocks = static_cast<uint32_t>(t.nblocks());
  p.chunk_begin = d.chunk_begin.ptr;
  p.chunk_count = d.chunk_count.ptr;
  p.chunk_row = d.chunk_row.ptr;
  p.chunk_part = d.chunk_part.ptr;
  p.nchunks = d.chunk_begin.n;
  for (int m = 0, k = 0; m < N; ++m) {
    if (m == a.mode) continue;
    p.factors[k] = a.factors[m];
    p.other[k] = m;
    p.oshift[k] = static_cast<uint32_t>(t.layout.field_shift[m]);
    p.omask[k] = t.layout.field_mask[m];
    ++k;
  }
  p.mode = a.mode;
  p.rank = static_cast<int>(a.rank);
  p.out = a.out;
  p.partial = partial;
  p.accumulate = a.accumulate;
  if (p.nchunks) {
    const unsigned grid = static_cast<unsigned>((p.nchunks + kDetWarps - 1) / kDetWarps);
    k_mttkrp_det<N, CPL><<<grid, 32 * kDetWarps, 0, a.stream>>>(p);
    count_launch();
    check_launch("k_mttkrp_det");
  }
  if (d.multi_row.n) {
    const unsigned grid = static_cast<unsigned>((d.multi_row.n + 7) / 8);
    k_det_combine<<<grid, 256, 0, a.stream>>>(d.multi_row.ptr, d.multi_first.ptr, d.multi_nparts.ptr,
                                             d.multi_row.n, partial, p.rank, a.accumulate, a.out);
    count_launch();
    check_launch("k_det_combine");
  }
}

template <int N>
void launch_det_order(const DetIndex& d, const blco_tensor& t, const MttkrpLaunch& a, double* partial) {
  const int cpl = static_cast<int>((a.rank + 31) / 32);
  switch (cpl) {
    case 1: return launch_det<N, 1>(d, t, a, partial);
    case 2: return launch_det<N, 2>(d, t, a, partial);
    case 3:
    case 4: return launch_det<N, 4>(d, t, a, partial);
    default:
      if (cpl <= 8) return launch_det<N, 8>(d, t, a, partial);
      throw_format("b200: deterministic mode supports rank <= 256");
  }
}

// Builds (or returns the cached) deterministic index of mode `mode`.
const DetIndex& det_index(const blco_tensor& t, int mode, cudaStream_t s) {
  {
    std::lock_guard<std::mutex> g(t.mu);
    auto it = t.det.find(mode);
    if (it != t.det.end()) return it->second;
  }
  const blco_layout& l = t.layout;
  if (t.nnz >= (uint64_t{1} << 32))
    throw_format("b200: deterministic mode needs fewer than 2^32 non-zeros per device tensor");
  const uint64_t rows_n = l.dims[mode];
  DetIndex d;
  DevBuf<uint32_t> rows(t.nnz), rows_alt(t.nnz), perm_alt(t.nnz), counts(rows_n);
  d.perm.alloc(t.nnz);
  B200_CUDA(cudaMemsetAsync(counts.ptr, 0, rows_n * 4, s));
  uint64_t ntiles = 0;
  const TileDesc* tiles = tile_table(t, mttkrp_tile_elems(), &ntiles);
  if (ntiles) {
    k_det_rows<<<static_cast<unsigned>(ntiles), 256, 0, s>>>(tiles, t.idx.ptr, t.block_base.ptr, l.order, mode,
                                                            static_cast<uint32_t>(l.field_shift[mode]),
                                                            l.field_mask[mode], rows.ptr, counts.ptr);
    count_launch();
    check_launch("k_det_rows");
    k_det_iota<<<static_cast<unsigned>(std::min<uint64_t>((t.nnz + 255) / 256, sm_count() * 16)), 256, 0, s>>>(
        perm_alt.ptr, t.nnz);
    count_launch();
    check_launch("k_det_iota");
    bool alt = false;
    const int bits = std::max(1, bits_for_extent(rows_n));
    radix_sort_pairs<uint32_t>(rows.ptr, rows_alt.ptr, perm_alt.ptr, d.perm.ptr, t.nnz, 0, bits, s, &alt);
    // result in (rows_alt, d.perm) iff alt; otherwise still in (rows, perm_alt)
    if (!alt) std::swap(d.perm.ptr, perm_alt.ptr);
  }
  std::vector<uint32_t> hc(rows_n);
  if (rows_n) B200_CUDA(cudaMemcpyAsync(hc.data(), counts.ptr, rows_n * 4, cudaMemcpyDeviceToHost, s));
  B200_CUDA(cudaStreamSynchronize(s));
  std::vector<uint64_t> cb;
  std::vector<uint32_t> cc, cr, cp, mr, mf, mn;
  uint64_t pos = 0;
  uint32_t parts = 0;
  for (uint64_t r = 0; r < rows_n; ++r) {
    const uint32_t c = hc[r];
    if (!c) continue;
    const uint32_t k = (c + kChunk - 1) / kChunk;
    if (k > 1) {
      mr.push_back(static_cast<uint32_t>(r));
      mf.push_back(parts);
      mn.push_back(k);
    }
    for (uint32_t q = 0; q < k; ++q) {
      cb.push_back(pos + uint64_t(q) * kChunk);
      cc.push_back(std::min(kChunk, c - q * kChunk));
      cr.push_back(static_cast<uint32_t>(r));
      cp.push_back(k > 1 ? parts + q : kDirect);
    }
    if (k > 1) parts += k;
    pos += c;
  }
  auto up = [&](auto& dst, const auto& src) {
    dst.alloc(src.size());
    if (!src.empty()) B200_CUDA(cudaMemcpy(dst.ptr, src.data(), src.size() * sizeof(src[0]), cudaMemcpyHostToDevice));
  };
  up(d.chunk_begin, cb);
  up(d.chunk_count, cc);
  up(d.chunk_row, cr);
  up(d.chunk_part, cp);
  up(d.multi_row, mr);
  up(d.multi_first, mf);
  up(d.multi_nparts, mn);
  up(d.block_off, t.offsets);
  d.nparts = parts;
  // staged pageable uploads above: land them before kernels on any stream
  B200_CUDA(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> g(t.mu);
  return t.det.emplace(mode, std::move(d)).first->second;
}

// per stream: launches on different streams of one thread may overlap
thread_local std::map<cudaStream_t, DevBuf<double>> t_partials;

}  // namespace

void release_det_cache() { t_partials.clear(); }

void det_mttkrp_enqueue(const blco_tensor& t, MttkrpLaunch& a) {
  const DetIndex& d = det_index(t, a.mode, a.stream);
  const uint64_t elems = t.layout.dims[a.mode] * a.rank;
  if (!a.accumulate && elems) B200_CUDA(cudaMemsetAsync(a.out, 0, elems * 8, a.stream));
  DevBuf<double>& t_partial = t_partials[a.stream];
  if (t_partial.n < d.nparts * a.rank) t_partial.alloc(d.nparts * a.rank);
  a.workgroups = d.chunk_begin.n;
  switch (t.layout.order) {
    case 1: return launch_det_order<1>(d, t, a, t_partial.ptr);
    case 2: return launch_det_order<2>(d, t, a, t_partial.ptr);
    case 3: return launch_det_order<3>(d, t, a, t_partial.ptr);
    case 4: return launch_det_order<4>(d, t, a, t_partial.ptr);
    case 5: return launch_det_order<5>(d, t, a, t_partial.ptr);
    case 6: return launch_det_order<6>(d, t, a, t_partial.ptr);
    case 7: return launch_det_order<7>(d, t, a, t_partial.ptr);
    case 8: return launch_det_order<8>(d, t, a, t_partial.ptr);
    default: throw_format("b200: order above the device limit");
  }
}

}  // namespace b200
