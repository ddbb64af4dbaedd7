// mttkrp.cu -- mode-agnostic BLCO MTTKRP for sm_100a (K4 register path,
// K5 hierarchical shared-memory stash, K5m copy merge).
//
// Reference semantics: mttkrp, proj/src/mttkrp.cpp:167-235 --
//   M[i, r] = sum over non-zeros with mode-`mode` coordinate i of
//             value * prod_{m != mode, ascending} A_m[c_m, r]
// with the per-element product formed in exactly the oracle's order
// (proj/src/oracle.cpp:15-24; mttkrp.cpp:104-107), so every per-element term
// is bit-identical to the oracle's and only the summation order differs.
//
// Kernel structure:
//   CTA = 8 warps, tile = 1024 contiguous elements of one block (TileDesc).
//   Processing phase, per warp, per 32-element sub-tile (the reference's
//   tile, mttkrp.cpp:23-81): streaming 64-bit index/value loads (ld.cs),
//   shift/mask de-linearization against the block's base coordinates,
//   __match_any_sync on the target row, a warp prefix sum over group sizes to
//   place equal rows contiguously in shared memory (the stable-reorder of
//   :55-73 without the O(tile^2) rank), segment-end flags.
//   Computing phase (:95-137): LPE lanes own one element's rank row (CPL
//   columns each, 128-bit factor-row gathers when R is even); U elements are
//   gathered before any is consumed so U*(N-1) row loads are in flight per
//   lane; products accumulate in registers along a segment and commit once
//   per segment -- RED.E.ADD.F64 into M (register path) or into the CTA's
//   shared-memory stash (hierarchical path, :139-155), whose rows flush to
//   the CTA's factor copy at the end (:210-215).
#include <algorithm>
#include <cstring>

#include "internal.hpp"

namespace b200 {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kWarps = 8;
constexpr int kCtaThreads = 32 * kWarps;
constexpr int kSub = 4;                          // 32-element sub-tiles per warp
constexpr int kWarpElems = 32 * kSub;            // 128
constexpr int kTileElems = kWarps * kWarpElems;  // 1024
constexpr int kUnroll = 4;                       // elements gathered ahead per lane group

template <int N>
struct Params {
  const TileDesc* __restrict__ tiles;
  uint64_t ntiles;
  uint64_t elem_end;  // global element bound (tile counts are clamped to it)
  const uint64_t* __restrict__ idx;
  const double* __restrict__ val;
  const uint32_t* __restrict__ block_base;
  const double* factors[N];  // factors[k] = A of the k-th non-target mode (ascending)
  int others[N];             // others[k] = that mode's index (k < N-1)
  double* out;          // register: M; hierarchical: copy 0 (copies are contiguous)
  uint64_t copy_elems;  // I_n * R
  int ncopies;
  int mode;
  int rank;
  int stash_slots;
  uint32_t shift[N];
  uint64_t mask[N];
  unsigned long long* counters;  // [segments, stash flushes, commit lanes] or null
};

template <int N>
struct Stage {
  uint32_t coord[N][kWarpElems];
  double val[kWarpElems];
  uint8_t end[kWarpElems];
};

template <int CPL, bool VEC>
struct Row {
  double v[CPL];
};

template <int CPL, bool VEC>
__device__ __forceinline__ void load_row(Row<CPL, VEC>& r, const double* __restrict__ p, int ncol_ok) {
  if constexpr (VEC && CPL == 2) {
    const double2 x = __ldg(reinterpret_cast<const double2*>(p));
    r.v[0] = x.x;
    r.v[1] = x.y;
  } else {
#pragma unroll
    for (int c = 0; c < CPL; ++c) r.v[c] = c < ncol_ok ? __ldg(p + c) : 0.0;
  }
}

// Processing phase for one warp: stage up to kWarpElems elements with equal
// target rows made contiguous within each 32-element sub-tile.  Returns the
// staged count and adds the segment count to *segs.
template <int N>
__device__ __forceinline__ int process_warp(const Params<N>& p, const TileDesc& td, int warp,
                                            int lane, Stage<N>& st, unsigned long long& segs) {
  const uint32_t wbeg = static_cast<uint32_t>(warp) * kWarpElems;
  const uint64_t room = td.start >= p.elem_end ? 0 : p.elem_end - td.start;
  const uint32_t cnt = room < td.count ? static_cast<uint32_t>(room) : td.count;
  const int wn = cnt > wbeg ? min(kWarpElems, static_cast<int>(cnt - wbeg)) : 0;
  if (wn == 0) return 0;
  uint32_t base[N];
#pragma unroll
  for (int m = 0; m < N; ++m) base[m] = __ldg(p.block_base + static_cast<uint64_t>(td.block) * N + m);
  const uint64_t g0 = td.start + wbeg;
  uint64_t ix[kSub];
  double vv[kSub];
#pragma unroll
  for (int s = 0; s < kSub; ++s) {
    const int j = s * 32 + lane;
    ix[s] = j < wn ? __ldcs(p.idx + g0 + j) : 0;
    vv[s] = j < wn ? __ldcs(p.val + g0 + j) : 0.0;
  }
#pragma unroll
  for (int s = 0; s < kSub; ++s) {
    if (s * 32 >= wn) break;
    const int j = s * 32 + lane;
    const bool valid = j < wn;
    uint32_t c[N];
#pragma unroll
    for (int m = 0; m < N; ++m) c[m] = base[m] | static_cast<uint32_t>((ix[s] >> p.shift[m]) & p.mask[m]);
    const uint32_t row = __ldg(p.block_base + static_cast<uint64_t>(td.block) * N + p.mode) |
                         static_cast<uint32_t>((ix[s] >> p.shift[p.mode]) & p.mask[p.mode]);
    // invalid lanes form the sentinel group; dims < 2^32 keep it distinct
    const uint32_t key = valid ? row : 0xffffffffu;
    const unsigned match = __match_any_sync(kFull, key);
    const int leader = __ffs(match) - 1;
    const int gsize = __popc(match);
    int x = lane == leader ? gsize : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(kFull, x, d);
      if (lane >= d) x += y;
    }
    const int excl = x - (lane == leader ? gsize : 0);
    const int goff = __shfl_sync(kFull, excl, leader);
    const int rin = __popc(match & ((1u << lane) - 1u));
    if (valid) {
      const int pos = s * 32 + goff + rin;
#pragma unroll
      for (int m = 0; m < N; ++m) st.coord[m][pos] = c[m];
      st.val[pos] = vv[s];
      st.end[pos] = rin == gsize - 1;
    }
    segs += __popc(__ballot_sync(kFull, valid && lane == leader));
  }
  __syncwarp();
  return wn;
}

// Computing phase: lane group g walks staged positions [lo, hi).
template <int N, int LPE, int CPL, bool VEC, bool HIER>
__device__ __forceinline__ void compute_warp(const Params<N>& p, const Stage<N>& st, int wn, int lane,
                                             int col0, double* __restrict__ copy_out,
                                             double* stash, uint32_t* tags,
                                             unsigned long long& commits,
                                             unsigned long long& flushes) {
  constexpr int G = 32 / LPE;
  const int g = lane / LPE, q = lane % LPE;
  const int lo = (g * wn) / G, hi = ((g + 1) * wn) / G;
  const int span = (wn + G - 1) / G;
  const int R = p.rank;
  const int cbase = col0 + q * CPL;
  const int ncol_ok = max(0, min(CPL, R - cbase));
  const unsigned gmask = LPE == 32 ? kFull : (((1u << LPE) - 1u) << (g * LPE));
  double acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0;

  constexpr int NO = N > 1 ? N - 1 : 1;  // non-target modes (array extent)
  for (int t0 = 0; t0 < span; t0 += kUnroll) {
    bool ok[kUnroll], fin[kUnroll];
    double v[kUnroll];
    uint32_t rowu[kUnroll];
    uint32_t cm[kUnroll][NO];
    Row<CPL, VEC> rows[kUnroll][NO];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int j = lo + t0 + u;
      ok[u] = j < hi;
      const int jc = ok[u] ? j : 0;
      v[u] = st.val[jc];
      rowu[u] = st.coord[p.mode][jc];
#pragma unroll
      for (int k = 0; k < N - 1; ++k) cm[u][k] = st.coord[p.others[k]][jc];
      fin[u] = ok[u] && (st.end[jc] || j == hi - 1);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int k = 0; k < N - 1; ++k)
        if (ok[u] && ncol_ok > 0)
          load_row<CPL, VEC>(rows[u][k], p.factors[k] + static_cast<uint64_t>(cm[u][k]) * R + cbase, ncol_ok);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (!ok[u]) continue;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        double prod = v[u];
#pragma unroll
        for (int k = 0; k < N - 1; ++k) prod = __dmul_rn(prod, rows[u][k].v[c]);
        acc[c] = __dadd_rn(acc[c], prod);
      }
      if (fin[u]) {
        const uint32_t row = rowu[u];
        if constexpr (HIER) {
          const uint32_t slot = row % static_cast<uint32_t>(p.stash_slots);
          int owned = 0;
          if (q == 0) {
            const uint32_t old = atomicCAS(&tags[slot], 0u, row + 1u);
            owned = old == 0u || old == row + 1u;
          }
          owned = __shfl_sync(gmask, owned, g * LPE);
          if (owned) {
#pragma unroll
            for (int c = 0; c < CPL; ++c)
              if (c < ncol_ok) atomicAdd(&stash[static_cast<uint64_t>(slot) * R + cbase + c], acc[c]);
          } else {
#pragma unroll
            for (int c = 0; c < CPL; ++c)
              if (c < ncol_ok) atomicAdd(copy_out + static_cast<uint64_t>(row) * R + cbase + c, acc[c]);
            if (q == 0) ++flushes;
          }
        } else {
#pragma unroll
          for (int c = 0; c < CPL; ++c)
            if (c < ncol_ok) atomicAdd(copy_out + static_cast<uint64_t>(row) * R + cbase + c, acc[c]);
        }
        if (ncol_ok > 0) ++commits;
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
      }
    }
  }
}

template <int N, int LPE, int CPL, bool VEC, bool STATS>
__global__ void __launch_bounds__(kCtaThreads) k_mttkrp_register(Params<N> p) {
  __shared__ Stage<N> stage[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TileDesc td = p.tiles[blockIdx.x];
  unsigned long long segs = 0, commits = 0, flushes = 0;
  const int wn = process_warp<N>(p, td, warp, lane, stage[warp], segs);
  if (wn > 0)
    compute_warp<N, LPE, CPL, VEC, false>(p, stage[warp], wn, lane, blockIdx.y * LPE * CPL, p.out,
                                          nullptr, nullptr, commits, flushes);
  if constexpr (STATS) {
    if (lane == 0 && blockIdx.y == 0 && segs) atomicAdd(&p.counters[0], segs);
    // commit lanes: count per lane, reduce over the warp
    unsigned long long c = commits;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(kFull, c, d);
    if (lane == 0 && c) atomicAdd(&p.counters[2], c);
  }
}

// Persistent CTAs; dynamic shared memory = stash (slots x R doubles + tags).
template <int N, int LPE, int CPL, bool VEC, bool STATS>
__global__ void __launch_bounds__(kCtaThreads) k_mttkrp_hier(Params<N> p) {
  __shared__ Stage<N> stage[kWarps];
  extern __shared__ __align__(16) unsigned char dyn[];
  const int S = p.stash_slots, R = p.rank;
  double* stash = reinterpret_cast<double*>(dyn);
  uint32_t* tags = reinterpret_cast<uint32_t*>(stash + static_cast<uint64_t>(S) * R);
  for (int i = threadIdx.x; i < S * R; i += blockDim.x) stash[i] = 0.0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) tags[i] = 0u;
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int copy = static_cast<int>(blockIdx.x % static_cast<unsigned>(p.ncopies));
  double* copy_out = p.out + static_cast<uint64_t>(copy) * p.copy_elems;
  unsigned long long segs = 0, commits = 0, flushes = 0;
  for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const TileDesc td = p.tiles[tile];
    const int wn = process_warp<N>(p, td, warp, lane, stage[warp], segs);
    if (wn > 0)
      compute_warp<N, LPE, CPL, VEC, true>(p, stage[warp], wn, lane, blockIdx.y * LPE * CPL,
                                           copy_out, stash, tags, commits, flushes);
    __syncwarp();
  }
  __syncthreads();
  // Flush every occupied slot (one row commit each) to this CTA's copy.
  const int cols = min(R - static_cast<int>(blockIdx.y) * LPE * CPL, LPE * CPL);
  for (int i = threadIdx.x; i < S * cols; i += blockDim.x) {
    const int s = i / cols, c = blockIdx.y * LPE * CPL + i % cols;
    const uint32_t tag = tags[s];
    if (tag) atomicAdd(copy_out + static_cast<uint64_t>(tag - 1u) * R + c, stash[static_cast<uint64_t>(s) * R + c]);
  }
  if constexpr (STATS) {
    unsigned long long occ = 0;
    for (int s = threadIdx.x; s < S; s += blockDim.x) occ += tags[s] != 0u;
    unsigned long long c = commits, f = flushes + (blockIdx.y == 0 ? occ : 0);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      c += __shfl_down_sync(kFull, c, d);
      f += __shfl_down_sync(kFull, f, d);
    }
    if (lane == 0 && blockIdx.y == 0 && segs) atomicAdd(&p.counters[0], segs);
    if (lane == 0 && f) atomicAdd(&p.counters[1], f);
    if (lane == 0 && c) atomicAdd(&p.counters[2], c);
  }
}

__global__ void k_merge_copies(const double* __restrict__ copies, uint64_t elems, int ncopies,
                               double* __restrict__ out, int accumulate) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < elems;
       i += uint64_t(gridDim.x) * blockDim.x) {
    double s = copies[i];
    for (int c = 1; c < ncopies; ++c) s += copies[static_cast<uint64_t>(c) * elems + i];
    out[i] = accumulate ? out[i] + s : s;
  }
}


}  // namespace

// ------------------------------------------------------------------ launch

uint32_t mttkrp_tile_elems() { return kTileElems; }

KernelView view_of(const blco_tensor& t) {
  KernelView v{};
  v.layout = &t.layout;
  v.tiles = tile_table(t, kTileElems, &v.ntiles);
  v.elem_end = t.nnz;
  v.idx = t.idx.ptr;
  v.vals = t.vals.ptr;
  v.block_base = t.block_base.ptr;
  return v;
}

void merge_copies_enqueue(const double* copies, uint64_t elems, int ncopies, double* out,
                          int accumulate, cudaStream_t s) {
  if (!elems) return;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((elems + 255) / 256, 65535));
  k_merge_copies<<<std::max(1u, g), 256, 0, s>>>(copies, elems, ncopies, out, accumulate);
  count_launch();
  check_launch("k_merge_copies");
}

namespace {

struct Workspace {
  DevBuf<double> copies;
  DevBuf<unsigned long long> counters;
  int device = -1;
};
thread_local Workspace t_ws;

// Per-thread scratch, re-created when the calling thread changes device.
Workspace& workspace() {
  int dev = 0;
  B200_CUDA(cudaGetDevice(&dev));
  if (t_ws.device != dev) {
    t_ws.copies.reset();
    t_ws.counters.reset();
    t_ws.device = dev;
  }
  return t_ws;
}

template <int N, int LPE, int CPL, bool VEC>
void launch_cfg(MttkrpLaunch& a) {
  const KernelView& v = a.view;
  const blco_layout& l = *v.layout;
  Params<N> p{};
  p.tiles = v.tiles;
  p.ntiles = v.ntiles;
  p.elem_end = v.elem_end;
  p.idx = v.idx;
  p.val = v.vals;
  p.block_base = v.block_base;
  for (int m = 0, k = 0; m < N; ++m) {
    if (m != a.mode) {
      p.factors[k] = a.factors[m];
      p.others[k++] = m;
    }
    p.shift[m] = static_cast<uint32_t>(l.field_shift[m]);
    p.mask[m] = l.field_mask[m];
  }
  p.mode = a.mode;
  p.rank = static_cast<int>(a.rank);
  const uint64_t elems = l.dims[a.mode] * a.rank;
  p.copy_elems = elems;
  p.counters = a.counters;
  const bool stats = a.counters != nullptr;
  const unsigned ychunks = static_cast<unsigned>((a.rank + LPE * CPL - 1) / (LPE * CPL));
  if (!a.accumulate) B200_CUDA(cudaMemsetAsync(a.out, 0, elems * sizeof(double), a.stream));
  if (p.ntiles == 0) return;

  if (a.strategy != BLCO_STRATEGY_HIERARCHICAL) {
    p.out = a.out;
    p.ncopies = 1;
    a.workgroups = p.ntiles;
    const dim3 grid(static_cast<unsigned>(p.ntiles), ychunks);
    if (stats)
      k_mttkrp_register<N, LPE, CPL, VEC, true><<<grid, kCtaThreads, 0, a.stream>>>(p);
    else
      k_mttkrp_register<N, LPE, CPL, VEC, false><<<grid, kCtaThreads, 0, a.stream>>>(p);
    count_launch();
    check_launch("k_mttkrp_register");
    return;
  }

  // Hierarchical: stash as large as shared memory allows, at least
  // cfg.stash_slots, no larger than the mode (then it privatises the mode).
  int dev = 0, smem_optin = 0, nsm = 0;
  B200_CUDA(cudaGetDevice(&dev));
  B200_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  B200_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const size_t static_smem = sizeof(Stage<N>) * kWarps;
  const size_t budget = static_cast<size_t>(smem_optin) - static_smem - 1024;
  const size_t per_slot = a.rank * sizeof(double) + sizeof(uint32_t);
  const uint64_t fit = budget / per_slot;
  if (fit < 1)
    throw_format("b200: rank " + std::to_string(a.rank) + " too large for the shared-memory stash");
  uint64_t slots = std::min<uint64_t>(l.dims[a.mode], fit);
  slots = std::max<uint64_t>(slots, std::min<uint64_t>(static_cast<uint64_t>(a.cfg.stash_slots), fit));
  p.stash_slots = static_cast<int>(slots);
  a.stash_slots = p.stash_slots;
  const size_t dyn = slots * per_slot + 16;
  auto kern = stats ? k_mttkrp_hier<N, LPE, CPL, VEC, true> : k_mttkrp_hier<N, LPE, CPL, VEC, false>;
  B200_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
  int per_sm = 0;
  B200_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCtaThreads, dyn));
  per_sm = std::max(per_sm, 1);
  const uint64_t grid = std::min<uint64_t>(p.ntiles, static_cast<uint64_t>(nsm) * per_sm);
  a.workgroups = grid;
  const int C = std::max(1, a.cfg.num_factor_copies);
  p.ncopies = C;
  bool merge = false;
  if (a.hier_copies) {
    p.out = a.hier_copies;  // caller merges once at the end
  } else if (C == 1 && !a.accumulate) {
    p.out = a.out;
  } else {
    Workspace& ws = workspace();
    if (ws.copies.n < elems * C) ws.copies.alloc(elems * C);
    B200_CUDA(cudaMemsetAsync(ws.copies.ptr, 0, elems * C * sizeof(double), a.stream));
    p.out = ws.copies.ptr;
    merge = true;
  }
  kern<<<dim3(static_cast<unsigned>(grid), ychunks), kCtaThreads, dyn, a.stream>>>(p);
  count_launch();
  check_launch("k_mttkrp_hier");
  if (merge) merge_copies_enqueue(p.out, elems, C, a.out, a.accumulate, a.stream);
}

template <int N>
void launch_order(MttkrpLaunch& a) {
  switch (a.rank) {
    case 8: return launch_cfg<N, 4, 2, true>(a);
    case 16: return launch_cfg<N, 8, 2, true>(a);
    case 32: return launch_cfg<N, 16, 2, true>(a);
    case 64: return launch_cfg<N, 32, 2, true>(a);
    default: return launch_cfg<N, 32, 1, false>(a);
  }
}

void validate_call(const blco_tensor* t, uint64_t rank, int mode, const blco_exec_config* cfg) {
  if (!t) throw_format("mttkrp: null tensor");
  if (blco_exec_config_validate(cfg) != BLCO_OK) throw_format(blco_last_error());
  if (mode < 0 || mode >= t->layout.order)
    throw_format("mttkrp: mode " + std::to_string(mode + 1) + " out of range for order " +
                 std::to_string(t->layout.order));
  if (rank < 1) throw_format("factors: rank must be >= 1");
}

// Enqueue with optional stats (stats forces a stream synchronisation).
void run(MttkrpLaunch& a, blco_mttkrp_stats* stats) {
  if (a.strategy == BLCO_STRATEGY_AUTO)
    a.strategy = blco_choose_strategy(a.view.layout->dims[a.mode], &a.cfg);
  Workspace& ws = workspace();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (stats) {
    if (ws.counters.n < 3) ws.counters.alloc(3);
    B200_CUDA(cudaMemsetAsync(ws.counters.ptr, 0, 3 * sizeof(unsigned long long), a.stream));
    a.counters = ws.counters.ptr;
    B200_CUDA(cudaEventCreate(&e0));
    B200_CUDA(cudaEventCreate(&e1));
    B200_CUDA(cudaEventRecord(e0, a.stream));
  }
  mttkrp_enqueue(a);
  if (!stats) return;
  B200_CUDA(cudaEventRecord(e1, a.stream));
  unsigned long long h[3] = {0, 0, 0};
  B200_CUDA(cudaMemcpyAsync(h, ws.counters.ptr, sizeof h, cudaMemcpyDeviceToHost, a.stream));
  B200_CUDA(cudaStreamSynchronize(a.stream));
  float ms = 0;
  B200_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  stats->strategy = a.strategy;
  stats->workgroups = a.workgroups;
  stats->segments = h[0];
  stats->stash_flushes = h[1];
  if (a.strategy == BLCO_STRATEGY_HIERARCHICAL) {
    // global traffic = row flushes (bypass commits + end-of-CTA slot
    // flushes), one R-wide commit event each (mttkrp.cpp:210-215)
    stats->commit_events = h[1];
    stats->scalar_adds = h[1] * a.rank;
  } else {
    stats->commit_events = h[2];  // committing lanes (mttkrp.cpp:131-134 analogue)
    stats->scalar_adds = h[0] * a.rank;
  }
  stats->kernel_ms = ms;
}

}  // namespace

void mttkrp_enqueue(MttkrpLaunch& a) {
  if (a.rank < 1) throw_format("factors: rank must be >= 1");
  switch (a.view.layout->order) {
    case 1: return launch_order<1>(a);
    case 2: return launch_order<2>(a);
    case 3: return launch_order<3>(a);
    case 4: return launch_order<4>(a);
    case 5: return launch_order<5>(a);
    case 6: return launch_order<6>(a);
    case 7: return launch_order<7>(a);
    case 8: return launch_order<8>(a);
    default: throw_format("b200: order above the device limit");
  }
}

}  // namespace b200

using namespace b200;

extern "C" {

int blco_mttkrp_device(const blco_tensor* t, const double* const* d_factors, uint64_t rank,
                       int mode, int strategy, const blco_exec_config* cfg, double* d_out,
                       int accumulate, void* stream, blco_mttkrp_stats* stats) {
  return guarded([&] {
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    validate_call(t, rank, mode, &c);
    DeviceGuard dg(t->device);
    MttkrpLaunch a{};
    a.view = view_of(*t);
    a.factors = d_factors;
    a.rank = rank;
    a.mode = mode;
    a.strategy = strategy;
    a.cfg = c;
    a.out = d_out;
    a.accumulate = accumulate;
    a.stream = static_cast<cudaStream_t>(stream);
    run(a, stats);
  });
}

int blco_mttkrp(const blco_tensor* t, const double* const* factors, uint64_t rank, int mode,
                int strategy, const blco_exec_config* cfg, double* out, blco_mttkrp_stats* stats) {
  return guarded([&] {
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    validate_call(t, rank, mode, &c);
    DeviceGuard dg(t->device);
    const blco_layout& l = t->layout;
    std::vector<DevBuf<double>> df(l.order);
    std::vector<const double*> ptrs(l.order);
    for (int m = 0; m < l.order; ++m) {
      df[m].alloc(l.dims[m] * rank);
      if (l.dims[m] * rank)
        B200_CUDA(cudaMemcpy(df[m].ptr, factors[m], l.dims[m] * rank * 8, cudaMemcpyHostToDevice));
      ptrs[m] = df[m].ptr;
    }
    const uint64_t elems = l.dims[mode] * rank;
    DevBuf<double> dout(elems);
    MttkrpLaunch a{};
    a.view = view_of(*t);
    a.factors = ptrs.data();
    a.rank = rank;
    a.mode = mode;
    a.strategy = strategy;
    a.cfg = c;
    a.out = dout.ptr;
    a.stream = nullptr;
    run(a, stats);
    B200_CUDA(cudaMemcpy(out, dout.ptr, elems * 8, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
