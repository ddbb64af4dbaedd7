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
#include <map>
#include <mutex>
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include "internal.hpp"

namespace b200 {
namespace {

// Factor-row gathers of the computing phases.  BLCO_GATHER (compile time)
// selects the L1 policy: 0 = ld.global.nc (cached in L1), 1 = ld.global.cg
// (L2 only), 2 = L1::evict_last, 3 = L1::no_allocate.
#ifndef BLCO_GATHER
#define BLCO_GATHER 0
#endif
// L2 eviction priorities (compile time, BLCO_L2HINT bits): 1 = segment
// commits (RED) evict_last, 2 = factor-row gathers evict_first.  A missed
// commit costs a DRAM read and a later write-back, a missed gather only the
// read, so keeping output lines longer may pay on DRAM-bound shapes.
#ifndef BLCO_L2HINT
#define BLCO_L2HINT 0
#endif
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void commit_add(double* a, double v) {
#if BLCO_L2HINT & 1
  asm volatile("red.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(l2_evict_last()) : "memory");
#else
  atomicAdd(a, v);
#endif
}

template <class T>
__device__ __forceinline__ T gather_ld(const T* p) {
#if BLCO_L2HINT & 2
  if constexpr (sizeof(T) == 8) {
    unsigned long long x;
    asm("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(x) : "l"(p), "l"(l2_evict_first()));
    T r;
    memcpy(&r, &x, 8);
    return r;
  }
#endif
#if BLCO_GATHER == 1
  return __ldcg(p);
#elif BLCO_GATHER == 2 || BLCO_GATHER == 3
  if constexpr (sizeof(T) == 8) {
    unsigned long long x;
#if BLCO_GATHER == 2
    asm("ld.global.nc.L1::evict_last.u64 %0, [%1];" : "=l"(x) : "l"(p));
#else
    asm("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(x) : "l"(p));
#endif
    T r;
    memcpy(&r, &x, 8);
    return r;
  } else {
    return __ldg(p);
  }
#else
  return __ldg(p);
#endif
}


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
  // [segments, stash flushes, commit lanes, processing-phase cycles (per
  // CTA), computing-phase cycles (per warp)] or null
  unsigned long long* counters;
  // StageR: bit offset and mask of each word slot (non-target modes
  // ascending, the row last) in the packed 64-bit record field
  uint32_t pk_off[N];
  uint32_t pk_mask[N];
};

// ------------------------------------------------------------ staging layout
// A staged element is its value plus its coordinates packed as u32 words:
// words 0..N-2 hold the non-target modes (ascending), word N-1 the target row.
//   N <= 3 ("packed"): one 16-byte record {value, w0, w1} per element (one
//     LDS.128 in the computing phase) plus a u32 row plane, read four rows at
//     a time with LDS.128 when the warp is two lane groups.  Measured LSU
//     costs: LDS.128 = 2 wavefronts and LDS.64/LDS.32 = 1 per
//     warp instruction, so the record + row plane cost 1.25 wavefronts per
//     element instead of 1.6 for separate value / coordinate planes.
//   N >= 4: value f64[W] plus uint4 planes of the words (NM = ceil(N/4)).
template <int N>
struct Stage {
  static constexpr int NM = (N + 3) / 4;
  static constexpr bool kPacked = N <= 3;
  static constexpr int kRowPad = 8;  // row plane over-read by the 4-row loads
  // N >= 4: the row word sits in the last uint4 plane, so get() returns it
  // with the other words (no separate row read per element)
  static constexpr bool kRowInRecord = !kPacked;
  double* val;     // [W] (general layout)
  uint4* meta;     // general: [NM][W]; packed: records [W]
  uint32_t* rows;  // packed: [W + kRowPad]
  int W;

  __device__ __forceinline__ void put(int j, double v, const uint32_t (&w)[4 * NM]) const {
    if constexpr (kPacked) {
      const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
      meta[j] = make_uint4(static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32), N > 1 ? w[0] : 0u,
                           N > 2 ? w[1] : 0u);
      rows[j] = w[N - 1];
    } else {
      val[j] = v;
#pragma unroll
      for (int q = 0; q < NM; ++q) meta[q * W + j] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    }
  }
  // Packed layout: fills the value and the non-target words; the row word
  // (w[N-1]) comes from row() / rows4().
  __device__ __forceinline__ void get(int j, double& v, uint32_t (&w)[4 * NM]) const {
    if constexpr (kPacked) {
      const uint4 x = meta[j];
      v = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(x.y) << 32) | x.x));
      if constexpr (N > 1) w[0] = x.z;
      if constexpr (N > 2) w[1] = x.w;
    } else {
      v = val[j];
#pragma unroll
      for (int q = 0; q < NM; ++q) {
        const uint4 x = meta[q * W + j];
        w[4 * q] = x.x, w[4 * q + 1] = x.y, w[4 * q + 2] = x.z, w[4 * q + 3] = x.w;
      }
    }
  }
  __device__ __forceinline__ uint32_t row(int j) const {
    if constexpr (kPacked) {
      return rows[j];
    } else {
      const uint32_t* plane = reinterpret_cast<const uint32_t*>(meta + ((N - 1) / 4) * W);
      return plane[4 * j + (N - 1) % 4];
    }
  }
  // rows j .. j+3 (j % 4 == 0), packed layout only
  __device__ __forceinline__ uint4 rows4(int j) const { return *reinterpret_cast<const uint4*>(rows + j); }
};

template <int N>
constexpr size_t stage_bytes(int W) {
  return Stage<N>::kPacked ? static_cast<size_t>(W) * sizeof(uint4) + (W + Stage<N>::kRowPad) * sizeof(uint32_t)
                           : static_cast<size_t>(W) * (sizeof(double) + Stage<N>::NM * sizeof(uint4));
}

// A stage of W elements carved from `base` (16-byte aligned).
template <int N>
__device__ __forceinline__ Stage<N> make_stage(unsigned char* base, int W) {
  if constexpr (Stage<N>::kPacked)
    return Stage<N>{nullptr, reinterpret_cast<uint4*>(base), reinterpret_cast<uint32_t*>(base + W * sizeof(uint4)), W};
  else
    return Stage<N>{reinterpret_cast<double*>(base + Stage<N>::NM * sizeof(uint4) * W), reinterpret_cast<uint4*>(base),
                    nullptr, W};
}

// Compact staging for N = 3 when both non-target coordinates fit in 16
// bits (NELL-2: 14-15 bits): one 16-byte record {value, w0 | w1 << 16, row}
// per element and no row plane -- 20 -> 16 B of shared memory per element
// (more L1 beside the staging) and one LDS.128 per element in the computing
// phase instead of a record plus a share of the row plane.
struct StageC {
  static constexpr int NM = 1;
  static constexpr bool kPacked = true;
  static constexpr bool kRowInRecord = true;
  uint4* meta;
  __device__ __forceinline__ void put(int j, double v, const uint32_t (&w)[4]) const {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    meta[j] = make_uint4(static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32), w[0] | (w[1] << 16), w[2]);
  }
  __device__ __forceinline__ void get(int j, double& v, uint32_t (&w)[4]) const {
    const uint4 x = meta[j];
    v = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(x.y) << 32) | x.x));
    w[0] = x.z & 0xffffu;
    w[1] = x.z >> 16;
    w[2] = x.w;
  }
  __device__ __forceinline__ uint32_t row(int j) const { return reinterpret_cast<const uint32_t*>(meta)[4 * j + 3]; }
};

// Tile-relative compact staging for any order: one 16-byte record {value,
// packed} per element, packed = sum_k (w_k - cmin_k) << off_k over the word
// slots (non-target modes ascending, the row last), where cmin is the tile's
// minimum of each slot (reduced in process_cta) and off/mask come from the
// launch (Params::pk_off / pk_mask: the largest span of every mode over the
// tensor's tiles, tile_span_bits; used when they sum to <= 64 bits).
// Replaces the 20-24 bytes of Stage<N> for wide N = 3 modes (Amazon) and
// N >= 4 (Delicious: a value plane plus a uint4 plane) by one LDS.128 per
// element with the row inside.  get()/row() return the slots RELATIVE to
// cmin; the computing phase folds cmin into its lane base pointers.
template <int N>
struct StageR {
  static constexpr bool kPacked = true;
  static constexpr bool kRowInRecord = true;
  uint4* meta;
  const uint32_t* cmin;  // [N] in shared memory, valid after process_cta
  uint32_t off[N], msk[N];
  __device__ __forceinline__ void put_rel(int j, double v, const uint32_t* w, const uint32_t (&cm)[N]) const {
    uint64_t pk = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) pk |= static_cast<uint64_t>(w[k] - cm[k]) << off[k];
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
    meta[j] = make_uint4(static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32), static_cast<uint32_t>(pk),
                         static_cast<uint32_t>(pk >> 32));
  }
  template <int NW>
  __device__ __forceinline__ void get(int j, double& v, uint32_t (&w)[NW]) const {
    const uint4 x = meta[j];
    v = __longlong_as_double(static_cast<long long>((static_cast<uint64_t>(x.y) << 32) | x.x));
    const uint64_t pk = (static_cast<uint64_t>(x.w) << 32) | x.z;
#pragma unroll
    for (int k = 0; k < N; ++k) w[k] = static_cast<uint32_t>(pk >> off[k]) & msk[k];
  }
  __device__ __forceinline__ uint32_t row(int j) const {
    const uint4 x = meta[j];
    const uint64_t pk = (static_cast<uint64_t>(x.w) << 32) | x.z;
    return static_cast<uint32_t>(pk >> off[N - 1]) & msk[N - 1];
  }
};

template <class ST>
struct is_relative : std::false_type {};
template <int N>
struct is_relative<StageR<N>> : std::true_type {};

// Decodes one element into packed words (non-target modes ascending, row last).
template <int N>
__device__ __forceinline__ void decode(const Params<N>& p, const uint32_t (&base)[N], uint64_t ix,
                                       uint32_t (&w)[4 * Stage<N>::NM]) {
  uint32_t c[N];
#pragma unroll
  for (int m = 0; m < N; ++m) c[m] = base[m] | static_cast<uint32_t>((ix >> p.shift[m]) & p.mask[m]);
#pragma unroll
  for (int i = 0; i < 4 * Stage<N>::NM; ++i) w[i] = 0;
  // compile-time slots only (selects, no dynamically indexed registers)
#pragma unroll
  for (int k = 0; k + 1 < N; ++k) w[k] = k < p.mode ? c[k] : c[k + 1];
  uint32_t row = c[0];
#pragma unroll
  for (int m = 1; m < N; ++m) row = m == p.mode ? c[m] : row;
  w[N - 1] = row;
}

// ------------------------------------------------------------ column layout
// Lane q of a lane group owns columns col0 + q + c * LPE (c < CPL): every
// factor-row load and every RED of the group touches LPE consecutive doubles,
// so both are fully coalesced (a 32-column row = two 128-byte wavefronts).
template <int CPL>
struct Row {
  double v[CPL];
};

// Computing phase.  The staged positions [lo0, lo0 + wn) are split among the
// G lane groups of the warp; group starts are offset by h == 1 (mod 4)
// positions so simultaneous LDS of the groups fall in disjoint banks.
// Products accumulate in registers along a run of equal target rows and
// commit once per run (and at the end of the group's range).
template <int N, int LPE, int CPL, bool FULL, bool HIER, int U = kUnroll>
__device__ __forceinline__ void compute_range(const Params<N>& p, const Stage<N> st, int lo0, int wn,
                                              int lane, int col0, double* __restrict__ copy_out,
                                              double* stash, uint32_t* tags,
                                              unsigned long long& commits,
                                              unsigned long long& flushes) {
  constexpr int G = 32 / LPE;
  constexpr int NW = 4 * Stage<N>::NM;
  const int g = lane / LPE, q = lane % LPE;
  // Two lane groups with the packed stage: group starts 4 (mod 8) apart, so
  // the groups' 16-byte records and 4-row loads sit in disjoint banks and
  // every batch starts 4-aligned.  Otherwise 1 (mod 4) apart.
  constexpr bool kRows4 = Stage<N>::kPacked && G == 2 && U == 4;
  int h = wn / G;
  if constexpr (kRows4) {
    h = h >= 4 ? (h & ~7) | 4 : 0;  // disjoint banks, 4-aligned group starts ...
    if (h > wn) h = (wn / 2) & ~3;   // ... without overrunning the range
  } else if (G > 1 && h > 1) {
    h = (h & ~3) | 1;                 // disjoint banks ...
    if ((G - 1) * h > wn) h = wn / G;  // ... without overrunning the range (G = 8)
  }
  const int lo = lo0 + g * h;
  const int hi = g == G - 1 ? lo0 + wn : lo0 + (g + 1) * h;
  const int span = max(h, wn - (G - 1) * h);
  const int R = p.rank;
  const int col = col0 + q;
  int ncol_ok = 0;
#pragma unroll
  for (int c = 0; c < CPL; ++c) ncol_ok += (col + c * LPE < R);
  const unsigned gmask = LPE == 32 ? kFull : (((1u << LPE) - 1u) << (g * LPE));
  double acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0;

  constexpr int NO = N > 1 ? N - 1 : 1;
  for (int t0 = 0; t0 < span; t0 += U) {
    bool ok[U];
    double v[U];
    uint32_t w[U][NW];
    Row<CPL> rows[U][NO];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = lo + t0 + u;
      ok[u] = j < hi;
      st.get(ok[u] ? j : lo0, v[u], w[u]);
    }
    if constexpr (kRows4) {
      const uint4 r4 = st.rows4(lo + t0);
      w[0][N - 1] = r4.x, w[1][N - 1] = r4.y, w[2][N - 1] = r4.z, w[3][N - 1] = r4.w;
    } else if constexpr (Stage<N>::kPacked) {
#pragma unroll
      for (int u = 0; u < U; ++u) w[u][N - 1] = st.row(ok[u] ? lo + t0 + u : lo0);
    }
    const int jn = lo + t0 + U;
    const uint32_t next_row = jn < hi ? st.row(jn) : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < N - 1; ++k)
        if (ok[u] && (FULL || ncol_ok > 0)) {
          const double* rp = p.factors[k] + static_cast<uint64_t>(w[u][k]) * R;
#pragma unroll
          for (int c = 0; c < CPL; ++c)
            rows[u][k].v[c] = (FULL || c < ncol_ok) ? gather_ld(rp + col + c * LPE) : 0.0;
        }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        double prod = v[u];
#pragma unroll
        for (int k = 0; k < N - 1; ++k) prod = __dmul_rn(prod, rows[u][k].v[c]);
        acc[c] = __dadd_rn(acc[c], prod);
      }
      const uint32_t row = w[u][N - 1];
      const uint32_t nrow = u + 1 < U ? (ok[u + 1] ? w[u + 1][N - 1] : 0xffffffffu) : next_row;
      if (nrow != row) {
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
              if (FULL || c < ncol_ok) atomicAdd(&stash[static_cast<uint64_t>(slot) * R + col + c * LPE], acc[c]);
          } else {
#pragma unroll
            for (int c = 0; c < CPL; ++c)
              if (FULL || c < ncol_ok) commit_add(copy_out + static_cast<uint64_t>(row) * R + col + c * LPE, acc[c]);
            if (q == 0) ++flushes;
          }
        } else {
#pragma unroll
          for (int c = 0; c < CPL; ++c)
            if (FULL || c < ncol_ok) commit_add(copy_out + static_cast<uint64_t>(row) * R + col + c * LPE, acc[c]);
        }
        if (FULL || ncol_ok > 0) ++commits;
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
      }
    }
  }
}

// Register-path computing phase for an exact rank (FULL: R == LPE * CPL,
// one column chunk) over the packed stage -- the hot configuration.  The same
// arithmetic and commit rule as compute_range, with the per-element overhead
// stripped: the row stride is a compile-time constant, the lane's column
// offset is folded into per-mode base pointers once, and every batch but the
// group's last runs without element masks.
// PRIV: `out` is a CTA-private M_n in shared memory (k_mttkrp_priv).  Rows
// are then < kBuckets, so the bucket grouping makes every row's run in a
// tile contiguous and collision-free: a lane group owns the rows of its
// interior segments outright (plain shared-memory add) and only its first
// and last segment, which may continue in the neighbouring group, need an
// atomic (fp64 shared atomics are CAS loops).
template <int N, int LPE, int CPL, int U, class ST = Stage<N>, bool PRIV = false>
__device__ __forceinline__ void compute_range_fast(const Params<N>& p, const ST st, int lo0, int wn, int lane,
                                                   double* __restrict__ out, unsigned long long& commits) {
  constexpr int G = 32 / LPE;
  constexpr int NW = 4 * Stage<N>::NM;
  constexpr int NO = N > 1 ? N - 1 : 1;
  constexpr int RF = LPE * CPL;
  constexpr bool kRows4 = G == 2 && U == 4 && !ST::kRowInRecord && ST::kPacked;
  const int g = lane / LPE, q = lane % LPE;
  int h = wn / G;
  if constexpr (kRows4) {
    h = h >= 4 ? (h & ~7) | 4 : 0;
    if (h > wn) h = (wn / 2) & ~3;
  } else if (G > 1 && h > 1) {
    h = (h & ~3) | 1;
    if ((G - 1) * h > wn) h = wn / G;
  }
  const int lo = lo0 + g * h;
  const int n = (g == G - 1 ? wn - (G - 1) * h : h);  // my elements: [lo, lo + n)
  const double* fb[NO];
#pragma unroll
  for (int k = 0; k < N - 1; ++k) fb[k] = p.factors[k] + q;
  double* ob = out + q;
  if constexpr (is_relative<ST>::value) {  // StageR slots are relative to the tile's minimum
#pragma unroll
    for (int k = 0; k < N - 1; ++k) fb[k] += static_cast<uint64_t>(st.cmin[k]) * RF;
    ob += static_cast<uint64_t>(st.cmin[N - 1]) * RF;
  }
  double acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
  bool first_seg = true;

  auto consume = [&](const double (&v)[U], const uint32_t (&w)[U][NW], const Row<CPL> (&rows)[U][NO],
                     uint32_t next_row, int valid) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u < valid) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          double prod = v[u];
#pragma unroll
          for (int k = 0; k < N - 1; ++k) prod = __dmul_rn(prod, rows[u][k].v[c]);
          acc[c] = __dadd_rn(acc[c], prod);
        }
        const uint32_t row = w[u][N - 1];
        const uint32_t nrow = u + 1 < valid ? w[u + 1][N - 1] : next_row;
        if (nrow != row) {
          double* o = ob + static_cast<uint64_t>(row) * RF;
          if constexpr (PRIV) {
            if (first_seg || (u + 1 >= valid && next_row == 0xffffffffu)) {
#pragma unroll
              for (int c = 0; c < CPL; ++c) atomicAdd(o + c * LPE, acc[c]);
            } else {
#pragma unroll
              for (int c = 0; c < CPL; ++c) o[c * LPE] += acc[c];
            }
            first_seg = false;
          } else {
#pragma unroll
            for (int c = 0; c < CPL; ++c) commit_add(o + c * LPE, acc[c]);
          }
          ++commits;
#pragma unroll
          for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
        }
      }
    }
  };

  const int nfull = n / U;
  for (int b = 0; b < nfull; ++b) {
    const int j0 = lo + b * U;
    double v[U];
    uint32_t w[U][NW];
    Row<CPL> rows[U][NO];
#pragma unroll
    for (int u = 0; u < U; ++u) st.get(j0 + u, v[u], w[u]);
    if constexpr (ST::kRowInRecord) {
      // the row came with the record
    } else if constexpr (kRows4) {
      const uint4 r4 = st.rows4(j0);
      w[0][N - 1] = r4.x, w[1][N - 1] = r4.y, w[2][N - 1] = r4.z, w[3][N - 1] = r4.w;
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) w[u][N - 1] = st.row(j0 + u);
    }
    const uint32_t next_row = j0 + U < lo + n ? st.row(j0 + U) : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < N - 1; ++k) {
        const double* rp = fb[k] + static_cast<uint64_t>(w[u][k]) * RF;
#pragma unroll
        for (int c = 0; c < CPL; ++c) rows[u][k].v[c] = gather_ld(rp + c * LPE);
      }
    consume(v, w, rows, next_row, U);
  }
  const int rem = n - nfull * U;
  if (rem > 0) {
    const int j0 = lo + nfull * U;
    double v[U];
    uint32_t w[U][NW];
    Row<CPL> rows[U][NO];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = u < rem ? j0 + u : j0;
      st.get(j, v[u], w[u]);
      if constexpr (!ST::kRowInRecord) w[u][N - 1] = st.row(j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < N - 1; ++k)
        if (u < rem) {
          const double* rp = fb[k] + static_cast<uint64_t>(w[u][k]) * RF;
#pragma unroll
          for (int c = 0; c < CPL; ++c) rows[u][k].v[c] = gather_ld(rp + c * LPE);
        }
    consume(v, w, rows, 0xffffffffu, rem);
  }
}

__device__ __forceinline__ uint32_t tile_count(const TileDesc& td, uint64_t elem_end) {
  const uint64_t room = td.start >= elem_end ? 0 : elem_end - td.start;
  return room < td.count ? static_cast<uint32_t>(room) : td.count;
}

// ------------------------------------------------ processing: paper variant
// Per warp, per 32-element sub-tile (the reference's tile, mttkrp.cpp:23-81):
// __match_any_sync groups equal target rows and a warp prefix sum over group
// sizes places each group contiguously -- the stable reorder of :55-73
// without the O(tile^2) rank.  Segments = groups.
template <int N>
__device__ __forceinline__ int process_warp(const Params<N>& p, const TileDesc& td, int warp,
                                            int lane, const Stage<N> st, unsigned long long& segs) {
  const uint32_t wbeg = static_cast<uint32_t>(warp) * kWarpElems;
  const uint32_t cnt = tile_count(td, p.elem_end);
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
    uint32_t w[4 * Stage<N>::NM];
    decode<N>(p, base, ix[s], w);
    const uint32_t key = valid ? w[N - 1] : 0xffffffffu;  // dims < 2^31: never a real row
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
    if (valid) st.put(s * 32 + goff + rin, vv[s], w);
    segs += __popc(__ballot_sync(kFull, valid && lane == leader));
  }
  __syncwarp();
  return wn;
}

// ----------------------------------------- processing: CTA bucket grouping
// The whole 1024-element tile is grouped by target row with a one-pass
// counting sort on the row's low kBucketBits bits: a shared-memory histogram
// (ATOMS.ADD gives each element its rank in its bucket), a block exclusive
// scan, a scatter.  ALTO order makes a tile's rows a few short contiguous
// ranges, so distinct rows almost never share a bucket and each row's
// elements end up adjacent; a shared bucket only splits a run (one extra
// commit), never mixes results.  Segments drop from ~0.91 to ~0.33 per
// non-zero on NELL-2 (SURVEY §8a row a13 replaced).
constexpr int kBucketBits = 11;
constexpr int kBuckets = 1 << kBucketBits;
struct BucketShared {
  uint32_t cnt[kBuckets];
  uint32_t warp_sum[kWarps];
  uint32_t cmin[8];  // StageR: the tile's minimum of each word slot
};

template <int N, int TILE = kTileElems, class ST = Stage<N>>
__device__ __forceinline__ uint32_t process_cta(const Params<N>& p, const TileDesc& td, const ST st,
                                                BucketShared& bs, unsigned long long& segs) {
  constexpr int kItems = TILE / kCtaThreads;  // elements per thread
  constexpr bool REL = is_relative<ST>::value;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cnt = tile_count(td, p.elem_end);
  for (int i = tid; i < kBuckets; i += kCtaThreads) bs.cnt[i] = 0;
  if constexpr (REL)
    if (tid < N) bs.cmin[tid] = 0xffffffffu;
  uint32_t base[N];
#pragma unroll
  for (int m = 0; m < N; ++m) base[m] = __ldg(p.block_base + static_cast<uint64_t>(td.block) * N + m);
  uint64_t ix[kItems];
  double vv[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint32_t e = tid + i * kCtaThreads;
    ix[i] = e < cnt ? __ldcs(p.idx + td.start + e) : 0;
    vv[i] = e < cnt ? __ldcs(p.val + td.start + e) : 0.0;
  }
  __syncthreads();
  uint32_t w[kItems][4 * Stage<N>::NM];
  uint32_t rank[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    decode<N>(p, base, ix[i], w[i]);
    const uint32_t e = tid + i * kCtaThreads;
    rank[i] = e < cnt ? atomicAdd(&bs.cnt[w[i][N - 1] & (kBuckets - 1)], 1u) : 0;
  }
  if constexpr (REL) {  // the tile's minimum of each word slot (StageR)
#pragma unroll
    for (int k = 0; k < N; ++k) {
      uint32_t m = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < kItems; ++i)
        if (tid + i * kCtaThreads < cnt) m = min(m, w[i][k]);
      m = __reduce_min_sync(kFull, m);
      if (lane == 0) atomicMin(&bs.cmin[k], m);
    }
  }
  __syncthreads();
  // exclusive scan of the histogram: thread t owns buckets [8t, 8t+8)
  constexpr int per = kBuckets / kCtaThreads;
  uint32_t loc[per], run = 0;
#pragma unroll
  for (int i = 0; i < per; ++i) {
    loc[i] = run;
    run += bs.cnt[tid * per + i];
  }
  uint32_t x = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) bs.warp_sum[warp] = x;
  __syncthreads();
  uint32_t woff = 0;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) woff += i < warp ? bs.warp_sum[i] : 0;
  const uint32_t toff = woff + x - run;
#pragma unroll
  for (int i = 0; i < per; ++i) bs.cnt[tid * per + i] = toff + loc[i];
  __syncthreads();
  if constexpr (REL) {
    uint32_t cm[N];
#pragma unroll
    for (int k = 0; k < N; ++k) cm[k] = bs.cmin[k];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t e = tid + i * kCtaThreads;
      if (e < cnt) st.put_rel(static_cast<int>(bs.cnt[w[i][N - 1] & (kBuckets - 1)] + rank[i]), vv[i], w[i], cm);
    }
  } else {
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t e = tid + i * kCtaThreads;
      if (e < cnt) st.put(static_cast<int>(bs.cnt[w[i][N - 1] & (kBuckets - 1)] + rank[i]), vv[i], w[i]);
    }
  }
  __syncthreads();
  if (segs != ~0ull) {  // count runs (stats only)
    unsigned n = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t j = tid * kItems + i;
      if (j < cnt) n += j + 1 == cnt || st.row(j + 1) != st.row(j);
    }
    segs += n;
  }
  return cnt;
}

template <int N, int LPE, int CPL, bool FULL, bool STATS>
__global__ void __launch_bounds__(kCtaThreads) k_mttkrp_warp(Params<N> p) {
  extern __shared__ __align__(16) unsigned char dyn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = stage_bytes<N>(kWarpElems);
  unsigned char* mine = dyn + warp * per_warp;
  const Stage<N> st = make_stage<N>(mine, kWarpElems);
  const TileDesc td = p.tiles[blockIdx.x];
  unsigned long long segs = 0, commits = 0, flushes = 0;
  const int wn = process_warp<N>(p, td, warp, lane, st, segs);
  if (wn > 0)
    compute_range<N, LPE, CPL, FULL, false>(p, st, 0, wn, lane, blockIdx.y * LPE * CPL, p.out, nullptr,
                                            nullptr, commits, flushes);
  if constexpr (STATS) {
    if (lane == 0 && blockIdx.y == 0 && segs) atomicAdd(&p.counters[0], segs);
    unsigned long long c = commits;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) c += __shfl_down_sync(kFull, c, d);
    if (lane == 0 && c) atomicAdd(&p.counters[2], c);
  }
}

template <int N, int TILE = kTileElems>
__device__ __forceinline__ Stage<N> cta_stage(unsigned char* dyn) {
  return make_stage<N>(dyn, TILE);
}

// TILE = elements per CTA tile: 1024, or 2048 for large tensors whose
// gathered factor matrices sit in L2 (the L1-pipe-bound regime: fewer
// segments, so fewer commits, and the per-tile fixed costs halve; NELL-2
// 8.29 -> 7.96 ms/iter).  DRAM-bound shapes (Amazon) and small tensors
// (fewer tiles than resident CTA slots) keep 1024.
// CMP (stage kind): 0 = Stage<N>, 1 = StageC (N = 3, absolute 16-bit
// coordinates), 2 = StageR<N> (tile-relative packed record)
template <int N, int LPE, int CPL, bool FULL, bool STATS, int U = kUnroll, int MINB = 1, int TILE = kTileElems,
          int CMP = 0>
__global__ void __launch_bounds__(kCtaThreads, MINB) k_mttkrp_sorted(Params<N> p) {
  constexpr int WE = TILE / kWarps;  // staged positions per warp
  using ST = std::conditional_t<CMP == 1, StageC, std::conditional_t<CMP == 2, StageR<N>, Stage<N>>>;
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ BucketShared bs;
  ST st;
  if constexpr (CMP == 1) {
    st = StageC{reinterpret_cast<uint4*>(dyn)};
  } else if constexpr (CMP == 2) {
    st.meta = reinterpret_cast<uint4*>(dyn);
    st.cmin = bs.cmin;
#pragma unroll
    for (int k = 0; k < N; ++k) st.off[k] = p.pk_off[k], st.msk[k] = p.pk_mask[k];
  } else {
    st = cta_stage<N, TILE>(dyn);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TileDesc td = p.tiles[blockIdx.x];
  unsigned long long segs = STATS ? 0 : ~0ull, commits = 0, flushes = 0;
  long long t0 = STATS ? clock64() : 0;
  const uint32_t cnt = process_cta<N, TILE, ST>(p, td, st, bs, segs);
  long long t1 = STATS ? clock64() : 0;
  const int lo0 = warp * WE;
  const int wn = static_cast<int>(cnt) > lo0 ? min(WE, static_cast<int>(cnt) - lo0) : 0;
  if (wn > 0) {
    if constexpr (FULL && U == 4)  // lean phase for every order (N >= 4: general stage, no 4-row loads)
      compute_range_fast<N, LPE, CPL, U, ST>(p, st, lo0, wn, lane, p.out, commits);
    else if constexpr (CMP == 0)
      compute_range<N, LPE, CPL, FULL, false, U>(p, st, lo0, wn, lane, blockIdx.y * LPE * CPL, p.out, nullptr,
                                              nullptr, commits, flushes);
  }
  if constexpr (STATS) {
    const long long t2 = clock64();
    if (lane == 0) {
      if (threadIdx.x == 0) atomicAdd(&p.counters[3], static_cast<unsigned long long>(t1 - t0));
      atomicAdd(&p.counters[4], static_cast<unsigned long long>(t2 - t1));
    }
    unsigned long long s = blockIdx.y == 0 ? segs : 0, c = commits;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      s += __shfl_down_sync(kFull, s, d);
      c += __shfl_down_sync(kFull, c, d);
    }
    if (lane == 0 && s) atomicAdd(&p.counters[0], s);
    if (lane == 0 && c) atomicAdd(&p.counters[2], c);
  }
}

// ----------------------------------------- all-mode fused kernel (N = 3)
// B200 extension for the all-mode step with fixed factors (BASELINE's
// "MTTKRP time/iter (all modes)"; also the gradient of all-at-once CP
// methods): every element is staged once, its three factor rows are gathered
// once, and its three per-mode terms are formed in the oracle's product
// order (oracle.cpp:15-24: value first, the other modes ascending):
//   M0 += (v A1) A2,   M1 += (v A0) A2,   M2 += (v A0) A1,
// so every term is bit-identical to the per-mode kernels' and only the
// summation order differs.  The tile is grouped by the row of mode GM
// (process_cta with p.mode = GM), so GM's terms accumulate along runs and
// commit once per run; the other two modes commit per element (merged while
// consecutive elements share a row).  Used when all three factors and
// outputs sit in L2 (NELL-2: 26 MB), where the per-mode kernels are bound by
// the L1 data pipe: 3 row gathers per element per step instead of 6, and one
// staging pass instead of three.
struct FusedOut {
  const double* f[3];
  double* out[3];
};

template <int GM, int LPE, int CPL, int U, class ST>
__device__ __forceinline__ void compute_fused(const ST st, int lo0, int wn, int lane, const FusedOut& fo) {
  constexpr int G = 32 / LPE;
  constexpr int RF = LPE * CPL;
  constexpr int MA = GM == 0 ? 1 : 0, MB = GM == 2 ? 1 : 2;  // the other modes, ascending
  const int g = lane / LPE, q = lane % LPE;
  int h = wn / G;
  if (G > 1 && h > 1) {
    h = (h & ~3) | 1;  // groups' staged records in disjoint banks
    if ((G - 1) * h > wn) h = wn / G;
  }
  const int lo = lo0 + g * h;
  const int n = (g == G - 1 ? wn - (G - 1) * h : h);
  const double* fb[3] = {fo.f[0] + q, fo.f[1] + q, fo.f[2] + q};
  double* ob[3] = {fo.out[0] + q, fo.out[1] + q, fo.out[2] + q};
  double acc[CPL], pa[CPL], pb[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = pa[c] = pb[c] = 0.0;
  uint32_t ra = 0xffffffffu, rb = 0xffffffffu;
  auto flush = [&](double (&x)[CPL], uint32_t row, int m) {
    if (row == 0xffffffffu) return;
    double* o = ob[m] + static_cast<uint64_t>(row) * RF;
#pragma unroll
    for (int c = 0; c < CPL; ++c) commit_add(o + c * LPE, x[c]);
  };
  for (int b0 = 0; b0 < n; b0 += U) {
    const int valid = min(U, n - b0);
    const int j0 = lo + b0;
    double v[U];
    uint32_t w[U][4];
    double rows[U][3][CPL];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = u < valid ? j0 + u : j0;
      st.get(j, v[u], w[u]);
      if constexpr (!ST::kRowInRecord) w[u][2] = st.row(j);
    }
    const uint32_t next_row = b0 + U < n ? st.row(j0 + U) : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (u < valid) {
        uint32_t c3[3];
        c3[GM] = w[u][2], c3[MA] = w[u][0], c3[MB] = w[u][1];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const double* rp = fb[m] + static_cast<uint64_t>(c3[m]) * RF;
#pragma unroll
          for (int c = 0; c < CPL; ++c) rows[u][m][c] = gather_ld(rp + c * LPE);
        }
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u >= valid) continue;
      double t[3][CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const double v0 = __dmul_rn(v[u], rows[u][0][c]);  // shared by the mode-1 and mode-2 terms
        t[0][c] = __dmul_rn(__dmul_rn(v[u], rows[u][1][c]), rows[u][2][c]);
        t[1][c] = __dmul_rn(v0, rows[u][2][c]);
        t[2][c] = __dmul_rn(v0, rows[u][1][c]);
      }
      // grouped mode: run accumulation, one commit per run
#pragma unroll
      for (int c = 0; c < CPL; ++c) acc[c] = __dadd_rn(acc[c], t[GM][c]);
      const uint32_t row = w[u][2];
      const uint32_t nrow = u + 1 < valid ? w[u + 1][2] : (b0 + U < n ? next_row : 0xffffffffu);
      if (nrow != row) {
        double* o = ob[GM] + static_cast<uint64_t>(row) * RF;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          commit_add(o + c * LPE, acc[c]);
          acc[c] = 0.0;
        }
      }
      // the other two modes: per element, merged while the row repeats
      const uint32_t a = w[u][0], b = w[u][1];
      if (a != ra) {
        flush(pa, ra, MA);
        ra = a;
#pragma unroll
        for (int c = 0; c < CPL; ++c) pa[c] = t[MA][c];
      } else {
#pragma unroll
        for (int c = 0; c < CPL; ++c) pa[c] = __dadd_rn(pa[c], t[MA][c]);
      }
      if (b != rb) {
        flush(pb, rb, MB);
        rb = b;
#pragma unroll
        for (int c = 0; c < CPL; ++c) pb[c] = t[MB][c];
      } else {
#pragma unroll
        for (int c = 0; c < CPL; ++c) pb[c] = __dadd_rn(pb[c], t[MB][c]);
      }
    }
  }
  flush(pa, ra, MA);
  flush(pb, rb, MB);
}

template <int GM, int LPE, int CPL, int TILE, bool CMP, int MINB, int U>
__global__ void __launch_bounds__(kCtaThreads, MINB) k_mttkrp_all3(Params<3> p, FusedOut fo) {
  constexpr int WE = TILE / kWarps;
  using ST = std::conditional_t<CMP, StageC, Stage<3>>;
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ BucketShared bs;
  ST st;
  if constexpr (CMP) st = StageC{reinterpret_cast<uint4*>(dyn)};
  else st = cta_stage<3, TILE>(dyn);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TileDesc td = p.tiles[blockIdx.x];
  unsigned long long segs = ~0ull;
  const uint32_t cnt = process_cta<3, TILE, ST>(p, td, st, bs, segs);
  const int lo0 = warp * WE;
  const int wn = static_cast<int>(cnt) > lo0 ? min(WE, static_cast<int>(cnt) - lo0) : 0;
  if (wn > 0) compute_fused<GM, LPE, CPL, U, ST>(st, lo0, wn, lane, fo);
}

// ------------------------------------------------ fp32 variant (register)
// The same processing phase (CTA bucket grouping, fp64 values staged), with
// fp32 factors, products and output (SURVEY.md 8c/8d "fp32 variant": 1e-5
// relative Frobenius against the fp64 oracle; B_elem = 8 + 4 + N*R*4).
// Lane q of a group owns V adjacent columns (V*q .. V*q+V-1, then + V*LPE per
// chunk c), so a 32-float row is one 128-byte access of a 16-lane group and a
// commit is one vector RED (atomicAdd on float2), both a single L1 wavefront.
// Products are formed in the oracle's order: value (rounded to fp32) first,
// then the non-target modes ascending.
template <int N>
struct ParamsF32 {
  Params<N> base;            // payload, tiles, decode tables (processing phase)
  const float* factors[N];   // non-target modes, ascending
  float* out;
};

template <int V>
struct VecF;
template <>
struct VecF<1> {
  using type = float;
  static __device__ __forceinline__ float get(const type& x, int) { return x; }
};
template <>
struct VecF<2> {
  using type = float2;
  static __device__ __forceinline__ float get(const type& x, int i) { return i ? x.y : x.x; }
};

template <int N, int LPE, int V, int CPL, bool FULL>
__device__ __forceinline__ void compute_range_f32(const ParamsF32<N>& p, const Stage<N> st, int lo0, int wn,
                                                  int lane, int col0) {
  using VT = typename VecF<V>::type;
  constexpr int G = 32 / LPE;
  constexpr int NW = 4 * Stage<N>::NM;
  constexpr int NO = N > 1 ? N - 1 : 1;
  const int g = lane / LPE, q = lane % LPE;
  int h = wn / G;
  if (G > 1 && h > 1) {
    h = (h & ~3) | 1;                   // group starts in disjoint banks ...
    if ((G - 1) * h > wn) h = wn / G;   // ... unless that overruns the warp's range (G = 8)
  }
  const int lo = lo0 + g * h;
  const int hi = g == G - 1 ? lo0 + wn : lo0 + (g + 1) * h;
  const int span = max(h, wn - (G - 1) * h);
  const int R = p.base.rank;
  bool cok[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) cok[c] = FULL || col0 + V * (q + LPE * c) < R;
  float acc[CPL][V];
#pragma unroll
  for (int c = 0; c < CPL; ++c)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[c][v] = 0.0f;
  for (int t0 = 0; t0 < span; t0 += kUnroll) {
    bool ok[kUnroll];
    double val[kUnroll];
    uint32_t w[kUnroll][NW];
    VT rows[kUnroll][NO][CPL];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int j = lo + t0 + u;
      ok[u] = j < hi;
      st.get(ok[u] ? j : lo0, val[u], w[u]);
      if constexpr (Stage<N>::kPacked) w[u][N - 1] = st.row(ok[u] ? j : lo0);
    }
    const int jn = lo + t0 + kUnroll;
    const uint32_t next_row = jn < hi ? st.row(jn) : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
      for (int k = 0; k < N - 1; ++k)
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          if (ok[u] && cok[c])
            rows[u][k][c] = gather_ld(reinterpret_cast<const VT*>(p.factors[k] + static_cast<uint64_t>(w[u][k]) * R +
                                                              col0 + V * (q + LPE * c)));
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (!ok[u]) continue;
      const float vf = __double2float_rn(val[u]);
#pragma unroll
      for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) {
          float prod = vf;
#pragma unroll
          for (int k = 0; k < N - 1; ++k) prod = __fmul_rn(prod, VecF<V>::get(rows[u][k][c], v));
          acc[c][v] = __fadd_rn(acc[c][v], prod);
        }
      const uint32_t row = w[u][N - 1];
      const uint32_t nrow = u + 1 < kUnroll ? (ok[u + 1] ? w[u + 1][N - 1] : 0xffffffffu) : next_row;
      if (nrow != row) {
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          if (cok[c]) {
            float* o = p.out + static_cast<uint64_t>(row) * R + col0 + V * (q + LPE * c);
            if constexpr (V == 2) atomicAdd(reinterpret_cast<float2*>(o), make_float2(acc[c][0], acc[c][1]));
            else atomicAdd(o, acc[c][0]);
          }
#pragma unroll
        for (int c = 0; c < CPL; ++c)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[c][v] = 0.0f;
      }
    }
  }
}

// Lean fp32 computing phase for an exact rank (R == LPE * V), packed stage.
template <int N, int LPE, int V, class ST = Stage<N>>
__device__ __forceinline__ void compute_range_f32_fast(const ParamsF32<N>& p, const ST st, int lo0, int wn,
                                                       int lane) {
  using VT = typename VecF<V>::type;
  constexpr int G = 32 / LPE;
  constexpr int NW = 4 * Stage<N>::NM;
  constexpr int NO = N > 1 ? N - 1 : 1;
  constexpr int RF = LPE * V;
  constexpr int U = kUnroll;
  constexpr bool kRows4 = G == 2 && U == 4 && !ST::kRowInRecord && ST::kPacked;
  const int g = lane / LPE, q = lane % LPE;
  int h = wn / G;
  if constexpr (kRows4) {
    h = h >= 4 ? (h & ~7) | 4 : 0;
    if (h > wn) h = (wn / 2) & ~3;
  } else if (G > 1 && h > 1) {
    h = (h & ~3) | 1;
    if ((G - 1) * h > wn) h = wn / G;
  }
  const int lo = lo0 + g * h;
  const int n = (g == G - 1 ? wn - (G - 1) * h : h);
  const float* fb[NO];
#pragma unroll
  for (int k = 0; k < N - 1; ++k) fb[k] = p.factors[k] + V * q;
  float* const ob = p.out + V * q;
  float acc[V];
#pragma unroll
  for (int x = 0; x < V; ++x) acc[x] = 0.0f;

  auto consume = [&](const double (&v)[U], const uint32_t (&w)[U][NW], const VT (&rows)[U][NO],
                     uint32_t next_row, int valid) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u < valid) {
        const float vf = __double2float_rn(v[u]);
#pragma unroll
        for (int x = 0; x < V; ++x) {
          float prod = vf;
#pragma unroll
          for (int k = 0; k < N - 1; ++k) prod = __fmul_rn(prod, VecF<V>::get(rows[u][k], x));
          acc[x] = __fadd_rn(acc[x], prod);
        }
        const uint32_t row = w[u][N - 1];
        const uint32_t nrow = u + 1 < valid ? w[u + 1][N - 1] : next_row;
        if (nrow != row) {
          float* o = ob + static_cast<uint64_t>(row) * RF;
          if constexpr (V == 2) atomicAdd(reinterpret_cast<float2*>(o), make_float2(acc[0], acc[1]));
          else atomicAdd(o, acc[0]);
#pragma unroll
          for (int x = 0; x < V; ++x) acc[x] = 0.0f;
        }
      }
    }
  };
  const int nfull = n / U;
  for (int b = 0; b < nfull; ++b) {
    const int j0 = lo + b * U;
    double v[U];
    uint32_t w[U][NW];
    VT rows[U][NO];
#pragma unroll
    for (int u = 0; u < U; ++u) st.get(j0 + u, v[u], w[u]);
    if constexpr (ST::kRowInRecord) {
      // the row came with the record
    } else if constexpr (kRows4) {
      const uint4 r4 = st.rows4(j0);
      w[0][N - 1] = r4.x, w[1][N - 1] = r4.y, w[2][N - 1] = r4.z, w[3][N - 1] = r4.w;
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) w[u][N - 1] = st.row(j0 + u);
    }
    const uint32_t next_row = j0 + U < lo + n ? st.row(j0 + U) : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < N - 1; ++k)
        rows[u][k] = gather_ld(reinterpret_cast<const VT*>(fb[k] + static_cast<uint64_t>(w[u][k]) * RF));
    consume(v, w, rows, next_row, U);
  }
  const int rem = n - nfull * U;
  if (rem > 0) {
    const int j0 = lo + nfull * U;
    double v[U];
    uint32_t w[U][NW];
    VT rows[U][NO];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = u < rem ? j0 + u : j0;
      st.get(j, v[u], w[u]);
      w[u][N - 1] = st.row(j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < N - 1; ++k)
        if (u < rem) rows[u][k] = gather_ld(reinterpret_cast<const VT*>(fb[k] + static_cast<uint64_t>(w[u][k]) * RF));
    consume(v, w, rows, 0xffffffffu, rem);
  }
}

template <int N, int LPE, int V, int CPL, bool FULL, int TILE = kTileElems, int MINB = 1, bool CMP = false>
__global__ void __launch_bounds__(kCtaThreads, MINB) k_mttkrp_sorted_f32(ParamsF32<N> p) {
  constexpr int WE = TILE / kWarps;
  using ST = std::conditional_t<CMP, StageC, Stage<N>>;
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ BucketShared bs;
  ST st;
  if constexpr (CMP) st = StageC{reinterpret_cast<uint4*>(dyn)};
  else st = cta_stage<N, TILE>(dyn);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TileDesc td = p.base.tiles[blockIdx.x];
  unsigned long long segs = ~0ull;
  const uint32_t cnt = process_cta<N, TILE, ST>(p.base, td, st, bs, segs);
  const int lo0 = warp * WE;
  const int wn = static_cast<int>(cnt) > lo0 ? min(WE, static_cast<int>(cnt) - lo0) : 0;
  if (wn > 0) {
    if constexpr (FULL && CPL == 1)  // lean phase for every order
      compute_range_f32_fast<N, LPE, V, ST>(p, st, lo0, wn, lane);
    else if constexpr (!CMP)
      compute_range_f32<N, LPE, V, CPL, FULL>(p, st, lo0, wn, lane, blockIdx.y * LPE * V * CPL);
  }
}

// Persistent CTAs; dynamic shared memory = tile stage + stash (slots x R
// doubles + tags).
// Hierarchical strategy, privatised form (exact ranks, N <= 3): when the
// whole target mode fits in shared memory beside the staging, each
// persistent CTA accumulates its segment sums into a private copy of M_n in
// shared memory -- the reference's work-group stash with one slot per row,
// so nothing is ever evicted (mttkrp.cpp:139-155, 83-89) -- and flushes it
// once at the end, one RED per non-zero element.  The computing phase is
// K4's lean one with the commit target in shared memory, so a short,
// high-conflict mode costs no global atomics per tile.
template <int N, int LPE, int CPL>
__global__ void __launch_bounds__(kCtaThreads) k_mttkrp_priv(Params<N> p) {
  constexpr int WE = kTileElems / kWarps;
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ BucketShared bs;
  const Stage<N> st = cta_stage<N>(dyn);
  double* const priv = reinterpret_cast<double*>(dyn + stage_bytes<N>(kTileElems));
  const uint64_t elems = p.copy_elems;  // I_n * R
  for (uint64_t i = threadIdx.x; i < elems; i += blockDim.x) priv[i] = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long segs = ~0ull, commits = 0;
  for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const TileDesc td = p.tiles[tile];
    const uint32_t cnt = process_cta<N>(p, td, st, bs, segs);  // its barriers also order the zeroing
    const int lo0 = warp * WE;
    const int wn = static_cast<int>(cnt) > lo0 ? min(WE, static_cast<int>(cnt) - lo0) : 0;
    if (wn > 0) compute_range_fast<N, LPE, CPL, kUnroll, Stage<N>, true>(p, st, lo0, wn, lane, priv, commits);
    __syncthreads();  // stage reused by the next tile
  }
  for (uint64_t i = threadIdx.x; i < elems; i += blockDim.x) {
    const double v = priv[i];
    if (v != 0.0) atomicAdd(p.out + i, v);
  }
}

template <int N, int LPE, int CPL, bool FULL, bool STATS>
__global__ void __launch_bounds__(kCtaThreads) k_mttkrp_hier(Params<N> p) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ BucketShared bs;
  const Stage<N> st = cta_stage<N>(dyn);
  const int S = p.stash_slots, R = p.rank;
  double* stash = reinterpret_cast<double*>(dyn + stage_bytes<N>(kTileElems));
  uint32_t* tags = reinterpret_cast<uint32_t*>(stash + static_cast<uint64_t>(S) * R);
  for (int i = threadIdx.x; i < S * R; i += blockDim.x) stash[i] = 0.0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) tags[i] = 0u;
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int copy = static_cast<int>(blockIdx.x % static_cast<unsigned>(p.ncopies));
  double* copy_out = p.out + static_cast<uint64_t>(copy) * p.copy_elems;
  unsigned long long segs = STATS ? 0 : ~0ull, commits = 0, flushes = 0;
  for (uint64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const TileDesc td = p.tiles[tile];
    const uint32_t cnt = process_cta<N>(p, td, st, bs, segs);
    const int lo0 = warp * kWarpElems;
    const int wn = static_cast<int>(cnt) > lo0 ? min(kWarpElems, static_cast<int>(cnt) - lo0) : 0;
    if (wn > 0)
      compute_range<N, LPE, CPL, FULL, true>(p, st, lo0, wn, lane, blockIdx.y * LPE * CPL, copy_out, stash,
                                             tags, commits, flushes);
    __syncthreads();  // stage reused by the next tile
  }
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
    unsigned long long sg = blockIdx.y == 0 ? segs : 0, c = commits, f = flushes + (blockIdx.y == 0 ? occ : 0);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      sg += __shfl_down_sync(kFull, sg, d);
      c += __shfl_down_sync(kFull, c, d);
      f += __shfl_down_sync(kFull, f, d);
    }
    if (lane == 0 && sg) atomicAdd(&p.counters[0], sg);
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
  v.tensor = &t;
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
  // hierarchical factor copies, one buffer per stream: launches on
  // different streams of one thread may run concurrently
  std::map<cudaStream_t, DevBuf<double>> copies;
  DevBuf<unsigned long long> counters;
  int device = -1;
};
thread_local Workspace t_ws;

}  // namespace

void release_mttkrp_workspace() {
  t_ws.copies.clear();
  t_ws.counters.reset();
  t_ws.device = -1;
}

namespace {

// Per-thread scratch, re-created when the calling thread changes device.
Workspace& workspace() {
  int dev = 0;
  B200_CUDA(cudaGetDevice(&dev));
  if (t_ws.device != dev) {
    t_ws.copies.clear();
    t_ws.counters.reset();
    t_ws.device = dev;
  }
  return t_ws;
}

// Register-path processing variant: "sorted" (CTA-wide row sort, default)
// or "warp" (the paper's 32-element tiles); BLCO_B200_VARIANT selects.
bool use_warp_variant() {
  static const bool warp = [] {
    const char* e = std::getenv("BLCO_B200_VARIANT");
    return e && std::string(e) == "warp";
  }();
  return warp;
}

// 2048-element tiles when the non-target factor matrices fit in L2 with
// room to spare and there are enough tiles to fill every resident CTA slot
// several times (k_mttkrp_sorted).  BLCO_B200_BIG_TILES=0/1 overrides.
bool use_big_tiles(const blco_layout& l, int mode, uint64_t rank, uint64_t nnz, uint64_t elem_bytes = 8) {
  static const int knob = [] {
    const char* e = std::getenv("BLCO_B200_BIG_TILES");
    return e ? std::atoi(e) : -1;
  }();
  if (knob >= 0) return knob > 0;
  uint64_t fbytes = 0;
  for (int m = 0; m < l.order; ++m)
    if (m != mode) fbytes += l.dims[m] * rank * elem_bytes;
  return fbytes <= (uint64_t(48) << 20) && nnz >= uint64_t(2 * kTileElems) * sm_count() * 3 * 4;
}

// BLCO_B200_COMPACT_STAGE=0 disables the compact N = 3 staging (StageC).
bool compact_stage_knob() {
  static const bool on = [] {
    const char* e = std::getenv("BLCO_B200_COMPACT_STAGE");
    return !(e && std::string(e) == "0");
  }();
  return on;
}

// ---- panel-ordered tile tables (orders >= 3, factors beyond L2)
// The tile table fixes only the order CTAs are dispatched in; any order gives
// the same terms (the commits are atomic, mttkrp.cpp:95-137 sums a segment
// in element order inside one tile, which is kept).  ALTO order is a
// Z-curve: a window of concurrent tiles is a box about equally wide in
// every mode, so when the factors exceed L2 (Amazon: 1.2 + 2 x 0.45 GB at
// R = 32) every target row misses (RED read-modify-write) and the gathered
// rows are reused ~1.7x per mode (ncu: 433 DRAM bytes per element per mode).
// A panel order is the loop nest
//   for X-panel (target mode, 2^bx rows)  for Y-panel (2^by rows of the
//   second-longest non-target mode)  for tiles of the panel in ALTO order,
// so a window of concurrent tiles spans few output and Y rows (they stay in
// L2 across the panel) while the longest non-target mode Z streams.  Y
// panels are walked boustrophedon so consecutive panels share their Y rows.
// Each tile is assigned to the panel of its middle element.  Measured on
// the Amazon shape (scripts/panel_probe.py, B200): 16,16 panels at R = 32
// cut the DRAM bytes of a mode launch from 760 to 506 GB (the output rows'
// write-backs from 215 to 29 GB) and the all-mode step from 384 to 345 ms;
// wider panels (17,17: 354 ms; 18,16: 371 ms) overflow L2 with the
// streamed rows, narrower ones (14,14: 361 ms) lose the reuse.
// BLCO_B200_PANEL: "0" off; "bx,by" fixed widths; default: both widths from
// BLCO_B200_PANEL_MB (default 32) of L2 for the panel's X + Y rows
// (R = 32: 2^16 rows each).
struct PanelPlan {
  int x = -1, y = -1;
  int bx = 0, by = 0;
};

PanelPlan panel_plan(const blco_layout& l, int mode, uint64_t rank, uint64_t elem_bytes) {
  PanelPlan p;
  if (l.order < 3 || rank == 0) return p;
  uint64_t bytes = 0;
  for (int m = 0; m < l.order; ++m) bytes += l.dims[m] * rank * elem_bytes;
  if (bytes <= (uint64_t(96) << 20)) return p;  // L2-resident working set: ALTO order is already local
  // read per call (only reached by launches over GBs of factors), so a probe
  // can sweep the widths in one process
  const char* ek = std::getenv("BLCO_B200_PANEL");
  const std::string knob = ek ? ek : "";
  const char* em = std::getenv("BLCO_B200_PANEL_MB");
  const uint64_t budget_mb = em ? std::strtoull(em, nullptr, 10) : 32ull;
  if (knob == "0") return p;
  // Z = the longest non-target mode (streamed), Y = the next longest; for
  // orders > 3 the remaining modes are left to L2 (short modes: Delicious'
  // 1443 rows)
  int z = -1, y = -1;
  for (int m = 0; m < l.order; ++m)
    if (m != mode && (z < 0 || l.dims[m] > l.dims[z])) z = m;
  for (int m = 0; m < l.order; ++m)
    if (m != mode && m != z && (y < 0 || l.dims[m] > l.dims[y])) y = m;
  p.x = mode;
  p.y = y;
  if (!knob.empty() && knob.find(',') != std::string::npos) {
    p.bx = std::atoi(knob.c_str());
    p.by = std::atoi(knob.c_str() + knob.find(',') + 1);
  } else {
    const uint64_t rows = (budget_mb << 20) / (rank * elem_bytes);
    int b = 0;
    while ((uint64_t(2) << (b + 1)) <= rows) ++b;  // 2 * 2^b <= rows
    p.bx = p.by = b;
  }
  if (p.bx <= 0 || p.by <= 0 || p.bx > 31 || p.by > 31 ||
      (l.dims[p.x] <= (uint64_t(1) << p.bx) && l.dims[p.y] <= (uint64_t(1) << p.by)))
    return PanelPlan{};  // one panel: nothing to reorder
  const uint64_t npanels = (((l.dims[p.x] - 1) >> p.bx) + 1) * (((l.dims[p.y] - 1) >> p.by) + 1);
  if (npanels > (uint64_t(1) << 26)) return PanelPlan{};  // widths far too narrow: keep ALTO order
  return p;
}

__global__ void k_tile_panel(const TileDesc* __restrict__ tiles, uint64_t ntiles, const uint64_t* __restrict__ idx,
                             const uint32_t* __restrict__ block_base, int order, int x, int y, uint32_t sx, uint64_t mx,
                             uint32_t sy, uint64_t my, int bx, int by, uint32_t npy, uint32_t* __restrict__ panel) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= ntiles) return;
  const TileDesc td = tiles[i];
  const uint64_t ix = idx[td.start + td.count / 2];
  const uint32_t cx = block_base[uint64_t(td.block) * order + x] | static_cast<uint32_t>((ix >> sx) & mx);
  const uint32_t cy = block_base[uint64_t(td.block) * order + y] | static_cast<uint32_t>((ix >> sy) & my);
  const uint32_t px = cx >> bx;
  uint32_t py = cy >> by;
  if (px & 1u) py = npy - 1 - py;  // boustrophedon
  panel[i] = px * npy + py;
}

// The tile table of t at tile_elems reordered by panel (stable: ALTO order
// inside a panel), or null when the plan is empty.  Cached with the tensor.
const TileDesc* panel_tile_table(const blco_tensor& t, uint32_t tile_elems, int mode, uint64_t rank,
                                 uint64_t* ntiles, uint64_t elem_bytes = sizeof(double)) {
  const PanelPlan pp = panel_plan(t.layout, mode, rank, elem_bytes);
  if (pp.x < 0) return nullptr;
  uint64_t n = 0;
  const TileDesc* base = tile_table(t, tile_elems, &n);
  const uint64_t key = (uint64_t(tile_elems) << 32) | (uint64_t(mode) << 24) | (uint64_t(pp.bx) << 8) | pp.by;
  std::lock_guard<std::mutex> g(t.mu);
  auto it = t.panel_tiles.find(key);
  if (it == t.panel_tiles.end()) {
    const blco_layout& l = t.layout;
    const uint32_t npy = static_cast<uint32_t>(((l.dims[pp.y] - 1) >> pp.by) + 1);
    const uint64_t npx = ((l.dims[pp.x] - 1) >> pp.bx) + 1;
    ScratchScope keep(false);  // cached with the tensor
    DevBuf<uint32_t> d_panel(std::max<uint64_t>(n, 1));
    DevBuf<TileDesc> d(n);
    if (n) {
      k_tile_panel<<<static_cast<unsigned>((n + 255) / 256), 256>>>(
          base, n, t.idx.ptr, t.block_base.ptr, l.order, pp.x, pp.y, static_cast<uint32_t>(l.field_shift[pp.x]),
          l.field_mask[pp.x], static_cast<uint32_t>(l.field_shift[pp.y]), l.field_mask[pp.y], pp.bx, pp.by, npy,
          d_panel.ptr);
      count_launch();
      check_launch("k_tile_panel");
      std::vector<uint32_t> panel(n);
      std::vector<TileDesc> src(n), dst(n);
      B200_CUDA(cudaMemcpy(panel.data(), d_panel.ptr, n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      B200_CUDA(cudaMemcpy(src.data(), base, n * sizeof(TileDesc), cudaMemcpyDeviceToHost));
      std::vector<uint64_t> start(npx * npy + 1, 0);  // stable counting sort by panel
      for (uint64_t i = 0; i < n; ++i) ++start[panel[i] + 1];
      for (size_t k = 1; k < start.size(); ++k) start[k] += start[k - 1];
      for (uint64_t i = 0; i < n; ++i) dst[start[panel[i]]++] = src[i];
      B200_CUDA(cudaMemcpy(d.ptr, dst.data(), n * sizeof(TileDesc), cudaMemcpyHostToDevice));
      B200_CUDA(cudaDeviceSynchronize());  // read by kernels on any stream
    }
    it = t.panel_tiles.emplace(key, std::move(d)).first;
  }
  *ntiles = it->second.n;
  return it->second.ptr;
}

// ---- StageR field widths: the largest per-mode span over the tiles
struct SpanParams {
  uint32_t shift[BLCO_MAX_DEV_ORDER];
  uint64_t mask[BLCO_MAX_DEV_ORDER];
};

__global__ void __launch_bounds__(256) k_tile_spans(const TileDesc* __restrict__ tiles,
                                                    const uint64_t* __restrict__ idx,
                                                    const uint32_t* __restrict__ block_base, int order, SpanParams sp,
                                                    uint32_t* __restrict__ bits_out) {
  __shared__ uint32_t lo[BLCO_MAX_DEV_ORDER], hi[BLCO_MAX_DEV_ORDER];
  const TileDesc td = tiles[blockIdx.x];
  if (threadIdx.x < BLCO_MAX_DEV_ORDER) lo[threadIdx.x] = 0xffffffffu, hi[threadIdx.x] = 0;
  __syncthreads();
  for (int m = 0; m < order; ++m) {
    const uint32_t base = block_base[uint64_t(td.block) * order + m];
    uint32_t mn = 0xffffffffu, mx = 0;
    for (uint32_t i = threadIdx.x; i < td.count; i += blockDim.x) {
      const uint32_t c = base | static_cast<uint32_t>((idx[td.start + i] >> sp.shift[m]) & sp.mask[m]);
      mn = min(mn, c);
      mx = max(mx, c);
    }
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&lo[m], mn);
      atomicMax(&hi[m], mx);
    }
  }
  __syncthreads();
  if (threadIdx.x < order && td.count) {
    const uint32_t span = hi[threadIdx.x] - lo[threadIdx.x];
    atomicMax(&bits_out[threadIdx.x], span ? 32u - __clz(span) : 0u);
  }
}

// Per mode, the bits of the largest coordinate span (max - min) inside one
// tile of tile_elems elements; cached with the tensor.
std::vector<uint32_t> tile_span_bits(const blco_tensor& t, uint32_t tile_elems) {
  uint64_t n = 0;
  const TileDesc* tiles = tile_table(t, tile_elems, &n);
  std::lock_guard<std::mutex> g(t.mu);
  auto it = t.span_bits.find(tile_elems);
  if (it == t.span_bits.end()) {
    const blco_layout& l = t.layout;
    std::vector<uint32_t> bits(l.order, 0);
    if (n) {
      SpanParams sp{};
      for (int m = 0; m < l.order; ++m) sp.shift[m] = static_cast<uint32_t>(l.field_shift[m]), sp.mask[m] = l.field_mask[m];
      ScratchScope keep(false);
      DevBuf<uint32_t> d(BLCO_MAX_DEV_ORDER);
      B200_CUDA(cudaMemset(d.ptr, 0, BLCO_MAX_DEV_ORDER * sizeof(uint32_t)));
      for (uint64_t b0 = 0; b0 < n; b0 += (uint64_t(1) << 30)) {
        const unsigned g = static_cast<unsigned>(std::min<uint64_t>(n - b0, uint64_t(1) << 30));
        k_tile_spans<<<g, 256>>>(tiles + b0, t.idx.ptr, t.block_base.ptr, l.order, sp, d.ptr);
        count_launch();
        check_launch("k_tile_spans");
      }
      B200_CUDA(cudaMemcpy(bits.data(), d.ptr, l.order * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    }
    it = t.span_bits.emplace(tile_elems, std::move(bits)).first;
  }
  return it->second;
}

// BLCO_B200_REL_STAGE=1 (read per call) enables the StageR record.  Opt-in:
// measured slower on B200 in interleaved A/B runs (scripts/panel_probe.py
// with the knob; Amazon 374-376 vs 357-368 ms per all-mode step, Delicious
// 22.3-23.3 vs 20.0-21.9 ms): the LDS wavefronts it saves (~0.3-0.7 per
// element) cost more in the per-element unpacking, the tile-minimum
// reduction and the register cap (80 / 64) than they return.
bool rel_stage_knob() {
  const char* e = std::getenv("BLCO_B200_REL_STAGE");
  return e && std::string(e) == "1";
}

// StageR field layout of a launch: slot k = the k-th non-target mode
// (p.others), the row last; false when the spans need more than 64 bits.
template <int N>
bool rel_stage_plan(const blco_tensor* t, uint32_t tile_elems, Params<N>& p) {
  if (!t || !rel_stage_knob()) return false;
  const std::vector<uint32_t> bits = tile_span_bits(*t, tile_elems);
  uint32_t off = 0;
  for (int k = 0; k < N; ++k) {
    const uint32_t b = bits[k < N - 1 ? p.others[k] : p.mode];
    p.pk_off[k] = std::min<uint32_t>(off, 63);  // a 0-bit slot reads 0 through its mask
    p.pk_mask[k] = b >= 32 ? 0xffffffffu : ((1u << b) - 1u);
    off += b;
  }
  return off <= 64;
}

template <class K>
void set_smem(K kern, size_t dyn) {
  ensure_dyn_smem(reinterpret_cast<const void*>(kern), dyn);
}

// BLCO_B200_L2WINDOW=f (0 < f <= 1; off by default): the launch gives the
// smallest gathered factor matrix an L2 access-policy window -- persisting
// hits, streaming misses, hit ratio = f * (max persisting L2) / window.  The
// probe of SURVEY 7's "L2 residency control" lever for DRAM-bound shapes
// (Amazon); measured in DESIGN.md 3.
double l2_window_knob() {
  static const double f = [] {
    const char* e = std::getenv("BLCO_B200_L2WINDOW");
    return e ? std::atof(e) : 0.0;
  }();
  return f;
}

template <int N, class K>
void launch_tiles(K kern, dim3 grid, size_t smem, const Params<N>& p, const MttkrpLaunch& a) {
  const double f = l2_window_knob();
  if (f <= 0.0 || N < 2) {
    kern<<<grid, kCtaThreads, smem, a.stream>>>(p);
    return;
  }
  const blco_layout& l = *a.view.layout;
  int best = -1;
  uint64_t bytes = ~0ull;
  for (int m = 0; m < N; ++m)
    if (m != a.mode && l.dims[m] * a.rank * 8 < bytes) bytes = l.dims[m] * a.rank * 8, best = m;
  int dev = 0, max_persist = 0, max_window = 0;
  B200_CUDA(cudaGetDevice(&dev));
  B200_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  B200_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  const size_t persist = static_cast<size_t>(std::min(1.0, f) * max_persist);
  static std::mutex mu;
  static std::map<int, size_t> limit_set;
  {
    std::lock_guard<std::mutex> g(mu);
    if (limit_set[dev] != persist) {
      B200_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist));
      limit_set[dev] = persist;
    }
  }
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeAccessPolicyWindow;
  auto& w = attr.val.accessPolicyWindow;
  w.base_ptr = const_cast<double*>(a.factors[best]);
  w.num_bytes = std::min<size_t>(bytes, static_cast<size_t>(max_window));
  w.hitRatio = w.num_bytes ? static_cast<float>(std::min(1.0, double(persist) / double(w.num_bytes))) : 0.0f;
  w.hitProp = cudaAccessPropertyPersisting;
  w.missProp = cudaAccessPropertyStreaming;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kCtaThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.stream;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  B200_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
}

template <int N, int LPE, int CPL, bool FULL>
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
  const size_t tile_stage = stage_bytes<N>(kTileElems);

  if (a.strategy != BLCO_STRATEGY_HIERARCHICAL) {
    p.out = a.out;
    p.ncopies = 1;
    a.workgroups = p.ntiles;
    const dim3 grid(static_cast<unsigned>(p.ntiles), ychunks);
    if (use_warp_variant()) {
      const size_t dyn = stage_bytes<N>(kWarpElems) * kWarps;
      auto kern = stats ? k_mttkrp_warp<N, LPE, CPL, FULL, true> : k_mttkrp_warp<N, LPE, CPL, FULL, false>;
      set_smem(kern, dyn);
      kern<<<grid, kCtaThreads, dyn, a.stream>>>(p);
      count_launch();
      check_launch("k_mttkrp_warp");
      return;
    }
    if constexpr (N <= 3 && FULL) {
      if (a.tensor && ychunks == 1 && use_big_tiles(l, a.mode, a.rank, a.tensor->nnz)) {
        // 2048-element tiles (see k_mttkrp_sorted)
        constexpr int T2 = 2 * kTileElems;
        p.tiles = tile_table(*a.tensor, T2, &p.ntiles);
        uint64_t nt = 0;
        if (const TileDesc* pt = panel_tile_table(*a.tensor, T2, a.mode, a.rank, &nt)) p.tiles = pt;
        a.workgroups = p.ntiles;
        auto kern = stats ? k_mttkrp_sorted<N, LPE, CPL, FULL, true, kUnroll, 1, T2>
                          : k_mttkrp_sorted<N, LPE, CPL, FULL, false, kUnroll, 3, T2>;  // <= 80 regs: 3 CTAs/SM (91 -> 2)
        size_t st2 = stage_bytes<N>(T2);
        if constexpr (N == 3) {
          bool narrow = compact_stage_knob();
          for (int m = 0; m < N; ++m)
            if (m != a.mode && l.dims[m] > 65536) narrow = false;
          if (narrow) {  // 16-byte records with the row inside (StageC)
            kern = stats ? k_mttkrp_sorted<N, LPE, CPL, FULL, true, kUnroll, 1, T2, 1>
                         : k_mttkrp_sorted<N, LPE, CPL, FULL, false, kUnroll, 3, T2, 1>;
            st2 = static_cast<size_t>(T2) * sizeof(uint4);
          }
        }
        set_smem(kern, st2);
        kern<<<dim3(static_cast<unsigned>(p.ntiles), 1), kCtaThreads, st2, a.stream>>>(p);
        count_launch();
        check_launch("k_mttkrp_sorted");
        return;
      }
    }
    if constexpr (N >= 3) {
      if (a.tensor) {  // factors beyond L2: panel-ordered dispatch (panel_plan)
        uint64_t nt = 0;
        if (const TileDesc* pt = panel_tile_table(*a.tensor, kTileElems, a.mode, a.rank, &nt)) p.tiles = pt;
      }
    }
    size_t stage1 = tile_stage;
    auto kern = stats ? k_mttkrp_sorted<N, LPE, CPL, FULL, true> : k_mttkrp_sorted<N, LPE, CPL, FULL, false>;
    // N = 3 with wide non-target modes (Amazon) and N = 4 (Delicious): the
    // 16-byte tile-relative record (StageR) when every tile's spans fit
    bool rel = false;
    if constexpr ((N == 3 || N == 4) && FULL && LPE * CPL <= 32) {
      bool narrow = N == 3 && compact_stage_knob();
      for (int m = 0; m < N; ++m)
        if (m != a.mode && l.dims[m] > 65536) narrow = false;
      if (!narrow && !use_warp_variant() && rel_stage_plan<N>(a.tensor, kTileElems, p)) {
        rel = true;
        // <= 80 registers for N = 3 (3 CTAs/SM); <= 64 for N = 4 (4 CTAs/SM, as
        // the Stage<4> kernel reaches uncapped)
        kern = stats ? k_mttkrp_sorted<N, LPE, CPL, FULL, true, kUnroll, 1, kTileElems, 2>
                     : k_mttkrp_sorted<N, LPE, CPL, FULL, false, kUnroll, N == 4 && CPL == 1 ? 4 : 3, kTileElems, 2>;
        stage1 = static_cast<size_t>(kTileElems) * sizeof(uint4);
      }
    }
    if constexpr (N == 3 && FULL) {
      bool narrow = compact_stage_knob();
      for (int m = 0; m < N; ++m)
        if (m != a.mode && l.dims[m] > 65536) narrow = false;
      if (narrow) {  // 16-byte records with the row inside (StageC)
        kern = stats ? k_mttkrp_sorted<N, LPE, CPL, FULL, true, kUnroll, 1, kTileElems, 1>
                     : k_mttkrp_sorted<N, LPE, CPL, FULL, false, kUnroll, 1, kTileElems, 1>;
        stage1 = static_cast<size_t>(kTileElems) * sizeof(uint4);
      }
    }
    // N = 4 (R <= 32): cap registers so 3 CTAs fit per SM (88 -> 80 for
    // R=16; the DRAM-bound Delicious modes run 6% faster with the extra warps
    // in flight).  N <= 3 already fits 3; higher orders would spill.
    if constexpr (N == 4 && LPE * CPL <= 32)
      if (!stats && !rel) kern = k_mttkrp_sorted<N, LPE, CPL, FULL, false, kUnroll, 3>;
    set_smem(kern, stage1);
    launch_tiles<N>(kern, grid, stage1, p, a);
    count_launch();
    check_launch("k_mttkrp_sorted");
    return;
  }

  // Hierarchical: stash as large as shared memory allows, at least
  // cfg.stash_slots, no larger than the mode (then it privatises the mode).
  int dev = 0, smem_optin = 0, nsm = 0;
  B200_CUDA(cudaGetDevice(&dev));
  B200_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  B200_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if constexpr (FULL && Stage<N>::kPacked) {
    // privatised form (k_mttkrp_priv) when M_n fits beside the staging and
    // one copy is asked for; ~half the shared memory at most, so at least
    // two CTAs stay resident per SM
    const size_t privb = elems * sizeof(double);
    const int C1 = std::max(1, a.cfg.num_factor_copies);
    if (C1 == 1 && !stats && !a.hier_copies && ychunks == 1 && l.dims[a.mode] <= uint64_t(kBuckets) &&
        tile_stage + privb + sizeof(BucketShared) + 1024 <= static_cast<size_t>(smem_optin) / 2) {
      const size_t dyn = tile_stage + privb;
      auto kern = k_mttkrp_priv<N, LPE, CPL>;
      set_smem(kern, dyn);
      const int per_sm = std::max(blocks_per_sm(reinterpret_cast<const void*>(kern), kCtaThreads, dyn), 1);
      const uint64_t grid = std::min<uint64_t>(p.ntiles, static_cast<uint64_t>(nsm) * per_sm);
      p.out = a.out;
      p.ncopies = 1;
      a.workgroups = grid;
      a.stash_slots = static_cast<int>(l.dims[a.mode]);
      kern<<<dim3(static_cast<unsigned>(grid), 1), kCtaThreads, dyn, a.stream>>>(p);
      count_launch();
      check_launch("k_mttkrp_priv");
      return;
    }
  }
  const size_t budget = static_cast<size_t>(smem_optin) - sizeof(BucketShared) - tile_stage - 1024;
  const size_t per_slot = a.rank * sizeof(double) + sizeof(uint32_t);
  const uint64_t fit = budget / per_slot;
  if (fit < 1)
    throw_format("b200: rank " + std::to_string(a.rank) + " too large for the shared-memory stash");
  uint64_t slots = std::min<uint64_t>(l.dims[a.mode], fit);
  slots = std::max<uint64_t>(slots, std::min<uint64_t>(static_cast<uint64_t>(a.cfg.stash_slots), fit));
  p.stash_slots = static_cast<int>(slots);
  a.stash_slots = p.stash_slots;
  const size_t dyn = tile_stage + slots * per_slot + 16;
  auto kern = stats ? k_mttkrp_hier<N, LPE, CPL, FULL, true> : k_mttkrp_hier<N, LPE, CPL, FULL, false>;
  set_smem(kern, dyn);
  const int per_sm = std::max(blocks_per_sm(reinterpret_cast<const void*>(kern), kCtaThreads, dyn), 1);
  const uint64_t grid = std::min<uint64_t>(p.ntiles, static_cast<uint64_t>(nsm) * per_sm);
  a.workgroups = grid;
  const int C = std::max(1, a.cfg.num_factor_copies);
  p.ncopies = C;
  bool merge = false;
  if (a.hier_copies) {
    p.out = a.hier_copies;  // caller merges once at the end
  } else if (C == 1) {
    p.out = a.out;  // flushes add into M (zeroed above unless accumulating)
  } else {
    DevBuf<double>& cb = workspace().copies[a.stream];
    if (cb.n < elems * C) cb.alloc(elems * C);
    B200_CUDA(cudaMemsetAsync(cb.ptr, 0, elems * C * sizeof(double), a.stream));
    p.out = cb.ptr;
    merge = true;
  }
  kern<<<dim3(static_cast<unsigned>(grid), ychunks), kCtaThreads, dyn, a.stream>>>(p);
  count_launch();
  check_launch("k_mttkrp_hier");
  if (merge) merge_copies_enqueue(p.out, elems, C, a.out, a.accumulate, a.stream);
}

// ---- the all-mode fused kernel (k_mttkrp_all3): eligibility and launch
// Opt-in (BLCO_B200_FUSED=1, read per call): measured slower than the three
// per-mode launches on every eligible shape (B200, interleaved A/B,
// scripts/fused_ab.py: NELL-2 R=32 8.78 vs 7.28 ms, R=16 4.92 vs 4.74 ms,
// config 1 0.112 vs 0.091 ms).  Halving the gathers moves the bound to L2:
// the two ungrouped modes commit one RED per element (~1.9 per element vs
// 3 x 0.32 for the grouped per-mode kernels), and fp64 REDs are served at a
// lower L2 rate than loads (ncu: lts 89%, L1 82%).
bool fused_knob() {
  const char* e = std::getenv("BLCO_B200_FUSED");
  return e && std::string(e) == "1";
}

// Order 3, R = 16 / 32, not deterministic, and the three factors plus the
// three outputs within 64 MB, so the whole gathered / committed working set
// stays in the 126 MB L2: the regime where the per-mode kernels are bound by
// the L1 data pipe.  Larger factors (Amazon) keep the per-mode kernels: there
// the working set of one window of concurrent tiles would double and fall
// out of L2.
bool fused_eligible(const blco_tensor& t, uint64_t rank, const blco_exec_config& c) {
  if (!fused_knob() || t.layout.order != 3 || (rank != 16 && rank != 32) || c.deterministic) return false;
  uint64_t bytes = 0;
  for (int m = 0; m < 3; ++m) bytes += 2 * t.layout.dims[m] * rank * sizeof(double);
  return bytes <= (uint64_t(64) << 20) && t.nnz > 0;
}

// BLCO_B200_FUSED_CFG: register / latency trade of the fused kernel --
// "u4m2": 4 elements gathered ahead per lane group, up to 128 registers
// (2 CTAs per SM); "u2m3" (default): 2 elements ahead, <= 80 registers
// (3 CTAs per SM).
bool fused_u4() {
  static const bool v = [] {
    const char* e = std::getenv("BLCO_B200_FUSED_CFG");
    return e && std::string(e) == "u4m2";
  }();
  return v;
}

template <int GM, int LPE, int CPL>
void launch_all3_gm(const Params<3>& p, const FusedOut& fo, bool narrow, cudaStream_t s) {
  constexpr int T2 = 2 * kTileElems;
  auto kern = narrow ? k_mttkrp_all3<GM, LPE, CPL, T2, true, 3, 2> : k_mttkrp_all3<GM, LPE, CPL, T2, false, 3, 2>;
  if (fused_u4())
    kern = narrow ? k_mttkrp_all3<GM, LPE, CPL, T2, true, 2, 4> : k_mttkrp_all3<GM, LPE, CPL, T2, false, 2, 4>;
  const size_t dyn = narrow ? static_cast<size_t>(T2) * sizeof(uint4) : stage_bytes<3>(T2);
  set_smem(kern, dyn);
  kern<<<dim3(static_cast<unsigned>(p.ntiles), 1), kCtaThreads, dyn, s>>>(p, fo);
  count_launch();
  check_launch("k_mttkrp_all3");
}

template <int LPE, int CPL>
void launch_all3(const blco_tensor& t, const double* const* f, uint64_t rank, double* const* outs,
                 cudaStream_t s) {
  const blco_layout& l = t.layout;
  Params<3> p{};
  p.tiles = tile_table(t, 2 * kTileElems, &p.ntiles);
  p.elem_end = t.nnz;
  p.idx = t.idx.ptr;
  p.val = t.vals.ptr;
  p.block_base = t.block_base.ptr;
  for (int m = 0; m < 3; ++m) {
    p.shift[m] = static_cast<uint32_t>(l.field_shift[m]);
    p.mask[m] = l.field_mask[m];
  }
  // group the tile by the shortest mode: the most elements per distinct row,
  // so the most commits saved by run accumulation
  int gm = 0;
  for (int m = 1; m < 3; ++m)
    if (l.dims[m] < l.dims[gm]) gm = m;
  p.mode = gm;
  p.rank = static_cast<int>(rank);
  FusedOut fo{};
  for (int m = 0; m < 3; ++m) fo.f[m] = f[m], fo.out[m] = outs[m];
  bool narrow = compact_stage_knob();
  for (int m = 0; m < 3; ++m)
    if (m != gm && l.dims[m] > 65536) narrow = false;
  if (p.ntiles == 0) return;
  if (gm == 0) launch_all3_gm<0, LPE, CPL>(p, fo, narrow, s);
  else if (gm == 1) launch_all3_gm<1, LPE, CPL>(p, fo, narrow, s);
  else launch_all3_gm<2, LPE, CPL>(p, fo, narrow, s);
}

template <int N>
void launch_order(MttkrpLaunch& a) {
  switch (a.rank) {
    case 8: return launch_cfg<N, 8, 1, true>(a);
    case 16: return launch_cfg<N, 16, 1, true>(a);  // 16 lanes x 1 column: a 128 B row per group (CP-ALS R=16 -10%)
    case 32: return launch_cfg<N, 16, 2, true>(a);
    case 64: return launch_cfg<N, 32, 2, true>(a);
    default: return launch_cfg<N, 32, 1, false>(a);
  }
}

template <int N, int LPE, int V, int CPL, bool FULL>
void launch_f32_cfg(const KernelView& v, const float* const* factors, uint64_t rank, int mode, float* out,
                    cudaStream_t s) {
  const blco_layout& l = *v.layout;
  ParamsF32<N> p{};
  p.base.tiles = v.tiles;
  p.base.ntiles = v.ntiles;
  p.base.elem_end = v.elem_end;
  p.base.idx = v.idx;
  p.base.val = v.vals;
  p.base.block_base = v.block_base;
  for (int m = 0, k = 0; m < N; ++m) {
    if (m != mode) p.factors[k++] = factors[m];
    p.base.shift[m] = static_cast<uint32_t>(l.field_shift[m]);
    p.base.mask[m] = l.field_mask[m];
  }
  p.base.mode = mode;
  p.base.rank = static_cast<int>(rank);
  p.out = out;
  if (v.ntiles == 0) return;
  const unsigned ychunks = static_cast<unsigned>((rank + LPE * V * CPL - 1) / (LPE * V * CPL));
  if constexpr (N <= 3 && FULL) {
    if (v.tensor && ychunks == 1 && use_big_tiles(l, mode, rank, v.tensor->nnz, sizeof(float))) {
      constexpr int T2 = 2 * kTileElems;  // as the fp64 kernel (k_mttkrp_sorted)
      p.base.tiles = tile_table(*v.tensor, T2, &p.base.ntiles);
      size_t st2 = stage_bytes<N>(T2);
      auto kern = k_mttkrp_sorted_f32<N, LPE, V, CPL, FULL, T2, 3>;
      if constexpr (N == 3 && CPL == 1) {
        bool narrow = compact_stage_knob();
        for (int m = 0; m < N; ++m)
          if (m != mode && l.dims[m] > 65536) narrow = false;
        if (narrow) {  // 16-byte records with the row inside (StageC)
          kern = k_mttkrp_sorted_f32<N, LPE, V, CPL, FULL, T2, 3, true>;
          st2 = static_cast<size_t>(T2) * sizeof(uint4);
        }
      }
      set_smem(kern, st2);
      kern<<<dim3(static_cast<unsigned>(p.base.ntiles), 1), kCtaThreads, st2, s>>>(p);
      count_launch();
      check_launch("k_mttkrp_sorted_f32");
      return;
    }
  }
  if constexpr (N >= 3) {
    if (v.tensor) {  // factors beyond L2: panel-ordered dispatch (panel_plan)
      uint64_t nt = 0;
      if (const TileDesc* pt = panel_tile_table(*v.tensor, kTileElems, mode, rank, &nt, sizeof(float)))
        p.base.tiles = pt;
    }
  }
  const size_t stage = stage_bytes<N>(kTileElems);
  auto kern = k_mttkrp_sorted_f32<N, LPE, V, CPL, FULL>;
  set_smem(kern, stage);
  kern<<<dim3(static_cast<unsigned>(v.ntiles), ychunks), kCtaThreads, stage, s>>>(p);
  count_launch();
  check_launch("k_mttkrp_sorted_f32");
}

template <int N>
void launch_f32_order(const KernelView& v, const float* const* f, uint64_t rank, int mode, float* out,
                      cudaStream_t s) {
  switch (rank) {
    case 8: return launch_f32_cfg<N, 4, 2, 1, true>(v, f, rank, mode, out, s);
    case 16: return launch_f32_cfg<N, 8, 2, 1, true>(v, f, rank, mode, out, s);
    case 32: return launch_f32_cfg<N, 16, 2, 1, true>(v, f, rank, mode, out, s);
    case 64: return launch_f32_cfg<N, 32, 2, 1, true>(v, f, rank, mode, out, s);
    default: return launch_f32_cfg<N, 32, 1, 1, false>(v, f, rank, mode, out, s);
  }
}

void mttkrp_f32_enqueue(const KernelView& v, const float* const* f, uint64_t rank, int mode, float* out,
                        cudaStream_t s) {
  switch (v.layout->order) {
    case 1: return launch_f32_order<1>(v, f, rank, mode, out, s);
    case 2: return launch_f32_order<2>(v, f, rank, mode, out, s);
    case 3: return launch_f32_order<3>(v, f, rank, mode, out, s);
    case 4: return launch_f32_order<4>(v, f, rank, mode, out, s);
    case 5: return launch_f32_order<5>(v, f, rank, mode, out, s);
    case 6: return launch_f32_order<6>(v, f, rank, mode, out, s);
    case 7: return launch_f32_order<7>(v, f, rank, mode, out, s);
    case 8: return launch_f32_order<8>(v, f, rank, mode, out, s);
    default: throw_format("b200: order above the device limit");
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
  int label = a.strategy;  // what MttkrpStats::strategy reports (the reference's choice under Auto)
  if (a.strategy == BLCO_STRATEGY_AUTO) {
    label = blco_choose_strategy(a.view.layout->dims[a.mode], &a.cfg);
    a.strategy = auto_kernel(a.view.layout->dims[a.mode], a.cfg);
  }
  Workspace& ws = workspace();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (stats) {
    if (ws.counters.n < 5) ws.counters.alloc(5);
    B200_CUDA(cudaMemsetAsync(ws.counters.ptr, 0, 5 * sizeof(unsigned long long), a.stream));
    a.counters = ws.counters.ptr;
    B200_CUDA(cudaEventCreate(&e0));
    B200_CUDA(cudaEventCreate(&e1));
    B200_CUDA(cudaEventRecord(e0, a.stream));
  }
  mttkrp_enqueue(a);
  if (!stats) return;
  B200_CUDA(cudaEventRecord(e1, a.stream));
  unsigned long long h[5] = {0, 0, 0, 0, 0};
  B200_CUDA(cudaMemcpyAsync(h, ws.counters.ptr, sizeof h, cudaMemcpyDeviceToHost, a.stream));
  B200_CUDA(cudaStreamSynchronize(a.stream));
  float ms = 0;
  B200_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  stats->strategy = label;
  stats->kernel = a.strategy;
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
  stats->processing_cycles = h[3];
  stats->computing_cycles = h[4];
}

}  // namespace

void mttkrp_enqueue(MttkrpLaunch& a) {
  static const char* const names[8] = {"mttkrp mode 0", "mttkrp mode 1", "mttkrp mode 2", "mttkrp mode 3",
                                        "mttkrp mode 4", "mttkrp mode 5", "mttkrp mode 6", "mttkrp mode 7"};
  NvtxRange nv(a.mode >= 0 && a.mode < 8 ? names[a.mode] : "mttkrp");
  if (a.rank < 1) throw_format("factors: rank must be >= 1");
  if (a.cfg.deterministic) {
    // fixed summation order (determ.cu); needs the device tensor's cache
    if (!a.tensor)
      throw_format("b200: deterministic mode needs a device-resident tensor (not the streamed paths)");
    det_mttkrp_enqueue(*a.tensor, a);
    return;
  }
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

int blco_panel_plan(const blco_layout* layout, int mode, uint64_t rank, uint64_t elem_bytes, int* y_mode, int* bx,
                    int* by) {
  return guarded([&] {
    if (!layout || !y_mode || !bx || !by) throw_format("panel_plan: null argument");
    if (mode < 0 || mode >= layout->order) throw_format("mttkrp: mode out of range");
    if (elem_bytes != 4 && elem_bytes != 8) throw_format("panel_plan: elem_bytes must be 4 or 8");
    const PanelPlan p = panel_plan(*layout, mode, rank, elem_bytes);
    *y_mode = p.x < 0 ? -1 : p.y;
    *bx = p.bx;
    *by = p.by;
  });
}

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
    a.tensor = t;
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

int blco_mttkrp_all_device(const blco_tensor* t, const double* const* d_factors, uint64_t rank, int strategy,
                           const blco_exec_config* cfg, double* const* d_outs, int accumulate, void* stream,
                           int* fused) {
  return guarded([&] {
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    for (int m = 0; m < t->layout.order; ++m) validate_call(t, rank, m, &c);
    DeviceGuard dg(t->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool use = strategy != BLCO_STRATEGY_HIERARCHICAL && fused_eligible(*t, rank, c);
    if (fused) *fused = use ? 1 : 0;
    if (use) {
      NvtxRange nv("mttkrp all modes (fused)");
      if (!accumulate)
        for (int m = 0; m < 3; ++m)
          B200_CUDA(cudaMemsetAsync(d_outs[m], 0, t->layout.dims[m] * rank * sizeof(double), s));
      if (rank == 32) launch_all3<16, 2>(*t, d_factors, rank, d_outs, s);
      else launch_all3<16, 1>(*t, d_factors, rank, d_outs, s);
      return;
    }
    for (int m = 0; m < t->layout.order; ++m) {
      MttkrpLaunch a{};
      a.view = view_of(*t);
      a.tensor = t;
      a.factors = d_factors;
      a.rank = rank;
      a.mode = m;
      a.strategy = strategy;
      a.cfg = c;
      a.out = d_outs[m];
      a.accumulate = accumulate;
      a.stream = s;
      run(a, nullptr);
    }
  });
}

int blco_mttkrp_device_f32(const blco_tensor* t, const float* const* d_factors, uint64_t rank, int mode,
                           const blco_exec_config* cfg, float* d_out, int accumulate, void* stream) {
  return guarded([&] {
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    validate_call(t, rank, mode, &c);
    if (c.deterministic) throw_format("b200: the fp32 variant has no deterministic mode");
    DeviceGuard dg(t->device);
    NvtxRange nv("mttkrp fp32");
    const KernelView v = view_of(*t);
    const uint64_t elems = t->layout.dims[mode] * rank;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!accumulate && elems) B200_CUDA(cudaMemsetAsync(d_out, 0, elems * sizeof(float), s));
    mttkrp_f32_enqueue(v, d_factors, rank, mode, d_out, s);
  });
}

int blco_mttkrp_f32(const blco_tensor* t, const float* const* factors, uint64_t rank, int mode,
                    const blco_exec_config* cfg, float* out) {
  return guarded([&] {
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    validate_call(t, rank, mode, &c);
    if (c.deterministic) throw_format("b200: the fp32 variant has no deterministic mode");
    DeviceGuard dg(t->device);
    const blco_layout& l = t->layout;
    std::vector<DevBuf<float>> df(l.order);
    std::vector<const float*> ptrs(l.order);
    for (int m = 0; m < l.order; ++m) {
      df[m].alloc(l.dims[m] * rank);
      if (df[m].n) B200_CUDA(cudaMemcpy(df[m].ptr, factors[m], df[m].bytes(), cudaMemcpyHostToDevice));
      ptrs[m] = df[m].ptr;
    }
    const uint64_t elems = l.dims[mode] * rank;
    DevBuf<float> dout(elems);
    if (elems) B200_CUDA(cudaMemset(dout.ptr, 0, dout.bytes()));
    mttkrp_f32_enqueue(view_of(*t), ptrs.data(), rank, mode, dout.ptr, nullptr);
    if (elems) B200_CUDA(cudaMemcpy(out, dout.ptr, dout.bytes(), cudaMemcpyDeviceToHost));
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
      if (l.dims[m] * rank != 0)
        B200_CUDA(cudaMemcpy(df[m].ptr, factors[m], l.dims[m] * rank * 8, cudaMemcpyHostToDevice));
      ptrs[m] = df[m].ptr;
    }
    const uint64_t elems = l.dims[mode] * rank;
    DevBuf<double> dout(elems);
    MttkrpLaunch a{};
    a.view = view_of(*t);
    a.tensor = t;
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
