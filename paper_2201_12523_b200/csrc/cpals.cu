// cpals.cu -- CP-ALS driver with factors resident in HBM (config 4).
//
// Reference: cp_als / fit, proj/src/cpals.cpp:66-129; dense kernels
// proj/src/dense_kernels.cpp:8-92.  Per iteration and mode n (Alg. 1):
//   V = hadamard_{m != n} Gram(A_m)            (R x R, host)
//   M = MTTKRP(X, n)                           (device, mttkrp.cu)
//   A_n = M V^-1 via Cholesky of V, Tikhonov escalation on failure
//                                              (factorisation on host, the
//                                               I_n row solves on device,
//                                               fused with Gram(A_n))
//   lambda = sqrt(diag Gram), A_n /= lambda     (device; folded into the
//                                               next solves, Dense::solve_fold,
//                                               and applied once at the end)
// then fit = 1 - sqrt(max(0, |X|^2 - 2<X,Xhat> + |Xhat|^2)) / |X|.
// Summation orders differ from the sequential host loops, so parity is
// tolerance-based.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "internal.hpp"

namespace b200 {
namespace {

constexpr int kT = 256;

// Fused epilogue pass 1 (solve_normal + the Gram of the solution,
// dense_kernels.cpp:68-92 and :8-21): A = M V^-1 row by row with V = L L^T,
// and G += A^T A (upper triangle) on the same staged rows.  A CTA stages ROWS
// rows of M through shared memory with coalesced loads (row stride R+1
// doubles, so a thread's own row is conflict-free), solves one row per
// thread in registers, stores the rows to A coalesced, and accumulates the
// R(R+1)/2 pair sums of the chunk in registers (one pair set per thread),
// flushed with one atomic per pair at the end.  diag(G) is the column
// sum-of-squares normalize_columns needs (cpals.cpp:51-61), so the
// separate norm pass disappears and Gram(A / lambda) = G_ij / (l_i l_j).
constexpr int kSolveThreads = 128;
// cp.async ring depth of k_solve_gram (chunks in flight per CTA)
#ifndef BLCO_SOLVE_STAGES
#define BLCO_SOLVE_STAGES 2
#endif
#ifndef BLCO_SOLVE_MINB
#define BLCO_SOLVE_MINB 1
#endif
constexpr int kSolveStages = BLCO_SOLVE_STAGES;

template <int RM>
constexpr int solve_rows() {
  return 4096 / RM < kSolveThreads ? 4096 / RM : kSolveThreads;
}

// L (R x R lower, the diagonal replaced by 1 / L_ii) in constant memory,
// copied device-to-device from the Cholesky kernel's output: with R == RM
// every L_ik index is a compile-time constant and the solve's DFMAs read it
// straight from the constant bank (no shared-memory traffic).  One ALS runs
// per device at a time (cp_als is synchronous on the legacy stream).
__constant__ double c_L[32 * 32];
// Column scaling of M applied as the rows are loaded (cp_als with folded
// normalisation: M comes from the unnormalised factors, s = 1 / prod lambda)
__constant__ double c_S[32];

template <int RM, bool EXACT>
__device__ __forceinline__ double lget(const double* sl, int R, int i, int k) {
  if constexpr (EXACT) return c_L[i * RM + k];
  else return sl[i * R + k];
}

// RM = 16: capped at 168 registers so three CTAs fit per SM (shared memory
// allows three); uncapped, ptxas takes 254 and two fit (ncu on the 17.3M-row
// Delicious mode: 12.5% occupancy, issue-latency bound on the DFMA chains).
#ifndef BLCO_SOLVE16_MINB
#define BLCO_SOLVE16_MINB 3
#endif
template <int RM>
constexpr int solve_min_blocks() {
  return RM == 16 ? BLCO_SOLVE16_MINB : BLCO_SOLVE_MINB;
}

template <int RM, bool EXACT>
__global__ void __launch_bounds__(kSolveThreads, solve_min_blocks<RM>()) k_solve_gram(const double* __restrict__ m, double* __restrict__ a,
                                                              uint64_t rows, int R, const double* __restrict__ L,
                                                              const double* __restrict__ S, double* __restrict__ g) {
  constexpr int ROWS = solve_rows<RM>();
  constexpr int W = kSolveThreads / 32;
  // Gram lane blocking: lane owns AI rows x AJ columns of a GI x GJ block of G
  // (the whole R x R for RM <= 32, with the warps splitting the staged rows;
  // one 32 x 32 quadrant per warp for RM = 64, every warp on every row).
  constexpr int AI = RM <= 32 ? RM / 8 : 4, AJ = RM <= 32 ? RM / 4 : 8;
  constexpr bool QUAD = RM > 32;
  extern __shared__ double smem[];
  double* sl = smem;                      // R x R (generic R only)
  __shared__ double ss[64];               // column scaling of M (generic R; ones when S is null)
  // two ROWS x (R + 1) tiles (double-buffered); RR = R as a compile-time
  // constant when R == RM, so row/column splits are shifts
  const int RR = EXACT ? RM : R;
  const int SR = RR + 1;  // padded row stride
  if constexpr (!EXACT) {
    for (int i = threadIdx.x; i < R * R; i += blockDim.x) sl[i] = L[i];
    for (int i = threadIdx.x; i < R; i += blockDim.x) ss[i] = S ? S[i] : 1.0;  // x * 1.0 is exact
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int qi = QUAD ? (warp >> 1) * 32 : 0, qj = QUAD ? (warp & 1) * 32 : 0;
  const int i0 = qi + (lane >> 2) * AI, j0 = qj + (lane & 3) * AJ;
  double gacc[AI][AJ];
#pragma unroll
  for (int x = 0; x < AI; ++x)
#pragma unroll
    for (int y = 0; y < AJ; ++y) gacc[x][y] = 0.0;

  // cp.async prefetch of the CTA's next chunk into the other buffer while
  // this chunk is solved (8-byte copies: the padded row stride is odd)
  const uint64_t step = uint64_t(gridDim.x) * ROWS;
  auto prefetch = [&](uint64_t base, double* dst) {
    if (base < rows) {
      const int n = static_cast<int>((rows - base < uint64_t(ROWS) ? rows - base : ROWS) * R);
      constexpr int PER = ROWS * RM / kSolveThreads;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int k = threadIdx.x + j * kSolveThreads;
        if (k < n) {
          const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + (k / RR) * SR + k % RR));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(m + base * R + k) : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // ring of kSolveStages chunk buffers: chunks k+1 .. k+S-1 stream in while
  // chunk k is solved
  constexpr int S_ = kSolveStages, TS = ROWS * (RM + 1);
  double* const tile0 = smem + RM * RM;
#pragma unroll
  for (int k = 0; k + 1 < S_; ++k) prefetch(blockIdx.x * uint64_t(ROWS) + k * step, tile0 + k * TS);
  int buf = 0;
  for (uint64_t r0 = blockIdx.x * uint64_t(ROWS); r0 < rows; r0 += step, buf = buf + 1 == S_ ? 0 : buf + 1) {
    const int nr = static_cast<int>(rows - r0 < uint64_t(ROWS) ? rows - r0 : ROWS);
    double* tile = tile0 + buf * TS;
    __syncthreads();  // every thread is done with the buffer of the previous chunk
    const int nb = buf + S_ - 1 >= S_ ? buf - 1 : buf + S_ - 1;  // (buf + S - 1) % S
    prefetch(r0 + (S_ - 1) * step, tile0 + nb * TS);
    asm volatile("cp.async.wait_group %0;" ::"n"(S_ - 1) : "memory");
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < nr) {
      double b[RM];
      double* row = tile + threadIdx.x * SR;
#pragma unroll
      for (int i = 0; i < RM; ++i)
        if (i < RR) {
          if constexpr (EXACT) b[i] = row[i] * c_S[i];  // ones unless the normalisation is folded
          else b[i] = row[i] * ss[i];
        }
#pragma unroll
      for (int i = 0; i < RM; ++i) {
        if (i < RR) {
          double x = b[i];
#pragma unroll
          for (int k = 0; k < i; ++k) x -= lget<RM, EXACT>(sl, R, i, k) * b[k];
          b[i] = x * lget<RM, EXACT>(sl, R, i, i);
        }
      }
#pragma unroll
      for (int ii = RM - 1; ii >= 0; --ii) {
        if (ii < RR) {
          double x = b[ii];
#pragma unroll
          for (int k = ii + 1; k < RM; ++k)
            if (k < RR) x -= lget<RM, EXACT>(sl, R, k, ii) * b[k];
          b[ii] = x * lget<RM, EXACT>(sl, R, ii, ii);
        }
      }
#pragma unroll
      for (int i = 0; i < RM; ++i)
        if (i < RR) row[i] = b[i];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nr * RR; k += blockDim.x) a[r0 * RR + k] = tile[(k / RR) * SR + k % RR];
    for (int r = QUAD ? 0 : warp; r < nr; r += QUAD ? 1 : W) {
      const double* t = tile + r * SR;
      double xi[AI], yj[AJ];
#pragma unroll
      for (int x = 0; x < AI; ++x) xi[x] = t[min(i0 + x, R - 1)];
#pragma unroll
      for (int y = 0; y < AJ; ++y) yj[y] = t[min(j0 + y, R - 1)];
#pragma unroll
      for (int x = 0; x < AI; ++x)
#pragma unroll
        for (int y = 0; y < AJ; ++y) gacc[x][y] += xi[x] * yj[y];
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // one R x R partial slot per warp (zeroed by the caller), summed in slot
  // order by k_reduce_ordered: the Gram does not depend on atomic order
  double* slot = g + (static_cast<uint64_t>(blockIdx.x) * W + warp) * R * R;
#pragma unroll
  for (int x = 0; x < AI; ++x)
#pragma unroll
    for (int y = 0; y < AJ; ++y) {
      const int gi = i0 + x, gj = j0 + y;
      if (gi < R && gj < R && gj >= gi) slot[gi * R + gj] = gacc[x][y];
    }
}

__device__ __forceinline__ double block_sum(double v);

// out[w] = sum_p parts[p * width + w] with a fixed reduction tree: one CTA
// per column, thread t adds slots t, t + blockDim, ... in order, then the
// fixed-shape block_sum.  The result depends only on the partials.
__global__ void k_reduce_ordered(const double* __restrict__ parts, uint64_t nparts, int width,
                                 double* __restrict__ out) {
  const int w = blockIdx.x;
  double s = 0.0;
  for (uint64_t q = threadIdx.x; q < nparts; q += blockDim.x) s += parts[q * width + w];
  s = block_sum(s);
  if (threadIdx.x == 0) out[w] = s;
}

// Fixed-order block sum of one value per thread: warp shuffle tree, then
// thread 0 adds the warps' sums in warp order and returns the total.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[32];
  for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += ws[w];
  return t;
}

// ---------------------------------------------------------------- R x R work
// The small dense steps of an ALS mode run on the device so an iteration is
// enqueued without host round trips (one read of the fit per iteration).
// Each restates the host arithmetic of dense_kernels.cpp / cpals.cpp in the
// same operation order with explicitly rounded operations, so it matches the
// host restatement bit for bit.

// V = hadamard_{m != n} grams[m] (cpals.cpp:86-90), then
// cholesky(V + shift I) with the Tikhonov escalation of solve_normal
// (dense_kernels.cpp:33-56, :72-80).  L_out gets L with its diagonal
// replaced by 1 / L_ii; status[0] = 1 when every shift failed.
__global__ void k_small_prep(const double* __restrict__ grams, int N, int n, int R, double* __restrict__ L_out,
                             int* __restrict__ status) {
  extern __shared__ double sm[];
  double* V = sm;          // R x R
  double* L = sm + R * R;  // R x R
  __shared__ int fail;
  __shared__ double shift;
  __shared__ double unit;  // trace / R; every thread's stop test reads it after a barrier
  const int RR = R * R;
  for (int i = threadIdx.x; i < RR; i += blockDim.x) {
    double v = 1.0;
    for (int m = 0; m < N; ++m)
      if (m != n) v = __dmul_rn(v, grams[static_cast<size_t>(m) * RR + i]);
    V[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double trace = 0.0;
    for (int i = 0; i < R; ++i) trace = __dadd_rn(trace, V[i * R + i]);
    unit = trace > 0.0 ? __ddiv_rn(trace, static_cast<double>(R)) : 1.0;
    shift = 0.0;
  }
  for (int attempt = 0;; ++attempt) {
    if (threadIdx.x == 0) fail = 0;
    __syncthreads();
    for (int j = 0; j < R; ++j) {
      if (threadIdx.x == 0) {
        double x = __dadd_rn(V[j * R + j], shift);
        for (int k = 0; k < j; ++k) x = __dsub_rn(x, __dmul_rn(L[j * R + k], L[j * R + k]));
        if (!(x > 0.0) || !isfinite(x)) fail = 1;
        L[j * R + j] = __dsqrt_rn(x);
      }
      __syncthreads();
      for (int i = j + 1 + threadIdx.x; i < R; i += blockDim.x) {
        double x = V[i * R + j];
        for (int k = 0; k < j; ++k) x = __dsub_rn(x, __dmul_rn(L[i * R + k], L[j * R + k]));
        L[i * R + j] = __ddiv_rn(x, L[j * R + j]);
      }
      __syncthreads();
    }
    if (!fail) break;
    // escalation: 0, then 1e-12 * unit, x10 each step, up to 1e-3 * unit
    if (threadIdx.x == 0) shift = attempt == 0 ? 1e-12 * unit : shift * 10.0;
    __syncthreads();
    if (!(shift <= 1e-3 * unit * (1.0 + 1e-9))) {
      if (threadIdx.x == 0) status[0] = 1;
      return;
    }
  }
  for (int i = threadIdx.x; i < RR; i += blockDim.x) {
    const int r = i / R, c = i % R;
    L_out[i] = c > r ? 0.0 : (r == c ? __ddiv_rn(1.0, L[i]) : L[i]);
  }
}

// lambda = sqrt(diag G) (0 -> 1, cpals.cpp:57-58); gram_out = G / (l l^T).
__global__ void k_small_norm(const double* __restrict__ G, int R, double* __restrict__ gram_out,
                             double* __restrict__ lam) {
  __shared__ double l[64];
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    double x = __dsqrt_rn(G[r * R + r]);
    l[r] = x == 0.0 ? 1.0 : x;
    lam[r] = l[r];
  }
  __syncthreads();
  for (int p = threadIdx.x; p < R * R; p += blockDim.x) {
    const int i = p / R, j = p % R;
    const int a = i < j ? i : j, b = i < j ? j : i;  // the upper triangle holds the sums
    gram_out[p] = __ddiv_rn(G[a * R + b], __dmul_rn(l[a], l[b]));
  }
}

// s[r] = 1 / prod_{m != n} lambda_m[r] (solve_fold)
__global__ void k_mscale(const double* __restrict__ lams, int N, int n, int R, double* __restrict__ out) {
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    double p = 1.0;
    for (int m = 0; m < N; ++m)
      if (m != n) p = __dmul_rn(p, lams[static_cast<size_t>(m) * R + r]);
    out[r] = __ddiv_rn(1.0, p);
  }
}

// fit (cpals.cpp:113-129): |Xhat|^2 = sum_rc prod_m gram_m[r,c] l_r l_c.
__global__ void k_small_fit(const double* __restrict__ grams, int N, int R, const double* __restrict__ lam,
                            const double* __restrict__ inner, double xn, double* __restrict__ fit_out) {
  if (threadIdx.x != 0) return;
  const int RR = R * R;
  double hat = 0.0;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < R; ++c) {
      double full = 1.0;
      for (int m = 0; m < N; ++m) full = __dmul_rn(full, grams[static_cast<size_t>(m) * RR + r * R + c]);
      hat = __dadd_rn(hat, __dmul_rn(__dmul_rn(full, lam[r]), lam[c]));
    }
  const double resid = fmax(0.0, __dadd_rn(__dsub_rn(xn, __dmul_rn(2.0, inner[0])), hat));
  fit_out[0] = __dsub_rn(1.0, __ddiv_rn(__dsqrt_rn(resid), __dsqrt_rn(xn)));
}

// Fused epilogue pass 2: A /= lambda column-wise (cpals.cpp:59-60) and, for
// the last mode, the fit's <X, Xhat> = sum m[i,r] lambda[r] A[i,r]
// (cpals.cpp:36-44) on the normalised A.
// V2: even R and 16-byte aligned rows, two columns per thread with 16-byte
// loads and stores (the pass is HBM-bound: 2 or 3 x I_n x R x 8 bytes).
template <bool V2>
__global__ void k_scale_inner(double* __restrict__ a, uint64_t rows, int R, const double* __restrict__ lambda,
                              const double* __restrict__ m, double* __restrict__ inner) {
  __shared__ double rl[64], il[64];  // lambda and 1 / lambda (R <= 64)
  for (int r = threadIdx.x; r < R; r += blockDim.x) rl[r] = lambda[r], il[r] = 1.0 / lambda[r];
  __syncthreads();
  const uint64_t n = rows * R;
  double s = 0.0;
  if constexpr (V2) {
    double2* a2 = reinterpret_cast<double2*>(a);
    const double2* m2 = reinterpret_cast<const double2*>(m);
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n / 2;
         i += uint64_t(gridDim.x) * blockDim.x) {
      const int c = static_cast<int>((R & (R - 1)) == 0 ? (2 * i) & (R - 1) : (2 * i) % R);
      double2 x = a2[i];
      x.x = x.x * il[c];
      x.y = x.y * il[c + 1];
      a2[i] = x;
      if (m) {
        const double2 y = m2[i];
        s += y.x * rl[c] * x.x;
        s += y.y * rl[c + 1] * x.y;
      }
    }
  } else {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
      const int c = static_cast<int>((R & (R - 1)) == 0 ? i & (R - 1) : i % R);
      const double x = a[i] * il[c];
      a[i] = x;
      if (m) s += m[i] * rl[c] * x;
    }
  }
  if (!m) return;
  s = block_sum(s);
  if (threadIdx.x == 0) inner[blockIdx.x] = s;  // per-block partial, reduced in block order
}

// G (R x R, upper triangle) += A^T A.  Each CTA stages chunks of rows in
// shared memory; every (i, j) pair is owned by one thread, whose running sum
// lives in shared memory (gpart), flushed with one atomic per pair.
constexpr int kGramChunk = 32;
__global__ void k_gram(const double* __restrict__ a, uint64_t rows, int R,
                       double* __restrict__ g) {
  extern __shared__ double smem[];
  double* gpart = smem;           // R * R
  double* tile = smem + R * R;    // kGramChunk * R
  const int pairs = R * R;
  for (int p = threadIdx.x; p < pairs; p += blockDim.x) gpart[p] = 0.0;
  for (uint64_t r0 = blockIdx.x * uint64_t(kGramChunk); r0 < rows;
       r0 += uint64_t(gridDim.x) * kGramChunk) {
    const int nr = static_cast<int>(rows - r0 < uint64_t(kGramChunk) ? rows - r0 : kGramChunk);
    __syncthreads();
    for (int i = threadIdx.x; i < nr * R; i += blockDim.x) tile[i] = a[r0 * R + i];
    __syncthreads();
    for (int p = threadIdx.x; p < pairs; p += blockDim.x) {
      const int i = p / R, j = p % R;
      if (j < i) continue;
      double s = 0.0;
      for (int r = 0; r < nr; ++r) s += tile[r * R + i] * tile[r * R + j];
      gpart[p] += s;
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < pairs; p += blockDim.x)
    g[static_cast<uint64_t>(blockIdx.x) * pairs + p] = p % R >= p / R ? gpart[p] : 0.0;
}

// sum_{i,r} m[i,r] * lambda[r] * a[i,r]
__global__ void k_inner(const double* __restrict__ m, const double* __restrict__ a, uint64_t rows,
                        int R, const double* __restrict__ lambda, double* __restrict__ out) {
  double s = 0.0;
  const uint64_t n = rows * R;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    s += m[i] * lambda[i % R] * a[i];
  s = block_sum(s);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void k_sumsq(const double* __restrict__ v, uint64_t n, double* __restrict__ out) {
  double s = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    s += v[i] * v[i];
  s = block_sum(s);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// out (R x R, full) = the upper triangle of g mirrored (Gram partials keep
// only i <= j, k_gram / k_solve_gram)
__global__ void k_symmetrize(const double* __restrict__ g, int R, double* __restrict__ out) {
  for (int p = threadIdx.x; p < R * R; p += blockDim.x) {
    const int i = p / R, j = p % R;
    out[p] = j >= i ? g[i * R + j] : g[j * R + i];
  }
}

bool exact_rank(int R) { return R == 16 || R == 32; }

unsigned grid_of(uint64_t n) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + kT - 1) / kT, sm_count() * 16)));
}

// Every reduction of the epilogue writes per-CTA (or per-warp) partials that
// k_reduce_ordered sums in a fixed order, so CP-ALS is bit-reproducible given
// bit-reproducible MTTKRPs (ExecConfig::deterministic).
struct Dense {
  int R;
  cudaStream_t s = nullptr;  // every launch and copy of the epilogue goes here
  DevBuf<double> L, small;  // small: R x R reduced Gram | R lambda | 1 scalar
  DevBuf<double> parts;     // partial slots (grown on demand)
  DevBuf<double> ones;      // R ones: c_S when the normalisation is not folded
  DevBuf<double> mscale;    // solve_fold: 1 / prod_{m != n} lambda_m

  // parts is sized up front for the largest reduction of a call (the solve's
  // per-warp Gram slots at full occupancy), so no iteration reallocates --
  // a cudaFree/cudaMalloc inside the loop stalls the queued kernels.
  explicit Dense(int r)
      : R(r), L(static_cast<size_t>(r) * r), small(static_cast<size_t>(r) * r + r + 1), ones(r), mscale(r) {
    const std::vector<double> h(r, 1.0);
    B200_CUDA(cudaMemcpy(ones.ptr, h.data(), r * sizeof(double), cudaMemcpyHostToDevice));
    const int nsm = sm_count();
    slots(std::max<uint64_t>(uint64_t(nsm) * 32 * (kSolveThreads / 32) * r * r, uint64_t(nsm) * 16 * 4));
  }

  double* slots(uint64_t n) {
    if (parts.n < n) parts.alloc(n);
    return parts.ptr;
  }
  // sum nslots partials of `width` values in slot order into small[0..width)
  void reduce(uint64_t nslots, int width) {
    k_reduce_ordered<<<width, 256, 0, s>>>(parts.ptr, nslots, width, small.ptr);
    count_launch();
    check_launch("k_reduce_ordered");
  }
  std::vector<double> fetch(int width) {
    std::vector<double> h(width);
    B200_CUDA(cudaMemcpyAsync(h.data(), small.ptr, width * 8, cudaMemcpyDeviceToHost, s));
    B200_CUDA(cudaStreamSynchronize(s));
    return h;
  }

  // upper triangle of Gram(A) over `rows` rows into small (dense_kernels.cpp:8-21)
  void gram_upper(const double* a, uint64_t rows) {
    const int RR = R * R;
    if (!rows) {
      B200_CUDA(cudaMemsetAsync(small.ptr, 0, RR * sizeof(double), s));
      return;
    }
    const size_t smem = (static_cast<size_t>(RR) + kGramChunk * R) * sizeof(double);
    if (smem > 48 * 1024)
      ensure_dyn_smem(reinterpret_cast<const void*>(k_gram), smem);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((rows + kGramChunk - 1) / kGramChunk, sm_count() * 8));
    k_gram<<<grid, kT, smem, s>>>(a, rows, R, slots(uint64_t(grid) * RR));
    count_launch();
    check_launch("k_gram");
    reduce(grid, RR);
  }

  std::vector<double> gram(const double* a, uint64_t rows) {
    const int RR = R * R;
    if (!rows) return std::vector<double>(RR, 0.0);
    gram_upper(a, rows);
    std::vector<double> g = fetch(RR);
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < i; ++j) g[i * R + j] = g[j * R + i];
    return g;
  }

  // small's upper triangle -> out, full symmetric R x R
  void symmetric_out(double* out) {
    k_symmetrize<<<1, 256, 0, s>>>(small.ptr, R, out);
    count_launch();
    check_launch("k_symmetrize");
  }

  // Solve step of one ALS mode (cpals.cpp:84-91, solve_normal
  // dense_kernels.cpp:68-92): V = hadamard_{m != n} grams[m] and its Cholesky
  // factor (Tikhonov escalation) on the device, then A = M V^-1 over `rows`
  // rows fused with Gram(A), whose upper triangle is left in small.
  // status[0] is set when V stays singular after the maximal shift.
  // const_L: R = 16/32 read L from the process-wide __constant__ c_L (only
  // for callers that serialise the whole ALS run, blco_cp_als); otherwise
  // the kernel reads L from this Dense's own device buffer.
  // mscale (device, R values, or null): columns of M are multiplied by it as
  // the rows are loaded (cp_als with the normalisation folded, solve_fold).
  void solve(const double* m, double* a, uint64_t rows, const double* dgrams, int N, int n, int* dstatus,
             bool const_L = false, const double* mscale = nullptr) {
    const int RR = R * R;
    const size_t prep_smem = 2 * static_cast<size_t>(RR) * sizeof(double);  // V and L: 64 KB at R = 64
    if (prep_smem > 48 * 1024) ensure_dyn_smem(reinterpret_cast<const void*>(k_small_prep), prep_smem);
    k_small_prep<<<1, 256, prep_smem, s>>>(dgrams, N, n, R, L.ptr, dstatus);
    count_launch();
    check_launch("k_small_prep");
    if (const_L && exact_rank(R)) {
      B200_CUDA(cudaMemcpyToSymbolAsync(c_L, L.ptr, RR * sizeof(double), 0, cudaMemcpyDeviceToDevice, s));
      B200_CUDA(cudaMemcpyToSymbolAsync(c_S, mscale ? mscale : ones.ptr, R * sizeof(double), 0,
                                        cudaMemcpyDeviceToDevice, s));
    }
    if (!rows) {
      B200_CUDA(cudaMemsetAsync(small.ptr, 0, RR * sizeof(double), s));
      return;
    }
    auto launch = [&](auto kern, int rm, int rows_per) {
      const size_t smem =
          (static_cast<size_t>(rm) * rm + kSolveStages * static_cast<size_t>(rows_per) * (rm + 1)) * 8;
      ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
      const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kern), kSolveThreads, smem);
      const unsigned grid = static_cast<unsigned>(
          std::min<uint64_t>((rows + rows_per - 1) / rows_per, uint64_t(sm_count()) * std::max(1, per_sm)));
      const uint64_t nslots = uint64_t(grid) * (kSolveThreads / 32);
      double* sl = slots(nslots * RR);
      // R <= 32: every warp writes the whole upper triangle of its slot (the
      // lower one is never read); R = 64: each warp owns one quadrant
      if (rm > 32) B200_CUDA(cudaMemsetAsync(sl, 0, nslots * RR * 8, s));
      kern<<<grid, kSolveThreads, smem, s>>>(m, a, rows, R, L.ptr, mscale, sl);
      count_launch();
      check_launch("k_solve_gram");
      reduce(nslots, RR);
    };
    if (R == 16 && const_L) launch(k_solve_gram<16, true>, 16, solve_rows<16>());
    else if (R == 32 && const_L) launch(k_solve_gram<32, true>, 32, solve_rows<32>());
    else if (R < 16) launch(k_solve_gram<16, false>, 16, solve_rows<16>());
    else if (R < 32) launch(k_solve_gram<32, false>, 32, solve_rows<32>());
    else if (R <= 64) launch(k_solve_gram<64, false>, 64, solve_rows<64>());
    else throw_format("b200: cp_als supports rank <= 64 on the device");
  }

  // normalize_columns (cpals.cpp:51-61) given G = Gram(A) (upper triangle
  // read): lambda = sqrt(diag G), gram_n = Gram(A / lambda) = G / (l l^T),
  // A /= lambda over `rows` rows, and with m_inner the fit's
  // <X, Xhat> = sum m lambda A over those rows into *dinner (cpals.cpp:36-44).
  void normalize(const double* G, double* a, uint64_t rows, double* gram_n, double* dlam,
                 const double* m_inner, double* dinner) {
    k_small_norm<<<1, 256, 0, s>>>(G, R, gram_n, dlam);
    count_launch();
    check_launch("k_small_norm");
    if (m_inner) B200_CUDA(cudaMemsetAsync(dinner, 0, sizeof(double), s));
    if (rows) {
      const bool v2 = R % 2 == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(m_inner) % 16 == 0;
      const unsigned grid = grid_of(v2 ? rows * R / 2 : rows * R);
      double* part = m_inner ? slots(grid) : nullptr;
      if (v2) k_scale_inner<true><<<grid, kT, 0, s>>>(a, rows, R, dlam, m_inner, part);
      else k_scale_inner<false><<<grid, kT, 0, s>>>(a, rows, R, dlam, m_inner, part);
      count_launch();
      check_launch("k_scale_inner");
      if (m_inner) {
        k_reduce_ordered<<<1, 256, 0, s>>>(part, grid, 1, dinner);
        count_launch();
        check_launch("k_reduce_ordered");
      }
    }
  }

  // One ALS mode's dense steps with the column normalisation folded into the
  // next solves (blco_cp_als): the factors stay UNnormalised on the device,
  // A_m = A_m' diag(lambda_m) with A_m' the reference's normalised factor
  // (cpals.cpp:51-61), so an MTTKRP over them is M' diag(prod_{m != n}
  // lambda_m) column-wise, and the solve multiplies the columns of M by
  // s = 1 / prod_{m != n} lambda_m as it loads them.  Then lambda_n =
  // sqrt(diag Gram(A_n)) and Gram(A_n') = Gram(A_n) / (l l^T) as before, with
  // no pass over A_n (the reference's A_n /= lambda, one read and one write of
  // I_n x R, is applied once, when the factors are returned).  For the last
  // mode (dinner set) <X, Xhat> = sum M' lambda A' = sum M s A.
  // dlams: N x R, every mode's lambda.
  void solve_fold(const double* m, double* a, uint64_t rows, double* dgrams, int N, int n, double* dlams,
                  int* dstatus, double* dinner) {
    // BLCO_B200_ALS_PROBE=1: device time of each step of this epilogue (stderr)
    static const bool probe = std::getenv("BLCO_B200_ALS_PROBE") != nullptr;
    cudaEvent_t pe[3] = {};
    auto pmark = [&](int k) {
      if (!probe) return;
      cudaEventCreate(&pe[k]);
      cudaEventRecord(pe[k], s);
    };
    pmark(0);
    k_mscale<<<1, 64, 0, s>>>(dlams, N, n, R, mscale.ptr);
    count_launch();
    check_launch("k_mscale");
    solve(m, a, rows, dgrams, N, n, dstatus, /*const_L=*/true, mscale.ptr);  // only blco_cp_als (serialised)
    pmark(1);
    k_small_norm<<<1, 256, 0, s>>>(small.ptr, R, dgrams + static_cast<size_t>(n) * R * R,
                                   dlams + static_cast<size_t>(n) * R);
    count_launch();
    check_launch("k_small_norm");
    if (dinner) {
      B200_CUDA(cudaMemsetAsync(dinner, 0, sizeof(double), s));
      if (rows) {
        const unsigned grid = grid_of(rows * R);
        k_inner<<<grid, kT, 0, s>>>(m, a, rows, R, mscale.ptr, slots(grid));
        count_launch();
        check_launch("k_inner");
        k_reduce_ordered<<<1, 256, 0, s>>>(parts.ptr, grid, 1, dinner);
        count_launch();
        check_launch("k_reduce_ordered");
      }
    }
    pmark(2);
    if (probe) {
      cudaEventSynchronize(pe[2]);
      float t[2];
      for (int k = 0; k < 2; ++k) cudaEventElapsedTime(&t[k], pe[k], pe[k + 1]);
      std::fprintf(stderr, "[als probe] mode %d rows %llu: prep+solve+gram %.3f norm+inner %.3f ms\n",
                   n, static_cast<unsigned long long>(rows), t[0], t[1]);
      for (int k = 0; k < 3; ++k) cudaEventDestroy(pe[k]);
    }
  }

  // A /= lambda over `rows` rows (the folded normalisation, applied once)
  void scale_rows(double* a, uint64_t rows, const double* dlam) {
    if (!rows) return;
    const bool v2 = R % 2 == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0;
    const unsigned grid = grid_of(v2 ? rows * R / 2 : rows * R);
    if (v2) k_scale_inner<true><<<grid, kT, 0, s>>>(a, rows, R, dlam, nullptr, nullptr);
    else k_scale_inner<false><<<grid, kT, 0, s>>>(a, rows, R, dlam, nullptr, nullptr);
    count_launch();
    check_launch("k_scale_inner");
  }

  double inner(const double* m, const double* a, uint64_t rows, const std::vector<double>& lambda) {
    if (!rows) return 0.0;
    double* lam = small.ptr + R * R;
    B200_CUDA(cudaMemcpyAsync(lam, lambda.data(), R * 8, cudaMemcpyHostToDevice, s));
    const unsigned grid = grid_of(rows * R);
    k_inner<<<grid, kT, 0, s>>>(m, a, rows, R, lam, slots(grid));
    count_launch();
    check_launch("k_inner");
    k_reduce_ordered<<<1, 256, 0, s>>>(parts.ptr, grid, 1, lam + R);
    count_launch();
    check_launch("k_reduce_ordered");
    double h = 0;
    B200_CUDA(cudaMemcpyAsync(&h, lam + R, 8, cudaMemcpyDeviceToHost, s));
    B200_CUDA(cudaStreamSynchronize(s));
    return h;
  }
};

double tensor_norm_sq(const blco_tensor& t) {
  if (!t.nnz) return 0.0;
  const unsigned grid = grid_of(t.nnz);
  DevBuf<double> part(grid), out(1);
  k_sumsq<<<grid, kT>>>(t.vals.ptr, t.nnz, part.ptr);
  count_launch();
  check_launch("k_sumsq");
  k_reduce_ordered<<<1, 256>>>(part.ptr, grid, 1, out.ptr);
  count_launch();
  check_launch("k_reduce_ordered");
  double h = 0;
  B200_CUDA(cudaMemcpy(&h, out.ptr, 8, cudaMemcpyDeviceToHost));
  return h;
}

// Dense epilogue state per (device, rank) for the calling thread: the
// distributed ALS pieces below are called once per mode, so their partial
// buffers must not be reallocated per call.
Dense& dense_cache(int R, cudaStream_t s) {
  thread_local std::map<std::pair<int, int>, std::unique_ptr<Dense>> cache;
  int dev = 0;
  B200_CUDA(cudaGetDevice(&dev));
  auto& d = cache[{dev, R}];
  if (!d) d = std::make_unique<Dense>(R);
  d->s = s;
  return *d;
}

double recon_norm_sq(const std::vector<std::vector<double>>& grams, const std::vector<double>& lam,
                     int R) {
  std::vector<double> full(static_cast<size_t>(R) * R, 1.0);
  for (const auto& g : grams)
    for (size_t i = 0; i < full.size(); ++i) full[i] *= g[i];
  double s = 0;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < R; ++c) s += full[r * R + c] * lam[r] * lam[c];
  return s;
}

double fit_value(double xn, double inner, double hat) {
  const double resid = std::max(0.0, xn - 2.0 * inner + hat);
  return 1.0 - std::sqrt(resid) / std::sqrt(xn);
}

void mttkrp_into(const blco_tensor& t, const std::vector<const double*>& f, uint64_t R, int mode,
                 int strategy, const blco_exec_config& cfg, double* out) {
  MttkrpLaunch a{};
  a.view = view_of(t);
  a.tensor = &t;
  a.factors = f.data();
  a.rank = R;
  a.mode = mode;
  a.strategy = strategy == BLCO_STRATEGY_AUTO ? auto_kernel(t.layout.dims[mode], cfg) : strategy;
  a.cfg = cfg;
  a.out = out;
  a.stream = nullptr;
  mttkrp_enqueue(a);
}

}  // namespace
}  // namespace b200

using namespace b200;

extern "C" {

int blco_cp_als(const blco_tensor* t, uint64_t rank, int max_iters, double tol, uint64_t seed,
                int strategy, const blco_exec_config* cfg, double* const* factors_out,
                double* lambda_out, double* fit_out, int* iters_out) {
  return blco_cp_als_timed(t, rank, max_iters, tol, seed, strategy, cfg, factors_out, lambda_out, fit_out,
                           iters_out, nullptr);
}

int blco_cp_als_timed(const blco_tensor* t, uint64_t rank, int max_iters, double tol, uint64_t seed,
                      int strategy, const blco_exec_config* cfg, double* const* factors_out,
                      double* lambda_out, double* fit_out, int* iters_out, blco_cp_als_stats* st) {
  return guarded([&] {
    if (rank < 1) throw_format("cp_als: rank must be >= 1");
    if (max_iters < 0) throw_format("cp_als: max_iters must be >= 0");
    // c_L (constant memory) is one per device context: ALS runs are
    // serialised within the process
    static std::mutex als_mu;
    std::lock_guard<std::mutex> als_lock(als_mu);
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    if (blco_exec_config_validate(&c) != BLCO_OK) throw_format(blco_last_error());
    DeviceGuard dg(t->device);
    const blco_layout& l = t->layout;
    const int N = l.order, R = static_cast<int>(rank);
    *iters_out = 0;
    std::vector<DevBuf<double>> A(N);
    std::vector<const double*> ptr(N);
    for (int m = 0; m < N; ++m) {
      A[m].alloc(l.dims[m] * rank);
      ptr[m] = A[m].ptr;
    }
    // FactorMatrices::random(dims, rank, seed) -- same bits as the host
    std::vector<double*> wptr(N);
    for (int m = 0; m < N; ++m) wptr[m] = A[m].ptr;
    if (blco_factors_random_device(l.dims, N, rank, seed, wptr.data(), nullptr) != BLCO_OK)
      throw Status(BLCO_ECUDA, blco_last_error());
    std::vector<double> lambda(rank, 1.0);
    auto emit = [&] {
      for (int m = 0; m < N; ++m)
        if (A[m].n) B200_CUDA(cudaMemcpy(factors_out[m], A[m].ptr, A[m].bytes(), cudaMemcpyDeviceToHost));
      std::memcpy(lambda_out, lambda.data(), rank * 8);
    };
    if (max_iters == 0) {
      emit();
      return;
    }
    const double xn = tensor_norm_sq(*t);
    if (xn == 0.0) throw_format("cp_als: zero-norm tensor");
    Dense dense(R);
    const int RR = R * R;
    // Grams, lambda, <X, Xhat>, fit and the singular flag live on the device
    // dlams: every mode's lambda (the factors stay unnormalised, solve_fold)
    DevBuf<double> dgrams(static_cast<size_t>(N) * RR), dlams(static_cast<size_t>(N) * R), dinner(1),
        dfit(std::max(1, max_iters));
    DevBuf<int> dstatus(1);
    B200_CUDA(cudaMemset(dstatus.ptr, 0, sizeof(int)));
    {
      const std::vector<double> ones(static_cast<size_t>(N) * R, 1.0);
      B200_CUDA(cudaMemcpy(dlams.ptr, ones.data(), ones.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    const double* dlam_last = dlams.ptr + static_cast<size_t>(N - 1) * R;
    // the reference's A_n /= lambda_n (cpals.cpp:59-60), applied once on the way out
    auto normalise_factors = [&] {
      for (int m = 0; m < N; ++m) dense.scale_rows(A[m].ptr, l.dims[m], dlams.ptr + static_cast<size_t>(m) * R);
    };
    for (int m = 0; m < N; ++m) {
      const std::vector<double> g = dense.gram(A[m].ptr, l.dims[m]);
      B200_CUDA(cudaMemcpy(dgrams.ptr + static_cast<size_t>(m) * RR, g.data(), RR * sizeof(double),
                           cudaMemcpyHostToDevice));
    }
    uint64_t maxrows = 0;
    for (int m = 0; m < N; ++m) maxrows = std::max<uint64_t>(maxrows, l.dims[m]);
    DevBuf<double> mt(maxrows * rank);
    double prev = 0.0;
    int it = 0;
    // BLCO_B200_TRACE=1: synchronise around the MTTKRPs and report where the
    // iteration time goes (stderr).
    static const bool trace = std::getenv("BLCO_B200_TRACE") != nullptr;
    double acc[2] = {0, 0};
    auto t_last = std::chrono::steady_clock::now();
    // device-time accounting (CUDA events on the legacy stream the loop runs on)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_mt, ev_all;
    auto mark = [](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v, bool begin) {
      if (begin) {
        v.emplace_back(nullptr, nullptr);
        cudaEventCreate(&v.back().first);
        cudaEventRecord(v.back().first, nullptr);
      } else {
        cudaEventCreate(&v.back().second);
        cudaEventRecord(v.back().second, nullptr);
      }
    };
    auto tick = [&](int slot) {
      if (!trace) return;
      cudaDeviceSynchronize();
      const auto now = std::chrono::steady_clock::now();
      acc[slot] += std::chrono::duration<double>(now - t_last).count();
      t_last = now;
    };
    auto fetch_lambda = [&] {
      B200_CUDA(cudaMemcpy(lambda.data(), dlam_last, R * sizeof(double), cudaMemcpyDeviceToHost));
    };
    for (; it < max_iters; ++it) {
      NvtxRange nv("cp_als iteration");
      if (st) mark(ev_all, true);
      for (int n = 0; n < N; ++n) {
        tick(1);
        if (st) mark(ev_mt, true);
        mttkrp_into(*t, ptr, rank, n, strategy, c, mt.ptr);
        if (st) mark(ev_mt, false);
        tick(0);
        // A_n = M V^-1 (unnormalised) straight into A_n; M of the last mode
        // stays in mt for the fit's inner product
        dense.solve_fold(mt.ptr, A[n].ptr, l.dims[n], dgrams.ptr, N, n, dlams.ptr, dstatus.ptr,
                         n == N - 1 ? dinner.ptr : nullptr);
      }
      k_small_fit<<<1, 32>>>(dgrams.ptr, N, R, dlam_last, dinner.ptr, xn, dfit.ptr + it);
      count_launch();
      check_launch("k_small_fit");
      if (st) mark(ev_all, false);
      // the iteration's one host round trip: its fit and the singular flag
      double f = 0;
      int singular = 0;
      B200_CUDA(cudaMemcpy(&f, dfit.ptr + it, sizeof(double), cudaMemcpyDeviceToHost));
      B200_CUDA(cudaMemcpy(&singular, dstatus.ptr, sizeof(int), cudaMemcpyDeviceToHost));
      tick(1);
      if (singular) throw_error("solve_normal: matrix singular after maximal diagonal shift");
      fit_out[it] = f;
      *iters_out = it + 1;
      if (!std::isfinite(f)) {
        fetch_lambda();
        normalise_factors();
        emit();
        throw_error("cp_als: non-finite fit at iteration " + std::to_string(it + 1));
      }
      if (it > 0 && f - prev < tol) break;
      prev = f;
    }
    fetch_lambda();
    if (st) {
      B200_CUDA(cudaDeviceSynchronize());
      auto sum = [](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
        double ms = 0;
        for (auto& [a, b] : v) {
          float x = 0;
          if (a && b && cudaEventElapsedTime(&x, a, b) == cudaSuccess) ms += x;
          if (a) cudaEventDestroy(a);
          if (b) cudaEventDestroy(b);
        }
        return ms;
      };
      st->iterations = static_cast<int>(ev_all.size());
      st->mttkrp_ms = sum(ev_mt);
      st->iterations_ms = sum(ev_all);
    }
    if (trace)
      std::fprintf(stderr, "[blco trace] cp_als %d iters: mttkrp %.3f s, dense epilogue + fit %.3f s\n", it, acc[0],
                   acc[1]);
    normalise_factors();
    emit();
  });
}

int blco_fit(const blco_tensor* t, const double* const* factors, const double* lambda,
             uint64_t rank, const blco_exec_config* cfg, double* fit_out) {
  return guarded([&] {
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    DeviceGuard dg(t->device);
    const blco_layout& l = t->layout;
    const int N = l.order, R = static_cast<int>(rank);
    const double xn = tensor_norm_sq(*t);
    if (xn == 0.0) throw_format("fit: zero-norm tensor");
    std::vector<DevBuf<double>> A(N);
    std::vector<const double*> ptr(N);
    Dense dense(R);
    std::vector<std::vector<double>> grams(N);
    for (int m = 0; m < N; ++m) {
      A[m].alloc(l.dims[m] * rank);
      if (A[m].n) B200_CUDA(cudaMemcpy(A[m].ptr, factors[m], A[m].bytes(), cudaMemcpyHostToDevice));
      ptr[m] = A[m].ptr;
      grams[m] = dense.gram(A[m].ptr, l.dims[m]);
    }
    DevBuf<double> ml(l.dims[N - 1] * rank);
    mttkrp_into(*t, ptr, rank, N - 1, BLCO_STRATEGY_AUTO, c, ml.ptr);
    std::vector<double> lam(lambda, lambda + rank);
    *fit_out = fit_value(xn, dense.inner(ml.ptr, A[N - 1].ptr, l.dims[N - 1], lam),
                         recon_norm_sq(grams, lam, R));
  });
}

// ------------------------------------------- distributed CP-ALS pieces
// The dense steps of one ALS mode split where a multi-GPU run reduces across
// ranks: see include/blco_b200.h.

int blco_tensor_norm_sq(const blco_tensor* t, double* d_out, void* stream) {
  return guarded([&] {
    DeviceGuard dg(t->device);
    auto s = static_cast<cudaStream_t>(stream);
    Dense& d = dense_cache(1, s);
    if (!t->nnz) {
      B200_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double), s));
      return;
    }
    const unsigned grid = grid_of(t->nnz);
    double* part = d.slots(grid);
    k_sumsq<<<grid, kT, 0, s>>>(t->vals.ptr, t->nnz, part);
    count_launch();
    check_launch("k_sumsq");
    k_reduce_ordered<<<1, 256, 0, s>>>(part, grid, 1, d_out);
    count_launch();
    check_launch("k_reduce_ordered");
  });
}

int blco_als_gram(const double* d_a, uint64_t rows, uint64_t rank, double* d_gram, void* stream) {
  return guarded([&] {
    if (rank < 1 || rank > 64) throw_format("cp_als: rank must be in [1, 64] on the device");
    Dense& d = dense_cache(static_cast<int>(rank), static_cast<cudaStream_t>(stream));
    d.gram_upper(d_a, rows);
    d.symmetric_out(d_gram);
  });
}

int blco_als_solve(const double* d_grams, int order, int mode, uint64_t rank, const double* d_m, uint64_t rows,
                   double* d_a, double* d_gram, int* d_status, void* stream) {
  return guarded([&] {
    if (rank < 1 || rank > 64) throw_format("cp_als: rank must be in [1, 64] on the device");
    if (order < 1 || mode < 0 || mode >= order) throw_format("cp_als: mode out of range");
    Dense& d = dense_cache(static_cast<int>(rank), static_cast<cudaStream_t>(stream));
    d.solve(d_m, d_a, rows, d_grams, order, mode, d_status);
    d.symmetric_out(d_gram);
  });
}

int blco_als_normalize(const double* d_gram_sum, uint64_t rank, double* d_a, uint64_t rows, double* d_gram_n,
                       double* d_lambda, const double* d_m, double* d_inner, void* stream) {
  return guarded([&] {
    if (rank < 1 || rank > 64) throw_format("cp_als: rank must be in [1, 64] on the device");
    Dense& d = dense_cache(static_cast<int>(rank), static_cast<cudaStream_t>(stream));
    d.normalize(d_gram_sum, d_a, rows, d_gram_n, d_lambda, d_m, d_inner);
  });
}

int blco_als_fit(const double* d_grams, int order, uint64_t rank, const double* d_lambda, const double* d_inner,
                 double xnormsq, double* d_fit, void* stream) {
  return guarded([&] {
    if (xnormsq == 0.0) throw_format("cp_als: zero-norm tensor");
    k_small_fit<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(d_grams, order, static_cast<int>(rank), d_lambda,
                                                                 d_inner, xnormsq, d_fit);
    count_launch();
    check_launch("k_small_fit");
  });
}

}  // extern "C"
