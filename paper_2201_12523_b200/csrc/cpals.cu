// cpals.cu -- CP-ALS driver with factors resident in HBM (config 4).
//
// Reference: cp_als / fit, proj/src/cpals.cpp:66-129; dense kernels
// proj/src/dense_kernels.cpp:8-92.  Per iteration and mode n (Alg. 1):
//   V = hadamard_{m != n} Gram(A_m)            (R x R, host)
//   M = MTTKRP(X, n)                           (device, mttkrp.cu)
//   A_n = M V^-1 via Cholesky of V, Tikhonov escalation on failure
//                                              (factorisation on host, the
//                                               I_n row solves on device)
//   lambda = column 2-norms, A_n /= lambda     (device reductions)
//   Gram(A_n)                                  (device)
// then fit = 1 - sqrt(max(0, |X|^2 - 2<X,Xhat> + |Xhat|^2)) / |X|.
// Summation orders differ from the sequential host loops, so parity is
// tolerance-based.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.hpp"

namespace b200 {
namespace {

constexpr int kT = 256;

// Forward/back substitution of every row of M against L (R x R lower).
template <int RMAX>
__global__ void k_solve_rows(double* __restrict__ a, uint64_t rows, int R,
                             const double* __restrict__ L) {
  __shared__ double sl[RMAX * RMAX];
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) sl[i] = L[i];
  __syncthreads();
  for (uint64_t row = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; row < rows;
       row += uint64_t(gridDim.x) * blockDim.x) {
    double b[RMAX];
    double* p = a + row * R;
#pragma unroll
    for (int i = 0; i < RMAX; ++i)
      if (i < R) b[i] = p[i];
#pragma unroll
    for (int i = 0; i < RMAX; ++i) {
      if (i >= R) break;
      double s = b[i];
#pragma unroll
      for (int k = 0; k < RMAX; ++k)
        if (k < i) s -= sl[i * R + k] * b[k];
      b[i] = s / sl[i * R + i];
    }
#pragma unroll
    for (int ii = RMAX - 1; ii >= 0; --ii) {
      if (ii >= R) continue;
      double s = b[ii];
#pragma unroll
      for (int k = 0; k < RMAX; ++k)
        if (k > ii && k < R) s -= sl[k * R + ii] * b[k];
      b[ii] = s / sl[ii * R + ii];
    }
#pragma unroll
    for (int i = 0; i < RMAX; ++i)
      if (i < R) p[i] = b[i];
  }
}

// out[r] += sum_i a[i, r]^2 (one partial per CTA, then atomics).
__global__ void k_col_sumsq(const double* __restrict__ a, uint64_t rows, int R,
                            double* __restrict__ out) {
  extern __shared__ double part[];
  for (int i = threadIdx.x; i < R; i += blockDim.x) part[i] = 0.0;
  __syncthreads();
  const uint64_t n = rows * R;
  // thread t handles column (t % R) of rows t/R, t/R + blockDim/R, ...
  const int per = blockDim.x / R;
  const int c = threadIdx.x % R;
  double s = 0.0;
  if (static_cast<int>(threadIdx.x) < per * R)
    for (uint64_t row = blockIdx.x * uint64_t(per) + threadIdx.x / R; row < rows;
         row += uint64_t(gridDim.x) * per) {
      const double x = a[row * R + c];
      s += x * x;
    }
  (void)n;
  atomicAdd(&part[c], s);
  __syncthreads();
  for (int i = threadIdx.x; i < R; i += blockDim.x) atomicAdd(&out[i], part[i]);
}

__global__ void k_scale_cols(double* __restrict__ a, uint64_t rows, int R,
                             const double* __restrict__ lambda) {
  const uint64_t n = rows * R;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] /= lambda[i % R];
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
    if (p % R >= p / R) atomicAdd(&g[p], gpart[p]);
}

// sum_{i,r} m[i,r] * lambda[r] * a[i,r]
__global__ void k_inner(const double* __restrict__ m, const double* __restrict__ a, uint64_t rows,
                        int R, const double* __restrict__ lambda, double* __restrict__ out) {
  double s = 0.0;
  const uint64_t n = rows * R;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    s += m[i] * lambda[i % R] * a[i];
  for (int d = 16; d > 0; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

__global__ void k_sumsq(const double* __restrict__ v, uint64_t n, double* __restrict__ out) {
  double s = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    s += v[i] * v[i];
  for (int d = 16; d > 0; d >>= 1) s += __shfl_down_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}

unsigned grid_of(uint64_t n) {
  return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + kT - 1) / kT, 148 * 16)));
}

// dense_kernels.cpp:35-56 restated (host, R x R).
bool cholesky(const std::vector<double>& v, int r, double shift, std::vector<double>& L) {
  L.assign(static_cast<size_t>(r) * r, 0.0);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = v[i * r + j] + (i == j ? shift : 0.0);
      for (int k = 0; k < j; ++k) s -= L[i * r + k] * L[j * r + k];
      if (i == j) {
        if (!(s > 0.0) || !std::isfinite(s)) return false;
        L[i * r + i] = std::sqrt(s);
      } else {
        L[i * r + j] = s / L[j * r + j];
      }
    }
  return true;
}

struct Dense {
  int R;
  cudaStream_t s = nullptr;
  DevBuf<double> L, scratch;  // scratch: R*R gram / R lambda / 1 scalar

  explicit Dense(int r) : R(r), L(static_cast<size_t>(r) * r), scratch(static_cast<size_t>(r) * r + r + 1) {}

  std::vector<double> gram(const double* a, uint64_t rows) {
    B200_CUDA(cudaMemset(scratch.ptr, 0, static_cast<size_t>(R) * R * 8));
    if (rows) {
      const size_t smem = (static_cast<size_t>(R) * R + kGramChunk * R) * sizeof(double);
      if (smem > 48 * 1024)
        B200_CUDA(cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((rows + kGramChunk - 1) / kGramChunk, 148 * 8));
      k_gram<<<grid, kT, smem>>>(a, rows, R, scratch.ptr);
      count_launch();
      check_launch("k_gram");
    }
    std::vector<double> g(static_cast<size_t>(R) * R);
    B200_CUDA(cudaMemcpy(g.data(), scratch.ptr, g.size() * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < i; ++j) g[i * R + j] = g[j * R + i];
    return g;
  }

  void solve(double* m, uint64_t rows, const std::vector<double>& v) {
    double trace = 0.0;
    for (int i = 0; i < R; ++i) trace += v[i * R + i];
    const double unit = trace > 0.0 ? trace / R : 1.0;
    std::vector<double> Lh;
    bool ok = cholesky(v, R, 0.0, Lh);
    for (double lam = 1e-12 * unit; !ok && lam <= 1e-3 * unit * (1.0 + 1e-9); lam *= 10.0)
      ok = cholesky(v, R, lam, Lh);
    if (!ok) throw_error("solve_normal: matrix singular after maximal diagonal shift");
    B200_CUDA(cudaMemcpy(L.ptr, Lh.data(), Lh.size() * 8, cudaMemcpyHostToDevice));
    if (!rows) return;
    if (R <= 16) k_solve_rows<16><<<grid_of(rows), kT>>>(m, rows, R, L.ptr);
    else if (R <= 32) k_solve_rows<32><<<grid_of(rows), kT>>>(m, rows, R, L.ptr);
    else if (R <= 64) k_solve_rows<64><<<grid_of(rows), 128>>>(m, rows, R, L.ptr);
    else throw_format("b200: cp_als supports rank <= 64 on the device");
    count_launch();
    check_launch("k_solve_rows");
  }

  std::vector<double> normalize(double* a, uint64_t rows) {
    double* lam = scratch.ptr + static_cast<size_t>(R) * R;
    B200_CUDA(cudaMemset(lam, 0, R * 8));
    if (rows) {
      k_col_sumsq<<<grid_of(rows * R), kT, R * sizeof(double)>>>(a, rows, R, lam);
      count_launch();
      check_launch("k_col_sumsq");
    }
    std::vector<double> h(R);
    B200_CUDA(cudaMemcpy(h.data(), lam, R * 8, cudaMemcpyDeviceToHost));
    for (auto& x : h) {
      x = std::sqrt(x);
      if (x == 0.0) x = 1.0;  // cpals.cpp:58
    }
    B200_CUDA(cudaMemcpy(lam, h.data(), R * 8, cudaMemcpyHostToDevice));
    if (rows) {
      k_scale_cols<<<grid_of(rows * R), kT>>>(a, rows, R, lam);
      count_launch();
      check_launch("k_scale_cols");
    }
    return h;
  }

  double inner(const double* m, const double* a, uint64_t rows, const std::vector<double>& lambda) {
    double* lam = scratch.ptr + static_cast<size_t>(R) * R;
    double* out = lam + R;
    B200_CUDA(cudaMemcpy(lam, lambda.data(), R * 8, cudaMemcpyHostToDevice));
    B200_CUDA(cudaMemset(out, 0, 8));
    if (rows) {
      k_inner<<<grid_of(rows * R), kT>>>(m, a, rows, R, lam, out);
      count_launch();
      check_launch("k_inner");
    }
    double h = 0;
    B200_CUDA(cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost));
    return h;
  }
};

double tensor_norm_sq(const blco_tensor& t) {
  DevBuf<double> out(1);
  B200_CUDA(cudaMemset(out.ptr, 0, 8));
  if (t.nnz) {
    k_sumsq<<<grid_of(t.nnz), kT>>>(t.vals.ptr, t.nnz, out.ptr);
    count_launch();
    check_launch("k_sumsq");
  }
  double h = 0;
  B200_CUDA(cudaMemcpy(&h, out.ptr, 8, cudaMemcpyDeviceToHost));
  return h;
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
  a.factors = f.data();
  a.rank = R;
  a.mode = mode;
  a.strategy = strategy == BLCO_STRATEGY_AUTO ? blco_choose_strategy(t.layout.dims[mode], &cfg)
                                              : strategy;
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
    std::vector<std::vector<double>> grams(N);
    for (int m = 0; m < N; ++m) grams[m] = dense.gram(A[m].ptr, l.dims[m]);
    uint64_t maxrows = 0;
    for (int m = 0; m < N; ++m) maxrows = std::max<uint64_t>(maxrows, l.dims[m]);
    DevBuf<double> mt(maxrows * rank), mlast(l.dims[N - 1] * rank);
    double prev = 0.0;
    int it = 0;
    // BLCO_B200_TRACE=1: synchronise after every step and report where the
    // iteration time goes (stderr).
    static const bool trace = std::getenv("BLCO_B200_TRACE") != nullptr;
    double acc[6] = {0, 0, 0, 0, 0, 0};
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
    for (; it < max_iters; ++it) {
      if (st) mark(ev_all, true);
      for (int n = 0; n < N; ++n) {
        std::vector<double> v(static_cast<size_t>(R) * R, 1.0);
        for (int m = 0; m < N; ++m)
          if (m != n)
            for (size_t i = 0; i < v.size(); ++i) v[i] *= grams[m][i];
        tick(5);
        if (st) mark(ev_mt, true);
        mttkrp_into(*t, ptr, rank, n, strategy, c, mt.ptr);
        if (st) mark(ev_mt, false);
        if (n == N - 1 && mlast.n)
          B200_CUDA(cudaMemcpy(mlast.ptr, mt.ptr, mlast.bytes(), cudaMemcpyDeviceToDevice));
        tick(0);
        dense.solve(mt.ptr, l.dims[n], v);
        tick(1);
        B200_CUDA(cudaMemcpy(A[n].ptr, mt.ptr, A[n].bytes(), cudaMemcpyDeviceToDevice));
        tick(2);
        lambda = dense.normalize(A[n].ptr, l.dims[n]);
        tick(3);
        grams[n] = dense.gram(A[n].ptr, l.dims[n]);
        tick(4);
      }
      const double inner = dense.inner(mlast.ptr, A[N - 1].ptr, l.dims[N - 1], lambda);
      const double f = fit_value(xn, inner, recon_norm_sq(grams, lambda, R));
      fit_out[it] = f;
      *iters_out = it + 1;
      if (st) mark(ev_all, false);
      if (!std::isfinite(f)) {
        emit();
        throw_error("cp_als: non-finite fit at iteration " + std::to_string(it + 1));
      }
      if (it > 0 && f - prev < tol) break;
      prev = f;
    }
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
      std::fprintf(stderr,
                   "[blco trace] cp_als %d iters: mttkrp %.3f s, solve %.3f s, copy %.3f s, normalize %.3f s, "
                   "gram %.3f s, host %.3f s\n",
                   it, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5]);
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

}  // extern "C"
