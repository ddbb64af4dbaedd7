// Microbenchmark: L1 data-pipe (LSU) wavefronts per gathered factor row on
// sm_100a.  Two 16-lane groups per warp each gather one random 256-byte row
// (R = 32 doubles) of an L2-resident 13 MB matrix, like the MTTKRP compute
// phase.  Variants: lane owns columns (q, q+16) via 2 x LDG.64, or adjacent
// columns (2q, 2q+1) via 1 x LDG.128; a full warp per row with 1 x LDG.64.
// Run under ncu: l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,
// l1tex__lsu_writeback_active_mem_lgds.sum, smsp__inst_executed_op_global_ld.sum.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 256;
constexpr int kRows = 50000;  // 50000 x 256 B = 12.8 MB

__device__ __forceinline__ unsigned hash(unsigned x) { return (x * 2654435761u) >> 3; }

__global__ void k_ldg64_pair(const double* __restrict__ a, double* out) {
  const int lane = threadIdx.x & 31, g = lane >> 4, q = lane & 15;
  double s = 0;
  for (int i = 0; i < kIters; ++i) {
    const unsigned r = hash(blockIdx.x * 4096 + (threadIdx.x >> 4) * kIters + i) % kRows;
    const double* p = a + r * 32ull;
    s += __ldg(p + q) + __ldg(p + q + 16);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  (void)g;
}

__global__ void k_ldg128_pair(const double* __restrict__ a, double* out) {
  const int lane = threadIdx.x & 31, q = lane & 15;
  double s = 0;
  for (int i = 0; i < kIters; ++i) {
    const unsigned r = hash(blockIdx.x * 4096 + (threadIdx.x >> 4) * kIters + i) % kRows;
    const double2 v = __ldg(reinterpret_cast<const double2*>(a + r * 32ull) + q);
    s += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ldg64_warp(const double* __restrict__ a, double* out) {
  const int lane = threadIdx.x & 31;
  double s = 0;
  for (int i = 0; i < kIters; ++i) {
    const unsigned r = hash(blockIdx.x * 4096 + (threadIdx.x >> 5) * kIters + i) % kRows;
    s += __ldg(a + r * 32ull + lane);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// like the MTTKRP compute phase: 4 elements x 2 rows x (q, q+16) = 16 loads in
// flight per lane before any is consumed, plus a streaming 8-byte load per
// element from a DRAM-sized array (ld.global.cs)
template <int U, bool STREAM>
__global__ void k_ldg64_pair_u(const double* __restrict__ a, const double* __restrict__ stream, double* out) {
  const int lane = threadIdx.x & 31, q = lane & 15;
  double s = 0;
  for (int i = 0; i < kIters; i += U) {
    double v[U][4];
    double sv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned base = blockIdx.x * 4096 + (threadIdx.x >> 4) * kIters + i + u;
      const double* p = a + (hash(base) % kRows) * 32ull;
      const double* p2 = a + (hash(base ^ 0x5bd1e995u) % kRows) * 32ull;
      v[u][0] = __ldg(p + q), v[u][1] = __ldg(p + q + 16), v[u][2] = __ldg(p2 + q), v[u][3] = __ldg(p2 + q + 16);
      sv[u] = STREAM ? __ldcs(stream + (static_cast<size_t>(blockIdx.x) * kIters + i + u) * 256 + threadIdx.x) : 1.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s += sv[u] * v[u][0] * v[u][1] + v[u][2] * v[u][3];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double *a, *out;
  cudaMalloc(&a, kRows * 32ull * 8);
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaMemset(a, 0, kRows * 32ull * 8);
  double* st;
  cudaMalloc(&st, 148ull * 8 * 256 * kIters * 8);
  cudaMemset(st, 0, 148ull * 8 * 256 * kIters * 8);
  for (int rep = 0; rep < 2; ++rep) {
    k_ldg64_pair_u<1, false><<<148 * 8, 256>>>(a, st, out);
    k_ldg64_pair_u<4, false><<<148 * 8, 256>>>(a, st, out);
    k_ldg64_pair_u<1, true><<<148 * 8, 256>>>(a, st, out);
    k_ldg64_pair_u<4, true><<<148 * 8, 256>>>(a, st, out);
    k_ldg64_pair<<<148 * 8, 256>>>(a, out);
    k_ldg128_pair<<<148 * 8, 256>>>(a, out);
    k_ldg64_warp<<<148 * 8, 256>>>(a, out);
  }
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
