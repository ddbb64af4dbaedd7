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

int main() {
  double *a, *out;
  cudaMalloc(&a, kRows * 32ull * 8);
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaMemset(a, 0, kRows * 32ull * 8);
  for (int rep = 0; rep < 2; ++rep) {
    k_ldg64_pair<<<148 * 8, 256>>>(a, out);
    k_ldg128_pair<<<148 * 8, 256>>>(a, out);
    k_ldg64_warp<<<148 * 8, 256>>>(a, out);
  }
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
