// Microbenchmark: cost of committing a 256-byte fp64 row (R = 32) into an
// L2-resident output on sm_100a, per committed row:
//   k_red16  : 16-lane group, 2 x RED.E.ADD.F64 (columns q, q+16) -- the
//              current MTTKRP commit;
//   k_red32  : full warp, 1 x RED.E.ADD.F64 per lane;
//   k_bulk   : the row is written to shared memory (2 x STS.64 per lane of a
//              16-lane group) and one lane issues cp.reduce.async.bulk
//              .global.shared::cta.add.f64 of 256 bytes (TMA bulk reduction).
// Run under ncu for LSU wavefronts and L2 traffic; time printed by events.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 64;
constexpr int kRows = 12000;  // 3 MB output

__device__ __forceinline__ unsigned hash(unsigned x) { return (x * 2654435761u) >> 3; }

__global__ void k_red16(double* out) {
  const int lane = threadIdx.x & 31, q = lane & 15;
  for (int i = 0; i < kIters; ++i) {
    const unsigned r = hash(blockIdx.x * 8192 + (threadIdx.x >> 4) * kIters + i) % kRows;
    atomicAdd(out + r * 32ull + q, 1.0);
    atomicAdd(out + r * 32ull + q + 16, 1.0);
  }
}

// only one 16-lane group active per instruction (divergent commits)
__global__ void k_red16_div(double* out) {
  const int lane = threadIdx.x & 31, q = lane & 15, g = lane >> 4;
  for (int i = 0; i < kIters; ++i) {
    const unsigned r = hash(blockIdx.x * 8192 + (threadIdx.x >> 4) * kIters + i) % kRows;
    if (g == (i & 1)) {
      atomicAdd(out + r * 32ull + q, 1.0);
      atomicAdd(out + r * 32ull + q + 16, 1.0);
    }
    __syncwarp();
  }
}

__global__ void k_red32(double* out) {
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < kIters; ++i) {
    const unsigned r = hash(blockIdx.x * 8192 + (threadIdx.x >> 5) * kIters * 2 + 2 * i) % kRows;
    const unsigned r2 = hash(blockIdx.x * 8192 + (threadIdx.x >> 5) * kIters * 2 + 2 * i + 1) % kRows;
    atomicAdd(out + r * 32ull + lane, 1.0);
    atomicAdd(out + r2 * 32ull + lane, 1.0);
  }
}

__global__ void k_bulk(double* out) {
  __shared__ __align__(128) double slot[16][4][32];  // 16 groups x 4-deep ring x 256 B
  const int lane = threadIdx.x & 31, q = lane & 15, grp = threadIdx.x >> 4;
  for (int i = 0; i < kIters; ++i) {
    const unsigned r = hash(blockIdx.x * 8192 + grp * kIters + i) % kRows;
    double* s = slot[grp][i & 3];
    if (q == 0 && i >= 4) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    __syncwarp();
    s[q] = 1.0;
    s[q + 16] = 1.0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (q == 0) {
      const unsigned src = static_cast<unsigned>(__cvta_generic_to_shared(s));
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 256;"
                   :: "l"(out + r * 32ull), "r"(src) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (q == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  double* out;
  cudaMalloc(&out, kRows * 32ull * 8);
  cudaMemset(out, 0, kRows * 32ull * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double rows = 148.0 * 8 * 16 * kIters;  // committed rows per launch
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(a);
    k_red16<<<148 * 8, 256>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("red16: %.3f ms, %.1f Grows/s\n", ms, rows / (ms * 1e-3) / 1e9);
    k_red16_div<<<148 * 8, 256>>>(out);
    cudaEventRecord(a);
    k_red32<<<148 * 8, 256>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("red32: %.3f ms, %.1f Grows/s\n", ms, rows / (ms * 1e-3) / 1e9);
    cudaEventRecord(a);
    k_bulk<<<148 * 8, 256>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("bulk: %.3f ms, %.1f Grows/s\n", ms, rows / (ms * 1e-3) / 1e9);
  }
  double h[32];
  cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
  printf("check %s out[0]=%g\n", cudaGetErrorString(cudaGetLastError()), h[0]);
  return 0;
}
