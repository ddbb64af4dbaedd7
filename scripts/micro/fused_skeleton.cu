// Microbenchmark (decision probe for an all-mode fused MTTKRP): the memory
// skeleton of one all-mode step over NELL-2-shaped factors (12092, 9184,
// 28818 rows of R = 32 fp64, L2 resident), without staging:
//   sep  : three launches, one per target mode; per element the two
//          non-target rows are gathered (16-lane groups, lane q takes columns
//          q and q+16), the product accumulates, and every 3rd element
//          commits a 256-byte row with RED (0.32 segments / nnz measured on
//          NELL-2 with CTA bucket grouping);
//   fused: one launch; per element all three rows are gathered once, the
//          three products formed, the grouped mode commits every 3rd element,
//          the other two modes commit every element.
// Rows are drawn by hash (no ALTO locality), so absolute times are not the
// kernel's; the ratio fused / sep is the question.
#include <cuda_runtime.h>

#include <cstdio>

__constant__ int kDims[3] = {12092, 9184, 28818};
constexpr int kHostDims[3] = {12092, 9184, 28818};
constexpr int kElemsPerGroup = 4096;

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ unsigned row_of(unsigned e, int m) { return hash(e * 3u + m) % kDims[m]; }

struct Args {
  const double* f[3];
  double* out[3];
};

__global__ void __launch_bounds__(256) k_sep(Args a, int mode) {
  const int lane = threadIdx.x & 31, q = lane & 15;
  const unsigned grp = (blockIdx.x * 256 + threadIdx.x) >> 4;
  const int m1 = mode == 0 ? 1 : 0, m2 = mode == 2 ? 1 : 2;
  double acc0 = 0, acc1 = 0;
  for (int e0 = 0; e0 < kElemsPerGroup; e0 += 4) {
    double v[4][4];
    unsigned rows[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned e = grp * kElemsPerGroup + e0 + u;
      const double* p1 = a.f[m1] + row_of(e, m1) * 32ull;
      const double* p2 = a.f[m2] + row_of(e, m2) * 32ull;
      rows[u] = row_of(e, mode);
      v[u][0] = __ldg(p1 + q), v[u][1] = __ldg(p1 + q + 16), v[u][2] = __ldg(p2 + q), v[u][3] = __ldg(p2 + q + 16);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc0 += v[u][0] * v[u][2];
      acc1 += v[u][1] * v[u][3];
      if ((e0 + u) % 3 == 2) {
        double* o = a.out[mode] + rows[u] * 32ull;
        atomicAdd(o + q, acc0);
        atomicAdd(o + q + 16, acc1);
        acc0 = acc1 = 0;
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_fused(Args a) {
  const int lane = threadIdx.x & 31, q = lane & 15;
  const unsigned grp = (blockIdx.x * 256 + threadIdx.x) >> 4;
  double g0 = 0, g1 = 0;
  for (int e0 = 0; e0 < kElemsPerGroup; e0 += 4) {
    double v[4][6];
    unsigned r[4][3];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned e = grp * kElemsPerGroup + e0 + u;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        r[u][m] = row_of(e, m);
        const double* p = a.f[m] + r[u][m] * 32ull;
        v[u][2 * m] = __ldg(p + q);
        v[u][2 * m + 1] = __ldg(p + q + 16);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // mode 0 grouped (accumulated, commit every 3rd), modes 1 and 2 per element
      g0 += v[u][2] * v[u][4];
      g1 += v[u][3] * v[u][5];
      double* o1 = a.out[1] + r[u][1] * 32ull;
      atomicAdd(o1 + q, v[u][0] * v[u][4]);
      atomicAdd(o1 + q + 16, v[u][1] * v[u][5]);
      double* o2 = a.out[2] + r[u][2] * 32ull;
      atomicAdd(o2 + q, v[u][0] * v[u][2]);
      atomicAdd(o2 + q + 16, v[u][1] * v[u][3]);
      if ((e0 + u) % 3 == 2) {
        double* o0 = a.out[0] + r[u][0] * 32ull;
        atomicAdd(o0 + q, g0);
        atomicAdd(o0 + q + 16, g1);
        g0 = g1 = 0;
      }
    }
  }
}

int main() {
  Args a;
  for (int m = 0; m < 3; ++m) {
    double* p;
    cudaMalloc(&p, size_t(kHostDims[m]) * 256);
    cudaMemset(p, 0, size_t(kHostDims[m]) * 256);
    a.f[m] = p;
    cudaMalloc(&a.out[m], size_t(kHostDims[m]) * 256);
    cudaMemset(a.out[m], 0, size_t(kHostDims[m]) * 256);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4;
  const double elems = double(grid) * 16 * kElemsPerGroup;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    for (int m = 0; m < 3; ++m) k_sep<<<grid, 256>>>(a, m);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms_sep = 0;
    cudaEventElapsedTime(&ms_sep, e0, e1);
    cudaEventRecord(e0);
    k_fused<<<grid, 256>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms_f = 0;
    cudaEventElapsedTime(&ms_f, e0, e1);
    std::printf("elements %.0f: sep (3 launches) %.3f ms = %.2f ns/elem; fused %.3f ms = %.2f ns/elem; ratio %.3f (%s)\n",
                elems, ms_sep, ms_sep * 1e6 / elems, ms_f, ms_f * 1e6 / elems, ms_f / ms_sep,
                cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
