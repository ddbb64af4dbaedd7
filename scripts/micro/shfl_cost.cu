// Microbenchmark: does SHFL consume L1 data-pipe (LSU) wavefronts on sm_100a?
// Compares a loop of 4 x SHFL.IDX per iteration against 1 x LDS.128 broadcast.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_shfl(const double* in, double* out, int iters) {
  double a = in[threadIdx.x], s = 0;
  unsigned lane = threadIdx.x & 31;
  for (int i = 0; i < iters; ++i) {
    const int src = (i + lane) & 15;
    s += __shfl_sync(0xffffffffu, a, src) * __shfl_sync(0xffffffffu, s, (src + 3) & 31);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lds(const double* in, double* out, int iters) {
  __shared__ double4 sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = make_double4(in[threadIdx.x], 1, 2, 3);
  __syncthreads();
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    const double4 x = sm[(i + (threadIdx.x >> 4)) & 63];  // two broadcast addresses per warp
    s += x.x * x.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double *in, *out;
  cudaMalloc(&in, 1024 * 8);
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaMemset(in, 0, 1024 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_shfl<<<148 * 8, 256>>>(in, out, 1 << 14);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("shfl: %.3f ms (%.2f shfl/clk/SM)\n", ms, 2.0 * (1 << 14) * 148 * 8 * 8 / (ms * 1e-3 * 1.965e9 * 148));
    cudaEventRecord(a);
    k_lds<<<148 * 8, 256>>>(in, out, 1 << 14);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("lds128: %.3f ms (%.2f lds/clk/SM)\n", ms, 1.0 * (1 << 14) * 148 * 8 * 8 / (ms * 1e-3 * 1.965e9 * 148));
  }
  return 0;
}
