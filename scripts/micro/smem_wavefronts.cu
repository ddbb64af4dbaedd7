// Microbenchmark: shared-memory data-pipe wavefronts per warp instruction on
// sm_100a for the access patterns of the MTTKRP staging (run under ncu with
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_{ld,st}.sum and
// smsp__inst_executed_op_shared_{ld,st}.sum).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 1024;

// 16 lanes read record A, 16 lanes record A + h (h = 1 mod 4): LDS.128 broadcast x2
__global__ void k_ld128_two(const uint4* in, uint4* out) {
  __shared__ uint4 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = in[i];
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  const int g = (threadIdx.x & 31) >> 4, w = threadIdx.x >> 5;
  for (int i = 0; i < kIters; ++i) {
    const uint4 x = sm[(w * 128 + (i & 127) + g * 33) & 1023];
    acc.x ^= x.x, acc.y += x.y, acc.z ^= x.z, acc.w += x.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// all 32 lanes read one record: LDS.128 broadcast x1
__global__ void k_ld128_one(const uint4* in, uint4* out) {
  __shared__ uint4 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = in[i];
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  const int w = threadIdx.x >> 5;
  for (int i = 0; i < kIters; ++i) {
    const uint4 x = sm[(w * 128 + (i & 127)) & 1023];
    acc.x ^= x.x, acc.y += x.y, acc.z ^= x.z, acc.w += x.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// two half-warp broadcast LDS.64
__global__ void k_ld64_two(const double* in, double* out) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = in[i];
  __syncthreads();
  double acc = 0;
  const int g = (threadIdx.x & 31) >> 4, w = threadIdx.x >> 5;
  for (int i = 0; i < kIters; ++i) acc += sm[(w * 128 + (i & 127) + g * 33) & 1023];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// STS.128 of 32 distinct records at a pseudo-random permutation within a 1024 window
__global__ void k_st128_scatter(const uint4* in, uint4* out) {
  __shared__ uint4 sm[1024];
  const uint4 v = in[threadIdx.x];
  for (int i = 0; i < kIters; ++i) {
    const unsigned p = ((threadIdx.x + i * 97u) * 2654435761u >> 7) & 1023;
    sm[p] = v;
  }
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sm[threadIdx.x];
}

int main() {
  uint4 *in, *out;
  cudaMalloc(&in, 1024 * 16);
  cudaMalloc(&out, 148 * 256 * 16);
  cudaMemset(in, 1, 1024 * 16);
  k_ld128_two<<<148, 256>>>(in, out);
  k_ld128_one<<<148, 256>>>(in, out);
  k_ld64_two<<<148, 256>>>(reinterpret_cast<double*>(in), reinterpret_cast<double*>(out));
  k_st128_scatter<<<148, 256>>>(in, out);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
