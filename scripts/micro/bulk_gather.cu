// Microbenchmark: three ways to gather random 256-byte factor rows (R = 32
// fp64) of an L2-resident 12.8 MB matrix into an SM, two rows per element as
// in the N = 3 MTTKRP computing phase, each row consumed by a 16-lane group
// (lane q takes columns q and q + 16):
//   ldg    : 2 x LDG.64 per lane per row, 4 elements (8 rows) in flight per
//            16-lane group (the current k_mttkrp_sorted pattern);
//   bulk   : one elected lane per warp issues cp.async.bulk (UBLKCP) per row
//            into a per-warp shared-memory ring of S stages, an mbarrier per
//            stage with complete_tx; the warp reads the rows with LDS;
//   gather4: TMA tile::gather4 (UTMALDG) -- 4 rows per instruction from a 2-D
//            tensor map -- into the same ring.
// Prints rows/s per variant (CUDA events, after a warm-up) and a checksum that
// must agree across variants.  Under ncu compare
// l1tex__data_pipe_lsu_wavefronts.sum and the time per row.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int kRows = 50000;        // 50000 x 256 B = 12.8 MB, L2 resident
constexpr int kElemsPerWarp = 8192;  // elements per warp (2 rows each)
constexpr int kWarps = 8;
constexpr int kE = 4;                // elements per stage
constexpr int kS = 4;                // ring stages per warp
constexpr int kStageBytes = kE * 2 * 256;

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ unsigned row_of(unsigned warp_global, unsigned e, unsigned m) {
  return hash(warp_global * 2654435761u + e * 2u + m) % kRows;
}

__global__ void __launch_bounds__(256) k_ldg(const double* __restrict__ a, double* out) {
  const int lane = threadIdx.x & 31, q = lane & 15, grp = lane >> 4;
  const unsigned w = blockIdx.x * kWarps + (threadIdx.x >> 5);
  double s = 0;
  for (int e0 = grp * 4; e0 < kElemsPerWarp; e0 += 8) {
    double v[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double* p0 = a + row_of(w, e0 + u, 0) * 32ull;
      const double* p1 = a + row_of(w, e0 + u, 1) * 32ull;
      v[u][0] = __ldg(p0 + q);
      v[u][1] = __ldg(p0 + q + 16);
      v[u][2] = __ldg(p1 + q);
      v[u][3] = __ldg(p1 + q + 16);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) s += v[u][0] * v[u][2] + v[u][1] * v[u][3];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, int r0, int r1, int r2, int r3,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

template <bool G4>
__global__ void __launch_bounds__(256) k_ring(const double* __restrict__ a, const __grid_constant__ CUtensorMap map,
                                              double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[kWarps][kS];
  const int lane = threadIdx.x & 31, q = lane & 15, grp = lane >> 4, wid = threadIdx.x >> 5;
  const unsigned w = blockIdx.x * kWarps + wid;
  unsigned char* ring = smem + wid * kS * kStageBytes;
  if (lane == 0)
    for (int s = 0; s < kS; ++s) mbar_init(&bars[wid][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  constexpr int kStages = kElemsPerWarp / kE;
  auto issue = [&](int st) {
    const int slot = st % kS;
    unsigned char* dst = ring + slot * kStageBytes;
    uint64_t* bar = &bars[wid][slot];
    mbar_expect(bar, kStageBytes);
    const int e0 = st * kE;
    if constexpr (G4) {
      // rows of mode 0 for the 4 elements, then rows of mode 1
      gather4(dst, &map, row_of(w, e0, 0), row_of(w, e0 + 1, 0), row_of(w, e0 + 2, 0), row_of(w, e0 + 3, 0), bar);
      gather4(dst + 4 * 256, &map, row_of(w, e0, 1), row_of(w, e0 + 1, 1), row_of(w, e0 + 2, 1),
              row_of(w, e0 + 3, 1), bar);
    } else {
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        bulk_row(dst + u * 256, a + row_of(w, e0 + u, 0) * 32ull, bar);
        bulk_row(dst + (4 + u) * 256, a + row_of(w, e0 + u, 1) * 32ull, bar);
      }
    }
  };
  if (lane == 0)
    for (int st = 0; st < kS - 1; ++st) issue(st);
  double s = 0;
  for (int st = 0; st < kStages; ++st) {
    if (lane == 0 && st + kS - 1 < kStages) issue(st + kS - 1);
    const int slot = st % kS;
    mbar_wait(&bars[wid][slot], (st / kS) & 1);
    const double* r = reinterpret_cast<const double*>(ring + slot * kStageBytes);
#pragma unroll
    for (int u = grp; u < kE; u += 2) {
      const double* r0 = r + u * 32;
      const double* r1 = r + (4 + u) * 32;
      s += r0[q] * r1[q] + r0[q + 16] * r1[q + 16];
    }
    __syncwarp();
    // the slot is refilled by the async proxy after these generic reads
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int blocks_per_sm = argc > 1 ? std::atoi(argv[1]) : 2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * blocks_per_sm;
  double *a, *out;
  cudaMalloc(&a, size_t(kRows) * 256);
  cudaMalloc(&out, size_t(grid) * 256 * 8);
  std::vector<double> h(size_t(kRows) * 32);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1.0 + (i % 7) * 0.125;
  cudaMemcpy(a, h.data(), h.size() * 8, cudaMemcpyHostToDevice);

  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  CUtensorMap map{};
  cuuint64_t dims[2] = {32, kRows}, strides[1] = {256};
  cuuint32_t box[2] = {32, 1}, estr[2] = {1, 1};
  CUresult cr = reinterpret_cast<EncodeTiled>(fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, strides, box,
                                                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("tensor map encode: %d\n", int(cr));
  const size_t smem = size_t(kWarps) * kS * kStageBytes;
  cudaFuncSetAttribute(k_ring<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(k_ring<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const double rows = double(grid) * kWarps * kElemsPerWarp * 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto sum_out = [&] {
    std::vector<double> o(size_t(grid) * 256);
    cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
    double t = 0;
    for (double x : o) t += x;
    return t;
  };
  for (int v = 0; v < 3; ++v) {
    auto launch = [&] {
      if (v == 0) k_ldg<<<grid, 256>>>(a, out);
      if (v == 1) k_ring<false><<<grid, 256, smem>>>(a, map, out);
      if (v == 2) k_ring<true><<<grid, 256, smem>>>(a, map, out);
    };
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    std::printf("%-8s grid %d (%d/SM, smem %zu B): %.3f ms, %.2f G rows/s, %.1f ns/row/SM, checksum %.6e %s\n",
                v == 0 ? "ldg" : v == 1 ? "bulk" : "gather4", grid, blocks_per_sm, v ? smem : size_t(0), ms / 5,
                rows / (ms / 5 * 1e-3) / 1e9, (ms / 5 * 1e6) / (rows / sms), sum_out(), cudaGetErrorString(err));
  }
  return 0;
}
