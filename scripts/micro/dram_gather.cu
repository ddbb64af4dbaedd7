// Microbenchmark (decision probe for the DRAM-bound Amazon-shaped mode
// kernel): the memory skeleton of one MTTKRP mode whose factors exceed L2.
// Per element two factor rows (R = 32 fp64, 256 B) are gathered from two
// 1.8M-row matrices (460 MB each), multiplied, and the product row is
// committed with RED.E.ADD.F64 into a 4.8M-row output (1.2 GB), 16-lane
// groups (lane q: columns q and q + 16), 4 elements in flight per group.
// Rows are drawn by hash, so there is no ALTO locality: absolute times are
// pessimistic, the ratios between variants are the question.
//   ldg    : both rows with LDG (the current k_mttkrp_sorted pattern);
//   hybrid : row A through TMA tile::gather4 (4 rows per instruction, one
//            elected lane per warp, mbarrier-gated ring of S stages in shared
//            memory), row B with LDG -- a third of the L1->XBAR line requests
//            per element move to the TMA unit;
//   g4     : both rows through gather4.
// ncu: l1tex__m_l1tex2xbar_req_cycles_active (the Amazon kernel's 88%
// limiter), l1tex__data_pipe_lsu_wavefronts, dram__bytes.
//   bulkred: LDG gathers, each product row committed by a 256-byte TMA bulk
//            reduction (cp.reduce.async.bulk .add.f64) from shared memory.
// Usage: dram_gather [blocks_per_sm] [variant mask] [row span]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>

constexpr unsigned kRowsA = 1800000, kRowsB = 1800000, kRowsM = 4800000;
constexpr int kElemsPerGroup = 2048;
constexpr int kWarps = 8;
constexpr int kE = 4;  // elements per group per stage
constexpr int kS = 4;  // ring stages

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__device__ __forceinline__ unsigned rowx(unsigned g, unsigned e, unsigned m, unsigned n) {
  return hash(g * 2654435761u + e * 3u + m) % n;
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
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, unsigned r0, unsigned r1, unsigned r2,
                                        unsigned r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void red2(double* p, double a) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(a) : "memory");
}
__device__ __forceinline__ void bulk_red_row(double* dst, const void* src) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 256;" ::"l"(dst),
               "r"(smem_u32(src))
               : "memory");
}

// V = 0 ldg, 1 hybrid, 2 g4, 3 ldg + TMA bulk-reduce commits
template <int V>
__global__ void __launch_bounds__(256) k_mode(const double* __restrict__ A, const double* __restrict__ B,
                                              const __grid_constant__ CUtensorMap mapA,
                                              const __grid_constant__ CUtensorMap mapB, double* M, unsigned nA,
                                              unsigned nB, unsigned nM) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[kWarps][kS];
  constexpr int kRowsPerStage = (V == 2 ? 2 : 1) * 2 * kE;  // rows per warp per stage
  constexpr int kStageBytes = kRowsPerStage * 256;
  const int lane = threadIdx.x & 31, q = lane & 15, grp = lane >> 4, wid = threadIdx.x >> 5;
  const unsigned gg = (blockIdx.x * kWarps + wid) * 2 + grp;  // global group id
  constexpr int kStages = kElemsPerGroup / kE;
  unsigned char* ring = smem + wid * kS * kStageBytes;
  if constexpr (V == 1 || V == 2) {
    if (lane == 0)
      for (int s = 0; s < kS; ++s) mbar_init(&bars[wid][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
  }
  const unsigned g0 = gg & ~1u;  // group 0 of this warp (lane 0 issues for both)
  auto issue = [&](int st) {
    const int slot = st % kS;
    unsigned char* dst = ring + slot * kStageBytes;
    uint64_t* bar = &bars[wid][slot];
    mbar_expect(bar, kStageBytes);
    const int e0 = st * kE;
    for (int h = 0; h < 2; ++h) {
      gather4(dst + h * kE * 256, &mapA, rowx(g0 + h, e0, 0, nA), rowx(g0 + h, e0 + 1, 0, nA),
              rowx(g0 + h, e0 + 2, 0, nA), rowx(g0 + h, e0 + 3, 0, nA), bar);
      if constexpr (V == 2)
        gather4(dst + (2 + h) * kE * 256, &mapB, rowx(g0 + h, e0, 1, nB), rowx(g0 + h, e0 + 1, 1, nB),
                rowx(g0 + h, e0 + 2, 1, nB), rowx(g0 + h, e0 + 3, 1, nB), bar);
    }
  };
  if constexpr (V == 1 || V == 2)
    if (lane == 0)
      for (int st = 0; st < kS - 1; ++st) issue(st);
  for (int st = 0; st < kStages; ++st) {
    const int e0 = st * kE;
    double a[kE][2], b[kE][2];
    if constexpr (V == 1 || V == 2)
      if (lane == 0 && st + kS - 1 < kStages) issue(st + kS - 1);
    if constexpr (V < 2 || V == 3) {
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const double* pb = B + rowx(gg, e0 + u, 1, nB) * 32ull;
        b[u][0] = __ldg(pb + q), b[u][1] = __ldg(pb + q + 16);
      }
    }
    if constexpr (V == 0 || V == 3) {
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const double* pa = A + rowx(gg, e0 + u, 0, nA) * 32ull;
        a[u][0] = __ldg(pa + q), a[u][1] = __ldg(pa + q + 16);
      }
    } else {
      const int slot = st % kS;
      mbar_wait(&bars[wid][slot], (st / kS) & 1);
      const double* r = reinterpret_cast<const double*>(ring + slot * kStageBytes);
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        const double* ra = r + (grp * kE + u) * 32;
        a[u][0] = ra[q], a[u][1] = ra[q + 16];
        if constexpr (V == 2) {
          const double* rb = r + ((2 + grp) * kE + u) * 32;
          b[u][0] = rb[q], b[u][1] = rb[q + 16];
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if constexpr (V == 3) {
      // products staged as rows in a per-warp 2-stage ring, one elected lane
      // issues a 256-byte bulk reduction per row
      double* stg = reinterpret_cast<double*>(smem + wid * 2 * (2 * kE * 256)) + (st & 1) * (2 * kE * 32);
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        double* r = stg + (grp * kE + u) * 32;
        r[q] = a[u][0] * b[u][0];
        r[q + 16] = a[u][1] * b[u][1];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        for (int h = 0; h < 2; ++h)
          for (int u = 0; u < kE; ++u)
            bulk_red_row(M + rowx(g0 + h, e0 + u, 2, nM) * 32ull, stg + (h * kE + u) * 32);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
#pragma unroll
      for (int u = 0; u < kE; ++u) {
        double* pm = M + rowx(gg, e0 + u, 2, nM) * 32ull;
        red2(pm + q, a[u][0] * b[u][0]);
        red2(pm + q + 16, a[u][1] * b[u][1]);
      }
    }
  }
  if constexpr (V == 3)
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int per_sm = argc > 1 ? std::atoi(argv[1]) : 3;
  const int mask = argc > 2 ? std::atoi(argv[2]) : 7;
  // rows drawn from the first `span` rows of each matrix (default: all; a
  // small span keeps the gathers and commits in L2)
  const unsigned span = argc > 3 ? unsigned(std::atoi(argv[3])) : kRowsM;
  const unsigned nA = std::min(span, kRowsA), nB = std::min(span, kRowsB), nM = std::min(span, kRowsM);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * per_sm;
  double *A, *B, *M;
  cudaMalloc(&A, size_t(nA) * 256);
  cudaMalloc(&B, size_t(nB) * 256);
  cudaMalloc(&M, size_t(nM) * 256);
  std::vector<double> h(size_t(nA) * 32);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1.0 + (i % 7) * 0.125;
  cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  CUtensorMap mapA{}, mapB{};
  cuuint64_t dA[2] = {32, nA}, dB[2] = {32, nB}, strides[1] = {256};
  cuuint32_t box[2] = {32, 1}, estr[2] = {1, 1};
  auto enc = reinterpret_cast<EncodeTiled>(fn);
  CUresult c1 = enc(&mapA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dA, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult c2 = enc(&mapB, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, B, dB, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::printf("tensor map encode: %d %d\n", int(c1), int(c2));
  const size_t sm1 = size_t(kWarps) * kS * 2 * kE * 256, sm2 = 2 * sm1;
  cudaFuncSetAttribute(k_mode<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm1));
  cudaFuncSetAttribute(k_mode<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm2));
  const size_t sm3 = size_t(kWarps) * 2 * 2 * kE * 256;
  const double elems = double(grid) * kWarps * 2 * kElemsPerGroup;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < 4; ++v) {
    if (!(mask & (1 << v))) continue;
    auto launch = [&] {
      if (v == 0) k_mode<0><<<grid, 256>>>(A, B, mapA, mapB, M, nA, nB, nM);
      if (v == 1) k_mode<1><<<grid, 256, sm1>>>(A, B, mapA, mapB, M, nA, nB, nM);
      if (v == 2) k_mode<2><<<grid, 256, sm2>>>(A, B, mapA, mapB, M, nA, nB, nM);
      if (v == 3) k_mode<3><<<grid, 256, sm3>>>(A, B, mapA, mapB, M, nA, nB, nM);
    };
    cudaMemset(M, 0, size_t(nM) * 256);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<double> o(4096);
    cudaMemcpy(o.data(), M, o.size() * 8, cudaMemcpyDeviceToHost);
    double cs = 0;
    for (double x : o) cs += x;
    const cudaError_t err = cudaGetLastError();
    std::printf("span %u %-7s %d/SM: %.3f ms, %.2f G elem/s (%.2f G rows/s gathered), checksum %.6e %s\n",
                span, v == 0 ? "ldg" : v == 1 ? "hybrid" : v == 2 ? "g4" : "bulkred", per_sm, ms / 3, elems / (ms / 3 * 1e-3) / 1e9,
                2 * elems / (ms / 3 * 1e-3) / 1e9, cs, cudaGetErrorString(err));
  }
  return 0;
}
