// allmode.cu -- all-mode MTTKRP of a HOST-resident BLCO tensor with the
// upload pipelined under the compute (the end-to-end path of bench.py).
//
// Reference semantics: one call = mttkrp(t, f, n) for every mode n
// (proj/src/mttkrp.cpp:167-235), i.e. the "MTTKRP time/iter (all modes)"
// step of BASELINE.json, with the tensor and factors in host memory on entry
// and every M_n in host memory on return.
//
// Pipeline (two CUDA streams, one device):
//   copy stream   : H2D of factors / tile table / block bases (one event),
//                   then the payload (idx, vals) in tile-aligned chunks, one
//                   event per chunk;
//   compute stream: zero M_n, wait(tables), then per chunk c: wait(event c),
//                   K4 for every mode over the chunk's tiles (accumulating
//                   into M_n), and finally D2H of every M_n.
// The link is the bound (16 B/nnz over PCIe/C2C against ~9 ms of compute for
// NELL-2), so the step costs ~ H2D(payload) + one chunk's compute + D2H(M).
// Each chunk's idx/vals are re-read by the N mode launches right after they
// land, mostly out of L2.  Device buffers are cached per calling thread and
// grow only, so a steady-state call does no cudaMalloc.
#include <algorithm>
#include <cstring>

#include "internal.hpp"

namespace b200 {
namespace {

struct AllModeCtx {
  int device = -1;
  cudaStream_t copy = nullptr, comp = nullptr;
  cudaEvent_t start = nullptr, stop = nullptr, tables = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  void* host_stage = nullptr;  // pinned staging of the tile table + block bases
  size_t host_cap = 0;
  DevBuf<uint64_t> idx;
  DevBuf<double> vals;
  DevBuf<uint32_t> base;
  DevBuf<TileDesc> tiles;
  std::vector<DevBuf<double>> fac, out;

  void release() {
    for (auto e : chunk_ev) cudaEventDestroy(e);
    chunk_ev.clear();
    if (start) cudaEventDestroy(start);
    if (stop) cudaEventDestroy(stop);
    if (tables) cudaEventDestroy(tables);
    if (host_stage) cudaFreeHost(host_stage);
    host_stage = nullptr;
    host_cap = 0;
    tables = nullptr;
    if (copy) cudaStreamDestroy(copy);
    if (comp) cudaStreamDestroy(comp);
    start = stop = nullptr;
    copy = comp = nullptr;
    idx.reset(), vals.reset(), base.reset(), tiles.reset();
    fac.clear(), out.clear();
    device = -1;
  }
  ~AllModeCtx() {
    // the CUDA context may already be gone at thread/process exit
    int d = 0;
    if (cudaGetDevice(&d) == cudaSuccess) release();
  }
};
thread_local AllModeCtx t_ctx;

template <class T>
void grow(DevBuf<T>& b, size_t n) {
  if (b.n < n) b.alloc(n);
}

AllModeCtx& context(int device) {
  AllModeCtx& c = t_ctx;
  if (c.device != device) {
    if (c.device >= 0) {
      DeviceGuard g(c.device);
      c.release();
    }
    B200_CUDA(cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking));
    B200_CUDA(cudaStreamCreateWithFlags(&c.comp, cudaStreamNonBlocking));
    B200_CUDA(cudaEventCreate(&c.start));
    B200_CUDA(cudaEventCreate(&c.stop));
    B200_CUDA(cudaEventCreateWithFlags(&c.tables, cudaEventDisableTiming));
    c.device = device;
  }
  return c;
}

}  // namespace

void release_allmode_cache() {
  if (t_ctx.device >= 0) {
    DeviceGuard g(t_ctx.device);
    t_ctx.release();
  }
}

}  // namespace b200

using namespace b200;

extern "C" int blco_mttkrp_all_host(const blco_layout* layout, uint64_t nblocks, const uint64_t* keys,
                                    const uint64_t* block_nnz, const uint64_t* const* idx,
                                    const double* const* vals, const double* const* factors,
                                    uint64_t rank, int strategy, const blco_exec_config* cfg,
                                    uint64_t chunk_elems, int device, double* const* outs,
                                    int outs_on_device, blco_all_modes_report* report) {
  return guarded([&] {
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    if (blco_exec_config_validate(&c) != BLCO_OK) throw_format(blco_last_error());
    // rejected before any copy is queued (the per-chunk launches would throw
    // with the caller's buffers still in flight)
    if (c.deterministic) throw_format("b200: deterministic mode needs a device-resident tensor (not the streamed paths)");
    if (!layout) throw_format("mttkrp: null layout");
    const blco_layout& l = *layout;
    check_device_layout(l);
    if (rank < 1) throw_format("factors: rank must be >= 1");
    const int N = l.order;
    for (int m = 0; m < N; ++m)
      if (!factors[m] || !outs[m]) throw_format("mttkrp: null factor or output pointer");

    // ---- host-side plan: offsets, tile table, block bases, chunks
    const uint32_t tile = mttkrp_tile_elems();
    std::vector<uint64_t> off(nblocks + 1, 0);
    for (uint64_t b = 0; b < nblocks; ++b) off[b + 1] = off[b] + block_nnz[b];
    const uint64_t nnz = off[nblocks];
    std::vector<TileDesc> ht;
    ht.reserve(nnz / tile + nblocks + 1);
    for (uint64_t b = 0; b < nblocks; ++b)
      for (uint64_t o = off[b]; o < off[b + 1]; o += tile)
        ht.push_back(TileDesc{o, static_cast<uint32_t>(std::min<uint64_t>(tile, off[b + 1] - o)),
                              static_cast<uint32_t>(b)});
    std::vector<uint32_t> hbase(std::max<uint64_t>(1, nblocks * N));
    for (uint64_t b = 0; b < nblocks; ++b)
      for (int m = 0; m < N; ++m)
        hbase[b * N + m] = static_cast<uint32_t>(key_upper(l, m, keys[b]) << l.rem_bits[m]);
    // chunk = run of whole tiles holding ~chunk_elems elements.  With the
    // automatic size the last chunks shrink geometrically (down to 2^16
    // elements): only the final chunk's kernels run after the last byte has
    // crossed the link, so a small tail keeps the step close to the link time.
    const bool auto_chunks = chunk_elems == 0;
    if (auto_chunks) chunk_elems = std::max<uint64_t>(uint64_t{1} << 20, (nnz + 31) / 32);
    std::vector<std::pair<uint64_t, uint64_t>> chunks;  // tile ranges
    uint64_t done = 0;
    for (uint64_t t0 = 0; t0 < ht.size();) {
      uint64_t target = chunk_elems;
      if (auto_chunks) {
        const uint64_t left = nnz - done;
        while (target > (uint64_t{1} << 16) && target > left / 2) target /= 2;
      }
      uint64_t t1 = t0, e = 0;
      while (t1 < ht.size() && (t1 == t0 || e + ht[t1].count <= target)) e += ht[t1++].count;
      chunks.emplace_back(t0, t1);
      done += e;
      t0 = t1;
    }

    DeviceGuard dg(device);
    NvtxRange nv("mttkrp all modes (host pipeline)");
    AllModeCtx& x = context(device);
    grow(x.idx, nnz);
    grow(x.vals, nnz);
    grow(x.base, hbase.size());
    grow(x.tiles, std::max<size_t>(1, ht.size()));
    x.fac.resize(N);
    x.out.resize(N);
    for (int m = 0; m < N; ++m) {
      grow(x.fac[m], l.dims[m] * rank);
      grow(x.out[m], l.dims[m] * rank);
    }
    while (x.chunk_ev.size() < chunks.size()) {
      cudaEvent_t e;
      B200_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      x.chunk_ev.push_back(e);
    }
    uint64_t h2d = 0, d2h = 0, launches0 = g_launches.load();

    // Staging of the small tables in pinned memory, so every copy below is
    // asynchronous.  Everything the kernels need besides the payload goes
    // first on the copy stream: copies of one direction are served in issue
    // order by the copy engine, so anything queued behind the payload chunks
    // would hold the first kernel back until the whole payload had landed.
    const size_t tile_bytes = ht.size() * sizeof(TileDesc), base_bytes = hbase.size() * 4;
    if (x.host_cap < tile_bytes + base_bytes) {
      if (x.host_stage) cudaFreeHost(x.host_stage);
      x.host_stage = nullptr;
      x.host_cap = 0;
      B200_CUDA(cudaHostAlloc(&x.host_stage, tile_bytes + base_bytes, cudaHostAllocPortable));
      x.host_cap = tile_bytes + base_bytes;
    }
    B200_CUDA(cudaEventRecord(x.start, x.comp));
    B200_CUDA(cudaStreamWaitEvent(x.copy, x.start, 0));  // the previous call's D2H / kernels are done
    std::memcpy(x.host_stage, ht.data(), tile_bytes);
    std::memcpy(static_cast<char*>(x.host_stage) + tile_bytes, hbase.data(), base_bytes);
    std::vector<const double*> fptr(N);
    for (int m = 0; m < N; ++m) {
      const uint64_t n = l.dims[m] * rank;
      B200_CUDA(cudaMemcpyAsync(x.fac[m].ptr, factors[m], n * 8, cudaMemcpyHostToDevice, x.copy));
      B200_CUDA(cudaMemsetAsync(x.out[m].ptr, 0, n * 8, x.comp));
      fptr[m] = x.fac[m].ptr;
      h2d += n * 8;
    }
    if (!ht.empty()) {
      B200_CUDA(cudaMemcpyAsync(x.tiles.ptr, x.host_stage, tile_bytes, cudaMemcpyHostToDevice, x.copy));
      B200_CUDA(cudaMemcpyAsync(x.base.ptr, static_cast<char*>(x.host_stage) + tile_bytes, base_bytes,
                                cudaMemcpyHostToDevice, x.copy));
      h2d += tile_bytes + base_bytes;
    }
    B200_CUDA(cudaEventRecord(x.tables, x.copy));
    // payload chunks
    for (size_t k = 0; k < chunks.size(); ++k) {
      const uint64_t e0 = ht[chunks[k].first].start;
      const uint64_t e1 = ht[chunks[k].second - 1].start + ht[chunks[k].second - 1].count;
      for (uint64_t b = ht[chunks[k].first].block; b < nblocks && off[b] < e1; ++b) {
        const uint64_t lo = std::max(e0, off[b]), hi = std::min(e1, off[b + 1]);
        if (lo >= hi) continue;
        B200_CUDA(cudaMemcpyAsync(x.idx.ptr + lo, idx[b] + (lo - off[b]), (hi - lo) * 8,
                                  cudaMemcpyHostToDevice, x.copy));
        B200_CUDA(cudaMemcpyAsync(x.vals.ptr + lo, vals[b] + (lo - off[b]), (hi - lo) * 8,
                                  cudaMemcpyHostToDevice, x.copy));
        h2d += (hi - lo) * 16;
      }
      B200_CUDA(cudaEventRecord(x.chunk_ev[k], x.copy));
    }
    B200_CUDA(cudaStreamWaitEvent(x.comp, x.tables, 0));
    std::vector<int> strat(N);
    for (int m = 0; m < N; ++m)
      strat[m] = strategy == BLCO_STRATEGY_AUTO ? auto_kernel(l.dims[m], c) : strategy;
    for (size_t k = 0; k < chunks.size(); ++k) {
      B200_CUDA(cudaStreamWaitEvent(x.comp, x.chunk_ev[k], 0));
      for (int m = 0; m < N; ++m) {
        MttkrpLaunch a{};
        a.view.layout = &l;
        a.view.tiles = x.tiles.ptr + chunks[k].first;
        a.view.ntiles = chunks[k].second - chunks[k].first;
        a.view.elem_end = nnz;
        a.view.idx = x.idx.ptr;
        a.view.vals = x.vals.ptr;
        a.view.block_base = x.base.ptr;
        a.factors = fptr.data();
        a.rank = rank;
        a.mode = m;
        a.strategy = strat[m];
        a.cfg = c;
        a.out = x.out[m].ptr;
        a.accumulate = 1;
        a.stream = x.comp;
        mttkrp_enqueue(a);
      }
    }
    for (int m = 0; m < N; ++m) {
      const uint64_t n = l.dims[m] * rank;
      if (outs_on_device) {
        B200_CUDA(cudaMemcpyAsync(outs[m], x.out[m].ptr, n * 8, cudaMemcpyDeviceToDevice, x.comp));
      } else {
        B200_CUDA(cudaMemcpyAsync(outs[m], x.out[m].ptr, n * 8, cudaMemcpyDeviceToHost, x.comp));
        d2h += n * 8;
      }
    }
    B200_CUDA(cudaEventRecord(x.stop, x.comp));
    B200_CUDA(cudaStreamSynchronize(x.comp));
    if (report) {
      float ms = 0;
      B200_CUDA(cudaEventElapsedTime(&ms, x.start, x.stop));
      report->device_ms = ms;
      report->chunks = chunks.size();
      report->h2d_bytes = h2d;
      report->d2h_bytes = d2h;
      report->launches = g_launches.load() - launches0;
    }
  });
}
