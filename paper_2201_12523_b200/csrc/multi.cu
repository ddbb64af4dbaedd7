// multi.cu -- the multi-GPU partition inside the library (SURVEY.md 8e, 8b
// "Threading"): non-zero spans split across G devices, factor matrices
// replicated, each mode's partial M_n summed by NCCL over NVLink/NVSwitch.
//
// Two entry families share one per-rank step (dist_step):
//   * blco_comm_* + blco_dist_mttkrp_all: one process per GPU (torchrun,
//     MPI, ...).  The caller moves the 128-byte NCCL unique id between its
//     processes; every collective is issued here, on the communicator's own
//     stream, never through torch.
//   * blco_multi_*: one host thread drives G devices of this process (the
//     reference's threading model: mttkrp is called from one coordinating
//     thread).  ncclCommInitAll over the devices, group calls
//     around the per-device collectives.
//
// Per mode n the kernel of mode n runs on the compute stream; an event
// orders the collective of M_n on the communicator stream after it, so the
// reduction of mode n overlaps the kernel of mode n+1 (outputs are distinct
// buffers).  The only data-path exchange is that reduction: no collective
// inside the kernel (peer REDs would move ~360x the bytes of a
// reduce-scatter of M for Amazon-shaped tensors).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2", reusing the copy a
// host framework has already loaded) so the library has no link-time NCCL
// dependency and never pulls a second NCCL into a torch process.  G = 1 needs
// no NCCL at all.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.hpp"

namespace b200 {
namespace {

// ------------------------------------------------------------ NCCL at run time
struct NcclApi {
  void* handle = nullptr;
  std::string error;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

template <class F>
void bind(void* h, F*& f, const char* name) {
  f = reinterpret_cast<F*>(dlsym(h, name));
}

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    const char* env = std::getenv("BLCO_B200_NCCL");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      // a copy already in the process (a host framework's) is reused
      a.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (a.handle) break;
    }
    for (const char* n : names) {
      if (a.handle || !n) continue;
      a.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!a.handle) {
      a.error = std::string("b200: NCCL not found (dlopen libnccl.so.2): ") + (dlerror() ? dlerror() : "");
      return a;
    }
    bind(a.handle, a.GetUniqueId, "ncclGetUniqueId");
    bind(a.handle, a.CommInitRank, "ncclCommInitRank");
    bind(a.handle, a.CommInitAll, "ncclCommInitAll");
    bind(a.handle, a.CommDestroy, "ncclCommDestroy");
    bind(a.handle, a.AllReduce, "ncclAllReduce");
    bind(a.handle, a.ReduceScatter, "ncclReduceScatter");
    bind(a.handle, a.GroupStart, "ncclGroupStart");
    bind(a.handle, a.GroupEnd, "ncclGroupEnd");
    bind(a.handle, a.GetErrorString, "ncclGetErrorString");
    bind(a.handle, a.GetVersion, "ncclGetVersion");
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommInitAll || !a.CommDestroy || !a.AllReduce ||
        !a.ReduceScatter || !a.GroupStart || !a.GroupEnd || !a.GetErrorString)
      a.error = "b200: libnccl.so.2 lacks a required symbol";
    return a;
  }();
  if (!api.error.empty()) throw Status(BLCO_ENCCL, api.error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Status(BLCO_ENCCL, std::string("b200: ") + what + ": " + nccl().GetErrorString(r));
}

void check_status(int st) {
  if (st != BLCO_OK) throw Status(st, blco_last_error());
}

// BLCO_B200_NCCL_SINGLE=1 (read per call): a one-rank communicator still
// creates an NCCL communicator, so the per-mode collectives run through NCCL
// (a reduction over one rank is a copy).  It exercises the NCCL path --
// binding, communicator setup, enqueue on the collective stream, events --
// on a one-GPU box.
bool nccl_single() {
  const char* e = std::getenv("BLCO_B200_NCCL_SINGLE");
  return e && std::string(e) == "1";
}

}  // namespace
}  // namespace b200

// A communicator member: one device of a G-device group.  G = 1 has no NCCL
// communicator (the reduction is the identity) unless BLCO_B200_NCCL_SINGLE.
struct blco_comm {
  int device = 0;
  int nranks = 1;
  int rank = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;  // collectives
  std::vector<cudaEvent_t> ready;  // per mode: the kernel of mode n has finished
  cudaEvent_t done = nullptr;

  void init_stream() {
    b200::DeviceGuard dg(device);
    B200_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    B200_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  }
  cudaEvent_t ready_event(int mode) {
    while (static_cast<int>(ready.size()) <= mode) {
      cudaEvent_t e;
      B200_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ready.push_back(e);
    }
    return ready[mode];
  }
  ~blco_comm() {
    b200::DeviceGuard dg(device);
    for (cudaEvent_t e : ready) cudaEventDestroy(e);
    if (done) cudaEventDestroy(done);
    if (stream) cudaStreamDestroy(stream);
    if (comm) b200::nccl().CommDestroy(comm);
  }
};

namespace b200 {
namespace {

uint64_t shard_rows(uint64_t rows, int G) { return rows ? (rows + G - 1) / G : 0; }

// One rank's all-mode step, enqueued: the mode kernels of `local` into the
// zeroed partials d_outs[n] on `stream`, each followed on the communicator's
// stream by its reduction.  Group calls are the caller's (one thread driving
// several communicators must wrap the collectives of one mode in a group).
struct RankStep {
  const blco_tensor* local;
  const double* const* factors;
  uint64_t rank;
  blco_comm* comm;
  int reduce;
  int strategy;
  const blco_exec_config* cfg;
  double* const* outs;
  double* const* shards;
  cudaStream_t stream;
};

void zero_partials(const RankStep& s) {
  const blco_layout& l = s.local->layout;
  for (int n = 0; n < l.order; ++n) {
    const uint64_t rows = s.reduce == BLCO_REDUCE_SCATTER ? shard_rows(l.dims[n], s.comm->nranks) * s.comm->nranks
                                                          : l.dims[n];
    if (rows) B200_CUDA(cudaMemsetAsync(s.outs[n], 0, rows * s.rank * sizeof(double), s.stream));
  }
}

void mode_kernel(const RankStep& s, int n) {
  check_status(blco_mttkrp_device(s.local, s.factors, s.rank, n, s.strategy, s.cfg, s.outs[n], 1, s.stream,
                                  nullptr));
  B200_CUDA(cudaEventRecord(s.comm->ready_event(n), s.stream));
  B200_CUDA(cudaStreamWaitEvent(s.comm->stream, s.comm->ready_event(n), 0));
}

void mode_collective(const RankStep& s, int n) {
  blco_comm& c = *s.comm;
  const uint64_t rows = s.local->layout.dims[n];
  if (!c.comm) {  // one rank, no NCCL communicator
    if (s.reduce == BLCO_REDUCE_SCATTER && rows && s.shards && s.shards[n] != s.outs[n])
      B200_CUDA(cudaMemcpyAsync(s.shards[n], s.outs[n], rows * s.rank * sizeof(double), cudaMemcpyDeviceToDevice,
                                c.stream));
    return;
  }
  if (s.reduce == BLCO_REDUCE_SCATTER) {
    const uint64_t per = shard_rows(rows, c.nranks) * s.rank;
    if (per)
      nccl_check(nccl().ReduceScatter(s.outs[n], s.shards[n], per, ncclFloat64, ncclSum, c.comm, c.stream),
                 "ncclReduceScatter");
  } else if (rows) {
    nccl_check(nccl().AllReduce(s.outs[n], s.outs[n], rows * s.rank, ncclFloat64, ncclSum, c.comm, c.stream),
               "ncclAllReduce");
  }
}

void finish(const RankStep& s) {
  B200_CUDA(cudaEventRecord(s.comm->done, s.comm->stream));
  B200_CUDA(cudaStreamWaitEvent(s.stream, s.comm->done, 0));
}

void validate_step(const RankStep& s) {
  if (!s.local || !s.comm || !s.factors || !s.outs) throw_format("dist: null argument");
  if (s.local->device != s.comm->device) throw_format("dist: tensor and communicator are on different devices");
  if (s.reduce != BLCO_REDUCE_ALL && s.reduce != BLCO_REDUCE_SCATTER) throw_format("dist: unknown reduction");
  if (s.rank < 1) throw_format("factors: rank must be >= 1");
  if (s.cfg && s.cfg->deterministic) throw_format("b200: deterministic mode is single-device");
  for (int n = 0; n < s.local->layout.order; ++n) {
    if (!s.factors[n] || !s.outs[n]) throw_format("dist: null factor or output pointer");
    if (s.reduce == BLCO_REDUCE_SCATTER && (!s.shards || !s.shards[n]))
      throw_format("dist: reduce-scatter needs shard buffers");
  }
}

}  // namespace
}  // namespace b200

// A tensor partitioned over the G devices of this process.
struct blco_multi {
  std::vector<int> devices;
  std::vector<blco_tensor*> parts;
  std::vector<blco_comm*> comms;
  std::vector<cudaStream_t> streams;
  std::vector<uint64_t> begin, end;
  blco_layout layout{};
  ~blco_multi() {
    for (size_t g = 0; g < devices.size(); ++g) {
      b200::DeviceGuard dg(devices[g]);
      if (g < streams.size() && streams[g]) cudaStreamDestroy(streams[g]);
    }
    for (blco_tensor* p : parts) blco_tensor_free(p);
    for (blco_comm* c : comms) delete c;
  }
};

using namespace b200;

extern "C" {

int blco_nccl_version(int* version) {
  return guarded([&] {
    const NcclApi& a = nccl();
    *version = 0;
    if (a.GetVersion) nccl_check(a.GetVersion(version), "ncclGetVersion");
  });
}

int blco_comm_unique_id(uint8_t* id) {
  return guarded([&] {
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == BLCO_COMM_ID_BYTES, "NCCL unique id size");
    std::memcpy(id, &u, sizeof u);
  });
}

int blco_comm_init_rank(const uint8_t* id, int nranks, int rank, int device, blco_comm** out) {
  *out = nullptr;
  return guarded([&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw_format("comm: rank out of range");
    auto c = std::make_unique<blco_comm>();
    c->device = device, c->nranks = nranks, c->rank = rank;
    c->init_stream();
    if (nranks > 1 || nccl_single()) {
      ncclUniqueId u;
      if (nranks > 1) std::memcpy(&u, id, sizeof u);
      else nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");  // the lone rank is its own root
      DeviceGuard dg(device);
      nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    }
    *out = c.release();
  });
}

int blco_comm_init_all(const int* devices, int ndev, blco_comm** out) {
  return guarded([&] {
    if (ndev < 1) throw_format("comm: need at least one device");
    std::vector<ncclComm_t> raw(ndev, nullptr);
    if (ndev > 1 || nccl_single()) nccl_check(nccl().CommInitAll(raw.data(), ndev, devices), "ncclCommInitAll");
    for (int g = 0; g < ndev; ++g) {
      auto* c = new blco_comm;
      c->device = devices[g], c->nranks = ndev, c->rank = g, c->comm = raw[g];
      c->init_stream();
      out[g] = c;
    }
  });
}

void blco_comm_free(blco_comm* c) { delete c; }

int blco_dist_mttkrp_all(const blco_tensor* local, const double* const* d_factors, uint64_t rank, blco_comm* comm,
                         int reduce, int strategy, const blco_exec_config* cfg, double* const* d_outs,
                         double* const* d_shards, void* stream) {
  return guarded([&] {
    const RankStep s{local, d_factors, rank, comm, reduce, strategy, cfg, d_outs, d_shards,
                     static_cast<cudaStream_t>(stream)};
    validate_step(s);
    DeviceGuard dg(local->device);
    NvtxRange nv("dist mttkrp all modes");
    zero_partials(s);
    for (int n = 0; n < local->layout.order; ++n) {
      mode_kernel(s, n);
      mode_collective(s, n);
    }
    finish(s);
  });
}

// ---- one thread, G devices of this process
int blco_multi_create(const blco_tensor* t, const int* devices, int ndev, blco_multi** out) {
  *out = nullptr;
  return guarded([&] {
    if (!t || !devices || ndev < 1) throw_format("multi: need a tensor and at least one device");
    auto m = std::make_unique<blco_multi>();
    m->devices.assign(devices, devices + ndev);
    m->layout = t->layout;
    std::vector<uint64_t> bn(t->nblocks());
    for (uint64_t b = 0; b < t->nblocks(); ++b) bn[b] = t->offsets[b + 1] - t->offsets[b];
    m->begin.resize(ndev);
    m->end.resize(ndev);
    // contiguous nnz-balanced span ranges (1024-element spans, never across a block)
    check_status(blco_partition(bn.data(), bn.size(), mttkrp_tile_elems(), ndev, m->begin.data(), m->end.data()));
    for (int g = 0; g < ndev; ++g) {
      blco_tensor* p = nullptr;
      check_status(blco_tensor_slice(t, m->begin[g], m->end[g], devices[g], &p));
      m->parts.push_back(p);
      DeviceGuard dg(devices[g]);
      cudaStream_t s;
      B200_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
      m->streams.push_back(s);
    }
    m->comms.resize(ndev);
    check_status(blco_comm_init_all(devices, ndev, m->comms.data()));
    *out = m.release();
  });
}

int blco_multi_info(const blco_multi* m, int* ndev, uint64_t* elem_begin, uint64_t* elem_end) {
  return guarded([&] {
    *ndev = static_cast<int>(m->devices.size());
    for (size_t g = 0; g < m->devices.size(); ++g) {
      if (elem_begin) elem_begin[g] = m->begin[g];
      if (elem_end) elem_end[g] = m->end[g];
    }
  });
}

void blco_multi_free(blco_multi* m) { delete m; }

int blco_multi_mttkrp_all(blco_multi* m, const double* const* factors, uint64_t rank, int reduce, int strategy,
                          const blco_exec_config* cfg, double* const* outs, blco_multi_report* rep) {
  return guarded([&] {
    const int G = static_cast<int>(m->devices.size());
    const blco_layout& l = m->layout;
    const int N = l.order;
    if (reduce != BLCO_REDUCE_ALL && reduce != BLCO_REDUCE_SCATTER) throw_format("dist: unknown reduction");
    if (rank < 1) throw_format("factors: rank must be >= 1");
    for (int n = 0; n < N; ++n)
      if (!factors[n] || !outs[n]) throw_format("mttkrp: null factor or output pointer");
    NvtxRange nv("multi mttkrp all modes");
    // per device: replicated factors, partials (padded for reduce-scatter), shards
    struct Dev {
      std::vector<DevBuf<double>> f, part, shard;
      std::vector<const double*> fp;
      std::vector<double*> op, sp;
      cudaEvent_t t0 = nullptr, t1 = nullptr;
    };
    std::vector<Dev> d(G);
    uint64_t h2d = 0, d2h = 0;
    for (int g = 0; g < G; ++g) {
      DeviceGuard dg(m->devices[g]);
      Dev& x = d[g];
      x.f.resize(N), x.part.resize(N), x.shard.resize(N);
      for (int n = 0; n < N; ++n) {
        const uint64_t elems = l.dims[n] * rank;
        x.f[n].alloc(elems);
        if (elems)
          B200_CUDA(cudaMemcpyAsync(x.f[n].ptr, factors[n], elems * 8, cudaMemcpyHostToDevice, m->streams[g]));
        h2d += elems * 8;
        const uint64_t per = shard_rows(l.dims[n], G);
        x.part[n].alloc(reduce == BLCO_REDUCE_SCATTER ? per * G * rank : elems);
        x.shard[n].alloc(reduce == BLCO_REDUCE_SCATTER ? per * rank : 0);
        x.fp.push_back(x.f[n].ptr);
        x.op.push_back(x.part[n].ptr);
        x.sp.push_back(x.shard[n].ptr);
      }
      B200_CUDA(cudaEventCreate(&x.t0));
      B200_CUDA(cudaEventCreate(&x.t1));
      B200_CUDA(cudaEventRecord(x.t0, m->streams[g]));
    }
    std::vector<RankStep> steps;
    for (int g = 0; g < G; ++g)
      steps.push_back(RankStep{m->parts[g], d[g].fp.data(), rank, m->comms[g], reduce, strategy, cfg,
                               d[g].op.data(), d[g].sp.data(), m->streams[g]});
    for (int g = 0; g < G; ++g) {
      validate_step(steps[g]);
      DeviceGuard dg(m->devices[g]);
      zero_partials(steps[g]);
    }
    for (int n = 0; n < N; ++n) {
      for (int g = 0; g < G; ++g) {
        DeviceGuard dg(m->devices[g]);
        mode_kernel(steps[g], n);
      }
      // one thread drives G communicators: the collectives of one mode form a group
      if (G > 1) nccl_check(nccl().GroupStart(), "ncclGroupStart");
      for (int g = 0; g < G; ++g) {
        DeviceGuard dg(m->devices[g]);
        mode_collective(steps[g], n);
      }
      if (G > 1) nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    }
    for (int g = 0; g < G; ++g) {
      DeviceGuard dg(m->devices[g]);
      finish(steps[g]);
      B200_CUDA(cudaEventRecord(d[g].t1, m->streams[g]));
    }
    // results: the all-reduced M_n from device 0, or every device's row shard
    for (int n = 0; n < N; ++n) {
      const uint64_t per = shard_rows(l.dims[n], G);
      for (int g = 0; g < G; ++g) {
        DeviceGuard dg(m->devices[g]);
        uint64_t lo = 0, rows = l.dims[n];
        const double* src = d[g].part[n].ptr;
        if (reduce == BLCO_REDUCE_SCATTER) {
          lo = std::min<uint64_t>(l.dims[n], g * per);
          rows = std::min<uint64_t>(l.dims[n], lo + per) - lo;
          src = m->comms[g]->comm ? d[g].shard[n].ptr : d[g].part[n].ptr;  // reduce-scattered, or one rank's partial
        } else if (g > 0) {
          continue;
        }
        if (rows)
          B200_CUDA(cudaMemcpyAsync(outs[n] + lo * rank, src, rows * rank * 8, cudaMemcpyDeviceToHost,
                                    m->streams[g]));
        d2h += rows * rank * 8;
      }
    }
    float worst = 0.0f;
    for (int g = 0; g < G; ++g) {
      DeviceGuard dg(m->devices[g]);
      B200_CUDA(cudaStreamSynchronize(m->streams[g]));
      float ms = 0.0f;
      B200_CUDA(cudaEventElapsedTime(&ms, d[g].t0, d[g].t1));
      worst = std::max(worst, ms);
      cudaEventDestroy(d[g].t0);
      cudaEventDestroy(d[g].t1);
    }
    if (rep) {
      rep->devices = G;
      rep->device_ms = worst;
      rep->h2d_bytes = h2d;
      rep->d2h_bytes = d2h;
    }
  });
}

}  // extern "C"
