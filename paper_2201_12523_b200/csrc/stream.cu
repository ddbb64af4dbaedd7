// stream.cu -- out-of-memory BLCO MTTKRP: blocks stream from host memory
// through per-queue device reservations on Q CUDA streams (K6).
//
// Reference: stream_mttkrp, proj/src/streaming.cpp:103-309.  Same budget
// arithmetic (:117-136), same round-robin queue assignment (:265), same
// rejection of a block larger than its queue reservation before it is
// transferred (:257-264), same report fields (:292-307).  What is real here
// and simulated there: capacity_bytes caps actual cudaMalloc'd bytes, a
// "transfer" is a cudaMemcpyAsync H2D into the queue's reservation and a
// "compute" is the MTTKRP kernel on the same stream, so block b+1's copy
// (queue (b+1) % Q) overlaps block b's kernel (queue b % Q).  Timeline
// intervals come from CUDA events.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <fcntl.h>
#include <unistd.h>

#include <condition_variable>
#include <deque>
#include <map>
#include <tuple>
#include <thread>

#include "internal.hpp"

namespace b200 {
namespace {

__global__ void k_one_block_base(uint64_t key, int order, int kept, int total,
                                 const uint8_t* __restrict__ imap_mode,
                                 const uint8_t* __restrict__ imap_bit,
                                 const int32_t* __restrict__ rem, uint32_t* __restrict__ base) {
  if (threadIdx.x != 0) return;
  uint64_t up[BLCO_MAX_DEV_ORDER] = {};
  for (int p = kept; p < total; ++p) {
    const int m = imap_mode[p];
    up[m] |= ((key >> (p - kept)) & 1u) << (imap_bit[p] - rem[m]);
  }
  for (int m = 0; m < order; ++m) base[m] = static_cast<uint32_t>(up[m] << rem[m]);
}

void CUDART_CB host_sleep(void* arg) {
  const double s = *static_cast<double*>(arg);
  std::this_thread::sleep_for(std::chrono::duration<double>(s));
}

struct Queue {
  cudaStream_t stream = nullptr;
  DevBuf<uint64_t> idx;
  DevBuf<double> vals;
  DevBuf<uint32_t> base;
  DevBuf<TileDesc> tiles;
  std::vector<TileDesc> htiles;  // host copy, alive while its upload is in flight
  uint64_t capacity = 0;  // elements
};

struct Interval {
  int kind, queue;
  uint64_t block;
  cudaEvent_t b, e;
};

double union_seconds(std::vector<std::pair<double, double>> iv) {
  std::sort(iv.begin(), iv.end());
  double total = 0, hi = -1;
  for (auto [b, e] : iv) {
    if (b > hi) {
      total += e - b;
      hi = e;
    } else if (e > hi) {
      total += e - hi;
      hi = e;
    }
  }
  return total;
}

// Where blocks come from: the caller's pull callback (BlockSource::next) or
// the native .blco file reader below.
struct BlockFeed {
  virtual ~BlockFeed() = default;
  // 1 = a block in *v, 0 = end of stream; errors throw Status
  virtual int next(blco_block_view& v) = 0;
  // the host->device copy of block `ordinal` is complete once `done` fires
  virtual void transferred(uint64_t ordinal, cudaEvent_t done) {
    (void)ordinal;
    (void)done;
  }
  // run read_blco_block's element checks on the transferred copy
  virtual bool validate() const { return false; }
  // the engine is done pulling (called before it releases its events)
  virtual void finish() {}
};

struct CallbackFeed final : BlockFeed {
  blco_block_source_fn fn;
  void* ctx;
  CallbackFeed(blco_block_source_fn f, void* c) : fn(f), ctx(c) {}
  int next(blco_block_view& v) override {
    const int r = fn(ctx, &v);
    if (r < 0) throw Status(-r, blco_last_error());
    return r;
  }
};

// Streams the blocks once and runs MTTKRP for every mode in modes[] on each
// resident block (one mode: stream_mttkrp; all modes: the all-mode
// extension, which moves the tensor over the host link once per iteration).
void stream_impl(const blco_layout* layout, uint64_t max_nnz_per_block, BlockFeed& feed,
                 const double* const* factors, uint64_t rank, const std::vector<int>& modes,
                 const blco_device_budget* budget, const blco_exec_config* cfg, int strategy_in,
                 int device, double* const* outs, bool outs_on_device, blco_stream_report* report) {
  {
    blco_exec_config c;
    if (cfg) c = *cfg; else blco_exec_config_default(&c);
    if (blco_exec_config_validate(&c) != BLCO_OK) throw_format(blco_last_error());
    const blco_layout& l = *layout;
    check_device_layout(l);
    if (rank < 1) throw_format("factors: rank must be >= 1");
    for (int mode : modes)
      if (mode < 0 || mode >= l.order) throw_format("stream: mode out of range");
    if (budget->num_queues < 1) throw_format("stream: num_queues must be >= 1");
    const int NM = static_cast<int>(modes.size());
    std::vector<int> strat(NM);
    std::vector<bool> hier(NM);
    std::vector<uint64_t> out_elems(NM);
    const int C = std::max(1, c.num_factor_copies);
    // Resident set: factors + outputs (+ copies), streaming.cpp:117-124.
    uint64_t pinned = 0;
    for (int m = 0; m < l.order; ++m) pinned += l.dims[m] * rank * sizeof(double);
    for (int k = 0; k < NM; ++k) {
      // the budget counts what the reference would keep resident (its
      // choose_strategy label: C output copies for a hierarchical mode), so
      // capacity errors match; Auto then runs the B200 kernel of choice
      const int label =
          strategy_in == BLCO_STRATEGY_AUTO ? blco_choose_strategy(l.dims[modes[k]], &c) : strategy_in;
      strat[k] = strategy_in == BLCO_STRATEGY_AUTO ? auto_kernel(l.dims[modes[k]], c) : strategy_in;
      hier[k] = strat[k] == BLCO_STRATEGY_HIERARCHICAL;
      out_elems[k] = l.dims[modes[k]] * rank;
      pinned += out_elems[k] * sizeof(double) * (label == BLCO_STRATEGY_HIERARCHICAL ? C : 1);
    }
    if (pinned > budget->capacity_bytes)
      throw_format("stream: factor matrices and output (" + std::to_string(pinned) +
                   " bytes) exceed device capacity " + std::to_string(budget->capacity_bytes));
    const int Q = budget->num_queues;
    uint64_t reservation = budget->reservation_bytes;
    if (reservation == 0) reservation = (budget->capacity_bytes - pinned) / Q;
    if (reservation < sizeof(uint64_t) + sizeof(double))
      throw_format("stream: budget leaves no room for a per-queue reservation");
    if (pinned + static_cast<uint64_t>(Q) * reservation > budget->capacity_bytes)
      throw_format("stream: reservations exceed device capacity");
    const uint64_t max_staged = reservation / (sizeof(uint64_t) + sizeof(double));
    const uint64_t resident = pinned + static_cast<uint64_t>(Q) * reservation;

    DeviceGuard dg(device);
    // factors + output
    std::vector<DevBuf<double>> df(l.order);
    std::vector<const double*> fptr(l.order);
    for (int m = 0; m < l.order; ++m) {
      df[m].alloc(l.dims[m] * rank);
      if (df[m].n) B200_CUDA(cudaMemcpy(df[m].ptr, factors[m], df[m].bytes(), cudaMemcpyHostToDevice));
      fptr[m] = df[m].ptr;
    }
    std::vector<DevBuf<double>> dout(NM), copies(NM);
    for (int k = 0; k < NM; ++k) {
      dout[k].alloc(out_elems[k]);
      copies[k].alloc(hier[k] ? out_elems[k] * C : 0);
      if (dout[k].n) B200_CUDA(cudaMemset(dout[k].ptr, 0, dout[k].bytes()));
      if (copies[k].n) B200_CUDA(cudaMemset(copies[k].ptr, 0, copies[k].bytes()));
    }
    DevBuf<uint8_t> dmode(BLCO_MAX_BITS), dbit(BLCO_MAX_BITS);
    DevBuf<int32_t> drem(BLCO_MAX_ORDER);
    B200_CUDA(cudaMemcpy(dmode.ptr, l.imap_mode, BLCO_MAX_BITS, cudaMemcpyHostToDevice));
    B200_CUDA(cudaMemcpy(dbit.ptr, l.imap_bit, BLCO_MAX_BITS, cudaMemcpyHostToDevice));
    B200_CUDA(cudaMemcpy(drem.ptr, l.rem_bits, sizeof(int32_t) * BLCO_MAX_ORDER, cudaMemcpyHostToDevice));

    // Reservations are allocated lazily at the size of the largest block seen
    // (bounded by the reservation), so capacity is a real cap.
    const uint32_t tile = mttkrp_tile_elems();
    std::vector<Queue> qs(Q);
    for (auto& q : qs) B200_CUDA(cudaStreamCreateWithFlags(&q.stream, cudaStreamNonBlocking));
    cudaEvent_t start, stop;
    B200_CUDA(cudaEventCreate(&start));
    B200_CUDA(cudaEventCreate(&stop));
    // zeroed before the device sync below: the queues are non-blocking
    // streams, not ordered after the legacy-stream memset
    DevBuf<unsigned> dbad(1);  // read_blco_block check bits of file-fed blocks
    B200_CUDA(cudaMemset(dbad.ptr, 0, sizeof(unsigned)));
    B200_CUDA(cudaDeviceSynchronize());
    B200_CUDA(cudaEventRecord(start, qs[0].stream));
    for (int q = 1; q < Q; ++q) B200_CUDA(cudaStreamWaitEvent(qs[q].stream, start, 0));

    std::vector<Interval> timeline;
    std::vector<int32_t> block_queue;
    std::vector<double> sleep_arg(1, budget->injected_transfer_latency_s);
    uint64_t ordinal = 0, bytes = 0;
    std::string err;
    int err_code = BLCO_OK;
    try {
      for (;;) {
        blco_block_view bv{};
        if (feed.next(bv) == 0) break;
        const uint64_t bbytes = bv.nnz * (sizeof(uint64_t) + sizeof(double));
        if (bbytes > reservation)
          throw_format("stream: block " + std::to_string(ordinal) + " (" + std::to_string(bbytes) +
                       " bytes) exceeds queue reservation " + std::to_string(reservation));
        if (bv.nnz > max_nnz_per_block && max_nnz_per_block)
          throw_format("blco: block exceeds max_nnz_per_block");
        const int qi = static_cast<int>(ordinal % Q);
        Queue& q = qs[qi];
        block_queue.push_back(qi);
        if (bv.nnz > q.capacity) {
          // grow this queue's reservation (waits for its stream first)
          B200_CUDA(cudaStreamSynchronize(q.stream));
          const uint64_t cap = std::min<uint64_t>(max_staged, std::max<uint64_t>(bv.nnz, 1));
          q.idx.alloc(cap);
          q.vals.alloc(cap);
          q.base.alloc(BLCO_MAX_DEV_ORDER);
          std::vector<TileDesc>& h = q.htiles;
          h.clear();
          for (uint64_t off = 0; off < cap; off += tile)
            h.push_back(TileDesc{off, static_cast<uint32_t>(std::min<uint64_t>(tile, cap - off)), 0u});
          q.tiles.alloc(h.size());
          // ordered on the queue's stream: a plain cudaMemcpy from pageable
          // memory returns once the data is staged, and the queue is a
          // non-blocking stream -- its kernels could read the table before
          // the DMA lands (seen as a wrong block every few calls with 3 queues)
          B200_CUDA(cudaMemcpyAsync(q.tiles.ptr, h.data(), h.size() * sizeof(TileDesc), cudaMemcpyHostToDevice,
                                    q.stream));
          q.capacity = cap;
        }
        NvtxRange nv("stream: block transfer + compute");
        Interval tr{0, qi, ordinal, nullptr, nullptr}, cp{1, qi, ordinal, nullptr, nullptr};
        B200_CUDA(cudaEventCreate(&tr.b));
        B200_CUDA(cudaEventCreate(&tr.e));
        B200_CUDA(cudaEventCreate(&cp.b));
        B200_CUDA(cudaEventCreate(&cp.e));
        timeline.push_back(tr);
        timeline.push_back(cp);
        B200_CUDA(cudaEventRecord(tr.b, q.stream));
        if (bv.nnz) {
          B200_CUDA(cudaMemcpyAsync(q.idx.ptr, bv.idx, bv.nnz * 8, cudaMemcpyHostToDevice, q.stream));
          B200_CUDA(cudaMemcpyAsync(q.vals.ptr, bv.vals, bv.nnz * 8, cudaMemcpyHostToDevice, q.stream));
        }
        k_one_block_base<<<1, 32, 0, q.stream>>>(bv.key, l.order, l.total_bits - l.stripped_bits,
                                                 l.total_bits, dmode.ptr, dbit.ptr, drem.ptr, q.base.ptr);
        count_launch();
        check_launch("k_one_block_base");
        if (budget->injected_transfer_latency_s > 0)
          B200_CUDA(cudaLaunchHostFunc(q.stream, host_sleep, sleep_arg.data()));
        B200_CUDA(cudaEventRecord(tr.e, q.stream));
        feed.transferred(ordinal, tr.e);
        if (feed.validate()) enqueue_block_check(l, bv.key, q.idx.ptr, bv.nnz, dbad.ptr, q.stream);
        // A block without BLCO_BLOCK_STABLE may be overwritten by the next
        // pull: wait until its copy has read the source.  This matters for
        // pinned sources above all -- a pinned cudaMemcpyAsync returns at once
        // and the DMA reads host memory later (a pageable one has already
        // staged the bytes on return, so its wait is nearly free).
        static const int dbg_sync = [] {
          const char* e = std::getenv("BLCO_B200_STREAM_SYNC");
          return e ? std::atoi(e) : 0;
        }();
        if ((dbg_sync & 1) || (bv.nnz && !(bv.flags & BLCO_BLOCK_STABLE)))
          B200_CUDA(cudaEventSynchronize(tr.e));

        B200_CUDA(cudaEventRecord(cp.b, q.stream));
        for (int k = 0; k < NM; ++k) {
          MttkrpLaunch a{};
          a.view.layout = &l;
          a.view.tiles = q.tiles.ptr;
          a.view.ntiles = (bv.nnz + tile - 1) / tile;
          a.view.elem_end = bv.nnz;
          a.view.idx = q.idx.ptr;
          a.view.vals = q.vals.ptr;
          a.view.block_base = q.base.ptr;
          a.factors = fptr.data();
          a.rank = rank;
          a.mode = modes[k];
          a.strategy = strat[k];
          a.cfg = c;
          a.out = dout[k].ptr;
          a.accumulate = 1;
          a.stream = q.stream;
          a.hier_copies = hier[k] ? copies[k].ptr : nullptr;
          mttkrp_enqueue(a);
        }
        B200_CUDA(cudaEventRecord(cp.e, q.stream));
        if (dbg_sync & 2) B200_CUDA(cudaEventSynchronize(cp.e));
        bytes += bbytes;
        ++ordinal;
      }
    } catch (const Status& s) {
      err = s.what();
      err_code = s.code;
    }
    for (auto& q : qs) B200_CUDA(cudaStreamSynchronize(q.stream));
    feed.finish();
    if (err_code == BLCO_OK && feed.validate()) {
      unsigned bad = 0;
      B200_CUDA(cudaMemcpy(&bad, dbad.ptr, sizeof bad, cudaMemcpyDeviceToHost));
      try {
        throw_block_check(bad);
      } catch (const Status& s) {
        err = s.what();
        err_code = s.code;
      }
    }
    if (err_code != BLCO_OK) {
      for (auto& iv : timeline) cudaEventDestroy(iv.b), cudaEventDestroy(iv.e);
      for (auto& q : qs) cudaStreamDestroy(q.stream);
      throw Status(err_code, err);
    }
    for (int q = 1; q < Q; ++q) {
      cudaEvent_t done;
      B200_CUDA(cudaEventCreate(&done));
      B200_CUDA(cudaEventRecord(done, qs[q].stream));
      B200_CUDA(cudaStreamWaitEvent(qs[0].stream, done, 0));
      cudaEventDestroy(done);
    }
    for (int k = 0; k < NM; ++k)
      if (hier[k]) merge_copies_enqueue(copies[k].ptr, out_elems[k], C, dout[k].ptr, 1, qs[0].stream);
    B200_CUDA(cudaEventRecord(stop, qs[0].stream));
    B200_CUDA(cudaStreamSynchronize(qs[0].stream));
    for (int k = 0; k < NM; ++k)
      if (out_elems[k])
        B200_CUDA(cudaMemcpy(outs[k], dout[k].ptr, dout[k].bytes(),
                             outs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));

    if (report) {
      float total_ms = 0;
      B200_CUDA(cudaEventElapsedTime(&total_ms, start, stop));
      std::vector<std::pair<double, double>> tr_iv, cp_iv;
      std::vector<blco_stream_event> evs;
      for (auto& iv : timeline) {
        float b = 0, e = 0;
        B200_CUDA(cudaEventElapsedTime(&b, start, iv.b));
        B200_CUDA(cudaEventElapsedTime(&e, start, iv.e));
        (iv.kind == 0 ? tr_iv : cp_iv).emplace_back(b * 1e-3, e * 1e-3);
        evs.push_back(blco_stream_event{iv.kind, iv.queue, iv.block, b * 1e-3, e * 1e-3});
      }
      std::sort(evs.begin(), evs.end(), [](const blco_stream_event& x, const blco_stream_event& y) {
        return x.begin_s < y.begin_s;
      });
      report->blocks = ordinal;
      report->bytes_streamed = bytes;
      report->total_seconds = total_ms * 1e-3;
      report->transfer_busy_seconds = union_seconds(tr_iv);
      report->compute_busy_seconds = union_seconds(cp_iv);
      const double gb = static_cast<double>(bytes) / 1e9;
      report->overall_gbps = report->total_seconds > 0 ? gb / report->total_seconds : 0;
      report->compute_gbps = report->compute_busy_seconds > 0 ? gb / report->compute_busy_seconds : 0;
      report->peak_resident_bytes = resident;
      if (report->block_queue)
        for (uint64_t i = 0; i < std::min<uint64_t>(report->block_queue_capacity, block_queue.size()); ++i)
          report->block_queue[i] = block_queue[i];
      report->timeline_count = evs.size();
      if (report->timeline)
        for (uint64_t i = 0; i < std::min<uint64_t>(report->timeline_capacity, evs.size()); ++i)
          report->timeline[i] = evs[i];
    }
    for (auto& iv : timeline) cudaEventDestroy(iv.b), cudaEventDestroy(iv.e);
    cudaEventDestroy(start);
    cudaEventDestroy(stop);
    for (auto& q : qs) cudaStreamDestroy(q.stream);
  }
}

// Pinned host slots of the file reader, kept for the next call: pinning
// gigabytes (cudaHostAlloc) costs seconds, far more than the read it serves.
class PinnedPool {
 public:
  static PinnedPool& get() {
    static PinnedPool* p = new PinnedPool;  // never destroyed: freed with the process
    return *p;
  }
  // a buffer of at least `bytes` (the largest free one that fits, else new)
  std::pair<void*, size_t> take(size_t bytes) {
    {
      std::lock_guard<std::mutex> g(mu_);
      auto it = free_.lower_bound(bytes);
      if (it != free_.end()) {
        auto r = std::make_pair(it->second, it->first);
        free_.erase(it);
        return r;
      }
    }
    void* mem = nullptr;
    B200_CUDA(cudaHostAlloc(&mem, bytes, cudaHostAllocPortable));
    return {mem, bytes};
  }
  void give(void* mem, size_t bytes) {
    if (!mem) return;
    std::lock_guard<std::mutex> g(mu_);
    free_.emplace(bytes, mem);
  }

 private:
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
};

// Native FileBlockSource (streaming.hpp:45-58, streaming.cpp:13-31): a
// reader thread reads each block record of a .blco container straight into a
// ring of pinned host slots while earlier blocks are copied and multiplied; a
// slot is refilled only after the engine reports that the copy of the block
// it held has completed.  read_blco_block's record checks (key range, empty
// record, capacity, ascending keys; blco_format.cpp:201-238) run here, its
// per-element checks on the device on the transferred copy -- the block
// crosses the link once.
class FileFeed final : public BlockFeed {
 public:
  FileFeed(const char* path, int device, int nslots) : device_(device), slots_(nslots) {
    f_ = std::fopen(path, "rb");
    if (!f_) throw Status(BLCO_EIO, std::string("cannot open ") + path);
    try {
      h_ = read_blco_file_header(f_);
    } catch (...) {
      std::fclose(f_);
      throw;
    }
    fd_ = ::open(path, O_RDONLY);
    if (fd_ < 0) {
      std::fclose(f_);
      throw Status(BLCO_EIO, std::string("cannot open ") + path);
    }
    pos_ = 4 + 2 + 2 + 8 * static_cast<uint64_t>(h_.layout.order) + 2 + 2 * static_cast<uint64_t>(h_.layout.order) +
           8 + 8;
    const unsigned hw = std::thread::hardware_concurrency();
    readers_ = static_cast<int>(std::max(1u, std::min(8u, hw / 2)));
    done_.assign(nslots, nullptr);
    done_ordinal_.assign(nslots, ~uint64_t{0});
    th_ = std::thread([this] { run(); });
  }
  ~FileFeed() override {
    finish();
    for (auto& sl : slots_) PinnedPool::get().give(sl.mem, sl.cap);
    if (fd_ >= 0) ::close(fd_);
    if (f_) std::fclose(f_);
  }
  const BlcoFileHeader& header() const { return h_; }

  int next(blco_block_view& v) override {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return !ready_.empty() || finished_; });
    if (!ready_.empty()) {
      v = ready_.front();
      ready_.pop_front();
      return 1;
    }
    if (err_code_ != BLCO_OK) throw Status(err_code_, err_);
    return 0;
  }
  void transferred(uint64_t ordinal, cudaEvent_t done) override {
    std::lock_guard<std::mutex> lk(mu_);
    const size_t k = ordinal % slots_.size();
    done_[k] = done;
    done_ordinal_[k] = ordinal;
    cv_.notify_all();
  }
  bool validate() const override { return true; }
  void finish() override {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      cv_.notify_all();
    }
    if (th_.joinable()) th_.join();
  }

 private:
  struct Slot {
    void* mem = nullptr;
    size_t cap = 0;
  };

  bool read_at(void* dst, size_t bytes, uint64_t off) const {
    auto* p = static_cast<char*>(dst);
    while (bytes) {
      const ssize_t r = ::pread(fd_, p, bytes, static_cast<off_t>(off));
      if (r <= 0) return false;
      p += r, off += static_cast<uint64_t>(r), bytes -= static_cast<size_t>(r);
    }
    return true;
  }
  bool read_parallel(void* dst, size_t bytes, uint64_t off) const {
    const size_t piece = (bytes + readers_ - 1) / readers_;
    if (readers_ == 1 || bytes < (size_t{8} << 20)) return read_at(dst, bytes, off);
    std::vector<std::thread> th;
    std::vector<char> ok(readers_, 0);
    for (int i = 0; i < readers_; ++i) {
      const size_t b = piece * i, e = std::min(bytes, b + piece);
      if (b >= e) {
        ok[i] = 1;
        continue;
      }
      th.emplace_back([&, i, b, e] { ok[i] = read_at(static_cast<char*>(dst) + b, e - b, off + b); });
    }
    for (auto& t : th) t.join();
    for (char x : ok)
      if (!x) return false;
    return true;
  }

  void fail(int code, const std::string& msg) {
    std::lock_guard<std::mutex> lk(mu_);
    err_code_ = code;
    err_ = msg;
    finished_ = true;
    cv_.notify_all();
  }

  void run() {
    try {
      B200_CUDA(cudaSetDevice(device_));
      const size_t K = slots_.size();
      const blco_layout& l = h_.layout;
      uint64_t prev_key = 0;
      for (uint64_t b = 0; b < h_.nblocks; ++b) {
        const size_t k = b % K;
        if (b >= K) {  // the slot's previous block (b - K) must have crossed the link
          cudaEvent_t ev = nullptr;
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || done_ordinal_[k] == b - K; });
            if (stop_) return;
            ev = done_[k];
          }
          B200_CUDA(cudaEventSynchronize(ev));
        }
        uint64_t rec[2];
        if (!read_at(rec, 16, pos_)) throw Status(BLCO_EIO, "blco: truncated payload");
        pos_ += 16;
        const uint64_t key = rec[0], n = rec[1];
        if (l.stripped_bits < 64 && key >= (uint64_t{1} << l.stripped_bits))
          throw_format("blco: block key out of range");
        if (n == 0) throw_format("blco: empty block record");
        if (n > h_.max_nnz) throw_format("blco: block exceeds max_nnz_per_block");
        if (b > 0 && key < prev_key) throw_format("blco: blocks not in ascending key order");
        prev_key = key;
        Slot& sl = slots_[k];
        if (sl.cap < n * 16) {
          PinnedPool::get().give(sl.mem, sl.cap);
          sl.mem = nullptr;
          sl.cap = 0;
          // at least this block, rounded up to 64 MiB so a slot is not
          // regrown for every slightly larger block
          const size_t want = ((n * 16 + (size_t{64} << 20) - 1) >> 26) << 26;
          std::tie(sl.mem, sl.cap) = PinnedPool::get().take(std::max<size_t>(n * 16, std::min(want, h_.max_nnz * 16)));
        }
        auto* idx = static_cast<uint64_t*>(sl.mem);
        auto* vals = reinterpret_cast<double*>(idx + n);
        // the record's idx[n] | vals[n] are contiguous in the file and in the
        // slot: one range, read by `readers_` threads in parallel (pread)
        if (!read_parallel(sl.mem, n * 16, pos_)) throw Status(BLCO_EIO, "blco: truncated payload");
        pos_ += n * 16;
        std::lock_guard<std::mutex> lk(mu_);
        if (stop_) return;
        ready_.push_back(blco_block_view{key, n, idx, vals, BLCO_BLOCK_STABLE});
        cv_.notify_all();
      }
      std::lock_guard<std::mutex> lk(mu_);
      finished_ = true;
      cv_.notify_all();
    } catch (const Status& s) {
      fail(s.code, s.what());
    } catch (const std::exception& e) {
      fail(BLCO_ERROR, e.what());
    }
  }

  FILE* f_ = nullptr;
  int fd_ = -1;
  uint64_t pos_ = 0;  // file offset of the next block record
  int readers_ = 1;
  BlcoFileHeader h_{};
  int device_;
  std::vector<Slot> slots_;
  std::vector<cudaEvent_t> done_;
  std::vector<uint64_t> done_ordinal_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<blco_block_view> ready_;
  bool finished_ = false, stop_ = false;
  int err_code_ = BLCO_OK;
  std::string err_;
  std::thread th_;
};

}  // namespace
}  // namespace b200

using namespace b200;

extern "C" int blco_stream_mttkrp(const blco_layout* layout, uint64_t max_nnz_per_block,
                                  blco_block_source_fn next, void* ctx,
                                  const double* const* factors, uint64_t rank, int mode,
                                  const blco_device_budget* budget, const blco_exec_config* cfg,
                                  int strategy, int device, double* out,
                                  blco_stream_report* report) {
  return guarded([&] {
    CallbackFeed feed(next, ctx);
    stream_impl(layout, max_nnz_per_block, feed, factors, rank, std::vector<int>{mode}, budget, cfg, strategy,
                device, &out, false, report);
  });
}

extern "C" int blco_stream_mttkrp_all(const blco_layout* layout, uint64_t max_nnz_per_block,
                                      blco_block_source_fn next, void* ctx,
                                      const double* const* factors, uint64_t rank,
                                      const blco_device_budget* budget, const blco_exec_config* cfg,
                                      int strategy, int device, double* const* outs,
                                      int outs_on_device, blco_stream_report* report) {
  return guarded([&] {
    if (!layout) throw_format("stream: null layout");
    std::vector<int> modes(layout->order);
    for (int m = 0; m < layout->order; ++m) modes[m] = m;
    CallbackFeed feed(next, ctx);
    stream_impl(layout, max_nnz_per_block, feed, factors, rank, modes, budget, cfg, strategy, device, outs,
                outs_on_device != 0, report);
  });
}

extern "C" int blco_stream_mttkrp_file(const char* path, const double* const* factors, uint64_t rank, int mode,
                                       const blco_device_budget* budget, const blco_exec_config* cfg, int strategy,
                                       int device, double* const* outs, blco_stream_report* report) {
  return guarded([&] {
    if (!path) throw Status(BLCO_EIO, "cannot open (null path)");
    if (budget->num_queues < 1) throw_format("stream: num_queues must be >= 1");
    DeviceGuard dg(device);
    FileFeed feed(path, device, budget->num_queues + 2);
    const blco_layout& l = feed.header().layout;
    std::vector<int> modes;
    if (mode >= 0) {
      modes.push_back(mode);
    } else {
      for (int m = 0; m < l.order; ++m) modes.push_back(m);
    }
    stream_impl(&l, feed.header().max_nnz, feed, factors, rank, modes, budget, cfg, strategy, device, outs, false,
                report);
  });
}

extern "C" void* blco_host_alloc_pinned(uint64_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    set_error(BLCO_ECUDA, "cuda: cudaHostAlloc failed");
    return nullptr;
  }
  return p;
}

extern "C" void blco_host_free_pinned(void* p) {
  if (p) cudaFreeHost(p);
}

extern "C" int blco_host_register(void* p, uint64_t bytes) {
  return guarded([&] { B200_CUDA(cudaHostRegister(p, bytes, cudaHostRegisterPortable)); });
}

extern "C" int blco_host_unregister(void* p) {
  return guarded([&] { B200_CUDA(cudaHostUnregister(p)); });
}
