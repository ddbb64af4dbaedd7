// ref_shim.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/libblco_ref.so, so tests, the golden-fixture generator and
// bench.py's reference arm can drive the reference's own C++ API through
// ctypes.  No reference source is copied into this repository.
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "blco/blco_format.hpp"
#include "blco/cpals.hpp"
#include "blco/layout.hpp"
#include "blco/mttkrp.hpp"
#include "blco/oracle.hpp"
#include "blco/streaming.hpp"
#include "blco/types.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const blco::FormatError& e) {
    g_err = e.what();
    return 2;
  } catch (const blco::IoError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

blco::FactorMatrices make_factors(int order, const uint64_t* dims, const double* const* f,
                                  uint64_t rank) {
  blco::FactorMatrices fm;
  fm.rank = rank;
  for (int m = 0; m < order; ++m) {
    blco::DenseMatrix a(dims[m], rank);
    std::memcpy(a.data.data(), f[m], dims[m] * rank * sizeof(double));
    fm.factors.push_back(std::move(a));
  }
  return fm;
}

blco::ExecConfig make_cfg(const int* c) {
  blco::ExecConfig cfg;
  if (!c) return cfg;
  cfg.workgroup_size = c[0];
  cfg.tile_size = c[1];
  cfg.coarsening = c[2];
  cfg.num_compute_units = c[3];
  cfg.num_factor_copies = c[4];
  cfg.stash_slots = c[5];
  cfg.deterministic = c[6] != 0;
  cfg.num_threads = c[7];
  return cfg;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// layout fields: out_i32 = [total, stripped, mode_bits[order], rem_bits[order],
// field_shift[order], imap_mode[total], imap_bit[total]]; out_mask[order]
int ref_layout(const uint64_t* dims, int order, int target_bits, int* out_i32,
               uint64_t* out_mask) {
  return guarded([&] {
    auto l = blco::make_layout(std::vector<uint64_t>(dims, dims + order), target_bits);
    int k = 0;
    out_i32[k++] = l.total_bits;
    out_i32[k++] = l.stripped_bits;
    for (int m = 0; m < order; ++m) out_i32[k++] = l.mode_bits[m];
    for (int m = 0; m < order; ++m) out_i32[k++] = l.rem_bits[m];
    for (int m = 0; m < order; ++m) out_i32[k++] = l.field_shift[m];
    for (auto [m, b] : l.interleave_map) out_i32[k++] = m;
    for (auto [m, b] : l.interleave_map) out_i32[k++] = b;
    for (int m = 0; m < order; ++m) out_mask[m] = l.field_mask[m];
  });
}

// out = [alto_hi, alto_lo, split_key, split_reenc, enc_key, enc_reenc]
int ref_encode(const uint64_t* dims, int order, int target_bits, const uint64_t* coords,
               uint64_t* out) {
  return guarded([&] {
    auto l = blco::make_layout(std::vector<uint64_t>(dims, dims + order), target_bits);
    std::vector<uint64_t> c(coords, coords + order);
    const blco::alto_t a = blco::linearize(l, c);
    auto s = blco::split_block_key(l, a);
    auto e = blco::encode_coords(l, c);
    out[0] = static_cast<uint64_t>(a >> 64);
    out[1] = static_cast<uint64_t>(a);
    out[2] = s.block_key;
    out[3] = s.reencoded;
    out[4] = e.block_key;
    out[5] = e.reencoded;
  });
}

int ref_build_blco(int order, const uint64_t* dims, uint64_t nnz, const uint64_t* idx,
                   const double* vals, int target_bits, uint64_t max_nnz, void** out,
                   double* stage_seconds) {
  return guarded([&] {
    blco::SparseTensorCoo coo;
    coo.dims.assign(dims, dims + order);
    coo.indices.resize(order);
    for (int m = 0; m < order; ++m) coo.indices[m].assign(idx + m * nnz, idx + (m + 1) * nnz);
    coo.values.assign(vals, vals + nnz);
    blco::BuildStats st;
    auto* t = new blco::BlcoTensor(blco::build_blco(coo, target_bits, max_nnz, &st));
    if (stage_seconds) {
      stage_seconds[0] = st.sort_seconds;
      stage_seconds[1] = st.block_seconds;
      stage_seconds[2] = st.reencode_seconds;
      stage_seconds[3] = st.batch_seconds;
    }
    *out = t;
  });
}

// Wraps caller-provided blocks (block-concatenated idx/vals with offsets) as
// a reference BlcoTensor, batch table rebuilt as deserialize_blco does.
int ref_blco_from_blocks(int order, const uint64_t* dims, int target_bits, uint64_t max_nnz,
                         uint64_t nblocks, const uint64_t* keys, const uint64_t* offsets,
                         const uint64_t* idx, const double* vals, void** out) {
  return guarded([&] {
    auto* t = new blco::BlcoTensor;
    t->layout = blco::make_layout(std::vector<uint64_t>(dims, dims + order), target_bits);
    t->max_nnz_per_block = max_nnz;
    for (uint64_t b = 0; b < nblocks; ++b) {
      blco::BlcoBlock blk;
      blk.key = keys[b];
      blk.linear_indices.assign(idx + offsets[b], idx + offsets[b + 1]);
      blk.values.assign(vals + offsets[b], vals + offsets[b + 1]);
      t->total_nnz += blk.nnz();
      t->blocks.push_back(std::move(blk));
    }
    t->batch_quota = blco::kDefaultBatchQuota;
    t->batch_table = blco::compute_batch_table(*t, t->batch_quota);
    *out = t;
  });
}

void ref_blco_free(void* h) { delete static_cast<blco::BlcoTensor*>(h); }

// serialize_blco into buf (capacity cap); returns the byte count (0 if it
// does not fit).
uint64_t ref_serialize(void* h, char* buf, uint64_t cap) {
  std::ostringstream out;
  blco::serialize_blco(*static_cast<blco::BlcoTensor*>(h), out);
  const std::string s = out.str();
  if (s.size() > cap) return 0;
  std::memcpy(buf, s.data(), s.size());
  return s.size();
}

uint64_t ref_blco_nblocks(void* h) { return static_cast<blco::BlcoTensor*>(h)->blocks.size(); }

void ref_blco_block(void* h, uint64_t b, uint64_t* key, uint64_t* nnz, const uint64_t** idx,
                    const double** vals) {
  auto& blk = static_cast<blco::BlcoTensor*>(h)->blocks[b];
  *key = blk.key;
  *nnz = blk.nnz();
  *idx = blk.linear_indices.data();
  *vals = blk.values.data();
}

uint64_t ref_blco_batch(void* h, uint64_t* spans) {
  auto& bt = static_cast<blco::BlcoTensor*>(h)->batch_table;
  if (spans)
    for (std::size_t i = 0; i < bt.size(); ++i) {
      spans[3 * i] = bt[i].block;
      spans[3 * i + 1] = bt[i].offset;
      spans[3 * i + 2] = bt[i].count;
    }
  return bt.size();
}

// cfg: 8 ints (ExecConfig fields in declaration order) or NULL for defaults.
// stats: [strategy, workgroups, segments, stash_flushes, commit_events, scalar_adds]
int ref_mttkrp(void* h, const double* const* factors, uint64_t rank, int mode, const int* cfg,
               int strategy, double* out, uint64_t* stats) {
  return guarded([&] {
    auto& t = *static_cast<blco::BlcoTensor*>(h);
    auto fm = make_factors(t.order(), t.dims().data(), factors, rank);
    blco::MttkrpStats st;
    auto m = blco::mttkrp(t, fm, mode, make_cfg(cfg), static_cast<blco::Strategy>(strategy), &st);
    std::memcpy(out, m.data.data(), m.data.size() * sizeof(double));
    if (stats) {
      stats[0] = static_cast<uint64_t>(st.strategy);
      stats[1] = st.workgroups;
      stats[2] = st.segments;
      stats[3] = st.stash_flushes;
      stats[4] = st.commit_events;
      stats[5] = st.scalar_adds;
    }
  });
}

int ref_mttkrp_coo(int order, const uint64_t* dims, uint64_t nnz, const uint64_t* idx,
                   const double* vals, const double* const* factors, uint64_t rank, int mode,
                   double* out) {
  return guarded([&] {
    blco::SparseTensorCoo coo;
    coo.dims.assign(dims, dims + order);
    coo.indices.resize(order);
    for (int m = 0; m < order; ++m) coo.indices[m].assign(idx + m * nnz, idx + (m + 1) * nnz);
    coo.values.assign(vals, vals + nnz);
    auto fm = make_factors(order, dims, factors, rank);
    auto m = blco::oracle::mttkrp_coo(coo, fm, mode);
    std::memcpy(out, m.data.data(), m.data.size() * sizeof(double));
  });
}

int ref_factors_random(const uint64_t* dims, int order, uint64_t rank, uint64_t seed,
                       double* const* out) {
  return guarded([&] {
    auto fm = blco::FactorMatrices::random(std::vector<uint64_t>(dims, dims + order), rank, seed);
    for (int m = 0; m < order; ++m)
      std::memcpy(out[m], fm.factors[m].data.data(), fm.factors[m].data.size() * sizeof(double));
  });
}

// budget: [capacity_bytes, num_queues, reservation_bytes]
int ref_stream_mttkrp(void* h, const double* const* factors, uint64_t rank, int mode,
                      const uint64_t* budget, const int* cfg, int strategy, double* out,
                      double* report) {
  return guarded([&] {
    auto& t = *static_cast<blco::BlcoTensor*>(h);
    auto fm = make_factors(t.order(), t.dims().data(), factors, rank);
    blco::DeviceBudget b;
    b.capacity_bytes = budget[0];
    b.num_queues = static_cast<int>(budget[1]);
    b.reservation_bytes = budget[2];
    blco::MemoryBlockSource src(t);
    blco::StreamReport rep;
    auto m = blco::stream_mttkrp(src, fm, mode, b, make_cfg(cfg),
                                 static_cast<blco::Strategy>(strategy), &rep);
    std::memcpy(out, m.data.data(), m.data.size() * sizeof(double));
    if (report) {
      report[0] = static_cast<double>(rep.blocks);
      report[1] = static_cast<double>(rep.bytes_streamed);
      report[2] = rep.total_seconds;
      report[3] = rep.overall_gbps;
      report[4] = rep.compute_gbps;
      report[5] = static_cast<double>(rep.peak_resident_bytes);
    }
  });
}

int ref_cp_als(void* h, uint64_t rank, int max_iters, double tol, uint64_t seed, int strategy,
               const int* cfg, double* const* factors_out, double* lambda_out, double* fit_out,
               int* iters_out) {
  return guarded([&] {
    auto& t = *static_cast<blco::BlcoTensor*>(h);
    blco::CpAlsOptions o;
    o.rank = rank;
    o.max_iters = max_iters;
    o.tol = tol;
    o.seed = seed;
    o.strategy = static_cast<blco::Strategy>(strategy);
    auto model = blco::cp_als(t, o, make_cfg(cfg));
    for (int m = 0; m < t.order(); ++m)
      std::memcpy(factors_out[m], model.factors.factors[m].data.data(),
                  model.factors.factors[m].data.size() * sizeof(double));
    std::memcpy(lambda_out, model.lambda.data(), rank * sizeof(double));
    std::memcpy(fit_out, model.fit_history.data(), model.fit_history.size() * sizeof(double));
    *iters_out = static_cast<int>(model.fit_history.size());
  });
}

}  // extern "C"
