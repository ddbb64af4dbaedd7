// test_api.cpp -- the reference's results-parity (bucket P) test cases
// restated in C++ against the drop-in API (include/blco/*.hpp ->
// libblco_b200.so).  Same inputs, seeds and assertions as the cited
// proj/tests lines; a reference user's code compiles against these headers.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <functional>
#include <sstream>
#include <map>
#include <set>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "blco/blco_format.hpp"
#include "blco/cpals.hpp"
#include "blco/layout.hpp"
#include "blco/mttkrp.hpp"
#include "blco/streaming.hpp"

using namespace blco;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(c)) {                                                               \
      ++g_fail;                                                               \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c); \
    }                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                 \
  do {                                           \
    bool thrown = false;                         \
    try {                                        \
      (void)(expr);                              \
    } catch (const T&) {                         \
      thrown = true;                             \
    }                                            \
    CHECK(thrown);                               \
  } while (0)

static std::vector<std::pair<const char*, std::function<void()>>>& registry() {
  static std::vector<std::pair<const char*, std::function<void()>>> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define TEST(name)                       \
  static void name();                    \
  static Reg reg_##name(#name, name);    \
  static void name()

// proj/tests/test_util.hpp:28-92
static SparseTensorCoo golden_tensor() {
  std::vector<index_t> i1{0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 3, 3};
  std::vector<index_t> i2{0, 0, 2, 0, 0, 0, 3, 1, 1, 2, 2, 3};
  std::vector<index_t> i3{0, 1, 2, 1, 2, 1, 3, 0, 1, 2, 3, 3};
  std::vector<double> v{1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12};
  return SparseTensorCoo::from_arrays({4, 4, 4}, {i1, i2, i3}, v);
}

struct Rng {
  std::uint64_t state;
  explicit Rng(std::uint64_t seed) : state(seed + 0x9e3779b97f4a7c15ull) {}
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  std::uint64_t below(std::uint64_t n) { return n ? next() % n : 0; }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

static SparseTensorCoo random_coo(Rng& rng, const std::vector<index_t>& dims, std::size_t n) {
  const int order = static_cast<int>(dims.size());
  std::set<std::vector<index_t>> seen;
  std::vector<std::vector<index_t>> idx(order);
  std::vector<double> vals;
  for (std::size_t tries = 0; tries < n * 4 && vals.size() < n; ++tries) {
    std::vector<index_t> c(order);
    for (int m = 0; m < order; ++m) c[m] = rng.below(dims[m]);
    if (!seen.insert(c).second) continue;
    for (int m = 0; m < order; ++m) idx[m].push_back(c[m]);
    vals.push_back(2.0 * rng.unit() - 1.0);
  }
  return SparseTensorCoo::from_arrays(dims, std::move(idx), std::move(vals));
}

static FactorMatrices random_factors(Rng& rng, const std::vector<index_t>& dims, std::size_t rank) {
  FactorMatrices f;
  f.rank = rank;
  for (index_t d : dims) {
    DenseMatrix a(d, rank);
    for (double& v : a.data) v = 2.0 * rng.unit() - 1.0;
    f.factors.push_back(std::move(a));
  }
  return f;
}

static double rel_frobenius(const DenseMatrix& a, const DenseMatrix& b) {
  double diff = 0, ref = 0;
  for (std::size_t i = 0; i < a.data.size(); ++i) {
    diff += (a.data[i] - b.data[i]) * (a.data[i] - b.data[i]);
    ref += b.data[i] * b.data[i];
  }
  return ref > 0 ? std::sqrt(diff / ref) : std::sqrt(diff);
}

// element-wise definition, COO order (the oracle loop)
static DenseMatrix mttkrp_coo(const SparseTensorCoo& t, const FactorMatrices& f, int mode) {
  DenseMatrix m(t.dims[mode], f.rank);
  std::vector<double> row(f.rank);
  for (std::size_t e = 0; e < t.nnz(); ++e) {
    std::fill(row.begin(), row.end(), t.values[e]);
    for (int n = 0; n < t.order(); ++n)
      if (n != mode)
        for (std::size_t r = 0; r < f.rank; ++r) row[r] *= f.factors[n](t.indices[n][e], r);
    for (std::size_t r = 0; r < f.rank; ++r) m(t.indices[mode][e], r) += row[r];
  }
  return m;
}

TEST(layout_444) {  // test_layout.cpp:8-30
  auto l = make_layout(std::vector<index_t>{4, 4, 4}, 64);
  CHECK(l.mode_bits == (std::vector<int>{2, 2, 2}));
  CHECK(l.total_bits == 6 && l.stripped_bits == 0);
  CHECK(l.interleave_map[3] == (std::pair<int, int>{0, 1}));
  auto l5 = make_layout(std::vector<index_t>{4, 4, 4}, 5);
  CHECK(l5.stripped_bits == 1);
  CHECK(l5.rem_bits == (std::vector<int>{2, 2, 1}));
  CHECK(l5.field_shift == (std::vector<int>{0, 2, 4}));
  CHECK(l5.field_mask == (std::vector<index_t>{3, 3, 1}));
  CHECK_THROWS_AS(make_layout(std::vector<index_t>{4, 4}, 0), FormatError);
  CHECK_THROWS_AS(make_layout(std::vector<index_t>{0, 4}, 32), FormatError);
}

TEST(linearize_split_goldens) {  // test_layout.cpp:48-95
  auto l = make_layout(std::vector<index_t>{4, 4, 4}, 64);
  CHECK(linearize(l, std::vector<index_t>{3, 1, 0}) == 11);
  CHECK(linearize(l, std::vector<index_t>{2, 3, 3}) == 62);
  CHECK_THROWS_AS(linearize(l, std::vector<index_t>{4, 0, 0}), FormatError);
  auto l5 = make_layout(std::vector<index_t>{4, 4, 4}, 5);
  auto s = split_block_key(l5, 48);
  CHECK(s.block_key == 1 && s.reencoded == 8);
  s = split_block_key(l5, 11);
  CHECK(s.block_key == 0 && s.reencoded == 7);
  index_t c[3];
  delinearize(l5, 1, 1, c);
  CHECK(c[0] == 1 && c[1] == 0 && c[2] == 2);
}

TEST(encode_equals_linearize_split) {  // test_layout.cpp:112-130
  Rng rng(23);
  for (int trial = 0; trial < 200; ++trial) {
    const int order = 1 + static_cast<int>(rng.below(5));
    std::vector<index_t> dims(order);
    for (auto& d : dims) d = 1 + rng.below(1u << rng.below(21));
    int total = 0;
    for (auto d : dims) total += bits_for_extent(d);
    const int target = 1 + static_cast<int>(rng.below(64));
    if (total > 128) continue;
    auto l = make_layout(dims, target);
    if (l.stripped_bits > 64) continue;  // reference UB region
    std::vector<index_t> co(order);
    for (int m = 0; m < order; ++m) co[m] = rng.below(dims[m]);
    auto a = split_block_key(l, linearize(l, co));
    auto b = encode_coords(l, co);
    CHECK(a.block_key == b.block_key && a.reencoded == b.reencoded);
  }
}

TEST(fig5b_blocks) {  // test_blco.cpp:11-48
  auto t = build_blco(golden_tensor(), 5, 6);
  CHECK(t.blocks.size() == 2 && t.total_nnz == 12);
  CHECK(t.blocks[0].linear_indices == (std::vector<index_t>{0, 16, 17, 7, 18, 23}));
  CHECK(t.blocks[0].values == (std::vector<double>{1, 2, 4, 8, 6, 9}));
  CHECK(t.blocks[1].key == 1);
  CHECK(t.blocks[1].linear_indices == (std::vector<index_t>{1, 8, 11, 27, 30, 31}));
  auto t4 = build_blco(golden_tensor(), 5, 4);
  CHECK(t4.blocks.size() == 4 && t4.blocks[1].nnz() == 2 && t4.blocks[3].key == 1);
  auto spans = compute_batch_table(t, 4);
  CHECK(spans.size() == 4 && spans[1] == (BatchSpan{0, 4, 2}));
}

TEST(conservation) {  // test_blco.cpp:50-84
  Rng rng(47);
  for (int trial = 0; trial < 12; ++trial) {
    const int order = 2 + static_cast<int>(rng.below(4));
    std::vector<index_t> dims(order);
    for (auto& d : dims) d = 1 + rng.below(300);
    auto coo = random_coo(rng, dims, 200);
    const int target = 3 + static_cast<int>(rng.below(62));
    auto t = build_blco(coo, target, 1 + rng.below(64));
    auto back = delinearize_all(t);
    std::map<std::vector<index_t>, double> want, got;
    for (std::size_t e = 0; e < coo.nnz(); ++e) {
      std::vector<index_t> c(order);
      for (int m = 0; m < order; ++m) c[m] = coo.indices[m][e];
      want[c] = coo.values[e];
    }
    for (std::size_t e = 0; e < back.nnz(); ++e) {
      std::vector<index_t> c(order);
      for (int m = 0; m < order; ++m) c[m] = back.indices[m][e];
      got[c] = back.values[e];
    }
    CHECK(want == got);
  }
}

TEST(duplicates_rejected) {  // test_blco.cpp:95-101
  SparseTensorCoo t;
  t.dims = {2, 2};
  t.indices = {{0, 0}, {1, 1}};
  t.values = {1.0, 2.0};
  CHECK_THROWS_AS(build_blco(t, 64), FormatError);
}

TEST(all_ones_rows) {  // test_mttkrp.cpp:33-47
  auto t = build_blco(golden_tensor(), 5, 6);
  auto f = FactorMatrices::ones(t.dims(), 2);
  auto m1 = mttkrp(t, f, 0, {}, Strategy::Register);
  const double rows1[4] = {6, 9, 13, 50};
  for (int i = 0; i < 4; ++i) CHECK(std::abs(m1(i, 1) - rows1[i]) <= 1e-13 * rows1[i]);
  auto m3 = mttkrp(t, f, 2, {}, Strategy::Hierarchical);
  const double rows3[4] = {9, 21, 18, 30};
  for (int i = 0; i < 4; ++i) CHECK(std::abs(m3(i, 0) - rows3[i]) <= 1e-13 * rows3[i]);
}

TEST(strategy_heuristic) {  // test_mttkrp.cpp:24-31
  ExecConfig cfg;
  CHECK(choose_strategy(24, cfg) == Strategy::Hierarchical);
  CHECK(choose_strategy(23'800'000, cfg) == Strategy::Register);
  CHECK(choose_strategy(108, cfg) == Strategy::Register);
  CHECK(choose_strategy(107, cfg) == Strategy::Hierarchical);
}

TEST(strategy_config_grid) {  // test_mttkrp.cpp:267-290
  Rng rng(73);
  auto coo = random_coo(rng, {24, 9, 31}, 160);
  auto t = build_blco(coo, 7, 64);
  auto f = random_factors(rng, coo.dims, 8);
  for (int mode = 0; mode < 3; ++mode) {
    auto want = mttkrp_coo(coo, f, mode);
    for (int wg : {4, 32})
      for (int tile : {2, 4}) {
        ExecConfig cfg;
        cfg.workgroup_size = wg;
        cfg.tile_size = tile;
        cfg.coarsening = 2;
        cfg.num_threads = 2;
        cfg.num_factor_copies = 3;
        cfg.stash_slots = 4;
        for (auto s : {Strategy::Register, Strategy::Hierarchical})
          CHECK(rel_frobenius(mttkrp(t, f, mode, cfg, s), want) <= 1e-12);
      }
  }
}

TEST(all_modes_extension) {  // B200 extension: every mode of a host tensor in one call
  Rng rng(79);
  auto coo = random_coo(rng, {40, 17, 63}, 900);
  auto t = build_blco(coo, 9, 100);  // several blocks
  auto f = random_factors(rng, coo.dims, 5);
  auto all = mttkrp_all_modes(t, f);
  CHECK(all.size() == 3);
  for (int mode = 0; mode < 3; ++mode) CHECK(rel_frobenius(all[mode], mttkrp_coo(coo, f, mode)) <= 1e-12);
}

TEST(streamed_all_modes_extension) {  // B200 extension of test_streaming.cpp:21-52
  Rng rng(83);
  auto coo = random_coo(rng, {50, 40, 60}, 600);
  auto t = build_blco(coo, 8, 64);
  auto f = random_factors(rng, coo.dims, 4);
  DeviceBudget b;
  b.num_queues = 2;
  b.reservation_bytes = t.max_nnz_per_block * 16;
  b.capacity_bytes = 2 * b.reservation_bytes + (50 + 40 + 60) * 4 * 8 * 2;
  MemoryBlockSource src(t);
  StreamReport rep;
  auto all = stream_mttkrp_all_modes(src, f, b, {}, Strategy::Register, &rep);
  CHECK(all.size() == 3 && rep.blocks == t.blocks.size());
  for (int mode = 0; mode < 3; ++mode) CHECK(rel_frobenius(all[mode], mttkrp_coo(coo, f, mode)) <= 1e-12);
}

TEST(single_copy_hierarchical) {  // test_mttkrp.cpp:235-244
  auto t = build_blco(golden_tensor(), 64);
  Rng rng(67);
  auto f = random_factors(rng, t.dims(), 3);
  ExecConfig cfg;
  cfg.num_factor_copies = 1;
  CHECK(rel_frobenius(mttkrp(t, f, 1, cfg, Strategy::Hierarchical), mttkrp_coo(golden_tensor(), f, 1)) <= 1e-12);
}

TEST(merge_copies_exact) {  // test_mttkrp.cpp:246-265
  Rng rng(71);
  DenseMatrix a(3, 2);
  for (double& v : a.data) v = 2.0 * rng.unit() - 1.0;
  DenseMatrix neg = a;
  for (double& v : neg.data) v = -v;
  std::vector<DenseMatrix> pair{a, neg};
  for (double v : merge_copies(pair).data) CHECK(v == 0.0);
}

TEST(validation) {  // test_mttkrp.cpp:319-326
  auto t = build_blco(golden_tensor(), 64);
  auto f = FactorMatrices::ones(t.dims(), 2);
  CHECK_THROWS_AS(mttkrp(t, f, 5), FormatError);
  auto bad = f;
  bad.factors[1] = DenseMatrix(3, 2);
  CHECK_THROWS_AS(mttkrp(t, bad, 0), FormatError);
}

static std::uint64_t factor_bytes(const FactorMatrices& f, index_t rows) {
  std::uint64_t b = rows * f.rank * sizeof(double);
  for (const auto& a : f.factors) b += a.data.size() * sizeof(double);
  return b;
}

TEST(streamed_equals_in_memory) {  // test_streaming.cpp:21-52
  Rng rng(83);
  auto coo = random_coo(rng, {50, 40, 60}, 600);
  auto t = build_blco(coo, 8, 64);
  CHECK(t.blocks.size() >= 4);
  auto f = random_factors(rng, coo.dims, 4);
  ExecConfig cfg;
  cfg.workgroup_size = 32;
  cfg.tile_size = 4;
  cfg.coarsening = 1;
  auto want = mttkrp(t, f, 0, cfg, Strategy::Register);
  for (int queues : {1, 2, 4}) {
    DeviceBudget budget;
    budget.num_queues = queues;
    budget.reservation_bytes = t.max_nnz_per_block * 16;
    budget.capacity_bytes = factor_bytes(f, t.dims()[0]) + queues * budget.reservation_bytes;
    MemoryBlockSource source(t);
    StreamReport report;
    auto got = stream_mttkrp(source, f, 0, budget, cfg, Strategy::Register, &report);
    CHECK(rel_frobenius(got, want) <= 1e-12);
    CHECK(report.blocks == t.blocks.size());
    CHECK(report.peak_resident_bytes <= budget.capacity_bytes);
    for (std::size_t b = 0; b < report.block_queue.size(); ++b)
      CHECK(report.block_queue[b] == static_cast<int>(b % queues));
    CHECK(report.bytes_streamed == t.total_nnz * 16);
  }
}

TEST(budget_errors) {  // test_streaming.cpp:173-199
  Rng rng(107);
  auto coo = random_coo(rng, {30, 30}, 100);
  auto t = build_blco(coo, 6, 32);
  auto f = random_factors(rng, coo.dims, 4);
  DeviceBudget tiny;
  tiny.capacity_bytes = 64;
  MemoryBlockSource s1(t);
  CHECK_THROWS_AS(stream_mttkrp(s1, f, 0, tiny), FormatError);
  DeviceBudget b;
  b.num_queues = 2;
  b.reservation_bytes = 8;
  b.capacity_bytes = factor_bytes(f, t.dims()[0]) + 16;
  MemoryBlockSource s2(t);
  CHECK_THROWS_AS(stream_mttkrp(s2, f, 0, b), FormatError);
}

TEST(serialize_roundtrip) {  // test_blco.cpp:124-135
  auto t = build_blco(golden_tensor(), 5, 6);
  std::ostringstream out;
  serialize_blco(t, out);
  std::istringstream in(out.str());
  auto t2 = deserialize_blco(in);
  CHECK(t.structurally_equal(t2));
  std::ostringstream out2;
  serialize_blco(t2, out2);
  CHECK(out.str() == out2.str());
  std::string bad = out.str();
  bad[0] = 'X';
  std::istringstream in_bad(bad);
  CHECK_THROWS_AS(deserialize_blco(in_bad), FormatError);
  std::istringstream in_trunc(out.str().substr(0, out.str().size() - 5));
  CHECK_THROWS_AS(deserialize_blco(in_trunc), IoError);
}

TEST(coo_canonical_form) {  // types.cpp:38-77 semantics: lexicographic order, duplicates summed in input order
  auto t = SparseTensorCoo::from_arrays({}, {{2, 0, 2, 1, 0}, {1, 3, 1, 0, 3}}, {1.0, 2.0, 4.0, 8.0, -0.0});
  CHECK((t.dims == std::vector<index_t>{3, 4}));
  CHECK((t.indices[0] == std::vector<index_t>{0, 1, 2}));
  CHECK((t.indices[1] == std::vector<index_t>{3, 0, 1}));
  CHECK((t.values == std::vector<double>{2.0, 8.0, 5.0}));
  auto z = SparseTensorCoo::from_arrays({5}, {{4}}, {-0.0});  // a lone -0.0 keeps its sign
  CHECK(std::signbit(z.values[0]));
  CHECK_THROWS_AS(SparseTensorCoo::from_arrays({}, {}, {}), FormatError);
  CHECK_THROWS_AS(SparseTensorCoo::from_arrays({}, {{0, 1}}, {1.0}), FormatError);
  CHECK_THROWS_AS(SparseTensorCoo::from_arrays({2}, {{0, 2}}, {1.0, 2.0}), FormatError);  // out of range
  // > 128 bits of modes: the tuple-comparison path
  std::vector<index_t> wide(5, index_t{1} << 40);
  auto w = SparseTensorCoo::from_arrays(wide, {{1, 0}, {0, 0}, {0, 0}, {0, 0}, {0, 0}}, {1.0, 2.0});
  CHECK((w.indices[0] == std::vector<index_t>{0, 1}) && (w.values == std::vector<double>{2.0, 1.0}));
}

TEST(coo_validate) {  // types.cpp:13-36
  SparseTensorCoo t;
  t.dims = {3, 3};
  t.indices = {{0, 1, 0}, {2, 2, 2}};
  t.values = {1, 2, 3};
  t.validate();
  CHECK_THROWS_AS(t.validate(true), FormatError);  // (0, 2) twice
  t.indices[0][2] = 2;
  t.validate(true);
  t.indices[1][1] = 3;
  CHECK_THROWS_AS(t.validate(), FormatError);
  t.indices[1][1] = 2;
  t.dims[0] = 0;
  CHECK_THROWS_AS(t.validate(), FormatError);
  t.dims = {3};
  CHECK_THROWS_AS(t.validate(), FormatError);
}

TEST(container_bytes_and_records) {  // blco_format.cpp:149-227 byte layout and record checks
  auto t = build_blco(golden_tensor(), 5, 6);
  std::ostringstream out;
  serialize_blco(t, out);
  const std::string bytes = out.str();
  std::size_t expect = 4 + 2 + 2 + 3 * 8 + 2 + 3 * 2 + 8 + 8;
  for (const auto& b : t.blocks) expect += 16 + 16 * b.nnz();
  CHECK(bytes.size() == expect && bytes.compare(0, 4, "BLCO") == 0);
  std::istringstream in(bytes);
  const BlcoHeader h = read_blco_header(in);
  CHECK(h.version == 1 && h.target_bits == 5 && h.max_nnz_per_block == 6 && h.block_count == t.blocks.size());
  CHECK((h.dims == std::vector<index_t>{4, 4, 4}) && (h.mode_bits == std::vector<int>{2, 2, 2}));
  const BitLayout l = h.make_layout_checked();
  for (const auto& want : t.blocks) {
    const BlcoBlock got = read_blco_block(in, l);
    CHECK(got.key == want.key && got.linear_indices == want.linear_indices && got.values == want.values);
  }
  BlcoHeader bad = h;
  bad.mode_bits[1] = 3;
  CHECK_THROWS_AS(bad.make_layout_checked(), FormatError);
  bad = h;
  bad.max_nnz_per_block = 0;
  CHECK_THROWS_AS(bad.make_layout_checked(), FormatError);
  // record rules of deserialize_blco: an empty record, blocks out of key order
  BlcoTensor e = t;
  e.blocks[1].linear_indices.clear();
  e.blocks[1].values.clear();
  std::ostringstream oe;
  serialize_blco(e, oe);
  std::istringstream ie(oe.str());
  CHECK_THROWS_AS(deserialize_blco(ie), FormatError);
  BlcoTensor r = t;
  std::swap(r.blocks.front(), r.blocks.back());
  std::ostringstream orr;
  serialize_blco(r, orr);
  std::istringstream ir(orr.str());
  bool caught = false;
  try {
    (void)deserialize_blco(ir);
  } catch (const FormatError& ex) {
    caught = std::string(ex.what()).find("ascending key order") != std::string::npos ||
             std::string(ex.what()).find("exceeds") != std::string::npos;
  }
  CHECK(caught);
  std::istringstream version2(std::string("BLCO\x02\x00", 6));
  CHECK_THROWS_AS(read_blco_header(version2), FormatError);
}

TEST(multi_device_all_modes) {  // B200 multi-GPU extension: G = every visible device (1 here)
  Rng rng(211);
  auto coo = random_coo(rng, {60, 50, 40}, 4000);
  auto t = build_blco(coo, 12, 500);
  auto f = random_factors(rng, coo.dims, 8);
  int n = 0;
  cudaGetDeviceCount(&n);
  std::vector<int> devs;
  for (int g = 0; g < n; ++g) devs.push_back(g);
  MultiDeviceTensor mt(t, devs);
  CHECK(mt.ranges().size() == devs.size() && mt.ranges().back().second == t.total_nnz);
  for (Reduction how : {Reduction::AllReduce, Reduction::ReduceScatter}) {
    MultiReport rep;
    auto got = mt.mttkrp_all_modes(f, how, {}, Strategy::Auto, &rep);
    CHECK(rep.devices == n && rep.device_ms > 0);
    for (int m = 0; m < 3; ++m) CHECK(rel_frobenius(got[m], mttkrp_coo(coo, f, m)) <= 1e-12);
  }
}

TEST(file_source_streams) {  // test_streaming.cpp:81-103
  Rng rng(97);
  auto coo = random_coo(rng, {40, 30, 20}, 300);
  auto t = build_blco(coo, 8, 40);
  auto path = std::filesystem::temp_directory_path() / "b200_stream_test.blco";
  save_blco(t, path);
  auto f = random_factors(rng, coo.dims, 4);
  ExecConfig cfg;
  cfg.workgroup_size = 16;
  cfg.tile_size = 4;
  cfg.coarsening = 1;
  auto want = mttkrp(t, f, 2, cfg, Strategy::Register);
  DeviceBudget budget;
  budget.num_queues = 2;
  budget.reservation_bytes = t.max_nnz_per_block * 16;
  budget.capacity_bytes = factor_bytes(f, t.dims()[2]) + 2 * budget.reservation_bytes;
  FileBlockSource source(path);
  auto got = stream_mttkrp(source, f, 2, budget, cfg, Strategy::Register);
  CHECK(rel_frobenius(got, want) <= 1e-12);
  CHECK(load_blco(path).structurally_equal(t));
  std::filesystem::remove(path);
}

TEST(cp_als_monotone_noiseless) {  // SPEC.md:665 probe: rank-4 30^3 reaches a high fit
  Rng rng(1);
  std::vector<index_t> dims{30, 30, 30};
  std::vector<std::vector<double>> A(3, std::vector<double>(30 * 4));
  for (auto& a : A)
    for (double& v : a) v = rng.unit();
  std::vector<std::vector<index_t>> idx(3);
  std::vector<double> vals;
  for (index_t i = 0; i < 30; ++i)
    for (index_t j = 0; j < 30; ++j)
      for (index_t k = 0; k < 30; ++k) {
        double s = 0;
        for (int r = 0; r < 4; ++r) s += A[0][i * 4 + r] * A[1][j * 4 + r] * A[2][k * 4 + r];
        idx[0].push_back(i), idx[1].push_back(j), idx[2].push_back(k), vals.push_back(s);
      }
  auto t = build_blco(SparseTensorCoo::from_arrays(dims, idx, vals), 64);
  CpAlsOptions o;
  o.rank = 4;
  o.max_iters = 50;
  o.tol = 1e-9;
  o.seed = 1;
  auto model = cp_als(t, o);
  CHECK(model.final_fit() > 0.9);
  for (std::size_t i = 1; i < model.fit_history.size(); ++i)
    CHECK(model.fit_history[i] >= model.fit_history[i - 1] - 1e-6);
  CHECK(std::abs(fit(t, model) - model.final_fit()) <= 1e-9);
}

int main() {
  for (auto& [name, fn] : registry()) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "%s: unexpected exception: %s\n", name, e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? " ok " : "FAIL", name);
  }
  std::printf("%d checks, %d failures, %zu test cases\n", g_checks, g_fail, registry().size());
  return g_fail ? 1 : 0;
}
