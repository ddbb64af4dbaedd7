/*
 * blco_oracle.h -- CPU restatement of the reference BLCO path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (libblco_b200.so, the
 * Python package, __graft_entry__.build's product half) links or calls this.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it,
 * and only as the checker.
 *
 * Parity pinning: every function below is checked against the reference's own
 * golden vectors (tests/golden/, restated from proj/tests/*.cpp) and against
 * the reference library itself compiled here into oracle/_ref/ (see
 * oracle/Makefile and tests/golden/gen_golden.py).
 *
 * Citations are paths under the read-only reference tree (proj/...).
 */
#ifndef BLCO_ORACLE_H
#define BLCO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_ORDER 32
#define ORC_MAX_BITS 128

/* status codes (mirror the product's C ABI) */
#define ORC_OK 0
#define ORC_EFORMAT 2

typedef unsigned __int128 orc_u128;

/* proj/include/blco/layout.hpp:19-51 (BitLayout) */
typedef struct orc_layout {
  int order;
  int total_bits;
  int target_bits;
  int stripped_bits;
  uint64_t dims[ORC_MAX_ORDER];
  int mode_bits[ORC_MAX_ORDER];
  int rem_bits[ORC_MAX_ORDER];
  int field_shift[ORC_MAX_ORDER];
  uint64_t field_mask[ORC_MAX_ORDER];
  /* interleaved position p (LSB first) -> (mode, bit within mode) */
  int imap_mode[ORC_MAX_BITS];
  int imap_bit[ORC_MAX_BITS];
  /* mode m, bit k -> interleaved position */
  int mode_pos[ORC_MAX_ORDER][64];
} orc_layout;

const char* orc_last_error(void);

/* proj/src/layout.cpp:15-69 */
int orc_make_layout(const uint64_t* dims, int order, int target_bits, orc_layout* out);
/* proj/src/layout.cpp:71-82 ; returns ALTO as (hi, lo) */
int orc_linearize(const orc_layout* l, const uint64_t* coords, uint64_t* hi, uint64_t* lo);
/* proj/src/layout.cpp:84-95 */
void orc_split_block_key(const orc_layout* l, uint64_t hi, uint64_t lo, uint64_t* key,
                         uint64_t* reenc);
/* proj/src/layout.cpp:97-107 */
int orc_encode_coords(const orc_layout* l, const uint64_t* coords, uint64_t* key,
                      uint64_t* reenc);
/* proj/src/layout.cpp:109-114 */
void orc_delinearize(const orc_layout* l, uint64_t reenc, uint64_t key, uint64_t* coords);
/* proj/src/layout.cpp:116-124 */
void orc_interleaved_remainder(const orc_layout* l, uint64_t reenc, uint64_t* hi, uint64_t* lo);

/* proj/src/blco_format.cpp:62-134 (build_blco).  idx is mode-major:
 * idx[m * nnz + e].  Output arrays are malloc'd; free with orc_free_blco. */
typedef struct orc_blco {
  uint64_t nblocks;
  uint64_t* keys;      /* [nblocks] */
  uint64_t* offsets;   /* [nblocks + 1] element offsets into idx/vals */
  uint64_t* idx;       /* [nnz] re-encoded indices, block-concatenated */
  double* vals;        /* [nnz] */
  uint64_t nnz;
} orc_blco;

int orc_build_blco(const orc_layout* l, uint64_t nnz, const uint64_t* idx, const double* vals,
                   uint64_t max_nnz_per_block, orc_blco* out);
void orc_free_blco(orc_blco* b);

/* proj/src/blco_format.cpp:136-147.  Writes (block, offset, count) triples
 * into spans (may be NULL to count); returns the span count. */
uint64_t orc_batch_table(const uint64_t* block_nnz, uint64_t nblocks, uint64_t quota,
                         uint64_t* spans);

/* proj/src/oracle.cpp:9-26 (oracle::mttkrp_coo), the trusted root.
 * factors[m] is dims[m] x rank row-major; out is dims[mode] x rank. */
int orc_mttkrp_coo(int order, const uint64_t* dims, uint64_t nnz, const uint64_t* idx,
                   const double* vals, const double* const* factors, uint64_t rank, int mode,
                   double* out);

/* Same element-wise loop over a BLCO tensor in stored order (decode with
 * proj/src/layout.cpp:109-114, then the oracle.cpp:15-24 product order). */
int orc_mttkrp_blco(const orc_layout* l, const orc_blco* t, const double* const* factors,
                    uint64_t rank, int mode, double* out);

/* proj/src/types.cpp:104-130 (FactorMatrices::random, SplitMix64). */
void orc_factors_random(const uint64_t* dims, int order, uint64_t rank, uint64_t seed,
                        double* const* out);

/* Synthetic-workload generator restated on the CPU (the product generates
 * the same tensor on the device).  Element e
 * gets cell feistel_perm(e) in [0, prod(dims)) decoded mixed-radix (mode 0
 * fastest) and value unit(splitmix64 output e of seed ^ VALUE_SALT). */
int orc_synth_uniform(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed,
                      uint64_t* idx, double* vals);
/* Rows rows[m][0..nrows[m]) of mttkrp_coo over an in-memory COO, every mode,
 * bit-identical to orc_mttkrp_coo's rows. */
int orc_rowsample_coo(int order, const uint64_t* dims, uint64_t nnz, const uint64_t* idx, const double* vals,
                      const double* const* f, uint64_t rank, const uint64_t* nrows,
                      const uint64_t* const* rows, double* const* out);

/* Rows rows[m][0..nrows[m]) of mttkrp_coo(T, f, m) for every mode m of
 * T = orc_synth_uniform(dims, nnz, seed), streamed (T is never stored);
 * bit-identical to the full oracle's rows (SURVEY.md 8c row-sampled oracle).
 * out[m] is nrows[m] x rank.  order <= 8. */
int orc_rowsample_uniform(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed,
                          const double* const* f, uint64_t rank, const uint64_t* nrows,
                          const uint64_t* const* rows, double* const* out, int threads);

/* Census of T = orc_synth_uniform(dims, nnz, seed), streamed on `threads`
 * threads: the order-free multiset hash (sum of mix64(cell ^ mix64(value
 * bits)) mod 2^64, cell = the mixed-radix cell id) and the element count per
 * block key of the target_bits layout (key_counts[2^stripped_bits]). */
int orc_census_uniform(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed, int target_bits,
                       int threads, uint64_t* hash, uint64_t* key_counts);

int orc_alto_lo_batch(const orc_layout* l, uint64_t nnz, const uint64_t* idx, uint64_t* out);

/* Independent per-mode draws floor(I * u^skew), first nnz distinct tuples. */
int orc_synth_draws(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed, int skew,
                    uint64_t* idx, double* vals);

/* Dense kernels for the CP-ALS restatement: proj/src/dense_kernels.cpp. */
void orc_gram(const double* a, uint64_t rows, uint64_t rank, double* g);
int orc_solve_normal(double* m, uint64_t rows, const double* v, uint64_t rank);

/* CP-ALS: proj/src/cpals.cpp:66-111.  factors_out[m] (dims[m] x rank),
 * lambda_out[rank], fit_out[max_iters]; returns iterations run (>= 0) or -err. */
int orc_cp_als(const orc_layout* l, const orc_blco* t, uint64_t rank, int max_iters, double tol,
               uint64_t seed, double* const* factors_out, double* lambda_out, double* fit_out);

#ifdef __cplusplus
}
#endif
#endif
