/*
 * blco_oracle.c -- CPU restatement of the reference BLCO path.
 * TEST INFRASTRUCTURE ONLY (see blco_oracle.h).  Plain C11, single-threaded
 * except for the element filter of the row-sampled oracle (pthreads).
 */
#include "blco_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return ORC_EFORMAT;
}

const char* orc_last_error(void) { return g_err; }

/* proj/include/blco/common.hpp:20-22 */
static int bits_for(uint64_t extent) {
  if (extent <= 1) return 0;
  return 64 - __builtin_clzll(extent - 1);
}

/* ------------------------------------------------------------------ layout */

int orc_make_layout(const uint64_t* dims, int order, int target_bits, orc_layout* l) {
  memset(l, 0, sizeof *l);
  if (order < 1) return fail("layout: at least one mode required");
  if (order > ORC_MAX_ORDER) return fail("oracle: order above %d", ORC_MAX_ORDER);
  if (target_bits < 1 || target_bits > 64)
    return fail("layout: target_bits must lie in [1, 64], got %d", target_bits);
  l->order = order;
  l->target_bits = target_bits;
  int max_bits = 0;
  for (int m = 0; m < order; ++m) {
    if (dims[m] < 1) return fail("layout: mode length must be >= 1");
    l->dims[m] = dims[m];
    l->mode_bits[m] = bits_for(dims[m]);
    if (l->mode_bits[m] > max_bits) max_bits = l->mode_bits[m];
  }
  /* layout.cpp:33-36: LSB-first round robin over modes that still have bits */
  int p = 0;
  for (int k = 0; k < max_bits; ++k)
    for (int m = 0; m < order; ++m)
      if (k < l->mode_bits[m]) {
        if (p >= ORC_MAX_BITS)
          return fail("layout: tensor needs more than the 128 supported index bits");
        l->imap_mode[p] = m;
        l->imap_bit[p] = k;
        l->mode_pos[m][k] = p;
        ++p;
      }
  l->total_bits = p;
  l->stripped_bits = p > target_bits ? p - target_bits : 0;
  const int low = p - l->stripped_bits;
  for (int q = 0; q < low; ++q) l->rem_bits[l->imap_mode[q]]++;
  int shift = 0;
  for (int m = 0; m < order; ++m) {
    l->field_shift[m] = shift;
    l->field_mask[m] = l->rem_bits[m] == 0 ? 0 : (~(uint64_t)0 >> (64 - l->rem_bits[m]));
    shift += l->rem_bits[m];
  }
  if (shift == 0 && p > 0)
    return fail("layout: every index bit stripped; no addressable field remains");
  return ORC_OK;
}

int orc_linearize(const orc_layout* l, const uint64_t* c, uint64_t* hi, uint64_t* lo) {
  orc_u128 a = 0;
  for (int m = 0; m < l->order; ++m) {
    if (c[m] >= l->dims[m]) return fail("linearize: coordinate out of range");
    for (int k = 0; k < l->mode_bits[m]; ++k)
      a |= (orc_u128)((c[m] >> k) & 1u) << l->mode_pos[m][k];
  }
  *hi = (uint64_t)(a >> 64);
  *lo = (uint64_t)a;
  return ORC_OK;
}

void orc_split_block_key(const orc_layout* l, uint64_t hi, uint64_t lo, uint64_t* key,
                         uint64_t* reenc) {
  const orc_u128 a = ((orc_u128)hi << 64) | lo;
  const int low = l->total_bits - l->stripped_bits;
  /* layout.cpp:87 narrows to 64 bits (the stripped > 64 defect) */
  *key = l->stripped_bits > 0 ? (uint64_t)(a >> low) : 0;
  uint64_t r = 0;
  for (int p = 0; p < low; ++p)
    if ((a >> p) & 1u) r |= (uint64_t)1 << (l->field_shift[l->imap_mode[p]] + l->imap_bit[p]);
  *reenc = r;
}

int orc_encode_coords(const orc_layout* l, const uint64_t* c, uint64_t* key, uint64_t* reenc) {
  const int low = l->total_bits - l->stripped_bits;
  uint64_t k = 0, r = 0;
  for (int m = 0; m < l->order; ++m) {
    if (c[m] >= l->dims[m]) return fail("encode: coordinate out of range");
    r |= (c[m] & l->field_mask[m]) << l->field_shift[m];
  }
  for (int p = low; p < l->total_bits; ++p) {
    const int m = l->imap_mode[p], b = l->imap_bit[p];
    k |= ((c[m] >> b) & 1u) << (p - low);
  }
  *key = k;
  *reenc = r;
  return ORC_OK;
}

/* key_upper (layout.hpp:42-46) restated: the stripped positions of mode m, in
 * ascending order, hold that mode's bits rem_bits[m], rem_bits[m]+1, ... */
static uint64_t key_upper(const orc_layout* l, int m, uint64_t key) {
  const int low = l->total_bits - l->stripped_bits;
  uint64_t up = 0;
  for (int p = low; p < l->total_bits; ++p)
    if (l->imap_mode[p] == m)
      up |= ((key >> (p - low)) & 1u) << (l->imap_bit[p] - l->rem_bits[m]);
  return up;
}

void orc_delinearize(const orc_layout* l, uint64_t reenc, uint64_t key, uint64_t* c) {
  for (int m = 0; m < l->order; ++m)
    c[m] = (key_upper(l, m, key) << l->rem_bits[m]) |
           ((reenc >> l->field_shift[m]) & l->field_mask[m]);
}

void orc_interleaved_remainder(const orc_layout* l, uint64_t reenc, uint64_t* hi, uint64_t* lo) {
  const int low = l->total_bits - l->stripped_bits;
  orc_u128 a = 0;
  for (int p = 0; p < low; ++p)
    a |= (orc_u128)((reenc >> (l->field_shift[l->imap_mode[p]] + l->imap_bit[p])) & 1u) << p;
  *hi = (uint64_t)(a >> 64);
  *lo = (uint64_t)a;
}

/* ------------------------------------------------------------------- build */

/* stable merge sort of a permutation by 128-bit keys (blco_format.cpp:80-83) */
static void msort(uint64_t* perm, uint64_t* tmp, uint64_t n, const orc_u128* keys) {
  for (uint64_t w = 1; w < n; w *= 2) {
    for (uint64_t lo = 0; lo < n; lo += 2 * w) {
      uint64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      uint64_t i = lo, j = mid, k = lo;
      while (i < mid && j < hi) tmp[k++] = keys[perm[j]] < keys[perm[i]] ? perm[j++] : perm[i++];
      while (i < mid) tmp[k++] = perm[i++];
      while (j < hi) tmp[k++] = perm[j++];
    }
    memcpy(perm, tmp, n * sizeof *perm);
  }
}

void orc_free_blco(orc_blco* b) {
  free(b->keys);
  free(b->offsets);
  free(b->idx);
  free(b->vals);
  memset(b, 0, sizeof *b);
}

int orc_build_blco(const orc_layout* l, uint64_t nnz, const uint64_t* idx, const double* vals,
                   uint64_t max_nnz, orc_blco* out) {
  memset(out, 0, sizeof *out);
  if (max_nnz < 1) return fail("blco: max_nnz_per_block must be >= 1");
  /* types.cpp:13-36 (validate) */
  for (int m = 0; m < l->order; ++m)
    for (uint64_t e = 0; e < nnz; ++e)
      if (idx[(uint64_t)m * nnz + e] >= l->dims[m]) return fail("coo: coordinate out of range");
  orc_u128* altos = malloc((nnz ? nnz : 1) * sizeof *altos);
  uint64_t* perm = malloc((nnz ? nnz : 1) * sizeof *perm);
  uint64_t* tmp = malloc((nnz ? nnz : 1) * sizeof *tmp);
  uint64_t c[ORC_MAX_ORDER];
  for (uint64_t e = 0; e < nnz; ++e) {
    uint64_t hi, lo;
    for (int m = 0; m < l->order; ++m) c[m] = idx[(uint64_t)m * nnz + e];
    orc_linearize(l, c, &hi, &lo);
    altos[e] = ((orc_u128)hi << 64) | lo;
    perm[e] = e;
  }
  msort(perm, tmp, nnz, altos);
  free(tmp);
  const int low = l->total_bits - l->stripped_bits;
  /* blco_format.cpp:86-111: runs of equal key, duplicates rejected, chunks of
   * max_nnz restarting at every run start */
  uint64_t cap = 16, nb = 0;
  uint64_t* keys = malloc(cap * sizeof *keys);
  uint64_t* offs = malloc((cap + 1) * sizeof *offs);
  for (uint64_t e = 0; e < nnz;) {
    const uint64_t key = l->stripped_bits == 0 ? 0 : (uint64_t)(altos[perm[e]] >> low);
    uint64_t f = e + 1;
    if (f < nnz && altos[perm[f]] == altos[perm[e]]) goto dup;
    while (f < nnz && (l->stripped_bits == 0 ? 0 : (uint64_t)(altos[perm[f]] >> low)) == key) {
      if (altos[perm[f]] == altos[perm[f - 1]]) goto dup;
      ++f;
    }
    for (uint64_t s = e; s < f; s += max_nnz) {
      if (nb == cap) {
        cap *= 2;
        keys = realloc(keys, cap * sizeof *keys);
        offs = realloc(offs, (cap + 1) * sizeof *offs);
      }
      keys[nb] = key;
      offs[nb] = s;
      ++nb;
    }
    e = f;
  }
  offs[nb] = nnz;
  out->nblocks = nb;
  out->keys = keys;
  out->offsets = offs;
  out->nnz = nnz;
  out->idx = malloc((nnz ? nnz : 1) * sizeof *out->idx);
  out->vals = malloc((nnz ? nnz : 1) * sizeof *out->vals);
  for (uint64_t e = 0; e < nnz; ++e) {
    uint64_t k, r;
    orc_split_block_key(l, (uint64_t)(altos[perm[e]] >> 64), (uint64_t)altos[perm[e]], &k, &r);
    out->idx[e] = r;
    out->vals[e] = vals[perm[e]];
  }
  free(altos);
  free(perm);
  return ORC_OK;
dup:
  free(altos);
  free(perm);
  free(keys);
  free(offs);
  return fail("blco: duplicate coordinate tuple in input");
}

uint64_t orc_batch_table(const uint64_t* block_nnz, uint64_t nblocks, uint64_t quota,
                         uint64_t* spans) {
  uint64_t n = 0;
  for (uint64_t b = 0; b < nblocks; ++b)
    for (uint64_t off = 0; off < block_nnz[b]; off += quota) {
      if (spans) {
        spans[3 * n] = b;
        spans[3 * n + 1] = off;
        spans[3 * n + 2] = block_nnz[b] - off < quota ? block_nnz[b] - off : quota;
      }
      ++n;
    }
  return n;
}

/* ------------------------------------------------------------------ mttkrp */

int orc_mttkrp_coo(int order, const uint64_t* dims, uint64_t nnz, const uint64_t* idx,
                   const double* vals, const double* const* f, uint64_t rank, int mode,
                   double* out) {
  if (mode < 0 || mode >= order) return fail("mttkrp: mode out of range");
  memset(out, 0, dims[mode] * rank * sizeof *out);
  double* row = malloc(rank * sizeof *row);
  for (uint64_t e = 0; e < nnz; ++e) {
    for (uint64_t r = 0; r < rank; ++r) row[r] = vals[e];
    for (int n = 0; n < order; ++n) {
      if (n == mode) continue;
      const double* a = f[n] + idx[(uint64_t)n * nnz + e] * rank;
      for (uint64_t r = 0; r < rank; ++r) row[r] *= a[r];
    }
    double* dst = out + idx[(uint64_t)mode * nnz + e] * rank;
    for (uint64_t r = 0; r < rank; ++r) dst[r] += row[r];
  }
  free(row);
  return ORC_OK;
}

int orc_mttkrp_blco(const orc_layout* l, const orc_blco* t, const double* const* f,
                    uint64_t rank, int mode, double* out) {
  if (mode < 0 || mode >= l->order) return fail("mttkrp: mode out of range");
  memset(out, 0, l->dims[mode] * rank * sizeof *out);
  double* row = malloc(rank * sizeof *row);
  uint64_t c[ORC_MAX_ORDER];
  for (uint64_t b = 0; b < t->nblocks; ++b)
    for (uint64_t e = t->offsets[b]; e < t->offsets[b + 1]; ++e) {
      orc_delinearize(l, t->idx[e], t->keys[b], c);
      for (uint64_t r = 0; r < rank; ++r) row[r] = t->vals[e];
      for (int n = 0; n < l->order; ++n) {
        if (n == mode) continue;
        const double* a = f[n] + c[n] * rank;
        for (uint64_t r = 0; r < rank; ++r) row[r] *= a[r];
      }
      double* dst = out + c[mode] * rank;
      for (uint64_t r = 0; r < rank; ++r) dst[r] += row[r];
    }
  free(row);
  return ORC_OK;
}

/* -------------------------------------------------------------- generators */

#define GOLDEN 0x9e3779b97f4a7c15ull
#define VALUE_SALT 0x5851f42d4c957f2dull

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static double unit_double(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

void orc_factors_random(const uint64_t* dims, int order, uint64_t rank, uint64_t seed,
                        double* const* out) {
  uint64_t state = seed; /* types.cpp:97-103 */
  for (int m = 0; m < order; ++m)
    for (uint64_t i = 0; i < dims[m] * rank; ++i) {
      state += GOLDEN;
      out[m][i] = unit_double(mix64(state));
    }
}

typedef struct feistel {
  uint64_t cells, mask, key[4];
  int half;
} feistel;

static int feistel_init(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed, feistel* fs) {
  unsigned __int128 cells = 1;
  for (int m = 0; m < order; ++m) cells *= dims[m];
  if (cells > (unsigned __int128)UINT64_MAX) return fail("synth: cell count exceeds 2^64-1");
  fs->cells = (uint64_t)cells;
  if (nnz > fs->cells) return fail("synth: more non-zeros than cells");
  int kb = bits_for(fs->cells);
  if (kb & 1) ++kb;
  if (kb < 2) kb = 2;
  fs->half = kb / 2;
  fs->mask = fs->half == 64 ? ~0ull : ((1ull << fs->half) - 1);
  for (int r = 0; r < 4; ++r) fs->key[r] = mix64(seed + (uint64_t)(r + 1) * GOLDEN);
  return ORC_OK;
}

/* element e -> its cell: keyed 4-round Feistel, cycle-walked into [0, cells) */
static uint64_t feistel_cell(const feistel* fs, uint64_t e) {
  uint64_t x = e;
  do {
    uint64_t L = x >> fs->half, R = x & fs->mask;
    for (int r = 0; r < 4; ++r) {
      const uint64_t F = mix64(R ^ fs->key[r]) & fs->mask;
      const uint64_t nl = R;
      R = L ^ F;
      L = nl;
    }
    x = (L << fs->half) | R;
  } while (x >= fs->cells);
  return x;
}

static double element_value(uint64_t seed, uint64_t e) {
  return unit_double(mix64((seed ^ VALUE_SALT) + (e + 1) * GOLDEN));
}

int orc_synth_uniform(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed,
                      uint64_t* idx, double* vals) {
  feistel fs;
  if (feistel_init(order, dims, nnz, seed, &fs) != ORC_OK) return ORC_EFORMAT;
  for (uint64_t e = 0; e < nnz; ++e) {
    uint64_t x = feistel_cell(&fs, e);
    for (int m = 0; m < order; ++m) {
      idx[(uint64_t)m * nnz + e] = x % dims[m];
      x /= dims[m];
    }
    vals[e] = element_value(seed, e);
  }
  return ORC_OK;
}

/* Row-sampled oracle (SURVEY.md 8c "Large configs"): the rows rows[m][0..k)
 * of mttkrp_coo(T, f, m) for every mode m of the uniform synthetic tensor T
 * = orc_synth_uniform(dims, nnz, seed), without materialising T.  Worker
 * threads filter contiguous element ranges for elements whose mode-m
 * coordinate is sampled; the hits are then accumulated on one thread in
 * element order with mttkrp_coo's product order (oracle.cpp:15-24), so the
 * sampled rows are bit-identical to those of the full oracle. */
#define RS_MAX_ORDER 8

typedef struct hit {
  uint64_t e;
  uint32_t coord[RS_MAX_ORDER];
} hit;

typedef struct rs_job {
  const feistel* fs;
  int order;
  const uint64_t* dims;
  const int32_t* const* slot_of; /* per mode: row -> sample slot or -1 */
  uint64_t e0, e1;
  hit* hits;
  uint64_t nhits, cap;
  int oom;
} rs_job;

static void* rs_worker(void* arg) {
  rs_job* j = arg;
  uint64_t c[ORC_MAX_ORDER];
  for (uint64_t e = j->e0; e < j->e1; ++e) {
    uint64_t x = feistel_cell(j->fs, e);
    int any = 0;
    for (int m = 0; m < j->order; ++m) {
      c[m] = x % j->dims[m];
      x /= j->dims[m];
      any |= j->slot_of[m][c[m]] >= 0;
    }
    if (!any) continue;
    if (j->nhits == j->cap) {
      const uint64_t nc = j->cap ? 2 * j->cap : 4096;
      hit* h = realloc(j->hits, nc * sizeof *h);
      if (!h) {
        j->oom = 1;
        return NULL;
      }
      j->hits = h, j->cap = nc;
    }
    hit* h = &j->hits[j->nhits++];
    h->e = e;
    for (int m = 0; m < j->order; ++m) h->coord[m] = (uint32_t)c[m];
  }
  return NULL;
}

/* Census of the uniform synthetic tensor, streamed from the generator (the
 * COO is never stored): the order-free multiset hash the product computes on
 * a device build (blco_tensor_census: sum of mix64(cell ^ mix64(value bits))
 * mod 2^64) and the number of elements per block key of the target_bits
 * layout (key = the stripped top ALTO bits, layout.cpp:84-95), from which the
 * reference's block chunking (blco_format.cpp:86-111: runs of equal keys cut
 * every max_nnz_per_block elements) follows.  key_counts has 2^stripped
 * entries (stripped <= 20). */
typedef struct census_job {
  const feistel* fs;
  const orc_layout* l;
  uint64_t seed, e0, e1, hash, nkeys;
  uint64_t* counts;
} census_job;

static void* census_worker(void* arg) {
  census_job* j = arg;
  uint64_t c[ORC_MAX_ORDER], h = 0;
  for (uint64_t e = j->e0; e < j->e1; ++e) {
    const uint64_t cell = feistel_cell(j->fs, e);
    uint64_t x = cell;
    for (int m = 0; m < j->l->order; ++m) {
      c[m] = x % j->l->dims[m];
      x /= j->l->dims[m];
    }
    uint64_t key = 0, reenc = 0;
    orc_encode_coords(j->l, c, &key, &reenc);
    if (key < j->nkeys) ++j->counts[key];
    const double v = element_value(j->seed, e);
    uint64_t vb;
    memcpy(&vb, &v, sizeof vb);
    h += mix64(cell ^ mix64(vb));
  }
  j->hash = h;
  return NULL;
}

int orc_census_uniform(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed, int target_bits,
                       int threads, uint64_t* hash, uint64_t* key_counts) {
  orc_layout l;
  if (orc_make_layout(dims, order, target_bits, &l) != ORC_OK) return ORC_EFORMAT;
  if (l.stripped_bits > 20) return fail("census: more than 2^20 block keys");
  feistel fs;
  if (feistel_init(order, dims, nnz, seed, &fs) != ORC_OK) return ORC_EFORMAT;
  const uint64_t nkeys = 1ull << l.stripped_bits;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  census_job jobs[256];
  pthread_t tid[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (census_job){&fs, &l, seed, nnz / threads * t, t + 1 == threads ? nnz : nnz / threads * (t + 1),
                           0, nkeys, calloc(nkeys, sizeof(uint64_t))};
    if (!jobs[t].counts) return fail("census: out of memory");
    pthread_create(&tid[t], NULL, census_worker, &jobs[t]);
  }
  uint64_t h = 0;
  memset(key_counts, 0, nkeys * sizeof(uint64_t));
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    h += jobs[t].hash;
    for (uint64_t k = 0; k < nkeys; ++k) key_counts[k] += jobs[t].counts[k];
    free(jobs[t].counts);
  }
  *hash = h;
  return ORC_OK;
}

/* Row-sampled mttkrp_coo over an in-memory COO (idx mode-major): rows
 * rows[m][0..nrows[m]) of every mode, one pass in COO order with the oracle's
 * product order (oracle.cpp:15-24), so the rows are bit-identical to
 * orc_mttkrp_coo's. */
int orc_rowsample_coo(int order, const uint64_t* dims, uint64_t nnz, const uint64_t* idx, const double* vals,
                      const double* const* f, uint64_t rank, const uint64_t* nrows,
                      const uint64_t* const* rows, double* const* out) {
  if (order < 1 || order > ORC_MAX_ORDER) return fail("rowsample: bad order");
  int32_t* slot_of[ORC_MAX_ORDER] = {0};
  int rc = ORC_OK;
  double* row = malloc(rank * sizeof *row);
  for (int m = 0; m < order; ++m) {
    slot_of[m] = malloc(dims[m] * sizeof(int32_t));
    if (!slot_of[m] || !row) {
      rc = fail("rowsample: out of memory");
      goto done;
    }
    memset(slot_of[m], 0xff, dims[m] * sizeof(int32_t));
    for (uint64_t k = 0; k < nrows[m]; ++k) {
      if (rows[m][k] >= dims[m]) {
        rc = fail("rowsample: row out of range");
        goto done;
      }
      slot_of[m][rows[m][k]] = (int32_t)k;
    }
    memset(out[m], 0, nrows[m] * rank * sizeof(double));
  }
  for (uint64_t e = 0; e < nnz; ++e)
    for (int mode = 0; mode < order; ++mode) {
      const uint64_t c = idx[(uint64_t)mode * nnz + e];
      if (c >= dims[mode]) {
        rc = fail("rowsample: coordinate out of range");
        goto done;
      }
      const int32_t sl = slot_of[mode][c];
      if (sl < 0) continue;
      for (uint64_t r = 0; r < rank; ++r) row[r] = vals[e];
      for (int n = 0; n < order; ++n) {
        if (n == mode) continue;
        const double* a = f[n] + idx[(uint64_t)n * nnz + e] * rank;
        for (uint64_t r = 0; r < rank; ++r) row[r] *= a[r];
      }
      double* dst = out[mode] + (uint64_t)sl * rank;
      for (uint64_t r = 0; r < rank; ++r) dst[r] += row[r];
    }
done:
  for (int m = 0; m < order; ++m) free(slot_of[m]);
  free(row);
  return rc;
}

int orc_rowsample_uniform(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed,
                          const double* const* f, uint64_t rank, const uint64_t* nrows,
                          const uint64_t* const* rows, double* const* out, int threads) {
  if (order < 1 || order > RS_MAX_ORDER) return fail("rowsample: order must lie in [1, 8]");
  feistel fs;
  if (feistel_init(order, dims, nnz, seed, &fs) != ORC_OK) return ORC_EFORMAT;
  int32_t* slot_of[RS_MAX_ORDER] = {0};
  int rc = ORC_OK;
  for (int m = 0; m < order; ++m) {
    slot_of[m] = malloc(dims[m] * sizeof(int32_t));
    if (!slot_of[m]) {
      rc = fail("rowsample: out of memory");
      goto done;
    }
    memset(slot_of[m], 0xff, dims[m] * sizeof(int32_t));
    for (uint64_t k = 0; k < nrows[m]; ++k) {
      if (rows[m][k] >= dims[m]) {
        rc = fail("rowsample: row out of range");
        goto done;
      }
      slot_of[m][rows[m][k]] = (int32_t)k;
    }
    memset(out[m], 0, nrows[m] * rank * sizeof(double));
  }
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  {
    rs_job jobs[256];
    pthread_t tid[256];
    for (int t = 0; t < threads; ++t) {
      jobs[t] = (rs_job){&fs, order, dims, (const int32_t* const*)slot_of,
                         nnz / threads * t, t + 1 == threads ? nnz : nnz / threads * (t + 1), NULL, 0, 0, 0};
      pthread_create(&tid[t], NULL, rs_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    double* row = malloc(rank * sizeof *row);
    for (int t = 0; t < threads; ++t) {
      if (jobs[t].oom) rc = fail("rowsample: out of memory");
      for (uint64_t i = 0; rc == ORC_OK && i < jobs[t].nhits; ++i) {
        const hit* h = &jobs[t].hits[i];
        const double v = element_value(seed, h->e);
        for (int mode = 0; mode < order; ++mode) {
          const int32_t s = slot_of[mode][h->coord[mode]];
          if (s < 0) continue;
          for (uint64_t r = 0; r < rank; ++r) row[r] = v;
          for (int n = 0; n < order; ++n) {
            if (n == mode) continue;
            const double* a = f[n] + (uint64_t)h->coord[n] * rank;
            for (uint64_t r = 0; r < rank; ++r) row[r] *= a[r];
          }
          double* dst = out[mode] + (uint64_t)s * rank;
          for (uint64_t r = 0; r < rank; ++r) dst[r] += row[r];
        }
      }
      free(jobs[t].hits);
    }
    free(row);
  }
done:
  for (int m = 0; m < order; ++m) free(slot_of[m]);
  return rc;
}

/* Independent draws, first nnz distinct tuples in draw order (the product's
 * blco_build_synthetic_draws). */
#define DRAW_SALT 0xd1b54a32d192ed03ull

static uint64_t skewed(double u, uint64_t dim, int k) {
  double p = u;
  for (int i = 1; i < k; ++i) p = p * u;
  const uint64_t c = (uint64_t)(p * (double)dim);
  return c < dim ? c : dim - 1;
}

int orc_synth_draws(int order, const uint64_t* dims, uint64_t nnz, uint64_t seed, int skew,
                    uint64_t* idx, double* vals) {
  uint64_t cap = 16;
  while (cap < 2 * nnz + 16) cap *= 2;
  uint64_t* table = calloc(cap, sizeof *table); /* stores element index + 1 */
  uint64_t kept = 0, c[ORC_MAX_ORDER];
  for (uint64_t j = 0; kept < nnz; ++j) {
    if (j > 64 * (nnz + 1024)) {
      free(table);
      return fail("synth: cannot draw %llu unique coordinates", (unsigned long long)nnz);
    }
    uint64_t h = 0x12345;
    for (int m = 0; m < order; ++m) {
      const double u = unit_double(mix64((seed ^ DRAW_SALT) + (j * order + m + 1) * GOLDEN));
      c[m] = skewed(u, dims[m], skew);
      h = mix64(h ^ (c[m] + GOLDEN * (m + 1)));
    }
    uint64_t s = h & (cap - 1);
    int dup = 0;
    while (table[s]) {
      const uint64_t e = table[s] - 1;
      int same = 1;
      for (int m = 0; m < order && same; ++m) same = idx[(uint64_t)m * nnz + e] == c[m];
      if (same) {
        dup = 1;
        break;
      }
      s = (s + 1) & (cap - 1);
    }
    if (dup) continue;
    for (int m = 0; m < order; ++m) idx[(uint64_t)m * nnz + kept] = c[m];
    vals[kept] = unit_double(mix64((seed ^ VALUE_SALT) + (j + 1) * GOLDEN));
    table[s] = ++kept;
  }
  free(table);
  return ORC_OK;
}

/* ------------------------------------------------------------ dense / ALS */

void orc_gram(const double* a, uint64_t rows, uint64_t rank, double* g) {
  for (uint64_t i = 0; i < rank; ++i)
    for (uint64_t j = i; j < rank; ++j) {
      double s = 0.0;
      for (uint64_t k = 0; k < rows; ++k) s += a[k * rank + i] * a[k * rank + j];
      g[i * rank + j] = s;
      g[j * rank + i] = s;
    }
}

/* dense_kernels.cpp:35-56 */
static int cholesky(const double* v, uint64_t r, double shift, double* L) {
  memset(L, 0, r * r * sizeof *L);
  for (uint64_t i = 0; i < r; ++i)
    for (uint64_t j = 0; j <= i; ++j) {
      double s = v[i * r + j] + (i == j ? shift : 0.0);
      for (uint64_t k = 0; k < j; ++k) s -= L[i * r + k] * L[j * r + k];
      if (i == j) {
        if (!(s > 0.0) || !isfinite(s)) return 0;
        L[i * r + i] = sqrt(s);
      } else {
        L[i * r + j] = s / L[j * r + j];
      }
    }
  return 1;
}

int orc_solve_normal(double* m, uint64_t rows, const double* v, uint64_t r) {
  double trace = 0.0;
  for (uint64_t i = 0; i < r; ++i) trace += v[i * r + i];
  const double unit = trace > 0.0 ? trace / (double)r : 1.0;
  double* L = malloc(r * r * sizeof *L);
  int ok = cholesky(v, r, 0.0, L);
  for (double lam = 1e-12 * unit; !ok && lam <= 1e-3 * unit * (1.0 + 1e-9); lam *= 10.0)
    ok = cholesky(v, r, lam, L);
  if (!ok) {
    free(L);
    return fail("solve_normal: matrix singular after maximal diagonal shift");
  }
  for (uint64_t row = 0; row < rows; ++row) {
    double* b = m + row * r;
    for (uint64_t i = 0; i < r; ++i) {
      double s = b[i];
      for (uint64_t k = 0; k < i; ++k) s -= L[i * r + k] * b[k];
      b[i] = s / L[i * r + i];
    }
    for (uint64_t ii = r; ii-- > 0;) {
      double s = b[ii];
      for (uint64_t k = ii + 1; k < r; ++k) s -= L[k * r + ii] * b[k];
      b[ii] = s / L[ii * r + ii];
    }
  }
  free(L);
  return ORC_OK;
}

/* cpals.cpp:51-62 */
static void normalize_columns(double* a, uint64_t rows, uint64_t rank, double* lambda) {
  for (uint64_t r = 0; r < rank; ++r) lambda[r] = 0.0;
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t r = 0; r < rank; ++r) lambda[r] += a[i * rank + r] * a[i * rank + r];
  for (uint64_t r = 0; r < rank; ++r) {
    lambda[r] = sqrt(lambda[r]);
    if (lambda[r] == 0.0) lambda[r] = 1.0;
  }
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t r = 0; r < rank; ++r) a[i * rank + r] /= lambda[r];
}

int orc_cp_als(const orc_layout* l, const orc_blco* t, uint64_t rank, int max_iters, double tol,
               uint64_t seed, double* const* A, double* lambda, double* fit_out) {
  const int N = l->order;
  orc_factors_random(l->dims, N, rank, seed, A);
  for (uint64_t r = 0; r < rank; ++r) lambda[r] = 1.0;
  if (max_iters == 0) return 0;
  double xn = 0.0; /* cpals.cpp:13-18, block order */
  for (uint64_t e = 0; e < t->nnz; ++e) xn += t->vals[e] * t->vals[e];
  if (xn == 0.0) return -fail("cp_als: zero-norm tensor");
  double* grams = malloc((size_t)N * rank * rank * sizeof *grams);
  double* v = malloc(rank * rank * sizeof *v);
  for (int n = 0; n < N; ++n) orc_gram(A[n], l->dims[n], rank, grams + n * rank * rank);
  uint64_t maxrows = 0;
  for (int n = 0; n < N; ++n) maxrows = l->dims[n] > maxrows ? l->dims[n] : maxrows;
  double* mt = malloc(maxrows * rank * sizeof *mt);
  double* mlast = malloc(l->dims[N - 1] * rank * sizeof *mlast);
  double prev = 0.0;
  int it;
  for (it = 0; it < max_iters; ++it) {
    for (int n = 0; n < N; ++n) {
      for (uint64_t i = 0; i < rank * rank; ++i) v[i] = 1.0;
      for (int m = 0; m < N; ++m)
        if (m != n)
          for (uint64_t i = 0; i < rank * rank; ++i) v[i] *= grams[m * rank * rank + i];
      orc_mttkrp_blco(l, t, (const double* const*)A, rank, n, mt);
      if (n == N - 1) memcpy(mlast, mt, l->dims[n] * rank * sizeof *mt);
      if (orc_solve_normal(mt, l->dims[n], v, rank) != ORC_OK) {
        it = -1;
        goto done;
      }
      memcpy(A[n], mt, l->dims[n] * rank * sizeof *mt);
      normalize_columns(A[n], l->dims[n], rank, lambda);
      orc_gram(A[n], l->dims[n], rank, grams + n * rank * rank);
    }
    /* cpals.cpp:21-49 fit identity */
    double inner = 0.0;
    for (uint64_t i = 0; i < l->dims[N - 1]; ++i)
      for (uint64_t r = 0; r < rank; ++r)
        inner += mlast[i * rank + r] * lambda[r] * A[N - 1][i * rank + r];
    for (uint64_t i = 0; i < rank * rank; ++i) v[i] = 1.0;
    for (int m = 0; m < N; ++m)
      for (uint64_t i = 0; i < rank * rank; ++i) v[i] *= grams[m * rank * rank + i];
    double hat = 0.0;
    for (uint64_t r = 0; r < rank; ++r)
      for (uint64_t c = 0; c < rank; ++c) hat += v[r * rank + c] * lambda[r] * lambda[c];
    double resid = xn - 2.0 * inner + hat;
    if (resid < 0.0) resid = 0.0;
    const double f = 1.0 - sqrt(resid) / sqrt(xn);
    fit_out[it] = f;
    if (!isfinite(f)) {
      it = -2;
      fail("cp_als: non-finite fit at iteration %d", it + 1);
      goto done;
    }
    if (it > 0 && f - prev < tol) {
      ++it;
      break;
    }
    prev = f;
  }
done:
  free(grams);
  free(v);
  free(mt);
  free(mlast);
  return it;
}

/* Batch ALTO low words (layout.cpp:71-82 per element; total_bits <= 64 only).
 * Used by bench.py to cut a contiguous ALTO-order sample of a synthetic
 * tensor for the reference CPU timing. */
int orc_alto_lo_batch(const orc_layout* l, uint64_t nnz, const uint64_t* idx, uint64_t* out) {
  if (l->total_bits > 64) return fail("orc_alto_lo_batch: layout wider than 64 bits");
  for (uint64_t e = 0; e < nnz; ++e) {
    uint64_t a = 0;
    for (int m = 0; m < l->order; ++m) {
      const uint64_t c = idx[(uint64_t)m * nnz + e];
      for (int k = 0; k < l->mode_bits[m]; ++k) a |= ((c >> k) & 1u) << l->mode_pos[m][k];
    }
    out[e] = a;
  }
  return ORC_OK;
}
