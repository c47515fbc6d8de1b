/*
 * sgnn_oracle.c -- TEST INFRASTRUCTURE ONLY (see sgnn_oracle.h).
 *
 * Single-threaded C restatement of the reference algorithms. Each function
 * names the reference file:line it follows (paths relative to
 * /root/reference/proj/include/sgnn/). Compile with -ffp-contract=off so every
 * `acc += a*b` rounds the product and the sum separately, exactly like the
 * reference build (g++ -std=c++20 -O3 without -march, hence no FMA).
 */
#include "sgnn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ===================================================================== */
/* rng.hpp:13-42  splitmix64                                              */
/* ===================================================================== */
typedef struct {
  uint64_t state;
} orc_rng;

static orc_rng rng_make(uint64_t seed) {
  orc_rng r;
  r.state = seed + 0x9E3779B97F4A7C15ull; /* rng.hpp:15 */
  return r;
}
static uint64_t rng_next(orc_rng* r) { /* rng.hpp:17-23 */
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t rng_below(orc_rng* r, uint64_t bound) { /* rng.hpp:26-32 */
  if (bound <= 1) return 0;
  const uint64_t limit = bound * ((~(uint64_t)0) / bound);
  uint64_t x = rng_next(r);
  while (x >= limit) x = rng_next(r);
  return x % bound;
}
static double rng_double(orc_rng* r) { /* rng.hpp:35 */
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}
static double rng_double_range(orc_rng* r, double lo, double hi) { /* rng.hpp:38 */
  return lo + (hi - lo) * rng_double(r);
}

void orc_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
  orc_rng r = rng_make(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_next(&r);
}
void orc_rng_below(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out) {
  orc_rng r = rng_make(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_below(&r, bound);
}

/* dense.hpp:45-53 DenseMatrix::random_uniform (draw in double, narrow) */
void orc_random_uniform(int64_t rows, int64_t cols, uint64_t seed, double lo, double hi,
                        double* out) {
  orc_rng r = rng_make(seed);
  const int64_t n = rows * cols;
  for (int64_t i = 0; i < n; ++i) out[i] = rng_double_range(&r, lo, hi);
}
void orc_random_uniform_f32(int64_t rows, int64_t cols, uint64_t seed, double lo, double hi,
                            float* out) {
  orc_rng r = rng_make(seed);
  const int64_t n = rows * cols;
  for (int64_t i = 0; i < n; ++i) out[i] = (float)rng_double_range(&r, lo, hi);
}

/* ===================================================================== */
/* graph.hpp:160-190 synthetic_graph                                      */
/* ===================================================================== */
int64_t orc_synthetic_graph_edges(int32_t n, double avg_degree) {
  const uint64_t pairs = (uint64_t)(avg_degree * (double)n / 2.0 + 0.5); /* graph.hpp:169-170 */
  return (int64_t)(2 * pairs);
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* open-addressing set of non-zero 64-bit keys (stand-in for unordered_set) */
typedef struct {
  uint64_t* slots;
  uint64_t mask;
  uint64_t size;
} u64set;
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdull;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ull;
  return z ^ (z >> 33);
}
static int u64set_insert(u64set* s, uint64_t key) { /* key stored +1 so 0 is empty */
  uint64_t k = key + 1, h = mix64(k) & s->mask;
  while (s->slots[h]) {
    if (s->slots[h] == k) return 0;
    h = (h + 1) & s->mask;
  }
  s->slots[h] = k;
  s->size++;
  return 1;
}

int orc_synthetic_graph(int32_t n, double avg_degree, uint64_t seed, int32_t* src,
                        int32_t* dst) {
  if (n < 1 || avg_degree < 0 || !(avg_degree < (double)n)) return -1; /* graph.hpp:161-163 */
  const uint64_t target = (uint64_t)(avg_degree * (double)n / 2.0 + 0.5);
  if (target == 0) return 0;
  uint64_t cap = 16;
  while (cap < target * 4) cap <<= 1;
  u64set set;
  set.slots = (uint64_t*)calloc(cap, sizeof(uint64_t));
  set.mask = cap - 1;
  set.size = 0;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * 2 * target);
  orc_rng r = rng_make(seed);
  uint64_t ne = 0;
  while (set.size < target) { /* graph.hpp:177-187 */
    const int32_t a = (int32_t)rng_below(&r, (uint64_t)n);
    const int32_t b = (int32_t)rng_below(&r, (uint64_t)n);
    if (a == b) continue;
    const int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    const uint64_t key = ((uint64_t)lo << 32) | (uint32_t)hi;
    if (!u64set_insert(&set, key)) continue;
    keys[ne++] = ((uint64_t)lo << 32) | (uint32_t)hi;
    keys[ne++] = ((uint64_t)hi << 32) | (uint32_t)lo;
  }
  /* dedup_edges (graph.hpp:42-55): stable sort by (src,dst); all keys unique */
  qsort(keys, ne, sizeof(uint64_t), cmp_u64);
  for (uint64_t i = 0; i < ne; ++i) {
    src[i] = (int32_t)(keys[i] >> 32);
    dst[i] = (int32_t)(keys[i] & 0xffffffffu);
  }
  free(keys);
  free(set.slots);
  return 0;
}

/* ===================================================================== */
/* sparse.hpp                                                             */
/* ===================================================================== */
typedef struct {
  uint64_t key;
  int64_t idx;
} keyed;
static int cmp_keyed(const void* a, const void* b) {
  const keyed* x = (const keyed*)a;
  const keyed* y = (const keyed*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0); /* stability */
}

/* sparse.hpp:110-142 coo_from_triplets: range check, stable sort, keep last */
int64_t orc_coo_canonicalize(int32_t n_rows, int32_t n_cols, int64_t nnz, const int32_t* rows,
                             const int32_t* cols, const double* vals, int32_t* out_rows,
                             int32_t* out_cols, double* out_vals) {
  for (int64_t i = 0; i < nnz; ++i)
    if (rows[i] < 0 || rows[i] >= n_rows || cols[i] < 0 || cols[i] >= n_cols) return -1;
  keyed* t = (keyed*)malloc(sizeof(keyed) * (nnz > 0 ? nnz : 1));
  for (int64_t i = 0; i < nnz; ++i) {
    t[i].key = ((uint64_t)(uint32_t)rows[i] << 32) | (uint32_t)cols[i];
    t[i].idx = i;
  }
  qsort(t, nnz, sizeof(keyed), cmp_keyed);
  int64_t w = 0;
  for (int64_t i = 0; i < nnz; ++i) {
    if (w > 0 && ((uint64_t)(uint32_t)out_rows[w - 1] << 32 | (uint32_t)out_cols[w - 1]) ==
                     t[i].key) {
      out_vals[w - 1] = vals[t[i].idx]; /* keep last (sparse.hpp:119-121) */
    } else {
      out_rows[w] = rows[t[i].idx];
      out_cols[w] = cols[t[i].idx];
      out_vals[w] = vals[t[i].idx];
      ++w;
    }
  }
  free(t);
  return w;
}

/* sparse.hpp:151-171 coo_to_csr (entries already canonical) */
void orc_coo_to_csr(int32_t n_rows, int64_t nnz, const int32_t* rows, int32_t* rowptr) {
  memset(rowptr, 0, sizeof(int32_t) * ((size_t)n_rows + 1));
  for (int64_t e = 0; e < nnz; ++e) rowptr[rows[e] + 1]++;
  for (int32_t i = 0; i < n_rows; ++i) rowptr[i + 1] += rowptr[i];
}

/* sparse.hpp:195-218 coo_to_csc: counting sort, rows ascend within a column.
 * perm[at] = canonical index (the SparsePattern convention, pattern.hpp:35-44) */
void orc_coo_to_csc(int32_t n_cols, int64_t nnz, const int32_t* rows, const int32_t* cols,
                    const double* vals, int32_t* colptr, int32_t* out_rows, double* out_vals,
                    int32_t* perm) {
  memset(colptr, 0, sizeof(int32_t) * ((size_t)n_cols + 1));
  for (int64_t e = 0; e < nnz; ++e) colptr[cols[e] + 1]++;
  for (int32_t j = 0; j < n_cols; ++j) colptr[j + 1] += colptr[j];
  int32_t* fill = (int32_t*)calloc((size_t)n_cols + 1, sizeof(int32_t));
  for (int64_t e = 0; e < nnz; ++e) {
    const int32_t j = cols[e];
    const int32_t at = colptr[j] + fill[j]++;
    if (out_rows) out_rows[at] = rows[e];
    if (out_vals) out_vals[at] = vals[e];
    if (perm) perm[at] = (int32_t)e;
  }
  free(fill);
}

/* sparse.hpp:457-472 add_self_loops: (i,i,1) where the diagonal is absent,
 * existing diagonal values kept, result canonical */
int64_t orc_add_self_loops(int32_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                           const double* vals, int32_t* out_rows, int32_t* out_cols,
                           double* out_vals) {
  unsigned char* has = (unsigned char*)calloc((size_t)n + 1, 1);
  for (int64_t e = 0; e < nnz; ++e)
    if (rows[e] == cols[e]) has[rows[e]] = 1;
  /* merge: input is canonical, so insert each missing diagonal in place */
  int64_t w = 0, e = 0;
  for (int32_t i = 0; i < n; ++i) {
    while (e < nnz && rows[e] == i && cols[e] < i) {
      out_rows[w] = rows[e]; out_cols[w] = cols[e]; out_vals[w] = vals[e]; ++w; ++e;
    }
    if (!has[i]) { out_rows[w] = i; out_cols[w] = i; out_vals[w] = 1.0; ++w; }
    while (e < nnz && rows[e] == i) {
      out_rows[w] = rows[e]; out_cols[w] = cols[e]; out_vals[w] = vals[e]; ++w; ++e;
    }
  }
  free(has);
  return w;
}

/* sparse.hpp:474-495 gcn_normalize: degrees of A+I in double, in canonical
 * order; v <- S(double(v) / sqrt(d_i * d_j)) */
int64_t orc_gcn_normalize(int32_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                          const double* vals, int32_t* out_rows, int32_t* out_cols,
                          double* out_vals) {
  const int64_t q = orc_add_self_loops(n, nnz, rows, cols, vals, out_rows, out_cols, out_vals);
  double* deg = (double*)calloc((size_t)n + 1, sizeof(double));
  for (int64_t e = 0; e < q; ++e) {
    if (out_vals[e] < 0.0) { free(deg); return -1; }
    deg[out_rows[e]] += out_vals[e];
  }
  for (int64_t e = 0; e < q; ++e)
    out_vals[e] = out_vals[e] / sqrt(deg[out_rows[e]] * deg[out_cols[e]]);
  free(deg);
  return q;
}

int64_t orc_gcn_normalize_f32(int32_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                              const float* vals, int32_t* out_rows, int32_t* out_cols,
                              float* out_vals) {
  double* v = (double*)malloc(sizeof(double) * (nnz + 1));
  double* o = (double*)malloc(sizeof(double) * (nnz + n + 1));
  for (int64_t e = 0; e < nnz; ++e) v[e] = (double)vals[e];
  const int64_t q = orc_add_self_loops(n, nnz, rows, cols, v, out_rows, out_cols, o);
  double* deg = (double*)calloc((size_t)n + 1, sizeof(double));
  int64_t ret = q;
  for (int64_t e = 0; e < q; ++e) {
    if (o[e] < 0.0) { ret = -1; break; }
    deg[out_rows[e]] += o[e]; /* static_cast<double>(float) is exact */
  }
  if (ret >= 0)
    for (int64_t e = 0; e < q; ++e)
      out_vals[e] = (float)(o[e] / sqrt(deg[out_rows[e]] * deg[out_cols[e]]));
  free(deg); free(v); free(o);
  return ret;
}

/* ===================================================================== */
/* pattern.hpp:19-59 SparsePattern::build                                 */
/* ===================================================================== */
int orc_pattern_build(int32_t n, const int32_t* rowptr, const int32_t* cols, int32_t* colptr,
                      int32_t* rows, int32_t* perm, int32_t* diag) {
  const int64_t q = rowptr[n];
  memset(colptr, 0, sizeof(int32_t) * ((size_t)n + 1));
  for (int64_t e = 0; e < q; ++e) colptr[cols[e] + 1]++;
  for (int32_t j = 0; j < n; ++j) colptr[j + 1] += colptr[j];
  int32_t* fill = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  for (int32_t i = 0; i < n; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int32_t j = cols[e];
      const int32_t at = colptr[j] + fill[j]++;
      rows[at] = i;
      perm[at] = e;
    }
  free(fill);
  int all = 1;
  for (int32_t i = 0; i < n; ++i) {
    diag[i] = -1;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
      if (cols[e] == i) { diag[i] = e; break; }
    if (diag[i] < 0) all = 0;
  }
  return all;
}

/* ===================================================================== */
/* kernels.hpp                                                            */
/* ===================================================================== */
/* kernels.hpp:33-53 spmm_csr_into: zero-init, per row in stored order */
void orc_spmm_csr(int32_t n_rows, const int32_t* rowptr, const int32_t* cols, const double* vals,
                  const double* B, int32_t f, double* C) {
  memset(C, 0, sizeof(double) * (size_t)n_rows * f);
  for (int32_t i = 0; i < n_rows; ++i) {
    double* crow = C + (size_t)i * f;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const double v = vals[e];
      const double* brow = B + (size_t)cols[e] * f;
      for (int32_t c = 0; c < f; ++c) crow[c] += v * brow[c];
    }
  }
}
void orc_spmm_csr_f32(int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                      const float* vals, const float* B, int32_t f, float* C) {
  memset(C, 0, sizeof(float) * (size_t)n_rows * f);
  for (int32_t i = 0; i < n_rows; ++i) {
    float* crow = C + (size_t)i * f;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const float v = vals[e];
      const float* brow = B + (size_t)cols[e] * f;
      for (int32_t c = 0; c < f; ++c) crow[c] += v * brow[c];
    }
  }
}

/* kernels.hpp:301-337 sddmm without scale: out_e = dot(B row i, C column j) */
void orc_sddmm(int32_t n, const int32_t* rowptr, const int32_t* cols, const double* B,
               int32_t f, const double* C, int32_t ldc, double* out) {
  for (int32_t i = 0; i < n; ++i) {
    const double* brow = B + (size_t)i * f;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int32_t j = cols[e];
      double acc = 0.0;
      for (int32_t l = 0; l < f; ++l) acc += brow[l] * C[(size_t)l * ldc + j];
      out[e] = 1.0 * acc;
    }
  }
}

/* kernels.hpp:500-534 edge_softmax (head-major h x q); needs self loops */
int orc_edge_softmax(int32_t n, const int32_t* rowptr, int64_t q, int32_t heads,
                     const double* w, double* alpha) {
  for (int32_t i = 0; i < n; ++i)
    for (int32_t t = 0; t < heads; ++t) {
      const double* wh = w + (size_t)t * q;
      double* oh = alpha + (size_t)t * q;
      if (rowptr[i] == rowptr[i + 1]) return -1;
      double gmax = wh[rowptr[i]];
      for (int32_t e = rowptr[i] + 1; e < rowptr[i + 1]; ++e) gmax = wh[e] > gmax ? wh[e] : gmax;
      double sum = 0.0;
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        const double x = exp(wh[e] - gmax);
        oh[e] = x;
        sum += x;
      }
      const double inv = 1.0 / sum;
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) oh[e] *= inv;
    }
  return 0;
}

/* kernels.hpp:219-254 spmm_semibatched */
void orc_spmm_semibatched(int32_t n, const int32_t* rowptr, const int32_t* cols, int64_t q,
                          int32_t h, int32_t k, const double* alpha, const double* B, double* C) {
  memset(C, 0, sizeof(double) * (size_t)n * h * k);
  for (int32_t i = 0; i < n; ++i) {
    double* crow = C + (size_t)i * h * k;
    for (int32_t t = 0; t < h; ++t) {
      const double* ah = alpha + (size_t)t * q;
      double* cs = crow + (size_t)t * k;
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        const double v = ah[e];
        const double* bs = B + ((size_t)cols[e] * h + t) * k;
        for (int32_t c = 0; c < k; ++c) cs[c] += v * bs[c];
      }
    }
  }
}

/* kernels.hpp:258-295 spmm_semibatched_transposed (column-grouped + perm) */
static void spmm_semibatched_transposed(int32_t n, const int32_t* colptr, const int32_t* crows,
                                        const int32_t* perm, int64_t q, int32_t h, int32_t k,
                                        const double* alpha, const double* B, double* C) {
  memset(C, 0, sizeof(double) * (size_t)n * h * k);
  for (int32_t j = 0; j < n; ++j) {
    double* crow = C + (size_t)j * h * k;
    for (int32_t t = 0; t < h; ++t) {
      const double* ah = alpha + (size_t)t * q;
      double* cs = crow + (size_t)t * k;
      for (int32_t e = colptr[j]; e < colptr[j + 1]; ++e) {
        const double v = ah[perm[e]];
        const double* bs = B + ((size_t)crows[e] * h + t) * k;
        for (int32_t c = 0; c < k; ++c) cs[c] += v * bs[c];
      }
    }
  }
}

/* ===================================================================== */
/* dense.hpp                                                              */
/* ===================================================================== */
/* dense.hpp:97-157 gemm with the four transpose loop orders */
int orc_gemm(const double* A, int32_t ra, int32_t ca, const double* B, int32_t rb, int32_t cb,
             int trans_a, int trans_b, double* C) {
  const int32_t m = trans_a ? ca : ra;
  const int32_t kk = trans_a ? ra : ca;
  const int32_t kb = trans_b ? cb : rb;
  const int32_t n = trans_b ? rb : cb;
  if (kk != kb) return -1;
  const int32_t lda = ca, ldb = cb;
  memset(C, 0, sizeof(double) * (size_t)m * n);
  for (int32_t i = 0; i < m; ++i) {
    double* crow = C + (size_t)i * n;
    if (!trans_a && !trans_b) {
      const double* arow = A + (size_t)i * lda;
      for (int32_t l = 0; l < kk; ++l) {
        const double a = arow[l];
        const double* brow = B + (size_t)l * ldb;
        for (int32_t j = 0; j < n; ++j) crow[j] += a * brow[j];
      }
    } else if (trans_a && !trans_b) {
      for (int32_t l = 0; l < kk; ++l) {
        const double a = A[(size_t)l * lda + i];
        const double* brow = B + (size_t)l * ldb;
        for (int32_t j = 0; j < n; ++j) crow[j] += a * brow[j];
      }
    } else if (!trans_a && trans_b) {
      const double* arow = A + (size_t)i * lda;
      for (int32_t j = 0; j < n; ++j) {
        const double* brow = B + (size_t)j * ldb;
        double acc = 0.0;
        for (int32_t l = 0; l < kk; ++l) acc += arow[l] * brow[l];
        crow[j] += acc;
      }
    } else {
      for (int32_t j = 0; j < n; ++j) {
        const double* brow = B + (size_t)j * ldb;
        double acc = 0.0;
        for (int32_t l = 0; l < kk; ++l) acc += A[(size_t)l * lda + i] * brow[l];
        crow[j] += acc;
      }
    }
  }
  return 0;
}

/* dense.hpp:159-170 bias_add_rows_inplace */
static void bias_add_rows(double* X, int32_t rows, int32_t cols, const double* b) {
  for (int32_t i = 0; i < rows; ++i) {
    double* row = X + (size_t)i * cols;
    for (int32_t j = 0; j < cols; ++j) row[j] += b[j];
  }
}

/* dense.hpp:272-282 column_sums */
void orc_column_sums(const double* X, int32_t rows, int32_t cols, double* out) {
  for (int32_t j = 0; j < cols; ++j) out[j] = 0.0;
  for (int32_t i = 0; i < rows; ++i) {
    const double* row = X + (size_t)i * cols;
    for (int32_t j = 0; j < cols; ++j) out[j] += row[j];
  }
}

/* dense.hpp:303-316 max_rel_diff: |a-b| / max(1,|a|,|b|) */
double orc_max_rel_diff(const double* a, const double* b, int64_t n) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double d = fabs(a[i]), e = fabs(b[i]);
    double den = 1.0;
    if (d > den) den = d;
    if (e > den) den = e;
    const double r = fabs(a[i] - b[i]) / den;
    if (r > m || r != r) m = r != r ? INFINITY : r;
  }
  return m;
}
double orc_max_rel_diff_f32(const float* a, const double* b, int64_t n) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = (double)a[i];
    double den = 1.0;
    if (fabs(x) > den) den = fabs(x);
    if (fabs(b[i]) > den) den = fabs(b[i]);
    const double r = fabs(x - b[i]) / den;
    if (r > m || r != r) m = r != r ? INFINITY : r;
  }
  return m;
}

/* dense.hpp:196-229 activation (relu=0, leaky=1, elu=2) */
void orc_activation(const double* X, int64_t n, int kind, double param, double* out,
                    uint8_t* mask) {
  const double alpha = kind == 2 ? (param > 0 ? param : 1.0) : 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double x = X[i];
    const int pos = x > 0.0;
    mask[i] = (uint8_t)pos;
    if (kind == 0) out[i] = pos ? x : 0.0;
    else if (kind == 1) out[i] = pos ? x : param * x;
    else out[i] = pos ? x : alpha * (exp(x) - 1.0);
  }
}
/* dense.hpp:231-270 activation_backward */
void orc_activation_backward(const double* g, const uint8_t* mask, int64_t n, int kind,
                             double param, const double* saved, double* out) {
  const double alpha = kind == 2 ? (param > 0 ? param : 1.0) : 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (mask[i]) out[i] = g[i];
    else if (kind == 0) out[i] = 0.0;
    else if (kind == 1) out[i] = param * g[i];
    else out[i] = (saved[i] + alpha) * g[i];
  }
}
/* model.hpp:228-245 loss_mse */
double orc_loss_mse(const double* out, const double* target, int64_t n, double* grad) {
  const double inv = 1.0 / (double)n;
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = out[i] - target[i];
    acc += d * d;
    grad[i] = 2.0 * d * inv;
  }
  return acc * inv;
}

/* ===================================================================== */
/* cost.hpp                                                               */
/* ===================================================================== */
static int sparse_bytes(int fmt, int64_t n, int64_t q, int64_t p, int64_t sb, int64_t ib,
                        int64_t* out) { /* cost.hpp:44-60 */
  switch (fmt) {
    case 1: case 2: *out = ib * (q + n + 1) + sb * q; return 0;
    case 0: *out = ib * 2 * q + sb * q; return 0;
    case 3: if (p <= 0) return -1; *out = (ib + sb) * n * p; return 0;
    default: return -1;
  }
}
static double oi_of(int64_t flops, int64_t bytes) {
  return bytes > 0 ? (double)flops / (double)bytes : 0.0;
}
int orc_spmm_cost(int fmt, int64_t n, int64_t q, int64_t p, int64_t f, int64_t sb, int64_t ib,
                  int64_t* flops, int64_t* bytes, double* oi) { /* cost.hpp:63-69 */
  int64_t sbytes;
  if (sparse_bytes(fmt, n, q, p, sb, ib, &sbytes)) return -1;
  *flops = 2 * q * f;
  *bytes = sbytes + 3 * sb * n * f;
  *oi = oi_of(*flops, *bytes);
  return 0;
}
int orc_sddmm_cost(int fmt, int64_t n, int64_t q, int64_t p, int64_t f, int64_t sb, int64_t ib,
                   int64_t* flops, int64_t* bytes, double* oi) { /* cost.hpp:81-101 */
  *flops = q * (2 * f + 1);
  int64_t b = sb * q * f;
  switch (fmt) {
    case 1: case 2: b += ib * (q + n + 1) + 2 * sb * q; break;
    case 0: b += ib * 2 * q + 2 * sb * q; break;
    case 3: if (p <= 0) return -1; b += ib * n * p + 2 * sb * q; break;
    default: return -1;
  }
  *bytes = b;
  *oi = oi_of(*flops, *bytes);
  return 0;
}
/* cost.hpp:201-223 gcn_select_scheme */
int orc_gcn_select_scheme(int64_t m, int64_t k, int fg, int caching, int* fwd, int* bwd,
                          int* cached) {
  if (!(m >= 1 && k >= 1)) return -1;
  if (!caching) {
    *fwd = k < m ? 0 : 1;
    const int fused = fg ? (k < 2 * m) : (k < m);
    *bwd = fused ? 0 : 1;
    *cached = 0;
  } else {
    const int transform = fg ? (k < m) : (2 * k < m);
    if (transform) { *fwd = 0; *bwd = 0; *cached = 0; }
    else { *fwd = 2; *bwd = 2; *cached = 1; }
  }
  return 0;
}
/* gcn.hpp:34-47 resolve_scheme; policy 0 adaptive, 1 force TF, 2 force PF */
int orc_resolve_scheme(int policy, int64_t m, int64_t k, int fg, int caching, int* fwd,
                       int* bwd, int* cached) {
  switch (policy) {
    case 0: return orc_gcn_select_scheme(m, k, fg, caching, fwd, bwd, cached);
    case 1: *fwd = 0; *bwd = 0; *cached = 0; return 0;
    case 2:
      if (caching) { *fwd = 2; *bwd = 2; *cached = 1; }
      else { *fwd = 1; *bwd = 1; *cached = 0; }
      return 0;
  }
  return -1;
}
int64_t orc_gcn_forward_flops(int s, int64_t n, int64_t m, int64_t k, int64_t q) {
  return s == 0 ? 2 * (n * m * k + q * k) : 2 * (n * m * k + q * m); /* cost.hpp:143-152 */
}
int64_t orc_gcn_backward_flops(int s, int64_t n, int64_t m, int64_t k, int64_t q, int fg) {
  switch (s) { /* cost.hpp:154-169 */
    case 0: return 2 * q * k + 2 * n * m * k + (fg ? 2 * n * m * k : 0);
    case 1: return 2 * q * m + 2 * n * m * k + (fg ? 2 * n * m * k + 2 * q * m : 0);
    case 2: return 2 * n * m * k + (fg ? 2 * n * m * k + 2 * q * m : 0);
  }
  return 0;
}
int64_t orc_gcn_forward_transients(int s, int64_t n, int64_t m, int64_t k) {
  return s == 0 ? n * k : n * m; /* cost.hpp:178-185 */
}
int64_t orc_gcn_backward_transients(int s, int64_t n, int64_t m, int64_t k, int fg) {
  switch (s) { /* cost.hpp:187-197 */
    case 0: return n * k;
    case 1: return fg ? 2 * n * m : n * m;
    case 2: return fg ? n * m : 0;
  }
  return 0;
}
int64_t orc_gat_cache_footprint(int level, int64_t n, int64_t h, int64_t k, int64_t q,
                                int64_t sb) { /* cost.hpp:243-252 */
  switch (level) {
    case 0: return 0;
    case 1: return sb * n * h * k;
    case 2: return sb * n * h * (k + 2);
    case 3: return sb * n * h * k + (sb + 1) * q * h;
  }
  return 0;
}

/* ===================================================================== */
/* gcn.hpp                                                                */
/* ===================================================================== */
/* gcn.hpp:54-62 GcnParams::init */
void orc_gcn_params_init(int32_t m, int32_t k, uint64_t seed, double* theta, double* bias) {
  const double bound = 1.0 / sqrt((double)m);
  orc_random_uniform(m, k, seed, -bound, bound, theta);
  orc_rng r = rng_make(seed + 1);
  for (int32_t j = 0; j < k; ++j) bias[j] = rng_double_range(&r, -bound, bound);
}

/* gcn.hpp:91-131 gcn_forward */
int orc_gcn_forward(int32_t n, const int32_t* rowptr, const int32_t* cols, const double* vals,
                    const double* X, int32_t m, const double* theta, const double* bias,
                    int32_t k, int fwd_scheme, double* out, double* P_out) {
  if (fwd_scheme == 0) {
    double* M = (double*)malloc(sizeof(double) * (size_t)n * k + 8);
    orc_gemm(X, n, m, theta, m, k, 0, 0, M);
    orc_spmm_csr(n, rowptr, cols, vals, M, k, out);
    free(M);
  } else {
    double* P = P_out ? P_out : (double*)malloc(sizeof(double) * (size_t)n * m + 8);
    orc_spmm_csr(n, rowptr, cols, vals, X, m, P);
    orc_gemm(P, n, m, theta, m, k, 0, 0, out);
    if (!P_out) free(P);
  }
  bias_add_rows(out, n, k, bias);
  return 0;
}

/* gcn.hpp:133-193 gcn_backward; A'^T products use the CSC arrays as a CSR of
 * A'^T (the zero-copy transpose of sparse.hpp:400-420). */
int orc_gcn_backward(int32_t n, const int32_t* rowptr, const int32_t* cols, const double* vals,
                     const int32_t* colptr, const int32_t* crows, const double* cvals,
                     const double* d_out, const double* saved, int32_t m, const double* theta,
                     int32_t k, int bwd_scheme, int fg, double* d_theta, double* d_bias,
                     double* d_input) {
  orc_column_sums(d_out, n, k, d_bias);
  if (bwd_scheme == 0) {
    double* S = (double*)malloc(sizeof(double) * (size_t)n * k + 8);
    orc_spmm_csr(n, colptr, crows, cvals, d_out, k, S);
    orc_gemm(saved, n, m, S, n, k, 1, 0, d_theta);
    if (fg) orc_gemm(S, n, k, theta, m, k, 0, 1, d_input);
    free(S);
  } else {
    double* P = NULL;
    const double* Pc = saved;
    if (bwd_scheme == 1) {
      P = (double*)malloc(sizeof(double) * (size_t)n * m + 8);
      orc_spmm_csr(n, rowptr, cols, vals, saved, m, P);
      Pc = P;
    }
    double* G = NULL;
    if (fg && bwd_scheme == 1) {
      G = (double*)malloc(sizeof(double) * (size_t)n * m + 8);
      orc_gemm(d_out, n, k, theta, m, k, 0, 1, G);
    }
    orc_gemm(Pc, n, m, d_out, n, k, 1, 0, d_theta);
    if (fg) {
      if (!G) {
        G = (double*)malloc(sizeof(double) * (size_t)n * m + 8);
        orc_gemm(d_out, n, k, theta, m, k, 0, 1, G);
      }
      orc_spmm_csr(n, colptr, crows, cvals, G, m, d_input);
    }
    free(G);
    free(P);
  }
  return 0;
}

/* ===================================================================== */
/* gat.hpp                                                                */
/* ===================================================================== */
/* gat.hpp:36-52 GatParams::init */
void orc_gat_params_init(int32_t m, int32_t h, int32_t k, uint64_t seed, double* theta,
                         double* a_src, double* a_dst, double* bias) {
  const double bound = 1.0 / sqrt((double)m);
  orc_random_uniform(m, (int64_t)h * k, seed, -bound, bound, theta);
  const double ab = 1.0 / sqrt((double)k);
  orc_random_uniform(h, k, seed + 1, -ab, ab, a_src);
  orc_random_uniform(h, k, seed + 2, -ab, ab, a_dst);
  orc_rng r = rng_make(seed + 3);
  for (int64_t j = 0; j < (int64_t)h * k; ++j) bias[j] = rng_double_range(&r, -bound, bound);
}

/* kernels.hpp:385-423 node_scores */
static void node_scores(const double* M, int32_t n, int32_t h, int32_t k, const double* a_src,
                        const double* a_dst, double* s, double* d) {
  for (int32_t i = 0; i < n; ++i)
    for (int32_t t = 0; t < h; ++t) {
      const double* mrow = M + ((size_t)i * h + t) * k;
      const double* as = a_src + (size_t)t * k;
      const double* ad = a_dst + (size_t)t * k;
      double sv = 0.0, dv = 0.0;
      for (int32_t c = 0; c < k; ++c) {
        sv += as[c] * mrow[c];
        dv += ad[c] * mrow[c];
      }
      s[(size_t)i * h + t] = sv;
      d[(size_t)i * h + t] = dv;
    }
}

/* kernels.hpp:427-478 edge_scores + leaky_relu_edges, then edge_softmax */
static int attention(int32_t n, const int32_t* rowptr, const int32_t* cols, int32_t h,
                     const double* s, const double* d, double beta, double* alpha,
                     uint8_t* mask) {
  const int64_t q = rowptr[n];
  double* w = (double*)malloc(sizeof(double) * (size_t)q * h + 8);
  for (int32_t t = 0; t < h; ++t)
    for (int32_t i = 0; i < n; ++i) {
      const double si = s[(size_t)i * h + t];
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
        const double y = si + d[(size_t)cols[e] * h + t];
        const int pos = y > 0.0;
        mask[(size_t)t * q + e] = (uint8_t)pos;
        w[(size_t)t * q + e] = pos ? y : beta * y;
      }
    }
  const int rc = orc_edge_softmax(n, rowptr, q, h, w, alpha);
  free(w);
  return rc;
}

/* gat.hpp:89-139 gat_forward */
int orc_gat_forward(int32_t n, const int32_t* rowptr, const int32_t* cols, const double* X,
                    int32_t m, const double* theta, const double* a_src, const double* a_dst,
                    const double* bias, int32_t h, int32_t k, double beta, double* out,
                    double* M_out, double* s_out, double* d_out_scores, double* alpha_out,
                    uint8_t* mask_out) {
  if (!(beta > 0)) return -1;
  for (int32_t i = 0; i < n; ++i) {
    int found = 0;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) if (cols[e] == i) { found = 1; break; }
    if (!found) return -1;
  }
  const int64_t q = rowptr[n];
  const int32_t hk = h * k;
  double* M = M_out ? M_out : (double*)malloc(sizeof(double) * (size_t)n * hk + 8);
  double* s = s_out ? s_out : (double*)malloc(sizeof(double) * (size_t)n * h + 8);
  double* d = d_out_scores ? d_out_scores : (double*)malloc(sizeof(double) * (size_t)n * h + 8);
  double* alpha = alpha_out ? alpha_out : (double*)malloc(sizeof(double) * (size_t)q * h + 8);
  uint8_t* mask = mask_out ? mask_out : (uint8_t*)malloc((size_t)q * h + 8);
  orc_gemm(X, n, m, theta, m, hk, 0, 0, M);
  node_scores(M, n, h, k, a_src, a_dst, s, d);
  attention(n, rowptr, cols, h, s, d, beta, alpha, mask);
  orc_spmm_semibatched(n, rowptr, cols, q, h, k, alpha, M, out);
  bias_add_rows(out, n, hk, bias);
  if (!M_out) free(M);
  if (!s_out) free(s);
  if (!d_out_scores) free(d);
  if (!alpha_out) free(alpha);
  if (!mask_out) free(mask);
  return 0;
}

/* gat.hpp:172-219 gat_backward (recompute of gat.hpp:150-170 with the
 * level-none path; every cache level is bit-identical by construction) */
int orc_gat_backward(int32_t n, const int32_t* rowptr, const int32_t* cols,
                     const int32_t* colptr, const int32_t* crows, const int32_t* perm,
                     const double* G, const double* X, int32_t m, const double* theta,
                     const double* a_src, const double* a_dst, int32_t h, int32_t k,
                     double beta, int fg, double* d_theta, double* d_a_src, double* d_a_dst,
                     double* d_bias, double* d_input) {
  const int64_t q = rowptr[n];
  const int32_t hk = h * k;
  orc_column_sums(G, n, hk, d_bias);
  double* M = (double*)malloc(sizeof(double) * (size_t)n * hk + 8);
  double* s = (double*)malloc(sizeof(double) * (size_t)n * h + 8);
  double* d = (double*)malloc(sizeof(double) * (size_t)n * h + 8);
  double* alpha = (double*)malloc(sizeof(double) * (size_t)q * h + 8);
  uint8_t* mask = (uint8_t*)malloc((size_t)q * h + 8);
  orc_gemm(X, n, m, theta, m, hk, 0, 0, M);
  node_scores(M, n, h, k, a_src, a_dst, s, d);
  attention(n, rowptr, cols, h, s, d, beta, alpha, mask);

  /* kernels.hpp:342-377 sddmm_semibatched: d_alpha[t,e] = <G[i,t,:], M[j,t,:]> */
  double* da = (double*)malloc(sizeof(double) * (size_t)q * h + 8);
  for (int32_t i = 0; i < n; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const int32_t j = cols[e];
      for (int32_t t = 0; t < h; ++t) {
        const double* ar = G + ((size_t)i * h + t) * k;
        const double* br = M + ((size_t)j * h + t) * k;
        double acc = 0.0;
        for (int32_t c = 0; c < k; ++c) acc += ar[c] * br[c];
        da[(size_t)t * q + e] = acc;
      }
    }
  /* kernels.hpp:537-567 edge_softmax_backward, then :481-495 leaky backward */
  double* dy = (double*)malloc(sizeof(double) * (size_t)q * h + 8);
  for (int32_t i = 0; i < n; ++i)
    for (int32_t t = 0; t < h; ++t) {
      const double* ah = alpha + (size_t)t * q;
      const double* gh = da + (size_t)t * q;
      double dot = 0.0;
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) dot += ah[e] * gh[e];
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
        dy[(size_t)t * q + e] = ah[e] * (gh[e] - dot);
    }
  for (int64_t x = 0; x < q * h; ++x) dy[x] = mask[x] ? dy[x] : beta * dy[x];
  /* kernels.hpp:570-588 edge_row_sums, :639-658 edge_col_sums */
  double* dS = (double*)malloc(sizeof(double) * (size_t)n * h + 8);
  double* dD = (double*)malloc(sizeof(double) * (size_t)n * h + 8);
  for (int32_t t = 0; t < h; ++t) {
    const double* hd = dy + (size_t)t * q;
    for (int32_t i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) acc += hd[e];
      dS[(size_t)i * h + t] = acc;
    }
    for (int32_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int32_t e = colptr[j]; e < colptr[j + 1]; ++e) acc += hd[perm[e]];
      dD[(size_t)j * h + t] = acc;
    }
  }
  /* dM = alpha^T G + dS (x) a_src + dD (x) a_dst (gat.hpp:201-204, kernels.hpp:614-636) */
  double* dM = (double*)malloc(sizeof(double) * (size_t)n * hk + 8);
  spmm_semibatched_transposed(n, colptr, crows, perm, q, h, k, alpha, G, dM);
  for (int pass = 0; pass < 2; ++pass) {
    const double* coeff = pass == 0 ? dS : dD;
    const double* vec = pass == 0 ? a_src : a_dst;
    for (int32_t i = 0; i < n; ++i)
      for (int32_t t = 0; t < h; ++t) {
        const double c = coeff[(size_t)i * h + t];
        double* orow = dM + ((size_t)i * h + t) * k;
        const double* vrow = vec + (size_t)t * k;
        for (int32_t cc = 0; cc < k; ++cc) orow[cc] += c * vrow[cc];
      }
  }
  /* kernels.hpp:592-611 attention_param_grad */
  for (int pass = 0; pass < 2; ++pass) {
    const double* coeff = pass == 0 ? dS : dD;
    double* o = pass == 0 ? d_a_src : d_a_dst;
    memset(o, 0, sizeof(double) * (size_t)hk);
    for (int32_t i = 0; i < n; ++i)
      for (int32_t t = 0; t < h; ++t) {
        const double c = coeff[(size_t)i * h + t];
        const double* mrow = M + ((size_t)i * h + t) * k;
        double* orow = o + (size_t)t * k;
        for (int32_t cc = 0; cc < k; ++cc) orow[cc] += c * mrow[cc];
      }
  }
  orc_gemm(X, n, m, dM, n, hk, 1, 0, d_theta);
  if (fg) orc_gemm(dM, n, hk, theta, m, hk, 0, 1, d_input);
  free(M); free(s); free(d); free(alpha); free(mask); free(da); free(dy);
  free(dS); free(dD); free(dM);
  return 0;
}
