/*
 * rdmm_oracle.c -- TEST INFRASTRUCTURE ONLY (see rdmm_oracle.h).
 *
 * CPU restatement of the reference algorithms, each function citing the
 * reference file:line it follows (paths relative to
 * /root/reference/proj/include/rdmm/).  Floating-point accumulation follows
 * the reference's order exactly and uses explicit fma(), which is what
 * `crow[j] += av * brow[j]` compiles to under g++ -O3 with FMA available
 * (-ffp-contract=fast is the GNU default), so real-valued results are
 * reproducible independently of this file's compile flags.
 */
#include "rdmm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- rng */

/* gen.hpp:20-25 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* gen.hpp:28-30 */
uint64_t orc_rng_at(uint64_t seed, uint64_t counter) {
  return orc_splitmix64(seed * 0x2545f4914f6cdd1dull + counter);
}

/* gen.hpp:32-34 */
double orc_rng_u01(uint64_t seed, uint64_t counter) {
  return (double)(orc_rng_at(seed, counter) >> 11) * 0x1.0p-53;
}

/* ---------------------------------------------------------------- utils */

static size_t wsize(int dtype) { return dtype == 8 ? 8 : 4; }

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 8);
  return p;
}

void orc_free(void* p) { free(p); }

void orc_csr_free(orc_csr* a) {
  if (!a) return;
  free(a->row_ptr);
  free(a->col_idx);
  free(a->values);
  a->row_ptr = NULL;
  a->col_idx = NULL;
  a->values = NULL;
}

static int csr_alloc(orc_csr* o, uint32_t rows, uint32_t cols, uint64_t nnz,
                     int dtype) {
  o->rows = rows;
  o->cols = cols;
  o->nnz = nnz;
  o->dtype = dtype;
  o->row_ptr = (uint32_t*)calloc((size_t)rows + 1, sizeof(uint32_t));
  o->col_idx = (uint32_t*)xmalloc(nnz * sizeof(uint32_t));
  o->values = xmalloc(nnz * wsize(dtype));
  if (!o->row_ptr || !o->col_idx || !o->values) {
    orc_csr_free(o);
    return -2;
  }
  return 0;
}

static void set_val(void* v, int dtype, uint64_t i, double x) {
  if (dtype == 8)
    ((double*)v)[i] = x;
  else
    ((float*)v)[i] = (float)x;
}

static double get_val(const void* v, int dtype, uint64_t i) {
  return dtype == 8 ? ((const double*)v)[i] : (double)((const float*)v)[i];
}

static int bits_for(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

/* Stable LSD radix sort of keys (with an optional uint64 payload) using
 * 11-bit digits over the low `kbits` bits. */
static int radix_sort_u64(uint64_t* keys, uint64_t* pay, uint64_t n,
                          int kbits) {
  if (n < 2 || kbits == 0) return 0;
  uint64_t* tk = (uint64_t*)xmalloc(n * sizeof(uint64_t));
  uint64_t* tp = pay ? (uint64_t*)xmalloc(n * sizeof(uint64_t)) : NULL;
  if (!tk || (pay && !tp)) {
    free(tk);
    free(tp);
    return -2;
  }
  const int D = 11;
  const uint64_t R = 1ull << D;
  uint64_t* cnt = (uint64_t*)xmalloc(R * sizeof(uint64_t));
  uint64_t *sk = keys, *sp = pay, *dk = tk, *dp = tp;
  for (int sh = 0; sh < kbits; sh += D) {
    memset(cnt, 0, R * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) cnt[(sk[i] >> sh) & (R - 1)]++;
    uint64_t s = 0;
    for (uint64_t d = 0; d < R; ++d) {
      uint64_t c = cnt[d];
      cnt[d] = s;
      s += c;
    }
    for (uint64_t i = 0; i < n; ++i) {
      uint64_t o = cnt[(sk[i] >> sh) & (R - 1)]++;
      dk[o] = sk[i];
      if (pay) dp[o] = sp[i];
    }
    uint64_t* t = sk;
    sk = dk;
    dk = t;
    t = sp;
    sp = dp;
    dp = t;
  }
  if (sk != keys) {
    memcpy(keys, sk, n * sizeof(uint64_t));
    if (pay) memcpy(pay, sp, n * sizeof(uint64_t));
  }
  free(tk);
  free(tp);
  free(cnt);
  return 0;
}

/* tile.hpp:70-95.  Keys are r*cols + c so lexicographic (r,c) order. */
static int csr_from_sorted_keys(uint32_t rows, uint32_t cols,
                                const uint64_t* keys, const uint64_t* order,
                                uint64_t n, const void* v, int dtype,
                                int ones, orc_csr* out) {
  uint64_t uniq = 0;
  for (uint64_t s = 0; s < n; ++s)
    if (s == 0 || keys[s] != keys[s - 1]) ++uniq;
  int rc = csr_alloc(out, rows, cols, uniq, dtype);
  if (rc) return rc;
  uint64_t o = 0;
  for (uint64_t s = 0; s < n;) {
    uint64_t key = keys[s];
    uint32_t r = (uint32_t)(key / cols), c = (uint32_t)(key % cols);
    uint64_t e = s;
    if (dtype == 8) {
      double sum = ones ? 0.0 : 0.0;
      int first = 1;
      while (e < n && keys[e] == key) {
        double x = ones ? 1.0 : ((const double*)v)[order[e]];
        sum = first ? x : sum + x;
        first = 0;
        ++e;
      }
      ((double*)out->values)[o] = sum;
    } else {
      float sum = 0.0f;
      int first = 1;
      while (e < n && keys[e] == key) {
        float x = ones ? 1.0f : ((const float*)v)[order[e]];
        sum = first ? x : sum + x;
        first = 0;
        ++e;
      }
      ((float*)out->values)[o] = sum;
    }
    out->col_idx[o] = c;
    out->row_ptr[r + 1]++;
    ++o;
    s = e;
  }
  for (uint32_t r = 0; r < rows; ++r) out->row_ptr[r + 1] += out->row_ptr[r];
  return 0;
}

int orc_from_coo(uint32_t rows, uint32_t cols, uint64_t n, const uint32_t* r,
                 const uint32_t* c, const void* v, int dtype, orc_csr* out) {
  memset(out, 0, sizeof(*out));
  uint64_t* keys = (uint64_t*)xmalloc(n * sizeof(uint64_t));
  uint64_t* ord = (uint64_t*)xmalloc(n * sizeof(uint64_t));
  if (!keys || !ord) {
    free(keys);
    free(ord);
    return -2;
  }
  for (uint64_t i = 0; i < n; ++i) {
    if (r[i] >= rows || c[i] >= cols) {
      free(keys);
      free(ord);
      return -1;
    }
    keys[i] = (uint64_t)r[i] * cols + c[i];
    ord[i] = i;
  }
  int rc = radix_sort_u64(keys, ord, n, bits_for((uint64_t)rows * cols));
  if (!rc)
    rc = csr_from_sorted_keys(rows, cols, keys, ord, n, v, dtype, 0, out);
  free(keys);
  free(ord);
  return rc;
}

/* ---------------------------------------------------------------- generators */

/* gen.hpp:58-92.  Edge e consumes counters [e*scale, (e+1)*scale). */
int orc_rmat(double a, double b, double c, double d, uint32_t scale,
             uint32_t edgefactor, uint64_t seed, int multiplicity, int dtype,
             orc_csr* out) {
  memset(out, 0, sizeof(*out));
  if (a < 0 || b < 0 || c < 0 || d < 0) return -1;       /* gen.hpp:45-46 */
  if (fabs(a + b + c + d - 1.0) > 1e-9) return -1;       /* gen.hpp:47-48 */
  if (scale > 26) return -1;                             /* gen.hpp:49-50 */
  const uint64_t rows = 1ull << scale;
  const uint64_t edges = (uint64_t)edgefactor << scale;
  uint64_t* keys = (uint64_t*)xmalloc(edges * sizeof(uint64_t));
  if (!keys) return -2;
  const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < (int64_t)edges; ++e) {
    uint64_t r = 0, col = 0, ctr = (uint64_t)e * scale;
    for (uint32_t level = 0; level < scale; ++level) {
      double u = orc_rng_u01(seed, ctr++);
      r <<= 1;
      col <<= 1;
      if (u < a) {
      } else if (u < ab) {
        col |= 1;
      } else if (u < abc) {
        r |= 1;
      } else {
        r |= 1;
        col |= 1;
      }
    }
    keys[e] = r * rows + col;
  }
  int rc = radix_sort_u64(keys, NULL, edges, bits_for(rows * rows - 1));
  if (!rc)
    rc = csr_from_sorted_keys((uint32_t)rows, (uint32_t)rows, keys, NULL,
                              edges, NULL, dtype, 1, out);
  free(keys);
  if (!rc && !multiplicity) /* gen.hpp:89-90 */
    for (uint64_t s = 0; s < out->nnz; ++s) set_val(out->values, dtype, s, 1.0);
  return rc;
}

/* Open-addressing set of uint64 (keys < 2^63; empty = ~0). */
typedef struct {
  uint64_t* slots;
  uint64_t mask;
  uint64_t size;
} u64set;

static uint64_t mix(uint64_t x) { return orc_splitmix64(x); }

static int set_insert(u64set* s, uint64_t k) {
  uint64_t h = mix(k) & s->mask;
  for (;;) {
    if (s->slots[h] == ~0ull) {
      s->slots[h] = k;
      s->size++;
      return 1;
    }
    if (s->slots[h] == k) return 0;
    h = (h + 1) & s->mask;
  }
}

/* gen.hpp:97-133.  The resulting cell set does not depend on the set's
 * iteration order because from_coo sorts. */
int orc_uniform_tiles(uint64_t m, uint64_t k, uint32_t p, double d,
                      uint64_t seed, int dtype, orc_csr* out) {
  memset(out, 0, sizeof(*out));
  uint32_t s = (uint32_t)lround(sqrt((double)p));
  if ((uint64_t)s * s != p) return -1;
  if (m % s != 0 || k % s != 0) return -1;
  uint64_t tm = m / s, tk = k / s;
  double per_tile_f = d * (double)tm * (double)tk;
  uint64_t per_tile = (uint64_t)llround(per_tile_f);
  if (fabs(per_tile_f - (double)per_tile) > 1e-9) return -1;
  if (per_tile > tm * tk) return -1;
  uint64_t total = per_tile * p;
  uint64_t* keys = (uint64_t*)xmalloc(total * sizeof(uint64_t));
  uint64_t cap = 16;
  while (cap < 2 * per_tile + 2) cap <<= 1;
  u64set set = {(uint64_t*)xmalloc(cap * sizeof(uint64_t)), cap - 1, 0};
  if (!keys || !set.slots) {
    free(keys);
    free(set.slots);
    return -2;
  }
  uint64_t ctr = 0, o = 0;
  for (uint32_t ti = 0; ti < s; ++ti)
    for (uint32_t tj = 0; tj < s; ++tj) {
      memset(set.slots, 0xff, cap * sizeof(uint64_t));
      set.size = 0;
      while (set.size < per_tile) {
        uint64_t cell = orc_rng_at(seed, ctr++) % (tm * tk);
        if (set_insert(&set, cell)) {
          uint64_t r = ti * tm + cell / tk, c = tj * tk + cell % tk;
          keys[o++] = r * k + c;
        }
      }
    }
  free(set.slots);
  int rc = radix_sort_u64(keys, NULL, total, bits_for(m * k - 1));
  if (!rc)
    rc = csr_from_sorted_keys((uint32_t)m, (uint32_t)k, keys, NULL, total, NULL,
                              dtype, 1, out);
  free(keys);
  return rc;
}

/* gen.hpp:138-155: Fisher-Yates with rng::at(seed, i), then relabel. */
int orc_permute_symmetric(const orc_csr* m, uint64_t seed, orc_csr* out) {
  memset(out, 0, sizeof(*out));
  if (m->rows != m->cols) return -1;
  uint32_t* perm = (uint32_t*)xmalloc((size_t)m->rows * sizeof(uint32_t));
  for (uint32_t i = 0; i < m->rows; ++i) perm[i] = i;
  for (uint32_t i = m->rows; i > 1; --i) {
    uint32_t j = (uint32_t)(orc_rng_at(seed, i) % i);
    uint32_t t = perm[i - 1];
    perm[i - 1] = perm[j];
    perm[j] = t;
  }
  uint32_t* rr = (uint32_t*)xmalloc(m->nnz * sizeof(uint32_t));
  uint32_t* cc = (uint32_t*)xmalloc(m->nnz * sizeof(uint32_t));
  for (uint32_t r = 0; r < m->rows; ++r)
    for (uint32_t s = m->row_ptr[r]; s < m->row_ptr[r + 1]; ++s) {
      rr[s] = perm[r];
      cc[s] = perm[m->col_idx[s]];
    }
  int rc = orc_from_coo(m->rows, m->cols, m->nnz, rr, cc, m->values, m->dtype,
                        out);
  free(perm);
  free(rr);
  free(cc);
  return rc;
}

/* gen.hpp:158-172: counter advances twice per cell; value drawn at the
 * (already incremented) counter. */
int orc_random_csr(uint32_t rows, uint32_t cols, double density, uint64_t seed,
                   int max_value, int dtype, orc_csr* out) {
  memset(out, 0, sizeof(*out));
  uint64_t ctr = 0, n = 0;
  /* first pass: count */
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t c = 0; c < cols; ++c) {
      if (orc_rng_u01(seed, ctr++) < density) ++n;
      ++ctr;
    }
  int rc = csr_alloc(out, rows, cols, n, dtype);
  if (rc) return rc;
  ctr = 0;
  uint64_t o = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    for (uint32_t c = 0; c < cols; ++c) {
      if (orc_rng_u01(seed, ctr++) < density) {
        int v = 1 + (int)(orc_rng_at(seed, ctr) % (uint64_t)max_value);
        out->col_idx[o] = c;
        set_val(out->values, dtype, o, (double)v);
        ++o;
      }
      ++ctr;
    }
    out->row_ptr[r + 1] = (uint32_t)o;
  }
  return 0;
}

/* gen.hpp:174-181 */
void orc_random_dense(uint32_t rows, uint32_t cols, uint64_t seed,
                      int max_value, int dtype, void* out) {
  uint64_t n = (uint64_t)rows * cols;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; ++i)
    set_val(out, dtype, (uint64_t)i,
            (double)(int)(orc_rng_at(seed, (uint64_t)i) %
                          (uint64_t)(max_value + 1)));
}

/* ---------------------------------------------------------------- kernels */

/* tile.hpp:170-188 restricted to rows [r0, r1). */
uint64_t orc_spmm_rows(const orc_csr* a, uint32_t r0, uint32_t r1, uint32_t n,
                       const void* b, uint64_t ldb, void* c, uint64_t ldc) {
  uint64_t nz = 0;
  if (a->dtype == 8) {
    const double* av = (const double*)a->values;
    const double* bb = (const double*)b;
    double* cc = (double*)c;
    for (uint32_t r = r0; r < r1; ++r) {
      double* crow = cc + (uint64_t)r * ldc;
      for (uint32_t s = a->row_ptr[r]; s < a->row_ptr[r + 1]; ++s) {
        const double* brow = bb + (uint64_t)a->col_idx[s] * ldb;
        double x = av[s];
        for (uint32_t j = 0; j < n; ++j) crow[j] = fma(x, brow[j], crow[j]);
      }
      nz += a->row_ptr[r + 1] - a->row_ptr[r];
    }
  } else {
    const float* av = (const float*)a->values;
    const float* bb = (const float*)b;
    float* cc = (float*)c;
    for (uint32_t r = r0; r < r1; ++r) {
      float* crow = cc + (uint64_t)r * ldc;
      for (uint32_t s = a->row_ptr[r]; s < a->row_ptr[r + 1]; ++s) {
        const float* brow = bb + (uint64_t)a->col_idx[s] * ldb;
        float x = av[s];
        for (uint32_t j = 0; j < n; ++j) crow[j] = fmaf(x, brow[j], crow[j]);
      }
      nz += a->row_ptr[r + 1] - a->row_ptr[r];
    }
  }
  return 2ull * nz * n;
}

/* tile.hpp:170-188 */
uint64_t orc_spmm_local(const orc_csr* a, uint32_t b_rows, uint32_t n,
                        const void* b, uint64_t ldb, void* c, uint64_t ldc,
                        int* err) {
  if (err) *err = 0;
  if (a->cols != b_rows) { /* tile.hpp:173-174 dimension_error */
    if (err) *err = -1;
    return 0;
  }
  return orc_spmm_rows(a, 0, a->rows, n, b, ldb, c, ldc);
}

/* tile.hpp:197-209 */
uint64_t orc_spgemm_flops(const orc_csr* a, const orc_csr* b) {
  uint64_t f = 0;
  for (uint64_t s = 0; s < a->nnz; ++s) {
    uint32_t k = a->col_idx[s];
    f += b->row_ptr[k + 1] - b->row_ptr[k];
  }
  return 2 * f;
}

static int cmp_u32(const void* x, const void* y) {
  uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
  return (a > b) - (a < b);
}

/* tile.hpp:211-249: Gustavson with a dense accumulator, `seen` flags, a
 * touched list sorted per row; cancelled zeros are kept. */
int orc_spgemm_local(const orc_csr* a, const orc_csr* b, uint32_t r0,
                     uint32_t r1, orc_csr* out, uint64_t* flops) {
  memset(out, 0, sizeof(*out));
  if (a->cols != b->rows) return -1; /* tile.hpp:216-217 */
  if (r1 > a->rows) r1 = a->rows;
  if (r0 > r1) r0 = r1;
  const int dt = a->dtype;
  const uint32_t nrows = r1 - r0;
  uint64_t cap = 1024, n = 0, f = 0;
  uint32_t* ci = (uint32_t*)xmalloc(cap * sizeof(uint32_t));
  void* vv = xmalloc(cap * wsize(dt));
  uint32_t* rp = (uint32_t*)calloc((size_t)nrows + 1, sizeof(uint32_t));
  char* seen = (char*)calloc(b->cols ? b->cols : 1, 1);
  uint32_t* touched = (uint32_t*)xmalloc(((size_t)b->cols + 1) * sizeof(uint32_t));
  double* accd = dt == 8 ? (double*)xmalloc(((size_t)b->cols + 1) * 8) : NULL;
  float* accf = dt == 4 ? (float*)xmalloc(((size_t)b->cols + 1) * 4) : NULL;
  for (uint32_t r = r0; r < r1; ++r) {
    uint32_t nt = 0;
    for (uint32_t s = a->row_ptr[r]; s < a->row_ptr[r + 1]; ++s) {
      uint32_t k = a->col_idx[s];
      for (uint32_t t = b->row_ptr[k]; t < b->row_ptr[k + 1]; ++t) {
        uint32_t j = b->col_idx[t];
        if (!seen[j]) {
          seen[j] = 1;
          if (dt == 8)
            accd[j] = 0.0;
          else
            accf[j] = 0.0f;
          touched[nt++] = j;
        }
        if (dt == 8)
          accd[j] = fma(((const double*)a->values)[s],
                        ((const double*)b->values)[t], accd[j]);
        else
          accf[j] = fmaf(((const float*)a->values)[s],
                         ((const float*)b->values)[t], accf[j]);
        f += 2;
      }
    }
    qsort(touched, nt, sizeof(uint32_t), cmp_u32);
    if (n + nt > cap) {
      while (n + nt > cap) cap *= 2;
      ci = (uint32_t*)realloc(ci, cap * sizeof(uint32_t));
      vv = realloc(vv, cap * wsize(dt));
    }
    for (uint32_t q = 0; q < nt; ++q) {
      uint32_t j = touched[q];
      ci[n] = j;
      if (dt == 8)
        ((double*)vv)[n] = accd[j];
      else
        ((float*)vv)[n] = accf[j];
      seen[j] = 0;
      ++n;
    }
    rp[r - r0 + 1] = (uint32_t)n;
  }
  free(seen);
  free(touched);
  free(accd);
  free(accf);
  out->rows = nrows;
  out->cols = b->cols;
  out->nnz = n;
  out->dtype = dt;
  out->row_ptr = rp;
  out->col_idx = ci;
  out->values = vv;
  if (flops) *flops = f;
  return 0;
}

/* tile.hpp:257-283 */
int orc_csr_add(const orc_csr* a, const orc_csr* b, orc_csr* out) {
  memset(out, 0, sizeof(*out));
  if (a->rows != b->rows || a->cols != b->cols) return -1;
  int rc = csr_alloc(out, a->rows, a->cols, a->nnz + b->nnz, a->dtype);
  if (rc) return rc;
  const int dt = a->dtype;
  uint64_t o = 0;
  for (uint32_t r = 0; r < a->rows; ++r) {
    uint32_t sa = a->row_ptr[r], ea = a->row_ptr[r + 1];
    uint32_t sb = b->row_ptr[r], eb = b->row_ptr[r + 1];
    while (sa < ea || sb < eb) {
      uint32_t ca = sa < ea ? a->col_idx[sa] : a->cols;
      uint32_t cb = sb < eb ? b->col_idx[sb] : b->cols;
      if (ca < cb) {
        out->col_idx[o] = ca;
        set_val(out->values, dt, o, get_val(a->values, dt, sa++));
      } else if (cb < ca) {
        out->col_idx[o] = cb;
        set_val(out->values, dt, o, get_val(b->values, dt, sb++));
      } else {
        out->col_idx[o] = ca;
        if (dt == 8)
          ((double*)out->values)[o] =
              ((const double*)a->values)[sa] + ((const double*)b->values)[sb];
        else
          ((float*)out->values)[o] =
              ((const float*)a->values)[sa] + ((const float*)b->values)[sb];
        ++sa;
        ++sb;
      }
      ++o;
    }
    out->row_ptr[r + 1] = (uint32_t)o;
  }
  out->nnz = o;
  return 0;
}

/* tile.hpp:300-307 */
void orc_dense_add_into(uint64_t n, void* c, const void* contrib, int dtype) {
  if (dtype == 8)
    for (uint64_t i = 0; i < n; ++i)
      ((double*)c)[i] += ((const double*)contrib)[i];
  else
    for (uint64_t i = 0; i < n; ++i)
      ((float*)c)[i] += ((const float*)contrib)[i];
}

/* tile.hpp:105-117 */
int orc_csr_well_formed(const orc_csr* a) {
  if (a->row_ptr[0] != 0 || a->row_ptr[a->rows] != a->nnz) return 0;
  for (uint32_t r = 0; r < a->rows; ++r) {
    if (a->row_ptr[r] > a->row_ptr[r + 1]) return 0;
    for (uint32_t s = a->row_ptr[r]; s < a->row_ptr[r + 1]; ++s) {
      if (a->col_idx[s] >= a->cols) return 0;
      if (s > a->row_ptr[r] && a->col_idx[s] <= a->col_idx[s - 1]) return 0;
    }
  }
  return 1;
}

/* ---------------------------------------------------------------- checksums */

/* algos.hpp:647: (i * 1000003u + j) % 8191 + 1 in uint32 arithmetic. */
static double tile_hash(uint32_t i, uint32_t j) {
  return (double)((i * 1000003u + j) % 8191u + 1u);
}

/* algos.hpp:634-650 */
double orc_checksum_dense(uint64_t m, uint64_t n, uint32_t tm, uint32_t tn,
                          const void* g, int dtype) {
  uint32_t M = (uint32_t)((m + tm - 1) / tm), N = (uint32_t)((n + tn - 1) / tn);
  double s = 0;
  for (uint32_t i = 0; i < M; ++i)
    for (uint32_t j = 0; j < N; ++j) {
      uint64_t rows = m - (uint64_t)i * tm < tm ? m - (uint64_t)i * tm : tm;
      uint64_t cols = n - (uint64_t)j * tn < tn ? n - (uint64_t)j * tn : tn;
      double ts = 0;
      for (uint64_t r = 0; r < rows; ++r)
        for (uint64_t c = 0; c < cols; ++c)
          ts += get_val(g, dtype,
                        ((uint64_t)i * tm + r) * n + (uint64_t)j * tn + c);
      s += tile_hash(i, j) * ts;
    }
  return s;
}

/* algos.hpp:652-669 */
double orc_checksum_sparse(const orc_csr* g, uint32_t tm, uint32_t tn) {
  uint32_t M = (uint32_t)(((uint64_t)g->rows + tm - 1) / tm);
  uint32_t N = (uint32_t)(((uint64_t)g->cols + tn - 1) / tn);
  double* ts = (double*)calloc((size_t)M * N, sizeof(double));
  for (uint32_t r = 0; r < g->rows; ++r)
    for (uint32_t s = g->row_ptr[r]; s < g->row_ptr[r + 1]; ++s) {
      uint32_t i = r / tm, j = g->col_idx[s] / tn;
      ts[(size_t)i * N + j] += get_val(g->values, g->dtype, s);
    }
  double sum = 0;
  for (uint32_t i = 0; i < M; ++i)
    for (uint32_t j = 0; j < N; ++j)
      sum += tile_hash(i, j) * ts[(size_t)i * N + j];
  free(ts);
  return sum;
}
