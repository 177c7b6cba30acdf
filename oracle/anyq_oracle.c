/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (C restatement) of the any4 hot path.
 *
 * Restates, in plain C, the reference algorithms of /root/reference/proj:
 *   RNG                core.hpp:154-200
 *   scales             scaling.cpp:8-96, scaling.hpp:36-45
 *   codebooks / RTN    codebooks.cpp:8-121, quantize.cpp:5-23
 *   learner            learner.cpp:10-448
 *   packing / layout   pack.cpp:15-238, pack.hpp:45,79-84
 *   GEMM               qgemm.cpp:22-128
 *   test generators    tests/helpers.hpp:14-71
 * Compiled with -ffp-contract=off like the reference (CMakeLists.txt:13-14),
 * it is bit-identical to the reference build; tests/test_oracle.py pins that
 * against oracle/_ref (when present) and against tests/golden/.
 *
 * Only the tests, __graft_entry__.smoke() and bench.py's CPU baseline load
 * this file's library. The product never links it.
 */
#define _POSIX_C_SOURCE 200809L
#include "anyq_oracle.h"

#include <float.h>
#include <math.h>
#include <setjmp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------
 * error handling: every API entry sets a jmp_buf; failures longjmp back with
 * the status of the reference exception class. Allocations go to an arena
 * freed on exit from the API call.
 * ---------------------------------------------------------------------- */
static _Thread_local char g_err[512];
static _Thread_local jmp_buf* g_env;
static _Thread_local void** g_arena;
static _Thread_local size_t g_arena_n, g_arena_cap;

static void fail(int status, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  longjmp(*g_env, status);
}

static void* oalloc(size_t n) {
  void* p = calloc(n ? n : 1, 1);
  if (!p) fail(ANYQ_ERR_INTERNAL, "oracle: out of memory");
  if (g_arena_n == g_arena_cap) {
    g_arena_cap = g_arena_cap ? 2 * g_arena_cap : 64;
    g_arena = (void**)realloc(g_arena, g_arena_cap * sizeof(void*));
  }
  g_arena[g_arena_n++] = p;
  return p;
}

static void arena_free(void) {
  for (size_t i = 0; i < g_arena_n; ++i) free(g_arena[i]);
  g_arena_n = 0;
}

#define API_BEGIN                \
  jmp_buf env__;                 \
  jmp_buf* prev__ = g_env;       \
  g_env = &env__;                \
  int st__ = setjmp(env__);      \
  if (st__ != 0) {               \
    arena_free();                \
    g_env = prev__;              \
    return st__;                 \
  }
#define API_END      \
  arena_free();      \
  g_env = prev__;    \
  g_err[0] = 0;      \
  return ANYQ_OK;

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------
 * RNG — core.hpp:154-200
 * ---------------------------------------------------------------------- */
static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

typedef struct {
  uint64_t key, counter;
} rng_t;

static rng_t rng_for_row(uint64_t seed, int64_t row) {
  rng_t r;
  r.key = splitmix64(seed) ^ splitmix64(0x9E3779B97F4A7C15ull * ((uint64_t)row + 1));
  r.counter = 0;
  return r;
}
static uint64_t next_u64(rng_t* r) { return splitmix64(r->key + 0xD1B54A32D192ED03ull * ++r->counter); }
static double next_double(rng_t* r) { return (double)(next_u64(r) >> 11) * 0x1.0p-53; }
static int64_t next_index(rng_t* r, int64_t bound) {
  double u = next_double(r);
  int64_t i = (int64_t)(u * (double)bound);
  return i >= bound ? bound - 1 : i;
}
static double next_gaussian(rng_t* r) {
  double u1 = (double)((next_u64(r) >> 11) + 1) * 0x1.0p-53;
  double u2 = next_double(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

void orc_rng_u64(uint64_t seed, int64_t row, int64_t n, uint64_t* out) {
  rng_t r = rng_for_row(seed, row);
  for (int64_t i = 0; i < n; ++i) out[i] = next_u64(&r);
}
void orc_rng_double(uint64_t seed, int64_t row, int64_t n, double* out) {
  rng_t r = rng_for_row(seed, row);
  for (int64_t i = 0; i < n; ++i) out[i] = next_double(&r);
}

/* test generators — tests/helpers.hpp:14-71 */
void orc_gaussian(int64_t rows, int64_t cols, uint64_t seed, float scale, float* out) {
  for (int64_t i = 0; i < rows; ++i) {
    rng_t r = rng_for_row(seed, i);
    for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = scale * (float)next_gaussian(&r);
  }
}
void orc_uniform(int64_t rows, int64_t cols, uint64_t seed, float lo, float hi, float* out) {
  for (int64_t i = 0; i < rows; ++i) {
    rng_t r = rng_for_row(seed, i);
    for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = lo + (hi - lo) * (float)next_double(&r);
  }
}
void orc_dyadic(int64_t rows, int64_t cols, uint64_t seed, int span, float step, float* out) {
  for (int64_t i = 0; i < rows; ++i) {
    rng_t r = rng_for_row(seed, i);
    for (int64_t j = 0; j < cols; ++j) {
      long t = (long)next_index(&r, 2 * (int64_t)span + 1) - span;
      out[i * cols + j] = step * (float)t;
    }
  }
}
void orc_heavy_tailed(int64_t rows, int64_t cols, uint64_t seed, float rate, float gain,
                      float* out) {
  for (int64_t i = 0; i < rows; ++i) {
    rng_t r = rng_for_row(seed, i);
    for (int64_t j = 0; j < cols; ++j) {
      float v = (float)next_gaussian(&r);
      if (next_double(&r) < rate) v *= gain;
      out[i * cols + j] = v;
    }
  }
}
void orc_synthetic_stats(int64_t cols, uint64_t seed, float* out) {
  rng_t r = rng_for_row(seed, 0);
  for (int64_t j = 0; j < cols; ++j) out[j] = (float)exp(1.2 * next_gaussian(&r));
}

/* ------------------------------------------------------------------------
 * config validation — core.hpp:124-147
 * ---------------------------------------------------------------------- */
static void validate_cfg(const anyq_config* c, int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) fail(ANYQ_ERR_SHAPE, "tensor must be at least 1x1");
  if (c->bits != 2 && c->bits != 3 && c->bits != 4 && c->bits != 8)
    fail(ANYQ_ERR_CONFIG, "bits must be one of {2,3,4,8}");
  if ((c->codebook == ANYQ_CB_FP4 || c->codebook == ANYQ_CB_NF4) && c->bits != 4)
    fail(ANYQ_ERR_CONFIG, "fp4/nf4 require bits == 4");
  if (c->granularity == ANYQ_G_GROUP && c->group_size < 2)
    fail(ANYQ_ERR_CONFIG, "group_size must be >= 2");
  if (c->granularity == ANYQ_G_BLOCK && c->block_size < 1)
    fail(ANYQ_ERR_CONFIG, "block_size must be >= 1");
  if (c->max_iters < 1) fail(ANYQ_ERR_CONFIG, "learner.max_iters must be >= 1");
  if (!(c->rel_tol >= 0)) fail(ANYQ_ERR_CONFIG, "learner.rel_tol must be >= 0");
  if (c->restarts < 1) fail(ANYQ_ERR_CONFIG, "learner.restarts must be >= 1");
  if (c->codebook == ANYQ_CB_ANY && c->granularity != ANYQ_G_ROW && c->granularity != ANYQ_G_GROUP)
    fail(ANYQ_ERR_CONFIG, "learned lookup tables are per-row");
  if (c->init == ANYQ_INIT_NF4 && c->bits != 4) fail(ANYQ_ERR_CONFIG, "nf4 seeding needs bits == 4");
}

static void require_finite(const float* m, int64_t n, const char* what) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(m[i])) {
      char b[128];
      snprintf(b, sizeof b, "%s: non-finite value", what);
      fail(ANYQ_ERR_NONFINITE, b);
    }
}

/* ------------------------------------------------------------------------
 * codebooks — codebooks.cpp:8-121
 * ---------------------------------------------------------------------- */
typedef struct {
  int n;
  float v[256];
} table_t;

static table_t int_grid(int bits, int shifted) {
  if (bits != 2 && bits != 3 && bits != 4 && bits != 8) fail(ANYQ_ERR_CONFIG, "int_grid: bits");
  table_t t;
  int lo = -(1 << (bits - 1)) + (shifted ? 1 : 0);
  t.n = 1 << bits;
  for (int q = 0; q < t.n; ++q) t.v[q] = (float)(lo + q);
  return t;
}

static const float kFp4[15] = {-6.0f, -4.0f, -3.0f, -2.0f, -1.5f, -1.0f, -0.5f, 0.0f,
                               0.5f,  1.0f,  1.5f,  2.0f,  3.0f,  4.0f,  6.0f};
static const float kNf4[16] = {-1.0f,
                               -0.6961928009986877f,
                               -0.5250730514526367f,
                               -0.39491748809814453f,
                               -0.28444138169288635f,
                               -0.18477343022823334f,
                               -0.09105003625154495f,
                               0.0f,
                               0.07958029955625534f,
                               0.16093020141124725f,
                               0.24611230194568634f,
                               0.33791524171829224f,
                               0.44070982933044434f,
                               0.5626170039176941f,
                               0.7229568362236023f,
                               1.0f};

static table_t fixed_codebook(const anyq_config* c) {
  table_t t;
  switch (c->codebook) {
    case ANYQ_CB_INT: return int_grid(c->bits, c->int_range_shifted);
    case ANYQ_CB_FP4:
      t.n = 15;
      memcpy(t.v, kFp4, sizeof kFp4);
      return t;
    case ANYQ_CB_NF4:
      t.n = 16;
      memcpy(t.v, kNf4, sizeof kNf4);
      return t;
    default: fail(ANYQ_ERR_CONFIG, "AnyN has no fixed codebook");
  }
  return t;
}

static table_t effective_codebook(table_t t, int symmetric) {
  if (symmetric) return t;
  float lo = t.v[0];
  for (int q = 0; q < t.n; ++q) t.v[q] -= lo;
  return t;
}

/* nearest table value, ties to the lower index — codebooks.cpp:75-97 */
static uint8_t round_one(float x, const table_t* t) {
  int lo = 0, hi = t->n; /* lower_bound: first v >= x */
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (t->v[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  if (lo == 0) return 0;
  if (lo == t->n) return (uint8_t)(t->n - 1);
  return (x - t->v[lo - 1] <= t->v[lo] - x) ? (uint8_t)(lo - 1) : (uint8_t)lo;
}

double orc_storage_bits_per_entry(const anyq_config* c, int64_t rows, int64_t cols) {
  double entries = (double)rows * (double)cols;
  double groups = 0;
  switch (c->granularity) {
    case ANYQ_G_TENSOR: groups = 1; break;
    case ANYQ_G_ROW: groups = (double)rows; break;
    case ANYQ_G_COLUMN: groups = (double)cols; break;
    case ANYQ_G_GROUP: groups = (double)rows * (double)((cols + c->group_size - 1) / c->group_size); break;
    case ANYQ_G_BLOCK:
      groups = (double)((rows + c->block_size - 1) / c->block_size) *
               (double)((cols + c->block_size - 1) / c->block_size);
      break;
  }
  double scale_bits = groups * 2.0 * 16.0;
  double lut_bits = 0;
  if (c->codebook == ANYQ_CB_ANY) lut_bits = (double)rows * (double)(1 << c->bits) * 16.0;
  return (double)c->bits + (scale_bits + lut_bits) / entries;
}

/* ------------------------------------------------------------------------
 * scales — scaling.cpp:8-96, scaling.hpp:36-45
 * ---------------------------------------------------------------------- */
typedef struct {
  int granularity, group_size, block_size, symmetric;
  int64_t rows, cols, ng;
  float* alphas;
  float* betas;
} scales_t;

static int64_t group_count(const anyq_config* c, int64_t rows, int64_t cols) {
  switch (c->granularity) {
    case ANYQ_G_TENSOR: return 1;
    case ANYQ_G_ROW: return rows;
    case ANYQ_G_COLUMN: return cols;
    case ANYQ_G_GROUP: return rows * ((cols + c->group_size - 1) / c->group_size);
    case ANYQ_G_BLOCK:
      return ((rows + c->block_size - 1) / c->block_size) *
             ((cols + c->block_size - 1) / c->block_size);
  }
  fail(ANYQ_ERR_CONFIG, "unknown granularity");
  return 0;
}

static int64_t group_of(const scales_t* s, int64_t i, int64_t j) {
  switch (s->granularity) {
    case ANYQ_G_TENSOR: return 0;
    case ANYQ_G_ROW: return i;
    case ANYQ_G_COLUMN: return j;
    case ANYQ_G_GROUP: return i * ((s->cols + s->group_size - 1) / s->group_size) + j / s->group_size;
    case ANYQ_G_BLOCK:
      return (i / s->block_size) * ((s->cols + s->block_size - 1) / s->block_size) + j / s->block_size;
  }
  fail(ANYQ_ERR_CONFIG, "unknown granularity");
  return 0;
}

static scales_t compute_scales(const float* w, int64_t rows, int64_t cols, const anyq_config* c,
                               float qmin, float qmax) {
  validate_cfg(c, rows, cols);
  require_finite(w, rows * cols, "compute_scales");
  if (!(qmax > qmin)) fail(ANYQ_ERR_CONFIG, "qmax must exceed qmin");
  if (c->symmetric && !(qmax > 0)) fail(ANYQ_ERR_CONFIG, "symmetric scaling needs qmax > 0");
  scales_t s;
  s.granularity = c->granularity;
  s.group_size = c->group_size;
  s.block_size = c->block_size;
  s.symmetric = c->symmetric;
  s.rows = rows;
  s.cols = cols;
  s.ng = group_count(c, rows, cols);
  float* mins = (float*)oalloc(sizeof(float) * s.ng);
  float* maxs = (float*)oalloc(sizeof(float) * s.ng);
  for (int64_t g = 0; g < s.ng; ++g) {
    mins[g] = FLT_MAX;
    maxs[g] = -FLT_MAX;
  }
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      int64_t g = group_of(&s, i, j);
      float v = w[i * cols + j];
      if (v < mins[g]) mins[g] = v;
      if (v > maxs[g]) maxs[g] = v;
    }
  s.alphas = (float*)oalloc(sizeof(float) * s.ng);
  s.betas = (float*)oalloc(sizeof(float) * s.ng);
  for (int64_t g = 0; g < s.ng; ++g) {
    if (c->symmetric) {
      float a = fabsf(mins[g]), b = fabsf(maxs[g]);
      float absmax = (a < b) ? b : a; /* std::max */
      s.alphas[g] = absmax > 0 ? absmax / qmax : 1.0f;
      s.betas[g] = 0;
    } else {
      float range = maxs[g] - mins[g];
      s.alphas[g] = range > 0 ? range / (qmax - qmin) : 1.0f;
      s.betas[g] = mins[g];
    }
  }
  return s;
}

static float* scale_weights(const float* w, const scales_t* s) {
  float* out = (float*)oalloc(sizeof(float) * s->rows * s->cols);
  for (int64_t i = 0; i < s->rows; ++i)
    for (int64_t j = 0; j < s->cols; ++j) {
      int64_t g = group_of(s, i, j);
      out[i * s->cols + j] = (w[i * s->cols + j] - s->betas[g]) / s->alphas[g];
    }
  return out;
}

/* ------------------------------------------------------------------------
 * learner — learner.cpp:10-448
 * ---------------------------------------------------------------------- */
typedef struct {
  const float* x;
  const float* w;
  int64_t n;
} prob_t;

static void prob_validate(const prob_t* p) { /* learner.cpp:10-23 */
  if (p->n == 0) fail(ANYQ_ERR_SHAPE, "KmProblem: empty problem");
  int any_pos = 0;
  for (int64_t i = 0; i < p->n; ++i) {
    float w = p->w[i];
    if (!(w >= 0) || !isfinite(w)) fail(ANYQ_ERR_STATS, "KmProblem: weights must be >= 0");
    any_pos |= w > 0;
  }
  if (!any_pos) fail(ANYQ_ERR_STATS, "KmProblem: all sample weights are zero");
  for (int64_t i = 0; i < p->n; ++i)
    if (!isfinite(p->x[i])) fail(ANYQ_ERR_NONFINITE, "KmProblem: non-finite sample");
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x < y) ? -1 : (y < x) ? 1 : 0;
}

/* learner.cpp:56-62: sorted unique sample values */
static double* distinct_values(const prob_t* p, int64_t* nd) {
  double* v = (double*)oalloc(sizeof(double) * p->n);
  for (int64_t i = 0; i < p->n; ++i) v[i] = p->x[i];
  qsort(v, (size_t)p->n, sizeof(double), cmp_double);
  int64_t m = 0;
  for (int64_t i = 0; i < p->n; ++i)
    if (m == 0 || !(v[m - 1] == v[i])) v[m++] = v[i];
  *nd = m;
  return v;
}

/* learner.cpp:64-75 */
static int64_t sample_index(const double* mass, int64_t n, double total, rng_t* rng) {
  double r = next_double(rng) * total;
  double acc = 0;
  int64_t last_positive = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (mass[i] <= 0) continue;
    acc += mass[i];
    last_positive = i;
    if (r < acc) return i;
  }
  return last_positive;
}

static void pad_with_distinct(double* c, int* nc, int k, const double* d, int64_t nd) {
  int64_t cursor = 0;
  while (*nc < k) c[(*nc)++] = d[cursor++ % nd];
}

static double pair_cost(double x, double c) {
  double d = x - c;
  return d * d;
}

/* learner.cpp:132-174 */
static void kmeans_pp(const prob_t* p, int k, rng_t* rng, double* cen) {
  prob_validate(p);
  if (k < 1) fail(ANYQ_ERR_CONFIG, "k must be >= 1");
  int64_t n = p->n;
  int nc = 0;
  double* mass = (double*)oalloc(sizeof(double) * n);
  double total = 0;
  for (int64_t i = 0; i < n; ++i) {
    mass[i] = p->w[i];
    total += mass[i];
  }
  cen[nc++] = p->x[sample_index(mass, n, total, rng)];
  double* d2 = (double*)oalloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) d2[i] = INFINITY;
  while (nc < k) {
    double c = cen[nc - 1];
    for (int64_t i = 0; i < n; ++i) {
      double pc = pair_cost(p->x[i], c);
      d2[i] = (pc < d2[i]) ? pc : d2[i]; /* std::min(d2, pc) */
    }
    total = 0;
    for (int64_t i = 0; i < n; ++i) {
      mass[i] = (double)p->w[i] * d2[i];
      total += mass[i];
    }
    if (total > 0) {
      cen[nc++] = p->x[sample_index(mass, n, total, rng)];
      continue;
    }
    total = 0;
    for (int64_t i = 0; i < n; ++i) {
      mass[i] = d2[i];
      total += mass[i];
    }
    if (total > 0) {
      cen[nc++] = p->x[sample_index(mass, n, total, rng)];
      continue;
    }
    int64_t nd;
    double* d = distinct_values(p, &nd);
    pad_with_distinct(cen, &nc, k, d, nd);
  }
}

/* learner.cpp:77-100 */
static void random_init(const prob_t* p, int k, rng_t* rng, double* cen) {
  int64_t n = p->n;
  int nc = 0;
  if ((int64_t)k >= n) {
    double* tmp = (double*)oalloc(sizeof(double) * (size_t)(n + k));
    for (int64_t i = 0; i < n; ++i) tmp[nc++] = p->x[i];
    qsort(tmp, (size_t)nc, sizeof(double), cmp_double);
    int64_t nd;
    double* d = distinct_values(p, &nd);
    pad_with_distinct(tmp, &nc, k, d, nd);
    memcpy(cen, tmp, sizeof(double) * (size_t)k);
    return;
  }
  int64_t* idx = (int64_t*)oalloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  for (int t = 0; t < k; ++t) {
    int64_t pick = t + next_index(rng, n - t);
    int64_t tmp = idx[t];
    idx[t] = idx[pick];
    idx[pick] = tmp;
    cen[nc++] = p->x[idx[t]];
  }
}

static uint8_t nearest(double x, const double* c, int k) { /* learner.cpp:185-196 */
  int best = 0;
  double bc = pair_cost(x, c[0]);
  for (int q = 1; q < k; ++q) {
    double cost = pair_cost(x, c[q]);
    if (cost < bc) {
      bc = cost;
      best = q;
    }
  }
  return (uint8_t)best;
}

static double total_cost(const prob_t* p, const double* c, const uint8_t* a) {
  double loss = 0;
  for (int64_t i = 0; i < p->n; ++i) loss += (double)p->w[i] * pair_cost(p->x[i], c[a[i]]);
  return loss;
}

/* learner.cpp:207-312 */
static double lloyd(const prob_t* p, double* cen, int k, const anyq_config* cfg, uint8_t* a,
                    int* iters_out) {
  int64_t n = p->n;
  memset(a, 0, (size_t)n);
  double* swx = (double*)oalloc(sizeof(double) * k);
  double* sw = (double*)oalloc(sizeof(double) * k);
  double* sx = (double*)oalloc(sizeof(double) * k);
  int64_t* cnt = (int64_t*)oalloc(sizeof(int64_t) * k);
  int* empties = (int*)oalloc(sizeof(int) * k);
  double prev = INFINITY;
  int iter = 0;
  for (; iter < cfg->max_iters; ++iter) {
    size_t changed = 0;
    for (int64_t i = 0; i < n; ++i) {
      uint8_t q = nearest(p->x[i], cen, k);
      changed += q != a[i];
      a[i] = q;
    }
    double loss_e = total_cost(p, cen, a);
    if (loss_e > prev) fail(ANYQ_ERR_INTERNAL, "internal: assignment step increased the weighted loss");
    if (cfg->check_invariants) {
      for (int64_t i = 0; i < n; ++i)
        for (int q = 0; q < k; ++q)
          if (pair_cost(p->x[i], cen[q]) < pair_cost(p->x[i], cen[a[i]]))
            fail(ANYQ_ERR_INTERNAL, "internal: stale assignment after E-step");
    }
    for (int q = 0; q < k; ++q) {
      swx[q] = sw[q] = sx[q] = 0;
      cnt[q] = 0;
    }
    for (int64_t i = 0; i < n; ++i) {
      uint8_t q = a[i];
      double w = p->w[i];
      double x = p->x[i];
      swx[q] += w * x;
      sw[q] += w;
      sx[q] += x;
      cnt[q] += 1;
    }
    int ne = 0;
    for (int q = 0; q < k; ++q) {
      if (cnt[q] == 0) empties[ne++] = q;
      else if (sw[q] > 0) cen[q] = swx[q] / sw[q];
      else cen[q] = sx[q] / (double)cnt[q];
    }
    if (cfg->check_invariants) {
      for (int q = 0; q < k; ++q) {
        if (cnt[q] == 0 || sw[q] <= 0) continue;
        double mean = swx[q] / sw[q];
        double am = fabs(mean);
        if (fabs(cen[q] - mean) > 1e-6 * (1.0 < am ? am : 1.0))
          fail(ANYQ_ERR_INTERNAL, "internal: centroid is not the weighted cluster mean");
      }
    }
    for (int e = 0; e < ne; ++e) {
      int q = empties[e];
      double worst = -1;
      int64_t wi = 0;
      for (int64_t i = 0; i < n; ++i) {
        double err = (double)p->w[i] * pair_cost(p->x[i], cen[a[i]]);
        if (err > worst) {
          worst = err;
          wi = i;
        }
      }
      cen[q] = p->x[wi];
      a[wi] = (uint8_t)q;
      changed += 1;
    }
    double loss_m = total_cost(p, cen, a);
    if (loss_m > loss_e * (1 + 1e-12) + 1e-300)
      fail(ANYQ_ERR_INTERNAL, "internal: update step increased the weighted loss");
    int stable = changed == 0 && iter > 0;
    int tol = isfinite(prev) && prev - loss_m <= (double)cfg->rel_tol * prev;
    prev = loss_m;
    if (stable || tol || loss_m == 0) {
      ++iter;
      break;
    }
  }
  for (int64_t i = 0; i < n; ++i) a[i] = nearest(p->x[i], cen, k);
  *iters_out = iter;
  return total_cost(p, cen, a);
}

/* learner.cpp:316-341 */
static double weighted_kmeans(const prob_t* p, int k, const anyq_config* cfg, rng_t* rng,
                              double* cen_out, uint8_t* a_out, int* iters_out) {
  prob_validate(p);
  if (k < 1) fail(ANYQ_ERR_CONFIG, "k must be >= 1");
  if (k > 256) fail(ANYQ_ERR_CONFIG, "k must fit an 8-bit code");
  double best = INFINITY;
  double* cen = (double*)oalloc(sizeof(double) * k);
  uint8_t* a = (uint8_t*)oalloc((size_t)p->n);
  int have = 0;
  for (int r = 0; r < cfg->restarts; ++r) {
    switch (cfg->init) {
      case ANYQ_INIT_KMPP: kmeans_pp(p, k, rng, cen); break;
      case ANYQ_INIT_RANDOM: random_init(p, k, rng, cen); break;
      case ANYQ_INIT_GRID:
        for (int q = 0; q < k; ++q) cen[q] = (double)(-(k / 2) + q);
        break;
      case ANYQ_INIT_NF4:
        if (k != 16) fail(ANYQ_ERR_CONFIG, "nf4 seeding needs exactly 16 centroids");
        for (int q = 0; q < 16; ++q) cen[q] = kNf4[q];
        break;
    }
    int iters;
    double loss = lloyd(p, cen, k, cfg, a, &iters);
    if (loss < best) {
      best = loss;
      memcpy(cen_out, cen, sizeof(double) * k);
      memcpy(a_out, a, (size_t)p->n);
      *iters_out = iters;
      have = 1;
    }
  }
  if (!have) { /* every restart produced a NaN loss: keep the default */
    memset(a_out, 0, (size_t)p->n);
  }
  return best;
}

/* learner.cpp:343-369 */
static double learn_row_lut(const prob_t* p, const anyq_config* cfg, int bits, rng_t* rng,
                            float* lut, uint8_t* codes) {
  int k = 1 << bits;
  double* cen = (double*)oalloc(sizeof(double) * k);
  uint8_t* a = (uint8_t*)oalloc((size_t)p->n);
  int iters = 0;
  double loss = weighted_kmeans(p, k, cfg, rng, cen, a, &iters);
  int order[256];
  for (int q = 0; q < k; ++q) order[q] = q;
  /* stable insertion sort by centroid value (std::stable_sort with <) */
  for (int i = 1; i < k; ++i) {
    int v = order[i];
    int j = i - 1;
    while (j >= 0 && cen[v] < cen[order[j]]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
  uint8_t rank[256];
  for (int pos = 0; pos < k; ++pos) rank[order[pos]] = (uint8_t)pos;
  for (int pos = 0; pos < k; ++pos) lut[pos] = (float)cen[order[pos]];
  for (int64_t i = 0; i < p->n; ++i) codes[i] = rank[a[i]];
  return loss;
}

/* learner.cpp:25-51 */
static void build_sample_weights(const scales_t* s, int64_t row, const float* stats, int mode,
                                 float* out) {
  int64_t cols = s->cols;
  if (stats)
    for (int64_t j = 0; j < cols; ++j)
      if (!(stats[j] >= 0) || !isfinite(stats[j]))
        fail(ANYQ_ERR_STATS, "sample weights: negative or non-finite stats entry");
  switch (mode) {
    case ANYQ_W_WEIGHTS:
      for (int64_t j = 0; j < cols; ++j) out[j] = 1.0f;
      return;
    case ANYQ_W_ACTS:
      for (int64_t j = 0; j < cols; ++j) out[j] = stats ? stats[j] : 1.0f;
      return;
    case ANYQ_W_FULL:
      for (int64_t j = 0; j < cols; ++j) {
        float e = stats ? stats[j] : 1.0f;
        out[j] = s->alphas[group_of(s, row, j)] * e;
      }
      return;
  }
  fail(ANYQ_ERR_CONFIG, "unknown weighting mode");
}

/* ------------------------------------------------------------------------
 * packing — pack.cpp:15-55
 * ---------------------------------------------------------------------- */
static int64_t bpr_of(int64_t cols, int bits) { return (cols * bits + 7) / 8; }

static void check_bits(int bits, const char* what) {
  if (bits != 2 && bits != 3 && bits != 4 && bits != 8) {
    char b[128];
    snprintf(b, sizeof b, "%s: bits must be one of {2,3,4,8}", what);
    fail(ANYQ_ERR_CONFIG, b);
  }
}

static void pack(const uint8_t* codes, int64_t rows, int64_t cols, int bits, uint8_t* out) {
  check_bits(bits, "pack_codes");
  int64_t bpr = bpr_of(cols, bits);
  uint32_t limit = 1u << bits;
  memset(out, 0, (size_t)(rows * bpr));
  for (int64_t i = 0; i < rows; ++i) {
    uint8_t* row = out + i * bpr;
    for (int64_t j = 0; j < cols; ++j) {
      uint32_t c = codes[i * cols + j];
      if (c >= limit) fail(ANYQ_ERR_CODE_RANGE, "code does not fit in bits");
      int64_t bit = j * bits;
      row[bit >> 3] |= (uint8_t)(c << (bit & 7));
      if ((bit & 7) + bits > 8) row[(bit >> 3) + 1] |= (uint8_t)(c >> (8 - (bit & 7)));
    }
  }
}

static void unpack(const uint8_t* packed, int64_t rows, int64_t cols, int bits, uint8_t* codes) {
  check_bits(bits, "unpack_codes");
  int64_t bpr = bpr_of(cols, bits);
  uint32_t mask = (1u << bits) - 1;
  for (int64_t i = 0; i < rows; ++i) {
    const uint8_t* row = packed + i * bpr;
    for (int64_t j = 0; j < cols; ++j) {
      int64_t bit = j * bits;
      uint32_t v = (uint32_t)row[bit >> 3] >> (bit & 7);
      if ((bit & 7) + bits > 8) v |= (uint32_t)row[(bit >> 3) + 1] << (8 - (bit & 7));
      codes[i * cols + j] = (uint8_t)(v & mask);
    }
  }
}

int orc_pack_codes(const uint8_t* codes, int64_t rows, int64_t cols, int bits, uint8_t* out) {
  API_BEGIN
  pack(codes, rows, cols, bits, out);
  API_END
}

int orc_unpack_codes(const uint8_t* packed, int64_t rows, int64_t cols, int bits, uint8_t* out) {
  API_BEGIN
  unpack(packed, rows, cols, bits, out);
  API_END
}

/* pack.hpp:79-84 */
static int64_t ktiled_pos(int64_t k, int64_t cols, int64_t tile_k) {
  int64_t num_full = cols / tile_k;
  int64_t full_end = num_full * tile_k;
  if (k >= full_end) return k;
  return (k % tile_k) * num_full + k / tile_k;
}

/* pack.cpp:175-199, on packed codes */
static void retile(const uint8_t* packed, int64_t rows, int64_t cols, int bits, int tile_k,
                   int inverse, uint8_t* out) {
  uint8_t* c = (uint8_t*)oalloc((size_t)(rows * cols));
  uint8_t* t = (uint8_t*)oalloc((size_t)(rows * cols));
  unpack(packed, rows, cols, bits, c);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      int64_t p = ktiled_pos(j, cols, tile_k);
      if (inverse) t[i * cols + j] = c[i * cols + p];
      else t[i * cols + p] = c[i * cols + j];
    }
  pack(t, rows, cols, bits, out);
}

int orc_to_ktiled(const anyq_qtensor* qt, int tile_k, uint8_t* codes_out) {
  API_BEGIN
  if (tile_k < 1) fail(ANYQ_ERR_CONFIG, "tile_k must be >= 1");
  int bits = qt->cfg.bits;
  const uint8_t* src = qt->codes;
  if (qt->layout == ANYQ_LAYOUT_KTILED) {
    uint8_t* rm = (uint8_t*)oalloc((size_t)(qt->rows * bpr_of(qt->cols, bits)));
    retile(qt->codes, qt->rows, qt->cols, bits, qt->tile_k, 1, rm);
    src = rm;
  }
  retile(src, qt->rows, qt->cols, bits, tile_k, 0, codes_out);
  API_END
}

int orc_from_ktiled(const anyq_qtensor* qt, uint8_t* codes_out) {
  API_BEGIN
  int64_t nb = qt->rows * bpr_of(qt->cols, qt->cfg.bits);
  if (qt->layout == ANYQ_LAYOUT_ROWMAJOR) memcpy(codes_out, qt->codes, (size_t)nb);
  else retile(qt->codes, qt->rows, qt->cols, qt->cfg.bits, qt->tile_k, 1, codes_out);
  API_END
}

/* ------------------------------------------------------------------------
 * 16-bit narrowing — pack.cpp:61-169
 * ---------------------------------------------------------------------- */
static uint32_t fbits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
static float bitsf(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static uint16_t f32_to_f16(float f) {
  uint32_t x = fbits(f);
  uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  uint32_t a = x & 0x7FFFFFFFu;
  if (a >= 0x7F800000u) fail(ANYQ_ERR_NONFINITE, "f32_to_f16: non-finite input");
  if (a >= 0x477FF000u) fail(ANYQ_ERR_IO, "f32_to_f16: value overflows to infinity");
  uint32_t out;
  if (a < 0x38800000u) {
    uint32_t e32 = a >> 23;
    uint32_t shift = 113u - e32;
    if (a == 0 || shift > 24u) {
      out = 0;
    } else {
      uint32_t mant = (a & 0x7FFFFFu) | 0x800000u;
      uint32_t q = mant >> (shift + 13u);
      uint32_t rem = mant & ((1u << (shift + 13u)) - 1u);
      uint32_t half = 1u << (shift + 12u);
      if (rem > half || (rem == half && (q & 1u))) ++q;
      out = q;
    }
  } else {
    uint32_t e = (a >> 23) - 112u;
    uint32_t mant = a & 0x7FFFFFu;
    uint32_t q = (e << 10) | (mant >> 13);
    uint32_t rem = mant & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) ++q;
    out = q;
  }
  return (uint16_t)(sign | out);
}

static float f16_to_f32(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1Fu;
  uint32_t mant = h & 0x3FFu;
  uint32_t out;
  if (e == 0) {
    if (mant == 0) {
      out = sign;
    } else {
      uint32_t shift = 0;
      while (!(mant & 0x400u)) {
        mant <<= 1;
        ++shift;
      }
      out = sign | ((113u - shift) << 23) | ((mant & 0x3FFu) << 13);
    }
  } else if (e == 0x1Fu) {
    out = sign | 0x7F800000u | (mant << 13);
  } else {
    out = sign | ((e + 112u) << 23) | (mant << 13);
  }
  return bitsf(out);
}

static uint16_t f32_to_bf16(float f) {
  uint32_t x = fbits(f);
  if ((x & 0x7F800000u) == 0x7F800000u) fail(ANYQ_ERR_NONFINITE, "f32_to_bf16: non-finite input");
  uint32_t lsb = (x >> 16) & 1u;
  uint32_t r = x + 0x7FFFu + lsb;
  if ((r & 0x7F800000u) == 0x7F800000u) fail(ANYQ_ERR_IO, "f32_to_bf16: overflow");
  return (uint16_t)(r >> 16);
}

static float bf16_to_f32(uint16_t h) { return bitsf((uint32_t)h << 16); }

int orc_f32_to_f16(float f, uint16_t* out) {
  API_BEGIN
  *out = f32_to_f16(f);
  API_END
}
float orc_f16_to_f32(uint16_t h) { return f16_to_f32(h); }
int orc_f32_to_bf16(float f, uint16_t* out) {
  API_BEGIN
  *out = f32_to_bf16(f);
  API_END
}
float orc_bf16_to_f32(uint16_t h) { return bf16_to_f32(h); }

static float narrow_widen(float v, int store) {
  switch (store) {
    case ANYQ_STORE_FP16: return f16_to_f32(f32_to_f16(v));
    case ANYQ_STORE_BF16: return bf16_to_f32(f32_to_bf16(v));
    case ANYQ_STORE_FP32: return v;
  }
  fail(ANYQ_ERR_CONFIG, "unknown storage precision");
  return v;
}

int orc_narrowed(anyq_qtensor* qt) { /* pack.cpp:159-169 */
  API_BEGIN
  if (qt->cfg.codebook == ANYQ_CB_ANY && qt->luts) {
    int64_t n = qt->rows * ((int64_t)1 << qt->cfg.bits);
    for (int64_t i = 0; i < n; ++i) qt->luts[i] = narrow_widen(qt->luts[i], qt->lut_store);
  }
  for (int64_t g = 0; g < qt->num_groups; ++g) {
    qt->alphas[g] = narrow_widen(qt->alphas[g], qt->scale_store);
    qt->betas[g] = narrow_widen(qt->betas[g], qt->scale_store);
    if (!(qt->alphas[g] > 0)) fail(ANYQ_ERR_INVARIANT, "scale underflows its 16-bit storage format");
  }
  API_END
}

/* ------------------------------------------------------------------------
 * quantization front doors — learner.cpp:373-448, quantize.cpp:5-23
 * ---------------------------------------------------------------------- */
static void export_scales(const scales_t* s, anyq_qtensor* out) {
  memcpy(out->alphas, s->alphas, sizeof(float) * s->ng);
  memcpy(out->betas, s->betas, sizeof(float) * s->ng);
  out->num_groups = s->ng;
}

static void quantize_any(const float* w, int64_t rows, int64_t cols, const anyq_config* cfg,
                         const float* exj, anyq_qtensor* out) {
  if (cfg->codebook != ANYQ_CB_ANY) fail(ANYQ_ERR_CONFIG, "quantize_any requires the learned codebook");
  validate_cfg(cfg, rows, cols);
  require_finite(w, rows * cols, "quantize_any");
  table_t grid = int_grid(cfg->bits, cfg->int_range_shifted);
  scales_t s = compute_scales(w, rows, cols, cfg, grid.v[0], grid.v[grid.n - 1]);
  float* ws = scale_weights(w, &s);
  int k = 1 << cfg->bits;
  uint8_t* codes = (uint8_t*)oalloc((size_t)(rows * cols));
  float* wts = (float*)oalloc(sizeof(float) * cols);
  for (int64_t i = 0; i < rows; ++i) {
    build_sample_weights(&s, i, exj, cfg->weighting, wts);
    int any = 0;
    for (int64_t j = 0; j < cols; ++j) any |= wts[j] > 0;
    if (!any)
      for (int64_t j = 0; j < cols; ++j) wts[j] = 1.0f;
    rng_t rng = rng_for_row(cfg->seed, i);
    prob_t p = {ws + i * cols, wts, cols};
    learn_row_lut(&p, cfg, cfg->bits, &rng, out->luts + i * k, codes + i * cols);
  }
  pack(codes, rows, cols, cfg->bits, out->codes);
  export_scales(&s, out);
}

static void quantize_fixed(const float* w, int64_t rows, int64_t cols, const anyq_config* cfg,
                           anyq_qtensor* out) {
  if (cfg->codebook == ANYQ_CB_ANY) fail(ANYQ_ERR_CONFIG, "quantize_fixed handles fixed codebooks only");
  validate_cfg(cfg, rows, cols);
  require_finite(w, rows * cols, "quantize_fixed");
  table_t cb = fixed_codebook(cfg);
  scales_t s = compute_scales(w, rows, cols, cfg, cb.v[0], cb.v[cb.n - 1]);
  float* ws = scale_weights(w, &s);
  table_t eff = effective_codebook(cb, cfg->symmetric);
  uint8_t* codes = (uint8_t*)oalloc((size_t)(rows * cols));
  for (int64_t i = 0; i < rows * cols; ++i) codes[i] = round_one(ws[i], &eff);
  pack(codes, rows, cols, cfg->bits, out->codes);
  export_scales(&s, out);
}

int orc_quantize(const float* w, int64_t rows, int64_t cols, const anyq_config* c,
                 const float* exj, int threads, anyq_qtensor* out) {
  (void)threads; /* rows are independent; the result is thread-count invariant */
  API_BEGIN
  out->rows = rows;
  out->cols = cols;
  out->layout = ANYQ_LAYOUT_ROWMAJOR;
  out->tile_k = 1;
  out->lut_store = ANYQ_STORE_FP16;
  out->scale_store = ANYQ_STORE_FP16;
  if (c->codebook == ANYQ_CB_ANY) quantize_any(w, rows, cols, c, exj, out);
  else quantize_fixed(w, rows, cols, c, out);
  API_END
}

int orc_time_quantize(const float* w, int64_t rows, int64_t cols, const anyq_config* c,
                      const float* exj, int threads, double* secs) {
  (void)threads;
  API_BEGIN
  anyq_qtensor q;
  memset(&q, 0, sizeof q);
  q.cfg = *c;
  int64_t ng = group_count(c, rows, cols);
  q.codes = (uint8_t*)oalloc((size_t)(rows * bpr_of(cols, c->bits)));
  q.luts = (float*)oalloc(sizeof(float) * rows * ((int64_t)1 << c->bits));
  q.alphas = (float*)oalloc(sizeof(float) * ng);
  q.betas = (float*)oalloc(sizeof(float) * ng);
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  quantize_any(w, rows, cols, c, exj, &q);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  *secs = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  API_END
}

/* ------------------------------------------------------------------------
 * dequantization — pack.cpp:205-238, scaling.cpp:85-96
 * ---------------------------------------------------------------------- */
static scales_t scales_of(const anyq_qtensor* qt) {
  scales_t s;
  s.granularity = qt->cfg.granularity;
  s.group_size = qt->cfg.group_size;
  s.block_size = qt->cfg.block_size;
  s.symmetric = qt->cfg.symmetric;
  s.rows = qt->rows;
  s.cols = qt->cols;
  s.ng = qt->num_groups;
  s.alphas = qt->alphas;
  s.betas = qt->betas;
  return s;
}

/* row-major logical codes of qt (undoing the k-tiling) */
static uint8_t* logical_codes(const anyq_qtensor* qt) {
  int bits = qt->cfg.bits;
  uint8_t* c = (uint8_t*)oalloc((size_t)(qt->rows * qt->cols));
  if (qt->layout == ANYQ_LAYOUT_KTILED) {
    uint8_t* rm = (uint8_t*)oalloc((size_t)(qt->rows * bpr_of(qt->cols, bits)));
    retile(qt->codes, qt->rows, qt->cols, bits, qt->tile_k, 1, rm);
    unpack(rm, qt->rows, qt->cols, bits, c);
  } else {
    unpack(qt->codes, qt->rows, qt->cols, bits, c);
  }
  return c;
}

static float* dequant(const anyq_qtensor* qt) {
  int64_t rows = qt->rows, cols = qt->cols;
  uint8_t* c = logical_codes(qt);
  float* v = (float*)oalloc(sizeof(float) * rows * cols);
  if (qt->cfg.codebook == ANYQ_CB_ANY) {
    int64_t k = (int64_t)1 << qt->cfg.bits;
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t j = 0; j < cols; ++j) {
        uint8_t q = c[i * cols + j];
        if (q >= k) fail(ANYQ_ERR_CODE_RANGE, "code exceeds LUT size");
        v[i * cols + j] = qt->luts[i * k + q];
      }
  } else {
    table_t cb = effective_codebook(fixed_codebook(&qt->cfg), qt->cfg.symmetric);
    for (int64_t i = 0; i < rows * cols; ++i) {
      if (c[i] >= cb.n) fail(ANYQ_ERR_CODE_RANGE, "code exceeds table size");
      v[i] = cb.v[c[i]];
    }
  }
  scales_t s = scales_of(qt);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      int64_t g = group_of(&s, i, j);
      v[i * cols + j] = s.alphas[g] * v[i * cols + j] + s.betas[g];
    }
  return v;
}

int orc_dequantize(const anyq_qtensor* qt, float* w) {
  API_BEGIN
  float* v = dequant(qt);
  memcpy(w, v, sizeof(float) * qt->rows * qt->cols);
  API_END
}

/* ------------------------------------------------------------------------
 * GEMM — qgemm.cpp:22-128
 * ---------------------------------------------------------------------- */
static void dense(const float* x, int64_t m, const float* w, int64_t n, int64_t k, float* y) {
  for (int64_t r = 0; r < m; ++r)
    for (int64_t i = 0; i < n; ++i) {
      float acc = 0;
      for (int64_t j = 0; j < k; ++j) acc += x[r * k + j] * w[i * k + j];
      y[r * n + i] = acc;
    }
}

int orc_gemm_dense(const float* x, int64_t m, const float* w, int64_t n, int64_t k, float* y) {
  API_BEGIN
  dense(x, m, w, n, k, y);
  API_END
}

/* weight_error, eval.cpp:11-29 (sequential double sums over i, j). */
int orc_weight_error(const float* w, const anyq_qtensor* qt, double* mse, double* rel) {
  API_BEGIN
  float* d = dequant(qt);
  double sq = 0, ref = 0;
  for (int64_t e = 0; e < qt->rows * qt->cols; ++e) {
    double x = (double)w[e] - (double)d[e];
    sq += x * x;
    ref += (double)w[e] * (double)w[e];
  }
  double count = (double)qt->rows * (double)qt->cols;
  *mse = sq / count;
  *rel = ref > 0 ? sqrt(sq) / sqrt(ref) : sqrt(sq);
  API_END
}

/* output_error, eval.cpp:31-46: gemm_dense(x, w) vs gemm_reference(x, qt). */
int orc_output_error(const float* w, const anyq_qtensor* qt, const float* x, int64_t m, double* mse) {
  API_BEGIN
  const int64_t n = qt->rows, k = qt->cols;
  float* y = (float*)oalloc(sizeof(float) * (size_t)(m * n + 1));
  float* yq = (float*)oalloc(sizeof(float) * (size_t)(m * n + 1));
  float* d = dequant(qt);
  dense(x, m, w, n, k, y);
  dense(x, m, d, n, k, yq);
  double sq = 0;
  for (int64_t e = 0; e < m * n; ++e) {
    double v = (double)yq[e] - (double)y[e];
    sq += v * v;
  }
  *mse = sq / ((double)m * (double)n);
  API_END
}

/* collect_stats, calibration.cpp:50-67: the per-layer statistic of the first
 * layer's inputs — E|x_j| = float(sum over samples in order of |double(x)| / M);
 * require_finite(inputs) (:52), at least one sample (:54). */
int orc_column_mean_abs(const float* x, int64_t m, int64_t k, float* out) {
  API_BEGIN
  require_finite(x, m * k, "collect_stats inputs");
  if (m < 1) fail(ANYQ_ERR_SHAPE, "need at least one input sample");
  for (int64_t j = 0; j < k; ++j) {
    double acc = 0;
    for (int64_t r = 0; r < m; ++r) acc += fabs((double)x[r * k + j]);
    out[j] = (float)(acc / (double)m);
  }
  API_END
}

int orc_gemm_reference(const float* x, int64_t m, const anyq_qtensor* qt, float* y) {
  API_BEGIN
  float* w = dequant(qt);
  dense(x, m, w, qt->rows, qt->cols, y);
  API_END
}

static void fused(const float* x, int64_t m, int64_t k, const anyq_qtensor* qt, int plan_layout,
                  int plan_tile_k, float* y) {
  if (k != qt->cols) fail(ANYQ_ERR_SHAPE, "gemm_fused: reduction dimensions differ");
  if (plan_layout != qt->layout || (qt->layout == ANYQ_LAYOUT_KTILED && plan_tile_k != qt->tile_k))
    fail(ANYQ_ERR_CONFIG, "gemm_fused: plan layout does not match tensor layout");
  int64_t n = qt->rows;
  int bits = qt->cfg.bits;
  int64_t bpr = bpr_of(k, bits);
  table_t fixed = {0, {0}};
  if (qt->cfg.codebook != ANYQ_CB_ANY) fixed = effective_codebook(fixed_codebook(&qt->cfg), qt->cfg.symmetric);
  scales_t s = scales_of(qt);
  for (int64_t i = 0; i < n; ++i) {
    const float* table = qt->cfg.codebook == ANYQ_CB_ANY ? qt->luts + i * ((int64_t)1 << bits) : fixed.v;
    int tsize = qt->cfg.codebook == ANYQ_CB_ANY ? (1 << bits) : fixed.n;
    const uint8_t* row = qt->codes + i * bpr;
    for (int64_t r = 0; r < m; ++r) {
      float acc = 0;
      for (int64_t j = 0; j < k; ++j) {
        int64_t pos = qt->layout == ANYQ_LAYOUT_KTILED ? ktiled_pos(j, k, qt->tile_k) : j;
        int64_t bit = pos * bits;
        uint32_t v = (uint32_t)row[bit >> 3] >> (bit & 7);
        if ((bit & 7) + bits > 8) v |= (uint32_t)row[(bit >> 3) + 1] << (8 - (bit & 7));
        uint32_t c = v & ((1u << bits) - 1);
        if ((int)c >= tsize) fail(ANYQ_ERR_CODE_RANGE, "gemm_fused: code exceeds table size");
        int64_t g = group_of(&s, i, j);
        float wv = s.alphas[g] * table[c] + s.betas[g];
        acc += x[r * k + j] * wv;
      }
      y[r * n + i] = acc;
    }
  }
}

int orc_gemm_fused(const float* x, int64_t m, int64_t k, const anyq_qtensor* qt, int plan_layout,
                   int plan_tile_k, float* y) {
  API_BEGIN
  fused(x, m, k, qt, plan_layout, plan_tile_k, y);
  API_END
}

int orc_time_gemm_fused(const float* x, int64_t m, const anyq_qtensor* qt, int repeats,
                        double* secs) {
  API_BEGIN
  float* y = (float*)oalloc(sizeof(float) * m * qt->rows);
  double* t = (double*)oalloc(sizeof(double) * repeats);
  for (int r = 0; r < repeats; ++r) {
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    fused(x, m, qt->cols, qt, qt->layout, qt->tile_k, y);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    t[r] = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
  }
  qsort(t, (size_t)repeats, sizeof(double), cmp_double);
  *secs = t[repeats / 2];
  API_END
}

/* ------------------------------------------------------------------------
 * learner entry points for tests
 * ---------------------------------------------------------------------- */
int orc_kmeans_pp_init(const float* x, const float* w, int64_t n, int k, uint64_t seed,
                       int64_t row, double* centroids) {
  API_BEGIN
  prob_t p = {x, w, n};
  rng_t r = rng_for_row(seed, row);
  kmeans_pp(&p, k, &r, centroids);
  API_END
}

int orc_weighted_kmeans(const float* x, const float* w, int64_t n, int k, const anyq_config* c,
                        uint64_t seed, int64_t row, double* centroids, uint8_t* assignments,
                        double* loss, int* iters) {
  API_BEGIN
  prob_t p = {x, w, n};
  rng_t r = rng_for_row(seed, row);
  *loss = weighted_kmeans(&p, k, c, &r, centroids, assignments, iters);
  API_END
}

int orc_learn_row_lut(const float* x, const float* w, int64_t n, int bits, const anyq_config* c,
                      uint64_t seed, int64_t row, float* lut, uint8_t* codes, double* loss) {
  API_BEGIN
  prob_t p = {x, w, n};
  rng_t r = rng_for_row(seed, row);
  *loss = learn_row_lut(&p, c, bits, &r, lut, codes);
  API_END
}
