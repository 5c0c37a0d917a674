/* qg_oracle.c — plain-C restatement of the reference qgemm algorithm
 * (/root/reference/proj/include/qgemm/*.hpp). TEST INFRASTRUCTURE ONLY:
 * see qg_oracle.h for who may call it. Compile with -ffp-contract=off so the
 * DoubleWord high part rounds exactly as the reference's (a*b)*inv_qd does.
 *
 * The reference is C++ exceptions + value types; here every routine returns a
 * status (QGO_*) in the order of errors.hpp:8-34 and writes caller-owned
 * row-major buffers with the exact layouts of CompressedMatrix::data
 * (matrix.hpp:44-63).
 */
#include "qg_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- field.hpp */

/* PrimeModulus::is_prime, field.hpp:42-48 (trial division). */
int qgo_is_prime(uint64_t n) {
  if (n < 2) return 0;
  if (n % 2 == 0) return n == 2;
  for (uint64_t f = 3; f * f <= n; f += 2)
    if (n % f == 0) return 0;
  return 1;
}

static uint64_t pm1sq(uint32_t p) { return (uint64_t)(p - 1) * (p - 1); } /* field.hpp:22 */

/* ----------------------------------------------------------------- plan.hpp */

/* detail::minimal_radix_exponent, plan.hpp:98-104: smallest t with 2^t > k(p-1)^2. */
static int minimal_radix_exponent(uint32_t p, uint64_t k) {
  const u128 bound = (u128)k * pm1sq(p);
  int t = 1;
  while (((u128)1 << t) <= bound) ++t;
  return t;
}

/* detail::word_capacity, plan.hpp:107-111: largest e with t*e < beta. */
static int word_capacity(int t, int beta) {
  int e = beta / t;
  if (e * t == beta) --e;
  return e;
}

/* detail::largest_common_dim, plan.hpp:113-115. */
static uint64_t largest_common_dim(uint32_t p, int t) {
  return ((UINT64_C(1) << t) - 1) / pm1sq(p);
}

/* plan_compression, plan.hpp:125-159 (PrimeModulus ctor checks, field.hpp:19-23). */
int qgo_plan_compression(uint32_t p, uint64_t k, int beta, int mode, qgo_plan* out) {
  if (p < 2 || !qgo_is_prime(p)) return QGO_INVALID_MODULUS;
  if (k < 1 || beta < 2) return QGO_INVALID_ARGUMENT;
  const int t = minimal_radix_exponent(p, k);
  if (t >= beta) return QGO_NO_COMPRESSION;
  const int e_raw = word_capacity(t, beta);
  const int e = (int)((uint64_t)e_raw < k ? (uint64_t)e_raw : k);
  if (e < 2) return QGO_NO_COMPRESSION;
  memset(out, 0, sizeof *out);
  out->p = p;
  out->t = t;
  out->e = e;
  out->d = e - 1;
  out->beta = beta;
  out->kmax = largest_common_dim(p, t);
  out->inv_qd = ldexp(1.0, -t * out->d);
  out->extraction = mode;
  if (mode == 1) { /* AddHighBits: plan.hpp:150-157 */
    const long double limit = exp2l((long double)t - 1.0L / e);
    uint64_t km = out->kmax;
    while (km > 0 && (long double)km * pm1sq(p) >= limit) --km;
    out->kmax = km;
  }
  return QGO_OK;
}

/* uncompressed_plan, plan.hpp:164-179. */
int qgo_uncompressed_plan(uint32_t p, uint64_t k, int beta, qgo_plan* out) {
  if (p < 2 || !qgo_is_prime(p)) return QGO_INVALID_MODULUS;
  if (k < 1) return QGO_INVALID_ARGUMENT;
  const int t = minimal_radix_exponent(p, k);
  if (t >= beta) return QGO_NO_COMPRESSION;
  memset(out, 0, sizeof *out);
  out->p = p;
  out->t = t;
  out->e = 1;
  out->d = 0;
  out->beta = beta;
  out->kmax = largest_common_dim(p, t);
  out->inv_qd = 1.0;
  return QGO_OK;
}

/* plan_packed_axis, plan.hpp:186-203. */
int qgo_plan_packed_axis(uint32_t p, uint64_t k, uint64_t axis_len, int beta, qgo_plan* out) {
  if (p < 2 || !qgo_is_prime(p)) return QGO_INVALID_MODULUS;
  if (k < 1 || axis_len < 1) return QGO_INVALID_ARGUMENT;
  const int t = minimal_radix_exponent(p, k);
  if (t >= beta) return QGO_NO_COMPRESSION;
  const uint64_t cap = (uint64_t)word_capacity(t, beta);
  memset(out, 0, sizeof *out);
  out->p = p;
  out->t = t;
  out->e = (int)(cap < axis_len ? cap : axis_len);
  out->d = out->e - 1;
  out->beta = beta;
  out->kmax = largest_common_dim(p, t);
  out->inv_qd = ldexp(1.0, -t * out->d);
  return QGO_OK;
}

/* The hand-built plan of the reference tests (test_pack.cpp:15-24, acceptance.cpp:29-38). */
int qgo_make_plan(uint32_t p, int t, int e, int beta, qgo_plan* out) {
  if (p < 2 || !qgo_is_prime(p)) return QGO_INVALID_MODULUS;
  memset(out, 0, sizeof *out);
  out->p = p;
  out->t = t;
  out->e = e;
  out->d = e - 1;
  out->beta = beta;
  out->kmax = ((UINT64_C(1) << t) - 1) / pm1sq(p);
  out->inv_qd = ldexp(1.0, -t * out->d);
  return QGO_OK;
}

/* choose_panel, plan.hpp:209-224. */
uint64_t qgo_choose_panel(uint32_t p, uint64_t k, int beta) {
  int direct_e = 1;
  qgo_plan pl;
  if (qgo_plan_compression(p, k, beta, 0, &pl) == QGO_OK) direct_e = pl.e;
  for (int t = 1; t < beta; ++t) {
    const uint64_t km = largest_common_dim(p, t);
    if (km == 0) continue;
    const uint64_t panel = km < k ? km : k;
    const uint64_t cap = (uint64_t)word_capacity(t, beta);
    const int e = (int)(cap < panel ? cap : panel);
    if (e > direct_e) return panel;
  }
  return 0;
}

/* ----------------------------------------------------------------- prng.hpp */

/* SplitMix64::next, prng.hpp:16-21, evaluated at counter index (state after
 * index+1 calls is seed + (index+1)*gamma). */
uint64_t qgo_splitmix64_at(uint64_t seed, uint64_t index) {
  uint64_t z = seed + (index + 1) * UINT64_C(0x9e3779b97f4a7c15);
  z = (z ^ (z >> 30)) * UINT64_C(0xbf58476d1ce4e5b9);
  z = (z ^ (z >> 27)) * UINT64_C(0x94d049bb133111eb);
  return z ^ (z >> 31);
}

/* random_residue_matrix, prng.hpp:31-38 (row-major fill, below(p) = next() % p, :25). */
void qgo_random_residue_matrix(size_t rows, size_t cols, uint32_t p, uint64_t seed, uint32_t* out) {
  qgo_random_residue_rows(0, rows, cols, p, seed, out);
}

/* Rows [row0, row0+rows) of the same matrix: the stream is counter-based. */
void qgo_random_residue_rows(size_t row0, size_t rows, size_t cols, uint32_t p, uint64_t seed,
                             uint32_t* out) {
  const uint64_t base = (uint64_t)row0 * cols;
  for (size_t i = 0; i < rows * cols; ++i)
    out[i] = (uint32_t)(qgo_splitmix64_at(seed, base + i) % p);
}

/* ----------------------------------------------------------------- pack.hpp */

static int check_backend(const qgo_plan* plan) { /* pack.hpp:19-24, DoubleWord: 53 bits */
  return plan->beta > 53 ? QGO_PLAN_MISMATCH : QGO_OK;
}

static uint64_t qmask(const qgo_plan* plan) { return (UINT64_C(1) << plan->t) - 1; }

/* compress_forward + horner_pack, pack.hpp:27-32, 47-54. */
int qgo_compress_forward(const uint32_t* v, size_t len, const qgo_plan* plan, double* out) {
  if (check_backend(plan)) return QGO_PLAN_MISMATCH;
  if (len > (size_t)plan->e) return QGO_SLOT_OVERFLOW;
  uint64_t r = 0;
  for (size_t i = len; i-- > 0;) r = (r << plan->t) | v[i];
  *out = (double)r;
  return QGO_OK;
}

/* compress_reverse, pack.hpp:59-70. */
int qgo_compress_reverse(const uint32_t* v, size_t len, const qgo_plan* plan, double* out) {
  if (check_backend(plan)) return QGO_PLAN_MISMATCH;
  if (len > (size_t)plan->e) return QGO_SLOT_OVERFLOW;
  uint64_t r = 0;
  for (size_t i = 0; i < len; ++i) r = (r << plan->t) | v[i];
  r <<= plan->t * (plan->e - (int)len);
  *out = (double)r;
  return QGO_OK;
}

/* extract_coefficient (DoubleWord), pack.hpp:78-100. */
uint32_t qgo_extract_coefficient(double w, const qgo_plan* plan) {
  uint64_t digit;
  if (plan->extraction == 1) {
    const double anchor = ldexp(1.0, plan->t * (2 * plan->d + 1));
    const double s = w + anchor;
    uint64_t bits;
    memcpy(&bits, &s, sizeof bits);
    const uint64_t mantissa = bits & ((UINT64_C(1) << 52) - 1);
    digit = (mantissa >> (52 - plan->t * plan->e)) & qmask(plan);
  } else {
    const double high = w * plan->inv_qd;
    digit = (uint64_t)(int64_t)high & qmask(plan);
  }
  return (uint32_t)(digit % plan->p);
}

static int fits_digits(double w, const qgo_plan* plan) { /* pack.hpp:107-111 */
  const int total_bits = plan->t * plan->e;
  return !(w < 0.0) && (w < (double)(UINT64_C(1) << total_bits));
}

/* extract_all, pack.hpp:104-119 (digits least significant first, unreduced). */
int qgo_extract_all(double w, const qgo_plan* plan, uint64_t* digits) {
  if (check_backend(plan)) return QGO_PLAN_MISMATCH;
  if (!fits_digits(w, plan)) return QGO_DIGIT_OVERFLOW;
  uint64_t bits = (uint64_t)w;
  for (int i = 0; i < plan->e; ++i) {
    digits[i] = bits & qmask(plan);
    bits >>= plan->t;
  }
  return QGO_OK;
}

/* redq, pack.hpp:124-137: every digit replaced by itself mod p. */
int qgo_redq(double w, const qgo_plan* plan, double* out) {
  if (check_backend(plan)) return QGO_PLAN_MISMATCH;
  if (!fits_digits(w, plan)) return QGO_DIGIT_OVERFLOW;
  const int total_bits = plan->t * plan->e;
  const uint64_t bits = (uint64_t)w;
  uint64_t r = 0;
  for (int i = 0; i < total_bits; i += plan->t) r |= (((bits >> i) & qmask(plan)) % plan->p) << i;
  *out = (double)r;
  return QGO_OK;
}

/* reduce_and_compress, pack.hpp:141-155: out has ceil(len/e) words. */
int qgo_reduce_and_compress(const double* row, size_t len, const qgo_plan* plan, double* out) {
  uint32_t* reduced = (uint32_t*)malloc((len ? len : 1) * sizeof(uint32_t));
  for (size_t i = 0; i < len; ++i) reduced[i] = qgo_extract_coefficient(row[i], plan);
  int st = QGO_OK;
  for (size_t g = 0, w = 0; g < len && st == QGO_OK; g += plan->e, ++w) {
    const size_t n = len - g < (size_t)plan->e ? len - g : (size_t)plan->e;
    st = qgo_compress_forward(reduced + g, n, plan, out + w);
  }
  free(reduced);
  return st;
}

/* ----------------------------------------------------------------- gemm.hpp */

static size_t group_count(size_t len, int slots) { return (len + slots - 1) / slots; } /* :41-43 */

/* compress_rows_reversed, gemm.hpp:104-118: m x ceil(k/e) words, Reversed/Column. */
int qgo_compress_rows_reversed(const qgo_plan* plan, const uint32_t* a, size_t m, size_t k,
                               double* ca) {
  if (k > plan->kmax) return QGO_PLAN_MISMATCH; /* check_common_dim, :29-35 */
  const size_t groups = group_count(k, plan->e);
  for (size_t i = 0; i < m; ++i)
    for (size_t g = 0; g < groups; ++g) {
      const size_t base = g * plan->e;
      const size_t len = k - base < (size_t)plan->e ? k - base : (size_t)plan->e;
      int st = qgo_compress_reverse(a + i * k + base, len, plan, ca + i * groups + g);
      if (st) return st;
    }
  return QGO_OK;
}

/* compress_cols_forward, gemm.hpp:122-140: ceil(k/e) x n words, Forward/Row. */
int qgo_compress_cols_forward(const qgo_plan* plan, const uint32_t* b, size_t k, size_t n,
                              double* cb) {
  if (k > plan->kmax) return QGO_PLAN_MISMATCH;
  const size_t groups = group_count(k, plan->e);
  uint32_t column[64];
  for (size_t g = 0; g < groups; ++g) {
    const size_t base = g * plan->e;
    const size_t len = k - base < (size_t)plan->e ? k - base : (size_t)plan->e;
    for (size_t j = 0; j < n; ++j) {
      for (size_t s = 0; s < len; ++s) column[s] = b[(base + s) * n + j];
      int st = qgo_compress_forward(column, len, plan, cb + g * n + j);
      if (st) return st;
    }
  }
  return QGO_OK;
}

/* compress_outer_cols, gemm.hpp:145-158: k x ceil(n/e) words, Forward/Column; no kmax check. */
int qgo_compress_outer_cols(const qgo_plan* plan, const uint32_t* b, size_t k, size_t n,
                            double* cb) {
  const size_t groups = group_count(n, plan->e);
  for (size_t i = 0; i < k; ++i)
    for (size_t g = 0; g < groups; ++g) {
      const size_t base = g * plan->e;
      const size_t len = n - base < (size_t)plan->e ? n - base : (size_t)plan->e;
      int st = qgo_compress_forward(b + i * n + base, len, plan, cb + i * groups + g);
      if (st) return st;
    }
  return QGO_OK;
}

/* compress_outer_rows, gemm.hpp:161-178: ceil(m/e) x k words, Forward/Row. */
int qgo_compress_outer_rows(const qgo_plan* plan, const uint32_t* a, size_t m, size_t k,
                            double* ca) {
  const size_t groups = group_count(m, plan->e);
  uint32_t column[64];
  for (size_t g = 0; g < groups; ++g) {
    const size_t base = g * plan->e;
    const size_t len = m - base < (size_t)plan->e ? m - base : (size_t)plan->e;
    for (size_t j = 0; j < k; ++j) {
      for (size_t s = 0; s < len; ++s) column[s] = a[(base + s) * k + j];
      int st = qgo_compress_forward(column, len, plan, ca + g * k + j);
      if (st) return st;
    }
  }
  return QGO_OK;
}

/* uncompress, gemm.hpp:182-204. */
int qgo_uncompress(const qgo_plan* plan, qgo_orientation o, const double* words,
                   size_t stored_rows, size_t stored_cols, size_t logical_rows,
                   size_t logical_cols, uint32_t* out) {
  uint64_t digits[64];
  memset(out, 0, logical_rows * logical_cols * sizeof(uint32_t));
  for (size_t si = 0; si < stored_rows; ++si)
    for (size_t sj = 0; sj < stored_cols; ++sj) {
      int st = qgo_extract_all(words[si * stored_cols + sj], plan, digits);
      if (st) return st;
      for (int s = 0; s < o.slots; ++s) {
        const uint64_t digit = o.direction == 1 ? digits[o.slots - 1 - s] : digits[s];
        size_t i = si, j = sj;
        if (o.axis == 1) j = sj * o.slots + s;
        else i = si * o.slots + s;
        if (i < logical_rows && j < logical_cols)
          out[i * logical_cols + j] = (uint32_t)(digit % plan->p);
      }
    }
  return QGO_OK;
}

/* ---- row-sharded worker pool (the reference is single-threaded; threads only
 * split independent output rows, each running the same loop body). */
typedef void (*row_fn)(void* ctx, size_t row0, size_t row1);
typedef struct {
  row_fn fn;
  void* ctx;
  size_t r0, r1;
} row_job;

static void* row_thread(void* arg) {
  row_job* j = (row_job*)arg;
  j->fn(j->ctx, j->r0, j->r1);
  return NULL;
}

static void parallel_rows(row_fn fn, void* ctx, size_t rows, int threads) {
  if (threads <= 1 || rows < 2) {
    fn(ctx, 0, rows);
    return;
  }
  if ((size_t)threads > rows) threads = (int)rows;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  row_job* jobs = (row_job*)malloc(sizeof(row_job) * threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].r0 = rows * t / threads;
    jobs[t].r1 = rows * (t + 1) / threads;
    pthread_create(&th[t], NULL, row_thread, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

typedef struct {
  const double *ca, *cb;
  size_t n, groups;
  double inv_qd;
  double* acc;
} common_ctx;

/* Hot loop of packed_common_product, gemm.hpp:233-242, with
 * DoubleWord::high_part = (double)(int64)(a*b*inv_qd), word.hpp:28-30. */
static void common_rows(void* vctx, size_t r0, size_t r1) {
  const common_ctx* c = (const common_ctx*)vctx;
  for (size_t i = r0; i < r1; ++i) {
    const double* arow = c->ca + i * c->groups;
    double* crow = c->acc + i * c->n;
    for (size_t j = 0; j < c->n; ++j) crow[j] = 0.0;
    for (size_t g = 0; g < c->groups; ++g) {
      const double a = arow[g];
      const double* brow = c->cb + g * c->n;
      for (size_t j = 0; j < c->n; ++j) crow[j] += (double)(int64_t)(a * brow[j] * c->inv_qd);
    }
  }
}

/* packed_common_product, gemm.hpp:210-244 (checks :213-225). */
int qgo_packed_common_product(const qgo_plan* plan, const double* ca, const double* cb,
                              size_t m, size_t n, size_t groups, size_t k_logical,
                              double* acc, int threads) {
  if (k_logical > plan->kmax) return QGO_PLAN_MISMATCH;
  if (group_count(k_logical, plan->e) != groups) return QGO_DIMENSION_MISMATCH;
  common_ctx c = {ca, cb, n, groups, plan->inv_qd, acc};
  parallel_rows(common_rows, &c, m, threads);
  return QGO_OK;
}

/* reduce_common_entry, gemm.hpp:247-250. */
uint32_t qgo_reduce_common_entry(double w, const qgo_plan* plan) {
  return (uint32_t)(((uint64_t)w & qmask(plan)) % plan->p);
}

/* mul_common_compressed(A, B, plan), gemm.hpp:254-271. */
int qgo_mul_common_compressed(const qgo_plan* plan, const uint32_t* a, const uint32_t* b,
                              size_t m, size_t k, size_t n, uint32_t* c, int threads) {
  const size_t groups = group_count(k, plan->e);
  double* ca = (double*)malloc((m * groups + 1) * sizeof(double));
  double* cb = (double*)malloc((groups * n + 1) * sizeof(double));
  double* acc = (double*)malloc((m * n + 1) * sizeof(double));
  int st = qgo_compress_rows_reversed(plan, a, m, k, ca);
  if (!st) st = qgo_compress_cols_forward(plan, b, k, n, cb);
  if (!st) st = qgo_packed_common_product(plan, ca, cb, m, n, groups, k, acc, threads);
  if (!st)
    for (size_t i = 0; i < m * n; ++i) c[i] = qgo_reduce_common_entry(acc[i], plan);
  free(ca);
  free(cb);
  free(acc);
  return st;
}

/* mul_common_repacked, gemm.hpp:275-280: C reduced, rows repacked forward (m x ceil(n/e)). */
int qgo_mul_common_repacked(const qgo_plan* plan, const uint32_t* a, const uint32_t* b,
                            size_t m, size_t k, size_t n, double* cc, int threads) {
  uint32_t* c = (uint32_t*)malloc((m * n + 1) * sizeof(uint32_t));
  int st = qgo_mul_common_compressed(plan, a, b, m, k, n, c, threads);
  if (!st) st = qgo_compress_outer_cols(plan, c, m, n, cc);
  free(c);
  return st;
}

typedef struct {
  const uint32_t* a;
  const double* cb;
  size_t k, h_cols;
  double* cc;
} right_ctx;

/* Hot loop of packed_right_product, gemm.hpp:300-308. */
static void right_rows(void* vctx, size_t r0, size_t r1) {
  const right_ctx* c = (const right_ctx*)vctx;
  for (size_t i = r0; i < r1; ++i) {
    double* crow = c->cc + i * c->h_cols;
    for (size_t h = 0; h < c->h_cols; ++h) crow[h] = 0.0;
    for (size_t l = 0; l < c->k; ++l) {
      const double ail = (double)c->a[i * c->k + l];
      const double* brow = c->cb + l * c->h_cols;
      for (size_t h = 0; h < c->h_cols; ++h) crow[h] += ail * brow[h];
    }
  }
}

/* packed_right_product, gemm.hpp:285-310: cc is m x ceil(n/e). */
int qgo_packed_right_product(const qgo_plan* plan, const uint32_t* a, const double* cb,
                             size_t m, size_t k, size_t n, double* cc, int threads) {
  if (k > plan->kmax) return QGO_PLAN_MISMATCH;
  right_ctx c = {a, cb, k, group_count(n, plan->e), cc};
  parallel_rows(right_rows, &c, m, threads);
  return QGO_OK;
}

/* redq_in_place, gemm.hpp:313-316. */
int qgo_redq_in_place(const qgo_plan* plan, double* words, size_t count) {
  for (size_t i = 0; i < count; ++i) {
    int st = qgo_redq(words[i], plan, &words[i]);
    if (st) return st;
  }
  return QGO_OK;
}

/* mul_right_compressed(a, cb), gemm.hpp:320-325. */
int qgo_mul_right_compressed(const qgo_plan* plan, const uint32_t* a, const double* cb,
                             size_t m, size_t k, size_t n, double* cc, int threads) {
  int st = qgo_packed_right_product(plan, a, cb, m, k, n, cc, threads);
  if (!st) st = qgo_redq_in_place(plan, cc, m * group_count(n, plan->e));
  return st;
}

/* plan_full, plan.hpp:229-252: word capacity E split as (dq+1)(dtheta+1),
 * dq+1 = floor(sqrt(E)), dtheta+1 = E / (dq+1). */
int qgo_plan_full(uint32_t p, uint64_t k, int beta, qgo_full_plan* out) {
  if (p < 2 || !qgo_is_prime(p)) return QGO_INVALID_MODULUS;
  if (k < 1 || beta < 2) return QGO_INVALID_ARGUMENT;
  const int t = minimal_radix_exponent(p, k);
  const int capacity = t < beta ? word_capacity(t, beta) : 0;
  if (capacity < 4) return QGO_NO_COMPRESSION;
  int qs = (int)sqrt((double)capacity);
  while (qs * qs > capacity) --qs;
  while ((qs + 1) * (qs + 1) <= capacity) ++qs;
  const int ts = capacity / qs;
  memset(out, 0, sizeof *out);
  out->base.p = p;
  out->base.t = t;
  out->base.e = qs * ts;
  out->base.d = out->base.e - 1;
  out->base.beta = beta;
  out->base.kmax = largest_common_dim(p, t);
  out->base.inv_qd = ldexp(1.0, -t * out->base.d);
  out->dq = qs - 1;
  out->dtheta = ts - 1;
  out->theta_exponent = t * qs;
  return QGO_OK;
}

typedef struct {
  const double* ca;
  const uint32_t* b;
  size_t k, n;
  double* cc;
} left_ctx;

/* Hot loop of packed_left_product, gemm.hpp:354-362. */
static void left_rows(void* vctx, size_t r0, size_t r1) {
  const left_ctx* c = (const left_ctx*)vctx;
  for (size_t g = r0; g < r1; ++g) {
    double* crow = c->cc + g * c->n;
    for (size_t j = 0; j < c->n; ++j) crow[j] = 0.0;
    for (size_t l = 0; l < c->k; ++l) {
      const double w = c->ca[g * c->k + l];
      const uint32_t* brow = c->b + l * c->n;
      for (size_t j = 0; j < c->n; ++j) crow[j] += w * (double)brow[j];
    }
  }
}

/* packed_left_product, gemm.hpp:340-364: ca is ceil(m/e) x k (compress_outer_rows). */
int qgo_packed_left_product(const qgo_plan* plan, const double* ca, const uint32_t* b, size_t m, size_t k,
                            size_t n, double* cc, int threads) {
  if (k > plan->kmax) return QGO_PLAN_MISMATCH;
  left_ctx c = {ca, b, k, n, cc};
  parallel_rows(left_rows, &c, group_count(m, plan->e), threads);
  return QGO_OK;
}

/* mul_left_compressed, gemm.hpp:366-371. */
int qgo_mul_left_compressed(const qgo_plan* plan, const double* ca, const uint32_t* b, size_t m, size_t k,
                            size_t n, double* cc, int threads) {
  int st = qgo_packed_left_product(plan, ca, b, m, k, n, cc, threads);
  if (!st) st = qgo_redq_in_place(plan, cc, group_count(m, plan->e) * n);
  return st;
}

/* mul_full_compressed, gemm.hpp:377-445: rows of A packed in base Q with
 * dq+1 slots, columns of B in base Theta = Q^(dq+1) with dtheta+1 slots; digit
 * (i, j) of entry (g, h) at base-Q position i + j (dq+1) is C[g(dq+1)+i][h(dtheta+1)+j]. */
int qgo_mul_full_compressed(const qgo_full_plan* fp, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                            size_t n, uint32_t* c) {
  const qgo_plan* pl = &fp->base;
  if (pl->beta > 53) return QGO_PLAN_MISMATCH;
  if (k > pl->kmax) return QGO_PLAN_MISMATCH;
  const int qs = fp->dq + 1, ts = fp->dtheta + 1, t = pl->t;
  const size_t gr = group_count(m, qs), hc = group_count(n, ts);
  double* ma = (double*)malloc((gr * k + 1) * sizeof(double));
  double* mb = (double*)malloc((k * hc + 1) * sizeof(double));
  double* acc = (double*)calloc(gr * hc + 1, sizeof(double));
  for (size_t g = 0; g < gr; ++g)
    for (size_t l = 0; l < k; ++l) {
      uint64_t w = 0;
      const size_t len = m - g * qs < (size_t)qs ? m - g * qs : (size_t)qs;
      for (size_t s = len; s-- > 0;) w = (w << t) | a[(g * qs + s) * k + l];
      ma[g * k + l] = (double)w;
    }
  for (size_t l = 0; l < k; ++l)
    for (size_t h = 0; h < hc; ++h) {
      uint64_t w = 0;
      const size_t len = n - h * ts < (size_t)ts ? n - h * ts : (size_t)ts;
      for (size_t s = len; s-- > 0;) w = (w << fp->theta_exponent) | b[l * n + h * ts + s];
      mb[l * hc + h] = (double)w;
    }
  for (size_t g = 0; g < gr; ++g)
    for (size_t l = 0; l < k; ++l) {
      const double w = ma[g * k + l];
      for (size_t h = 0; h < hc; ++h) acc[g * hc + h] += w * mb[l * hc + h];
    }
  const uint64_t mask = (UINT64_C(1) << t) - 1;
  for (size_t g = 0; g < gr; ++g)
    for (size_t h = 0; h < hc; ++h) {
      const uint64_t bits = (uint64_t)acc[g * hc + h];
      for (int j = 0; j < ts; ++j)
        for (int i = 0; i < qs; ++i) {
          const uint64_t digit = (bits >> (t * (i + j * qs))) & mask;
          const size_t row = g * qs + i, col = h * ts + j;
          if (row < m && col < n) c[row * n + col] = (uint32_t)(digit % pl->p);
        }
    }
  free(ma);
  free(mb);
  free(acc);
  return QGO_OK;
}

/* blocked_accumulate, gemm.hpp:450-489: k-panels, mod-p accumulation between them. */
int qgo_blocked_accumulate(const qgo_plan* plan, const uint32_t* a, const uint32_t* b,
                           size_t m, size_t k, size_t n, size_t kpanel, uint32_t* c,
                           int threads) {
  if (kpanel < 1) return QGO_INVALID_ARGUMENT;
  if (kpanel > plan->kmax) return QGO_PLAN_MISMATCH;
  memset(c, 0, m * n * sizeof(uint32_t));
  uint32_t* ap = (uint32_t*)malloc((m * kpanel + 1) * sizeof(uint32_t));
  uint32_t* cp = (uint32_t*)malloc((m * n + 1) * sizeof(uint32_t));
  int st = QGO_OK;
  for (size_t base = 0; base < k && !st; base += kpanel) {
    const size_t len = k - base < kpanel ? k - base : kpanel;
    for (size_t i = 0; i < m; ++i) memcpy(ap + i * len, a + i * k + base, len * sizeof(uint32_t));
    st = qgo_mul_common_compressed(plan, ap, b + base * n, m, len, n, cp, threads);
    for (size_t idx = 0; idx < m * n && !st; ++idx) c[idx] = (uint32_t)(((uint64_t)c[idx] + cp[idx]) % plan->p);
  }
  free(ap);
  free(cp);
  return st;
}

typedef struct {
  uint32_t p;
  const uint32_t *a, *b;
  size_t k, n;
  uint32_t* c;
} naive_ctx;

/* naive_gemm body, gemm.hpp:80-100: uint64 accumulation, % p every 1024 terms. */
static void naive_rows(void* vctx, size_t r0, size_t r1) {
  const naive_ctx* c = (const naive_ctx*)vctx;
  uint64_t* acc = (uint64_t*)malloc((c->n + 1) * sizeof(uint64_t));
  for (size_t i = r0; i < r1; ++i) {
    memset(acc, 0, c->n * sizeof(uint64_t));
    for (size_t l = 0; l < c->k; ++l) {
      const uint64_t ail = c->a[i * c->k + l];
      const uint32_t* brow = c->b + l * c->n;
      for (size_t j = 0; j < c->n; ++j) acc[j] += ail * brow[j];
      if ((l + 1) % 1024 == 0)
        for (size_t j = 0; j < c->n; ++j) acc[j] %= c->p;
    }
    for (size_t j = 0; j < c->n; ++j) c->c[i * c->n + j] = (uint32_t)(acc[j] % c->p);
  }
  free(acc);
}

int qgo_naive_gemm(uint32_t p, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                   size_t n, uint32_t* c, int threads) {
  naive_ctx ctx = {p, a, b, k, n, c};
  parallel_rows(naive_rows, &ctx, m, threads);
  return QGO_OK;
}

/* residue_checksum, bench.hpp:43-47: sum mod 2^32. */
uint32_t qgo_residue_checksum(const uint32_t* c, size_t count) {
  uint32_t s = 0;
  for (size_t i = 0; i < count; ++i) s += c[i];
  return s;
}

/* ================================================ Int64Word (word.hpp:36-54)
 * The same routines over uint64 words: products wrap modulo 2^64, the common
 * product adds high_part = ((a b) >> t d) & (Q-1) per term (word.hpp:51-53),
 * extraction is ((w >> t d) & (Q-1)) mod p (pack.hpp:96-98). Plans may use
 * beta up to 63. */
static int check_backend_i64(const qgo_plan* plan) { return plan->beta > 63 ? QGO_PLAN_MISMATCH : QGO_OK; }

static uint64_t i64_forward(const uint32_t* v, size_t len, int t) { /* pack.hpp:27-32 */
  uint64_t r = 0;
  for (size_t i = len; i-- > 0;) r = (r << t) | v[i];
  return r;
}
static uint64_t i64_reverse(const uint32_t* v, size_t len, int t, int e) { /* pack.hpp:59-70 */
  uint64_t r = 0;
  for (size_t i = 0; i < len; ++i) r = (r << t) | v[i];
  return r << (t * (e - (int)len));
}

int qgo_compress_rows_reversed_i64(const qgo_plan* plan, const uint32_t* a, size_t m, size_t k, uint64_t* ca) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  if (k > plan->kmax) return QGO_PLAN_MISMATCH;
  const size_t groups = group_count(k, plan->e);
  for (size_t i = 0; i < m; ++i)
    for (size_t g = 0; g < groups; ++g) {
      const size_t base = g * plan->e, len = k - base < (size_t)plan->e ? k - base : (size_t)plan->e;
      ca[i * groups + g] = i64_reverse(a + i * k + base, len, plan->t, plan->e);
    }
  return QGO_OK;
}

int qgo_compress_cols_forward_i64(const qgo_plan* plan, const uint32_t* b, size_t k, size_t n, uint64_t* cb) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  if (k > plan->kmax) return QGO_PLAN_MISMATCH;
  const size_t groups = group_count(k, plan->e);
  uint32_t column[64];
  for (size_t g = 0; g < groups; ++g) {
    const size_t base = g * plan->e, len = k - base < (size_t)plan->e ? k - base : (size_t)plan->e;
    for (size_t j = 0; j < n; ++j) {
      for (size_t s = 0; s < len; ++s) column[s] = b[(base + s) * n + j];
      cb[g * n + j] = i64_forward(column, len, plan->t);
    }
  }
  return QGO_OK;
}

int qgo_compress_outer_cols_i64(const qgo_plan* plan, const uint32_t* b, size_t k, size_t n, uint64_t* cb) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  const size_t groups = group_count(n, plan->e);
  for (size_t i = 0; i < k; ++i)
    for (size_t g = 0; g < groups; ++g) {
      const size_t base = g * plan->e, len = n - base < (size_t)plan->e ? n - base : (size_t)plan->e;
      cb[i * groups + g] = i64_forward(b + i * n + base, len, plan->t);
    }
  return QGO_OK;
}

int qgo_compress_outer_rows_i64(const qgo_plan* plan, const uint32_t* a, size_t m, size_t k, uint64_t* ca) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  const size_t groups = group_count(m, plan->e);
  uint32_t column[64];
  for (size_t g = 0; g < groups; ++g) {
    const size_t base = g * plan->e, len = m - base < (size_t)plan->e ? m - base : (size_t)plan->e;
    for (size_t j = 0; j < k; ++j) {
      for (size_t s = 0; s < len; ++s) column[s] = a[(base + s) * k + j];
      ca[g * k + j] = i64_forward(column, len, plan->t);
    }
  }
  return QGO_OK;
}

/* packed_common_product<Int64Word>, gemm.hpp:210-244 */
int qgo_packed_common_product_i64(const qgo_plan* plan, const uint64_t* ca, const uint64_t* cb, size_t m, size_t n,
                                  size_t groups, uint64_t* acc) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  const int sh = plan->t * plan->d;
  const uint64_t mask = qmask(plan);
  for (size_t i = 0; i < m; ++i)
    for (size_t j = 0; j < n; ++j) {
      uint64_t s = 0;
      for (size_t g = 0; g < groups; ++g) s += ((ca[i * groups + g] * cb[g * n + j]) >> sh) & mask;
      acc[i * n + j] = s;
    }
  return QGO_OK;
}

uint32_t qgo_reduce_common_entry_i64(uint64_t w, const qgo_plan* plan) { return (uint32_t)((w & qmask(plan)) % plan->p); }

uint32_t qgo_extract_coefficient_i64(uint64_t w, const qgo_plan* plan) {
  return (uint32_t)(((w >> (plan->t * plan->d)) & qmask(plan)) % plan->p);
}

/* redq<Int64Word>, pack.hpp:124-137 */
int qgo_redq_i64(uint64_t w, const qgo_plan* plan, uint64_t* out) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  const int total = plan->t * plan->e;
  if (total < 64 && w >= (UINT64_C(1) << total)) return QGO_DIGIT_OVERFLOW;
  uint64_t r = 0;
  for (int i = 0; i < total; i += plan->t) r |= (((w >> i) & qmask(plan)) % plan->p) << i;
  *out = r;
  return QGO_OK;
}

int qgo_uncompress_i64(const qgo_plan* plan, qgo_orientation o, const uint64_t* words, size_t stored_rows,
                       size_t stored_cols, size_t logical_rows, size_t logical_cols, uint32_t* out) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  const int total = plan->t * plan->e;
  memset(out, 0, logical_rows * logical_cols * sizeof(uint32_t));
  for (size_t si = 0; si < stored_rows; ++si)
    for (size_t sj = 0; sj < stored_cols; ++sj) {
      const uint64_t w = words[si * stored_cols + sj];
      if (total < 64 && w >= (UINT64_C(1) << total)) return QGO_DIGIT_OVERFLOW;
      for (int s = 0; s < o.slots; ++s) {
        const int di = o.direction == 1 ? o.slots - 1 - s : s;
        const uint64_t digit = di < plan->e ? (w >> (plan->t * di)) & qmask(plan) : 0;
        const size_t i = o.axis == 1 ? si : si * o.slots + s, j = o.axis == 1 ? sj * o.slots + s : sj;
        if (i < logical_rows && j < logical_cols) out[i * logical_cols + j] = (uint32_t)(digit % plan->p);
      }
    }
  return QGO_OK;
}

/* packed_right_product<Int64Word>, gemm.hpp:285-310: cc = A x CBo, wrapping. */
int qgo_packed_right_product_i64(const qgo_plan* plan, const uint32_t* a, const uint64_t* cb, size_t m, size_t k,
                                 size_t n, uint64_t* cc) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  if (k > plan->kmax) return QGO_PLAN_MISMATCH;
  const size_t h = group_count(n, plan->e);
  for (size_t i = 0; i < m; ++i)
    for (size_t g = 0; g < h; ++g) {
      uint64_t s = 0;
      for (size_t l = 0; l < k; ++l) s += (uint64_t)a[i * k + l] * cb[l * h + g];
      cc[i * h + g] = s;
    }
  return QGO_OK;
}

/* packed_left_product<Int64Word>, gemm.hpp:340-364 */
int qgo_packed_left_product_i64(const qgo_plan* plan, const uint64_t* ca, const uint32_t* b, size_t m, size_t k,
                                size_t n, uint64_t* cc) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  if (k > plan->kmax) return QGO_PLAN_MISMATCH;
  const size_t gr = group_count(m, plan->e);
  for (size_t g = 0; g < gr; ++g)
    for (size_t j = 0; j < n; ++j) {
      uint64_t s = 0;
      for (size_t l = 0; l < k; ++l) s += ca[g * k + l] * (uint64_t)b[l * n + j];
      cc[g * n + j] = s;
    }
  return QGO_OK;
}

int qgo_redq_in_place_i64(const qgo_plan* plan, uint64_t* words, size_t count) {
  for (size_t i = 0; i < count; ++i) {
    int st = qgo_redq_i64(words[i], plan, words + i);
    if (st) return st;
  }
  return QGO_OK;
}

/* mul_full_compressed<Int64Word>, gemm.hpp:377-445 */
int qgo_mul_full_compressed_i64(const qgo_full_plan* fp, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                                size_t n, uint32_t* c) {
  const qgo_plan* pl = &fp->base;
  if (check_backend_i64(pl)) return QGO_PLAN_MISMATCH;
  if (k > pl->kmax) return QGO_PLAN_MISMATCH;
  const int qs = fp->dq + 1, ts = fp->dtheta + 1, t = pl->t;
  const size_t gr = group_count(m, qs), hc = group_count(n, ts);
  const uint64_t mask = qmask(pl);
  for (size_t g = 0; g < gr; ++g)
    for (size_t h = 0; h < hc; ++h) {
      uint64_t acc = 0;
      for (size_t l = 0; l < k; ++l) {
        uint64_t wa = 0, wb = 0;
        const size_t la = m - g * qs < (size_t)qs ? m - g * qs : (size_t)qs;
        for (size_t s = la; s-- > 0;) wa = (wa << t) | a[(g * qs + s) * k + l];
        const size_t lb = n - h * ts < (size_t)ts ? n - h * ts : (size_t)ts;
        for (size_t s = lb; s-- > 0;) wb = (wb << fp->theta_exponent) | b[l * n + h * ts + s];
        acc += wa * wb;
      }
      for (int j = 0; j < ts; ++j)
        for (int i = 0; i < qs; ++i) {
          const size_t row = g * qs + i, col = h * ts + j;
          if (row < m && col < n) c[row * n + col] = (uint32_t)(((acc >> (t * (i + j * qs))) & mask) % pl->p);
        }
    }
  return QGO_OK;
}

/* blocked_accumulate<Int64Word>, gemm.hpp:450-489 */
int qgo_blocked_accumulate_i64(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                               size_t kpanel, uint32_t* c) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  if (kpanel < 1) return QGO_INVALID_ARGUMENT;
  if (kpanel > plan->kmax) return QGO_PLAN_MISMATCH;
  memset(c, 0, m * n * sizeof(uint32_t));
  const int sh = plan->t * plan->d;
  const uint64_t mask = qmask(plan);
  for (size_t k0 = 0; k0 < k; k0 += kpanel) {
    const size_t len = k - k0 < kpanel ? k - k0 : kpanel, groups = group_count(len, plan->e);
    for (size_t i = 0; i < m; ++i)
      for (size_t j = 0; j < n; ++j) {
        uint64_t acc = 0;
        uint32_t col[64];
        for (size_t g = 0; g < groups; ++g) {
          const size_t base = g * plan->e, gl = len - base < (size_t)plan->e ? len - base : (size_t)plan->e;
          for (size_t s = 0; s < gl; ++s) col[s] = b[(k0 + base + s) * n + j];
          const uint64_t wa = i64_reverse(a + i * k + k0 + base, gl, plan->t, plan->e), wb = i64_forward(col, gl, plan->t);
          acc += ((wa * wb) >> sh) & mask;
        }
        c[i * n + j] = (uint32_t)(((uint64_t)c[i * n + j] + (acc & mask) % plan->p) % plan->p);
      }
  }
  return QGO_OK;
}

/* reduce_and_compress<Int64Word>, pack.hpp:141-155 */
int qgo_reduce_and_compress_i64(const uint64_t* row, size_t len, const qgo_plan* plan, uint64_t* out) {
  if (check_backend_i64(plan)) return QGO_PLAN_MISMATCH;
  uint32_t red[64];
  for (size_t g = 0; g < len; g += plan->e) {
    const size_t gl = len - g < (size_t)plan->e ? len - g : (size_t)plan->e;
    for (size_t s = 0; s < gl; ++s) red[s] = qgo_extract_coefficient_i64(row[g + s], plan);
    out[g / plan->e] = i64_forward(red, gl, plan->t);
  }
  return QGO_OK;
}
