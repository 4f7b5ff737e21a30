/* oracle.c — plain-C restatement of the reference eigenid hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled with -ffp-contract=off
 * so every product/sum rounds exactly where the reference's (x86-64, no FMA)
 * build rounds; tests/test_oracle.py checks it bit-for-bit against the
 * unmodified reference (oracle/_ref).
 *
 * Paths cited as file:line are relative to /root/reference/proj.
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static void set_err(orc_err* err, int code, int64_t index, double gap,
                    const char* msg) {
  if (!err) return;
  err->code = code;
  err->index = index;
  err->gap = gap;
  snprintf(err->msg, sizeof(err->msg), "%s", msg);
}

/* ------------------------------------------------------------------ */
/* mt19937_64 (std::mt19937_64 as specified by [rand.predef]) and the  */
/* hand-written variate transforms of SeededDraws, matrix_io.cpp:39-71 */
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
  int have_spare;
  double spare;
} orc_rng;

static void rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = 312;
  r->have_spare = 0;
  r->spare = 0.0;
}

static uint64_t rng_next(orc_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* SeededDraws::unit, matrix_io.cpp:44 */
static double rng_unit(orc_rng* r) {
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}

/* SeededDraws::uniform_open, matrix_io.cpp:46-51 */
static double rng_uniform_open(orc_rng* r) {
  for (;;) {
    double v = 2.0 * rng_unit(r) - 1.0;
    if (v > -1.0) return v;
  }
}

/* SeededDraws::gaussian (Box-Muller, cached spare), matrix_io.cpp:53-65 */
static double rng_gaussian(orc_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_unit(r);
  double u2 = rng_unit(r);
  while (u1 <= 0.0) u1 = rng_unit(r);
  double rad = sqrt(-2.0 * log(u1));
  double theta = 2.0 * M_PI * u2;
  r->spare = rad * sin(theta);
  r->have_spare = 1;
  return rad * cos(theta);
}

void orc_gaussian_stream(uint64_t seed, size_t count, double* out) {
  orc_rng r;
  rng_seed(&r, seed);
  for (size_t t = 0; t < count; ++t) out[t] = rng_gaussian(&r);
}

/* random_symmetric (matrix_io.cpp:171-181) followed by
 * SymmetricMatrix::build(kSymmetrize) (matrix.cpp:10-38). */
void orc_random_symmetric(uint64_t seed, size_t n, int uniform, double* e) {
  orc_rng r;
  rng_seed(&r, seed);
  for (size_t t = 0; t < n * n; ++t)
    e[t] = uniform ? rng_uniform_open(&r) : rng_gaussian(&r);
  double max_asym = 0.0;
  for (size_t rr = 0; rr < n; ++rr)
    for (size_t c = rr + 1; c < n; ++c) {
      double d = fabs(e[rr * n + c] - e[c * n + rr]);
      if (d > max_asym) max_asym = d;
    }
  if (max_asym > 0.0)
    for (size_t rr = 0; rr < n; ++rr)
      for (size_t c = rr + 1; c < n; ++c) {
        double m = 0.5 * (e[rr * n + c] + e[c * n + rr]);
        e[rr * n + c] = m;
        e[c * n + rr] = m;
      }
}

/* splitmix64, bench.cpp:78-83 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* SymmetricMatrix::minor_matrix, matrix.cpp:51-68 */
void orc_minor(const double* a, size_t n, size_t j, double* out) {
  size_t m = n - 1, rr = 0;
  for (size_t r = 0; r < n; ++r) {
    if (r == j) continue;
    size_t cc = 0;
    for (size_t c = 0; c < n; ++c) {
      if (c == j) continue;
      out[rr * m + cc] = a[r * n + c];
      ++cc;
    }
    ++rr;
  }
}

static int cmp_double(const void* pa, const void* pb) {
  double x = *(const double*)pa, y = *(const double*)pb;
  return (x < y) ? -1 : (x > y);
}

void orc_c5_lambda(uint64_t seed, size_t n, double* lambda) {
  orc_rng r;
  rng_seed(&r, seed);
  for (size_t k = 0; k < n; ++k) lambda[k] = rng_uniform_open(&r);
  for (;;) {
    qsort(lambda, n, sizeof(double), cmp_double);
    int ties = 0;
    for (size_t k = 0; k + 1 < n; ++k)
      if (lambda[k + 1] == lambda[k]) {
        lambda[k + 1] = rng_uniform_open(&r);
        ties = 1;
      }
    if (!ties) return;
  }
}

/* mu_{j,k} = l_k + u (l_{k+1} - l_k), u = (splitmix64(seed ^ (j<<32 ^ k))
 * >> 11 + 0.5) 2^-53 in (0,1).  Midpoint fallback keeps mu strictly inside
 * (l_k, l_{k+1}).  The device generator performs the same three roundings. */
void orc_c5_mu_row(uint64_t seed, const double* lambda, size_t n, size_t j,
                   double* mu) {
  for (size_t k = 0; k + 1 < n; ++k) {
    uint64_t h = orc_splitmix64(seed ^ (((uint64_t)j << 32) ^ (uint64_t)k));
    double u = ((double)(h >> 11) + 0.5) * 0x1.0p-53;
    double lo = lambda[k], hi = lambda[k + 1];
    double t = hi - lo;
    double m = u * t;
    double v = lo + m;
    if (!(v > lo && v < hi)) v = 0.5 * (lo + hi);
    mu[k] = v;
  }
}

/* ------------------------------------------------------------------ */
/* tred1 without Q: eigensolve.cpp:19-69                               */
/* ------------------------------------------------------------------ */
void orc_tridiagonalize(const double* src, size_t n, size_t max_steps,
                        double* dout, double* offdiag) {
  double* a = (double*)malloc(n * n * sizeof(double));
  double* e = (double*)calloc(n ? n : 1, sizeof(double));
  memcpy(a, src, n * n * sizeof(double));
  size_t steps = 0;
  for (size_t i = n; i-- > 1 && steps < max_steps; ++steps) {
    const size_t l = i - 1;
    double h = 0.0, scale = 0.0;
    if (l > 0) {
      for (size_t k = 0; k <= l; ++k) scale += fabs(a[i * n + k]);
      if (scale == 0.0) {
        e[i] = a[i * n + l];
      } else {
        for (size_t k = 0; k <= l; ++k) {
          a[i * n + k] /= scale;
          h += a[i * n + k] * a[i * n + k];
        }
        double f = a[i * n + l];
        double g = f >= 0.0 ? -sqrt(h) : sqrt(h);
        e[i] = scale * g;
        h -= f * g;
        a[i * n + l] = f - g;
        f = 0.0;
        for (size_t j = 0; j <= l; ++j) {
          g = 0.0;
          for (size_t k = 0; k <= j; ++k) g += a[j * n + k] * a[i * n + k];
          for (size_t k = j + 1; k <= l; ++k) g += a[k * n + j] * a[i * n + k];
          e[j] = g / h;
          f += e[j] * a[i * n + j];
        }
        const double hh = f / (h + h);
        for (size_t j = 0; j <= l; ++j) {
          f = a[i * n + j];
          e[j] = g = e[j] - hh * f;
          for (size_t k = 0; k <= j; ++k)
            a[j * n + k] -= f * e[k] + g * a[i * n + k];
        }
      }
    } else {
      e[i] = a[i * n + l];
    }
  }
  for (size_t i = 0; i < n; ++i) dout[i] = a[i * n + i];
  for (size_t i = 0; i + 1 < n; ++i) offdiag[i] = e[i + 1];
  free(a);
  free(e);
}

/* Implicit-shift QL, eigenvalues only, then ascending sort:
 * eigensolve.cpp:72-128. */
int orc_ql(double* d, const double* offdiag, size_t n, orc_err* err) {
  double* e = (double*)calloc(n ? n : 1, sizeof(double));
  for (size_t i = 0; i + 1 < n; ++i) e[i] = offdiag[i];
  const double eps = 2.220446049250313080847e-16;
  const size_t max_iter = 30 * n;
  size_t iter = 0;
  for (size_t l = 0; l < n; ++l) {
    size_t m;
    do {
      for (m = l; m + 1 < n; ++m) {
        const double dd = fabs(d[m]) + fabs(d[m + 1]);
        if (fabs(e[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (++iter > max_iter) {
          char buf[160];
          snprintf(buf, sizeof buf,
                   "QL iteration budget exhausted (%zu iterations) before "
                   "isolating eigenvalue %zu", max_iter, l);
          set_err(err, ORC_E_CONVERGENCE, (int64_t)l, 0.0, buf);
          free(e);
          return ORC_E_CONVERGENCE;
        }
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int underflow = 0;
        for (size_t i = m; i-- > l;) {
          double f = s * e[i];
          const double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            underflow = 1;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
        }
        if (underflow) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  qsort(d, n, sizeof(double), cmp_double);
  free(e);
  return ORC_OK;
}

int orc_eigenvalues(const double* a, size_t n, double* out, orc_err* err) {
  double* off = (double*)malloc((n ? n : 1) * sizeof(double));
  orc_tridiagonalize(a, n, (size_t)-1, out, off);
  int st = orc_ql(out, off, n, err);
  free(off);
  return st;
}

/* ------------------------------------------------------------------ */
/* identity engine: identity.cpp                                       */
/* ------------------------------------------------------------------ */

/* check_fully_nondegenerate, identity.cpp:141-149 */
int orc_check_fully_nondegenerate(const double* s, size_t n, double tol,
                                  orc_err* err) {
  const double range = s[n - 1] - s[0];
  for (size_t k = 0; k + 1 < n; ++k)
    if (s[k + 1] - s[k] <= tol * range) {
      char buf[160];
      snprintf(buf, sizeof buf,
               "spectrum is degenerate between eigenvalues %zu and %zu", k,
               k + 1);
      set_err(err, ORC_E_DEGENERATE, (int64_t)k, s[k + 1] - s[k], buf);
      return ORC_E_DEGENERATE;
    }
  return ORC_OK;
}

/* checked_min_gap, identity.cpp:42-55 */
static int checked_min_gap(const double* s, size_t n, size_t i, double tol,
                           double* gap_out, orc_err* err) {
  double min_gap = INFINITY;
  for (size_t k = 0; k < n; ++k) {
    if (k == i) continue;
    double g = fabs(s[i] - s[k]);
    if (g < min_gap) min_gap = g;
  }
  if (min_gap <= tol * (s[n - 1] - s[0])) {
    char buf[160];
    snprintf(buf, sizeof buf, "eigenvalue %zu is degenerate (gap %g)", i,
             min_gap);
    set_err(err, ORC_E_DEGENERATE, (int64_t)i, min_gap, buf);
    return ORC_E_DEGENERATE;
  }
  if (gap_out) *gap_out = min_gap;
  return ORC_OK;
}

/* log_domain_product, identity.cpp:98-122 */
int orc_log_domain_product(const double* num, const double* den, size_t len,
                           double* out, orc_err* err) {
  double log_sum = 0.0;
  int negative = 0, zero = 0;
  for (size_t k = 0; k < len; ++k) {
    double x = num[k];
    if (x == 0.0) {
      zero = 1;
    } else {
      log_sum += log(fabs(x));
      if (x < 0.0) negative = !negative;
    }
  }
  for (size_t k = 0; k < len; ++k) {
    double x = den[k];
    if (x == 0.0) {
      set_err(err, ORC_E_DEGENERATE, -1, 0.0, "zero denominator factor");
      return ORC_E_DEGENERATE;
    }
    log_sum -= log(fabs(x));
    if (x < 0.0) negative = !negative;
  }
  if (zero) {
    *out = 0.0;
    return ORC_OK;
  }
  if (negative) {
    set_err(err, ORC_E_INTERNAL, -1, 0.0,
            "reconstructed squared magnitude is negative; eigenvalue "
            "ordering is inconsistent");
    return ORC_E_INTERNAL;
  }
  *out = exp(log_sum);
  return ORC_OK;
}

/* evaluate(), identity.cpp:185-238, with make_sorted_pairing (:74-83),
 * prepare_batches (:85-96) and the batch product/combine (:204-225). */
static int evaluate_ws(const double* lambda, const double* mu, size_t n,
                       size_t i, size_t batch, double tol, int log_domain,
                       double* num, double* den, double* ratios, double* raw,
                       double* value, int* method, orc_err* err) {
  int st = checked_min_gap(lambda, n, i, tol, NULL, err);
  if (st) return st;
  const double lam = lambda[i];
  size_t t = 0;
  for (size_t k = 0; k + 1 < n; ++k) num[k] = lam - mu[k];
  for (size_t k = 0; k < n; ++k)
    if (k != i) den[t++] = lam - lambda[k];
  qsort(num, n - 1, sizeof(double), cmp_double);
  qsort(den, n - 1, sizeof(double), cmp_double);
  double r;
  int meth;
  if (log_domain) {
    st = orc_log_domain_product(num, den, n - 1, &r, err);
    if (st) return st;
    meth = 3;
  } else {
    const size_t total = n - 1;
    size_t nb = 0;
    for (size_t b = 0; b < total; b += batch) {
      size_t e = b + batch < total ? b + batch : total;
      double nm = 1.0, dn = 1.0;
      for (size_t k = b; k < e; ++k) {
        nm *= num[k];
        dn *= den[k];
      }
      ratios[nb++] = nm / dn;
    }
    r = 1.0;
    for (size_t b = 0; b < nb; ++b) r *= ratios[b];
    meth = 1;
    if (!isfinite(r)) {
      st = orc_log_domain_product(num, den, n - 1, &r, err);
      if (st) return st;
      meth = 3;
    }
  }
  *raw = r;
  *value = r < 0.0 ? 0.0 : (1.0 < r ? 1.0 : r); /* std::clamp */
  if (method) *method = meth;
  return ORC_OK;
}

int orc_evaluate(const double* lambda, const double* mu, size_t n, size_t i,
                 size_t batch, double tol, int log_domain, double* raw,
                 double* value, int* method, orc_err* err) {
  if (batch < 1) {
    set_err(err, ORC_E_CONFIG, -1, 0.0, "batch size must be >= 1");
    return ORC_E_CONFIG;
  }
  double* ws = (double*)malloc(3 * n * sizeof(double));
  int st = evaluate_ws(lambda, mu, n, i, batch, tol, log_domain, ws, ws + n,
                       ws + 2 * n, raw, value, method, err);
  free(ws);
  return st;
}

/* ---- a tiny pthread fan-out standing in for ThreadPool::parallel_for ---- */
typedef struct {
  pthread_mutex_t mu;
  size_t next, count;
  int status;
  orc_err err;
  void (*body)(void* ctx, size_t idx, double* ws, orc_err* err, int* st);
  void* ctx;
  size_t ws_doubles;
} orc_pool;

static void* pool_worker(void* p) {
  orc_pool* pool = (orc_pool*)p;
  double* ws = (double*)malloc(pool->ws_doubles * sizeof(double));
  for (;;) {
    size_t idx;
    pthread_mutex_lock(&pool->mu);
    if (pool->next >= pool->count || pool->status) {
      pthread_mutex_unlock(&pool->mu);
      break;
    }
    idx = pool->next++;
    pthread_mutex_unlock(&pool->mu);
    orc_err e;
    int st = 0;
    pool->body(pool->ctx, idx, ws, &e, &st);
    if (st) {
      pthread_mutex_lock(&pool->mu);
      if (!pool->status) {
        pool->status = st;
        pool->err = e;
      }
      pthread_mutex_unlock(&pool->mu);
    }
  }
  free(ws);
  return NULL;
}

static int pool_run(size_t count, int threads, size_t ws_doubles,
                    void (*body)(void*, size_t, double*, orc_err*, int*),
                    void* ctx, orc_err* err) {
  orc_pool pool;
  pthread_mutex_init(&pool.mu, NULL);
  pool.next = 0;
  pool.count = count;
  pool.status = 0;
  pool.body = body;
  pool.ctx = ctx;
  pool.ws_doubles = ws_doubles;
  if (threads < 1) threads = 1;
  if ((size_t)threads > count) threads = (int)(count ? count : 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int t = 1; t < threads; ++t)
    pthread_create(&th[t], NULL, pool_worker, &pool);
  pool_worker(&pool);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&pool.mu);
  if (pool.status && err) *err = pool.err;
  return pool.status;
}

typedef struct {
  const double* lambda;
  const double* mu; /* row-major, row r = minor j0 + r */
  size_t n, j0, batch;
  double tol;
  int log_domain;
  double* out; /* row r = j0 + r */
} id_ctx;

static void id_body(void* p, size_t r, double* ws, orc_err* err, int* st) {
  id_ctx* c = (id_ctx*)p;
  const size_t n = c->n;
  for (size_t i = 0; i < n; ++i) {
    double raw, val;
    *st = evaluate_ws(c->lambda, c->mu + r * (n - 1), n, i, c->batch, c->tol,
                      c->log_domain, ws, ws + n, ws + 2 * n, &raw, &val, NULL,
                      err);
    if (*st) return;
    c->out[r * n + i] = val;
  }
}

int orc_identity_rows(const double* lambda, const double* mu, size_t n,
                      size_t j0, size_t j1, size_t batch, double tol,
                      int log_domain, int threads, double* out,
                      orc_err* err) {
  if (batch < 1) {
    set_err(err, ORC_E_CONFIG, -1, 0.0, "batch size must be >= 1");
    return ORC_E_CONFIG;
  }
  id_ctx c = {lambda, mu, n, j0, batch, tol, log_domain, out};
  return pool_run(j1 - j0, threads, 3 * n, id_body, &c, err);
}

typedef struct {
  const double* a;
  size_t n;
  const size_t* js;
  double* mu;
} minor_ctx;

static void minor_body(void* p, size_t r, double* ws, orc_err* err, int* st) {
  minor_ctx* c = (minor_ctx*)p;
  const size_t n = c->n, m = n - 1;
  (void)ws;
  double* mm = (double*)malloc(m * m * sizeof(double));
  orc_minor(c->a, n, c->js ? c->js[r] : r, mm);
  *st = orc_eigenvalues(mm, m, c->mu + r * m, err);
  free(mm);
}

int orc_minor_spectra(const double* a, size_t n, const size_t* js,
                      size_t count, int threads, double* mu, orc_err* err) {
  minor_ctx c = {a, n, js, mu};
  return pool_run(count, threads, 1, minor_body, &c, err);
}

/* all_magnitudes, identity.cpp:294-316 */
int orc_all_magnitudes(const double* a, size_t n, size_t batch, double tol,
                       int log_domain, int threads, double* out,
                       double* lambda_out, double* mu_out, orc_err* err) {
  if (n < 2) {
    set_err(err, ORC_E_MATRIX_TOO_SMALL, -1, 0.0,
            "component magnitudes need n >= 2");
    return ORC_E_MATRIX_TOO_SMALL;
  }
  if (batch < 1) {
    set_err(err, ORC_E_CONFIG, -1, 0.0, "batch size must be >= 1");
    return ORC_E_CONFIG;
  }
  double* lambda = (double*)malloc(n * sizeof(double));
  double* mu = (double*)malloc(n * (n - 1) * sizeof(double));
  int st = orc_eigenvalues(a, n, lambda, err);
  if (!st) st = orc_check_fully_nondegenerate(lambda, n, tol, err);
  if (!st) st = orc_minor_spectra(a, n, NULL, n, threads, mu, err);
  if (!st)
    st = orc_identity_rows(lambda, mu, n, 0, n, batch, tol, log_domain,
                           threads, out, err);
  if (!st && lambda_out) memcpy(lambda_out, lambda, n * sizeof(double));
  if (!st && mu_out) memcpy(mu_out, mu, n * (n - 1) * sizeof(double));
  free(lambda);
  free(mu);
  return st;
}

/* ---- sign recovery ------------------------------------------------------
 * Restates recover_signs (src/signs.cpp:48-120) and its Gaussian elimination
 * with partial pivoting (solve_linear, :13-44): the largest magnitude (first
 * on ties) anchors the vector, the other n-1 row equations of
 * (A - lambda I) v = 0 are solved for the remaining components, only their
 * signs are kept, the first component above sign_tol is made positive and the
 * residual ||(A - lambda I) v|| is checked against 1e-6 ||A||_F. */
static int orc_gauss_solve(double* w, double* rhs, size_t m) {
  for (size_t col = 0; col < m; ++col) {
    size_t piv = col;
    for (size_t r = col + 1; r < m; ++r)
      if (fabs(w[r * m + col]) > fabs(w[piv * m + col])) piv = r;
    if (w[piv * m + col] == 0.0) return 0;
    if (piv != col) {
      for (size_t c = 0; c < m; ++c) {
        const double t = w[col * m + c];
        w[col * m + c] = w[piv * m + c];
        w[piv * m + c] = t;
      }
      const double t = rhs[col];
      rhs[col] = rhs[piv];
      rhs[piv] = t;
    }
    const double inv = 1.0 / w[col * m + col];
    for (size_t r = col + 1; r < m; ++r) {
      const double f = w[r * m + col] * inv;
      if (f == 0.0) continue;
      for (size_t c = col; c < m; ++c) w[r * m + c] -= f * w[col * m + c];
      rhs[r] -= f * rhs[col];
    }
  }
  for (size_t col = m; col-- > 0;) {
    double acc = rhs[col];
    for (size_t c = col + 1; c < m; ++c) acc -= w[col * m + c] * rhs[c];
    rhs[col] = acc / w[col * m + col];
  }
  return 1;
}

int orc_recover_signs(const double* a, size_t n, size_t i, const double* mags,
                      size_t nmags, double lambda_i, double sign_tol,
                      double* out, orc_err* err) {
  (void)i; /* unused by the reference too (signs.cpp:54) */
  if (nmags != n) {
    set_err(err, ORC_E_DIMENSION, -1, 0.0, "magnitude vector length does not match n");
    return ORC_E_DIMENSION;
  }
  for (size_t j = 0; j < n; ++j) {
    const double c = mags[j] < 0.0 ? 0.0 : (mags[j] > 1.0 ? 1.0 : mags[j]);
    out[j] = sqrt(c);
  }
  if (n > 1) {
    size_t anchor = 0;
    for (size_t j = 1; j < n; ++j)
      if (mags[j] > mags[anchor]) anchor = j;
    const size_t m = n - 1;
    double* w = (double*)malloc(sizeof(double) * m * m);
    double* rhs = (double*)malloc(sizeof(double) * m);
    if (!w || !rhs) {
      free(w);
      free(rhs);
      set_err(err, ORC_E_ALLOC, -1, 0.0, "allocation failed");
      return ORC_E_ALLOC;
    }
    size_t rr = 0;
    for (size_t r = 0; r < n; ++r) {
      if (r == anchor) continue;
      size_t cc = 0;
      for (size_t c = 0; c < n; ++c) {
        if (c == anchor) continue;
        w[rr * m + cc] = a[r * n + c] - (r == c ? lambda_i : 0.0);
        ++cc;
      }
      rhs[rr] = -(a[r * n + anchor] - (r == anchor ? lambda_i : 0.0)) * out[anchor];
      ++rr;
    }
    const int ok = orc_gauss_solve(w, rhs, m);
    if (!ok) {
      free(w);
      free(rhs);
      set_err(err, ORC_E_SIGN_RECOVERY, -1, 0.0, "row equations are singular at the anchor");
      return ORC_E_SIGN_RECOVERY;
    }
    rr = 0;
    for (size_t r = 0; r < n; ++r) {
      if (r == anchor) continue;
      if (mags[r] > sign_tol && rhs[rr] < 0.0) out[r] = -out[r];
      ++rr;
    }
    free(w);
    free(rhs);
  }
  for (size_t j = 0; j < n; ++j)
    if (mags[j] > sign_tol) {
      if (out[j] < 0.0)
        for (size_t t = 0; t < n; ++t) out[t] = -out[t];
      break;
    }
  double res2 = 0.0, fro2 = 0.0;
  for (size_t r = 0; r < n; ++r) {
    double row = 0.0;
    for (size_t c = 0; c < n; ++c) row += (a[r * n + c] - (r == c ? lambda_i : 0.0)) * out[c];
    res2 += row * row;
  }
  for (size_t t = 0; t < n * n; ++t) fro2 += a[t] * a[t];
  const double res = sqrt(res2), bound = 1e-6 * sqrt(fro2);
  if (res > bound) {
    char buf[256];
    snprintf(buf, sizeof buf, "sign recovery residual %f exceeds %f", res, bound);
    set_err(err, ORC_E_SIGN_RECOVERY, -1, 0.0, buf);
    return ORC_E_SIGN_RECOVERY;
  }
  return ORC_OK;
}

/* C3 input: A = Q diag(lambda) Q^T with Q from the Householder
 * QR of an n x n matrix G of SeededDraws::gaussian draws (matrix_io.cpp:53-65,
 * row-major), each column of Q sign-fixed by diag(R); lambda_k = -1 + 2k/(n-1);
 * then build(kSymmetrize) (matrix.cpp:30-35).  Plain loops in a fixed order
 * (no BLAS), so the product library's eigenid_c3_matrix reproduces it bit for
 * bit and the reference arm can build the same bytes without the product. */
void orc_c3_matrix(uint64_t seed, size_t n, double* out) {
  double* g = (double*)malloc(sizeof(double) * n * n);
  double* w = (double*)malloc(sizeof(double) * n * n);   /* W = G^T: row k = column k */
  double* p = (double*)malloc(sizeof(double) * n * n);   /* P = Q^T */
  double* beta = (double*)malloc(sizeof(double) * n);
  double* rdiag = (double*)malloc(sizeof(double) * n);
  orc_gaussian_stream(seed, n * n, g);
  for (size_t r = 0; r < n; ++r)
    for (size_t c = 0; c < n; ++c) w[c * n + r] = g[r * n + c];
  for (size_t k = 0; k < n; ++k) {
    double* x = w + k * n;
    double ss = 0.0;
    for (size_t t = k; t < n; ++t) ss += x[t] * x[t];
    const double nrm = sqrt(ss);
    const double alpha = x[k] >= 0.0 ? -nrm : nrm;
    rdiag[k] = alpha;
    if (nrm == 0.0) { beta[k] = 0.0; continue; }
    x[k] -= alpha;                       /* v = x - alpha e_k, stored in place */
    double vv = 0.0;
    for (size_t t = k; t < n; ++t) vv += x[t] * x[t];
    beta[k] = 2.0 / vv;
    for (size_t j = k + 1; j < n; ++j) {
      double* y = w + j * n;
      double d = 0.0;
      for (size_t t = k; t < n; ++t) d += x[t] * y[t];
      const double s = beta[k] * d;
      for (size_t t = k; t < n; ++t) y[t] -= s * x[t];
    }
  }
  /* Q = H_0 ... H_{n-1}: backward accumulation on P = Q^T from the right */
  for (size_t t = 0; t < n * n; ++t) p[t] = 0.0;
  for (size_t t = 0; t < n; ++t) p[t * n + t] = 1.0;
  for (size_t k = n; k-- > 0;) {
    const double* v = w + k * n;
    if (beta[k] == 0.0) continue;
    for (size_t r = k; r < n; ++r) {
      double* pr = p + r * n;
      double d = 0.0;
      for (size_t t = k; t < n; ++t) d += pr[t] * v[t];
      const double s = beta[k] * d;
      for (size_t t = k; t < n; ++t) pr[t] -= s * v[t];
    }
  }
  /* column k of Q (row k of P) times sign(R_kk) */
  for (size_t k = 0; k < n; ++k)
    if (rdiag[k] < 0.0)
      for (size_t t = 0; t < n; ++t) p[k * n + t] = -p[k * n + t];
  /* A = sum_k lambda_k q_k q_k^T, rank-1 updates in k order */
  for (size_t t = 0; t < n * n; ++t) out[t] = 0.0;
  for (size_t k = 0; k < n; ++k) {
    const double lk = -1.0 + 2.0 * (double)k / (double)(n - 1);
    const double* q = p + k * n;
    for (size_t r = 0; r < n; ++r) {
      const double s = lk * q[r];
      double* ar = out + r * n;
      for (size_t c = 0; c < n; ++c) ar[c] += s * q[c];
    }
  }
  for (size_t r = 0; r < n; ++r)
    for (size_t c = r + 1; c < n; ++c) {
      const double m = 0.5 * (out[r * n + c] + out[c * n + r]);
      out[r * n + c] = m;
      out[c * n + r] = m;
    }
  free(g); free(w); free(p); free(beta); free(rdiag);
}
