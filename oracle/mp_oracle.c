/*
 * mp_oracle.c -- plain-C restatement of the reference projection algorithms.
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA path.  Never linked by
 * the product library.  Each function cites the reference file:line whose
 * behaviour it restates (paths relative to /root/reference/).  It is pinned
 * against the compiled reference (oracle/_ref, built by oracle/Makefile from
 * the sources where they lie) and against the golden fixtures in
 * tests/golden/ (tests/test_oracle.py).
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction; the reference is built
 * for baseline x86-64, where double math is SSE2 and long double is x87).
 */
#include "mp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int radius_ok(double r) { return r >= 0.0 && isfinite(r); }

static int all_finite(const double* y, int64_t len) {
  for (int64_t i = 0; i < len; ++i)
    if (!isfinite(y[i])) return 0;
  return 1;
}

/* Sequential |y| sum, proj/src/vector_balls.cpp:23-27. */
static double abs_sum(const double* y, int64_t len) {
  double s = 0.0;
  for (int64_t i = 0; i < len; ++i) s += fabs(y[i]);
  return s;
}

int orc_vector_norm(const double* v, int64_t len, int q, double* out) {
  /* proj/src/tensor.cpp:78-99 */
  if (!all_finite(v, len)) return ORC_VALUE;
  double s = 0.0;
  for (int64_t i = 0; i < len; ++i) {
    double a = fabs(v[i]);
    if (q == ORC_L1) s += a;
    else if (q == ORC_L2) s += v[i] * v[i];
    else s = (s < a) ? a : s;
  }
  *out = (q == ORC_L2) ? sqrt(s) : s;
  return ORC_OK;
}

void orc_aggregate(const double* t, int64_t n, int64_t m, int q, double* out) {
  /* Row sweep, ascending row index per accumulator:
   * proj/src/tensor.cpp:118-136 == proj/src/fiber_kernels.cpp:16-34. */
  memset(out, 0, (size_t)m * sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    const double* row = t + i * m;
    for (int64_t f = 0; f < m; ++f) {
      double a = fabs(row[f]);
      if (q == ORC_L1) out[f] += a;
      else if (q == ORC_L2) out[f] += row[f] * row[f];
      else if (out[f] < a) out[f] = a;
    }
  }
  if (q == ORC_L2)
    for (int64_t f = 0; f < m; ++f) out[f] = sqrt(out[f]);
}

/* tau = (sum_{|y| >= cutoff} |y| - radius) / k in long double, index order:
 * proj/src/vector_balls.cpp:32-40. */
static double tau_from_cutoff(const double* y, int64_t len, double cutoff,
                              int64_t k, double radius) {
  long double acc = 0.0L;
  for (int64_t i = 0; i < len; ++i) {
    double a = fabs(y[i]);
    if (a >= cutoff) acc += a;
  }
  return (double)((acc - radius) / (long double)k);
}

/* proj/src/vector_balls.cpp:42-48: +0.0 below the threshold. */
static void shrink(double* y, int64_t len, double tau) {
  for (int64_t i = 0; i < len; ++i) {
    double d = fabs(y[i]) - tau;
    y[i] = d > 0.0 ? copysign(d, y[i]) : 0.0;
  }
}

static uint64_t xorshift_step(uint64_t* s) {
  uint64_t x = *s;
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  *s = x;
  return x;
}

static void swap_d(double* a, double* b) {
  double t = *a;
  *a = *b;
  *b = t;
}

/* Duchi et al. randomized-pivot search for the active set of the l1
 * projection (expected linear time), with the reference's fixed xorshift
 * pivot stream and front-partitioning so every pivot value -- and hence
 * every long-double decision -- matches proj/src/vector_balls.cpp:74-121. */
static void pivot_search(double* w, int64_t len, double radius,
                         double* cutoff, int64_t* k) {
  uint64_t state = 0x9e3779b97f4a7c15ULL;
  int64_t lo = 0, hi = len;
  long double kept_sum = 0.0L;
  int64_t kept = 0;
  double c = 0.0;
  while (lo < hi) {
    double piv = w[lo + (int64_t)(xorshift_step(&state) % (uint64_t)(hi - lo))];
    int64_t split = lo;
    long double upper_sum = 0.0L;
    for (int64_t i = lo; i < hi; ++i) {
      if (w[i] >= piv) {
        swap_d(&w[i], &w[split]);
        upper_sum += w[split];
        ++split;
      }
    }
    int64_t upper = split - lo;
    long double excess =
        (kept_sum + upper_sum) - (long double)(kept + upper) * piv;
    if (excess < radius) {
      /* every entry >= piv is active; continue below the pivot */
      kept_sum += upper_sum;
      kept += upper;
      c = piv;
      lo = split;
    } else {
      /* threshold is >= piv: drop the entries equal to piv */
      int64_t dst = lo;
      for (int64_t i = lo; i < split; ++i)
        if (w[i] > piv) swap_d(&w[i], &w[dst++]);
      hi = dst;
    }
  }
  *cutoff = c;
  *k = kept;
}

static int desc_cmp(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x < y) - (x > y);
}

/* Definitional sort path: largest k with z_(k) > (P_k - r)/k on descending
 * magnitudes, proj/src/vector_balls.cpp:52-70. */
static void sort_search(double* w, int64_t len, double radius, double* cutoff,
                        int64_t* k) {
  qsort(w, (size_t)len, sizeof(double), desc_cmp);
  long double prefix = 0.0L;
  *cutoff = w[0];
  *k = 1;
  for (int64_t i = 0; i < len; ++i) {
    prefix += w[i];
    double cand = (double)((prefix - radius) / (long double)(i + 1));
    if (!(w[i] > cand)) break;
    *cutoff = w[i];
    *k = i + 1;
  }
}

static void project_l1_common(double* y, int64_t len, double radius,
                              double* tau, int64_t* k, int use_sort) {
  /* proj/src/vector_balls.cpp:150-161 (fast) / :125-140 (sort) */
  if (tau) *tau = -1.0;
  if (k) *k = -1;
  if (len == 0 || abs_sum(y, len) <= radius) return;
  if (radius == 0.0) {
    for (int64_t i = 0; i < len; ++i) y[i] = 0.0;
    if (tau) *tau = 0.0;
    if (k) *k = 0;
    return;
  }
  double* mags = (double*)malloc((size_t)len * sizeof(double));
  for (int64_t i = 0; i < len; ++i) mags[i] = fabs(y[i]);
  double cutoff;
  int64_t kk;
  if (use_sort) sort_search(mags, len, radius, &cutoff, &kk);
  else pivot_search(mags, len, radius, &cutoff, &kk);
  free(mags);
  double t = tau_from_cutoff(y, len, cutoff, kk, radius);
  shrink(y, len, t);
  if (tau) *tau = t;
  if (k) *k = kk;
}

void orc_project_l1_inplace(double* y, int64_t len, double radius, double* tau,
                            int64_t* k) {
  project_l1_common(y, len, radius, tau, k, 0);
}

void orc_project_l1_sort_inplace(double* y, int64_t len, double radius,
                                 double* tau, int64_t* k) {
  project_l1_common(y, len, radius, tau, k, 1);
}

/* proj/src/vector_balls.cpp:171-177 */
static void project_l2_inplace(double* y, int64_t len, double radius) {
  double s = 0.0;
  for (int64_t i = 0; i < len; ++i) s += y[i] * y[i];
  double norm = sqrt(s);
  if (norm <= radius || norm == 0.0) return;
  double scale = radius / norm;
  for (int64_t i = 0; i < len; ++i) y[i] *= scale;
}

/* proj/src/vector_balls.cpp:187-191 */
static void project_linf_inplace(double* y, int64_t len, double radius) {
  for (int64_t i = 0; i < len; ++i)
    if (fabs(y[i]) > radius) y[i] = copysign(radius, y[i]);
}

static void project_ball_inplace(double* y, int64_t len, int q, double r,
                                 double* tau) {
  if (q == ORC_L1) orc_project_l1_inplace(y, len, r, tau, NULL);
  else if (q == ORC_L2) project_l2_inplace(y, len, r);
  else project_linf_inplace(y, len, r);
}

int orc_project_ball(double* y, int64_t len, int q, double radius) {
  /* proj/src/vector_balls.cpp:207-214 */
  if (!radius_ok(radius)) return ORC_VALUE;
  if (!all_finite(y, len)) return ORC_VALUE;
  project_ball_inplace(y, len, q, radius, NULL);
  return ORC_OK;
}

/* Per-fiber projection at per-fiber budgets, in place on x viewed (n, m):
 * proj/src/fiber_kernels.cpp:37-67. */
static void project_fibers(double* x, int64_t n, int64_t m, int q,
                           const double* v, const double* budgets) {
  if (q == ORC_INF) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t f = 0; f < m; ++f) {
        double* e = &x[i * m + f];
        if (fabs(*e) > budgets[f]) *e = copysign(budgets[f], *e);
      }
  } else if (q == ORC_L2) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t f = 0; f < m; ++f)
        if (v[f] > budgets[f]) x[i * m + f] *= budgets[f] / v[f];
  } else {
    double* col = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
    for (int64_t f = 0; f < m; ++f) {
      if (v[f] <= budgets[f]) continue;
      for (int64_t i = 0; i < n; ++i) col[i] = x[i * m + f];
      orc_project_l1_inplace(col, n, budgets[f], NULL, NULL);
      for (int64_t i = 0; i < n; ++i) x[i * m + f] = col[i];
    }
    free(col);
  }
}

void orc_project_fibers(double* x, int64_t n, int64_t m, int q, const double* v, const double* budgets) {
  project_fibers(x, n, m, q, v, budgets);
}

int orc_bilevel(const double* y, int64_t n, int64_t m, int p, int q,
                double eta, double* x, double* budgets, double* v,
                int64_t* zero_columns, double* tau) {
  /* proj/src/bilevel.cpp:10-32 */
  if (!radius_ok(eta)) return ORC_VALUE;
  if (!all_finite(y, n * m)) return ORC_VALUE; /* tensor.cpp:40-41 */
  double* norms = v ? v : (double*)malloc((size_t)m * sizeof(double));
  orc_aggregate(y, n, m, q, norms);
  int rc = ORC_OK;
  if (!all_finite(norms, m)) { /* vector_balls.cpp:210 */
    rc = ORC_VALUE;
    goto done;
  }
  memcpy(budgets, norms, (size_t)m * sizeof(double));
  if (tau) *tau = -1.0;
  project_ball_inplace(budgets, m, p, eta, p == ORC_L1 ? tau : NULL);
  memcpy(x, y, (size_t)(n * m) * sizeof(double)); /* bilevel.cpp:24 */
  project_fibers(x, n, m, q, norms, budgets);
  int64_t z = 0;
  for (int64_t f = 0; f < m; ++f)
    if (budgets[f] == 0.0 || norms[f] == 0.0) ++z; /* bilevel.cpp:29-30 */
  *zero_columns = z;
done:
  if (!v) free(norms);
  return rc;
}

static int64_t prod_from(const int64_t* shape, int order, int from) {
  int64_t p = 1;
  for (int i = from; i < order; ++i) p *= shape[i];
  return p;
}

int orc_multilevel(const double* t, const int64_t* shape, int order,
                   const int* levels, double eta, double* x, double* chain) {
  /* proj/src/multilevel.cpp:93-124 (iterative form; bit-identical to the
   * recursive form :77-91 per proj/tests/test_multilevel.cpp:44-67). */
  if (order < 1) return ORC_CONFIG;
  if (!radius_ok(eta)) return ORC_VALUE;
  int64_t total = prod_from(shape, order, 0);
  if (total <= 0) return ORC_SHAPE;
  if (!all_finite(t, total)) return ORC_VALUE;
  if (order == 1) { /* :80-82 */
    memcpy(x, t, (size_t)total * sizeof(double));
    return orc_project_ball(x, total, levels[0], eta);
  }
  /* agg[i] = level-i aggregate (shape shape[i:]), i = 1..order-1 */
  double** agg = (double**)calloc((size_t)order, sizeof(double*));
  agg[0] = (double*)t;
  for (int i = 1; i < order; ++i) {
    int64_t mi = prod_from(shape, order, i);
    agg[i] = (double*)malloc((size_t)mi * sizeof(double));
    orc_aggregate(agg[i - 1], shape[i - 1], mi, levels[i - 1], agg[i]);
  }
  int rc = ORC_OK;
  int64_t mdeep = shape[order - 1];
  double* prev = (double*)malloc((size_t)mdeep * sizeof(double));
  memcpy(prev, agg[order - 1], (size_t)mdeep * sizeof(double));
  int64_t off = 0;
  rc = orc_project_ball(prev, mdeep, levels[order - 1], eta);
  if (rc != ORC_OK) goto out;
  if (chain) memcpy(chain, prev, (size_t)mdeep * sizeof(double));
  off = mdeep;
  for (int i = order - 2; i >= 0; --i) {
    int64_t mi = prod_from(shape, order, i);
    double* u = (i == 0) ? x : (double*)malloc((size_t)mi * sizeof(double));
    memcpy(u, agg[i], (size_t)mi * sizeof(double)); /* :115 copy */
    project_fibers(u, shape[i], mi / shape[i], levels[i], agg[i + 1], prev);
    if (chain && i > 0) {
      memcpy(chain + off, u, (size_t)mi * sizeof(double));
      off += mi;
    }
    free(prev);
    prev = (i == 0) ? NULL : u;
  }
out:
  free(prev);
  for (int i = 1; i < order; ++i) free(agg[i]);
  free(agg);
  return rc;
}

int orc_multilevel_norm(const double* t, const int64_t* shape, int order,
                        const int* levels, double* out) {
  /* proj/src/multilevel.cpp:134-141 */
  if (order < 1) return ORC_SHAPE;
  int64_t total = prod_from(shape, order, 0);
  double* cur = (double*)malloc((size_t)total * sizeof(double));
  memcpy(cur, t, (size_t)total * sizeof(double));
  for (int i = 0; i + 1 < order; ++i) {
    int64_t mi = prod_from(shape, order, i + 1);
    double* nxt = (double*)malloc((size_t)mi * sizeof(double));
    orc_aggregate(cur, shape[i], mi, levels[i], nxt);
    free(cur);
    cur = nxt;
  }
  int rc = orc_vector_norm(cur, shape[order - 1], levels[order - 1], out);
  free(cur);
  return rc;
}

int64_t orc_structured_sparsity(const double* x, int64_t n, int64_t m,
                                double tol) {
  /* proj/src/tensor.cpp:152-164 */
  int64_t count = 0;
  for (int64_t f = 0; f < m; ++f) {
    double mx = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double a = fabs(x[i * m + f]);
      mx = (mx < a) ? a : mx;
    }
    if (mx <= tol) ++count;
  }
  return count;
}
