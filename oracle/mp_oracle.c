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

/* ---------------------------------------------------------------------------
 * Exact Euclidean l_{1,inf} projection (proj/src/euclidean.cpp:82-170).
 *
 * Column j, magnitudes sorted descending a_1 >= ... >= a_n, long double
 * prefix P_k = a_1 + ... + a_k; theta-space breakpoints t_k = P_k - k a_k
 * (rounded to double, non-decreasing in k) and the column's total mass P_n
 * (:28-49).  For theta below P_n the column's budget is
 * u_j(theta) = (P_k - theta) / k with k = #{t_k <= theta} (at least 1,
 * :19-26,51-61).  The optimal theta solves sum_j u_j(theta) = eta: the
 * candidates are 0, every t_k and every P_n, sorted and deduplicated
 * (:103-112); a bisection finds the first candidate whose budget sum is
 * <= eta (:114-123) and the bracketing linear segment is solved exactly from
 * the segment indices at its midpoint (:125-141).  Budgets are clamped at 0
 * and X clips every column at its budget (:143-156).
 */
typedef struct {
  double* mags;       /* descending */
  long double* pref;  /* pref[k] = a_1 + ... + a_k, k = 0..n */
  double* brk;        /* t_k, k = 1..n at brk[k-1] */
  double total;
} orc_col;

static int desc_dbl(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x < y) - (x > y);
}
static int asc_dbl(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* upper_bound over the non-decreasing breakpoints: #{t_k <= theta} */
static int64_t col_segment(const orc_col* c, int64_t n, double theta) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (c->brk[mid] <= theta) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static double col_budget(const orc_col* c, double theta, int64_t k) {
  return (double)((c->pref[k] - (long double)theta) / (long double)k);
}

static double budget_sum(const orc_col* cols, int64_t m, int64_t n, double theta) {
  long double s = 0.0L;
  for (int64_t j = 0; j < m; ++j) {
    if (theta >= cols[j].total) continue;
    int64_t k = col_segment(&cols[j], n, theta);
    if (k == 0) k = 1;
    s += col_budget(&cols[j], theta, k);
  }
  return (double)s;
}

int orc_euclid_l1inf(const double* y, int64_t n, int64_t m, double eta, double* x, double* budgets,
                     double* theta_out) {
  if (!radius_ok(eta)) return ORC_VALUE;
  if (!all_finite(y, n * m)) return ORC_VALUE;
  orc_col* cols = (orc_col*)calloc((size_t)(m > 0 ? m : 1), sizeof(orc_col));
  double l1inf = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    orc_col* c = &cols[j];
    c->mags = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    c->pref = (long double*)malloc(sizeof(long double) * (size_t)(n + 1));
    c->brk = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) c->mags[i] = fabs(y[i * m + j]);
    qsort(c->mags, (size_t)n, sizeof(double), desc_dbl);
    c->pref[0] = 0.0L;
    for (int64_t k = 1; k <= n; ++k) {
      c->pref[k] = c->pref[k - 1] + c->mags[k - 1];
      c->brk[k - 1] = (double)(c->pref[k] - (long double)k * c->mags[k - 1]);
    }
    c->total = (double)c->pref[n];
    l1inf += n > 0 ? c->mags[0] : 0.0;
  }
  int rc = ORC_OK;
  double theta = 0.0;
  if (l1inf <= eta) {
    for (int64_t j = 0; j < m; ++j) budgets[j] = cols[j].mags[0];
    memcpy(x, y, sizeof(double) * (size_t)(n * m));
    theta = 0.0;
    goto done;
  }
  if (eta == 0.0) {
    for (int64_t j = 0; j < m; ++j) {
      budgets[j] = 0.0;
      if (cols[j].total > theta) theta = cols[j].total;
    }
    for (int64_t e = 0; e < n * m; ++e) x[e] = 0.0;
    goto done;
  }
  {
    const int64_t nb_max = m * (n + 1) + 1;
    double* br = (double*)malloc(sizeof(double) * (size_t)nb_max);
    int64_t nb = 0;
    br[nb++] = 0.0;
    for (int64_t j = 0; j < m; ++j) {
      for (int64_t k = 0; k < n; ++k) br[nb++] = cols[j].brk[k];
      br[nb++] = cols[j].total;
    }
    qsort(br, (size_t)nb, sizeof(double), asc_dbl);
    int64_t u = 0;
    for (int64_t i = 0; i < nb; ++i)
      if (u == 0 || br[i] != br[u - 1]) br[u++] = br[i];
    nb = u;
    int64_t lo = 0, hi = nb - 1;
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (budget_sum(cols, m, n, br[mid]) <= eta) hi = mid;
      else lo = mid;
    }
    if (budget_sum(cols, m, n, br[hi]) == eta) {
      theta = br[hi];
    } else {
      const double probe = 0.5 * (br[lo] + br[hi]);
      long double a = 0.0L, b = 0.0L;
      for (int64_t j = 0; j < m; ++j) {
        if (probe >= cols[j].total) continue;
        int64_t k = col_segment(&cols[j], n, probe);
        if (k == 0) k = 1;
        a += cols[j].pref[k] / (long double)k;
        b += 1.0L / (long double)k;
      }
      theta = (double)((a - (long double)eta) / b);
      if (theta < br[lo]) theta = br[lo];
      if (theta > br[hi]) theta = br[hi];
    }
    free(br);
  }
  for (int64_t j = 0; j < m; ++j) {
    budgets[j] = 0.0;
    if (theta >= cols[j].total) continue;
    int64_t k = col_segment(&cols[j], n, theta);
    if (k == 0) k = 1;
    const double b = col_budget(&cols[j], theta, k);
    budgets[j] = b > 0.0 ? b : 0.0;
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < m; ++j) {
      const double e = y[i * m + j];
      x[i * m + j] = fabs(e) > budgets[j] ? copysign(budgets[j], e) : e;
    }
done:
  if (theta_out) *theta_out = theta;
  for (int64_t j = 0; j < m; ++j) {
    free(cols[j].mags);
    free(cols[j].pref);
    free(cols[j].brk);
  }
  free(cols);
  return rc;
}

/* clip_cost (proj/src/euclidean.cpp:64-80): sum_j sum_i max(|y_ij| - u_j, 0)^2. */
double orc_clip_cost(const double* y, int64_t n, int64_t m, const double* budgets) {
  double cost = 0.0;
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < n; ++i) {
      const double over = fabs(y[i * m + j]) - budgets[j];
      if (over > 0.0) cost += over * over;
    }
  return cost;
}
