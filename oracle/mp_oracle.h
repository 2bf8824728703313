/*
 * mp_oracle.h -- CPU restatement of the reference bi-/multi-level projection
 * path (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product path
 * (paper_2405_02086_b200) never links or calls it.
 *
 * All arithmetic is f64 (long double where the reference uses it), matching
 * /root/reference/proj which is CPU/f64-only.  Norm codes follow the
 * reference enum order `enum class Norm { L1, L2, Inf }`
 * (proj/include/multiproj/tensor.hpp:15).
 */
#ifndef MP_ORACLE_H
#define MP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_L1 = 0, ORC_L2 = 1, ORC_INF = 2 };
/* Error codes mirror the reference exception types
 * (proj/include/multiproj/errors.hpp:10-31). */
enum { ORC_OK = 0, ORC_VALUE = 1, ORC_SHAPE = 2, ORC_CONFIG = 3 };

/* ||v||_q (proj/src/tensor.cpp:78-99).  Returns ORC_VALUE on non-finite. */
int orc_vector_norm(const double* v, int64_t len, int q, double* out);

/* out[f] = ||fiber f||_q over the leading axis of a (n, m) row-major view
 * (proj/src/tensor.cpp:107-138, proj/src/fiber_kernels.cpp:11-35). */
void orc_aggregate(const double* t, int64_t n, int64_t m, int q, double* out);

/* In-place l1-ball projection, the reference fast path
 * (proj/src/vector_balls.cpp:150-161).  tau/k report the threshold and the
 * active count when a projection happened (tau = -1, k = -1 otherwise). */
void orc_project_l1_inplace(double* y, int64_t len, double radius,
                            double* tau, int64_t* k);
/* Sort-based l1 cutoff, the reference's definitional path
 * (proj/src/vector_balls.cpp:52-70,125-140). */
void orc_project_l1_sort_inplace(double* y, int64_t len, double radius,
                                 double* tau, int64_t* k);

/* project_ball (proj/src/vector_balls.cpp:207-214): validates radius and
 * finiteness, then projects y in place onto the q-ball. */
int orc_project_ball(double* y, int64_t len, int q, double radius);

/* detail::project_block over all fibers, in place (proj/src/fiber_kernels.cpp:37-67). */
void orc_project_fibers(double* x, int64_t n, int64_t m, int q, const double* v, const double* budgets);

/* bilevel_project (proj/src/bilevel.cpp:10-32).  x, budgets, v (norms) and
 * zero_columns are outputs; v/tau may be NULL.  tau is the outer l1
 * threshold (-1 when the outer step was the identity / p != 1). */
int orc_bilevel(const double* y, int64_t n, int64_t m, int p, int q,
                double eta, double* x, double* budgets, double* v,
                int64_t* zero_columns, double* tau);

/* multilevel_project_iter (proj/src/multilevel.cpp:93-124).  shape has
 * `order` dims; levels has `order` norm codes, innermost first.  x receives
 * the projected tensor.  If chain is non-NULL it receives the concatenated
 * budget chain without its last entry (== x): deepest budgets first, sizes
 * prod(shape[order-1:]), prod(shape[order-2:]), ..., prod(shape[1:]). */
int orc_multilevel(const double* t, const int64_t* shape, int order,
                   const int* levels, double eta, double* x, double* chain);

/* multilevel_norm (proj/src/multilevel.cpp:134-141). */
int orc_multilevel_norm(const double* t, const int64_t* shape, int order,
                        const int* levels, double* out);

/* structured_sparsity (proj/src/tensor.cpp:152-164): columns of an (n, m)
 * matrix whose max |x| <= tol. */
int64_t orc_structured_sparsity(const double* x, int64_t n, int64_t m,
                                double tol);

/* Exact Euclidean l_{1,inf} projection (proj/src/euclidean.cpp:82-170):
 * x (n, m) row-major, budgets[m], theta.  ORC_VALUE on a bad radius or
 * non-finite data. */
int orc_euclid_l1inf(const double* y, int64_t n, int64_t m, double eta, double* x, double* budgets,
                     double* theta);

/* clip_cost (proj/src/euclidean.cpp:64-80). */
double orc_clip_cost(const double* y, int64_t n, int64_t m, const double* budgets);

#ifdef __cplusplus
}
#endif
#endif
