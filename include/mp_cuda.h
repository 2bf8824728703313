/*
 * mp_cuda.h -- C-ABI of the B200-native bi-/multi-level projection path.
 *
 * This is the drop-in boundary between host code and the sm_100a kernels.
 * Plain pointers and sizes only (no torch / no C++ types).  Each entry point
 * replaces one reference interface (paths relative to /root/reference/):
 *
 *   mp_bilevel_project        <- multiproj::bilevel_project
 *                                (proj/include/multiproj/bilevel.hpp:19-20,
 *                                 proj/src/bilevel.cpp:10-32) and
 *                                bilevel_project_l1inf (bilevel.hpp:23-24)
 *   mp_multilevel_project     <- multiproj::multilevel_project_iter /
 *                                multilevel_project / trilevel_project_l1infinf
 *                                (proj/include/multiproj/multilevel.hpp:35-46,
 *                                 proj/src/multilevel.cpp:77-132)
 *   mp_project_ball           <- multiproj::project_ball / project_l1_fast /
 *                                project_l2 / project_linf
 *                                (proj/include/multiproj/vector_balls.hpp:12-32)
 *   mp_aggregate              <- multiproj::aggregate_leading_axis
 *                                (proj/include/multiproj/tensor.hpp:86-87,
 *                                 proj/src/tensor.cpp:107-138) -- the kernel
 *                                seam detail::aggregate_block
 *                                (proj/include/multiproj/detail/fiber_kernels.hpp:13-14)
 *   mp_*_host                 <- the same calls with HOST buffers in and out
 *                                (the reference's by-value DenseTensor API);
 *                                host<->device copies happen inside the call.
 *
 * Conventions (device entry points):
 *   - The caller owns all device memory, including the workspace sized by the
 *     matching mp_*_workspace_size().  No allocation and no host sync happen
 *     inside the call, so it is CUDA-graph capturable.  `stream` is a
 *     cudaStream_t (NULL = legacy default stream).
 *   - x may alias y (in-place projection).
 *   - Layout is the reference's: row-major, fibers are leading-axis slices,
 *     i.e. for an (n, m) matrix the groups are the m columns, strided by m
 *     (proj/include/multiproj/tensor.hpp:19-22,46-51).
 *   - Argument validation mirrors the reference exception taxonomy
 *     (proj/include/multiproj/errors.hpp:10-31) as mp_status codes returned
 *     synchronously.  Data-dependent failures found on device (non-finite
 *     input, ValueError at proj/src/tensor.cpp:40-41) are written to
 *     mp_info.status and the output is left unwritten; the *_host calls
 *     return them as their status.
 *   - mp_norm order mirrors `enum class Norm { L1, L2, Inf }`
 *     (proj/include/multiproj/tensor.hpp:15).
 */
#ifndef MP_CUDA_H
#define MP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

typedef enum mp_status {
  MP_OK = 0,
  MP_ERR_VALUE = 1,     /* ValueError: eta < 0 / non-finite, non-finite data */
  MP_ERR_SHAPE = 2,     /* ShapeError: wrong order, zero dims, depth != order */
  MP_ERR_CONFIG = 3,    /* ConfigError: empty spec, bad norm/dtype code */
  MP_ERR_CUDA = 4,      /* CUDA runtime error (see mp_last_error) */
  MP_ERR_WORKSPACE = 5, /* workspace too small / NULL required pointer */
  MP_ERR_UNSUPPORTED = 6
} mp_status;

typedef enum mp_norm { MP_NORM_L1 = 0, MP_NORM_L2 = 1, MP_NORM_INF = 2 } mp_norm;

typedef enum mp_dtype { MP_F32 = 0, MP_F64 = 1 } mp_dtype;

/* Flags. */
/* Read zero-budget columns so zeroed entries keep copysign(0, y) bytes
 * (-0.0 for negative y), exactly as proj/src/fiber_kernels.cpp:47.  Default
 * off: zero-budget column groups are written as +0.0 without being read
 * (value-equal; saves the read of every zeroed column). */
#define MP_FLAG_EXACT_ZERO_SIGN 1u

/* Device-written summary of one projection (lives in device memory). */
typedef struct mp_info {
  double tau;           /* outer l1 threshold (p = 1); -1 if the outer step was the identity */
  int64_t zero_columns; /* #{j : u_j == 0 || v_j == 0}  (proj/src/bilevel.cpp:29-30) */
  int64_t active;       /* k = #{j : v_j >= cutoff} of the outer l1 step (-1 if identity) */
  int64_t survivors;    /* #{j : u_j > 0}: columns the apply pass reads */
  int32_t status;       /* mp_status of device-side checks (MP_ERR_VALUE on non-finite) */
  int32_t iterations;   /* threshold-search passes of the outer l1 step */
} mp_info;

/* ---------------------------------------------------------------- device */

size_t mp_bilevel_workspace_size(mp_dtype dtype, int64_t n, int64_t m, mp_norm p, mp_norm q);

/* Bi-level l_{p,q} projection of the (n, m) row-major matrix y into x.
 * budgets (m doubles, device, nullable): the outer-projected radii u.
 * norms (m doubles, device, nullable): the column q-norms v.
 * info (device, nullable). */
mp_status mp_bilevel_project(const void* y, void* x, mp_dtype dtype, int64_t n, int64_t m,
                             mp_norm p, mp_norm q, double eta, double* budgets, double* norms,
                             mp_info* info, unsigned flags, void* workspace,
                             size_t workspace_bytes, void* stream);

size_t mp_multilevel_workspace_size(mp_dtype dtype, const int64_t* shape, int order,
                                    const mp_norm* levels, int depth);

/* Multi-level projection (iterative form).  levels[0..depth) innermost
 * first; depth must equal order.  budget_chain (device, nullable) receives
 * the budget chain without its last entry (== x), deepest first:
 * prod(shape[order-1:]), prod(shape[order-2:]), ..., prod(shape[1:]) doubles
 * (proj/include/multiproj/multilevel.hpp:28-31). */
mp_status mp_multilevel_project(const void* t, void* x, mp_dtype dtype, const int64_t* shape,
                                int order, const mp_norm* levels, int depth, double eta,
                                double* budget_chain, mp_info* info, unsigned flags,
                                void* workspace, size_t workspace_bytes, void* stream);

size_t mp_project_ball_workspace_size(mp_dtype dtype, int64_t len, mp_norm q);

/* Vector-ball projection of len entries (signed) onto the q-ball. */
mp_status mp_project_ball(const void* y, void* x, mp_dtype dtype, int64_t len, mp_norm q,
                          double radius, mp_info* info, void* workspace, size_t workspace_bytes,
                          void* stream);

size_t mp_aggregate_workspace_size(mp_dtype dtype, int64_t n, int64_t m, mp_norm q);

/* out[f] = ||fiber f||_q of the (n, m) row-major view (f64 out, device). */
mp_status mp_aggregate(const void* t, double* out, mp_dtype dtype, int64_t n, int64_t m,
                       mp_norm q, void* workspace, size_t workspace_bytes, void* stream);

/* Config-5 workload harness (BASELINE.json config 5, the per-step
 * projection of proj/src/train.cpp:191-199): x += sigma * N(0, 1), with the
 * deviates from Philox4x32-10 keyed by (seed, iteration) on the element
 * index -- stateless, graph-replayable, reproducible. */
mp_status mp_perturb_gaussian(void* x, mp_dtype dtype, int64_t count, double sigma, uint64_t seed,
                              uint64_t iteration, void* stream);

size_t mp_project_fibers_workspace_size(mp_dtype dtype, int64_t n, int64_t m, mp_norm q);

/* The apply seam alone (detail::project_block,
 * proj/include/multiproj/detail/fiber_kernels.hpp:16-20,
 * proj/src/fiber_kernels.cpp:37-67): every fiber (column) j of the (n, m)
 * view is projected onto the q-ball of radius budgets[j], given its q-norm
 * norms[j] (both device, f64).  Used by the column-sharded multi-GPU
 * projection, where the budgets come from a gathered norm vector. */
mp_status mp_project_fibers(const void* y, void* x, mp_dtype dtype, int64_t n, int64_t m, mp_norm q,
                            const double* norms, const double* budgets, unsigned flags, void* workspace,
                            size_t workspace_bytes, void* stream);

/* Exact Euclidean projection onto the l_{1,inf} ball (euclid_project_l1inf,
 * proj/include/multiproj/euclidean.hpp:27-30, proj/src/euclidean.cpp:82-170;
 * the "euclid" tag of proj/src/dispatch.cpp).  x (n, m) = Y clipped per
 * column at the distance-minimising budgets; budgets (device f64, nullable)
 * = ColumnBudgetSolution.budgets; info->tau = theta (the common residual
 * mass), info->iterations = Newton steps, info->zero_columns = #{u_j == 0}.
 * Columns are sorted in shared memory: workspace_size returns 0 (and the
 * call MP_ERR_UNSUPPORTED) beyond n = 32768 (f32) / 16384 (f64). */
size_t mp_euclid_workspace_size(mp_dtype dtype, int64_t n, int64_t m);

mp_status mp_euclid_project(const void* y, void* x, mp_dtype dtype, int64_t n, int64_t m, double eta,
                            double* budgets, mp_info* info, unsigned flags, void* workspace,
                            size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ host */

/* Opaque per-thread-safe execution context: device, stream, cached device
 * buffers.  ctx = NULL in the *_host calls uses a thread-local default. */
typedef struct mp_context mp_context;

mp_context* mp_context_create(int device);
void mp_context_destroy(mp_context* ctx);

/* Synchronous host-buffer bi-level projection: y/x are host pointers
 * (pinned or pageable; x may alias y).  budgets (m doubles), zero_columns
 * and tau are host outputs (nullable). */
mp_status mp_bilevel_project_host(mp_context* ctx, const void* y, void* x, mp_dtype dtype,
                                  int64_t n, int64_t m, mp_norm p, mp_norm q, double eta,
                                  double* budgets, int64_t* zero_columns, double* tau,
                                  unsigned flags);

/* Radius sweep with host buffers (the reference's run_radius_sweep shape,
 * proj/src/bench.cpp:93-106): y is uploaded once and projected at each of
 * count radii; xs[k] (host) receives the k-th projection.  Downloads overlap
 * the next projection (two device output buffers, a copy stream).  budgets
 * (count * m doubles) and zero_columns (count) are nullable host outputs.
 * On a device-side failure the xs contents are unspecified. */
mp_status mp_bilevel_sweep_host(mp_context* ctx, const void* y, void* const* xs, mp_dtype dtype, int64_t n,
                                int64_t m, mp_norm p, mp_norm q, const double* etas, int count,
                                double* budgets, int64_t* zero_columns, unsigned flags);

/* The same sweep, enqueued and returned from at once (a serving pipeline over
 * a stream of inputs, e.g. bench_one's repeated calls, proj/src/bench.cpp:54-91):
 * the upload of y runs on its own stream, so it overlaps the downloads of the
 * previous sweep on this context; up to two sweeps are in flight.  y, xs,
 * budgets and zero_columns must stay valid until mp_context_wait(ctx, *ticket)
 * returns, which reports the sweep's status.  mp_bilevel_sweep_host is this
 * call followed by the wait. */
mp_status mp_bilevel_sweep_host_async(mp_context* ctx, const void* y, void* const* xs, mp_dtype dtype,
                                      int64_t n, int64_t m, mp_norm p, mp_norm q, const double* etas,
                                      int count, double* budgets, int64_t* zero_columns, unsigned flags,
                                      uint64_t* ticket);

mp_status mp_context_wait(mp_context* ctx, uint64_t ticket);

mp_status mp_multilevel_project_host(mp_context* ctx, const void* t, void* x, mp_dtype dtype,
                                     const int64_t* shape, int order, const mp_norm* levels,
                                     int depth, double eta, double* budget_chain,
                                     unsigned flags);

mp_status mp_project_ball_host(mp_context* ctx, const void* y, void* x, mp_dtype dtype,
                               int64_t len, mp_norm q, double radius);

mp_status mp_aggregate_host(mp_context* ctx, const void* t, double* out, mp_dtype dtype,
                            int64_t n, int64_t m, mp_norm q);

/* euclid_project_l1inf on host buffers (replaces the EuclidResult call,
 * proj/src/euclidean.cpp:82): budgets[m] and *theta (both nullable) receive
 * ColumnBudgetSolution. */
mp_status mp_euclid_project_host(mp_context* ctx, const void* y, void* x, mp_dtype dtype, int64_t n,
                                 int64_t m, double eta, double* budgets, double* theta);

/* ----------------------------------------------------------- diagnostics */

/* Per-phase device timing (bench / profiling aid, not in the reference):
 * while set, every mp_bilevel_project / mp_multilevel_project call on this
 * host thread records
 * events[0..3] (cudaEvent_t) on its stream before the norm pass, after the
 * norm pass, after the outer projection and after the apply pass.  Recorded
 * events are stream-ordered, so they work inside CUDA-graph capture.  Pass
 * NULL / 0 to disable. */
void mp_profile_events(void* const* events, int count);

/* Device-side timeline (profiling aid): while set (device pointer to 8
 * uint64, caller-initialised to {UINT64_MAX, 0} pairs), kernels fold their
 * %globaltimer start (min) / end (max) into [2k], [2k+1] for k = 0 norm pass,
 * 1 norm finalize, 2 outer projection, 3 apply pass.  NULL disables. */
void mp_profile_timeline(unsigned long long* device_buf);

/* Thread-local description of the last non-OK status. */
const char* mp_last_error(void);

/* ABI version (major * 10000 + minor * 100 + patch). */
int mp_version(void);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* MP_CUDA_H */
