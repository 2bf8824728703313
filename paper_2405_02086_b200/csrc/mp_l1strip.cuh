// mp_l1strip.cuh -- K3b: per-column l1-ball projection at per-column radii,
// the l_{1,1} apply pass (proj/src/fiber_kernels.cpp:56-65, which gathers
// each column and calls project_l1_fast_inplace, proj/src/vector_balls.cpp:150-161).
//
// B200 design: a thread-block CLUSTER owns a strip of 32 adjacent columns
// (128-byte rows for f32, one L2 line) over all n rows.  Each of the C CTAs
// of the cluster stages its rpc-row slice of the strip in shared memory with
// cp.async, so the strip is read from HBM exactly once however many
// threshold passes a column needs.  Lane l of every warp owns column l; warps
// split the rows.  Per pass, every column's (sum, count) above its current
// threshold is reduced warp-wise -> CTA -> cluster through DSMEM (double
// buffered, one cluster barrier per pass, fixed rank order => identical,
// deterministic totals in every CTA).  Michelot's fixed point converges in a
// handful of passes (6-7 for config 3).  The final
// threshold follows the reference definition: cutoff = smallest active |y|,
// k = #{|y| >= cutoff}, tau = (sum_{|y|>=cutoff} |y| - u) / k with the sum in
// double-double (the reference uses long double, vector_balls.cpp:32-40), and
// the soft threshold |y| - tau is formed in f64.
// Strips whose slice does not fit shared memory (n beyond ~25k rows for f32)
// use the same kernel with STAGED = false: passes re-read the strip from
// global memory (L2), C = 1.
#pragma once

#include <algorithm>
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "mp_cuda.h"
#include "mp_internal.h"
#include "mp_kernels.cuh"
#include "mp_l1cols.cuh"
#include "mp_l1quad.cuh"
#include "mp_l1reg.cuh"

namespace mpk {

namespace cg = cooperative_groups;

constexpr int kStripCols = 32;
constexpr int kStripThreads = 256;
constexpr int kStripWarps = kStripThreads / 32;
constexpr size_t kStripTileMax = 100 * 1024;  // bytes of staged rows per CTA (2 CTAs / SM)

struct L1StripWs {
  double* tau;  // per-column inner threshold (-1 where the column was not projected)
};

inline L1StripWs carve_l1strip(mpi::Carve& c, int64_t m) {
  L1StripWs w;
  w.tau = c.take<double>(m);
  return w;
}

struct StripRed {
  double a, b;
  long long c;
};

// Per-column reduction over the cluster.  `mine` is this thread's partial
// for column `lane`; returns the cluster-wide total for that column in every
// thread of every CTA.  op must be associative; order is fixed.
template <class Op>
__device__ __forceinline__ StripRed strip_reduce(StripRed mine, StripRed* wred, StripRed* cred, int& par,
                                                 const cg::cluster_group& cl, unsigned C, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  wred[warp * 32 + lane] = mine;
  __syncthreads();
  if (warp == 0) {
    StripRed t = wred[lane];
#pragma unroll
    for (int w = 1; w < kStripWarps; ++w) t = op(t, wred[w * 32 + lane]);
    cred[par * 32 + lane] = t;
  }
  cl.sync();
  StripRed tot = *cl.map_shared_rank(&cred[par * 32 + lane], 0);
  for (unsigned r = 1; r < C; ++r) tot = op(tot, *cl.map_shared_rank(&cred[par * 32 + lane], r));
  par ^= 1;
  return tot;
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <typename T, bool STAGED>
__global__ void __launch_bounds__(kStripThreads)
    k_l1strip(const T* __restrict__ y, T* __restrict__ x, int64_t n, int64_t m, int64_t rpc,
              const double* __restrict__ v, const double* __restrict__ u, double* __restrict__ tau_out,
              const mp_info* __restrict__ info, unsigned flags) {
  tl_begin(3);
  if (info->status != MP_OK) return;  // uniform across the cluster
  cg::cluster_group cl = cg::this_cluster();
  const unsigned C = cl.num_blocks();
  const unsigned rank = cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t strip = blockIdx.x / C;
  const int64_t cbase = strip * kStripCols;
  const int64_t col = cbase + lane;
  const bool colok = col < m;
  const int64_t r0 = static_cast<int64_t>(rank) * rpc;
  const int64_t r1 = min(n, r0 + rpc);
  const int64_t nr = r1 > r0 ? r1 - r0 : 0;

  const double uj = colok ? u[col] : 0.0;
  const double vj = colok ? v[col] : 0.0;
  // 0: outside m, 1: feasible (untouched), 2: zero budget, 3: project
  const int kind = !colok ? 0 : (vj <= uj ? 1 : (uj == 0.0 ? 2 : 3));
  (void)flags;
  const bool any_proj = __syncthreads_or(kind == 3);  // same strip in every CTA => cluster-uniform

  if (!any_proj) {
    for (int64_t r = r0 + warp; r < r1; r += kStripWarps) {
      const int64_t idx = r * m + col;
      if (kind == 1 && x != y) x[idx] = y[idx];
      else if (kind == 2) x[idx] = T(0);
    }
    if (rank == 0 && warp == 0 && colok) tau_out[col] = -1.0;
    tl_end(3);
    return;
  }

  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);  // [nr][32]
  __shared__ StripRed wred[kStripWarps * 32];
  __shared__ StripRed cred[2 * 32];
  __shared__ double stau[32];
  __shared__ int sdone;
  int par = 0;

  auto elem = [&](int64_t rl) -> T {
    if constexpr (STAGED) return tile[rl * kStripCols + lane];
    else return y[(r0 + rl) * m + col];
  };

  if constexpr (STAGED) {
    const bool full = cbase + kStripCols <= m;
    const uintptr_t al = reinterpret_cast<uintptr_t>(y);
    constexpr int per16 = 16 / sizeof(T);
    if (full && (m % per16) == 0 && (al % 16) == 0) {
      constexpr int chunks = kStripCols / per16;  // 16-byte pieces per row
      for (int64_t i = threadIdx.x; i < nr * chunks; i += kStripThreads) {
        const int64_t rl = i / chunks;
        const int part = static_cast<int>(i % chunks);
        cp_async16(&tile[rl * kStripCols + part * per16], y + (r0 + rl) * m + cbase + part * per16);
      }
    } else {
      for (int64_t rl = warp; rl < nr; rl += kStripWarps)
        if (colok) {
          if constexpr (sizeof(T) == 4) cp_async4(&tile[rl * kStripCols + lane], y + (r0 + rl) * m + col);
          else cp_async8(&tile[rl * kStripCols + lane], y + (r0 + rl) * m + col);
        }
    }
    cp_async_wait_all();
    __syncthreads();
  }

  auto add_sc = [](StripRed p, StripRed q) { return StripRed{__dadd_rn(p.a, q.a), 0.0, p.c + q.c}; };

  // Michelot passes with a monotone threshold (the active set only shrinks).
  double t = 0.0;
  long long kprev = -1;
  bool done = (kind != 3);
  int iters = 0;
  for (;;) {
    StripRed mine{0.0, 0.0, 0};
    if (kind == 3) {
      for (int64_t rl = warp; rl < nr; rl += kStripWarps) {
        const double a = fabs(static_cast<double>(elem(rl)));
        if (a > t) {
          mine.a = __dadd_rn(mine.a, a);
          ++mine.c;
        }
      }
    }
    const StripRed tot = strip_reduce(mine, wred, cred, par, cl, C, add_sc);
    ++iters;
    if (!done) {
      if (tot.c == kprev || tot.c == 0) done = true;
      else {
        const double nt = (tot.a - uj) / static_cast<double>(tot.c);
        t = fmax(t, nt);
        kprev = tot.c;
      }
    }
    if (warp == 0) {
      const bool all = __all_sync(0xffffffffu, done);
      if (lane == 0) sdone = all;
    }
    __syncthreads();
    const bool stop = sdone;
    __syncthreads();
    if (stop || iters > 4 * 1024) break;
  }

  // cutoff = min active |y| (> t); then (sum, count) over |y| >= cutoff.
  StripRed mn{__longlong_as_double(0x7ff0000000000000ll), 0.0, 0};
  if (kind == 3)
    for (int64_t rl = warp; rl < nr; rl += kStripWarps) {
      const double a = fabs(static_cast<double>(elem(rl)));
      if (a > t) mn.a = fmin(mn.a, a);
    }
  const StripRed cut = strip_reduce(mn, wred, cred, par, cl, C,
                                    [](StripRed p, StripRed q) { return StripRed{fmin(p.a, q.a), 0.0, 0}; });
  DD ps{0.0, 0.0};
  long long pk = 0;
  if (kind == 3)
    for (int64_t rl = warp; rl < nr; rl += kStripWarps) {
      const double a = fabs(static_cast<double>(elem(rl)));
      if (a >= cut.a) {
        ps = dd_add(ps, a);
        ++pk;
      }
    }
  const StripRed S = strip_reduce(StripRed{ps.hi, ps.lo, pk}, wred, cred, par, cl, C, [](StripRed p, StripRed q) {
    DD r = dd_add(DD{p.a, p.b}, DD{q.a, q.b});
    return StripRed{r.hi, r.lo, p.c + q.c};
  });
  double tau = -1.0;
  if (kind == 3 && S.c > 0) {
    const DD d = two_sum(S.a, -uj);
    tau = __dadd_rn(d.hi, __dadd_rn(d.lo, S.b)) / static_cast<double>(S.c);
  }
  if (warp == 0) stau[lane] = tau;
  cl.sync();  // no CTA leaves while a peer may still read its DSMEM
  if (rank == 0 && warp == 0 && colok) tau_out[col] = tau;

  // Apply from the staged slice; lane = column => 128-byte coalesced rows.
  for (int64_t rl = warp; rl < nr; rl += kStripWarps) {
    const int64_t idx = (r0 + rl) * m + col;
    if (kind == 1) {
      if (x != y) x[idx] = elem(rl);
    } else if (kind == 2) {
      x[idx] = T(0);
    } else if (kind == 3) {
      const T e = elem(rl);
      const double d = fabs(static_cast<double>(e)) - tau;
      x[idx] = d > 0.0 ? static_cast<T>(copysign(d, static_cast<double>(e))) : T(0);
    }
  }
  tl_end(3);
}

constexpr size_t kColsSmemTarget = 72 * 1024;   // >= 3 CTAs per SM
constexpr size_t kColsSmemMax = 200 * 1024;

template <typename T>
inline int cols_stride(int64_t n) {
  return static_cast<int>(((n + 3) / 4) * 4 + 4);  // 16-byte aligned columns, offset banks
}

constexpr int kColsTW = 2;  // warps per column (occupancy is bounded by shared memory)

template <typename T, int W>
cudaError_t cols_attr() {
  cudaError_t e = cudaFuncSetAttribute(k_l1cols<T, W, kColsTW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kColsSmemMax));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_l1cols<T, W, kColsTW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kColsSmemMax));
}

// K2 outcome handed to the l1 apply when it derives the budgets itself.
struct L1Derive {
  const OuterParams* params = nullptr;  // null: read budgets u[]
  double* u_out = nullptr;
  mp_info* info_w = nullptr;
};

// MP_L1_KERNEL=quad forces the shared-memory path (A/B timing aid).
inline bool l1reg_disabled() {
  static const bool d = [] {
    const char* e = std::getenv("MP_L1_KERNEL");
    return e && std::strcmp(e, "quad") == 0;
  }();
  return d;
}

// MP_L1REG_PERSIST=0: one CTA per strip instead of grid-stride (tuning aid).
inline bool l1reg_persist() {
  static const bool d = [] {
    const char* e = std::getenv("MP_L1REG_PERSIST");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return d;
}

// MP_L1REG_P=1|2|4|8 caps the register path's pieces per row (tuning aid).
inline int l1reg_prefer_p() {
  static const int p = [] {
    const char* e = std::getenv("MP_L1REG_P");
    return e ? std::atoi(e) : 0;
  }();
  return p;
}

template <typename T, int P>
cudaError_t launch_reg(const T* y, T* x, int64_t n, int64_t m, const double* v, const double* u,
                       const L1StripWs& ws, const mp_info* info, const L1Derive& dv, cudaStream_t s) {
  constexpr int W = 16 / sizeof(T) * P;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kRegThreads);
  cfg.gridDim = dim3(static_cast<unsigned>(m / W));
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int64_t nstrips = m / W;
  if (l1reg_persist()) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(nstrips, sms)));
    if (dv.params)
      return cudaLaunchKernelEx(&cfg, k_l1reg<T, P, true, true>, y, x, static_cast<int>(n), m, v, u, ws.tau, info,
                                dv.params, dv.u_out, nstrips);
    return cudaLaunchKernelEx(&cfg, k_l1reg<T, P, false, true>, y, x, static_cast<int>(n), m, v, u, ws.tau, info,
                              dv.params, dv.u_out, nstrips);
  }
  if (dv.params)
    return cudaLaunchKernelEx(&cfg, k_l1reg<T, P, true, false>, y, x, static_cast<int>(n), m, v, u, ws.tau, info,
                              dv.params, dv.u_out, nstrips);
  return cudaLaunchKernelEx(&cfg, k_l1reg<T, P, false, false>, y, x, static_cast<int>(n), m, v, u, ws.tau, info,
                            dv.params, dv.u_out, nstrips);
}

template <typename T>
cudaError_t quad_attr() {
  cudaError_t e = cudaFuncSetAttribute(k_l1quad<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kColsSmemMax));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_l1quad<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kColsSmemMax));
}

inline cudaError_t l1strip_setup() {
  for (cudaError_t e : {quad_attr<float>(), quad_attr<double>(), cols_attr<float, 8>(), cols_attr<float, 4>(), cols_attr<float, 2>(), cols_attr<float, 1>(),
                        cols_attr<double, 8>(), cols_attr<double, 4>(), cols_attr<double, 2>(),
                        cols_attr<double, 1>()})
    if (e != cudaSuccess) return e;
  return cudaSuccess;
}

template <typename T, int W>
cudaError_t launch_cols(const T* y, T* x, int64_t n, int64_t m, const double* v, const double* u,
                        const L1StripWs& ws, const mp_info* info, const L1Derive& dv, cudaStream_t s) {
  const int stride = cols_stride<T>(n);
  const size_t smem = static_cast<size_t>(W) * stride * sizeof(T);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>((m + W - 1) / W));
  cfg.blockDim = dim3(32 * W * kColsTW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (dv.params)
    return cudaLaunchKernelEx(&cfg, k_l1cols<T, W, kColsTW, true>, y, x, static_cast<int>(n), m, stride, v, u, ws.tau, info,
                              dv.params, dv.u_out, dv.info_w);
  return cudaLaunchKernelEx(&cfg, k_l1cols<T, W, kColsTW, false>, y, x, static_cast<int>(n), m, stride, v, u, ws.tau, info,
                            dv.params, dv.u_out, dv.info_w);
}

// Per-column l1 projection: warp-per-column staged kernel when a column
// fits shared memory (n up to ~50k f32 rows), else the unstaged strip
// kernel (passes re-read the strip from L2).
template <typename T>
inline bool l1_staged_ok(int64_t n) {
  return static_cast<size_t>(cols_stride<T>(n)) * sizeof(T) <= kColsSmemMax;
}

// With dv.params set, u must still point at a budgets array the fallback
// path can read; the staged kernels derive the budgets themselves.
template <typename T>
cudaError_t launch_l1strip(const T* y, T* x, int64_t n, int64_t m, const double* v, const double* u,
                           const L1StripWs& ws, const mp_info* info, unsigned flags, cudaStream_t s,
                           const L1Derive& dv = L1Derive()) {
  if (l1_quad_ok<T>(y, x, m) && !l1reg_disabled()) {
    switch (l1reg_pieces<T>(n, m, l1reg_prefer_p())) {
      case 8: return launch_reg<T, 8>(y, x, n, m, v, u, ws, info, dv, s);
      case 4: return launch_reg<T, 4>(y, x, n, m, v, u, ws, info, dv, s);
      case 2: return launch_reg<T, 2>(y, x, n, m, v, u, ws, info, dv, s);
      case 1: return launch_reg<T, 1>(y, x, n, m, v, u, ws, info, dv, s);
      default: break;
    }
  }
  if (l1_quad_ok<T>(y, x, m) && static_cast<size_t>(n) * 16 <= kColsSmemMax) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(m / (16 / sizeof(T))));
    cfg.blockDim = dim3(kQuadThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(n) * 16;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (dv.params)
      return cudaLaunchKernelEx(&cfg, k_l1quad<T, true>, y, x, static_cast<int>(n), m, v, u, ws.tau, info, dv.params,
                                dv.u_out);
    return cudaLaunchKernelEx(&cfg, k_l1quad<T, false>, y, x, static_cast<int>(n), m, v, u, ws.tau, info, dv.params,
                              dv.u_out);
  }
  const size_t col_bytes = static_cast<size_t>(cols_stride<T>(n)) * sizeof(T);
  if (8 * col_bytes <= kColsSmemTarget) return launch_cols<T, 8>(y, x, n, m, v, u, ws, info, dv, s);
  if (4 * col_bytes <= kColsSmemTarget) return launch_cols<T, 4>(y, x, n, m, v, u, ws, info, dv, s);
  if (2 * col_bytes <= kColsSmemTarget) return launch_cols<T, 2>(y, x, n, m, v, u, ws, info, dv, s);
  if (col_bytes <= kColsSmemMax) return launch_cols<T, 1>(y, x, n, m, v, u, ws, info, dv, s);
  const int64_t nstrips = (m + kStripCols - 1) / kStripCols;
  k_l1strip<T, false><<<static_cast<unsigned>(nstrips), kStripThreads, 0, s>>>(y, x, n, m, n, v, u, ws.tau, info,
                                                                              flags);
  return cudaGetLastError();
}

}  // namespace mpk
