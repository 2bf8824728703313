// mp_l1strip.cuh -- K3b dispatch and the tall-column fallback: per-column
// l1-ball projection at per-column radii, the l_{1,1} apply pass
// (proj/src/fiber_kernels.cpp:56-65, which gathers each column and calls
// project_l1_fast_inplace, proj/src/vector_balls.cpp:150-161).
//
// Routes (launch_l1strip): register strips (mp_l1reg.cuh) for n <= 8192/P;
// the shared-memory quad strip (mp_l1quad.cuh) for longer 16-byte-aligned
// columns that fit shared memory; the column kernels (mp_l1cols.cuh) for
// unaligned m; and, for columns beyond shared memory, k_l1strip below: a CTA
// owns 32 adjacent columns (lane l of every warp = column l, 128-byte rows),
// warps split the rows, and every Michelot pass re-reads the strip from
// global memory (L2).  Its final threshold follows the reference definition:
// cutoff = smallest active |y|, k = #{|y| >= cutoff},
// tau = (sum_{|y|>=cutoff} |y| - u) / k with the sum in double-double (the
// reference uses long double, vector_balls.cpp:32-40), and the soft
// threshold |y| - tau is formed in f64.
#pragma once

#include <algorithm>
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

constexpr int kStripCols = 32;
constexpr int kStripThreads = 256;
constexpr int kStripWarps = kStripThreads / 32;

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

// Per-column reduction over the CTA: `mine` is this thread's partial for
// column `lane`; returns the CTA total for that column in every thread.
// Fixed order => deterministic.  `red` is double-buffered by `par`.
template <class Op>
__device__ __forceinline__ StripRed strip_reduce(StripRed mine, StripRed (*red)[kStripWarps * 32], int& par, Op op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  red[par][warp * 32 + lane] = mine;
  __syncthreads();
  StripRed t = red[par][lane];
#pragma unroll
  for (int w = 1; w < kStripWarps; ++w) t = op(t, red[par][w * 32 + lane]);
  par ^= 1;
  return t;
}

template <typename T>
__global__ void __launch_bounds__(kStripThreads)
    k_l1strip(const T* __restrict__ y, T* __restrict__ x, int64_t n, int64_t m, const double* __restrict__ v,
              const double* __restrict__ u, double* __restrict__ tau_out, const mp_info* __restrict__ info) {
  tl_begin(3);
  if (info->status != MP_OK) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * kStripCols + lane;
  const bool colok = col < m;
  const double uj = colok ? u[col] : 0.0;
  const double vj = colok ? v[col] : 0.0;
  // 0: outside m, 1: feasible (untouched), 2: zero budget, 3: project
  const int kind = !colok ? 0 : (vj <= uj ? 1 : (uj == 0.0 ? 2 : 3));
  const bool any_proj = __syncthreads_or(kind == 3);

  if (!any_proj) {
    for (int64_t r = warp; r < n; r += kStripWarps) {
      const int64_t idx = r * m + col;
      if (kind == 1 && x != y) x[idx] = y[idx];
      else if (kind == 2) x[idx] = T(0);
    }
    if (warp == 0 && colok) tau_out[col] = -1.0;
    tl_end(3);
    return;
  }

  __shared__ StripRed red[2][kStripWarps * 32];
  __shared__ int sdone;
  int par = 0;
  auto elem = [&](int64_t r) -> T { return y[r * m + col]; };
  auto add_sc = [](StripRed p, StripRed q) { return StripRed{__dadd_rn(p.a, q.a), 0.0, p.c + q.c}; };

  // Michelot passes with a monotone threshold (the active set only shrinks).
  double t = 0.0;
  long long kprev = -1;
  bool done = (kind != 3);
  for (int iters = 0;; ++iters) {
    StripRed mine{0.0, 0.0, 0};
    if (kind == 3)
      for (int64_t r = warp; r < n; r += kStripWarps) {
        const double a = fabs(static_cast<double>(elem(r)));
        if (a > t) {
          mine.a = __dadd_rn(mine.a, a);
          ++mine.c;
        }
      }
    const StripRed tot = strip_reduce(mine, red, par, add_sc);
    if (!done) {
      if (tot.c == kprev || tot.c == 0) done = true;
      else {
        t = fmax(t, (tot.a - uj) / static_cast<double>(tot.c));
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
    for (int64_t r = warp; r < n; r += kStripWarps) {
      const double a = fabs(static_cast<double>(elem(r)));
      if (a > t) mn.a = fmin(mn.a, a);
    }
  const StripRed cut =
      strip_reduce(mn, red, par, [](StripRed p, StripRed q) { return StripRed{fmin(p.a, q.a), 0.0, 0}; });
  DD ps{0.0, 0.0};
  long long pk = 0;
  if (kind == 3)
    for (int64_t r = warp; r < n; r += kStripWarps) {
      const double a = fabs(static_cast<double>(elem(r)));
      if (a >= cut.a) {
        ps = dd_add(ps, a);
        ++pk;
      }
    }
  const StripRed S = strip_reduce(StripRed{ps.hi, ps.lo, pk}, red, par, [](StripRed p, StripRed q) {
    const DD r = dd_add(DD{p.a, p.b}, DD{q.a, q.b});
    return StripRed{r.hi, r.lo, p.c + q.c};
  });
  double tau = -1.0;
  if (kind == 3 && S.c > 0) {
    const DD d = two_sum(S.a, -uj);
    tau = __dadd_rn(d.hi, __dadd_rn(d.lo, S.b)) / static_cast<double>(S.c);
  }
  if (warp == 0 && colok) tau_out[col] = tau;

  // Apply; lane = column => 128-byte coalesced rows.
  for (int64_t r = warp; r < n; r += kStripWarps) {
    const int64_t idx = r * m + col;
    if (kind == 1) {
      if (x != y) x[idx] = elem(r);
    } else if (kind == 2) {
      x[idx] = T(0);
    } else if (kind == 3) {
      const T e = elem(r);
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

// Route switches for A/B timing.  The product build compiles them to their
// defaults; only a build with -DMP_TUNING_SWITCHES reads the environment.
#ifdef MP_TUNING_SWITCHES
inline const char* mp_tuning_env(const char* name) { return std::getenv(name); }
#else
inline const char* mp_tuning_env(const char*) { return nullptr; }
#endif

// MP_L1_KERNEL=quad forces the shared-memory path (A/B timing aid).
inline bool l1reg_disabled() {
  static const bool d = [] {
    const char* e = mp_tuning_env("MP_L1_KERNEL");
    return e && std::strcmp(e, "quad") == 0;
  }();
  return d;
}

// MP_L1REG_P=1|2|4|8 caps the register path's pieces per row (tuning aid).
inline int l1reg_prefer_p() {
  static const int p = [] {
    const char* e = mp_tuning_env("MP_L1REG_P");
    return e ? std::atoi(e) : 0;
  }();
  return p;
}

// TMA maps for the hybrid strips' shared-memory half (f32, 8-column x
// 256-row boxes over the (n, m) row-major matrix).  The encoder comes from
// the driver through the runtime (no libcuda link).  MP_L1_TMA=0 keeps the
// cp.async / LSU path (A/B aid).
inline bool l1_tma_enabled() {
  static const bool on = [] {
    const char* e = mp_tuning_env("MP_L1_TMA");
    return !(e && *e == '0');
  }();
  return on;
}
template <typename T>
inline bool encode_strip_map(CUtensorMap* tm, const void* base, int64_t n, int64_t m) {
  typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Enc enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<Enc>(fn);
  }();
  if (!enc) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(m) * sizeof(T)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(32 / sizeof(T)), 256};  // 32-byte strip rows
  const cuuint32_t es[2] = {1, 1};
  return enc(tm, sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
             const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Grid-stride CTAs, as many as are co-resident (kRegThreads / NT per SM).
template <typename T, int P, int NT, int RS = 0, bool TMA = false>
cudaError_t launch_reg(const T* y, T* x, int64_t n, int64_t m, const double* v, const double* u,
                       const L1StripWs& ws, const mp_info* info, const L1Derive& dv, cudaStream_t s,
                       const TmaMaps* maps = nullptr) {
  constexpr int W = 16 / sizeof(T) * P;
  const int64_t nstrips = m / W;
  const size_t smem = static_cast<size_t>(NT) * RS * 16;
  if constexpr (RS > 0) {
    static std::atomic<uint64_t> done{0};
    const cudaError_t a = mpi::once_per_device(done, [smem] {
      const cudaError_t a1 = cudaFuncSetAttribute(k_l1reg<T, P, true, true, NT, RS, TMA>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (a1 != cudaSuccess) return a1;
      return cudaFuncSetAttribute(k_l1reg<T, P, false, true, NT, RS, TMA>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    if (a != cudaSuccess) return a;
  }
  TmaMaps tm{};
  if (maps) tm = *maps;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NT);
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(nstrips, static_cast<int64_t>(mpi::sm_count()) *
                                                                           (kRegThreads / NT))));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (dv.params)
    return cudaLaunchKernelEx(&cfg, k_l1reg<T, P, true, true, NT, RS, TMA>, y, x, static_cast<int>(n), m, v, u,
                              ws.tau, info, dv.params, dv.u_out, nstrips, tm);
  return cudaLaunchKernelEx(&cfg, k_l1reg<T, P, false, true, NT, RS, TMA>, y, x, static_cast<int>(n), m, v, u,
                            ws.tau, info, dv.params, dv.u_out, nstrips, tm);
}

template <typename T, int P>
cudaError_t launch_reg_nt(const RegGeom& g, const T* y, T* x, int64_t n, int64_t m, const double* v, const double* u,
                          const L1StripWs& ws, const mp_info* info, const L1Derive& dv, cudaStream_t s) {
  if constexpr (P == 2) {
    if (g.RS > 0) {
      if (g.NT == 128) return launch_reg<T, 2, 128, kRegHybridRS>(y, x, n, m, v, u, ws, info, dv, s);
      if (g.NT == 256) {
        {
          // TMA for the shared-memory pieces (16-byte-aligned rows, n <= 4096)
          TmaMaps maps{};
          if (l1_tma_enabled() && reinterpret_cast<uintptr_t>(y) % 16 == 0 &&
              reinterpret_cast<uintptr_t>(x) % 16 == 0 && encode_strip_map<T>(&maps.y, y, n, m) &&
              encode_strip_map<T>(&maps.x, x, n, m))
            return launch_reg<T, 2, 256, tma_rs(256), true>(y, x, n, m, v, u, ws, info, dv, s, &maps);
        }
        return launch_reg<T, 2, 256, kRegHybridRS>(y, x, n, m, v, u, ws, info, dv, s);
      }
      if constexpr (sizeof(T) == 8) {  // f64, 4097..8192 rows: 512-thread TMA strips
        TmaMaps maps{};
        if (l1_tma_enabled() && reinterpret_cast<uintptr_t>(y) % 16 == 0 &&
            reinterpret_cast<uintptr_t>(x) % 16 == 0 && encode_strip_map<T>(&maps.y, y, n, m) &&
            encode_strip_map<T>(&maps.x, x, n, m))
          return launch_reg<T, 2, kRegThreads, tma_rs(kRegThreads), true>(y, x, n, m, v, u, ws, info, dv, s, &maps);
      }
      return launch_reg<T, 2, kRegThreads, kRegHybridRS>(y, x, n, m, v, u, ws, info, dv, s);
    }
  }
  if (g.NT == 128) return launch_reg<T, P, 128>(y, x, n, m, v, u, ws, info, dv, s);
  if (g.NT == 256) return launch_reg<T, P, 256>(y, x, n, m, v, u, ws, info, dv, s);
  return launch_reg<T, P, kRegThreads>(y, x, n, m, v, u, ws, info, dv, s);
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
    const RegGeom g = l1reg_geometry<T>(n, m, l1reg_prefer_p());
    // columns of 513..1024 rows: 64-thread TMA strips of 1024 rows, eight
    // CTAs per SM.  1000x16384: f32 51.7 -> 40.4 us, f64 122.9 -> 68.4 us;
    // 600 rows: f32 45.1 -> 38.1, f64 114.7 -> 60.2 us.
    if (l1_tma_enabled() && n > 512 && n <= 1024 && m % (2 * 16 / sizeof(T)) == 0 &&
        reinterpret_cast<uintptr_t>(y) % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0) {
      TmaMaps maps{};
      if (encode_strip_map<T>(&maps.y, y, n, m) && encode_strip_map<T>(&maps.x, x, n, m))
        return launch_reg<T, 2, 64, 24, true>(y, x, n, m, v, u, ws, info, dv, s, &maps);
    }
    // columns of 1025..2048 rows (f64: 513..2048): 128-thread TMA strips of
    // 2048 rows, four CTAs per SM.  2000x16384: f32 105.6 -> 76.9 us, f64
    // 295 -> 146 us; f64 1000x16384 138 -> 122 us; f32 at 1000 rows loses
    // to the register strips (67 vs 52 us: half the strip is padding).
    if (l1_tma_enabled() && n <= 2048 && n > (sizeof(T) == 4 ? 1024 : 512) && m % (2 * 16 / sizeof(T)) == 0 &&
        reinterpret_cast<uintptr_t>(y) % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0) {
      TmaMaps maps{};
      if (encode_strip_map<T>(&maps.y, y, n, m) && encode_strip_map<T>(&maps.x, x, n, m))
        return launch_reg<T, 2, 128, tma_rs(128), true>(y, x, n, m, v, u, ws, info, dv, s, &maps);
    }
    switch (g.P) {
      case 8: return launch_reg_nt<T, 8>(g, y, x, n, m, v, u, ws, info, dv, s);
      case 4: return launch_reg_nt<T, 4>(g, y, x, n, m, v, u, ws, info, dv, s);
      case 2: return launch_reg_nt<T, 2>(g, y, x, n, m, v, u, ws, info, dv, s);
      case 1: return launch_reg_nt<T, 1>(g, y, x, n, m, v, u, ws, info, dv, s);
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
  (void)flags;
  k_l1strip<T><<<static_cast<unsigned>(nstrips), kStripThreads, 0, s>>>(y, x, n, m, v, u, ws.tau, info);
  return cudaGetLastError();
}

}  // namespace mpk
