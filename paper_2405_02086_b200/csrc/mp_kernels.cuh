// mp_kernels.cuh -- sm_100a kernels of the bi-/multi-level projection path.
//
// The three passes of proj/src/bilevel.cpp:10-32, re-designed for B200:
//   K1 k_colnorm       column q-norms (proj/src/fiber_kernels.cpp:11-35) as one
//                      coalesced HBM sweep: each thread owns VEC adjacent
//                      columns (128-bit loads) over a row block, U loads in
//                      flight; l_inf merges by atomicMax on |y| bit patterns
//                      (exact, order-free), l1/l2 write f64 row-block partials
//                      reduced in fixed order by k_colnorm_finalize
//                      (deterministic, run-to-run bit-reproducible).
//   K2 k_outer         the outer projection of the norm vector
//                      (proj/src/vector_balls.cpp:150-191,207-214) entirely on
//                      device: one CTA, vector in shared memory, f64 Michelot
//                      fixed point for the l1 threshold, final tau from a
//                      double-double sum over {v >= cutoff} (the reference sums
//                      in long double, vector_balls.cpp:32-40).
//   K3 k_apply         fused clamp / scale (proj/src/fiber_kernels.cpp:37-55),
//                      streaming loads/stores, zero-budget column groups
//                      written without being read, row blocks swept in reverse
//                      so the L2-resident tail of K1 is re-used.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mp_cuda.h"

namespace mpk {

constexpr int kL1 = 0, kL2 = 1, kInf = 2;
constexpr int kThreads = 256;  // K1 / K3 CTA size
constexpr int kOuterThreads = 1024;

// ------------------------------------------------------------ pack helpers
template <typename T, int VEC> struct PackT;
template <> struct PackT<float, 4> { using type = float4; };
template <> struct PackT<float, 2> { using type = float2; };
template <> struct PackT<float, 1> { using type = float; };
template <> struct PackT<double, 2> { using type = double2; };
template <> struct PackT<double, 1> { using type = double; };

template <typename T> struct BitsT;
template <> struct BitsT<float> { using type = unsigned int; };
template <> struct BitsT<double> { using type = unsigned long long; };

__device__ __forceinline__ unsigned int abs_bits(float v) {
  return __float_as_uint(v) & 0x7fffffffu;
}
__device__ __forceinline__ unsigned long long abs_bits(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
}

// Read-only path; K1 keeps lines in L2 (default policy) so K3 can reuse them.
template <typename T, int VEC>
__device__ __forceinline__ void load_keep(const T* p, T (&o)[VEC]) {
  using V = typename PackT<T, VEC>::type;
  V v = __ldg(reinterpret_cast<const V*>(p));
  memcpy(o, &v, sizeof(V));
}
// Last use of the data: evict-first.
template <typename T, int VEC>
__device__ __forceinline__ void load_last(const T* p, T (&o)[VEC]) {
  using V = typename PackT<T, VEC>::type;
  V v = __ldcs(reinterpret_cast<const V*>(p));
  memcpy(o, &v, sizeof(V));
}
template <typename T, int VEC>
__device__ __forceinline__ void store_stream(T* p, const T (&o)[VEC]) {
  using V = typename PackT<T, VEC>::type;
  V v;
  memcpy(&v, o, sizeof(V));
  __stcs(reinterpret_cast<V*>(p), v);
}

// ------------------------------------------------------------------- K1
// grid = (column tiles, row blocks); thread owns columns [c0, c0+VEC) over
// rows [r0, r1).  out: BitsT<T>[m] (l_inf, pre-zeroed) or double[R][m].
template <typename T, int VEC, int Q, int U>
__global__ void __launch_bounds__(kThreads)
    k_colnorm(const T* __restrict__ y, int64_t n, int64_t m, int64_t rpb, void* __restrict__ out) {
  const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * VEC;
  if (c0 >= m) return;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rpb;
  const int64_t r1 = min(n, r0 + rpb);
  const T* p = y + r0 * m + c0;
  int64_t r = r0;
  if constexpr (Q == kInf) {
    using B = typename BitsT<T>::type;
    B acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0;
    for (; r + U <= r1; r += U, p += U * m) {
      T e[U][VEC];
#pragma unroll
      for (int u = 0; u < U; ++u) load_keep<T, VEC>(p + u * m, e[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = max(acc[j], abs_bits(e[u][j]));
    }
    for (; r < r1; ++r, p += m) {
      T e[VEC];
      load_keep<T, VEC>(p, e);
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] = max(acc[j], abs_bits(e[j]));
    }
    B* vb = static_cast<B*>(out) + c0;
#pragma unroll
    for (int j = 0; j < VEC; ++j) atomicMax(vb + j, acc[j]);
  } else {
    double acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.0;
    for (; r + U <= r1; r += U, p += U * m) {
      T e[U][VEC];
#pragma unroll
      for (int u = 0; u < U; ++u) load_keep<T, VEC>(p + u * m, e[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const double d = static_cast<double>(e[u][j]);
          acc[j] = (Q == kL1) ? __dadd_rn(acc[j], fabs(d)) : __dadd_rn(acc[j], __dmul_rn(d, d));
        }
    }
    for (; r < r1; ++r, p += m) {
      T e[VEC];
      load_keep<T, VEC>(p, e);
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const double d = static_cast<double>(e[j]);
        acc[j] = (Q == kL1) ? __dadd_rn(acc[j], fabs(d)) : __dadd_rn(acc[j], __dmul_rn(d, d));
      }
    }
    double* part = static_cast<double*>(out) + static_cast<int64_t>(blockIdx.y) * m + c0;
#pragma unroll
    for (int j = 0; j < VEC; ++j) part[j] = acc[j];
  }
}

// Fixed-order reduction of the row-block partials (l1 / l2), or conversion
// of l_inf bit patterns to f64 (kind 0 = float bits, 1 = double bits).
template <int Q>
__global__ void k_colnorm_finalize(const void* __restrict__ in, int64_t R, int64_t m, int bits_kind,
                                   double* __restrict__ v) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m) return;
  if constexpr (Q == kInf) {
    if (bits_kind == 0)
      v[c] = static_cast<double>(__uint_as_float(static_cast<const unsigned int*>(in)[c]));
    else
      v[c] = __longlong_as_double(static_cast<const long long*>(in)[c]);
  } else {
    const double* part = static_cast<const double*>(in);
    double s = 0.0;
    for (int64_t r = 0; r < R; ++r) s = __dadd_rn(s, part[r * m + c]);
    v[c] = (Q == kL2) ? sqrt(s) : s;
  }
}

// ------------------------------------------------------- reductions (K2)
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, err};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const double lo = __dadd_rn(s.lo, __dadd_rn(a.lo, b.lo));
  return two_sum(s.hi, lo);
}
__device__ __forceinline__ DD dd_add(DD a, double b) { return dd_add(a, DD{b, 0.0}); }
__device__ __forceinline__ DD dd_sq(double a) {
  const double p = __dmul_rn(a, a);
  return {p, fma(a, a, -p)};
}
__device__ __forceinline__ double dd_value(DD a) { return __dadd_rn(a.hi, a.lo); }

template <typename F, typename V>
__device__ __forceinline__ V warp_reduce(V v, F op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ DD warp_reduce_dd(DD v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    DD w{__shfl_xor_sync(0xffffffffu, v.hi, o), __shfl_xor_sync(0xffffffffu, v.lo, o)};
    v = dd_add(v, w);
  }
  return v;
}

// Block-wide reductions for blockDim.x == kOuterThreads; result broadcast.
// Fixed tree => deterministic.  `scratch` needs 32 slots of 16 bytes.
__device__ __forceinline__ DD block_sum_dd(DD v, DD* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_reduce_dd(v);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  DD t = (lane < (blockDim.x >> 5)) ? scratch[lane] : DD{0.0, 0.0};
  t = warp_reduce_dd(t);
  return t;
}
__device__ __forceinline__ void block_sum_count(double& s, long long& c, double* sscr, long long* cscr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  s = warp_reduce(s, [](double a, double b) { return __dadd_rn(a, b); });
  c = warp_reduce(c, [](long long a, long long b) { return a + b; });
  __syncthreads();
  if (lane == 0) {
    sscr[w] = s;
    cscr[w] = c;
  }
  __syncthreads();
  s = (lane < (blockDim.x >> 5)) ? sscr[lane] : 0.0;
  c = (lane < (blockDim.x >> 5)) ? cscr[lane] : 0;
  s = warp_reduce(s, [](double a, double b) { return __dadd_rn(a, b); });
  c = warp_reduce(c, [](long long a, long long b) { return a + b; });
}
__device__ __forceinline__ double block_min(double v, double* scr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_reduce(v, [](double a, double b) { return fmin(a, b); });
  __syncthreads();
  if (lane == 0) scr[w] = v;
  __syncthreads();
  v = (lane < (blockDim.x >> 5)) ? scr[lane] : __longlong_as_double(0x7ff0000000000000ll);
  return warp_reduce(v, [](double a, double b) { return fmin(a, b); });
}
__device__ __forceinline__ long long block_count(long long c, long long* scr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  c = warp_reduce(c, [](long long a, long long b) { return a + b; });
  __syncthreads();
  if (lane == 0) scr[w] = c;
  __syncthreads();
  c = (lane < (blockDim.x >> 5)) ? scr[lane] : 0;
  return warp_reduce(c, [](long long a, long long b) { return a + b; });
}
__device__ __forceinline__ int block_or(int v, int* scr) {
  return __syncthreads_or(v);
}

// ------------------------------------------------------------------- K2
// Outer projection of a length-m vector held in shared memory.
struct OuterArgs {
  const void* vin;   // input vector
  int vkind;         // 0: float |y| bits (K1 l_inf over f32), 1: double, 2: float values
  int64_t m;
  int p;             // outer norm
  double eta;
  double* u_out;     // projected vector (budgets), double[m], required
  double* v_out;     // nullable: the input as f64 (column norms)
  float2* rdrn;      // nullable: per column {RD(u), RN(u)} for the f32 l_inf apply
  double* factor;    // nullable: per column u/v (v > u) or 1 for the l2 apply
  mp_info* info;     // required
  void* scratch;     // k_outer_large only: LargeScratch in the workspace
};

constexpr int kOuterMaxPerThread = 24;
constexpr int64_t kOuterMaxM = static_cast<int64_t>(kOuterThreads) * kOuterMaxPerThread;

__device__ __forceinline__ double outer_load(const OuterArgs& a, int64_t i) {
  if (a.vkind == 0) return static_cast<double>(__uint_as_float(static_cast<const unsigned int*>(a.vin)[i]));
  if (a.vkind == 1) return static_cast<const double*>(a.vin)[i];
  return static_cast<double>(static_cast<const float*>(a.vin)[i]);
}

__global__ void __launch_bounds__(kOuterThreads) k_outer(OuterArgs a) {
  extern __shared__ double sv[];
  __shared__ DD dscr[32];
  __shared__ double sscr[32];
  __shared__ long long cscr[32];
  const int tid = threadIdx.x;
  const int64_t m = a.m;
  const double eta = a.eta;

  // Load + finiteness + the feasibility / norm sum (double-double).
  int bad = 0;
  DD acc{0.0, 0.0};
  for (int64_t i = tid; i < m; i += kOuterThreads) {
    const double x = outer_load(a, i);
    sv[i] = x;
    bad |= !isfinite(x);
    if (a.p == kL2) acc = dd_add(acc, dd_sq(x));
    else acc = dd_add(acc, fabs(x));
  }
  bad = __syncthreads_or(bad);
  if (bad) {
    if (tid == 0) {
      a.info->status = MP_ERR_VALUE;
      a.info->tau = -1.0;
      a.info->active = -1;
      a.info->iterations = 0;
    }
    return;
  }
  const DD total = block_sum_dd(acc, dscr);

  // mode: 0 identity, 1 zero, 2 l1 threshold tau, 3 l2 scale, 4 linf clip
  int mode = 0;
  double tau = -1.0, scale = 1.0;
  long long active = -1;
  int iters = 0;
  if (a.p == kInf) {
    mode = 4;
  } else if (a.p == kL2) {
    const double norm = sqrt(dd_value(total));
    if (!(norm <= eta) && norm != 0.0) {
      mode = 3;
      scale = eta / norm;
    }
  } else if (m > 0 && !(dd_value(total) <= eta)) {
    if (eta == 0.0) {
      mode = 1;
      tau = 0.0;
      active = 0;
    } else {
      mode = 2;
      // Michelot fixed point on a monotonically shrinking active set.
      unsigned int mask = 0;
      for (int j = 0; j < kOuterMaxPerThread; ++j)
        if (tid + static_cast<int64_t>(j) * kOuterThreads < m) mask |= 1u << j;
      double t = (dd_value(total) - eta) / static_cast<double>(m);
      long long kprev = m;
      for (;;) {
        double s = 0.0;
        long long c = 0;
#pragma unroll 4
        for (int j = 0; j < kOuterMaxPerThread; ++j) {
          if (!(mask >> j & 1u)) continue;
          const double x = fabs(sv[tid + static_cast<int64_t>(j) * kOuterThreads]);
          if (x > t) {
            s = __dadd_rn(s, x);
            ++c;
          } else {
            mask &= ~(1u << j);
          }
        }
        block_sum_count(s, c, sscr, cscr);
        ++iters;
        if (c == kprev || c == 0) break;
        t = (s - eta) / static_cast<double>(c);
        kprev = c;
      }
      // Final threshold, reference definition: cutoff = smallest active
      // magnitude, k = #{|v| >= cutoff}, tau = (sum_{|v|>=cutoff} |v| - eta)/k.
      double lmin = __longlong_as_double(0x7ff0000000000000ll);
      for (int j = 0; j < kOuterMaxPerThread; ++j)
        if (mask >> j & 1u) lmin = fmin(lmin, fabs(sv[tid + static_cast<int64_t>(j) * kOuterThreads]));
      const double cutoff = block_min(lmin, sscr);
      DD ps{0.0, 0.0};
      long long pk = 0;
      for (int64_t i = tid; i < m; i += kOuterThreads) {
        const double x = fabs(sv[i]);
        if (x >= cutoff) {
          ps = dd_add(ps, x);
          ++pk;
        }
      }
      const DD S = block_sum_dd(ps, dscr);
      active = block_count(pk, cscr);
      const DD d = two_sum(S.hi, -eta);
      tau = __dadd_rn(d.hi, __dadd_rn(d.lo, S.lo)) / static_cast<double>(active);
    }
  }

  long long zeros = 0, surv = 0;
  for (int64_t i = tid; i < m; i += kOuterThreads) {
    const double x = sv[i];
    double u;
    switch (mode) {
      case 1: u = 0.0; break;
      case 2: {
        const double d = fabs(x) - tau;
        u = d > 0.0 ? copysign(d, x) : 0.0;
        break;
      }
      case 3: u = x * scale; break;
      case 4: u = fabs(x) > eta ? copysign(eta, x) : x; break;
      default: u = x;
    }
    a.u_out[i] = u;
    if (a.v_out) a.v_out[i] = x;
    zeros += (u == 0.0 || x == 0.0);
    surv += (u != 0.0);
    if (a.rdrn) a.rdrn[i] = make_float2(__double2float_rz(u), __double2float_rn(u));
    if (a.factor) a.factor[i] = (x > u) ? u / x : 1.0;
  }
  zeros = block_count(zeros, cscr);
  surv = block_count(surv, cscr);
  if (tid == 0) {
    a.info->status = MP_OK;
    a.info->tau = tau;
    a.info->active = active;
    a.info->iterations = iters;
    a.info->zero_columns = zeros;
    a.info->survivors = surv;
  }
}

// ------------------------------------------------------------------- K3
// l_inf clamp (proj/src/fiber_kernels.cpp:43-49) / l2 scale (:50-55).
// colp: float2 {RD(u), RN(u)} (f32 l_inf), double u (f64 l_inf) or double
// factor (l2).  `dead` columns (u == 0) are written as +0 without a read
// unless MP_FLAG_EXACT_ZERO_SIGN.
template <typename T, int VEC, int Q, int U>
__global__ void __launch_bounds__(kThreads)
    k_apply(const T* __restrict__ y, T* __restrict__ x, int64_t n, int64_t m, int64_t rpb, int nrb,
            const void* __restrict__ colp, const double* __restrict__ budgets,
            const mp_info* __restrict__ info, unsigned flags) {
  if (info->status != MP_OK) return;
  const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * VEC;
  if (c0 >= m) return;
  const int64_t rb = static_cast<int64_t>(nrb) - 1 - blockIdx.y;  // reverse sweep: L2 tail reuse
  const int64_t r0 = rb * rpb;
  const int64_t r1 = min(n, r0 + rpb);

  // per-column parameters
  float rd[VEC], rn[VEC];
  double pu[VEC];
  bool dead = !(flags & MP_FLAG_EXACT_ZERO_SIGN);
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    if constexpr (Q == kInf && sizeof(T) == 4) {
      const float2 q = static_cast<const float2*>(colp)[c0 + j];
      rd[j] = q.x;
      rn[j] = q.y;
    } else {
      pu[j] = static_cast<const double*>(colp)[c0 + j];
    }
    dead = dead && (budgets[c0 + j] == 0.0);
  }
  T* q = x + r0 * m + c0;
  if (dead) {
    T z[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) z[j] = T(0);
    for (int64_t r = r0; r < r1; ++r, q += m) store_stream<T, VEC>(q, z);
    return;
  }
  auto op = [&](T e, int j) -> T {
    if constexpr (Q == kInf) {
      if constexpr (sizeof(T) == 4) return fabsf(e) > rd[j] ? copysignf(rn[j], e) : e;
      else return fabs(e) > pu[j] ? copysign(pu[j], e) : e;
    } else {
      if constexpr (sizeof(T) == 4) return __double2float_rn(__dmul_rn(static_cast<double>(e), pu[j]));
      else return __dmul_rn(e, pu[j]);
    }
  };
  const T* p = y + r0 * m + c0;
  int64_t r = r0;
  for (; r + U <= r1; r += U, p += U * m, q += U * m) {
    T e[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) load_last<T, VEC>(p + u * m, e[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) e[u][j] = op(e[u][j], j);
      store_stream<T, VEC>(q + u * m, e[u]);
    }
  }
  for (; r < r1; ++r, p += m, q += m) {
    T e[VEC];
    load_last<T, VEC>(p, e);
#pragma unroll
    for (int j = 0; j < VEC; ++j) e[j] = op(e[j], j);
    store_stream<T, VEC>(q, e);
  }
}

}  // namespace mpk
