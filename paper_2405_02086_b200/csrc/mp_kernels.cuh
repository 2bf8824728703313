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
//                      device: one register CTA, a <=16-CTA DSMEM cluster or a
//                      cooperative grid; f64 Michelot fixed point for the l1
//                      threshold, tau = (sum_A v - eta)/|A| from fixed-order
//                      f64 tree sums over the final active set A (the
//                      reference sums in long double, vector_balls.cpp:32-40;
//                      agreement ~1e-15 relative).
//   K3 k_apply         fused clamp / scale (proj/src/fiber_kernels.cpp:37-55),
//                      streaming loads/stores, zero-budget column groups
//                      written without being read, row blocks swept in reverse
//                      so the L2-resident tail of K1 is re-used.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "mp_cuda.h"

namespace mpk {

namespace cg = cooperative_groups;

constexpr int kL1 = 0, kL2 = 1, kInf = 2;
constexpr int kThreads = 256;  // K1 / K3 CTA size
constexpr int kOuterThreads = 256;   // K2 threads per cluster CTA
constexpr int kOuterMaxCluster = 16;

// ------------------------------------------------------------ pack helpers
template <typename T, int VEC> struct PackT;
template <> struct PackT<float, 8> { using type = float4; };  // 256-bit path uses inline PTX
template <> struct PackT<float, 4> { using type = float4; };
template <> struct PackT<float, 2> { using type = float2; };
template <> struct PackT<float, 1> { using type = float; };
template <> struct PackT<double, 4> { using type = double2; };  // 256-bit path uses inline PTX
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
  if constexpr (sizeof(T) * VEC == 32) {
    // 256-bit LDG (sm_100): half the LSU instructions of float4 loads
    if constexpr (sizeof(T) == 4)
      asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
          : "l"(p));
    else
      asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
          : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3])
          : "l"(p));
  } else {
    using V = typename PackT<T, VEC>::type;
    V v = __ldg(reinterpret_cast<const V*>(p));
    memcpy(o, &v, sizeof(V));
  }
}
// Last use of the data: evict-first.
template <typename T, int VEC>
__device__ __forceinline__ void load_last(const T* p, T (&o)[VEC]) {
  if constexpr (sizeof(T) * VEC == 32) {
    if constexpr (sizeof(T) == 4)
      asm("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
          : "l"(p));
    else
      asm("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(o[0]), "=d"(o[1]), "=d"(o[2]), "=d"(o[3]) : "l"(p));
  } else {
    using V = typename PackT<T, VEC>::type;
    V v = __ldcs(reinterpret_cast<const V*>(p));
    memcpy(o, &v, sizeof(V));
  }
}
template <typename T, int VEC>
__device__ __forceinline__ void store_stream(T* p, const T (&o)[VEC]) {
  if constexpr (sizeof(T) * VEC == 32) {
    if constexpr (sizeof(T) == 4)
      asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(o[0]), "f"(o[1]), "f"(o[2]),
                   "f"(o[3]), "f"(o[4]), "f"(o[5]), "f"(o[6]), "f"(o[7])
                   : "memory");
    else
      asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(o[0]), "d"(o[1]), "d"(o[2]), "d"(o[3])
                   : "memory");
  } else {
    using V = typename PackT<T, VEC>::type;
    V v;
    memcpy(&v, o, sizeof(V));
    __stcs(reinterpret_cast<V*>(p), v);
  }
}

// Device-side timeline (profiling aid, mp_profile_timeline): when set, thread
// 0 of every CTA folds %globaltimer into [2k] = min start, [2k+1] = max end
// for kernel k (0 K1, 1 finalize, 2 K2, 3 K3).  One predicated load per CTA
// when unset.
__device__ unsigned long long* g_mp_timeline = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tl_begin(int k) {
  if (threadIdx.x == 0) {
    unsigned long long* tl = g_mp_timeline;
    if (tl) atomicMin(tl + 2 * k, gtimer());
  }
}
__device__ __forceinline__ void tl_end(int k) {
  if (threadIdx.x == 0) {
    unsigned long long* tl = g_mp_timeline;
    if (tl) atomicMax(tl + 2 * k + 1, gtimer());
  }
}

// Programmatic dependent launch (sm_90+): wait for the producer grid's
// memory, and let the consumer grid be scheduled early.  Both are no-ops
// when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ------------------------------------------------------------------- K1
// grid = (column tiles, row blocks); thread owns columns [c0, c0+VEC) over
// rows [r0, r1).  out: BitsT<T>[m] (l_inf, pre-zeroed) or double[R][m].
// Pointer step the optimiser cannot see through: without it nvcc
// strength-reduces an unrolled p += stride into U live 64-bit addresses
// (80 registers, occupancy 3); with it one address stays live.
template <typename T>
__device__ __forceinline__ T* step_ptr(T* p, int64_t elems) {
  T* r;
  asm("add.s64 %0, %1, %2;" : "=l"(r) : "l"(p), "l"(elems * static_cast<int64_t>(sizeof(T))));
  return r;
}

// Row mapping shared by K1 and K3: CTA row-slot b of R walks either the
// contiguous block [b*rpb, (b+1)*rpb) (interleave = 0) or the rows b, b+R,
// b+2R, ... (interleave = 1: the whole grid sweeps one band of R rows at a
// time, i.e. one contiguous ~R*m*sizeof(T) region of HBM).
// `rpb` doubles as the interleaved quotient: with interleave the host passes
// rpb = n / R, so slot b owns rpb + (b < n % R) rows (no device division).
// Row slots are (blockIdx.y, threadIdx.y): R = gridDim.y * blockDim.y.
struct RowWalk {
  int64_t r0, step, cnt;
};
template <bool RG = false>
__device__ __forceinline__ RowWalk row_walk(int64_t n, int64_t rpb, int interleave) {
  const int64_t b = RG ? static_cast<int64_t>(blockIdx.y) * blockDim.y + threadIdx.y : blockIdx.y;
  const int64_t R = RG ? static_cast<int64_t>(gridDim.y) * blockDim.y : gridDim.y;
  if (interleave) return {b, R, rpb + (b < n - rpb * R ? 1 : 0)};
  const int64_t r0 = b * rpb;
  return {r0, 1, r0 < n ? min(rpb, n - r0) : 0};
}

// K1.  blockDim = (column threads, row groups): narrow matrices (few column
// threads) stack up to 16 row groups in one CTA and fold them in shared
// memory first, so each column sees one atomic / partial per CTA instead of
// one per row group (atomics on few addresses serialise in L2).
// l_inf: CTA row block r folds into copy r % ncopy of the maxima (narrow
// matrices: fewer same-address atomics serialised in one L2 slice; K2 folds
// the copies).
template <typename T, int VEC, int Q, int U, bool RG>
__global__ void __launch_bounds__(RG ? 1024 : kThreads, RG ? 1 : 8)
    k_colnorm(const T* __restrict__ y, int64_t n, int64_t m, int64_t rpb, int interleave, void* __restrict__ out,
              int ncopy) {
  pdl_trigger();  // let the (single-CTA) outer kernel be scheduled as SMs free up
  tl_begin(0);
  const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * VEC;
  if constexpr (!RG) {
    if (c0 >= m) return;
  }
  const bool active = !RG || c0 < m;
  const RowWalk rw = row_walk<RG>(n, rpb, interleave);
  const int64_t cnt = RG ? (active ? rw.cnt : 0) : rw.cnt;
  const int64_t ds = rw.step * m;  // element stride between consecutive rows of this thread
  const T* p = y + rw.r0 * m + (active ? c0 : 0);
  int64_t k = 0;
  if constexpr (Q == kInf) {
    using B = typename BitsT<T>::type;
    B acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0;
    for (; k + U <= cnt; k += U) {
      T e[U][VEC];
#pragma unroll
      for (int u = 0; u < U; ++u) {  // one live address: p advances load by load
        load_keep<T, VEC>(p, e[u]);
        p = step_ptr(p, ds);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = max(acc[j], abs_bits(e[u][j]));
    }
    for (; k < cnt; ++k, p += ds) {
      T e[VEC];
      load_keep<T, VEC>(p, e);
#pragma unroll
      for (int j = 0; j < VEC; ++j) acc[j] = max(acc[j], abs_bits(e[j]));
    }
    if (RG) {  // fold the row groups (max is order-free)
      extern __shared__ unsigned char k1_smem[];
      B* red = reinterpret_cast<B*>(k1_smem);
      const int slot = (threadIdx.y * blockDim.x + threadIdx.x) * VEC;
#pragma unroll
      for (int j = 0; j < VEC; ++j) red[slot + j] = acc[j];
      __syncthreads();
      if (threadIdx.y != 0) return;
      for (int r = 1; r < static_cast<int>(blockDim.y); ++r)
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = max(acc[j], red[(r * blockDim.x + threadIdx.x) * VEC + j]);
    }
    if (RG && !active) return;
    B* vb = static_cast<B*>(out) + static_cast<int64_t>(blockIdx.y % ncopy) * m + c0;
#pragma unroll
    for (int j = 0; j < VEC; ++j) atomicMax(vb + j, acc[j]);
    tl_end(0);
  } else {
    double acc[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) acc[j] = 0.0;
    for (; k + U <= cnt; k += U) {
      T e[U][VEC];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        load_keep<T, VEC>(p, e[u]);
        p = step_ptr(p, ds);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const double dv = static_cast<double>(e[u][j]);
          acc[j] = (Q == kL1) ? __dadd_rn(acc[j], fabs(dv)) : __dadd_rn(acc[j], __dmul_rn(dv, dv));
        }
    }
    for (; k < cnt; ++k, p += ds) {
      T e[VEC];
      load_keep<T, VEC>(p, e);
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        const double dv = static_cast<double>(e[j]);
        acc[j] = (Q == kL1) ? __dadd_rn(acc[j], fabs(dv)) : __dadd_rn(acc[j], __dmul_rn(dv, dv));
      }
    }
    if (RG) {  // fold the row groups in fixed order (deterministic)
      extern __shared__ unsigned char k1_smem[];
      double* red = reinterpret_cast<double*>(k1_smem);
      const int slot = (threadIdx.y * blockDim.x + threadIdx.x) * VEC;
#pragma unroll
      for (int j = 0; j < VEC; ++j) red[slot + j] = acc[j];
      __syncthreads();
      if (threadIdx.y != 0) return;
      for (int r = 1; r < static_cast<int>(blockDim.y); ++r)
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = __dadd_rn(acc[j], red[(r * blockDim.x + threadIdx.x) * VEC + j]);
    }
    if (RG && !active) return;
    double* part = static_cast<double*>(out) + static_cast<int64_t>(blockIdx.y) * m + c0;
#pragma unroll
    for (int j = 0; j < VEC; ++j) part[j] = acc[j];
    tl_end(0);
  }
}

// Fixed-order reduction of the row-block partials (l1 / l2), or conversion
// of l_inf bit patterns to f64 (kind 0 = float bits, 1 = double bits).
template <int Q>
__global__ void k_colnorm_finalize(const void* __restrict__ in, int64_t R, int64_t m, int bits_kind,
                                   double* __restrict__ v) {
  pdl_wait();
  pdl_trigger();
  tl_begin(1);
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
  tl_end(1);
}

// l1 / l2 partials -> norms with 8 warps per 32 columns: warp w sums rows
// w, w+8, ... (coalesced 32-column rows), then warp 0 adds the 8 warp sums in
// fixed order (deterministic).
template <int Q>
__global__ void __launch_bounds__(256) k_colnorm_reduce(const double* __restrict__ part, int64_t R, int64_t m,
                                                        double* __restrict__ v) {
  pdl_wait();
  pdl_trigger();
  tl_begin(1);
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  double s0 = 0.0, s1 = 0.0;
  if (c < m) {
    int64_t r = w;
    for (; r + 8 < R; r += 16) {
      s0 = __dadd_rn(s0, part[r * m + c]);
      s1 = __dadd_rn(s1, part[(r + 8) * m + c]);
    }
    if (r < R) s0 = __dadd_rn(s0, part[r * m + c]);
  }
  red[w][lane] = __dadd_rn(s0, s1);
  __syncthreads();
  if (w == 0 && c < m) {
    double s = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) s = __dadd_rn(s, red[k][lane]);
    v[c] = (Q == kL2) ? sqrt(s) : s;
  }
  tl_end(1);
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

// ------------------------------------------------------------------- K2
// Outer projection of a length-m vector held in shared memory.
// Outcome of the outer projection, enough to derive every budget from its
// norm: u = derive_u(P, v).  Written by K2, read by the apply kernels.
struct OuterParams {
  int mode;      // 0 identity, 1 zero, 2 l1 threshold tau, 3 l2 scale, 4 linf clip at eta
  int pad;
  double tau, scale, eta;
};

__device__ __forceinline__ double derive_u(const OuterParams& P, double x) {
  switch (P.mode) {
    case 1: return 0.0;
    case 2: {
      const double d = fabs(x) - P.tau;  // proj/src/vector_balls.cpp:42-48
      return d > 0.0 ? copysign(d, x) : 0.0;
    }
    case 3: return x * P.scale;                                 // :171-177
    case 4: return fabs(x) > P.eta ? copysign(P.eta, x) : x;  // :187-191
    default: return x;
  }
}

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
  OuterParams* params;  // nullable: mode / tau / scale for derive_u
  int emit;          // 1: write the per-element outputs above; 0: params + info only
  int ncopy;         // kInfCopies: fold K1's copies of the maxima (k_outer_reg<P, 256, true>); else one
};

// Fold the kInfCopies copies of K1's bit-pattern maxima for element i (max
// is order-free; all loads in flight) and leave the result in copy 0 for the
// apply pass.
constexpr int kInfCopies = 8;
template <bool STORE = true>
__device__ __forceinline__ double outer_load_fold(const OuterArgs& a, int64_t i) {
  if (a.vkind == 0) {
    unsigned* b = static_cast<unsigned*>(const_cast<void*>(a.vin));
    unsigned c8[kInfCopies];
#pragma unroll
    for (int c = 0; c < kInfCopies; ++c) c8[c] = b[c * a.m + i];
    unsigned mx = c8[0];
#pragma unroll
    for (int c = 1; c < kInfCopies; ++c) mx = max(mx, c8[c]);
    if (STORE) b[i] = mx;
    return static_cast<double>(__uint_as_float(mx));
  }
  unsigned long long* b = static_cast<unsigned long long*>(const_cast<void*>(a.vin));
  unsigned long long c8[kInfCopies];
#pragma unroll
  for (int c = 0; c < kInfCopies; ++c) c8[c] = b[c * a.m + i];
  unsigned long long mx = c8[0];
#pragma unroll
  for (int c = 1; c < kInfCopies; ++c) mx = max(mx, c8[c]);
  if (STORE) b[i] = mx;
  return __longlong_as_double(static_cast<long long>(mx));
}

__device__ __forceinline__ void outer_publish(const OuterArgs& a, int mode, double tau, double scale) {
  if (a.params) {
    a.params->mode = mode;
    a.params->tau = tau;
    a.params->scale = scale;
    a.params->eta = a.eta;
  }
}

constexpr int kOuterMaxPerThread = 24;
constexpr int64_t kOuterMaxM = static_cast<int64_t>(kOuterThreads) * kOuterMaxPerThread * kOuterMaxCluster;

__device__ __forceinline__ double outer_load(const OuterArgs& a, int64_t i) {
  if (a.vkind == 0) return static_cast<double>(__uint_as_float(static_cast<const unsigned int*>(a.vin)[i]));
  if (a.vkind == 1) return static_cast<const double*>(a.vin)[i];
  return static_cast<double>(static_cast<const float*>(a.vin)[i]);
}

__device__ __forceinline__ void block_sum_icount(double& s, int& c, double* sscr, int* cscr) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  __syncthreads();
  if (lane == 0) {
    sscr[w] = s;
    cscr[w] = c;
  }
  __syncthreads();
  s = (lane < (blockDim.x >> 5)) ? sscr[lane] : 0.0;
  c = (lane < (blockDim.x >> 5)) ? cscr[lane] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
}

// #{j : u_j == 0 || v_j == 0} from the outer outcome (v >= 0):
// l1 threshold -> m - |active set|; zero radius -> m; identity, l2 scale and
// l_inf clip zero exactly the zero norms (unless the radius / scale is 0).
__device__ __forceinline__ int outer_zero_count(int mode, int m, int active, int nzero, double eta, double scale) {
  switch (mode) {
    case 1: return m;
    case 2: return m - active;
    case 3: return scale == 0.0 ? m : nzero;
    case 4: return eta == 0.0 ? m : nzero;
    default: return nzero;
  }
}

// Cluster-wide (sum, count): CTA reduction, then every thread reads the C
// per-CTA partials through DSMEM in rank order (identical, deterministic
// totals in every CTA).  Double-buffered partials: one cluster barrier per
// reduction.
__device__ __forceinline__ void cluster_sum_icount(double& s, int& c, double* sscr, int* cscr, double* ps,
                                                   int* pc, int& par, const cg::cluster_group& cl, int C) {
  block_sum_icount(s, c, sscr, cscr);
  if (threadIdx.x == 0) {
    ps[par] = s;
    pc[par] = c;
  }
  cl.sync();
  // lane r fetches CTA r's partial (all DSMEM loads in flight at once), then
  // the same xor butterfly in every warp of every CTA => identical totals.
  const int lane = threadIdx.x & 31;
  double S = lane < C ? *cl.map_shared_rank(&ps[par], lane) : 0.0;
  int N = lane < C ? *cl.map_shared_rank(&pc[par], lane) : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    S += __shfl_xor_sync(0xffffffffu, S, o);
    N += __shfl_xor_sync(0xffffffffu, N, o);
  }
  par ^= 1;
  s = S;
  c = N;
}

// K2: the outer projection of the length-m norm vector
// (proj/src/vector_balls.cpp:150-191,207-214) on a thread-block CLUSTER of C
// CTAs (C <= 16): CTA r holds the r-th contiguous chunk of v in its shared
// memory, P elements per thread (compile time: every per-element loop is
// unrolled with constant shifts on the active-set mask).  A single CTA spent
// ~14 us here on one SM's issue slots; spreading the vector over C SMs keeps
// every pass to a few instructions per thread plus one DSMEM reduction.
// Michelot (tau_{t+1} = (sum_{A_t} |v| - eta) / |A_t|, A_{t+1} = A_t cap
// {|v| > tau_{t+1}}) converges when the active set stops shrinking; the
// converged A equals the reference's {|v| >= cutoff} (cutoff = min A), so
// the last pass's (sum, count) give tau directly.
template <int P>
__global__ void __launch_bounds__(kOuterThreads) k_outer(OuterArgs a) {
  pdl_wait();
  pdl_trigger();
  tl_begin(2);
  cg::cluster_group cl = cg::this_cluster();
  const int C = static_cast<int>(cl.num_blocks());
  const int rank = static_cast<int>(cl.block_rank());
  extern __shared__ double sv[];
  __shared__ double sscr[32];
  __shared__ int cscr[32];
  __shared__ double cps[2];
  __shared__ int cpc[2];
  int par = 0;
  const int tid = threadIdx.x;
  const int m = static_cast<int>(a.m);
  const int chunk = (m + C - 1) / C;
  const int base = rank * chunk;
  const int cnt = max(0, min(chunk, m - base));
  const double eta = a.eta;

  double s = 0.0;
  int bad = 0, nzero = 0;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const int i = tid + j * kOuterThreads;
    if (i < cnt) {
      const double x = outer_load(a, base + i);
      sv[i] = x;
      bad += !isfinite(x);
      nzero += (x == 0.0);
      s += (a.p == kL2) ? x * x : fabs(x);
    }
  }
  int flags_zeros = ((bad > 0) << 18) + nzero;
  cluster_sum_icount(s, flags_zeros, sscr, cscr, cps, cpc, par, cl, C);
  bad = flags_zeros >> 18;
  nzero = flags_zeros & ((1 << 18) - 1);
  if (bad) {
    if (rank == 0 && tid == 0) {
      a.info->status = MP_ERR_VALUE;
      a.info->tau = -1.0;
      a.info->active = -1;
      a.info->iterations = 0;
    }
    cl.sync();
    return;
  }

  // mode: 0 identity, 1 zero, 2 l1 threshold tau, 3 l2 scale, 4 linf clip
  int mode = 0;
  double tau = -1.0, scale = 1.0;
  int active = -1;
  int iters = 0;
  if (a.p == kInf) {
    mode = 4;
  } else if (a.p == kL2) {
    const double norm = sqrt(s);
    if (!(norm <= eta) && norm != 0.0) {
      mode = 3;
      scale = eta / norm;
    }
  } else if (m > 0 && !(s <= eta)) {
    if (eta == 0.0) {
      mode = 1;
      tau = 0.0;
      active = 0;
    } else {
      mode = 2;
      unsigned long long mask = 0;
#pragma unroll
      for (int j = 0; j < P; ++j)
        if (tid + j * kOuterThreads < cnt) mask |= 1ull << j;
      double t = (s - eta) / static_cast<double>(m);
      int kprev = m;
      double S = s;
      for (;;) {
        double ps = 0.0;
        int pc = 0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
          if (mask >> j & 1ull) {
            const double x = fabs(sv[tid + j * kOuterThreads]);
            const bool keep = x > t;
            ps += keep ? x : 0.0;
            pc += keep;
            if (!keep) mask &= ~(1ull << j);
          }
        }
        cluster_sum_icount(ps, pc, sscr, cscr, cps, cpc, par, cl, C);
        ++iters;
        if (pc == 0) break;  // cannot happen for eta > 0; keep the last set
        S = ps;
        const bool stable = (pc == kprev);
        kprev = pc;
        if (stable) break;
        t = (ps - eta) / static_cast<double>(pc);
      }
      active = kprev;
      tau = (S - eta) / static_cast<double>(active);
    }
  }

  if (rank == 0 && tid == 0) outer_publish(a, mode, tau, scale);
  double* __restrict__ uo = a.u_out + base;
  if (a.emit) {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int i = tid + j * kOuterThreads;
      if (i < cnt) {
        const double x = sv[i];
        double u = x;
        if (mode == 2) {
          const double dd = fabs(x) - tau;
          u = dd > 0.0 ? copysign(dd, x) : 0.0;
        } else if (mode == 4) {
          u = fabs(x) > eta ? copysign(eta, x) : x;
        } else if (mode == 3) {
          u = x * scale;
        } else if (mode == 1) {
          u = 0.0;
        }
        uo[i] = u;
        if (a.rdrn) a.rdrn[base + i] = make_float2(__double2float_rz(u), __double2float_rn(u));
        if (a.v_out) a.v_out[base + i] = x;
        if (a.factor) a.factor[base + i] = (x > u) ? u / x : 1.0;
      }
    }
  }
  const int zeros = outer_zero_count(mode, m, active, nzero, eta, scale);
  if (rank == 0 && tid == 0) {
    a.info->status = MP_OK;
    a.info->tau = tau;
    a.info->active = active;
    a.info->iterations = iters;
    a.info->zero_columns = zeros;
    a.info->survivors = m - zeros;
  }
  cl.sync();  // no CTA leaves while a peer may still read its DSMEM
  tl_end(2);
}

// Block all-reduce of (sum, count) with ONE barrier: double-buffered warp
// slots; every warp re-reduces the 32 slots with the same xor butterfly, so
// every thread ends with the same bits (a + b == b + a exactly).
__device__ __forceinline__ void block_allreduce(double& s, int& c, double (*sb)[32], int (*cb)[32], int& par) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if (lane == 0) {
    sb[par][w] = s;
    cb[par][w] = c;
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  s = lane < nw ? sb[par][lane] : 0.0;
  c = lane < nw ? cb[par][lane] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  par ^= 1;
}

constexpr int kOuterRegThreads = 1024;
constexpr int kOuterRegMaxP = 12;
constexpr int64_t kOuterRegMaxM = static_cast<int64_t>(kOuterRegThreads) * kOuterRegMaxP;

// The outcome of the outer projection of the norm vector.
struct OuterOutcome {
  int mode;  // 0 identity, 1 zero, 2 l1 threshold, 3 l2 scale, 4 linf clip
  double tau, scale;
  int active, iters, zeros;
  bool bad;  // a non-finite norm
};

// The body of the fast path: the CTA's threads hold the vector (element
// tid + j * blockDim.x in v[j]) and every thread returns the same outcome.
// Shared by k_outer_reg and by the apply pass of narrow matrices, whose CTAs
// each run it themselves instead of waiting for a K2 launch (k_apply, FUSE).
// FOLD: 0 one copy of the norms, 1 fold K1's copies and leave the result in
// copy 0 (K2), 2 fold without the store (the fused apply pass: thousands of
// CTAs would write the same words).
template <int P, int FOLD>
__device__ __forceinline__ OuterOutcome outer_reg_core(const OuterArgs& a, double (&v)[P], double (*sb)[32],
                                                       int (*cb)[32], int& par) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int m = static_cast<int>(a.m);
  const double eta = a.eta;
  double s = 0.0;
  int bad = 0;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const int i = tid + j * NT;
    v[j] = (i < m) ? (FOLD == 1 ? outer_load_fold<true>(a, i) : FOLD == 2 ? outer_load_fold<false>(a, i)
                                                                          : outer_load(a, i))
                   : 0.0;
  }
  int nzero = 0;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    bad += !isfinite(v[j]);
    nzero += (v[j] == 0.0) && (tid + j * NT < m);
    s += (a.p == kL2) ? v[j] * v[j] : fabs(v[j]);
  }
  // one int channel: non-finite flag (bit 18+) and #{v == 0} (bits 0..17)
  int flags_zeros = ((bad > 0) << 18) + nzero;
  block_allreduce(s, flags_zeros, sb, cb, par);
  bad = flags_zeros >> 18;
  nzero = flags_zeros & ((1 << 18) - 1);
  OuterOutcome o{0, -1.0, 1.0, -1, 0, 0, bad != 0};
  if (bad) return o;
  if (a.p == kInf) {
    o.mode = 4;
  } else if (a.p == kL2) {
    const double norm = sqrt(s);
    if (!(norm <= eta) && norm != 0.0) {
      o.mode = 3;
      o.scale = eta / norm;
    }
  } else if (m > 0 && !(s <= eta)) {
    if (eta == 0.0) {
      o.mode = 1;
      o.tau = 0.0;
      o.active = 0;
    } else {
      o.mode = 2;
      unsigned mask = 0;
#pragma unroll
      for (int j = 0; j < P; ++j)
        if (tid + j * NT < m) mask |= 1u << j;
      double t = (s - eta) / static_cast<double>(m);
      int kprev = m;
      double S = s;
      for (;;) {
        double ps = 0.0;
        int pc = 0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
          const double x = fabs(v[j]);
          const bool keep = (mask >> j & 1u) && x > t;
          ps += keep ? x : 0.0;
          pc += keep;
          mask = keep ? mask : (mask & ~(1u << j));
        }
        block_allreduce(ps, pc, sb, cb, par);
        ++o.iters;
        if (pc == 0) break;  // cannot happen for eta > 0; keep the last set
        S = ps;
        const bool stable = (pc == kprev);
        kprev = pc;
        if (stable) break;
        t = (ps - eta) / static_cast<double>(pc);
      }
      o.active = kprev;
      o.tau = (S - eta) / static_cast<double>(o.active);
    }
  }
  // Zero columns follow from the outcome (u == 0 <=> v <= tau for the l1
  // threshold, v == 0 for identity / scale / clip); survivors = m - zeros.
  o.zeros = outer_zero_count(o.mode, m, o.active, nzero, eta, o.scale);
  return o;
}

// What K2 leaves in mp_info (thread 0 of one CTA).
__device__ __forceinline__ void outer_write_info(mp_info* info, const OuterOutcome& o, int m) {
  if (o.bad) {
    info->status = MP_ERR_VALUE;
    info->tau = -1.0;
    info->active = -1;
    info->iterations = 0;
    return;
  }
  info->status = MP_OK;
  info->tau = o.tau;
  info->active = o.active;
  info->iterations = o.iters;
  info->zero_columns = o.zeros;
  info->survivors = m - o.zeros;
}

// K2 fast path (m <= 12288): ONE CTA of NT threads (1024; 256 for m <= 2048,
// where the barriers of the per-pass all-reduce dominate), the vector held in
// registers (P per thread, compile time), every reduction a single-barrier
// all-reduce.  The kernel's time is its dependency chain on one SM: a load
// wave, 1 + passes + 1 block reductions, one double division per pass.
template <int P, int NT = kOuterRegThreads, bool FOLD = false>
__global__ void __launch_bounds__(NT, 1) k_outer_reg(OuterArgs a) {
  pdl_wait();
  pdl_trigger();
  tl_begin(2);
  __shared__ double sb[2][32];
  __shared__ int cb[2][32];
  int par = 0;
  const int tid = threadIdx.x;
  const int m = static_cast<int>(a.m);
  const double eta = a.eta;
  double v[P];
  const OuterOutcome o = outer_reg_core<P, FOLD ? 1 : 0>(a, v, sb, cb, par);
  if (o.bad) {
    if (tid == 0) outer_write_info(a.info, o, m);
    return;
  }
  const int mode = o.mode;
  const double tau = o.tau, scale = o.scale;
  if (tid == 0) outer_publish(a, mode, tau, scale);
  if (a.emit) {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const int i = tid + j * NT;
      if (i < m) {
        const double x = v[j];
        double u = x;
        if (mode == 2) {
          const double dd = fabs(x) - tau;
          u = dd > 0.0 ? copysign(dd, x) : 0.0;
        } else if (mode == 4) {
          u = fabs(x) > eta ? copysign(eta, x) : x;
        } else if (mode == 3) {
          u = x * scale;
        } else if (mode == 1) {
          u = 0.0;
        }
        a.u_out[i] = u;
        if (a.v_out) a.v_out[i] = x;
        if (a.rdrn) a.rdrn[i] = make_float2(__double2float_rz(u), __double2float_rn(u));
        if (a.factor) a.factor[i] = (x > u) ? u / x : 1.0;
      }
    }
  }
  if (tid == 0) outer_write_info(a.info, o, m);
  tl_end(2);
}

// ------------------------------------------------------------------- K3
// Per-column inputs of the apply pass.  DERIVE (the bi-level hot path): each
// thread derives its columns' budgets from the norms and K2's OuterParams --
// u = derive_u(P, v) -- so K2 stays a short serial step and the per-column
// work is spread over the whole grid; row block 0 also writes the user-facing
// budgets / norms (K2 already counted zero_columns / survivors).  Otherwise
// (multi-level levels): precomputed colp (float2 {RD(u), RN(u)} for f32
// l_inf, double u for f64 l_inf, double factor for l2) and budgets.
struct ApplyCols {
  const void* colp;
  const double* budgets;
  const void* v;          // DERIVE: norms (vkind 0: float |y| bits, 1: double)
  int vkind;
  const OuterParams* params;
  double* u_out;          // DERIVE, nullable
  double* v_out;          // DERIVE, nullable
  mp_info* info_w;        // unused (K2 counts zero columns); kept for ABI of the kernel args
  OuterArgs outer;        // FUSE: the outer projection's arguments (no K2 launch)
};

__device__ __forceinline__ double load_norm(const ApplyCols& a, int64_t c) {
  return a.vkind == 0 ? static_cast<double>(__uint_as_float(static_cast<const unsigned int*>(a.v)[c]))
                      : static_cast<const double*>(a.v)[c];
}

// FUSE: column tile == the whole vector (one tile of blockDim.x * VEC >= m
// columns, blockDim.x a multiple of 32).  Every CTA of the apply pass runs the
// outer projection itself (outer_reg_core: a few block reductions over norms
// that sit in L2) instead of waiting for a one-CTA K2 launch: config 4
// (65536 x 256) K2 was 7 of 36 us, config 1 3.3 of 18 us.  CTA (0, 0) leaves
// K2's mp_info / OuterParams.  The threshold's f64 sums associate by this
// kernel's thread layout, so it may differ from a stand-alone K2's by an ulp.
template <int VEC, int FOLD>
__device__ __forceinline__ OuterOutcome apply_fused_outer(const ApplyCols& A) {
  __shared__ double sb[2][32];
  __shared__ int cb[2][32];
  int par = 0;
  double vv[VEC];
  const OuterOutcome o = outer_reg_core<VEC, FOLD>(A.outer, vv, sb, cb, par);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    outer_write_info(A.outer.info, o, static_cast<int>(A.outer.m));
    if (!o.bad) outer_publish(A.outer, o.mode, o.tau, o.scale);
  }
  return o;
}

// l_inf clamp (proj/src/fiber_kernels.cpp:43-49) / l2 scale (:50-55).
// `dead` packs (all budgets 0) are written as +0 without a read unless
// MP_FLAG_EXACT_ZERO_SIGN.
// f32 l2 runs at 4 CTAs per SM (<= 64 registers): 143.4 vs 145.4 us on config 3
// l1,2 at the 5 CTAs its 48 registers would allow (a grid of fewer row slots).
template <typename T, int VEC, int Q, int U, bool DERIVE, bool FUSE = false>
__global__ void __launch_bounds__(kThreads, (Q == kL2 && sizeof(T) == 4) ? 4 : 0)
    k_apply(const T* __restrict__ y, T* __restrict__ x, int64_t n, int64_t m, int64_t rpb, int interleave,
            ApplyCols A, const mp_info* __restrict__ info, unsigned flags) {
  pdl_wait();
  tl_begin(3);
  OuterParams PF{};  // FUSE: this CTA's own outer projection
  if constexpr (FUSE) {
    const OuterOutcome o = A.outer.ncopy > 1 ? apply_fused_outer<VEC, 2>(A) : apply_fused_outer<VEC, 0>(A);
    if (o.bad) return;
    PF.mode = o.mode;
    PF.tau = o.tau;
    PF.scale = o.scale;
    PF.eta = A.outer.eta;
  } else {
    if (info->status != MP_OK) return;
  }
  const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * VEC;
  if (c0 >= m) return;
  const RowWalk rw = row_walk(n, rpb, interleave);

  // per-column parameters
  float rd[VEC], rn[VEC];
  double pu[VEC];
  bool dead = !(flags & MP_FLAG_EXACT_ZERO_SIGN);
  if constexpr (DERIVE) {
    const OuterParams P = FUSE ? PF : *A.params;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      const double vj = (FUSE && A.outer.ncopy > 1) ? outer_load_fold<false>(A.outer, c0 + j) : load_norm(A, c0 + j);
      const double uj = derive_u(P, vj);
      if constexpr (Q == kInf && sizeof(T) == 4) {
        rd[j] = __double2float_rz(uj);
        rn[j] = __double2float_rn(uj);
      } else if constexpr (Q == kInf) {
        pu[j] = uj;
      } else {
        pu[j] = (vj > uj) ? uj / vj : 1.0;
      }
      dead = dead && (uj == 0.0);
      if (blockIdx.y == 0) {
        if (A.u_out) A.u_out[c0 + j] = uj;
        if (A.v_out) A.v_out[c0 + j] = vj;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      if constexpr (Q == kInf && sizeof(T) == 4) {
        const float2 q = static_cast<const float2*>(A.colp)[c0 + j];
        rd[j] = q.x;
        rn[j] = q.y;
      } else {
        pu[j] = static_cast<const double*>(A.colp)[c0 + j];
      }
      dead = dead && (A.budgets[c0 + j] == 0.0);
    }
  }
  // Zero-budget packs are stored without a read.  Every lane stays in the
  // one loop below and only its LOAD is predicated on the pack being live,
  // so each warp store still writes its whole contiguous row segment at
  // once: lines written partly early (by read-free lanes) and partly late
  // are evicted partially valid and cost DRAM read-modify-writes (a separate
  // store-only loop for dead lanes: config-5 iteration 0 1.13 ms per lane,
  // 0.53 ms per 16-lane group, 0.527 ms like this).  The skipped reads only
  // pay when a whole 128-byte line is dead: with 10% of the columns alive
  // at random the L1 asks for 62% of the sectors, but L2 and DRAM serve 96%
  // (the line-granular fraction, 1 - 0.9^32), whatever the cache operator
  // (.cs, .cg, .nc.L1::no_allocate measured alike; profiles/r2_zero_skip.txt).
  // Lanes past m never reach here.
  if (rw.cnt <= 0) return;
  // This CTA's rows are swept LAST-FIRST: K1 swept them first-last in the
  // same resident wave, so the rows it touched last are still in L2 when
  // this kernel starts.
  const int64_t ds = rw.step * m;
  const int64_t last = (rw.r0 + (rw.cnt - 1) * rw.step) * m + c0;
  T* q = x + last;
  const bool live = !dead;
  // f32 l2 scale: the f64 factor as a float pair (hi + lo), the product
  // y * factor formed in f32 with an exact FMA error term -- full-rate FP32
  // instead of two f32<->f64 converts (1/8 rate) and a DMUL per element.
  // Magnitudes, then the sign: factor 1 and 0 keep y's zero sign (y * 1.0,
  // y * 0.0 in the reference's doubles).
  float fh[VEC], fl[VEC];
  if constexpr (Q == kL2 && sizeof(T) == 4) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      fh[j] = __double2float_rn(pu[j]);
      fl[j] = __double2float_rn(pu[j] - static_cast<double>(fh[j]));
    }
  }
  auto op = [&](T e, int j) -> T {
    if constexpr (Q == kInf) {
      // a zero budget inside a live group: copysign keeps y's zero sign,
      // the reference's bytes (read-free groups write +0.0; +-0 compare equal)
      if constexpr (sizeof(T) == 4) return fabsf(e) > rd[j] ? copysignf(rn[j], e) : e;
      else return fabs(e) > pu[j] ? copysign(pu[j], e) : e;
    } else {
      if constexpr (sizeof(T) == 4) {
        const float a = fabsf(e);
        const float ph = a * fh[j];
        const float t = fmaf(a, fl[j], fmaf(a, fh[j], -ph));
        return copysignf(ph + t, e);
      } else {
        return __dmul_rn(e, pu[j]);
      }
    }
  };
  const T* p = y + last;
  int64_t k = 0;
  for (; k + U <= rw.cnt; k += U) {
    T e[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // one live address per stream
#pragma unroll
      for (int j = 0; j < VEC; ++j) e[u][j] = T(0);
      if (live) load_last<T, VEC>(p, e[u]);
      p = step_ptr(p, -ds);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) e[u][j] = op(e[u][j], j);
      store_stream<T, VEC>(q, e[u]);
      q = step_ptr(q, -ds);
    }
  }
  for (; k < rw.cnt; ++k, p -= ds, q -= ds) {
    T e[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) e[j] = T(0);
    if (live) load_last<T, VEC>(p, e);
#pragma unroll
    for (int j = 0; j < VEC; ++j) e[j] = op(e[j], j);
    store_stream<T, VEC>(q, e);
  }
  tl_end(3);
}

}  // namespace mpk
