// mp_l1quad.cuh -- K3b fast path: per-column l1-ball projection for strips
// of 16-byte rows (4 f32 / 2 f64 columns), the l_{1,1} apply pass
// (proj/src/fiber_kernels.cpp:56-65 -> project_l1_fast_inplace,
// proj/src/vector_balls.cpp:150-161).
//
// One CTA owns C4 adjacent columns over all n rows:
//  * staging: cp.async 16-byte row pieces straight into a ROW-MAJOR tile --
//    the whole strip in flight at once, no registers, no transpose;
//  * 8 warps split the rows; inside a warp, lane group c (LPC lanes) owns
//    column c, lane k of the group rows k, k+LPC, ... of the warp's range.
//    In a row-major tile with 16-byte rows that mapping is bank-conflict free
//    (bank = 4*(row % 8) + column for f32);
//  * Michelot's fixed point per column, every thread compacting its own
//    survivors in place, reduced LPC lanes -> warp -> CTA (one barrier per
//    pass, double-buffered partials, fixed order => identical totals in all
//    threads).  First iterate from the norm pass: t1 = (v_j - u_j) / n.
//    Compares run in the staged type against RD(t); sums in f64; converged
//    set == reference {|y| >= cutoff} => tau_j = (S - u_j) / k.
//  * apply: re-land the strip (L2-resident) with cp.async, shrink with the
//    f64-accurate float-pair tau, store 16-byte row pieces.
#pragma once

#include <cuda_runtime.h>

#include "mp_cuda.h"
#include "mp_kernels.cuh"
#include "mp_l1cols.cuh"

namespace mpk {

constexpr int kQuadWarps = 8;
constexpr int kQuadThreads = 32 * kQuadWarps;

template <typename T>
inline bool l1_quad_ok(const void* y, const void* x, int64_t m) {
  constexpr int C4 = 16 / sizeof(T);
  return m % C4 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
}

template <typename T, bool DERIVE>
__global__ void __launch_bounds__(kQuadThreads)
    k_l1quad(const T* __restrict__ y, T* __restrict__ x, int n, int64_t m, const double* __restrict__ v,
             const double* __restrict__ u, double* __restrict__ tau_out, const mp_info* __restrict__ info,
             const OuterParams* __restrict__ params, double* __restrict__ u_out) {
  constexpr int C4 = 16 / sizeof(T);  // columns per CTA (one 16-byte row piece)
  constexpr int LPC = 32 / C4;        // lanes per column inside a warp
  pdl_wait();
  tl_begin(3);
  if (info->status != MP_OK) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);  // [n][C4] row-major
  __shared__ double red_s[2][kQuadWarps][C4];
  __shared__ int red_c[2][kQuadWarps][C4];
  __shared__ int skind[C4];
  __shared__ double stau[C4];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = lane / LPC, k = lane % LPC;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * C4;

  // column parameters (every thread computes its column's; thread 0 of the
  // column group publishes)
  const double vj = v[c0 + c];
  const double uj = DERIVE ? derive_u(*params, vj) : u[c0 + c];
  const int kind = vj <= uj ? 1 : (uj == 0.0 ? 2 : 3);
  if (g == 0 && k == 0) {
    skind[c] = kind;
    stau[c] = -1.0;
    if (DERIVE && u_out) u_out[c0 + c] = uj;
  }
  const int any_proj = __syncthreads_or(kind == 3);
  const long long ck0 = clock64();
  long long ck1 = ck0, ck2 = ck0;
  int npass = 0;

  if (any_proj) {
    for (int r = threadIdx.x; r < n; r += kQuadThreads) cp_async_16(tile + static_cast<int64_t>(r) * C4, y + r * m + c0);
    cp_async_all();
    __syncthreads();
    ck1 = clock64();

    // rows [rb, re) of this warp; lane k of column c owns rb + k + LPC*j
    const int rw = ((n + kQuadWarps - 1) / kQuadWarps + LPC - 1) / LPC * LPC;
    const int rb = min(n, g * rw), re = min(n, rb + rw);
    T* mine = tile + static_cast<int64_t>(rb + k) * C4 + c;
    int cnt = re - rb > k ? (re - rb - k + LPC - 1) / LPC : 0;
    double t = (vj - uj) / static_cast<double>(n);
    int kprev = n, K = 0, par = 0;
    double S = 0.0;
    bool done = kind != 3;
    if (done) cnt = 0;
    for (int pass = 0; pass < 4 * 1024; ++pass) {
      ++npass;
      const T thr = round_down_to(T(0), t);
      // Batches of 8: all loads first (independent LDS in flight), then the
      // compacting stores -- they land at slots <= the batch's own, so the
      // batch is read before it can be overwritten.
      constexpr int kStep = LPC * C4;  // slot stride of one thread (elements)
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int kept = 0;
      for (int j = 0; j < cnt; j += 8) {  // masked batches: no serial tail loop
        T a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = (j + q < cnt) ? fabs(mine[kStep * (j + q)]) : T(0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const bool kq = a[q] > thr;  // masked entries are 0 <= thr
          const double dq = kq ? static_cast<double>(a[q]) : 0.0;
          if ((q & 3) == 0) s0 += dq;
          else if ((q & 3) == 1) s1 += dq;
          else if ((q & 3) == 2) s2 += dq;
          else s3 += dq;
          if (j + q < cnt) mine[kStep * kept] = a[q];  // the slot is re-written or dropped
          kept += kq;
        }
      }
      s0 += s2;
      s1 += s3;
      cnt = kept;
      double s = s0 + s1;
      int cc = kept;
#pragma unroll
      for (int o = LPC / 2; o > 0; o >>= 1) {  // within the column's lane group
        s += __shfl_xor_sync(0xffffffffu, s, o);
        cc += __shfl_xor_sync(0xffffffffu, cc, o);
      }
      if (k == 0) {
        red_s[par][g][c] = s;
        red_c[par][g][c] = cc;
      }
      __syncthreads();
      s = 0.0;
      cc = 0;
#pragma unroll
      for (int w = 0; w < kQuadWarps; ++w) {
        s += red_s[par][w][c];
        cc += red_c[par][w][c];
      }
      par ^= 1;
      if (!done) {
        if (cc == 0) {
          done = true;  // cannot happen for 0 < u_j < v_j; keep the last set
        } else {
          S = s;
          K = cc;
          if (cc == kprev) done = true;
          else {
            kprev = cc;
            t = fmax(t, (s - uj) / static_cast<double>(cc));
          }
        }
        if (done) cnt = 0;
      }
      if (!__syncthreads_or(!done)) break;
    }
    if (kind == 3 && g == 0 && k == 0) stau[c] = (S - uj) / static_cast<double>(K);
    __syncthreads();
  }
  ck2 = clock64();
  if (g == 0 && k == 0) tau_out[c0 + c] = stau[c];

  // ---- apply
  bool need_store = any_proj || x != y;
#pragma unroll
  for (int e = 0; e < C4; ++e) need_store = need_store || skind[e] == 2;
  if (!need_store) {
    tl_end(3);
    return;
  }
  int kk[C4];
  TauPair tp[C4];
  double td[C4];
#pragma unroll
  for (int e = 0; e < C4; ++e) {
    kk[e] = skind[e];
    td[e] = stau[e];
    tp[e].hi = __double2float_rn(td[e]);
    tp[e].lo = __double2float_rn(td[e] - static_cast<double>(tp[e].hi));
  }
  if (any_proj)
    for (int r = threadIdx.x; r < n; r += kQuadThreads) cp_async_16(tile + static_cast<int64_t>(r) * C4, y + r * m + c0);
  cp_async_all();  // each thread reads back only the rows it landed
  for (int r = threadIdx.x; r < n; r += kQuadThreads) {
    T e[C4];
    if (any_proj) {
      if constexpr (sizeof(T) == 4) {
        const float4 q = *reinterpret_cast<const float4*>(tile + static_cast<int64_t>(r) * C4);
        e[0] = q.x; e[1 % C4] = q.y; e[2 % C4] = q.z; e[3 % C4] = q.w;
      } else {
        const double2 q = *reinterpret_cast<const double2*>(tile + static_cast<int64_t>(r) * C4);
        e[0] = q.x; e[1 % C4] = q.y;
      }
    } else {
      if constexpr (sizeof(T) == 4) {
        const float4 q = __ldcs(reinterpret_cast<const float4*>(y + r * m + c0));
        e[0] = q.x; e[1 % C4] = q.y; e[2 % C4] = q.z; e[3 % C4] = q.w;
      } else {
        const double2 q = __ldcs(reinterpret_cast<const double2*>(y + r * m + c0));
        e[0] = q.x; e[1 % C4] = q.y;
      }
    }
#pragma unroll
    for (int q = 0; q < C4; ++q) {
      if (kk[q] == 2) e[q] = T(0);
      else if (kk[q] == 3) {
        if constexpr (sizeof(T) == 4) {
          const float dm = shrink_mag(fabsf(e[q]), tp[q]);
          e[q] = dm > 0.0f ? copysignf(dm, e[q]) : 0.0f;
        } else {
          const double dm = fabs(e[q]) - td[q];
          e[q] = dm > 0.0 ? copysign(dm, e[q]) : 0.0;
        }
      }
    }
    T* dst = x + r * m + c0;
    if constexpr (sizeof(T) == 4)
      __stcs(reinterpret_cast<float4*>(dst), make_float4(e[0], e[1 % C4], e[2 % C4], e[3 % C4]));
    else
      __stcs(reinterpret_cast<double2*>(dst), make_double2(e[0], e[1 % C4]));
  }
  if (threadIdx.x == 0 && g_mp_timeline) {  // profiling aid: passes and per-phase SM cycles, slots 8..13
    const long long ck3 = clock64();
    atomicAdd(g_mp_timeline + 8, static_cast<unsigned long long>(npass));
    atomicMax(g_mp_timeline + 9, static_cast<unsigned long long>(npass));
    atomicAdd(g_mp_timeline + 10, 1ull);
    atomicAdd(g_mp_timeline + 11, static_cast<unsigned long long>(ck1 - ck0));
    atomicAdd(g_mp_timeline + 12, static_cast<unsigned long long>(ck2 - ck1));
    atomicAdd(g_mp_timeline + 13, static_cast<unsigned long long>(ck3 - ck2));
  }
  tl_end(3);
}

}  // namespace mpk
