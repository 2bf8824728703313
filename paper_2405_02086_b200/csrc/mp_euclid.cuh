// mp_euclid.cuh -- exact Euclidean projection onto the l_{1,inf} ball
// (proj/src/euclidean.cpp:82-170, the paper's comparison target), on device.
//
// The distance minimiser clips column j at u_j, where every active column
// leaves the same residual mass theta = sum_i (|y_ij| - u_j)_+.  Per column,
// with magnitudes sorted descending a_1 >= ... >= a_n and prefix sums P_k,
// the budget is piecewise linear in theta: u_j(theta) = (P_k - theta) / k for
// t_k <= theta < t_{k+1}, t_k = P_k - k a_k (euclidean.cpp:13-49).  theta
// solves S(theta) = sum_j u_j(theta) = eta.
//
//  EK0 k_eu_gather   |Y| transposed into column-major order (32x32 tiles,
//                    both sides coalesced) + the finiteness check
//                    (tensor.cpp:40-41);
//  EK1 k_eu_sort     one CTA per column: bitonic sort (descending) in
//                    registers / shuffles / shared memory, then the
//                    double-double prefix sums P_k (the reference's long
//                    double, euclidean.cpp:41-46);
//  EK2 k_eu_search   a cooperative grid: the feasibility test (l1,inf norm
//                    <= eta, :95-100) and Newton's iteration on the convex,
//                    decreasing, piecewise-linear S from theta = 0: each step
//                    solves the current linear segment exactly,
//                    theta' = (sum_j P_k/k - eta) / (sum_j 1/k) -- the
//                    reference's segment solve (:125-141) -- and stops when
//                    theta' lies inside that segment [max t_k, min t_{k+1}],
//                    i.e. on the segment the reference's breakpoint bisection
//                    (:103-123) brackets.  Newton from the left of a convex
//                    decreasing function never overshoots, so the iteration
//                    is monotone and finite.  Each column's segment index is
//                    a binary search over its breakpoints (upper_bound,
//                    :19-26).  Budgets u_j = max(0, (P_k - theta)/k) (:143-149);
//  EK3               the l_inf clip at u_j: the bi-level K3 apply kernel.
// Sums are deterministic (fixed trees, CTA partials reduced in CTA order).
#pragma once

#include <cub/block/block_radix_sort.cuh>

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "mp_cuda.h"
#include "mp_kernels.cuh"

namespace mpk {

constexpr int kEuSortThreads = 1024;
#ifndef MP_EU_RADIX_BITS
#define MP_EU_RADIX_BITS 4
#endif
constexpr int kEuRadixBits = MP_EU_RADIX_BITS;  // digit width of the column radix sort
constexpr int kEuSearchThreads = 256;
constexpr int kEuMaxCtas = 1024;
constexpr size_t kEuSortSmemMax = 200 * 1024;

struct EuPart {
  DD a, b;         // sum_j P_k/k, sum_j 1/k over the active columns
  double lo, hi;   // segment bounds: max_j t_k, min_j t_{k+1}
  DD l1inf;        // phase 0: sum_j a_1
  double tmax;     // phase 0: max_j P_n
};

struct EuScratch {
  EuPart part[2][kEuMaxCtas];
  long long zero[kEuMaxCtas];
};

// Sorted-column layout.  Column j occupies [j*ld, j*ld + ld), ld = P2 (the
// sort's power of two).  Rank r (0-based, descending) of a column sorted by
// NT threads holding E keys each (thread t: ranks t*E .. t*E+E-1) lives at
// slot (r % E) * NT + r / E: the sort's stores -- and the unsorted loads --
// are coalesced across a warp (rank-contiguous stores were 32 scattered
// sectors per warp instruction).
struct EuLayout {
  int64_t ld;  // column stride (P2)
  int lge;     // log2 E
  int lgnt;    // log2 NT
  __device__ __forceinline__ int64_t slot(int64_t r) const {
    return ((r & ((1 << lge) - 1)) << lgnt) + (r >> lge);
  }
};

// ------------------------------------------------------------------- EK0
template <typename T>
__global__ void __launch_bounds__(256) k_eu_gather(const T* __restrict__ y, int64_t n, int64_t m, T* __restrict__ mags,
                                                   int64_t ld, mp_info* __restrict__ info) {
  __shared__ T tile[32][33];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32, r0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // (32, 8)
  bool bad = false;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t r = r0 + ty + k, c = c0 + tx;
    T e = T(0);
    if (r < n && c < m) {
      e = y[r * m + c];
      bad |= !isfinite(e);
    }
    tile[ty + k][tx] = fabs(e);
  }
  if (__syncthreads_or(bad) && tx == 0 && ty == 0) info->status = MP_ERR_VALUE;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int64_t c = c0 + ty + k, r = r0 + tx;
    if (r < n && c < m) mags[c * ld + r] = tile[tx][ty + k];
  }
}

// ------------------------------------------------------------------- EK1
// Bitonic sort, descending, of P2 = NT * E keys: thread t holds keys
// t*E .. t*E+E-1 in registers.  Partner distance d < E: inside the thread;
// d < 32E: the same register of lane ^ (d/E), by shuffle; larger d: one
// shared-memory round trip in an [E][NT] layout (conflict-free).  Then the
// double-double prefix sums P_k (the reference's long double,
// euclidean.cpp:41-46) over the thread-contiguous chunks: a block scan of the
// chunk totals and one more pass over the registers.
template <typename T>
__device__ __forceinline__ T tmax(T a, T b) {
  if constexpr (sizeof(T) == 4) return fmaxf(a, b);
  else return fmax(a, b);
}
template <typename T>
__device__ __forceinline__ T tmin(T a, T b) {
  if constexpr (sizeof(T) == 4) return fminf(a, b);
  else return fmin(a, b);
}
// keys are finite and >= -1 (padding): min / max are branch-free selects
template <typename T>
__device__ __forceinline__ void bitonic_keep(T& v, T o, bool take_max) {
  const T hi = tmax(v, o), lo = tmin(v, o);
  v = take_max ? hi : lo;
}

// Store the sorted column and its double-double prefix sums P_k (the
// reference's long double, euclidean.cpp:41-46): chunk totals, warp scan,
// warp totals, block offsets, one more pass over the registers.
template <typename T, int E>
__device__ __forceinline__ void eu_store_prefix(const T (&v)[E], T* __restrict__ col, DD* __restrict__ pc, int64_t n,
                                                DD* wsum) {
  const int NT = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // rank tid*E + e -> slot e*NT + tid (EuLayout)
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = tid * E + e;
    if (i < n) col[e * NT + tid] = v[e];
  }
  // prefix sums: chunk totals, warp scan, warp totals, block offsets
  DD s{0.0, 0.0};
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (tid * E + e < n) s = dd_add(s, static_cast<double>(v[e]));
  DD inc = s;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const DD w{__shfl_up_sync(0xffffffffu, inc.hi, o), __shfl_up_sync(0xffffffffu, inc.lo, o)};
    if (lane >= o) inc = dd_add(w, inc);
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    DD t = lane < (NT >> 5) ? wsum[lane] : DD{0.0, 0.0};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const DD w{__shfl_up_sync(0xffffffffu, t.hi, o), __shfl_up_sync(0xffffffffu, t.lo, o)};
      if (lane >= o) t = dd_add(w, t);
    }
    wsum[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  DD run = warp > 0 ? wsum[warp - 1] : DD{0.0, 0.0};
  const DD ex{__shfl_up_sync(0xffffffffu, inc.hi, 1), __shfl_up_sync(0xffffffffu, inc.lo, 1)};
  if (lane > 0) run = dd_add(run, ex);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = tid * E + e;
    if (i < n) {
      run = dd_add(run, static_cast<double>(v[e]));
      pc[e * NT + tid] = run;
    }
  }
}

template <typename T, int E>
__global__ void __launch_bounds__(kEuSortThreads) k_eu_sort(T* __restrict__ mags, DD* __restrict__ pref, int64_t n,
                                                            int P2, const mp_info* __restrict__ info) {
  // column stride P2 (EuLayout); the unsorted keys are read striped
  // (coalesced): the network does not care which thread starts with which key
  if (info->status != MP_OK) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sk = reinterpret_cast<T*>(smem_raw);  // [E][NT]
  __shared__ DD wsum[32];
  const int NT = blockDim.x, tid = threadIdx.x, lane = tid & 31;
  const int64_t j = blockIdx.x;
  T* col = mags + j * P2;
  T v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * NT + tid;
    v[e] = i < n ? col[i] : T(-1);  // padding sorts last
  }
  for (int k = 2; k <= P2; k <<= 1) {
    int d = k >> 1;
    for (; d >= 32 * E; d >>= 1) {  // shared memory
#pragma unroll
      for (int e = 0; e < E; ++e) sk[e * NT + tid] = v[e];
      __syncthreads();
      const int pt = tid ^ (d / E);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid * E + e;
        const bool lower = tid < pt, desc = (i & k) == 0;
        bitonic_keep(v[e], sk[e * NT + pt], lower == desc);
      }
      __syncthreads();
    }
    for (; d >= E; d >>= 1) {  // shuffles
      const int dl = d / E;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid * E + e;
        const T o = __shfl_xor_sync(0xffffffffu, v[e], dl);
        const bool lower = (lane & dl) == 0, desc = (i & k) == 0;
        bitonic_keep(v[e], o, lower == desc);
      }
    }
#pragma unroll
    for (int dd = E / 2; dd >= 1; dd >>= 1) {  // registers
      if (dd >= k) continue;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e & dd) continue;
        const int i = tid * E + e;
        const bool desc = (i & k) == 0;
        const T hi = tmax(v[e], v[e + dd]), lo = tmin(v[e], v[e + dd]);
        v[e] = desc ? hi : lo;
        v[e + dd] = desc ? lo : hi;
      }
    }
  }
  eu_store_prefix<T, E>(v, col, pref + j * P2, n, wsum);
}

// EK1 (radix): the same column sort as a CTA-wide LSD radix sort
// (cub::BlockRadixSort over the |y| bit patterns -- non-negative floats
// order like their bits; padding 0 sorts last among equals, so the first n
// sorted keys are the column's), then the same prefix pass.  Blocked
// arrangement: thread t ends with ranks t*E .. t*E+E-1, as in the bitonic
// network; sorted values are identical, so is everything downstream.
template <typename T, int NT, int E>
__global__ void __launch_bounds__(NT) k_eu_sort_radix(T* __restrict__ mags, DD* __restrict__ pref, int64_t n,
                                                      const mp_info* __restrict__ info) {
  if (info->status != MP_OK) return;
  using K = typename BitsT<T>::type;
  using Sort = cub::BlockRadixSort<K, NT, E, cub::NullType, kEuRadixBits>;
  // CUB's temp storage in dynamic shared memory (above 48 KiB for 1024 threads)
  extern __shared__ __align__(16) unsigned char eu_radix_smem[];
  typename Sort::TempStorage& tmp = *reinterpret_cast<typename Sort::TempStorage*>(eu_radix_smem);
  __shared__ DD wsum[32];
  const int tid = threadIdx.x;
  const int64_t j = blockIdx.x;
  T* col = mags + j * (NT * E);
  K key[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * NT + tid;  // striped, coalesced
    key[e] = i < n ? abs_bits(col[i]) : K(0);
  }
  // magnitudes: the sign bit is always clear, sort the low 31 / 63 bits
  Sort(tmp).SortDescending(key, 0, static_cast<int>(sizeof(K) * 8 - 1));
  T v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if constexpr (sizeof(T) == 4) v[e] = __uint_as_float(key[e]);
    else v[e] = __longlong_as_double(static_cast<long long>(key[e]));
  }
  eu_store_prefix<T, E>(v, col, pref + j * (NT * E), n, wsum);
}

// ------------------------------------------------------------------- EK2
__device__ __forceinline__ DD dd_sub(DD a, DD b) { return dd_add(a, DD{-b.hi, -b.lo}); }
// DD / k for an integer k >= 1
__device__ __forceinline__ DD dd_div_int(DD a, double k) {
  const double q = a.hi / k;
  const double r = fma(-q, k, a.hi);  // exact remainder of the leading part
  const double e = (r + a.lo) / k;
  return two_sum(q, e);
}
// DD / DD, to double
__device__ __forceinline__ double dd_div_to_double(DD a, DD b) {
  const double q = a.hi / b.hi;
  // a - q b in DD
  const double p = q * b.hi;
  const double pe = fma(q, b.hi, -p);
  DD r = dd_sub(a, DD{p, pe});
  r = dd_sub(r, DD{q * b.lo, fma(q, b.lo, -(q * b.lo))});
  return q + (r.hi + r.lo) / b.hi;
}

template <typename T>
struct EuCol {
  const T* a_;   // sorted magnitudes, descending (EuLayout slots)
  const DD* P_;  // prefix sums P_k = a_1 + ... + a_k (EuLayout slots)
  int64_t n;
  EuLayout L;
  __device__ __forceinline__ T a(int64_t r) const { return a_[L.slot(r)]; }     // a_{r+1}
  __device__ __forceinline__ DD P(int64_t r) const { return P_[L.slot(r)]; }    // P_{r+1}
  // t_k = P_k - k a_k rounded to double (euclidean.cpp:44-45), k = 1..n
  __device__ __forceinline__ double brk(int64_t k) const {
    const DD pk = P(k - 1);
    const double ak = static_cast<double>(a(k - 1)), kk = static_cast<double>(k);
    const double p = kk * ak, pe = fma(kk, ak, -p);
    const DD t = dd_sub(pk, DD{p, pe});
    return t.hi + t.lo;
  }
  __device__ __forceinline__ double total() const { const DD t = P(n - 1); return t.hi + t.lo; }
  // #{k : t_k <= theta} (the breakpoints are non-decreasing)
  __device__ __forceinline__ int64_t segment(double theta) const {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (brk(mid + 1) <= theta) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  }
};

template <typename T>
__global__ void __launch_bounds__(kEuSearchThreads)
    k_eu_search(const T* __restrict__ mags, const DD* __restrict__ pref, int64_t n, int64_t m, EuLayout lay, double eta,
                double* __restrict__ colmax, double* __restrict__ budgets, mp_info* __restrict__ info,
                EuScratch* __restrict__ sc) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  if (info->status != MP_OK) return;  // written by EK0 before this launch: uniform
  __shared__ DD dscr[32];
  __shared__ double fscr[32];
  __shared__ long long cscr[32];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int64_t j0 = static_cast<int64_t>(b) * blockDim.x + tid, js = static_cast<int64_t>(G) * blockDim.x;

  // phase 0: l1,inf norm, largest column mass, column maxima
  DD l1{0.0, 0.0};
  double tmax = 0.0;
  for (int64_t j = j0; j < m; j += js) {
    const EuCol<T> c{mags + j * lay.ld, pref + j * lay.ld, n, lay};
    const double a1 = static_cast<double>(c.a(0));
    colmax[j] = a1;
    l1 = dd_add(l1, a1);
    tmax = fmax(tmax, c.total());
  }
  l1 = block_sum_dd(l1, dscr);
  tmax = -block_min(-tmax, fscr);
  if (tid == 0) {
    sc->part[0][b].l1inf = l1;
    sc->part[0][b].tmax = tmax;
  }
  grid.sync();
  // CTA partials reduced by every CTA with the same fixed tree (thread i
  // loads partials i, i + 256, ...), so all CTAs agree bit for bit
  DD L{0.0, 0.0};
  double TM = 0.0;
  for (int i = tid; i < G; i += blockDim.x) {
    L = dd_add(L, sc->part[0][i].l1inf);
    TM = fmax(TM, sc->part[0][i].tmax);
  }
  L = block_sum_dd(L, dscr);
  TM = -block_min(-TM, fscr);
  const double l1inf = L.hi + L.lo;
  double theta;
  int iters = 0;
  int mode;  // 0 identity (budgets = column maxima), 1 zero radius, 2 clip
  if (l1inf <= eta) {
    mode = 0;
    theta = 0.0;
  } else if (eta == 0.0) {
    mode = 1;
    theta = TM;
  } else {
    mode = 2;
    theta = 0.0;
    int par = 1;
    for (iters = 1; iters <= 1 << 16; ++iters, par ^= 1) {
      DD A{0.0, 0.0}, B{0.0, 0.0};
      double lo = 0.0, hi = __longlong_as_double(0x7ff0000000000000ll);
      for (int64_t j = j0; j < m; j += js) {
        const EuCol<T> c{mags + j * lay.ld, pref + j * lay.ld, n, lay};
        const double tot = c.total();
        if (theta >= tot) continue;  // inactive column
        int64_t k = c.segment(theta);
        if (k == 0) k = 1;
        const double kd = static_cast<double>(k);
        A = dd_add(A, dd_div_int(c.P(k - 1), kd));
        B = dd_add(B, dd_div_int(DD{1.0, 0.0}, kd));
        lo = fmax(lo, c.brk(k));
        hi = fmin(hi, k < n ? c.brk(k + 1) : tot);
      }
      A = block_sum_dd(A, dscr);
      B = block_sum_dd(B, dscr);
      lo = -block_min(-lo, fscr);
      hi = block_min(hi, fscr);
      if (tid == 0) {
        EuPart& p = sc->part[par][b];
        p.a = A;
        p.b = B;
        p.lo = lo;
        p.hi = hi;
      }
      grid.sync();
      A = DD{0.0, 0.0};
      B = DD{0.0, 0.0};
      lo = 0.0;
      hi = __longlong_as_double(0x7ff0000000000000ll);
      for (int i = tid; i < G; i += blockDim.x) {
        const EuPart& p = sc->part[par][i];
        A = dd_add(A, p.a);
        B = dd_add(B, p.b);
        lo = fmax(lo, p.lo);
        hi = fmin(hi, p.hi);
      }
      A = block_sum_dd(A, dscr);
      B = block_sum_dd(B, dscr);
      lo = -block_min(-lo, fscr);
      hi = block_min(hi, fscr);
      const double tn = dd_div_to_double(dd_sub(A, DD{eta, 0.0}), B);
      if (tn <= hi || !(tn > theta)) {  // the root lies on this segment
        theta = fmin(fmax(tn, lo), hi);
        break;
      }
      theta = tn;
    }
  }

  // budgets (euclidean.cpp:143-149)
  long long zc = 0;
  for (int64_t j = j0; j < m; j += js) {
    const EuCol<T> c{mags + j * lay.ld, pref + j * lay.ld, n, lay};
    double u;
    if (mode == 0) {
      u = static_cast<double>(c.a(0));
    } else if (mode == 1 || theta >= c.total()) {
      u = 0.0;
    } else {
      int64_t k = c.segment(theta);
      if (k == 0) k = 1;
      const DD d = dd_div_int(dd_sub(c.P(k - 1), DD{theta, 0.0}), static_cast<double>(k));
      u = fmax(0.0, d.hi + d.lo);
    }
    budgets[j] = u;
    zc += u == 0.0;
  }
  zc = block_count(zc, cscr);
  if (tid == 0) sc->zero[b] = zc;
  grid.sync();
  if (b == 0 && tid == 0) {
    long long z = 0;
    for (int i = 0; i < G; ++i) z += sc->zero[i];
    info->tau = theta;
    info->iterations = iters;
    info->zero_columns = z;
    info->active = m - z;
    info->survivors = m - z;
  }
}

}  // namespace mpk
