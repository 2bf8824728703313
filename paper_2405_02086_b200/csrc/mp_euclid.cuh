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
//  EK1 k_eu_sort_block  per column (or per run of a long column), a bitonic
//                    sorting network on the |y| bit patterns, 16 keys per
//                    thread in registers (eu_bitonic_desc), then -- for a
//                    whole column -- double-double prefix offsets every 32
//                    ranks (the reference's long double P_k,
//                    euclidean.cpp:41-46; P_k itself is re-summed from the
//                    chunk's offset);
//  EK1b k_eu_merge   columns longer than one CTA's shared memory: sorted
//                    runs merged pairwise in global memory (merge path),
//                    then k_eu_prefix writes their chunk offsets;
// Sums are deterministic (fixed trees, CTA partials reduced in CTA order).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "mp_cuda.h"
#include "mp_kernels.cuh"

namespace mpk {

constexpr int kEuSearchThreads = 256;
constexpr int kEuMaxCtas = 1024;
constexpr int kEuChunk = 32;           // ranks per double-double prefix offset
constexpr int kEuMergeThreads = 256, kEuMergeE = 8;  // merge tile: 2048 outputs

// Keys one sort CTA holds (1024 threads x 16 keys; f64: 512 x 16, by shared
// memory): longer columns are cut into runs of this length and merged.
template <typename T>
constexpr int64_t eu_sort_cap() {
  return sizeof(T) == 4 ? 16 * 1024 : 8 * 1024;
}

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

// ------------------------------------------------------------------- EK0
// 64 x 64 tiles, 256 threads, 16 elements per thread (32 x 32 tiles of 4
// per thread ran 121 us on 4096 x 16384, 68% of HBM: the grid was 65536 CTAs
// of little work each).
constexpr int kEuTile = 64;
template <typename T>
__global__ void __launch_bounds__(256) k_eu_gather(const T* __restrict__ y, int64_t n, int64_t m, T* __restrict__ mags,
                                                   int64_t ld, mp_info* __restrict__ info) {
  __shared__ T tile[kEuTile][kEuTile + 1];
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kEuTile, r0 = static_cast<int64_t>(blockIdx.y) * kEuTile;
  const int tx = threadIdx.x, ty = threadIdx.y;  // (32, 8)
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kEuTile; k += 8) {
#pragma unroll
    for (int h = 0; h < kEuTile; h += 32) {
      const int64_t r = r0 + ty + k, c = c0 + tx + h;
      T e = T(0);
      if (r < n && c < m) {
        e = y[r * m + c];
        bad |= !isfinite(e);
      }
      tile[ty + k][tx + h] = fabs(e);
    }
  }
  if (__syncthreads_or(bad) && tx == 0 && ty == 0) info->status = MP_ERR_VALUE;
#pragma unroll
  for (int k = 0; k < kEuTile; k += 8) {
#pragma unroll
    for (int h = 0; h < kEuTile; h += 32) {
      const int64_t c = c0 + ty + k, r = r0 + tx + h;
      if (r < n && c < m) mags[c * ld + r] = tile[tx + h][ty + k];
    }
  }
}

// ------------------------------------------------------------------- EK1
template <typename K>
__device__ __forceinline__ double eu_key_value(K k) {
  if constexpr (sizeof(K) == 4) return static_cast<double>(__uint_as_float(k));
  else return __longlong_as_double(static_cast<long long>(k));
}

// Double-double prefix offsets of a sorted column: offs[c] = a_0 + ... +
// a_{32c - 1} (exclusive), chunk sums by warp trees, the chunk scan by warp
// 0 (contiguous chunk ranges per lane, then a lane scan) -- fixed orders,
// deterministic.  `val(i)` reads rank i; `cs` holds >= ceil(len / 32) DDs.
__device__ __forceinline__ DD dd_sub(DD a, DD b) { return dd_add(a, DD{-b.hi, -b.lo}); }

// First breakpoint of every chunk, t_k at k = 32c + 1 (euclidean.cpp:44-45),
// from the chunk offsets: the search bisects these (a dense, L2-resident
// array) instead of re-summing prefixes.  Call after eu_scan_offsets.
template <typename V>
__device__ __forceinline__ void eu_first_breaks(V val, int64_t len, const DD* offs, double* fb) {
  __syncthreads();  // offs were written by warp 0
  const int64_t nch = (len + kEuChunk - 1) / kEuChunk;
  for (int64_t c = threadIdx.x; c < nch; c += blockDim.x) {
    const double a = val(c * kEuChunk), k = static_cast<double>(c * kEuChunk + 1);
    const DD pk = dd_add(offs[c], a);
    const double p = k * a, pe = fma(k, a, -p);
    const DD t = dd_sub(pk, DD{p, pe});
    fb[c] = t.hi + t.lo;
  }
}

// Exclusive double-double scan of nch chunk sums cs[] into offs[] by warp 0:
// contiguous chunk ranges per lane, then a lane scan (fixed orders,
// deterministic).  cs may alias offs: each entry is read before it is
// overwritten, and lanes own disjoint ranges.
__device__ __forceinline__ void eu_scan_offsets(const DD* cs, int64_t nch, DD* offs) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) != 0) return;
  const int64_t per = (nch + 31) / 32, c0 = lane * per, c1 = min(nch, c0 + per);
  DD t{0.0, 0.0};
  for (int64_t c = c0; c < c1; ++c) t = dd_add(t, cs[c]);
  DD inc = t;  // inclusive lane scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const DD w{__shfl_up_sync(0xffffffffu, inc.hi, o), __shfl_up_sync(0xffffffffu, inc.lo, o)};
    if (lane >= o) inc = dd_add(w, inc);
  }
  DD run{__shfl_up_sync(0xffffffffu, inc.hi, 1), __shfl_up_sync(0xffffffffu, inc.lo, 1)};
  if (lane == 0) run = DD{0.0, 0.0};
  for (int64_t c = c0; c < c1; ++c) {
    const DD x = cs[c];
    offs[c] = run;
    run = dd_add(run, x);
  }
}

// Double-double prefix offsets of a sorted column: offs[c] = a_0 + ... +
// a_{32c - 1} (exclusive): chunk sums by warp trees, then eu_scan_offsets.
// `val(i)` reads rank i; `cs` holds >= ceil(len / 32) DDs (may be offs).
template <typename V>
__device__ __forceinline__ void eu_prefix_offsets(V val, int64_t len, DD* cs, DD* offs) {
  const int NT = blockDim.x, NW = NT / 32, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nch = (len + kEuChunk - 1) / kEuChunk;
  for (int64_t c = warp; c < nch; c += NW) {
    const int64_t i = c * kEuChunk + lane;
    DD v{i < len ? val(i) : 0.0, 0.0};
    v = warp_reduce_dd(v);
    if (lane == 0) cs[c] = v;
  }
  __syncthreads();
  eu_scan_offsets(cs, nch, offs);
}

// EK1 for runs of up to NT * 16 keys (a whole column when n <= 16384 f32 /
// 8192 f64; longer columns in runs of that length, merged by k_eu_merge): a
// bitonic sorting
// network over the CTA, 16 keys per thread in registers, blocked (thread t
// holds positions 16t .. 16t + 15).  Every merge step of size k starts with a
// "flip" substage (position i against i ^ (k - 1)) followed by the substages
// i against i ^ j, j = k/4 .. 1, so every comparison keeps the larger key at
// the lower position: no direction flags.  A substage with j < 16 is a
// compare-exchange between two registers of a thread (42 of the 78 substages
// at 4096 keys), up to 512 positions apart one shfl.xor per key (30), further
// apart an exchange through shared memory (6).  ~150 instructions per key,
// none of them a shared-memory atomic or a scan: 4096 x 16384 f32 sorts in
// ~0.5 ms where cub::BlockRadixSort (4-bit digits, round 1) took 0.79 ms and
// an LSD radix sort of our own with warp-wide ranks 1.8 ms.  Afterwards the sorted blocked keys go through
// shared memory (one pad word per 32: conflict-free blocked writes) to
// coalesced column stores and the chunk prefix offsets.
template <typename K>
__device__ __forceinline__ K eu_shfl_xor(K v, int mask) {
  if constexpr (sizeof(K) == 4) {
    return __shfl_xor_sync(0xffffffffu, v, mask);
  } else {
    const unsigned lo = __shfl_xor_sync(0xffffffffu, static_cast<unsigned>(v), mask);
    const unsigned hi = __shfl_xor_sync(0xffffffffu, static_cast<unsigned>(v >> 32), mask);
    return (static_cast<K>(hi) << 32) | lo;
  }
}

// Larger / smaller of two keys (VIMNMX; taking the f32 maxima as floats,
// FMNMX, measured the same: both run on the ALU pipe, which bounds the
// network at 88% busy).
template <typename K>
__device__ __forceinline__ K eu_kmax(K a, K b) {
  return a > b ? a : b;
}
template <typename K>
__device__ __forceinline__ K eu_kmin(K a, K b) {
  return a > b ? b : a;
}

template <typename K, int NT>
__device__ __forceinline__ void eu_bitonic_desc(K (&key)[16], K* S) {
  constexpr int E = 16, N = NT * E;
  const int t = threadIdx.x;
  auto pad = [](int i) { return i + (i >> 5); };
  auto cmpx = [&](int lo, int hi) {  // registers lo < hi: the larger key first
    const K a = key[lo], b = key[hi];
    key[lo] = eu_kmax(a, b);
    key[hi] = eu_kmin(a, b);
  };
  // this thread's keys against v[e] from the partner thread: the thread at
  // the lower positions keeps the larger keys
  auto keep = [&](const K (&v)[E], bool lower) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const K a = key[e], b = v[e];
      const K mx = eu_kmax(a, b), mn = eu_kmin(a, b);
      key[e] = lower ? mx : mn;
    }
  };
  // partner keys through shared memory (threads of different warps); `rev`:
  // the partner's keys in reverse order (the flip substage)
  auto exchange = [&](int pt, bool rev, K (&v)[E]) {
    __syncthreads();  // the previous exchange's reads are done
#pragma unroll
    for (int e = 0; e < E; ++e) S[pad(t * E + e)] = key[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = S[pad(pt * E + (rev ? E - 1 - e : e))];
  };
  constexpr int kLogN = 31 - __builtin_clz(static_cast<unsigned>(N));
#pragma unroll
  for (int lk = 1; lk <= kLogN; ++lk) {
    const int k = 1 << lk;
    if (k <= E) {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if ((e ^ (k - 1)) > e) cmpx(e, e ^ (k - 1));
    } else {
      const int tm = k / E - 1;                     // partner thread t ^ tm, its keys reversed
      const bool lower = (t & (k / E / 2)) == 0;  // bit k/2 of the position
      K v[E];
      if (tm < 32) {
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = eu_shfl_xor(key[E - 1 - e], tm);
      } else {
        exchange(t ^ tm, true, v);
      }
      keep(v, lower);
    }
#pragma unroll
    for (int lj = lk - 2; lj >= 0; --lj) {
      const int j = 1 << lj;
      if (j < E) {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if ((e ^ j) > e) cmpx(e, e ^ j);
      } else {
        const int tj = j / E;
        const bool lower = (t & tj) == 0;
        K v[E];
        if (tj < 32) {
#pragma unroll
          for (int e = 0; e < E; ++e) v[e] = eu_shfl_xor(key[e], tj);
        } else {
          exchange(t ^ tj, false, v);
        }
        keep(v, lower);
      }
    }
  }
}

template <typename T, int NT>
struct EuBlock {
  static constexpr int E = 16;
  using K = typename BitsT<T>::type;
  // the padded keys (the sort's exchange buffer, then the sorted column),
  // then the chunk sums
  static constexpr size_t kUnion = (static_cast<size_t>(NT) * E * 33 / 32 * sizeof(K) + 15) & ~size_t(15);
  static constexpr size_t kSmem = kUnion + static_cast<size_t>(NT) * E / kEuChunk * sizeof(DD);
};

template <typename T, int NT>
__global__ void __launch_bounds__(NT) k_eu_sort_block(T* __restrict__ mags, int64_t ld, int64_t ncol, int64_t runs,
                                                      DD* __restrict__ offs, double* __restrict__ fb, int64_t ldo,
                                                      const mp_info* __restrict__ info) {
  if (info->status != MP_OK) return;
  using Cfg = EuBlock<T, NT>;
  constexpr int E = Cfg::E;
  using K = typename Cfg::K;
  extern __shared__ __align__(16) unsigned char eu_blk_smem[];
  K* S = reinterpret_cast<K*>(eu_blk_smem);
  DD* cs = reinterpret_cast<DD*>(eu_blk_smem + Cfg::kUnion);
  const int tid = threadIdx.x;
  // block b sorts run b % runs of column b / runs (runs == 1: the whole
  // column, which then also gets its chunk prefix offsets)
  const int64_t j = blockIdx.x / runs, r0 = (blockIdx.x % runs) * (static_cast<int64_t>(NT) * E);
  T* col = mags + j * ld + r0;
  const int64_t n = ncol - r0 < static_cast<int64_t>(NT) * E ? ncol - r0 : static_cast<int64_t>(NT) * E;
  K key[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = e * NT + tid;  // striped, coalesced
    key[e] = i < n ? abs_bits(col[i]) : K(0);  // padding: 0 sorts last
  }
  // (the unsorted keys' arrangement does not matter: taken as blocked)
  eu_bitonic_desc<K, NT>(key, S);
  __syncthreads();  // the last exchange's reads are done: S takes the sorted keys
  auto pad = [](int i) { return i + (i >> 5); };
  // chunk sums straight from the registers: thread t holds ranks 16t ..
  // 16t + 15 (padding keys are 0), chunk c = threads 2c, 2c + 1
  DD part{0.0, 0.0};
#pragma unroll
  for (int e = 0; e < E; ++e) {
    S[pad(tid * E + e)] = key[e];
    part = dd_add(part, eu_key_value(key[e]));
  }
  const DD other{__shfl_xor_sync(0xffffffffu, part.hi, 1), __shfl_xor_sync(0xffffffffu, part.lo, 1)};
  if ((tid & 1) == 0) cs[tid >> 1] = dd_add(part, other);
  __syncthreads();
  for (int i = tid; i < n; i += NT) {
    if constexpr (sizeof(T) == 4) col[i] = __uint_as_float(S[pad(i)]);
    else col[i] = __longlong_as_double(static_cast<long long>(S[pad(i)]));
  }
  if (runs != 1) return;  // merged columns: k_eu_prefix writes the offsets
  eu_scan_offsets(cs, (n + kEuChunk - 1) / kEuChunk, offs + j * ldo);
  eu_first_breaks([&](int64_t i) { return eu_key_value(S[pad(static_cast<int>(i))]); }, n, offs + j * ldo,
                  fb + j * ldo);
}

// EK1b: merge pairs of sorted (descending) runs of width w into dst: each
// thread finds its output diagonal's split by a binary search (merge path,
// ties taken from the first run: stable) and merges kEuMergeE outputs.
template <typename T>
__global__ void __launch_bounds__(kEuMergeThreads) k_eu_merge(const T* __restrict__ src, T* __restrict__ dst,
                                                              int64_t ld, int64_t n, int64_t w,
                                                              const mp_info* __restrict__ info) {
  if (info->status != MP_OK) return;
  const int64_t j = blockIdx.y;
  const T* s = src + j * ld;
  T* d = dst + j * ld;
  const int64_t p0 = (static_cast<int64_t>(blockIdx.x) * kEuMergeThreads + threadIdx.x) * kEuMergeE;
  if (p0 >= n) return;
  const int64_t lo = (p0 / (2 * w)) * (2 * w);
  const int64_t la = min(w, n - lo), lb = max(int64_t(0), min(w, n - lo - w));
  const T* a = s + lo;
  const T* b = a + la;
  const int64_t diag = p0 - lo;
  int64_t ilo = max(int64_t(0), diag - lb), ihi = min(diag, la);
  while (ilo < ihi) {
    const int64_t mid = (ilo + ihi) >> 1;
    if (a[mid] >= b[diag - 1 - mid]) ilo = mid + 1;
    else ihi = mid;
  }
  int64_t i = ilo, k = diag - ilo;
  const int64_t end = min(p0 + kEuMergeE, lo + la + lb);
  for (int64_t p = p0; p < end; ++p) {
    if (i < la && (k >= lb || a[i] >= b[k])) d[p] = a[i++];
    else d[p] = b[k++];
  }
}

// Prefix offsets of merged (long) columns: one CTA per column; the chunk
// sums are staged in offs itself (the scan reads each before overwriting it).
template <typename T>
__global__ void __launch_bounds__(256) k_eu_prefix(const T* __restrict__ mags, int64_t ld, int64_t n,
                                                   DD* __restrict__ offs, double* __restrict__ fb, int64_t ldo,
                                                   const mp_info* __restrict__ info) {
  if (info->status != MP_OK) return;
  const int64_t j = blockIdx.x;
  const T* col = mags + j * ld;
  eu_prefix_offsets([&](int64_t i) { return static_cast<double>(col[i]); }, n, offs + j * ldo, offs + j * ldo);
  eu_first_breaks([&](int64_t i) { return static_cast<double>(col[i]); }, n, offs + j * ldo, fb + j * ldo);
}

// ------------------------------------------------------------------- EK2
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
  const T* a_;      // sorted magnitudes, descending, rank-contiguous
  const DD* off;    // off[c] = a_0 + ... + a_{32c-1}
  const double* fb; // fb[c] = t_{32c+1}, the chunk's first breakpoint
  int64_t n;
  __device__ __forceinline__ T a(int64_t r) const { return a_[r]; }  // a_{r+1}
  // P_{r+1} = a_1 + ... + a_{r+1}: the chunk's offset plus its ranks up to r
  __device__ __forceinline__ DD P(int64_t r) const {
    const int64_t c0 = r & ~int64_t(kEuChunk - 1);
    DD s = off[c0 / kEuChunk];
    for (int64_t i = c0; i <= r; ++i) s = dd_add(s, static_cast<double>(a_[i]));
    return s;
  }
  __device__ __forceinline__ double brk_from_a(DD pk, int64_t k, double ak) const {  // t_k from P_k, a_k
    const double kk = static_cast<double>(k);
    const double p = kk * ak, pe = fma(kk, ak, -p);
    const DD t = dd_sub(pk, DD{p, pe});
    return t.hi + t.lo;
  }
  __device__ __forceinline__ double brk_from(DD pk, int64_t k) const {  // t_k from P_k
    const double ak = static_cast<double>(a(k - 1)), kk = static_cast<double>(k);
    const double p = kk * ak, pe = fma(kk, ak, -p);
    const DD t = dd_sub(pk, DD{p, pe});
    return t.hi + t.lo;
  }
  // t_k = P_k - k a_k rounded to double (euclidean.cpp:44-45), k = 1..n
  __device__ __forceinline__ double brk(int64_t k) const { return brk_from(P(k - 1), k); }
  __device__ __forceinline__ double total() const { const DD t = P(n - 1); return t.hi + t.lo; }
  // The linear segment of u(theta) holding theta: k = #{k : t_k <= theta}
  // (>= 1: t_1 = 0 <= theta), P_k, t_k and the segment's end t_{k+1} (P_n
  // for k = n).  A binary search over the chunks' first breakpoints (the
  // breakpoints are non-decreasing), then one walk inside the chunk that
  // carries P_k along (euclidean.cpp:19-26 bisects all n breakpoints).
  struct Seg {
    int64_t k;
    DD pk;
    double tk, tk1;
  };
  __device__ __forceinline__ Seg segment(double theta) const {
    const int64_t nch = (n + kEuChunk - 1) / kEuChunk;
    int64_t lo = 1, hi = nch;  // chunks [0, lo) start at or below theta (chunk 0: t_1 = 0)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (fb[mid] <= theta) lo = mid + 1;
      else hi = mid;
    }
    const int64_t k0 = (lo - 1) * kEuChunk + 1;
    // the chunk's ranks and the next chunk's first, loaded up front (one
    // line; the walk below would otherwise wait on each load in turn)
    double v[kEuChunk + 1];
#pragma unroll
    for (int i = 0; i <= kEuChunk; ++i) v[i] = k0 - 1 + i < n ? static_cast<double>(a_[k0 - 1 + i]) : 0.0;
    Seg r{k0, dd_add(off[lo - 1], v[0]), 0.0, 0.0};
    r.tk = brk_from_a(r.pk, k0, v[0]);
    r.tk1 = -1.0;
#pragma unroll
    for (int i = 1; i <= kEuChunk; ++i) {  // up to the next chunk's first (> theta)
      const int64_t k = k0 + i;
      if (k > n) break;
      const DD pn = dd_add(r.pk, v[i]);
      const double tn = brk_from_a(pn, k, v[i]);
      if (tn > theta) {
        r.tk1 = tn;
        break;
      }
      r.k = k;
      r.pk = pn;
      r.tk = tn;
    }
    if (r.tk1 < 0.0) r.tk1 = r.k == n ? r.pk.hi + r.pk.lo : brk(r.k + 1);  // k = n: the segment ends at P_n
    return r;
  }
  // The same segment found by a whole warp (every lane calls with the same
  // column and theta, every lane gets the result): a 32-way search over the
  // chunks' first breakpoints (two dependent loads for up to 1024 chunks
  // instead of a bisection's ten), the chunk's 32 ranks in one coalesced
  // load, P_k by a double-double warp scan and one ballot over the
  // breakpoints -- a few hundred cycles where the one-thread walk is a chain
  // of up to 32 dependent double-double additions.
  __device__ __forceinline__ Seg segment_warp(double theta, int lane) const {
    const int64_t nch = (n + kEuChunk - 1) / kEuChunk;
    int64_t lo = 1, hi = nch;  // chunks [0, lo) start at or below theta, chunks [hi, nch) above it
    while (lo < hi) {
      const int64_t step = (hi - lo + 31) / 32, idx = lo + lane * step;
      const bool p = idx < hi && fb[idx] <= theta;  // non-decreasing: a prefix of the lanes
      const int cnt = __popc(__ballot_sync(0xffffffffu, p));
      const int64_t nlo = cnt > 0 ? lo + static_cast<int64_t>(cnt - 1) * step + 1 : lo;
      const int64_t nhi = lo + static_cast<int64_t>(cnt) * step < hi ? lo + static_cast<int64_t>(cnt) * step : hi;
      lo = nlo;
      hi = nhi;
    }
    const int64_t c0 = lo - 1, k0 = c0 * kEuChunk + 1, ki = k0 + lane;  // lane i: rank k0 + i
    const double vi = ki <= n ? static_cast<double>(a_[ki - 1]) : 0.0;
    DD pi{vi, 0.0};  // inclusive double-double scan of the chunk's ranks
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const DD q{__shfl_up_sync(0xffffffffu, pi.hi, o), __shfl_up_sync(0xffffffffu, pi.lo, o)};
      if (lane >= o) pi = dd_add(q, pi);
    }
    pi = dd_add(off[c0], pi);
    const double ti = ki <= n ? brk_from_a(pi, ki, vi) : 0.0;
    const int cnt = __popc(__ballot_sync(0xffffffffu, ki <= n && ti <= theta));  // >= 1: t_{k0} <= theta
    const int src = cnt > 0 ? cnt - 1 : 0;
    Seg r;
    r.k = k0 + src;
    r.pk = DD{__shfl_sync(0xffffffffu, pi.hi, src), __shfl_sync(0xffffffffu, pi.lo, src)};
    r.tk = __shfl_sync(0xffffffffu, ti, src);
    const double tnext = __shfl_sync(0xffffffffu, ti, src + 1 < 32 ? src + 1 : 31);
    if (r.k == n) r.tk1 = r.pk.hi + r.pk.lo;  // the segment ends at P_n
    else if (src + 1 < 32) r.tk1 = tnext;
    else r.tk1 = fb[c0 + 1];  // the next chunk's first breakpoint
    return r;
  }
  // P_n by a warp
  __device__ __forceinline__ double total_warp(int lane) const {
    const int64_t c0 = (n - 1) / kEuChunk, ki = c0 * kEuChunk + 1 + lane;
    DD v{ki <= n ? static_cast<double>(a_[ki - 1]) : 0.0, 0.0};
    v = warp_reduce_dd(v);
    const DD t = dd_add(off[c0], v);
    return t.hi + t.lo;
  }
};

// WARP: one warp per column (segment_warp) -- up to a few thousand columns
// the search is a latency chain and the warp version is ~3x shorter (1000 x
// 1000: 130 -> 93 us for the whole projection); beyond that the thread per
// column wins, the warp scan issues ~6x the double-double arithmetic
// (4096 x 16384: 176 vs 265 us).
template <typename T, bool WARP>
__global__ void __launch_bounds__(kEuSearchThreads)
    k_eu_search(const T* __restrict__ mags, const DD* __restrict__ offs, const double* __restrict__ fbs, int64_t n,
                int64_t m, int64_t ld, int64_t ldo,
                double eta, double* __restrict__ colmax, double* __restrict__ budgets, double* __restrict__ coltot,
                mp_info* __restrict__ info, EuScratch* __restrict__ sc) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  if (info->status != MP_OK) return;  // written by EK0 before this launch: uniform
  __shared__ DD dscr[32];
  __shared__ double fscr[32];
  __shared__ long long cscr[32];
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  // WARP: columns strided over the grid's warps, lane 0 carries the warp's
  // partial sums into the block reductions; else over its threads
  const int64_t j0 = WARP ? static_cast<int64_t>(b) * (blockDim.x / 32) + (tid >> 5)
                          : static_cast<int64_t>(b) * blockDim.x + tid,
                js = WARP ? static_cast<int64_t>(G) * (blockDim.x / 32) : static_cast<int64_t>(G) * blockDim.x;
  const bool lead = !WARP || lane == 0;  // the thread that carries the column's results

  // phase 0: l1,inf norm, largest column mass, column maxima
  DD l1{0.0, 0.0};
  double tmax = 0.0;
  for (int64_t j = j0; j < m; j += js) {
    const EuCol<T> c{mags + j * ld, offs + j * ldo, fbs + j * ldo, n};
    const double a1 = static_cast<double>(c.a(0));
    const double tot = WARP ? c.total_warp(lane) : c.total();
    if (lead) {
      colmax[j] = a1;
      l1 = dd_add(l1, a1);
      coltot[j] = tot;  // P_n, read back by every Newton step
      tmax = fmax(tmax, tot);
    }
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
        if (theta >= coltot[j]) continue;  // inactive column
        const EuCol<T> c{mags + j * ld, offs + j * ldo, fbs + j * ldo, n};
        const typename EuCol<T>::Seg g = WARP ? c.segment_warp(theta, lane) : c.segment(theta);
        if (lead) {
          const double kd = static_cast<double>(g.k);
          A = dd_add(A, dd_div_int(g.pk, kd));
          B = dd_add(B, dd_div_int(DD{1.0, 0.0}, kd));
          lo = fmax(lo, g.tk);
          hi = fmin(hi, g.tk1);
        }
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
    const EuCol<T> c{mags + j * ld, offs + j * ldo, fbs + j * ldo, n};
    double u;
    if (mode == 0) {
      u = static_cast<double>(c.a(0));
    } else if (mode == 1 || theta >= coltot[j]) {
      u = 0.0;
    } else {
      const typename EuCol<T>::Seg g = WARP ? c.segment_warp(theta, lane) : c.segment(theta);
      const DD d = dd_div_int(dd_sub(g.pk, DD{theta, 0.0}), static_cast<double>(g.k));
      u = fmax(0.0, d.hi + d.lo);
    }
    if (lead) {
      budgets[j] = u;
      zc += u == 0.0;
    }
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
