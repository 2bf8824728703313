// mp_l1cols.cuh -- K3b: per-column l1-ball projection at per-column radii,
// the l_{1,1} apply pass (proj/src/fiber_kernels.cpp:56-65: gather column,
// project_l1_fast_inplace at radius u_j, proj/src/vector_balls.cpp:150-161).
//
// B200 design: one WARP per column, W adjacent columns per CTA.
//  1. Stage |y| of the n x W strip once from HBM (coalesced 16-byte row
//     pieces) into shared memory, transposed to column-major (column stride
//     n + 4: conflict-free transpose stores, LDS.128 column sweeps).
//  2. Each warp runs Michelot's fixed point on its column with warp shuffles
//     only -- no CTA or cluster barrier -- and COMPACTS the active set in
//     place every pass (per thread: thread l keeps its survivors in its own
//     slots l, l+32*TW, ...; no scan, no bank conflicts), so later passes
//     touch only the survivors: ~2n element visits instead of passes * n.
//     TW = 2 warps share a column (named-barrier reduction) to double the
//     warps per SM -- occupancy is bounded by shared memory.  The
//     first iterate uses the column norm from the norm pass,
//     t1 = (v_j - u_j) / n.  Comparisons run in the staged type against RD(t)
//     (exact: for a float a, a > t <=> a > RD_float(t)); sums accumulate in
//     f64; the converged set equals the reference's {|y| >= cutoff}, so the
//     last pass's (sum, count) give tau_j = (S - u_j) / k.
//  3. The apply re-reads the strip (still L2-resident: ~30 MB of strips are
//     in flight chip-wide), forms |y| - tau_j to f64 accuracy (SURVEY.md
//     §0.4; f32 via a float-pair tau, see shrink_mag) and stores 16-byte row
//     pieces.
#pragma once

#include <cuda_runtime.h>

#include "mp_cuda.h"
#include "mp_kernels.cuh"

namespace mpk {

__device__ __forceinline__ float round_down_to(float, double t) { return __double2float_rd(t); }
__device__ __forceinline__ double round_down_to(double, double t) { return t; }

// Named barrier over the TW warps of one column group (ids 1..8; 0 is
// __syncthreads).  Immediate ids, so ptxas reserves only the barriers used
// (a register id makes it reserve all 16 and caps CTAs per SM).
template <int NTHREADS>
__device__ __forceinline__ void group_bar(int group) {
  switch (group) {
    case 0: asm volatile("bar.sync 1, %0;" ::"n"(NTHREADS) : "memory"); break;
    case 1: asm volatile("bar.sync 2, %0;" ::"n"(NTHREADS) : "memory"); break;
    case 2: asm volatile("bar.sync 3, %0;" ::"n"(NTHREADS) : "memory"); break;
    case 3: asm volatile("bar.sync 4, %0;" ::"n"(NTHREADS) : "memory"); break;
    case 4: asm volatile("bar.sync 5, %0;" ::"n"(NTHREADS) : "memory"); break;
    case 5: asm volatile("bar.sync 6, %0;" ::"n"(NTHREADS) : "memory"); break;
    case 6: asm volatile("bar.sync 7, %0;" ::"n"(NTHREADS) : "memory"); break;
    default: asm volatile("bar.sync 8, %0;" ::"n"(NTHREADS) : "memory"); break;
  }
}

// One Michelot pass over a thread-interleaved list: thread cl (of the
// column's 32*TW) owns slots cl, cl + 32*TW, ... and holds cnt of them.
// Returns the f64 sum and count of {a > thr} over the column (identical in
// every thread: warp xor-butterfly, then the TW warp partials summed in
// fixed order through double-buffered shared slots and one named barrier)
// and compacts each thread's survivors to its own first slots in place --
// no cross-thread scan, and a warp's 32 threads touch 32 distinct banks.
template <typename T, int TW>
__device__ __forceinline__ void michelot_pass(T* list, int& cnt, T thr, int cl, int group, double* rs, int* rc,
                                              int& par, double& S, int& K) {
  constexpr int kStride = 32 * TW;
  double s0 = 0.0, s1 = 0.0;
  int kept = 0;
  T* mine = list + cl;
  int j = 0;
  for (; j + 2 <= cnt; j += 2) {
    const T a0 = mine[kStride * j], a1 = mine[kStride * (j + 1)];
    const bool k0 = a0 > thr, k1 = a1 > thr;
    s0 += k0 ? static_cast<double>(a0) : 0.0;
    s1 += k1 ? static_cast<double>(a1) : 0.0;
    if (k0) mine[kStride * kept++] = a0;
    if (k1) mine[kStride * kept++] = a1;
  }
  if (j < cnt) {
    const T a0 = mine[kStride * j];
    const bool k0 = a0 > thr;
    s0 += k0 ? static_cast<double>(a0) : 0.0;
    if (k0) mine[kStride * kept++] = a0;
  }
  cnt = kept;
  double s = s0 + s1;
  int c = kept;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if constexpr (TW > 1) {
    const int wic = cl >> 5;
    if ((cl & 31) == 0) {
      rs[par * TW + wic] = s;
      rc[par * TW + wic] = c;
    }
    group_bar<kStride>(group);
    s = 0.0;
    c = 0;
#pragma unroll
    for (int k = 0; k < TW; ++k) {
      s += rs[par * TW + k];
      c += rc[par * TW + k];
    }
    par ^= 1;
  }
  S = s;
  K = c;
}

// |y| - tau for the apply pass.  f32: tau carried as a float pair
// (hi = RN(tau), lo = RN(tau - hi)); (a - hi) is exact near the threshold
// (Sterbenz) and otherwise off by < 1/2 ulp of a result >= hi, so the
// difference is correct to ~1 ulp -- the f64 subtraction's accuracy without
// leaving the FP32 pipe.  f64: plain subtraction.
struct TauPair {
  float hi, lo;
};
__device__ __forceinline__ float shrink_mag(float a, TauPair t) { return (a - t.hi) - t.lo; }

// DERIVE (bi-level hot path): u_j = derive_u(K2's OuterParams, v_j); thread 0
// of each column group writes the budget (K2 already counted zero columns).
// Occupancy is bounded by shared memory (~3 CTAs of W warps per SM), so the
// memory phases trade registers for bytes in flight: kStageBatch /
// kApplyBatch 16-byte loads per thread.
constexpr int kStageBatch = 8;

__device__ __forceinline__ void cp_async_16(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// W columns per CTA, TW warps per column (32*W*TW threads).
template <typename T, int W, int TW, bool DERIVE>
__global__ void __launch_bounds__(32 * W * TW)
    k_l1cols(const T* __restrict__ y, T* __restrict__ x, int n, int64_t m, int stride,
             const double* __restrict__ v, const double* __restrict__ u, double* __restrict__ tau_out,
             const mp_info* __restrict__ info, const OuterParams* __restrict__ params, double* __restrict__ u_out,
             mp_info* __restrict__ info_w) {
  pdl_wait();
  tl_begin(3);
  if (info->status != MP_OK) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);  // [W][stride], column-major |y|
  constexpr int NT = 32 * W * TW;
  __shared__ int skind[W];
  __shared__ double stau[W];
  __shared__ double red_s[W][2 * TW];
  __shared__ int red_c[W][2 * TW];
  const int cl = threadIdx.x % (32 * TW);  // thread index within the column group
  const int w = threadIdx.x / (32 * TW);   // column within the CTA
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * W;
  const int64_t col = c0 + w;
  const bool colok = col < m;
  const double vj = colok ? v[col] : 0.0;
  double uj;
  if constexpr (DERIVE) {
    uj = colok ? derive_u(*params, vj) : 0.0;
    if (cl == 0 && colok && u_out) u_out[col] = uj;
  } else {
    uj = colok ? u[col] : 0.0;
  }
  // 0 outside m, 1 feasible (untouched), 2 zero budget, 3 project
  const int kind = !colok ? 0 : (vj <= uj ? 1 : (uj == 0.0 ? 2 : 3));
  if (cl == 0) {
    skind[w] = kind;
    stau[w] = -1.0;
  }
  const int any_proj = __syncthreads_or(kind == 3);
  const int wcols = (m - c0) < W ? static_cast<int>(m - c0) : W;
  constexpr int kPer16 = 16 / sizeof(T);
  constexpr int kCPR = (W * sizeof(T)) / 16;  // 16-byte pieces per row (0 if W*sizeof(T) < 16)
  constexpr int kCPRv = kCPR > 0 ? kCPR : 1;
  const bool vec_ok = kCPR > 0 && wcols == W && (m % kPer16) == 0 &&
                      (reinterpret_cast<uintptr_t>(y + c0) % 16) == 0 &&
                      (reinterpret_cast<uintptr_t>(x + c0) % 16) == 0;

  const long long ck0 = clock64();
  long long ck1 = ck0, ck2 = ck0;
  if (any_proj) {
    // ---- stage |y| (16-byte pieces, 8 in flight per thread)
    if (vec_ok) {
      const int total = n * kCPRv;
      for (int b = threadIdx.x; b < total; b += kStageBatch * NT) {
        T vals[kStageBatch][kPer16];
#pragma unroll
        for (int k = 0; k < kStageBatch; ++k) {
          const int idx = b + k * NT;
          if (idx < total) {
            const int r = idx / kCPRv, part = idx % kCPRv;
            const T* src = y + static_cast<int64_t>(r) * m + c0 + part * kPer16;
            if constexpr (sizeof(T) == 4) {
              const float4 q = __ldg(reinterpret_cast<const float4*>(src));
              vals[k][0] = q.x; vals[k][1] = q.y; vals[k][2 % kPer16] = q.z; vals[k][3 % kPer16] = q.w;
            } else {
              const double2 q = __ldg(reinterpret_cast<const double2*>(src));
              vals[k][0] = q.x; vals[k][1 % kPer16] = q.y;
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kStageBatch; ++k) {
          const int idx = b + k * NT;
          if (idx < total) {
            const int r = idx / kCPRv, part = idx % kCPRv;
#pragma unroll
            for (int e = 0; e < kPer16; ++e) {
              const T a = vals[k][e];
              tile[(part * kPer16 + e) * stride + r] = a < T(0) ? -a : a;
            }
          }
        }
      }
    } else {
      for (int b = threadIdx.x; b < n * W; b += 8 * NT) {
        T vals[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int idx = b + k * NT;
          const int r = idx / W, cc = idx % W;
          vals[k] = (idx < n * W && cc < wcols) ? __ldg(y + static_cast<int64_t>(r) * m + c0 + cc) : T(0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int idx = b + k * NT;
          if (idx < n * W) tile[(idx % W) * stride + idx / W] = vals[k] < T(0) ? -vals[k] : vals[k];
        }
      }
    }
    __syncthreads();
    ck1 = clock64();

    // ---- per-column Michelot with per-thread active-set compaction
    if (kind == 3) {
      T* list = tile + w * stride;  // column-major: row r at slot r, owned by thread r % (32*TW)
      double t = (vj - uj) / static_cast<double>(n);  // Michelot's first iterate (all n entries)
      int cnt = n > cl ? (n - cl + 32 * TW - 1) / (32 * TW) : 0;
      int par = 0;
      int kprev = n;
      double S = 0.0;
      int K = 0;
      int pass_count = 0;
      for (int pass = 0; pass < 4 * 1024; ++pass) {
        double s;
        int c;
        ++pass_count;
        michelot_pass<T, TW>(list, cnt, round_down_to(T(0), t), cl, w, red_s[w], red_c[w], par, s, c);
        if (c == 0) break;  // cannot happen for 0 < u_j < v_j; keep the last set
        S = s;
        K = c;
        if (c == kprev) break;
        kprev = c;
        t = fmax(t, (s - uj) / static_cast<double>(c));
      }
      if (cl == 0) stau[w] = (S - uj) / static_cast<double>(K);
      if (cl == 0 && g_mp_timeline) {  // profiling aid: l1 pass statistics in slots 8..10
        atomicAdd(g_mp_timeline + 8, static_cast<unsigned long long>(pass_count));
        atomicMax(g_mp_timeline + 9, static_cast<unsigned long long>(pass_count));
        atomicAdd(g_mp_timeline + 10, 1ull);
      }
    }
    __syncthreads();
  }
  ck2 = clock64();
  if (cl == 0 && colok) tau_out[col] = stau[w];

  // ---- apply: re-read y (L2), write x in 16-byte row pieces
  auto out = [&](T e, int cc) -> T {
    const int k = skind[cc];
    if (k == 2) return T(0);
    if (k != 3) return e;
    const double d = fabs(static_cast<double>(e)) - stau[cc];
    return d > 0.0 ? static_cast<T>(copysign(d, static_cast<double>(e))) : T(0);
  };
  bool need_store = any_proj || x != y;
  for (int cc = 0; cc < wcols && !need_store; ++cc) need_store = skind[cc] == 2;
  if (!need_store) {
    tl_end(3);
    return;
  }
  if (vec_ok) {
    const int total = n * kCPRv;
    // NT is a multiple of kCPRv, so a thread's pieces always cover the
    // same kPer16 columns: fetch their kinds and thresholds once.
    const int part = threadIdx.x % kCPRv;
    int kk[kPer16];
    TauPair tp[kPer16];
    double td[kPer16];
#pragma unroll
    for (int e = 0; e < kPer16; ++e) {
      kk[e] = skind[part * kPer16 + e];
      td[e] = stau[part * kPer16 + e];
      tp[e].hi = __double2float_rn(td[e]);
      tp[e].lo = __double2float_rn(td[e] - static_cast<double>(tp[e].hi));
    }
    auto apply1 = [&](T v, int e) -> T {
      if (kk[e] == 2) return T(0);
      if (kk[e] != 3) return v;
      if constexpr (sizeof(T) == 4) {
        const float dm = shrink_mag(fabsf(v), tp[e]);
        return dm > 0.0f ? copysignf(dm, v) : 0.0f;
      } else {
        const double dm = fabs(v) - td[e];
        return dm > 0.0 ? copysign(dm, v) : 0.0;
      }
    };
    // The staged |y| is dead: re-land the strip row-major in the same shared
    // memory with cp.async (the whole strip in flight, no registers), then
    // every thread transforms its own 16-byte pieces.
    T* land = tile;
    if (any_proj) __syncthreads();  // all warps are done with the column lists
    for (int idx = threadIdx.x; idx < total; idx += NT) {
      const int r = idx / kCPRv;
      cp_async_16(land + static_cast<int64_t>(idx) * kPer16, y + static_cast<int64_t>(r) * m + c0 + part * kPer16);
    }
    cp_async_all();  // each thread reads back only the pieces it landed itself
    for (int idx = threadIdx.x; idx < total; idx += NT) {
      const int r = idx / kCPRv;
      T vals[kPer16];
      if constexpr (sizeof(T) == 4) {
        const float4 q = *reinterpret_cast<const float4*>(land + static_cast<int64_t>(idx) * kPer16);
        vals[0] = q.x; vals[1] = q.y; vals[2 % kPer16] = q.z; vals[3 % kPer16] = q.w;
      } else {
        const double2 q = *reinterpret_cast<const double2*>(land + static_cast<int64_t>(idx) * kPer16);
        vals[0] = q.x; vals[1 % kPer16] = q.y;
      }
#pragma unroll
      for (int e = 0; e < kPer16; ++e) vals[e] = apply1(vals[e], e);
      T* dst = x + static_cast<int64_t>(r) * m + c0 + part * kPer16;
      if constexpr (sizeof(T) == 4)
        __stcs(reinterpret_cast<float4*>(dst), make_float4(vals[0], vals[1 % kPer16], vals[2 % kPer16], vals[3 % kPer16]));
      else
        __stcs(reinterpret_cast<double2*>(dst), make_double2(vals[0], vals[1 % kPer16]));
    }
    if (threadIdx.x == 0 && g_mp_timeline) {  // profiling aid: per-phase SM cycles in slots 11..13
      const long long ck3 = clock64();
      atomicAdd(g_mp_timeline + 11, static_cast<unsigned long long>(ck1 - ck0));
      atomicAdd(g_mp_timeline + 12, static_cast<unsigned long long>(ck2 - ck1));
      atomicAdd(g_mp_timeline + 13, static_cast<unsigned long long>(ck3 - ck2));
    }
  } else {
    for (int idx = threadIdx.x; idx < n * W; idx += NT) {
      const int r = idx / W, cc = idx % W;
      if (cc >= wcols) continue;
      const int k = skind[cc];
      const int64_t g = static_cast<int64_t>(r) * m + c0 + cc;
      if (k == 2) __stcs(x + g, T(0));
      else if (k == 3 || x != y) __stcs(x + g, out(__ldcs(y + g), cc));
    }
  }
  tl_end(3);
}

}  // namespace mpk
