// mp_l1cols.cuh -- K3b: per-column l1-ball projection at per-column radii,
// the l_{1,1} apply pass (proj/src/fiber_kernels.cpp:56-65: gather column,
// project_l1_fast_inplace at radius u_j, proj/src/vector_balls.cpp:150-161).
//
// B200 design: one WARP per column.  A CTA owns W adjacent columns (W warps);
// it stages the n x W strip once from HBM (coalesced row chunks) into shared
// memory, transposed to column-major with a 16-byte-aligned column stride of
// n + 4 elements (conflict-free transpose stores, LDS.128 reads of 4
// consecutive rows per lane).  Each warp then runs Michelot's fixed point on
// its own column with nothing but warp shuffles -- no CTA or cluster
// barrier, and every column stops as soon as it converges.  The first
// iterate uses the column norm v_j from the norm pass (t_1 = (v_j - u_j)/n).
// Comparisons run on the staged type against RD(t) (exact: for a float a,
// a > t  <=>  a > RD_float(t)); sums accumulate in f64; the converged active
// set equals the reference's {|y| >= cutoff}, so the last pass's (sum, count)
// give tau_j = (S - u_j) / k; the soft threshold |y| - tau_j is formed in f64
// (SURVEY.md §0.4).  Results go back through shared memory and are stored
// with the same coalesced row-chunk pattern.
#pragma once

#include <cuda_runtime.h>

#include "mp_cuda.h"
#include "mp_kernels.cuh"

namespace mpk {

__device__ __forceinline__ float round_down_to(float, double t) { return __double2float_rd(t); }
__device__ __forceinline__ double round_down_to(double, double t) { return t; }

// DERIVE (bi-level hot path): u_j = derive_u(K2's OuterParams, v_j); lane 0
// of each warp writes the budget and accumulates zero_columns / survivors.
template <typename T, int W, bool DERIVE>
__global__ void __launch_bounds__(32 * W)
    k_l1cols(const T* __restrict__ y, T* __restrict__ x, int n, int64_t m, int stride,
             const double* __restrict__ v, const double* __restrict__ u, double* __restrict__ tau_out,
             const mp_info* __restrict__ info, const OuterParams* __restrict__ params, double* __restrict__ u_out,
             mp_info* __restrict__ info_w) {
  pdl_wait();
  tl_begin(3);
  if (info->status != MP_OK) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);  // [W][stride], column-major
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * W;
  const int64_t col = c0 + w;
  const bool colok = col < m;
  const double vj = colok ? v[col] : 0.0;
  double uj;
  if constexpr (DERIVE) {
    uj = colok ? derive_u(*params, vj) : 0.0;
    if (lane == 0 && colok) {
      if (u_out) u_out[col] = uj;
      if (uj == 0.0 || vj == 0.0) atomicAdd(reinterpret_cast<unsigned long long*>(&info_w->zero_columns), 1ull);
      if (uj != 0.0) atomicAdd(reinterpret_cast<unsigned long long*>(&info_w->survivors), 1ull);
    }
  } else {
    uj = colok ? u[col] : 0.0;
  }
  // 0 outside m, 1 feasible (untouched), 2 zero budget, 3 project
  const int kind = !colok ? 0 : (vj <= uj ? 1 : (uj == 0.0 ? 2 : 3));
  __shared__ int skind[W];
  if (lane == 0) skind[w] = kind;
  const int any_proj = __syncthreads_or(kind == 3);
  const int wcols = (m - c0) < W ? static_cast<int>(m - c0) : W;

  if (!any_proj) {  // nothing to project: copy / zero straight through
    for (int idx = threadIdx.x; idx < n * W; idx += 32 * W) {
      const int r = idx / W, cc = idx % W;
      if (cc >= wcols) continue;
      const int k = skind[cc];
      const int64_t g = static_cast<int64_t>(r) * m + c0 + cc;
      if (k == 1 && x != y) x[g] = y[g];
      else if (k == 2) x[g] = T(0);
    }
    if (lane == 0 && colok) tau_out[col] = -1.0;
    tl_end(3);
    return;
  }

  // Stage: the strip's rows are W * sizeof(T) contiguous bytes; read them in
  // 16-byte pieces (8 in flight per thread) and scatter-transpose into the
  // column-major tile.  Scalar fallback for ragged / unaligned strips.
  constexpr int kPer16 = 16 / sizeof(T);
  constexpr int kCPR = (W * sizeof(T)) / 16;  // 16-byte pieces per row (0 if W*sizeof(T) < 16)
  const bool vec_ok = kCPR > 0 && wcols == W && (m % kPer16) == 0 &&
                      (reinterpret_cast<uintptr_t>(y + c0) % 16) == 0;
  if (vec_ok) {
    constexpr int kCPRv = kCPR > 0 ? kCPR : 1;
    const int total = n * kCPRv;
    for (int base = threadIdx.x; base < total; base += 8 * 32 * W) {
      T vals[8][kPer16];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = base + k * 32 * W;
        if (idx < total) {
          const int r = idx / kCPRv, part = idx % kCPRv;
          const T* src = y + static_cast<int64_t>(r) * m + c0 + part * kPer16;
          if constexpr (sizeof(T) == 4) {
            const float4 q = __ldcs(reinterpret_cast<const float4*>(src));
            vals[k][0] = q.x; vals[k][1] = q.y; vals[k][2 % kPer16] = q.z; vals[k][3 % kPer16] = q.w;
          } else {
            const double2 q = __ldcs(reinterpret_cast<const double2*>(src));
            vals[k][0] = q.x; vals[k][1 % kPer16] = q.y;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = base + k * 32 * W;
        if (idx < total) {
          const int r = idx / kCPRv, part = idx % kCPRv;
#pragma unroll
          for (int e = 0; e < kPer16; ++e) tile[(part * kPer16 + e) * stride + r] = vals[k][e];
        }
      }
    }
  } else {
    for (int base = threadIdx.x; base < n * W; base += 8 * 32 * W) {
      T vals[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = base + k * 32 * W;
        const int r = idx / W, cc = idx % W;
        vals[k] = (idx < n * W && cc < wcols) ? __ldcs(y + static_cast<int64_t>(r) * m + c0 + cc) : T(0);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int idx = base + k * 32 * W;
        if (idx < n * W) tile[(idx % W) * stride + idx / W] = vals[k];
      }
    }
  }
  __syncthreads();

  double tau = -1.0;
  if (kind == 3) {
    T* colp = tile + w * stride;
    double t = (vj - uj) / static_cast<double>(n);  // Michelot's first iterate (all n entries)
    int kprev = n;
    double S = 0.0;
    int K = 0;
    const int n4 = n & ~127;  // rows covered by whole 128-row LDS.128 sweeps
    for (int pass = 0;; ++pass) {
      const T thr = round_down_to(T(0), t);
      double s0 = 0.0, s1 = 0.0;
      int c = 0;
      for (int i = 4 * lane; i < n4; i += 128) {
        T e[4];
        if constexpr (sizeof(T) == 4) {
          const float4 q = *reinterpret_cast<const float4*>(colp + i);
          e[0] = q.x; e[1] = q.y; e[2] = q.z; e[3] = q.w;
        } else {
          const double2 q0 = *reinterpret_cast<const double2*>(colp + i);
          const double2 q1 = *reinterpret_cast<const double2*>(colp + i + 2);
          e[0] = q0.x; e[1] = q0.y; e[2] = q1.x; e[3] = q1.y;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const T a = e[k] < T(0) ? -e[k] : e[k];
          const bool keep = a > thr;
          const double ad = keep ? static_cast<double>(a) : 0.0;
          if (k & 1) s1 += ad;
          else s0 += ad;
          c += keep;
        }
      }
      for (int i = n4 + lane; i < n; i += 32) {
        const T e = colp[i];
        const T a = e < T(0) ? -e : e;
        const bool keep = a > thr;
        s0 += keep ? static_cast<double>(a) : 0.0;
        c += keep;
      }
      double s = s0 + s1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
      }
      if (c == 0) break;  // cannot happen for 0 < u_j < v_j; keep the last set
      S = s;
      K = c;
      if (c == kprev || pass > 4 * 1024) break;
      kprev = c;
      t = fmax(t, (s - uj) / static_cast<double>(c));
    }
    tau = (S - uj) / static_cast<double>(K);
    for (int i = lane; i < n; i += 32) {
      const T e = colp[i];
      const double d = fabs(static_cast<double>(e)) - tau;
      colp[i] = d > 0.0 ? static_cast<T>(copysign(d, static_cast<double>(e))) : T(0);
    }
  }
  if (lane == 0 && colok) tau_out[col] = tau;
  __syncthreads();

  if (vec_ok) {  // 16-byte stores of whole row pieces (a piece mixes column kinds)
    constexpr int kCPRv = kCPR > 0 ? kCPR : 1;
    const int total = n * kCPRv;
    for (int idx = threadIdx.x; idx < total; idx += 32 * W) {
      const int r = idx / kCPRv, part = idx % kCPRv;
      T vals[kPer16];
      bool any = false;
#pragma unroll
      for (int e = 0; e < kPer16; ++e) {
        const int cc = part * kPer16 + e;
        const int k = skind[cc];
        vals[e] = (k == 2) ? T(0) : tile[cc * stride + r];
        any |= (k == 3 || k == 2 || (k == 1 && x != y));
      }
      if (!any) continue;
      T* dst = x + static_cast<int64_t>(r) * m + c0 + part * kPer16;
      if constexpr (sizeof(T) == 4)
        __stcs(reinterpret_cast<float4*>(dst), make_float4(vals[0], vals[1 % kPer16], vals[2 % kPer16], vals[3 % kPer16]));
      else
        __stcs(reinterpret_cast<double2*>(dst), make_double2(vals[0], vals[1 % kPer16]));
    }
  } else {
    for (int idx = threadIdx.x; idx < n * W; idx += 32 * W) {
      const int r = idx / W, cc = idx % W;
      if (cc >= wcols) continue;
      const int k = skind[cc];
      const int64_t g = static_cast<int64_t>(r) * m + c0 + cc;
      if (k == 3 || (k == 1 && x != y)) __stcs(x + g, tile[cc * stride + r]);
      else if (k == 2) __stcs(x + g, T(0));
    }
  }
  tl_end(3);
}

}  // namespace mpk
