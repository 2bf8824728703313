// mp_outer_large.cuh -- K2 for vectors longer than one CTA's shared memory
// (m > kOuterMaxM = 24576): the same outer projection as k_outer
// (proj/src/vector_balls.cpp:150-191) run by a cooperative grid of all
// co-resident CTAs.  Each CTA owns a contiguous chunk; every pass writes
// per-CTA partials (double buffered), grid-syncs, and every CTA reduces the
// partials in the same fixed order, so all CTAs take identical, deterministic
// decisions.  Michelot uses a monotone threshold (active set = {|x| > t}).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "mp_kernels.cuh"

namespace mpk {

constexpr int kLargeThreads = 512;
constexpr int kLargeMaxCtas = 2048;

struct LargeScratch {
  DD dd[2][kLargeMaxCtas];
  long long cnt[2][kLargeMaxCtas];
  int bad[kLargeMaxCtas];
};

inline size_t outer_large_ws_bytes(int64_t m) {
  return m > kOuterMaxM ? sizeof(LargeScratch) : 0;
}

// Fixed-order reduce of G partials, result in every thread.
__device__ __forceinline__ DD large_reduce(const DD* part, const long long* cnt, int G, long long& ctot, DD* dscr,
                                           long long* cscr) {
  DD a{0.0, 0.0};
  long long c = 0;
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    a = dd_add(a, part[i]);
    c += cnt[i];
  }
  const DD t = block_sum_dd(a, dscr);
  ctot = block_count(c, cscr);
  return t;
}

__global__ void __launch_bounds__(kLargeThreads) k_outer_large(OuterArgs a, LargeScratch* sc) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ DD dscr[32];
  __shared__ long long cscr[32];
  __shared__ double sscr[32];
  const int G = gridDim.x, b = blockIdx.x;
  const int64_t m = a.m;
  const double eta = a.eta;
  const int64_t chunk = (m + G - 1) / G;
  const int64_t i0 = min(m, static_cast<int64_t>(b) * chunk), i1 = min(m, i0 + chunk);
  int par = 0;

  // pass 0: finiteness + total (|x| for l1, x^2 for l2)
  int bad = 0;
  DD acc{0.0, 0.0};
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double x = outer_load(a, i);
    bad |= !isfinite(x);
    acc = (a.p == kL2) ? dd_add(acc, dd_sq(x)) : dd_add(acc, fabs(x));
  }
  bad = __syncthreads_or(bad);
  acc = block_sum_dd(acc, dscr);
  if (threadIdx.x == 0) {
    sc->dd[par][b] = acc;
    sc->cnt[par][b] = 0;
    sc->bad[b] = bad;
  }
  grid.sync();
  int anybad = 0;
  for (int i = threadIdx.x; i < G; i += blockDim.x) anybad |= sc->bad[i];
  anybad = __syncthreads_or(anybad);
  if (anybad) {
    if (b == 0 && threadIdx.x == 0) {
      a.info->status = MP_ERR_VALUE;
      a.info->tau = -1.0;
      a.info->active = -1;
      a.info->iterations = 0;
    }
    return;
  }
  long long dummy;
  const DD total = large_reduce(sc->dd[par], sc->cnt[par], G, dummy, dscr, cscr);
  par ^= 1;

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
  } else if (!(dd_value(total) <= eta)) {
    if (eta == 0.0) {
      mode = 1;
      tau = 0.0;
      active = 0;
    } else {
      mode = 2;
      double t = (dd_value(total) - eta) / static_cast<double>(m);
      long long kprev = m;
      for (;;) {
        double s = 0.0;
        long long c = 0;
        for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
          const double x = fabs(outer_load(a, i));
          if (x > t) {
            s = __dadd_rn(s, x);
            ++c;
          }
        }
        block_sum_count(s, c, sscr, cscr);
        if (threadIdx.x == 0) {
          sc->dd[par][b] = DD{s, 0.0};
          sc->cnt[par][b] = c;
        }
        grid.sync();
        long long K;
        const DD S = large_reduce(sc->dd[par], sc->cnt[par], G, K, dscr, cscr);
        par ^= 1;
        ++iters;
        if (K == kprev || K == 0) break;
        t = fmax(t, (dd_value(S) - eta) / static_cast<double>(K));
        kprev = K;
      }
      double lmin = __longlong_as_double(0x7ff0000000000000ll);
      for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double x = fabs(outer_load(a, i));
        if (x > t) lmin = fmin(lmin, x);
      }
      lmin = block_min(lmin, sscr);
      if (threadIdx.x == 0) sc->dd[par][b] = DD{lmin, 0.0};
      grid.sync();
      double cutoff = __longlong_as_double(0x7ff0000000000000ll);
      for (int i = threadIdx.x; i < G; i += blockDim.x) cutoff = fmin(cutoff, sc->dd[par][i].hi);
      cutoff = block_min(cutoff, sscr);
      par ^= 1;
      DD ps{0.0, 0.0};
      long long pk = 0;
      for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double x = fabs(outer_load(a, i));
        if (x >= cutoff) {
          ps = dd_add(ps, x);
          ++pk;
        }
      }
      ps = block_sum_dd(ps, dscr);
      pk = block_count(pk, cscr);
      if (threadIdx.x == 0) {
        sc->dd[par][b] = ps;
        sc->cnt[par][b] = pk;
      }
      grid.sync();
      const DD S = large_reduce(sc->dd[par], sc->cnt[par], G, active, dscr, cscr);
      par ^= 1;
      const DD d = two_sum(S.hi, -eta);
      tau = __dadd_rn(d.hi, __dadd_rn(d.lo, S.lo)) / static_cast<double>(active);
    }
  }

  if (b == 0 && threadIdx.x == 0) outer_publish(a, mode, tau, scale);
  long long zeros = 0, surv = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double x = outer_load(a, i);
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
    zeros += (u == 0.0 || x == 0.0);
    surv += (u != 0.0);
    if (!a.emit) continue;
    a.u_out[i] = u;
    if (a.v_out) a.v_out[i] = x;
    if (a.rdrn) a.rdrn[i] = make_float2(__double2float_rz(u), __double2float_rn(u));
    if (a.factor) a.factor[i] = (x > u) ? u / x : 1.0;
  }
  zeros = block_count(zeros, cscr);
  surv = block_count(surv, cscr);
  if (threadIdx.x == 0) {
    sc->dd[par][b] = DD{static_cast<double>(surv), 0.0};
    sc->cnt[par][b] = zeros;
  }
  grid.sync();
  if (b == 0) {
    long long Z;
    const DD Sv = large_reduce(sc->dd[par], sc->cnt[par], G, Z, dscr, cscr);
    if (threadIdx.x == 0) {
      a.info->status = MP_OK;
      a.info->tau = tau;
      a.info->active = active;
      a.info->iterations = iters;
      a.info->zero_columns = Z;
      a.info->survivors = static_cast<long long>(dd_value(Sv));
    }
  }
}

inline cudaError_t launch_outer_large(const OuterArgs& a, cudaStream_t s) {
  int dev = 0, sms = 0, occ = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_outer_large, kLargeThreads, 0);
  if (e != cudaSuccess) return e;
  int G = sms * (occ < 2 ? occ : 2);
  if (G > kLargeMaxCtas) G = kLargeMaxCtas;
  if (G < 1) G = 1;
  OuterArgs args = a;
  LargeScratch* sc = static_cast<LargeScratch*>(a.scratch);
  void* params[] = {&args, &sc};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_outer_large), dim3(G), dim3(kLargeThreads),
                                     params, 0, s);
}

}  // namespace mpk
