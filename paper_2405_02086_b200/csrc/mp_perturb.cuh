// mp_perturb.cuh -- seeded Gaussian perturbation for the config-5 loop
// (BASELINE.json: "projected 100 times in a loop with a small seeded Gaussian
// perturbation (sigma = 1e-4) added between calls", the per-step projection
// of proj/src/train.cpp:191-199).  Workload harness, not the projection.
//
// Counter-based, so it is stateless, graph-replayable and reproducible:
// Philox4x32-10 keyed by (seed, iteration) on the counter (element index / 4)
// gives 4 uniforms -> 2 Box-Muller pairs -> 4 N(0,1) deviates per 4 elements.
// One 16-byte read and one write per 4 fp32 elements (HBM-bound).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mp_kernels.cuh"

namespace mpk {

struct Philox4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ Philox4 philox4x32_10(Philox4 ctr, uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(M0) * ctr.x;
    const uint64_t p1 = static_cast<uint64_t>(M1) * ctr.z;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    ctr = Philox4{hi1 ^ ctr.y ^ k0, lo1, hi0 ^ ctr.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return ctr;
}

// (0, 1] from 32 random bits (never 0, so log() is finite).
__device__ __forceinline__ float u01_open0(uint32_t b) { return (static_cast<float>(b >> 8) + 1.0f) * (1.0f / 16777216.0f); }

template <typename T, bool V4>
__global__ void __launch_bounds__(256)
    k_perturb_gaussian(T* __restrict__ x, int64_t count, float sigma, uint32_t seed_lo, uint32_t seed_hi,
                       uint32_t iteration) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  auto deviates = [&](int64_t q, float (&g)[4]) {
    const Philox4 r = philox4x32_10(Philox4{static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32), iteration, 0u},
                                    seed_lo, seed_hi);
    float s0, c0, s1, c1;
    const float r0 = sqrtf(-2.0f * __logf(u01_open0(r.x)));
    const float r1 = sqrtf(-2.0f * __logf(u01_open0(r.z)));
    __sincosf(6.2831853071795865f * u01_open0(r.y), &s0, &c0);
    __sincosf(6.2831853071795865f * u01_open0(r.w), &s1, &c1);
    g[0] = r0 * c0;
    g[1] = r0 * s0;
    g[2] = r1 * c1;
    g[3] = r1 * s1;
  };
  int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if constexpr (V4) {  // f32, 16-byte aligned, count % 4 == 0
    // four quads per thread in flight: the loads are issued before the
    // ~120 instructions of Philox and Box-Muller per quad (one load at a time
    // left the kernel at 84% of the copy rate; two in flight 394 us, four
    // 363 us, eight 415 us per GiB)
    constexpr int kU = 4;
    float4* x4 = reinterpret_cast<float4*>(x);
    for (; (q + (kU - 1) * stride) * 4 < count; q += kU * stride) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) v[u] = x4[q + u * stride];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        float g[4];
        deviates(q + u * stride, g);
        v[u].x += sigma * g[0];
        v[u].y += sigma * g[1];
        v[u].z += sigma * g[2];
        v[u].w += sigma * g[3];
        x4[q + u * stride] = v[u];
      }
    }
    for (; q * 4 < count; q += stride) {
      float g[4];
      deviates(q, g);
      float4 v = x4[q];
      v.x += sigma * g[0];
      v.y += sigma * g[1];
      v.z += sigma * g[2];
      v.w += sigma * g[3];
      x4[q] = v;
    }
  } else {
    for (; q * 4 < count; q += stride) {
      float g[4];
      deviates(q, g);
      const int64_t i0 = q * 4;
      for (int e = 0; e < 4 && i0 + e < count; ++e) x[i0 + e] = static_cast<T>(x[i0 + e] + static_cast<T>(sigma * g[e]));
    }
  }
}

}  // namespace mpk
