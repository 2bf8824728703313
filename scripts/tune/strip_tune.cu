// Strip-access microbenchmark (K3b's memory pattern without its passes):
// copy a 4096 x 16384 fp32 matrix strip by strip, each CTA holding a strip of
// W = 4P columns over all rows (thread t: 16-byte piece t % P of rows
// t / P + (NT / P) i), grid-stride over strips -- against a row-major copy.
// Tells whether K3b is bound by its passes or by the strip access pattern.
#include <cstdio>
#include <cstdint>

__global__ void flush_read(const float4* p, size_t n, float* out) {
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcs(p + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 1234.5f) *out = s;
}

// NPC pieces per thread held in registers, then stored (optionally a dummy
// compute loop of `work` passes over the registers to model the passes);
// a strip covers n rows in n / (SL * NPC) row chunks.
template <int P, int NT, int NPC>
__global__ void __launch_bounds__(NT, 1) strip_copy(const float* __restrict__ y, float* __restrict__ x, int n,
                                                    int64_t m, int64_t nstrips, int work) {
  constexpr int W = 4 * P, SL = NT / P;
  const int tid = threadIdx.x, pc = (tid % P) * 4, rb = tid / P;
  const int64_t step = (int64_t)SL * m;
  for (int64_t strip = blockIdx.x; strip < nstrips; strip += gridDim.x) {
    for (int r0 = 0; r0 < n; r0 += SL * NPC) {
      uint4 q[NPC];
      const float* yp = y + (int64_t)(r0 + rb) * m + strip * W + pc;
#pragma unroll
      for (int i = 0; i < NPC; ++i, yp += step) q[i] = __ldg(reinterpret_cast<const uint4*>(yp));
      float acc = 0.f;
      for (int w = 0; w < work; ++w)
#pragma unroll
        for (int i = 0; i < NPC; ++i) acc += __uint_as_float(q[i].x) > acc ? 1.f : 0.f;
      if (acc == -1.f) q[0].x = 0;
      __syncthreads();
      float* xp = x + (int64_t)(r0 + rb) * m + strip * W + pc;
#pragma unroll
      for (int i = 0; i < NPC; ++i, xp += step) __stcs(reinterpret_cast<uint4*>(xp), q[i]);
    }
  }
}

__global__ void row_copy(const float4* __restrict__ y, float4* __restrict__ x, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    __stcs(x + i, __ldcs(y + i));
}

int main() {
  const int n = 4096;
  const int64_t m = 16384;
  const size_t N = (size_t)n * m;
  float *y, *x, *fo;
  float4* fl;
  const size_t fln = (size_t)64 << 20;
  cudaMalloc(&y, N * 4);
  cudaMalloc(&x, N * 4);
  cudaMalloc(&fl, fln * 16);
  cudaMalloc(&fo, 4);
  cudaMemset(y, 0, N * 4);
  cudaMemset(fl, 0, fln * 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* name, auto launch) {
    float best = 1e9, tot = 0;
    for (int rep = 0; rep < 10; ++rep) {
      flush_read<<<148 * 4, 512>>>(fl, fln, fo);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep >= 2) { tot += ms; best = ms < best ? ms : best; }
    }
    printf("%-44s median-ish %.1f us  best %.1f us  (%.0f GB/s)\n", name, tot / 8 * 1e3, best * 1e3,
           2.0 * N * 4 / (best * 1e-3) / 1e9);
  };
  time("row-major copy", [&] { row_copy<<<148 * 8, 256>>>((const float4*)y, (float4*)x, N / 4); });
  // K3b config-3 geometry: 8-column strips (P = 2) over all 4096 rows, 16 warps per SM
  time("strips 8 cols (P=2) NT=512 x16, 148 CTAs", [&] { strip_copy<2, 512, 16><<<148, 512>>>(y, x, n, m, m / 8, 0); });
  time("strips 8 cols, work 4", [&] { strip_copy<2, 512, 16><<<148, 512>>>(y, x, n, m, m / 8, 4); });
  time("strips 16 cols (P=4) NT=512 x16, 148", [&] { strip_copy<4, 512, 16><<<148, 512>>>(y, x, n, m, m / 16, 0); });
  time("strips 32 cols (P=8) NT=512 x16, 148", [&] { strip_copy<8, 512, 16><<<148, 512>>>(y, x, n, m, m / 32, 0); });
  time("strips 64 cols (P=16) NT=512 x16, 148", [&] { strip_copy<16, 512, 16><<<148, 512>>>(y, x, n, m, m / 64, 0); });
  time("strips 8 cols NT=256 x16, 296 CTAs", [&] { strip_copy<2, 256, 16><<<296, 256>>>(y, x, n, m, m / 8, 0); });
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
