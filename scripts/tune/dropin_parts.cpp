// Where the C++ drop-in's bilevel_project call spends its time on a 10^4 x
// 10^4 f64 DenseTensor (host side): result allocation, finiteness check of
// the result, pageable H2D / D2H, the host-buffer C-ABI call.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <vector>

#include "mp_cuda.h"

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t n = 10000, m = 10000, N = n * m;
  std::vector<double> y(N);
  for (size_t i = 0; i < N; ++i) y[i] = std::sin(0.001 * i);
  double t0 = now();
  std::vector<double> x(N);
  double t1 = now();
  bool fin = std::all_of(x.begin(), x.end(), [](double v) { return std::isfinite(v); });
  double t2 = now();
  void* d = nullptr;
  cudaMalloc(&d, N * 8);
  cudaMemcpy(d, y.data(), N * 8, cudaMemcpyHostToDevice);  // warm
  double t3 = now();
  cudaMemcpy(d, y.data(), N * 8, cudaMemcpyHostToDevice);
  double t4 = now();
  cudaMemcpy(x.data(), d, N * 8, cudaMemcpyDeviceToHost);
  double t5 = now();
  std::vector<double> b(m);
  int64_t z = 0;
  double tau = 0;
  mp_bilevel_project_host(nullptr, y.data(), x.data(), MP_F64, n, m, MP_NORM_L1, MP_NORM_INF, 100.0, b.data(), &z, &tau,
                          MP_FLAG_EXACT_ZERO_SIGN);
  double t6 = now();
  mp_bilevel_project_host(nullptr, y.data(), x.data(), MP_F64, n, m, MP_NORM_L1, MP_NORM_INF, 100.0, b.data(), &z, &tau,
                          MP_FLAG_EXACT_ZERO_SIGN);
  double t7 = now();
  std::printf("alloc+zero %.1f ms, isfinite %.1f ms (%d), H2D pageable %.1f ms (%.1f GB/s), D2H pageable %.1f ms (%.1f GB/s), host call (2nd) %.1f ms\n",
              1e3 * (t1 - t0), 1e3 * (t2 - t1), (int)fin, 1e3 * (t4 - t3), N * 8 / (t4 - t3) / 1e9, 1e3 * (t5 - t4),
              N * 8 / (t5 - t4) / 1e9, 1e3 * (t7 - t6));
  return 0;
}
