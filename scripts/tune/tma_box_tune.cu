// TMA box-shape microbenchmark: copy a 4096 x 16384 fp32 matrix through
// shared memory with cp.async.bulk.tensor only (one thread per CTA issues
// everything, one CTA per SM, a ring of 16 8-KB slots), for boxes of
// 8x256, 16x128, 32x64 and 64x32 (columns x rows) -- i.e. 32 / 64 / 128 /
// 256-byte box rows.  Tells whether TMA traffic in 32-byte strip rows (K3b's
// strips) is limited by the per-row request rate rather than by HBM.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) tma_copy(const __grid_constant__ CUtensorMap ty,
                                                  const __grid_constant__ CUtensorMap tx, int bc, int br, int n,
                                                  int m) {
  constexpr int S = 16, LAG = 4;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned long long bar[S];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int tr = n / br, tc = m / bc;
  const long long ntiles = (long long)tr * tc;
  // tile t of this CTA: column tile = (b + G * (t / tr)), row tile = t % tr (strip order)
  const long long G = gridDim.x;
  const long long mine = (tc - blockIdx.x + G - 1) / G * tr;
  auto coords = [&](long long t, int& c, int& r) {
    c = (int)((blockIdx.x + G * (t / tr)) * bc);
    r = (int)((t % tr) * br);
  };
  auto load = [&](long long t) {
    int c, r;
    coords(t, c, r);
    const int s = (int)(t % S);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(8192) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(sm + s * 8192)),
        "l"(&ty), "r"(c), "r"(r), "r"(su32(&bar[s]))
        : "memory");
  };
  for (long long t = 0; t < S && t < mine; ++t) load(t);
  for (long long t = 0; t < mine; ++t) {
    const int s = (int)(t % S);
    const unsigned ph = (unsigned)((t / S) & 1);
    asm volatile(
        "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(
            su32(&bar[s])),
        "r"(ph)
        : "memory");
    int c, r;
    coords(t, c, r);
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tx), "r"(c),
                 "r"(r), "r"(su32(sm + s * 8192))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // reload the slot stored LAG iterations ago
    const long long tr_ = t - LAG;
    if (tr_ >= 0 && tr_ + S < mine) {
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(LAG) : "memory");
      load(tr_ + S);
    }
  }
  // tail reloads
  for (long long tr_ = mine - LAG; tr_ < mine; ++tr_)
    if (tr_ >= 0 && tr_ + S < mine) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(tr_ + S);
    }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  (void)ntiles;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 4096, m = 16384;
  const size_t N = (size_t)n * m;
  float *y, *x;
  cudaMalloc(&y, N * 4);
  cudaMalloc(&x, N * 4);
  cudaMemset(y, 0, N * 4);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  Enc enc = (Enc)fn;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 8192);
  const int shapes[][2] = {{8, 256}, {16, 128}, {32, 64}, {64, 32}};
  for (auto& sh : shapes) {
    for (auto promo : {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B}) {
      CUtensorMap ty, tx;
      const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
      const cuuint64_t strides[1] = {(cuuint64_t)m * 4};
      const cuuint32_t box[2] = {(cuuint32_t)sh[0], (cuuint32_t)sh[1]};
      const cuuint32_t es[2] = {1, 1};
      enc(&ty, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      enc(&tx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int ctas_per_sm : {1}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const int grid = sms * ctas_per_sm;
        float best = 1e9f;
        for (int rep = 0; rep < 6; ++rep) {
          cudaEventRecord(a);
          tma_copy<<<grid, 32, 16 * 8192>>>(ty, tx, sh[0], sh[1], n, m);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms = 0;
          cudaEventElapsedTime(&ms, a, b);
          if (rep > 0 && ms < best) best = ms;
        }
        const cudaError_t e = cudaGetLastError();
        printf("box %2dx%3d (%3d B rows) promo %d, %d CTA/SM: %.1f us, %.0f GB/s %s\n", sh[0], sh[1], sh[0] * 4,
               (int)promo, ctas_per_sm, best * 1e3, 2.0 * N * 4 / (best * 1e-3) / 1e9,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
