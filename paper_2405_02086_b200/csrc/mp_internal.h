// mp_internal.h -- shared host-side helpers of libmp_b200 (not installed).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstddef>
#include <cstdint>
#include <string>

#include "mp_cuda.h"

namespace mpi {

// Thread-local last-error text behind mp_last_error().
void set_error(const char* fmt, ...);
const char* last_error();

inline mp_status fail(mp_status s, const char* what) {
  set_error("%s", what);
  return s;
}

inline mp_status cuda_fail(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return MP_ERR_CUDA;
}

#define MP_CUDA_TRY(expr)                                   \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return ::mpi::cuda_fail(_e, #expr); \
  } while (0)

// Bump allocator over a caller-provided workspace (256-byte aligned slices).
struct Carve {
  char* base;
  size_t cap;
  size_t off = 0;
  Carve(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <class T>
  T* take(size_t count) {
    off = (off + 255) & ~static_cast<size_t>(255);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
  bool fits() const { return off <= cap; }
};

inline size_t dtype_size(mp_dtype d) { return d == MP_F64 ? 8 : 4; }
inline bool norm_ok(int q) { return q == MP_NORM_L1 || q == MP_NORM_L2 || q == MP_NORM_INF; }
inline bool dtype_ok(int d) { return d == MP_F32 || d == MP_F64; }

int sm_count();

// Function attributes (dynamic shared memory limits, non-portable cluster
// sizes) belong to a device context.  Bit d of `done` marks device d as set
// up; f() must be idempotent (two threads may both run it for one device).
template <class F>
cudaError_t once_per_device(std::atomic<uint64_t>& done, F&& f) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (dev < 64 && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = f();
  if (e == cudaSuccess && dev < 64) done.fetch_or(bit, std::memory_order_release);
  return e;
}

}  // namespace mpi
