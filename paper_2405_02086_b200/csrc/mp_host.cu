// mp_host.cu -- host-buffer entry points of the C-ABI (mp_*_host): the
// reference's by-value API shape (DenseTensor in, DenseTensor out;
// proj/src/bilevel.cpp:10-32 returns a fresh X) with the host<->device copies
// inside the call.  An mp_context caches device buffers (grow-only) and owns
// a non-blocking stream; calls on one context are serialised by its mutex, a
// NULL context is a thread-local default, so concurrent callers never share
// state (the reference's ThreadPool is not safe for concurrent callers,
// proj/src/parallel.cpp:49-58; ours is).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "mp_internal.h"

using namespace mpi;

// One in-flight radius sweep (mp_bilevel_sweep_host_async): its own device
// copy of Y, two ping-pong outputs, per-radius budgets / info, and a pinned
// host staging copy of those.
struct SweepSlot {
  void* y = nullptr;
  size_t y_cap = 0;
  void* out[2] = {nullptr, nullptr};
  size_t out_cap[2] = {0, 0};
  void* small = nullptr;  // device: per radius [budgets (m f64) | mp_info]
  size_t small_cap = 0;
  void* h_small = nullptr;  // pinned host mirror of small
  size_t h_small_cap = 0;
  cudaEvent_t up_done = nullptr, y_free = nullptr, small_done = nullptr, done = nullptr;
  cudaEvent_t proj_done[2] = {nullptr, nullptr}, dl_done[2] = {nullptr, nullptr};
  bool used = false;      // the events above have been recorded at least once
  bool pending = false;   // results not yet collected by mp_context_wait
  uint64_t ticket = 0;
  int count = 0;
  int64_t m = 0;
  size_t per = 0;
  double* budgets = nullptr;       // caller's host outputs, filled at wait
  int64_t* zero_columns = nullptr;
};

// Host threads for the staged copies: memcpy between pageable user memory
// and the pinned staging slots, split across the caller and W workers (one
// copy on one core tops out near 10 GB/s).
class CopyPool {
 public:
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this, i] { loop(i + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // dst[0, bytes) = src[0, bytes), in parts = workers + 1 contiguous pieces
  void copy(void* dst, const void* src, size_t bytes) {
    const int parts = static_cast<int>(th_.size()) + 1;
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      parts_ = parts;
      left_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    piece(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return left_ == 0; });
  }

 private:
  void piece(int i) {
    const size_t per = (bytes_ / parts_ + 63) & ~size_t(63);
    const size_t a = std::min(bytes_, per * i), b = std::min(bytes_, per * (i + 1));
    if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      piece(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--left_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
  int parts_ = 1, left_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Pinned staging ring for pageable host tensors.  The driver stages a
// pageable cudaMemcpy through its own pinned buffer on one thread: 9.7 GB/s
// H2D and 16.7 GB/s D2H for an 800 MB f64 tensor on the B200 box.  Here host
// threads fill / drain one slot while the copy engine moves the previous one.
constexpr size_t kStageBytes = size_t(32) << 20;
constexpr int kStageSlots = 3;
constexpr size_t kStageMin = size_t(16) << 20;  // smaller copies: plain cudaMemcpyAsync

struct mp_context {
  int device = 0;
  void* stage[kStageSlots] = {};
  cudaEvent_t stage_ev[kStageSlots] = {};
  bool stage_used[kStageSlots] = {};
  std::unique_ptr<CopyPool> pool;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // D2H of sweep results (overlaps the next projection)
  cudaStream_t up_stream = nullptr;    // H2D of the next sweep's input (overlaps this sweep's D2H)
  SweepSlot slot[2];
  uint64_t next_ticket = 1;
  std::mutex mu;
  void* data = nullptr;  // tensor buffer (projected in place)
  size_t data_cap = 0;
  void* ws = nullptr;    // kernel workspace
  size_t ws_cap = 0;
  void* small = nullptr; // budgets / chain / info
  size_t small_cap = 0;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

cudaError_t grow(void*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  const size_t sz = need < 256 ? 256 : need;
  cudaError_t e = cudaMalloc(&p, sz);
  if (e == cudaSuccess) cap = sz;
  return e;
}

mp_context* default_ctx() {
  thread_local std::unique_ptr<mp_context, void (*)(mp_context*)> tl(nullptr, mp_context_destroy);
  int dev = 0;
  cudaGetDevice(&dev);
  if (!tl || tl->device != dev) tl.reset(mp_context_create(dev));
  return tl.get();
}

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

cudaError_t stage_setup(mp_context* c) {
  if (c->stage[0]) return cudaSuccess;
  for (int i = 0; i < kStageSlots; ++i) {
    cudaError_t e = cudaHostAlloc(&c->stage[i], kStageBytes, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    e = cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
  c->pool = std::make_unique<CopyPool>(static_cast<int>(std::min(7u, hw / 2)));
  return cudaSuccess;
}

// Host -> device, stream-ordered: returns with the last chunks in flight.
cudaError_t h2d(mp_context* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes < kStageMin || host_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  cudaError_t e = stage_setup(c);
  if (e != cudaSuccess) return e;
  for (size_t off = 0, k = 0; off < bytes; off += kStageBytes, ++k) {
    const int i = static_cast<int>(k % kStageSlots);
    const size_t len = std::min(kStageBytes, bytes - off);
    if (c->stage_used[i] && (e = cudaEventSynchronize(c->stage_ev[i])) != cudaSuccess) return e;
    c->pool->copy(c->stage[i], static_cast<const char*>(src) + off, len);
    if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + off, c->stage[i], len, cudaMemcpyHostToDevice, s)) !=
        cudaSuccess)
      return e;
    if ((e = cudaEventRecord(c->stage_ev[i], s)) != cudaSuccess) return e;
    c->stage_used[i] = true;
  }
  return cudaSuccess;
}

// Device -> host after everything queued on s; returns when dst is filled.
cudaError_t d2h(mp_context* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  cudaError_t e;
  if (bytes < kStageMin || host_pinned(dst)) {
    if ((e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    return cudaStreamSynchronize(s);
  }
  if ((e = stage_setup(c)) != cudaSuccess) return e;
  const size_t nchunk = (bytes + kStageBytes - 1) / kStageBytes;
  auto issue = [&](size_t k) -> cudaError_t {
    const int i = static_cast<int>(k % kStageSlots);
    const size_t off = k * kStageBytes, len = std::min(kStageBytes, bytes - off);
    cudaError_t r = cudaMemcpyAsync(c->stage[i], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s);
    if (r == cudaSuccess) r = cudaEventRecord(c->stage_ev[i], s);
    c->stage_used[i] = true;
    return r;
  };
  for (size_t k = 0; k < std::min<size_t>(kStageSlots, nchunk); ++k)
    if ((e = issue(k)) != cudaSuccess) return e;
  for (size_t k = 0; k < nchunk; ++k) {
    const int i = static_cast<int>(k % kStageSlots);
    const size_t off = k * kStageBytes, len = std::min(kStageBytes, bytes - off);
    if ((e = cudaEventSynchronize(c->stage_ev[i])) != cudaSuccess) return e;
    c->pool->copy(static_cast<char*>(dst) + off, c->stage[i], len);
    if (k + kStageSlots < nchunk && (e = issue(k + kStageSlots)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

mp_status device_status(const mp_info& info) {
  if (info.status == MP_ERR_VALUE) return fail(MP_ERR_VALUE, "non-finite tensor entry");
  if (info.status != MP_OK) return fail(static_cast<mp_status>(info.status), "device-side failure");
  return MP_OK;
}

}  // namespace

extern "C" {

mp_context* mp_context_create(int device) {
  auto* c = new mp_context();
  c->device = device;
  DeviceGuard g(device);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->up_stream, cudaStreamNonBlocking) != cudaSuccess) {
    set_error("mp_context_create: cannot create streams on device %d", device);
    delete c;
    return nullptr;
  }
  for (SweepSlot& sl : c->slot)
    for (cudaEvent_t* e : {&sl.up_done, &sl.y_free, &sl.small_done, &sl.done, &sl.proj_done[0], &sl.proj_done[1],
                           &sl.dl_done[0], &sl.dl_done[1]})
      cudaEventCreateWithFlags(e, cudaEventDisableTiming);
  return c;
}

void mp_context_destroy(mp_context* c) {
  if (!c) return;
  {
    DeviceGuard g(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->data) cudaFree(c->data);
    if (c->ws) cudaFree(c->ws);
    if (c->small) cudaFree(c->small);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    if (c->up_stream) cudaStreamSynchronize(c->up_stream);
    for (SweepSlot& sl : c->slot) {
      for (void* p : {sl.y, sl.out[0], sl.out[1], sl.small})
        if (p) cudaFree(p);
      if (sl.h_small) cudaFreeHost(sl.h_small);
      for (cudaEvent_t e : {sl.up_done, sl.y_free, sl.small_done, sl.done, sl.proj_done[0], sl.proj_done[1],
                            sl.dl_done[0], sl.dl_done[1]})
        if (e) cudaEventDestroy(e);
    }
    for (int i = 0; i < kStageSlots; ++i) {
      if (c->stage[i]) cudaFreeHost(c->stage[i]);
      if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
    }
    c->pool.reset();
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->up_stream) cudaStreamDestroy(c->up_stream);
    if (c->stream) cudaStreamDestroy(c->stream);
  }
  delete c;
}

mp_status mp_bilevel_project_host(mp_context* ctx, const void* y, void* x, mp_dtype dtype, int64_t n, int64_t m,
                                  mp_norm p, mp_norm q, double eta, double* budgets, int64_t* zero_columns,
                                  double* tau, unsigned flags) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const size_t ws = mp_bilevel_workspace_size(dtype, n, m, p, q);
  if (ws == 0) {
    // let the device entry produce the reference error
    return mp_bilevel_project(y, x, dtype, n, m, p, q, eta, nullptr, nullptr, nullptr, flags, nullptr, 0, nullptr);
  }
  if (!(eta >= 0.0) || !std::isfinite(eta)) return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!y || !x) return fail(MP_ERR_WORKSPACE, "null tensor pointer");
  const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(m) * dtype_size(dtype);
  const size_t small = static_cast<size_t>(m) * sizeof(double) + 256;
  MP_CUDA_TRY(grow(ctx->data, ctx->data_cap, bytes));
  MP_CUDA_TRY(grow(ctx->ws, ctx->ws_cap, ws));
  MP_CUDA_TRY(grow(ctx->small, ctx->small_cap, small + sizeof(mp_info)));
  double* d_budgets = static_cast<double*>(ctx->small);
  mp_info* d_info = reinterpret_cast<mp_info*>(static_cast<char*>(ctx->small) + small);
  cudaStream_t s = ctx->stream;
  MP_CUDA_TRY(h2d(ctx, ctx->data, y, bytes, s));
  mp_status st = mp_bilevel_project(ctx->data, ctx->data, dtype, n, m, p, q, eta, d_budgets, nullptr, d_info, flags,
                                    ctx->ws, ctx->ws_cap, s);
  if (st != MP_OK) return st;
  mp_info info{};
  MP_CUDA_TRY(cudaMemcpyAsync(&info, d_info, sizeof info, cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  st = device_status(info);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(d2h(ctx, x, ctx->data, bytes, s));
  if (budgets) MP_CUDA_TRY(cudaMemcpyAsync(budgets, d_budgets, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  if (zero_columns) *zero_columns = info.zero_columns;
  if (tau) *tau = info.tau;
  return MP_OK;
}

mp_status mp_euclid_project_host(mp_context* ctx, const void* y, void* x, mp_dtype dtype, int64_t n, int64_t m,
                                 double eta, double* budgets, double* theta) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const size_t ws = mp_euclid_workspace_size(dtype, n, m);
  if (ws == 0) return mp_euclid_project(y, x, dtype, n, m, eta, nullptr, nullptr, 0, nullptr, 0, nullptr);
  if (!(eta >= 0.0) || !std::isfinite(eta)) return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!y || !x) return fail(MP_ERR_WORKSPACE, "null tensor pointer");
  const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(m) * dtype_size(dtype);
  const size_t small = static_cast<size_t>(m) * sizeof(double) + 256;
  MP_CUDA_TRY(grow(ctx->data, ctx->data_cap, bytes));
  MP_CUDA_TRY(grow(ctx->ws, ctx->ws_cap, ws));
  MP_CUDA_TRY(grow(ctx->small, ctx->small_cap, small + sizeof(mp_info)));
  double* d_budgets = static_cast<double*>(ctx->small);
  mp_info* d_info = reinterpret_cast<mp_info*>(static_cast<char*>(ctx->small) + small);
  cudaStream_t s = ctx->stream;
  MP_CUDA_TRY(h2d(ctx, ctx->data, y, bytes, s));
  mp_status st = mp_euclid_project(ctx->data, ctx->data, dtype, n, m, eta, d_budgets, d_info, 0, ctx->ws, ctx->ws_cap, s);
  if (st != MP_OK) return st;
  mp_info info{};
  MP_CUDA_TRY(cudaMemcpyAsync(&info, d_info, sizeof info, cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  st = device_status(info);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(d2h(ctx, x, ctx->data, bytes, s));
  if (budgets) MP_CUDA_TRY(cudaMemcpyAsync(budgets, d_budgets, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  if (theta) *theta = info.tau;
  return MP_OK;
}

namespace {

// Collect a finished sweep: wait for its downloads, check every projection's
// device status, copy budgets / zero counts to the caller.  Caller holds mu.
mp_status collect(mp_context* ctx, SweepSlot& sl) {
  DeviceGuard g(ctx->device);
  sl.pending = false;
  MP_CUDA_TRY(cudaEventSynchronize(sl.small_done));
  MP_CUDA_TRY(cudaEventSynchronize(sl.done));
  for (int k = 0; k < sl.count; ++k) {
    const char* hs = static_cast<const char*>(sl.h_small) + sl.per * k;
    mp_info info;
    std::memcpy(&info, hs + static_cast<size_t>(sl.m) * sizeof(double), sizeof info);
    const mp_status st = device_status(info);
    if (st != MP_OK) return st;
    if (sl.zero_columns) sl.zero_columns[k] = info.zero_columns;
    if (sl.budgets) std::memcpy(sl.budgets + static_cast<size_t>(k) * sl.m, hs, static_cast<size_t>(sl.m) * sizeof(double));
  }
  return MP_OK;
}

}  // namespace

mp_status mp_bilevel_sweep_host_async(mp_context* ctx, const void* y, void* const* xs, mp_dtype dtype, int64_t n,
                                      int64_t m, mp_norm p, mp_norm q, const double* etas, int count, double* budgets,
                                      int64_t* zero_columns, unsigned flags, uint64_t* ticket) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  if (count < 0 || (count > 0 && (!etas || !xs))) return fail(MP_ERR_CONFIG, "bad sweep arguments");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const size_t ws = mp_bilevel_workspace_size(dtype, n, m, p, q);
  if (ws == 0)
    return mp_bilevel_project(y, count > 0 ? xs[0] : nullptr, dtype, n, m, p, q, count > 0 ? etas[0] : 0.0, nullptr,
                              nullptr, nullptr, flags, nullptr, 0, nullptr);
  for (int k = 0; k < count; ++k)
    if (!(etas[k] >= 0.0) || !std::isfinite(etas[k]))
      return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!y) return fail(MP_ERR_WORKSPACE, "null tensor pointer");
  const uint64_t tk = ctx->next_ticket++;
  SweepSlot& sl = ctx->slot[tk & 1];
  if (sl.pending) {  // two sweeps in flight at most: the caller skipped a wait
    const mp_status st = collect(ctx, sl);
    if (st != MP_OK) return st;
  }
  const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(m) * dtype_size(dtype);
  const size_t per = ((static_cast<size_t>(m) * sizeof(double) + sizeof(mp_info) + 255) / 256) * 256;
  if (sl.used) MP_CUDA_TRY(cudaEventSynchronize(sl.done));  // before any buffer of this slot is regrown
  MP_CUDA_TRY(grow(sl.y, sl.y_cap, bytes));
  MP_CUDA_TRY(grow(sl.out[0], sl.out_cap[0], bytes));
  MP_CUDA_TRY(grow(sl.out[1], sl.out_cap[1], bytes));
  MP_CUDA_TRY(grow(sl.small, sl.small_cap, per * static_cast<size_t>(std::max(count, 1))));
  MP_CUDA_TRY(grow(ctx->ws, ctx->ws_cap, ws));
  if (sl.h_small_cap < per * static_cast<size_t>(std::max(count, 1))) {
    if (sl.h_small) cudaFreeHost(sl.h_small);
    sl.h_small = nullptr;
    sl.h_small_cap = 0;
    MP_CUDA_TRY(cudaMallocHost(&sl.h_small, per * static_cast<size_t>(std::max(count, 1))));
    sl.h_small_cap = per * static_cast<size_t>(std::max(count, 1));
  }
  cudaStream_t s = ctx->stream, cs = ctx->copy_stream, us = ctx->up_stream;
  // upload on its own stream, once this slot's previous projections are done
  // with Y -- so it overlaps the other slot's downloads
  if (sl.used) MP_CUDA_TRY(cudaStreamWaitEvent(us, sl.y_free, 0));
  MP_CUDA_TRY(cudaMemcpyAsync(sl.y, y, bytes, cudaMemcpyHostToDevice, us));
  MP_CUDA_TRY(cudaEventRecord(sl.up_done, us));
  MP_CUDA_TRY(cudaStreamWaitEvent(s, sl.up_done, 0));
  for (int k = 0; k < count; ++k) {
    const int b = k & 1;
    char* sm = static_cast<char*>(sl.small) + per * k;
    if (k >= 2 || sl.used) MP_CUDA_TRY(cudaStreamWaitEvent(s, sl.dl_done[b], 0));  // buffer b downloaded
    const mp_status st = mp_bilevel_project(sl.y, sl.out[b], dtype, n, m, p, q, etas[k], reinterpret_cast<double*>(sm),
                                            nullptr, reinterpret_cast<mp_info*>(sm + static_cast<size_t>(m) * sizeof(double)),
                                            flags, ctx->ws, ctx->ws_cap, s);
    if (st != MP_OK) return st;
    MP_CUDA_TRY(cudaEventRecord(sl.proj_done[b], s));
    MP_CUDA_TRY(cudaStreamWaitEvent(cs, sl.proj_done[b], 0));
    MP_CUDA_TRY(cudaMemcpyAsync(xs[k], sl.out[b], bytes, cudaMemcpyDeviceToHost, cs));
    MP_CUDA_TRY(cudaEventRecord(sl.dl_done[b], cs));
  }
  MP_CUDA_TRY(cudaEventRecord(sl.y_free, s));
  if (count > 0)
    MP_CUDA_TRY(cudaMemcpyAsync(sl.h_small, sl.small, per * static_cast<size_t>(count), cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaEventRecord(sl.small_done, s));
  MP_CUDA_TRY(cudaEventRecord(sl.done, cs));
  sl.used = true;
  sl.pending = true;
  sl.ticket = tk;
  sl.count = count;
  sl.m = m;
  sl.per = per;
  sl.budgets = budgets;
  sl.zero_columns = zero_columns;
  if (ticket) *ticket = tk;
  return MP_OK;
}

mp_status mp_context_wait(mp_context* ctx, uint64_t ticket) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  for (SweepSlot& sl : ctx->slot)
    if (sl.pending && sl.ticket == ticket) return collect(ctx, sl);
  return MP_OK;  // already collected (or never issued)
}

mp_status mp_bilevel_sweep_host(mp_context* ctx, const void* y, void* const* xs, mp_dtype dtype, int64_t n, int64_t m,
                                mp_norm p, mp_norm q, const double* etas, int count, double* budgets,
                                int64_t* zero_columns, unsigned flags) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  uint64_t tk = 0;
  const mp_status st =
      mp_bilevel_sweep_host_async(ctx, y, xs, dtype, n, m, p, q, etas, count, budgets, zero_columns, flags, &tk);
  if (st != MP_OK || tk == 0) return st;
  return mp_context_wait(ctx, tk);
}

mp_status mp_multilevel_project_host(mp_context* ctx, const void* t, void* x, mp_dtype dtype, const int64_t* shape,
                                     int order, const mp_norm* levels, int depth, double eta, double* budget_chain,
                                     unsigned flags) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const size_t ws = mp_multilevel_workspace_size(dtype, shape, order, levels, depth);
  if (ws == 0)
    return mp_multilevel_project(t, x, dtype, shape, order, levels, depth, eta, nullptr, nullptr, flags, nullptr, 0,
                                 nullptr);
  if (!(eta >= 0.0) || !std::isfinite(eta)) return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!t || !x) return fail(MP_ERR_WORKSPACE, "null tensor pointer");
  size_t total = 1, chain_len = 0;
  for (int i = 0; i < order; ++i) total *= static_cast<size_t>(shape[i]);
  {
    size_t mi = 1;
    for (int i = order - 1; i >= 1; --i) {
      mi *= static_cast<size_t>(shape[i]);
      chain_len += mi;
    }
  }
  const size_t bytes = total * dtype_size(dtype);
  const size_t small = chain_len * sizeof(double) + 256;
  MP_CUDA_TRY(grow(ctx->data, ctx->data_cap, bytes));
  MP_CUDA_TRY(grow(ctx->ws, ctx->ws_cap, ws));
  MP_CUDA_TRY(grow(ctx->small, ctx->small_cap, small + sizeof(mp_info)));
  double* d_chain = static_cast<double*>(ctx->small);
  mp_info* d_info = reinterpret_cast<mp_info*>(static_cast<char*>(ctx->small) + small);
  cudaStream_t s = ctx->stream;
  MP_CUDA_TRY(h2d(ctx, ctx->data, t, bytes, s));
  // A NULL budget_chain lets the device pick the collapsed (inf, ..., inf, p) path.
  mp_status st = mp_multilevel_project(ctx->data, ctx->data, dtype, shape, order, levels, depth, eta,
                                       (budget_chain && chain_len) ? d_chain : nullptr, d_info, flags, ctx->ws,
                                       ctx->ws_cap, s);
  if (st != MP_OK) return st;
  mp_info info{};
  MP_CUDA_TRY(cudaMemcpyAsync(&info, d_info, sizeof info, cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  st = device_status(info);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(d2h(ctx, x, ctx->data, bytes, s));
  if (budget_chain && chain_len)
    MP_CUDA_TRY(cudaMemcpyAsync(budget_chain, d_chain, chain_len * sizeof(double), cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  return MP_OK;
}

mp_status mp_project_ball_host(mp_context* ctx, const void* y, void* x, mp_dtype dtype, int64_t len, mp_norm q,
                               double radius) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const size_t ws = mp_project_ball_workspace_size(dtype, len, q);
  if (ws == 0) return mp_project_ball(y, x, dtype, len, q, radius, nullptr, nullptr, 0, nullptr);
  if (!(radius >= 0.0) || !std::isfinite(radius)) return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!y || !x) return fail(MP_ERR_WORKSPACE, "null pointer");
  const size_t bytes = static_cast<size_t>(len) * dtype_size(dtype);
  MP_CUDA_TRY(grow(ctx->data, ctx->data_cap, 2 * bytes + 256));
  MP_CUDA_TRY(grow(ctx->ws, ctx->ws_cap, ws));
  MP_CUDA_TRY(grow(ctx->small, ctx->small_cap, sizeof(mp_info)));
  char* din = static_cast<char*>(ctx->data);
  char* dout = din + ((bytes + 255) & ~static_cast<size_t>(255));
  mp_info* d_info = static_cast<mp_info*>(ctx->small);
  cudaStream_t s = ctx->stream;
  MP_CUDA_TRY(h2d(ctx, din, y, bytes, s));
  mp_status st = mp_project_ball(din, dout, dtype, len, q, radius, d_info, ctx->ws, ctx->ws_cap, s);
  if (st != MP_OK) return st;
  mp_info info{};
  MP_CUDA_TRY(cudaMemcpyAsync(&info, d_info, sizeof info, cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  st = device_status(info);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(d2h(ctx, x, dout, bytes, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  return MP_OK;
}

mp_status mp_aggregate_host(mp_context* ctx, const void* t, double* out, mp_dtype dtype, int64_t n, int64_t m,
                            mp_norm q) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const size_t ws = mp_aggregate_workspace_size(dtype, n, m, q);
  if (ws == 0) return mp_aggregate(t, out, dtype, n, m, q, nullptr, 0, nullptr);
  if (!t || !out) return fail(MP_ERR_WORKSPACE, "null pointer");
  const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(m) * dtype_size(dtype);
  MP_CUDA_TRY(grow(ctx->data, ctx->data_cap, bytes));
  MP_CUDA_TRY(grow(ctx->ws, ctx->ws_cap, ws));
  MP_CUDA_TRY(grow(ctx->small, ctx->small_cap, static_cast<size_t>(m) * sizeof(double)));
  cudaStream_t s = ctx->stream;
  MP_CUDA_TRY(h2d(ctx, ctx->data, t, bytes, s));
  mp_status st = mp_aggregate(ctx->data, static_cast<double*>(ctx->small), dtype, n, m, q, ctx->ws, ctx->ws_cap, s);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(cudaMemcpyAsync(out, ctx->small, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  return MP_OK;
}

}  // extern "C"
