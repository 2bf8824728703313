// mp_host.cu -- host-buffer entry points of the C-ABI (mp_*_host): the
// reference's by-value API shape (DenseTensor in, DenseTensor out;
// proj/src/bilevel.cpp:10-32 returns a fresh X) with the host<->device copies
// inside the call.  An mp_context caches device buffers (grow-only) and owns
// a non-blocking stream; calls on one context are serialised by its mutex, a
// NULL context is a thread-local default, so concurrent callers never share
// state (the reference's ThreadPool is not safe for concurrent callers,
// proj/src/parallel.cpp:49-58; ours is).
#include <cuda_runtime.h>

#include <cmath>
#include <memory>
#include <mutex>
#include <vector>

#include "mp_internal.h"

using namespace mpi;

struct mp_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // D2H of sweep results (overlaps the next projection)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  void* out2 = nullptr;  // second output buffer for the sweep ping-pong
  size_t out2_cap = 0;
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
      cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    set_error("mp_context_create: cannot create streams on device %d", device);
    delete c;
    return nullptr;
  }
  for (auto& e : c->ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
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
    if (c->out2) cudaFree(c->out2);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    for (auto& e : c->ev)
      if (e) cudaEventDestroy(e);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
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
  MP_CUDA_TRY(cudaMemcpyAsync(ctx->data, y, bytes, cudaMemcpyHostToDevice, s));
  mp_status st = mp_bilevel_project(ctx->data, ctx->data, dtype, n, m, p, q, eta, d_budgets, nullptr, d_info, flags,
                                    ctx->ws, ctx->ws_cap, s);
  if (st != MP_OK) return st;
  mp_info info{};
  MP_CUDA_TRY(cudaMemcpyAsync(&info, d_info, sizeof info, cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  st = device_status(info);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(cudaMemcpyAsync(x, ctx->data, bytes, cudaMemcpyDeviceToHost, s));
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
  MP_CUDA_TRY(cudaMemcpyAsync(ctx->data, y, bytes, cudaMemcpyHostToDevice, s));
  mp_status st = mp_euclid_project(ctx->data, ctx->data, dtype, n, m, eta, d_budgets, d_info, 0, ctx->ws, ctx->ws_cap, s);
  if (st != MP_OK) return st;
  mp_info info{};
  MP_CUDA_TRY(cudaMemcpyAsync(&info, d_info, sizeof info, cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  st = device_status(info);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(cudaMemcpyAsync(x, ctx->data, bytes, cudaMemcpyDeviceToHost, s));
  if (budgets) MP_CUDA_TRY(cudaMemcpyAsync(budgets, d_budgets, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  if (theta) *theta = info.tau;
  return MP_OK;
}

mp_status mp_bilevel_sweep_host(mp_context* ctx, const void* y, void* const* xs, mp_dtype dtype, int64_t n, int64_t m,
                                mp_norm p, mp_norm q, const double* etas, int count, double* budgets,
                                int64_t* zero_columns, unsigned flags) {
  if (!ctx) ctx = default_ctx();
  if (!ctx) return fail(MP_ERR_CUDA, "no CUDA context");
  if (count < 0 || (count > 0 && (!etas || !xs))) return fail(MP_ERR_CONFIG, "bad sweep arguments");
  if (count == 0) return MP_OK;
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const size_t ws = mp_bilevel_workspace_size(dtype, n, m, p, q);
  if (ws == 0)
    return mp_bilevel_project(y, xs[0], dtype, n, m, p, q, etas[0], nullptr, nullptr, nullptr, flags, nullptr, 0,
                              nullptr);
  for (int k = 0; k < count; ++k)
    if (!(etas[k] >= 0.0) || !std::isfinite(etas[k]))
      return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!y) return fail(MP_ERR_WORKSPACE, "null tensor pointer");
  const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(m) * dtype_size(dtype);
  const size_t per = ((static_cast<size_t>(m) * sizeof(double) + sizeof(mp_info) + 255) / 256) * 256;
  MP_CUDA_TRY(grow(ctx->data, ctx->data_cap, 2 * ((bytes + 255) / 256) * 256));  // y + out[0]
  MP_CUDA_TRY(grow(ctx->out2, ctx->out2_cap, bytes));                           // out[1]
  MP_CUDA_TRY(grow(ctx->ws, ctx->ws_cap, ws));
  MP_CUDA_TRY(grow(ctx->small, ctx->small_cap, per * static_cast<size_t>(count)));
  char* dy = static_cast<char*>(ctx->data);
  void* dout[2] = {dy + ((bytes + 255) / 256) * 256, ctx->out2};
  cudaStream_t s = ctx->stream, cs = ctx->copy_stream;
  // One upload; each projection writes a ping-pong buffer whose download on
  // the copy stream overlaps the next projection (the reference's radius
  // sweep, proj/src/bench.cpp:93-106, re-uploads nothing either).
  MP_CUDA_TRY(cudaMemcpyAsync(dy, y, bytes, cudaMemcpyHostToDevice, s));
  for (int k = 0; k < count; ++k) {
    const int b = k & 1;
    char* sm = static_cast<char*>(ctx->small) + per * k;
    if (k >= 2) MP_CUDA_TRY(cudaStreamWaitEvent(s, ctx->ev[2 + b], 0));  // buffer b downloaded
    mp_status st = mp_bilevel_project(dy, dout[b], dtype, n, m, p, q, etas[k], reinterpret_cast<double*>(sm), nullptr,
                                      reinterpret_cast<mp_info*>(sm + static_cast<size_t>(m) * sizeof(double)), flags,
                                      ctx->ws, ctx->ws_cap, s);
    if (st != MP_OK) return st;
    MP_CUDA_TRY(cudaEventRecord(ctx->ev[b], s));
    MP_CUDA_TRY(cudaStreamWaitEvent(cs, ctx->ev[b], 0));
    MP_CUDA_TRY(cudaMemcpyAsync(xs[k], dout[b], bytes, cudaMemcpyDeviceToHost, cs));
    MP_CUDA_TRY(cudaEventRecord(ctx->ev[2 + b], cs));
  }
  std::vector<mp_info> infos(static_cast<size_t>(count));
  for (int k = 0; k < count; ++k) {
    char* sm = static_cast<char*>(ctx->small) + per * k;
    MP_CUDA_TRY(cudaMemcpyAsync(&infos[k], sm + static_cast<size_t>(m) * sizeof(double), sizeof(mp_info),
                                cudaMemcpyDeviceToHost, s));
    if (budgets)
      MP_CUDA_TRY(cudaMemcpyAsync(budgets + static_cast<size_t>(k) * m, sm, static_cast<size_t>(m) * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
  }
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  MP_CUDA_TRY(cudaStreamSynchronize(cs));
  for (int k = 0; k < count; ++k) {
    mp_status st = device_status(infos[k]);
    if (st != MP_OK) return st;
    if (zero_columns) zero_columns[k] = infos[k].zero_columns;
  }
  return MP_OK;
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
  MP_CUDA_TRY(cudaMemcpyAsync(ctx->data, t, bytes, cudaMemcpyHostToDevice, s));
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
  MP_CUDA_TRY(cudaMemcpyAsync(x, ctx->data, bytes, cudaMemcpyDeviceToHost, s));
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
  MP_CUDA_TRY(cudaMemcpyAsync(din, y, bytes, cudaMemcpyHostToDevice, s));
  mp_status st = mp_project_ball(din, dout, dtype, len, q, radius, d_info, ctx->ws, ctx->ws_cap, s);
  if (st != MP_OK) return st;
  mp_info info{};
  MP_CUDA_TRY(cudaMemcpyAsync(&info, d_info, sizeof info, cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  st = device_status(info);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(cudaMemcpyAsync(x, dout, bytes, cudaMemcpyDeviceToHost, s));
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
  MP_CUDA_TRY(cudaMemcpyAsync(ctx->data, t, bytes, cudaMemcpyHostToDevice, s));
  mp_status st = mp_aggregate(ctx->data, static_cast<double*>(ctx->small), dtype, n, m, q, ctx->ws, ctx->ws_cap, s);
  if (st != MP_OK) return st;
  MP_CUDA_TRY(cudaMemcpyAsync(out, ctx->small, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  MP_CUDA_TRY(cudaStreamSynchronize(s));
  return MP_OK;
}

}  // extern "C"
