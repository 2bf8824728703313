// mp_device.cu -- device entry points of the C-ABI (include/mp_cuda.h):
// argument validation (reference exception taxonomy), workspace carving,
// grid planning and kernel dispatch.  No allocation, no host sync: every
// entry point is stream-ordered and CUDA-graph capturable.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <vector>

#include "mp_internal.h"
#include "mp_euclid.cuh"
#include "mp_kernels.cuh"
#include "mp_l1strip.cuh"
#include "mp_outer_large.cuh"
#include "mp_perturb.cuh"

namespace mpi {

static thread_local std::string g_err;
static thread_local cudaEvent_t g_prof[4] = {nullptr, nullptr, nullptr, nullptr};

void prof_mark(int i, cudaStream_t s) {
  if (!g_prof[i]) return;
  // Inside stream capture, record an EXTERNAL event node so the event stays
  // usable for timing after every graph replay.
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(g_prof[i], s, cudaEventRecordExternal);
  else cudaEventRecord(g_prof[i], s);
}

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

const char* last_error() { return g_err.c_str(); }

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

}  // namespace mpi

using namespace mpi;

namespace {

// ----------------------------------------------------------- grid planning
constexpr int kRowInterleave = 1;  // see mpk::row_walk: the grid sweeps HBM band by band
// K1 row blocks hold >= 16 rows: short matrices otherwise pile one atomic /
// partial per row onto every column (1000x1000: K1 9.9 -> 4.4 us); K3 keeps 4.
constexpr int64_t kK1MinRows = 16;

struct Grid {
  int vec = 1;
  int threads = 32;
  int64_t ntiles = 1;  // column tiles (grid.x)
  int64_t nrb = 1;     // row blocks (grid.y)
  int64_t rpb = 1;     // rows per block
};

// Balanced column tiles: the fewest tiles of <= 256 threads, all the same
// width (m = 10000, VEC = 4: 10 tiles of 250 threads), so no CTA is short.
int threads_for(int vec, int64_t m) {
  const int64_t slots = (m + vec - 1) / vec;
  const int64_t tiles = (slots + mpk::kThreads - 1) / mpk::kThreads;
  return static_cast<int>((slots + tiles - 1) / tiles);
}

// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor drains and synchronises with
// griddepcontrol.wait before touching the predecessor's outputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, static_cast<KArgs>(args)...);
}

// One resident wave: grid.y = floor(SMs * occupancy / column tiles) row
// blocks, so every CTA starts at once and none trails in a second wave (a
// 1.005-wave grid costs a whole extra CTA lifetime).  Each thread keeps U
// 16-byte loads in flight; at full occupancy that is >= 128 KiB per SM, well
// above the ~35 KiB Little's law asks of HBM3e.
Grid plan_grid(int vec, int64_t n, int64_t m, int ctas_per_sm, int64_t min_rows = 4) {
  Grid g;
  g.vec = vec;
  g.threads = threads_for(vec, m);
  const int64_t slots = (m + vec - 1) / vec;
  g.ntiles = (slots + g.threads - 1) / g.threads;
  const int64_t resident = static_cast<int64_t>(sm_count()) * std::max(1, ctas_per_sm);
  int64_t nrb = std::max<int64_t>(1, resident / g.ntiles);
  nrb = std::min<int64_t>(nrb, std::max<int64_t>(1, (n + min_rows - 1) / min_rows));
  nrb = std::min<int64_t>(nrb, 65535);
  g.rpb = (n + nrb - 1) / nrb;
  g.nrb = (n + g.rpb - 1) / g.rpb;
  return g;
}


// Occupancy of one kernel instantiation (cached per function and block size).
int occupancy(const void* fn, int threads) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> cache;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& e : cache)
    if (e.first.first == fn && e.first.second == threads) return e.second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, 0) != cudaSuccess || occ < 1) occ = 1;
  cache.push_back({{fn, threads}, occ});
  return occ;
}

int pick_vec(mp_dtype dt, int64_t m, const void* a, const void* b) {
  const uintptr_t al = reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b);
  // 16-byte packs: measured on B200 (scripts/tune), 16-byte LDG at full
  // occupancy streams faster than 256-bit LDG at the lower occupancy its
  // register footprint allows (K1 64 us vs 74 us on 400 MB).
  if (dt == MP_F32) {
    if (m % 4 == 0 && al % 16 == 0) return 4;
    if (m % 2 == 0 && al % 8 == 0) return 2;
    return 1;
  }
  if (m % 2 == 0 && al % 16 == 0) return 2;
  return 1;
}

// Upper bound of the K1 row-block count over every vector width and any
// occupancy (sizes the l1/l2 partials in the workspace).
int64_t max_nrb(mp_dtype dt, int64_t n, int64_t m) {
  int64_t r = 1;
  for (int v : {1, 2, 4, 8}) {
    if (dt == MP_F64 && v == 8) continue;
    const int t = threads_for(v, m);
    r = std::max(r, plan_grid(v, n, m, std::min(32, 2048 / t), kK1MinRows).nrb);
  }
  return r;
}

// --------------------------------------------------------------- dispatch
// K1 and K3 each run one resident wave at their own occupancy.  Rows are
// interleaved across the grid (kRowInterleave), so both kernels sweep HBM
// band by band and K3's reverse sweep starts on the bands K1 read last --
// still in L2 -- whatever the two grids are.
// Row groups per K1 CTA: narrow matrices stack row groups (up to 1024
// threads) so each column gets one atomic / partial per CTA.
inline int k1_row_groups(int tx) { return tx >= 128 ? 1 : std::min(16, 1024 / tx); }

template <typename T, int VEC, int Q, bool RG>
cudaError_t launch_colnorm_rg(int64_t n, int64_t m, const T* y, void* out, Grid& g, cudaStream_t s, int ncopy) {
  constexpr int U = (sizeof(T) * VEC == 32) ? 4 : 8;  // 128 bytes of loads in flight per thread
  auto fn = mpk::k_colnorm<T, VEC, Q, U, RG>;
  const int tx = threads_for(VEC, m);
  const int ty = RG ? k1_row_groups(tx) : 1;
  const size_t smem = ty > 1 ? static_cast<size_t>(ty) * tx * VEC * 8 : 0;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessorWithFlags(&occ, fn, tx * ty, smem, 0) != cudaSuccess || occ < 1)
    occ = 1;
  g = plan_grid(VEC, n, m, occ, kK1MinRows);  // g.nrb = CTA rows; row slots = g.nrb * ty
  const int64_t slots = g.nrb * ty;
  const int64_t rpb = kRowInterleave ? n / slots : (n + slots - 1) / slots;
  dim3 grid(static_cast<unsigned>(g.ntiles), static_cast<unsigned>(g.nrb));
  fn<<<grid, dim3(tx, ty), smem, s>>>(y, n, m, rpb, kRowInterleave, out, ncopy);
  return cudaGetLastError();
}

template <typename T, int VEC, int Q>
cudaError_t launch_colnorm_q(int64_t n, int64_t m, const T* y, void* out, Grid& g, cudaStream_t s, int ncopy) {
  if (k1_row_groups(threads_for(VEC, m)) > 1) return launch_colnorm_rg<T, VEC, Q, true>(n, m, y, out, g, s, ncopy);
  return launch_colnorm_rg<T, VEC, Q, false>(n, m, y, out, g, s, ncopy);
}

template <typename T, int VEC>
cudaError_t launch_colnorm_v(int q, const T* y, int64_t n, int64_t m, void* out, Grid& g, cudaStream_t s,
                             int ncopy) {
  if (q == mpk::kInf) return launch_colnorm_q<T, VEC, mpk::kInf>(n, m, y, out, g, s, ncopy);
  if (q == mpk::kL1) return launch_colnorm_q<T, VEC, mpk::kL1>(n, m, y, out, g, s, 1);
  return launch_colnorm_q<T, VEC, mpk::kL2>(n, m, y, out, g, s, 1);
}

// K1; `g` returns the grid used (g.nrb = number of l1/l2 partial rows).
template <typename T>
cudaError_t launch_colnorm(int q, int vec, const T* y, int64_t n, int64_t m, void* out, Grid& g, cudaStream_t s,
                           int ncopy = 1) {
  if (vec == 8) {
    if constexpr (sizeof(T) == 4) return launch_colnorm_v<T, 8>(q, y, n, m, out, g, s, ncopy);
  }
  if (vec == 4) return launch_colnorm_v<T, 4>(q, y, n, m, out, g, s, ncopy);
  if (vec == 2) return launch_colnorm_v<T, 2>(q, y, n, m, out, g, s, ncopy);
  return launch_colnorm_v<T, 1>(q, y, n, m, out, g, s, ncopy);
}

// The apply pass can run the outer projection itself (k_apply FUSE) when one
// column tile holds the whole norm vector -- and pays when the grid is small:
// every CTA repeats the projection (a few block reductions over L2-resident
// norms, ~3 us at the head of the kernel) where a K2 launch costs ~4 us of
// latency chain.  Measured K1 start to K3 end: 300 x 900 11.3 -> 9.7 us,
// 1000 x 1000 13.1 -> 12.0, 5000 x 1024 25.9 -> 25.1; but 20000 x 512 26.1 ->
// 27.3 and 65536 x 256 31.2 -> 33.5 (thousands of CTAs fold the maxima's
// copies and repeat the projection), hence the element cap.
constexpr int64_t kFuseMaxElements = int64_t(6) << 20;
bool apply_fusable(int vec, int64_t n, int64_t m) {
  return (m + vec - 1) / vec <= mpk::kThreads && n * m <= kFuseMaxElements;
}

template <typename T, int VEC, int Q, int U>
cudaError_t launch_apply_qu(const T* y, T* x, int64_t n, int64_t m, const mpk::ApplyCols& A, bool derive,
                            const mp_info* info, unsigned flags, cudaStream_t s, bool fuse = false) {
  if (fuse) {  // one tile of whole warps (the core's block reductions)
    const int tf = (threads_for(VEC, m) + 31) & ~31;
    const void* ff = reinterpret_cast<const void*>(mpk::k_apply<T, VEC, Q, U, true, true>);
    Grid gf = plan_grid(VEC, n, m, occupancy(ff, tf));
    gf.threads = tf;
    dim3 gridf(1, static_cast<unsigned>(gf.nrb));
    return launch_pdl(mpk::k_apply<T, VEC, Q, U, true, true>, gridf, dim3(tf), 0, s, y, x, n, m,
                      kRowInterleave ? n / gf.nrb : gf.rpb, kRowInterleave, A, info, flags);
  }
  const int t = threads_for(VEC, m);
  const void* fn = derive ? reinterpret_cast<const void*>(mpk::k_apply<T, VEC, Q, U, true>)
                          : reinterpret_cast<const void*>(mpk::k_apply<T, VEC, Q, U, false>);
  const Grid g = plan_grid(VEC, n, m, occupancy(fn, t));
  dim3 grid(static_cast<unsigned>(g.ntiles), static_cast<unsigned>(g.nrb));
  if (derive)
    return launch_pdl(mpk::k_apply<T, VEC, Q, U, true>, grid, dim3(g.threads), 0, s, y, x, n, m,
                      kRowInterleave ? n / g.nrb : g.rpb, kRowInterleave, A, info,
                      flags);
  return launch_pdl(mpk::k_apply<T, VEC, Q, U, false>, grid, dim3(g.threads), 0, s, y, x, n, m,
                      kRowInterleave ? n / g.nrb : g.rpb, kRowInterleave, A, info,
                    flags);
}

// l_inf: 8 packs in flight per thread (config 2 K3 ~130 -> 127 us) when the
// row slots are deep enough to fill batches of 8 (short matrices keep 4: one
// HBM round trip for their few rows, config 1 K3 3.8 -> 2.8 us).
template <typename T, int VEC, int Q>
cudaError_t launch_apply_q(const T* y, T* x, int64_t n, int64_t m, const mpk::ApplyCols& A, bool derive,
                           const mp_info* info, unsigned flags, cudaStream_t s, bool fuse) {
  if constexpr (Q == mpk::kInf) {
    const int t = threads_for(VEC, m);
    const Grid g8 = plan_grid(VEC, n, m, occupancy(reinterpret_cast<const void*>(mpk::k_apply<T, VEC, Q, 8, true>), t));
    if (n / g8.nrb >= 16) return launch_apply_qu<T, VEC, Q, 8>(y, x, n, m, A, derive, info, flags, s, fuse);
  }
  return launch_apply_qu<T, VEC, Q, 4>(y, x, n, m, A, derive, info, flags, s, fuse);
}

template <typename T, int VEC>
cudaError_t launch_apply_v(int q, const T* y, T* x, int64_t n, int64_t m, const mpk::ApplyCols& A, bool derive,
                           const mp_info* info, unsigned flags, cudaStream_t s, bool fuse) {
  if (q == mpk::kInf) return launch_apply_q<T, VEC, mpk::kInf>(y, x, n, m, A, derive, info, flags, s, fuse);
  return launch_apply_q<T, VEC, mpk::kL2>(y, x, n, m, A, derive, info, flags, s, fuse);
}

// `fuse` (derive only, apply_fusable(vec, m)): A.outer holds the outer
// projection's arguments and no K2 was launched.
template <typename T>
cudaError_t launch_apply(int q, int vec, const T* y, T* x, int64_t n, int64_t m, const mpk::ApplyCols& A,
                         bool derive, const mp_info* info, unsigned flags, cudaStream_t s, bool fuse = false) {
  if (vec == 8) {
    if constexpr (sizeof(T) == 4) return launch_apply_v<T, 8>(q, y, x, n, m, A, derive, info, flags, s, fuse);
  }
  if (vec == 4) return launch_apply_v<T, 4>(q, y, x, n, m, A, derive, info, flags, s, fuse);
  if (vec == 2) return launch_apply_v<T, 2>(q, y, x, n, m, A, derive, info, flags, s, fuse);
  return launch_apply_v<T, 1>(q, y, x, n, m, A, derive, info, flags, s, fuse);
}

template <int P>
cudaError_t outer_attr() {
  cudaError_t e = cudaFuncSetAttribute(mpk::k_outer<P>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(mpk::k_outer<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(P * mpk::kOuterThreads * sizeof(double)));
}

cudaError_t outer_setup() {
  static std::atomic<uint64_t> done{0};
  return mpi::once_per_device(done, [] {
    for (cudaError_t e : {outer_attr<1>(), outer_attr<2>(), outer_attr<4>(), outer_attr<8>(), outer_attr<12>(),
                          outer_attr<16>(), outer_attr<24>(), mpk::l1strip_setup()})
      if (e != cudaSuccess) return e;
    return cudaSuccess;
  });
}

// K2 on a cluster of C CTAs (PDL + cluster launch attributes).
template <int P>
cudaError_t launch_outer_p(const mpk::OuterArgs& a, int C, int chunk, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(mpk::kOuterThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(std::max(chunk, 1)) * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = C;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, mpk::k_outer<P>, a);
}

template <int P, int NT = mpk::kOuterRegThreads, bool FOLD = false>
cudaError_t launch_outer_reg(const mpk::OuterArgs& a, cudaStream_t s) {
  return launch_pdl(mpk::k_outer_reg<P, NT, FOLD>, dim3(1), dim3(NT), 0, s, a);
}

cudaError_t launch_outer(const mpk::OuterArgs& a, cudaStream_t s) {
  cudaError_t e = outer_setup();
  if (e != cudaSuccess) return e;
  if (a.ncopy > 1) {  // narrow l_inf: fold K1's copies of the maxima (m <= 512)
    if (a.m <= 256) return launch_outer_reg<1, 256, true>(a, s);
    return launch_outer_reg<2, 256, true>(a, s);
  }
  if (a.m <= 2048) {  // small vectors: a 256-thread CTA, cheaper barriers
    const int64_t per = (std::max<int64_t>(a.m, 1) + 255) / 256;
    if (per <= 1) return launch_outer_reg<1, 256>(a, s);
    if (per <= 2) return launch_outer_reg<2, 256>(a, s);
    if (per <= 4) return launch_outer_reg<4, 256>(a, s);
    return launch_outer_reg<8, 256>(a, s);
  }
  if (a.m <= mpk::kOuterRegMaxM) {
    const int64_t per = (std::max<int64_t>(a.m, 1) + mpk::kOuterRegThreads - 1) / mpk::kOuterRegThreads;
    if (per <= 1) return launch_outer_reg<1>(a, s);
    if (per <= 2) return launch_outer_reg<2>(a, s);
    if (per <= 4) return launch_outer_reg<4>(a, s);
    if (per <= 8) return launch_outer_reg<8>(a, s);
    return launch_outer_reg<12>(a, s);
  }
  // ~2048 elements (8 per thread) per CTA, at most 16 CTAs per cluster.
  const int64_t m = std::max<int64_t>(a.m, 1);
  const int C = static_cast<int>(std::min<int64_t>(mpk::kOuterMaxCluster, (m + 2047) / 2048));
  const int chunk = static_cast<int>((m + C - 1) / C);
  const int per = (chunk + mpk::kOuterThreads - 1) / mpk::kOuterThreads;
  if (per <= 1) return launch_outer_p<1>(a, C, chunk, s);
  if (per <= 2) return launch_outer_p<2>(a, C, chunk, s);
  if (per <= 4) return launch_outer_p<4>(a, C, chunk, s);
  if (per <= 8) return launch_outer_p<8>(a, C, chunk, s);
  if (per <= 12) return launch_outer_p<12>(a, C, chunk, s);
  if (per <= 16) return launch_outer_p<16>(a, C, chunk, s);
  return launch_outer_p<24>(a, C, chunk, s);
}

// Column parameters for a fiber projection from (norms v, budgets u).
template <typename T>
__global__ void k_colparams(const double* __restrict__ v, const double* __restrict__ u, int64_t m, int q,
                            void* __restrict__ colp, const mp_info* __restrict__ info) {
  if (info->status != MP_OK) return;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= m) return;
  const double uu = u[c];
  if (q == mpk::kInf) {
    if constexpr (sizeof(T) == 4)
      static_cast<float2*>(colp)[c] = make_float2(__double2float_rz(uu), __double2float_rn(uu));
    else
      static_cast<double*>(colp)[c] = uu;
  } else if (q == mpk::kL2) {
    static_cast<double*>(colp)[c] = (v[c] > uu) ? uu / v[c] : 1.0;
  }
}

// Narrow l_inf matrices (m <= 512, K2 = k_outer_reg<P, 256, true>, which
// folds the copies): K1's atomics spread over 8 copies of the maxima
// (256^3 tri-level: 148 same-address atomics per column -> 19).
inline int inf_copies(int64_t m) { return m <= 512 ? mpk::kInfCopies : 1; }

// ------------------------------------------------------ workspace layouts
struct BilevelWs {
  mp_info* info;
  void* k1out;       // l_inf bits or l1/l2 partials
  double* v;         // norms (f64)
  double* budgets;   // outer-projected radii
  void* colp;        // per-column apply parameters
  mpk::L1StripWs l1; // l1 inner projection scratch
  void* large;       // k_outer_large scratch (m > kOuterMaxM)
  mpk::OuterParams* params;  // K2 -> apply: mode / tau / scale
};

BilevelWs carve_bilevel(Carve& c, mp_dtype dt, int64_t n, int64_t m, mp_norm q) {
  BilevelWs w{};
  w.info = c.take<mp_info>(1);
  // l_inf: bit-pattern maxima, kInfCopies copies for narrow matrices
  if (q == MP_NORM_INF) w.k1out = c.take<unsigned long long>(static_cast<size_t>(inf_copies(m)) * m);
  else w.k1out = c.take<double>(static_cast<size_t>(max_nrb(dt, n, m)) * m);
  w.v = c.take<double>(m);
  w.budgets = c.take<double>(m);
  w.colp = c.take<double>(m);
  if (q == MP_NORM_L1) w.l1 = mpk::carve_l1strip(c, m);
  w.large = c.take<char>(mpk::outer_large_ws_bytes(m));
  w.params = c.take<mpk::OuterParams>(1);
  return w;
}

// Core of a fiber-projection level: y (T, (n, m)) -> x given norms v and
// budgets u; colp must hold the per-column parameters for q.
template <typename T>
cudaError_t project_fibers(const T* y, T* x, int64_t n, int64_t m, int q, const double* v, const double* u,
                           const void* colp, const mpk::L1StripWs& l1, const mp_info* info, unsigned flags,
                           mp_dtype dt, cudaStream_t s) {
  if (q == mpk::kL1) return mpk::launch_l1strip<T>(y, x, n, m, v, u, l1, info, flags, s);
  mpk::ApplyCols A{};
  A.colp = colp;
  A.budgets = u;
  return launch_apply<T>(q, pick_vec(dt, m, y, x), y, x, n, m, A, false, info, flags, s);
}

// K1 partials (l1 / l2) -> norms.
cudaError_t launch_norm_reduce(int q, const void* part, int64_t R, int64_t m, double* v, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((m + 31) / 32);
  if (q == mpk::kL1)
    return launch_pdl(mpk::k_colnorm_reduce<mpk::kL1>, dim3(blocks), dim3(256), 0, s, static_cast<const double*>(part),
                      R, m, v);
  return launch_pdl(mpk::k_colnorm_reduce<mpk::kL2>, dim3(blocks), dim3(256), 0, s, static_cast<const double*>(part),
                    R, m, v);
}

// The bi-level hot path (proj/src/bilevel.cpp:10-32):
//   [memset] K1 norms -> (l1/l2: reduce partials) -> K2 outer threshold ->
//   K3 apply, each later kernel PDL-chained to its producer.  K2 publishes
//   only (mode, tau, scale); K3 / the l1 strips derive every budget from its
//   norm, write the user-facing budgets and count zero columns.
template <typename T>
mp_status bilevel_impl(const T* y, T* x, mp_dtype dt, int64_t n, int64_t m, mp_norm p, mp_norm q, double eta,
                       double* budgets, double* norms, mp_info* info, unsigned flags, void* ws, size_t wsb,
                       cudaStream_t s) {
  Carve c(ws, wsb);
  BilevelWs w = carve_bilevel(c, dt, n, m, q);
  if (!c.fits()) return fail(MP_ERR_WORKSPACE, "mp_bilevel_project: workspace too small");
  MP_CUDA_TRY(outer_setup());
  mp_info* inf = info ? info : w.info;
  double* u = budgets ? budgets : w.budgets;
  double* v = norms ? norms : w.v;
  // The huge-n l1 fallback reads materialised budgets; everything else derives.
  const bool derive = !(q == MP_NORM_L1 && !mpk::l1_staged_ok<T>(n));

  const int vec = pick_vec(dt, m, y, x);
  Grid g;
  prof_mark(0, s);
  mpk::OuterArgs oa{};
  oa.m = m;
  oa.p = p;
  oa.eta = eta;
  oa.u_out = u;
  oa.info = inf;
  oa.scratch = w.large;
  oa.params = w.params;
  oa.emit = derive ? 0 : 1;
  mpk::ApplyCols A{};
  A.params = w.params;
  A.u_out = u;
  A.info_w = inf;
  if (q == MP_NORM_INF) {
    const int ncopy = inf_copies(m);
    // 8 bytes per column and copy even for f32 bits: measured, a 4000-byte
    // memset node cost config 1 two microseconds more than an 8000-byte one
    MP_CUDA_TRY(cudaMemsetAsync(w.k1out, 0, static_cast<size_t>(ncopy) * m * sizeof(unsigned long long), s));
    MP_CUDA_TRY(launch_colnorm<T>(q, vec, y, n, m, w.k1out, g, s, ncopy));
    oa.ncopy = ncopy;
    oa.vin = w.k1out;
    oa.vkind = sizeof(T) == 4 ? 0 : 1;  // f64 |y| bits are the f64 values
    A.v = w.k1out;
    A.vkind = oa.vkind;
    A.v_out = norms;
  } else {
    MP_CUDA_TRY(launch_colnorm<T>(q, vec, y, n, m, w.k1out, g, s));
    MP_CUDA_TRY(launch_norm_reduce(q, w.k1out, g.nrb, m, v, s));
    oa.vin = v;
    oa.vkind = 1;
    A.v = v;
    A.vkind = 1;
  }
  prof_mark(1, s);
  // Narrow matrices (one column tile): every CTA of the apply pass runs the
  // outer projection itself, no K2 launch.
  const bool fuse = derive && q != MP_NORM_L1 && apply_fusable(vec, n, m);
  if (fuse) {
    A.outer = oa;
  } else if (m > mpk::kOuterMaxM) {
    MP_CUDA_TRY(mpk::launch_outer_large(oa, s));
  } else {
    MP_CUDA_TRY(launch_outer(oa, s));
  }
  prof_mark(2, s);
  if (q == MP_NORM_L1) {
    mpk::L1Derive dv;
    if (derive) {
      dv.params = w.params;
      dv.u_out = u;
      dv.info_w = inf;
    }
    MP_CUDA_TRY(mpk::launch_l1strip<T>(y, x, n, m, v, u, w.l1, inf, flags, s, dv));
  } else {
    MP_CUDA_TRY(launch_apply<T>(q, vec, y, x, n, m, A, true, inf, flags, s, fuse));
  }
  prof_mark(3, s);
  return MP_OK;
}

mp_status check_bilevel_args(const void* y, const void* x, mp_dtype dt, int64_t n, int64_t m, mp_norm p, mp_norm q,
                             double eta) {
  if (!dtype_ok(dt)) return fail(MP_ERR_CONFIG, "unknown dtype code");
  if (!norm_ok(p) || !norm_ok(q)) return fail(MP_ERR_CONFIG, "unknown norm code");
  if (n < 1 || m < 1) return fail(MP_ERR_SHAPE, "bilevel_project requires a non-empty order-2 tensor");
  if (!(eta >= 0.0) || !std::isfinite(eta)) return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!y || !x) return fail(MP_ERR_WORKSPACE, "null tensor pointer");
  return MP_OK;
}


// --------------------------------------------------------- vector / aggregate
template <typename T>
__global__ void k_cast_from_f64(const double* __restrict__ in, T* __restrict__ out, int64_t len,
                                const mp_info* __restrict__ info) {
  if (info->status != MP_OK) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len) out[i] = static_cast<T>(in[i]);
}

struct VectorWs {
  mp_info* info;
  double* u;     // f64 result staging (f32 data)
  void* large;
};

VectorWs carve_vector(Carve& c, mp_dtype dt, int64_t len) {
  VectorWs w{};
  w.info = c.take<mp_info>(1);
  w.u = dt == MP_F32 ? c.take<double>(len) : nullptr;
  w.large = c.take<char>(mpk::outer_large_ws_bytes(len));
  return w;
}

// project_ball on a flat vector (proj/src/vector_balls.cpp:207-214).
mp_status vector_impl(const void* y, void* x, mp_dtype dt, int64_t len, mp_norm q, double radius, mp_info* info,
                      VectorWs& w, cudaStream_t s) {
  mp_info* inf = info ? info : w.info;
  mpk::OuterArgs oa{};
  oa.vin = y;
  oa.vkind = dt == MP_F32 ? 2 : 1;
  oa.m = len;
  oa.p = q;
  oa.eta = radius;
  oa.u_out = dt == MP_F32 ? w.u : static_cast<double*>(x);
  oa.info = inf;
  oa.scratch = w.large;
  oa.emit = 1;
  if (len > mpk::kOuterMaxM) {
    MP_CUDA_TRY(mpk::launch_outer_large(oa, s));
  } else {
    MP_CUDA_TRY(launch_outer(oa, s));
  }
  if (dt == MP_F32) {
    const unsigned blocks = static_cast<unsigned>((len + 255) / 256);
    k_cast_from_f64<float><<<blocks, 256, 0, s>>>(w.u, static_cast<float*>(x), len, inf);
    MP_CUDA_TRY(cudaGetLastError());
  }
  return MP_OK;
}

// Leading-axis aggregate of (n, m) T data into out (f64), via K1 (+ finalize).
// scratch: l_inf -> m u32/u64 bits (f32 only; f64 bits land in out directly),
// l1/l2 -> max_nrb * m partials.
template <typename T>
mp_status aggregate_impl(const T* t, double* out, mp_dtype dt, int64_t n, int64_t m, int q, void* scratch,
                         cudaStream_t s) {
  const int vec = pick_vec(dt, m, t, t);
  Grid g;
  const unsigned fin_blocks = static_cast<unsigned>((m + 255) / 256);
  if (q == mpk::kInf) {
    void* bits = sizeof(T) == 8 ? static_cast<void*>(out) : scratch;
    MP_CUDA_TRY(cudaMemsetAsync(bits, 0, static_cast<size_t>(m) * sizeof(T), s));
    MP_CUDA_TRY(launch_colnorm<T>(q, vec, t, n, m, bits, g, s));
    if (sizeof(T) == 4) mpk::k_colnorm_finalize<mpk::kInf><<<fin_blocks, 256, 0, s>>>(bits, 1, m, 0, out);
  } else {
    MP_CUDA_TRY(launch_colnorm<T>(q, vec, t, n, m, scratch, g, s));
    MP_CUDA_TRY(launch_norm_reduce(q, scratch, g.nrb, m, out, s));
  }
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

size_t aggregate_scratch_bytes(mp_dtype dt, int64_t n, int64_t m, int q) {
  if (q == mpk::kInf) return static_cast<size_t>(m) * 8;
  return static_cast<size_t>(max_nrb(dt, n, m)) * static_cast<size_t>(m) * 8;
}

// ------------------------------------------------------------- multilevel
struct MultiWs {
  mp_info* info = nullptr;
  std::vector<double*> agg;   // agg[i], i = 1..order-1 (agg[0] unused)
  std::vector<double*> bud;   // budgets B_i (when no user chain), i = 1..order-1
  void* scratch = nullptr;    // K1 scratch, max over levels
  void* colp = nullptr;       // per-column params, max M_1..M_{order-1}
  mpk::L1StripWs l1{};
  void* large = nullptr;
  VectorWs vec{};             // depth-1 path
};

MultiWs carve_multi(Carve& c, mp_dtype dt, const int64_t* shape, int order, const mp_norm* levels) {
  MultiWs w;
  std::vector<int64_t> M(order + 1, 1);
  for (int i = order - 1; i >= 0; --i) M[i] = M[i + 1] * shape[i];
  if (order == 1) {
    w.vec = carve_vector(c, dt, M[0]);
    return w;
  }
  w.info = c.take<mp_info>(1);
  w.agg.assign(order, nullptr);
  w.bud.assign(order, nullptr);
  size_t scr = 0;
  int64_t mmax = 1;
  for (int i = 1; i < order; ++i) {
    w.agg[i] = c.take<double>(M[i]);
    w.bud[i] = c.take<double>(M[i]);
    mmax = std::max(mmax, M[i]);
    scr = std::max(scr, aggregate_scratch_bytes(i == 1 ? dt : MP_F64, shape[i - 1], M[i], levels[i - 1]));
  }
  w.scratch = c.take<char>(scr);
  w.colp = c.take<double>(mmax);
  w.l1 = mpk::carve_l1strip(c, mmax);
  w.large = c.take<char>(mpk::outer_large_ws_bytes(shape[order - 1]));
  return w;
}

template <typename T>
cudaError_t launch_colparams(const double* v, const double* u, int64_t m, int q, void* colp, const mp_info* info,
                             cudaStream_t s) {
  if (q == mpk::kL1) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>((m + 255) / 256);
  k_colparams<T><<<blocks, 256, 0, s>>>(v, u, m, q, colp, info);
  return cudaGetLastError();
}

template <typename T>
mp_status multilevel_impl(const T* t, T* x, mp_dtype dt, const int64_t* shape, int order, const mp_norm* levels,
                          double eta, double* chain, mp_info* info, unsigned flags, void* ws, size_t wsb,
                          cudaStream_t s) {
  Carve c(ws, wsb);
  MultiWs w = carve_multi(c, dt, shape, order, levels);
  if (!c.fits()) return fail(MP_ERR_WORKSPACE, "mp_multilevel_project: workspace too small");
  MP_CUDA_TRY(outer_setup());
  prof_mark(0, s);
  if (order == 1) {
    mp_status st1 = vector_impl(t, x, dt, shape[0], levels[0], eta, info, w.vec, s);
    prof_mark(3, s);
    return st1;
  }

  std::vector<int64_t> M(order + 1, 1);
  for (int i = order - 1; i >= 0; --i) M[i] = M[i + 1] * shape[i];
  mp_info* inf = info ? info : w.info;
  // Budget buffers: inside the user chain when given (deepest first).
  std::vector<double*> B(order, nullptr);
  {
    int64_t off = 0;
    for (int i = order - 1; i >= 1; --i) {
      B[i] = chain ? chain + off : w.bud[i];
      off += M[i];
    }
  }
  // Aggregation chain (proj/src/multilevel.cpp:99-104).
  mp_status st = aggregate_impl<T>(t, w.agg[1], dt, shape[0], M[1], levels[0], w.scratch, s);
  if (st != MP_OK) return st;
  for (int i = 1; i + 1 < order; ++i) {
    st = aggregate_impl<double>(w.agg[i], w.agg[i + 1], MP_F64, shape[i], M[i + 1], levels[i], w.scratch, s);
    if (st != MP_OK) return st;
  }
  // Deepest aggregate: vector-ball projection at eta (:106-111).
  mpk::OuterArgs oa{};
  oa.vin = w.agg[order - 1];
  oa.vkind = 1;
  oa.m = M[order - 1];
  oa.p = levels[order - 1];
  oa.eta = eta;
  oa.u_out = B[order - 1];
  oa.info = inf;
  oa.scratch = w.large;
  oa.emit = 1;
  if (oa.m > mpk::kOuterMaxM) {
    MP_CUDA_TRY(mpk::launch_outer_large(oa, s));
  } else {
    MP_CUDA_TRY(launch_outer(oa, s));
  }
  // Unwind (:113-119): level i fibers at the budgets of level i+1.
  for (int i = order - 2; i >= 1; --i) {
    MP_CUDA_TRY(launch_colparams<double>(w.agg[i + 1], B[i + 1], M[i + 1], levels[i], w.colp, inf, s));
    MP_CUDA_TRY(project_fibers<double>(w.agg[i], B[i], shape[i], M[i + 1], levels[i], w.agg[i + 1], B[i + 1],
                                       w.colp, w.l1, inf, 0u, MP_F64, s));
  }
  MP_CUDA_TRY(launch_colparams<T>(w.agg[1], B[1], M[1], levels[0], w.colp, inf, s));
  MP_CUDA_TRY(project_fibers<T>(t, x, shape[0], M[1], levels[0], w.agg[1], B[1], w.colp, w.l1, inf, flags, dt, s));
  prof_mark(3, s);
  return MP_OK;
}

// Specs whose inner levels are all l_inf (order >= 2); rows = d0*...*d_{r-2}.
bool inf_inner_levels(const int64_t* shape, int order, const mp_norm* levels, int64_t& rows) {
  if (order < 2) return false;
  rows = 1;
  for (int i = 0; i + 1 < order; ++i) {
    if (levels[i] != MP_NORM_INF) return false;
    rows *= shape[i];
  }
  return true;
}

mp_status check_multi_args(const void* t, const void* x, mp_dtype dt, const int64_t* shape, int order,
                           const mp_norm* levels, int depth, double eta) {
  if (!dtype_ok(dt)) return fail(MP_ERR_CONFIG, "unknown dtype code");
  if (!shape || order < 1) return fail(MP_ERR_SHAPE, "tensor order must be >= 1");
  for (int i = 0; i < order; ++i)
    if (shape[i] < 1) return fail(MP_ERR_SHAPE, "zero dimension in shape");
  if (depth < 1 || !levels) return fail(MP_ERR_CONFIG, "empty norm spec");
  for (int i = 0; i < depth; ++i)
    if (!norm_ok(levels[i])) return fail(MP_ERR_CONFIG, "unknown norm code");
  if (depth != order) return fail(MP_ERR_SHAPE, "norm spec depth does not match tensor order");
  if (!(eta >= 0.0) || !std::isfinite(eta)) return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!t || !x) return fail(MP_ERR_WORKSPACE, "null tensor pointer");
  return MP_OK;
}

// ---------------------------------------------------- exact Euclidean l1,inf
// (proj/src/euclidean.cpp:82-170; kernels in mp_euclid.cuh)
struct EuclidWs {
  mp_info* info;
  void* mags;         // |Y| column-major (stride ld), sorted per column
  mpk::DD* offs;      // double-double prefix offsets every 32 ranks (stride ldo)
  double* fb;         // each chunk's first breakpoint (stride ldo)
  void* tmp;          // merge buffer for a batch of long columns (n > one CTA's sort)
  int64_t ld, ldo, batch;
  double* colmax;
  double* budgets;
  void* colp;
  mpk::EuScratch* sc;
};

template <typename T>
int64_t eu_merge_batch(int64_t n, int64_t m, int64_t ld) {
  if (n <= mpk::eu_sort_cap<T>()) return 0;
  // long columns merge through a buffer of at most ~1/4 of the tensor
  return std::max<int64_t>(1, std::min<int64_t>(m, (m + 3) / 4));
}

EuclidWs carve_euclid(Carve& c, mp_dtype dt, int64_t n, int64_t m) {
  EuclidWs w{};
  const size_t s = dtype_size(dt);
  w.ld = (n + 3) & ~int64_t(3);  // 16-byte aligned columns
  w.ldo = (n + mpk::kEuChunk - 1) / mpk::kEuChunk;
  w.batch = dt == MP_F32 ? eu_merge_batch<float>(n, m, w.ld) : eu_merge_batch<double>(n, m, w.ld);
  w.info = c.take<mp_info>(1);
  w.mags = c.take<char>(static_cast<size_t>(w.ld) * m * s);
  w.offs = c.take<mpk::DD>(static_cast<size_t>(w.ldo) * m);
  w.fb = c.take<double>(static_cast<size_t>(w.ldo) * m);
  w.tmp = w.batch ? c.take<char>(static_cast<size_t>(w.ld) * w.batch * s) : nullptr;
  w.colmax = c.take<double>(m);
  w.budgets = c.take<double>(m);
  w.colp = c.take<double>(m);
  w.sc = c.take<mpk::EuScratch>(1);
  return w;
}

template <typename T, int NT>
cudaError_t launch_eu_block(T* mags, const EuclidWs& w, int64_t n, int64_t m, const mp_info* inf, cudaStream_t s) {
  constexpr size_t smem = mpk::EuBlock<T, NT>::kSmem;
  static std::atomic<uint64_t> done{0};
  const cudaError_t a = mpi::once_per_device(done, [] {
    return cudaFuncSetAttribute(mpk::k_eu_sort_block<T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem));
  });
  if (a != cudaSuccess) return a;
  const int64_t runs = (n + static_cast<int64_t>(NT) * 16 - 1) / (static_cast<int64_t>(NT) * 16);
  mpk::k_eu_sort_block<T, NT><<<static_cast<unsigned>(m * runs), NT, smem, s>>>(mags, w.ld, n, runs, w.offs, w.fb,
                                                                               w.ldo, inf);
  return cudaGetLastError();
}

constexpr int64_t kEuWarpSearchMaxCols = 4096;

template <typename T>
mp_status euclid_impl(const T* y, T* x, mp_dtype dt, int64_t n, int64_t m, double eta, double* budgets,
                      mp_info* info, unsigned flags, const EuclidWs& w, cudaStream_t s) {
  mp_info* inf = info ? info : w.info;
  double* u = budgets ? budgets : w.budgets;
  prof_mark(0, s);
  MP_CUDA_TRY(cudaMemsetAsync(inf, 0, sizeof(mp_info), s));
  T* mags = static_cast<T*>(w.mags);
  mpk::k_eu_gather<T><<<dim3(static_cast<unsigned>((m + mpk::kEuTile - 1) / mpk::kEuTile),
                           static_cast<unsigned>((n + mpk::kEuTile - 1) / mpk::kEuTile)),
                      dim3(32, 8), 0, s>>>(y, n, m, mags, w.ld, inf);
  MP_CUDA_TRY(cudaGetLastError());
  // columns that fit one CTA are sorted whole (+ prefix offsets); longer
  // columns in runs of the largest block, merged pairwise through w.tmp
  const int64_t cap = mpk::eu_sort_cap<T>();  // f64 at 1024 x 16 keys exceeds shared memory
  int nt = 64;
  while (nt * 16 < n && nt * 16 < cap) nt *= 2;
  switch (nt) {
    case 64: MP_CUDA_TRY((launch_eu_block<T, 64>(mags, w, n, m, inf, s))); break;
    case 128: MP_CUDA_TRY((launch_eu_block<T, 128>(mags, w, n, m, inf, s))); break;
    case 256: MP_CUDA_TRY((launch_eu_block<T, 256>(mags, w, n, m, inf, s))); break;
    case 512: MP_CUDA_TRY((launch_eu_block<T, 512>(mags, w, n, m, inf, s))); break;
    default:
      if constexpr (sizeof(T) == 4) MP_CUDA_TRY((launch_eu_block<T, 1024>(mags, w, n, m, inf, s)));
      break;
  }
  if (n > cap) {
    T* tmp = static_cast<T*>(w.tmp);
    const int64_t tile = static_cast<int64_t>(mpk::kEuMergeThreads) * mpk::kEuMergeE;
    for (int64_t j0 = 0; j0 < m; j0 += w.batch) {
      const int64_t nb = std::min(w.batch, m - j0);
      T* cols = mags + j0 * w.ld;
      for (int64_t width = cap; width < n; width *= 2) {
        mpk::k_eu_merge<T><<<dim3(static_cast<unsigned>((n + tile - 1) / tile), static_cast<unsigned>(nb)),
                             mpk::kEuMergeThreads, 0, s>>>(cols, tmp, w.ld, n, width, inf);
        MP_CUDA_TRY(cudaGetLastError());
        MP_CUDA_TRY(cudaMemcpyAsync(cols, tmp, static_cast<size_t>(nb) * w.ld * sizeof(T), cudaMemcpyDeviceToDevice,
                                    s));
      }
    }
    mpk::k_eu_prefix<T><<<static_cast<unsigned>(m), 256, 0, s>>>(mags, w.ld, n, w.offs, w.fb, w.ldo, inf);
    MP_CUDA_TRY(cudaGetLastError());
  }
  // cooperative search grid: every CTA co-resident; a warp per column up to
  // kEuWarpSearchMaxCols columns, a thread per column beyond
  const bool warp = m <= kEuWarpSearchMaxCols;
  static int occ_w = -1, occ_t = -1;
  if (occ_w < 0) {
    MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_w, mpk::k_eu_search<T, true>,
                                                              mpk::kEuSearchThreads, 0));
    MP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, mpk::k_eu_search<T, false>,
                                                              mpk::kEuSearchThreads, 0));
  }
  const int per_cta = warp ? mpk::kEuSearchThreads / 32 : mpk::kEuSearchThreads;
  int G = static_cast<int>(std::min<int64_t>(
      (m + per_cta - 1) / per_cta,
      static_cast<int64_t>(sm_count()) * std::max(1, warp ? occ_w : std::min(occ_t, 2))));
  G = std::max(1, std::min(G, mpk::kEuMaxCtas));
  const T* cm = mags;
  const mpk::DD* co = w.offs;
  const double* cf = w.fb;
  double* colmax = w.colmax;
  double* coltot = static_cast<double*>(w.colp);  // scratch until launch_colparams
  mpk::EuScratch* sc = w.sc;
  int64_t ld = w.ld, ldo = w.ldo;
  void* args[] = {&cm, &co, &cf, &n, &m, &ld, &ldo, &eta, &colmax, &u, &coltot, &inf, &sc};
  MP_CUDA_TRY(cudaLaunchCooperativeKernel(warp ? reinterpret_cast<const void*>(mpk::k_eu_search<T, true>)
                                               : reinterpret_cast<const void*>(mpk::k_eu_search<T, false>),
                                          dim3(G), dim3(mpk::kEuSearchThreads), args, 0, s));
  if (eta == 0.0) {  // the reference returns DenseTensor::zeros (+0.0 everywhere)
    MP_CUDA_TRY(cudaMemsetAsync(x, 0, static_cast<size_t>(n) * m * sizeof(T), s));
  } else {
    MP_CUDA_TRY(launch_colparams<T>(w.colmax, u, m, mpk::kInf, w.colp, inf, s));
    mpk::ApplyCols A{};
    A.colp = w.colp;
    A.budgets = u;
    MP_CUDA_TRY(launch_apply<T>(mpk::kInf, pick_vec(dt, m, y, x), y, x, n, m, A, false, inf, flags, s));
  }
  prof_mark(3, s);
  return MP_OK;
}

}  // namespace

// ================================================================== C-ABI
extern "C" {

const char* mp_last_error(void) { return last_error(); }

void mp_profile_timeline(unsigned long long* device_buf) {
  cudaMemcpyToSymbol(mpk::g_mp_timeline, &device_buf, sizeof(device_buf));
}

void mp_profile_events(void* const* events, int count) {
  for (int i = 0; i < 4; ++i)
    g_prof[i] = (events && i < count) ? static_cast<cudaEvent_t>(events[i]) : nullptr;
}

int mp_version(void) { return 100; }

size_t mp_bilevel_workspace_size(mp_dtype dtype, int64_t n, int64_t m, mp_norm p, mp_norm q) {
  (void)p;
  if (n < 1 || m < 1 || !dtype_ok(dtype) || !norm_ok(q)) return 0;
  Carve c(nullptr, 0);
  carve_bilevel(c, dtype, n, m, q);
  return c.off + 256;
}

mp_status mp_bilevel_project(const void* y, void* x, mp_dtype dtype, int64_t n, int64_t m, mp_norm p, mp_norm q,
                             double eta, double* budgets, double* norms, mp_info* info, unsigned flags,
                             void* workspace, size_t workspace_bytes, void* stream) {
  mp_status st = check_bilevel_args(y, x, dtype, n, m, p, q, eta);
  if (st != MP_OK) return st;
  if (!workspace) return fail(MP_ERR_WORKSPACE, "null workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == MP_F32)
    return bilevel_impl<float>(static_cast<const float*>(y), static_cast<float*>(x), dtype, n, m, p, q, eta, budgets,
                               norms, info, flags, workspace, workspace_bytes, s);
  return bilevel_impl<double>(static_cast<const double*>(y), static_cast<double*>(x), dtype, n, m, p, q, eta, budgets,
                              norms, info, flags, workspace, workspace_bytes, s);
}


size_t mp_multilevel_workspace_size(mp_dtype dtype, const int64_t* shape, int order, const mp_norm* levels,
                                    int depth) {
  if (check_multi_args(reinterpret_cast<void*>(1), reinterpret_cast<void*>(1), dtype, shape, order, levels, depth,
                       0.0) != MP_OK)
    return 0;
  Carve c(nullptr, 0);
  carve_multi(c, dtype, shape, order, levels);
  size_t need = c.off + 256;
  int64_t rows = 0;
  if (inf_inner_levels(shape, order, levels, rows))
    need = std::max(need, mp_bilevel_workspace_size(dtype, rows, shape[order - 1], levels[order - 1], MP_NORM_INF));
  return need;
}

mp_status mp_multilevel_project(const void* t, void* x, mp_dtype dtype, const int64_t* shape, int order,
                                const mp_norm* levels, int depth, double eta, double* budget_chain, mp_info* info,
                                unsigned flags, void* workspace, size_t workspace_bytes, void* stream) {
  mp_status st = check_multi_args(t, x, dtype, shape, order, levels, depth, eta);
  if (st != MP_OK) return st;
  if (!workspace) return fail(MP_ERR_WORKSPACE, "null workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t rows = 0;
  if (!budget_chain && inf_inner_levels(shape, order, levels, rows)) {
    // (inf, ..., inf, p) == bi-level l_{p,inf} on the (d0*...*d_{r-2}, d_{r-1})
    // reshape, bit for bit: the nested clamps collapse to the
    // deepest budget because |T| <= every intermediate max.  One norm sweep,
    // one apply sweep, instead of the level-by-level chain.
    prof_mark(0, s);
    if (dtype == MP_F32)
      st = bilevel_impl<float>(static_cast<const float*>(t), static_cast<float*>(x), dtype, rows, shape[order - 1],
                               levels[order - 1], MP_NORM_INF, eta, nullptr, nullptr, info, flags, workspace,
                               workspace_bytes, s);
    else
      st = bilevel_impl<double>(static_cast<const double*>(t), static_cast<double*>(x), dtype, rows, shape[order - 1],
                                levels[order - 1], MP_NORM_INF, eta, nullptr, nullptr, info, flags, workspace,
                                workspace_bytes, s);
    return st;
  }
  if (dtype == MP_F32)
    return multilevel_impl<float>(static_cast<const float*>(t), static_cast<float*>(x), dtype, shape, order, levels,
                                  eta, budget_chain, info, flags, workspace, workspace_bytes, s);
  return multilevel_impl<double>(static_cast<const double*>(t), static_cast<double*>(x), dtype, shape, order, levels,
                                 eta, budget_chain, info, flags, workspace, workspace_bytes, s);
}

mp_status mp_perturb_gaussian(void* x, mp_dtype dtype, int64_t count, double sigma, uint64_t seed, uint64_t iteration,
                              void* stream) {
  if (!dtype_ok(dtype)) return fail(MP_ERR_CONFIG, "unknown dtype code");
  if (count < 0 || (count > 0 && !x)) return fail(MP_ERR_SHAPE, "bad tensor");
  if (!(sigma >= 0.0) || !std::isfinite(sigma)) return fail(MP_ERR_VALUE, "sigma must be a finite nonnegative real");
  if (count == 0) return MP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t quads = (count + 3) / 4;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((quads + 255) / 256, sm_count() * 8));
  const uint32_t lo = static_cast<uint32_t>(seed), hi = static_cast<uint32_t>(seed >> 32);
  const uint32_t it = static_cast<uint32_t>(iteration);
  if (dtype == MP_F32) {
    if (count % 4 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0)
      mpk::k_perturb_gaussian<float, true><<<blocks, 256, 0, s>>>(static_cast<float*>(x), count,
                                                                  static_cast<float>(sigma), lo, hi, it);
    else
      mpk::k_perturb_gaussian<float, false><<<blocks, 256, 0, s>>>(static_cast<float*>(x), count,
                                                                   static_cast<float>(sigma), lo, hi, it);
  } else {
    mpk::k_perturb_gaussian<double, false><<<blocks, 256, 0, s>>>(static_cast<double*>(x), count,
                                                                  static_cast<float>(sigma), lo, hi, it);
  }
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

size_t mp_project_ball_workspace_size(mp_dtype dtype, int64_t len, mp_norm q) {
  if (len < 1 || !dtype_ok(dtype) || !norm_ok(q)) return 0;
  Carve c(nullptr, 0);
  carve_vector(c, dtype, len);
  return c.off + 256;
}

mp_status mp_project_ball(const void* y, void* x, mp_dtype dtype, int64_t len, mp_norm q, double radius,
                          mp_info* info, void* workspace, size_t workspace_bytes, void* stream) {
  if (!dtype_ok(dtype)) return fail(MP_ERR_CONFIG, "unknown dtype code");
  if (!norm_ok(q)) return fail(MP_ERR_CONFIG, "unknown norm code");
  if (!(radius >= 0.0) || !std::isfinite(radius)) return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (len < 1) return fail(MP_ERR_SHAPE, "empty vector");
  if (!y || !x || !workspace) return fail(MP_ERR_WORKSPACE, "null pointer");
  Carve c(workspace, workspace_bytes);
  VectorWs w = carve_vector(c, dtype, len);
  if (!c.fits()) return fail(MP_ERR_WORKSPACE, "mp_project_ball: workspace too small");
  return vector_impl(y, x, dtype, len, q, radius, info, w, static_cast<cudaStream_t>(stream));
}

size_t mp_project_fibers_workspace_size(mp_dtype dtype, int64_t n, int64_t m, mp_norm q) {
  if (n < 1 || m < 1 || !dtype_ok(dtype) || !norm_ok(q)) return 0;
  Carve c(nullptr, 0);
  c.take<mp_info>(1);
  c.take<double>(m);
  mpk::carve_l1strip(c, m);
  return c.off + 256;
}

mp_status mp_project_fibers(const void* y, void* x, mp_dtype dtype, int64_t n, int64_t m, mp_norm q,
                            const double* norms, const double* budgets, unsigned flags, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (!dtype_ok(dtype)) return fail(MP_ERR_CONFIG, "unknown dtype code");
  if (!norm_ok(q)) return fail(MP_ERR_CONFIG, "unknown norm code");
  if (n < 1 || m < 1) return fail(MP_ERR_SHAPE, "project_fibers requires a non-empty (n, m) view");
  if (!y || !x || !norms || !budgets || !workspace) return fail(MP_ERR_WORKSPACE, "null pointer");
  Carve c(workspace, workspace_bytes);
  mp_info* inf = c.take<mp_info>(1);
  void* colp = c.take<double>(m);
  mpk::L1StripWs l1 = mpk::carve_l1strip(c, m);
  if (!c.fits()) return fail(MP_ERR_WORKSPACE, "mp_project_fibers: workspace too small");
  MP_CUDA_TRY(outer_setup());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  MP_CUDA_TRY(cudaMemsetAsync(inf, 0, sizeof(mp_info), s));  // status MP_OK: the kernels proceed
  if (dtype == MP_F32) {
    MP_CUDA_TRY(launch_colparams<float>(norms, budgets, m, q, colp, inf, s));
    MP_CUDA_TRY(project_fibers<float>(static_cast<const float*>(y), static_cast<float*>(x), n, m, q, norms, budgets,
                                      colp, l1, inf, flags, dtype, s));
  } else {
    MP_CUDA_TRY(launch_colparams<double>(norms, budgets, m, q, colp, inf, s));
    MP_CUDA_TRY(project_fibers<double>(static_cast<const double*>(y), static_cast<double*>(x), n, m, q, norms,
                                       budgets, colp, l1, inf, flags, dtype, s));
  }
  return MP_OK;
}

size_t mp_euclid_workspace_size(mp_dtype dtype, int64_t n, int64_t m) {
  if (n < 1 || m < 1 || !dtype_ok(dtype)) return 0;
  Carve c(nullptr, 0);
  carve_euclid(c, dtype, n, m);
  return c.off + 256;
}

mp_status mp_euclid_project(const void* y, void* x, mp_dtype dtype, int64_t n, int64_t m, double eta,
                            double* budgets, mp_info* info, unsigned flags, void* workspace, size_t workspace_bytes,
                            void* stream) {
  if (!dtype_ok(dtype)) return fail(MP_ERR_CONFIG, "unknown dtype code");
  if (n < 1 || m < 1) return fail(MP_ERR_SHAPE, "euclid_project_l1inf requires a non-empty order-2 tensor");
  if (!(eta >= 0.0) || !std::isfinite(eta)) return fail(MP_ERR_VALUE, "radius must be a finite nonnegative real");
  if (!y || !x || !workspace) return fail(MP_ERR_WORKSPACE, "null pointer");
  Carve c(workspace, workspace_bytes);
  EuclidWs w = carve_euclid(c, dtype, n, m);
  if (!c.fits()) return fail(MP_ERR_WORKSPACE, "mp_euclid_project: workspace too small");
  MP_CUDA_TRY(outer_setup());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == MP_F32)
    return euclid_impl<float>(static_cast<const float*>(y), static_cast<float*>(x), dtype, n, m, eta, budgets, info,
                              flags, w, s);
  return euclid_impl<double>(static_cast<const double*>(y), static_cast<double*>(x), dtype, n, m, eta, budgets, info,
                             flags, w, s);
}

size_t mp_aggregate_workspace_size(mp_dtype dtype, int64_t n, int64_t m, mp_norm q) {
  if (n < 1 || m < 1 || !dtype_ok(dtype) || !norm_ok(q)) return 0;
  return aggregate_scratch_bytes(dtype, n, m, q) + 256;
}

mp_status mp_aggregate(const void* t, double* out, mp_dtype dtype, int64_t n, int64_t m, mp_norm q, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (!dtype_ok(dtype)) return fail(MP_ERR_CONFIG, "unknown dtype code");
  if (!norm_ok(q)) return fail(MP_ERR_CONFIG, "unknown norm code");
  if (n < 1 || m < 1) return fail(MP_ERR_SHAPE, "aggregate requires a non-empty tensor of order >= 2");
  if (!t || !out || !workspace) return fail(MP_ERR_WORKSPACE, "null pointer");
  if (workspace_bytes < aggregate_scratch_bytes(dtype, n, m, q)) return fail(MP_ERR_WORKSPACE, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == MP_F32)
    return aggregate_impl<float>(static_cast<const float*>(t), out, dtype, n, m, q, workspace, s);
  return aggregate_impl<double>(static_cast<const double*>(t), out, dtype, n, m, q, workspace, s);
}

}  // extern "C"
