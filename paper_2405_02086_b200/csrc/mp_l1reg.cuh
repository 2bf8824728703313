// mp_l1reg.cuh -- K3b register-resident path: per-column l1-ball projection
// (the l_{1,1} apply pass, proj/src/fiber_kernels.cpp:56-65 ->
// project_l1_fast_inplace, proj/src/vector_balls.cpp:150-161) with the
// strip held ENTIRELY IN REGISTERS.
//
// One CTA of NT = 512 threads (128 / 256 for short columns, several CTAs per
// SM) owns a strip of W = 4P f32 (2P f64) adjacent columns over all
// n <= NT/P * 16 rows; thread t holds 16-byte piece t % P of rows
// t / P + (NT/P) i, i < 16 (64 registers of data, the whole register file
// of the SM for P = 2, n = 4096).  A warp instruction then touches 32/P rows
// of 16P bytes (P = 2: whole 32-byte sectors) instead of 32 lines for 16
// bytes each -- the L1 line rate, not HBM, bounds a 16-byte-per-row walk.
//  * y is read from HBM exactly once, all loads of a thread in flight,
//    issued BEFORE griddepcontrol.wait (no earlier kernel of the projection
//    writes y), overlapping K2;
//  * Michelot's fixed point (t <- (S(t) - u_j) / K(t), S, K over |y| > t)
//    runs over registers with full ILP; per pass a warp reduce-scatter and
//    one CTA barrier; the column lanes of every warp total the warp partials
//    in warp order (deterministic, identical in every warp);
//  * the apply shrinks the registers and stores the row pieces: no re-read;
//  * PERSIST (default): one CTA per SM walks strips grid-stride and streams
//    the next strip's row piece into each register right after storing it,
//    so the loads overlap the apply (a cp.async prefetch into shared memory
//    measured slower: 283 vs 256 us on config 3).
//
// Passes come in two kinds.  FAST (f32 strips, far from convergence): f32
// per-thread sums (an f32->f64 convert per element would cost more than the
// pass), f64 across threads, and a step to a rigorous LOWER bound of the
// exact iterate: a thread partial sums NPC <= 32 nonnegative f32 terms, the
// warp and CTA totals add 5 + NW more, so S >= S_exact (1 - 53 2^-24) and
// S_lo = S (1 - 2^-17), rounded down, is below S_exact; t' = RD((S_lo - RU(u_j)) / K) <= (S_exact - u_j) / K.
// Michelot from below stays below tau and the set only shrinks (f64 strips:
// f64 sums, the step nudged 2^-45 below).  EXACT (near convergence -- the
// count dropped by < 1/16): f64 sums, plus min |y| over the set.  With t_ex = (S - u_j) / K,
// the set is the fixed point {|y| > tau} iff min_set |y| > t_ex, and then
// tau_j = t_ex: the same fixed point (hence the reference's set
// {|y| >= cutoff}) that the exact iteration reaches -- one pass before it
// would see its count repeat.  Otherwise the exact step continues from t_ex.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "mp_cuda.h"
#include "mp_kernels.cuh"
#include "mp_l1cols.cuh"

namespace mpk {

constexpr int kRegRPT = 16;       // 16-byte row pieces per thread
constexpr int kRegThreads = 512;  // one CTA per SM (the register file)

template <typename T>
struct alignas(16) RegPart {
  double s;
  int k;
  T mn;
};

template <typename T>
__device__ __forceinline__ RegPart<T> rp_add(const RegPart<T>& a, const RegPart<T>& b) {
  return {a.s + b.s, a.k + b.k, a.mn < b.mn ? a.mn : b.mn};
}

template <typename T>
__device__ __forceinline__ RegPart<T> rp_shfl(const RegPart<T>& a, int o) {
  return {__shfl_xor_sync(0xffffffffu, a.s, o), __shfl_xor_sync(0xffffffffu, a.k, o),
          __shfl_xor_sync(0xffffffffu, a.mn, o)};
}

// Warp reduce-scatter of the C4 per-column partials of every 16-byte piece
// over the lanes sharing the piece (lane % P): xor 16, 8 split the columns,
// xor 4 .. P finish.  Afterwards lane l holds the warp total of strip column
// reg_col<T, P>(l) iff reg_writer<T, P>(l).  Fixed pattern => deterministic.
template <typename T, int P>
__device__ __forceinline__ int reg_col(int lane) {
  constexpr int C4 = 16 / sizeof(T);
  const int c = C4 == 4 ? ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1) : ((lane >> 4) & 1);
  return (lane & (P - 1)) * C4 + c;
}
template <typename T, int P>
__device__ __forceinline__ bool reg_writer(int lane) {
  constexpr int C4 = 16 / sizeof(T);
  constexpr int hi = C4 == 4 ? 7 : 15;  // bits still reduced after the split
  return (lane & (hi & ~(P - 1))) == 0;
}

// Fast-pass partial: f32 sum and count (exact: counts < 2^24).
struct FastPart {
  float s, k;
};
__device__ __forceinline__ FastPart rp_add(const FastPart& a, const FastPart& b) { return {a.s + b.s, a.k + b.k}; }
__device__ __forceinline__ FastPart rp_shfl(const FastPart& a, int o) {
  return {__shfl_xor_sync(0xffffffffu, a.s, o), __shfl_xor_sync(0xffffffffu, a.k, o)};
}

// f64 strips: f64 sum, f32 count.
struct FastPartD {
  double s;
  float k;
};
__device__ __forceinline__ FastPartD rp_add(const FastPartD& a, const FastPartD& b) { return {a.s + b.s, a.k + b.k}; }
__device__ __forceinline__ FastPartD rp_shfl(const FastPartD& a, int o) {
  return {__shfl_xor_sync(0xffffffffu, a.s, o), __shfl_xor_sync(0xffffffffu, a.k, o)};
}

// Field-wise select (a ternary on the aggregates would index the array with a
// runtime value and send it to local memory).
__device__ __forceinline__ FastPart rp_sel(bool p, const FastPart& a, const FastPart& b) {
  return {p ? a.s : b.s, p ? a.k : b.k};
}
__device__ __forceinline__ FastPartD rp_sel(bool p, const FastPartD& a, const FastPartD& b) {
  return {p ? a.s : b.s, p ? a.k : b.k};
}
template <typename T>
__device__ __forceinline__ RegPart<T> rp_sel(bool p, const RegPart<T>& a, const RegPart<T>& b) {
  return {p ? a.s : b.s, p ? a.k : b.k, p ? a.mn : b.mn};
}

template <int C4, int P, typename Part>
__device__ __forceinline__ Part reg_reduce(const Part (&a)[C4], int lane) {
  Part r;
  if constexpr (C4 == 4) {
    const bool h4 = lane & 16, h3 = lane & 8;
    const Part b0 = rp_add(rp_sel(h4, a[2], a[0]), rp_shfl(rp_sel(h4, a[0], a[2]), 16));
    const Part b1 = rp_add(rp_sel(h4, a[3], a[1]), rp_shfl(rp_sel(h4, a[1], a[3]), 16));
    r = rp_add(rp_sel(h3, b1, b0), rp_shfl(rp_sel(h3, b0, b1), 8));
#pragma unroll
    for (int o = 4; o >= P; o >>= 1) r = rp_add(r, rp_shfl(r, o));
  } else {
    const bool h4 = lane & 16;
    r = rp_add(rp_sel(h4, a[1], a[0]), rp_shfl(rp_sel(h4, a[0], a[1]), 16));
#pragma unroll
    for (int o = 8; o >= P; o >>= 1) r = rp_add(r, rp_shfl(r, o));
  }
  return r;
}

template <typename T>
__device__ __forceinline__ void reg_unpack(const uint4& q, T (&e)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 4) {
    e[0] = __uint_as_float(q.x); e[1 % (16 / sizeof(T))] = __uint_as_float(q.y);
    e[2 % (16 / sizeof(T))] = __uint_as_float(q.z); e[3 % (16 / sizeof(T))] = __uint_as_float(q.w);
  } else {
    e[0] = __hiloint2double(static_cast<int>(q.y), static_cast<int>(q.x));
    e[1 % (16 / sizeof(T))] = __hiloint2double(static_cast<int>(q.w), static_cast<int>(q.z));
  }
}

template <typename T>
__device__ __forceinline__ uint4 reg_pack(const T (&e)[16 / sizeof(T)]) {
  if constexpr (sizeof(T) == 4) {
    return make_uint4(__float_as_uint(e[0]), __float_as_uint(e[1 % 4]), __float_as_uint(e[2 % 4]),
                      __float_as_uint(e[3 % 4]));
  } else {
    const double a = e[0], b = e[1 % 2];
    return make_uint4(static_cast<unsigned>(__double2loint(a)), static_cast<unsigned>(__double2hiint(a)),
                      static_cast<unsigned>(__double2loint(b)), static_cast<unsigned>(__double2hiint(b)));
  }
}

// TMA (cp.async.bulk.tensor) helpers for the shared-memory half of a hybrid
// strip: 2-D boxes of 8 columns x 256 rows move between global memory and
// the [rows][8] shared-memory layout, which for P = 2, NT = 256 is exactly
// the thread-private slot layout sq[i * NT + tid] (thread t holds row
// t / 2, 16-byte half t % 2).  The copies bypass the LSU: a 32-byte-wide
// strip row costs one L1 transaction per row piece on the LSU path.
struct TmaMaps {
  CUtensorMap y, x;
};
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}

// Estimate of the l1 threshold tau of a column with l1 norm v and budget
// u < v under a half-normal model of |y| (E|y| = v / n, sigma = E|y| sqrt(pi/2)):
// the root z of n sigma g(z) = u, g(z) = E max(|Z| - z, 0) = 2 phi(z) -
// z erfc(z / sqrt2), read from a table of z at c = g(0) 2^(-k/4), k = 0..120
// (generated offline by bisection), linearly interpolated in log2 c; tau ~
// z sigma.  Only a starting point: the first pass probes it and steps to the
// Michelot iterate from it, which is a LOWER bound of tau whichever side of
// tau the probe lies (for the set A of entries above any t, m = (S_A - u)/|A|
// gives sum_A (|y| - m) = u, so sum_all max(|y| - m, 0) >= u: m <= tau).
// N(0,1) columns: 6.1 -> 4.1 passes per strip.  (Newton on erfc in the
// kernel cost 15% of its instructions.)
__device__ const float kHalfNormalZ[121] = {
    0.000000f, 0.134111f, 0.260645f, 0.380545f, 0.494589f, 0.603428f, 0.707609f, 0.807596f,
    0.903789f, 0.996531f, 1.086120f, 1.172815f, 1.256847f, 1.338416f, 1.417702f, 1.494865f,
    1.570048f, 1.643379f, 1.714974f, 1.784939f, 1.853368f, 1.920349f, 1.985961f, 2.050277f,
    2.113363f, 2.175282f, 2.236090f, 2.295840f, 2.354580f, 2.412355f, 2.469209f, 2.525179f,
    2.580304f, 2.634616f, 2.688149f, 2.740932f, 2.792994f, 2.844361f, 2.895059f, 2.945111f,
    2.994539f, 3.043366f, 3.091610f, 3.139291f, 3.186427f, 3.233035f, 3.279131f, 3.324731f,
    3.369849f, 3.414500f, 3.458696f, 3.502452f, 3.545778f, 3.588686f, 3.631188f, 3.673295f,
    3.715016f, 3.756362f, 3.797342f, 3.837965f, 3.878239f, 3.918173f, 3.957776f, 3.997054f,
    4.036015f, 4.074667f, 4.113016f, 4.151069f, 4.188833f, 4.226313f, 4.263516f, 4.300447f,
    4.337113f, 4.373517f, 4.409667f, 4.445566f, 4.481219f, 4.516633f, 4.551810f, 4.586755f,
    4.621474f, 4.655969f, 4.690246f, 4.724307f, 4.758157f, 4.791800f, 4.825239f, 4.858478f,
    4.891520f, 4.924368f, 4.957026f, 4.989497f, 5.021784f, 5.053889f, 5.085817f, 5.117569f,
    5.149148f, 5.180558f, 5.211800f, 5.242877f, 5.273792f, 5.304548f, 5.335145f, 5.365588f,
    5.395878f, 5.426017f, 5.456008f, 5.485852f, 5.515551f, 5.545109f, 5.574526f, 5.603804f,
    5.632946f, 5.661953f, 5.690827f, 5.719570f, 5.748184f, 5.776670f, 5.805029f, 5.833264f,
    5.861376f};
__device__ __forceinline__ float halfnormal_tau(double v, double u, int n) {
  const float sig = static_cast<float>(v / n) * 1.25331414f;  // sqrt(pi/2)
  const float c = static_cast<float>(u / (static_cast<double>(n) * sig));
  const float r = 4.0f * __log2f(0.79788456f / c);
  if (!(r > 0.0f)) return 0.0f;
  if (!(r < 120.0f)) return __ldg(&kHalfNormalZ[120]) * sig;
  const int k = static_cast<int>(r);
  const float z0 = __ldg(&kHalfNormalZ[k]), z1 = __ldg(&kHalfNormalZ[k + 1]);
  return fmaf(r - static_cast<float>(k), z1 - z0, z0) * sig;
}

// Compiler barrier that keeps four pieces live in distinct registers.
__device__ __forceinline__ void pin_regs(uint4& a, uint4& b, uint4& c, uint4& d) {
  asm volatile("" : "+r"(a.x), "+r"(a.y), "+r"(a.z), "+r"(a.w), "+r"(b.x), "+r"(b.y), "+r"(b.z), "+r"(b.w),
                    "+r"(c.x), "+r"(c.y), "+r"(c.z), "+r"(c.w), "+r"(d.x), "+r"(d.y), "+r"(d.z), "+r"(d.w)
               :
               : "memory");
}

template <typename T, int P, bool DERIVE, bool PERSIST, int NT = kRegThreads, int RS = 0, bool TMA = false>
__global__ void __launch_bounds__(NT, kRegThreads / NT)
    k_l1reg(const T* __restrict__ y, T* __restrict__ x, int n, int64_t m, const double* __restrict__ v,
            const double* __restrict__ u, double* __restrict__ tau_out, const mp_info* __restrict__ info,
            const OuterParams* __restrict__ params, double* __restrict__ u_out, int64_t nstrips,
            const __grid_constant__ TmaMaps tm) {
  constexpr int C4 = 16 / sizeof(T);
  constexpr int W = C4 * P;  // strip columns
  constexpr int NW = NT / 32;
  constexpr int SL = NT / P;  // row slots
  // TMA strips keep 32 - RS pieces per thread in registers (the rest in
  // shared memory, moved by TMA); the others kRegRPT
  constexpr int RPT = TMA ? 32 - RS : kRegRPT;
  constexpr bool kF32 = sizeof(T) == 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t strip = blockIdx.x;
  const int pc = (tid % P) * C4;  // this thread's first strip column
  const int rb = tid / P;         // this thread's first row
  const int64_t step = static_cast<int64_t>(SL) * m;

  // RS > 0: the strip's last RS pieces per thread live in shared memory
  // ([RS][NT] uint4, each thread lands and reads back only its own), the
  // first RPT in registers -- half the registers per strip, two CTAs per SM.
  extern __shared__ __align__(128) uint4 sq[];
  constexpr int NPC = RPT + RS;  // pieces per thread
  static_assert(!TMA || (RS > 0 && P == 2), "TMA strips: P = 2 (32-byte rows)");
  static_assert(!TMA || (RS * (NT / P)) % 256 == 0, "TMA strips: whole 256-row boxes");
  constexpr int kBoxRows = 256, kBoxes = RS * SL / kBoxRows;
  __shared__ unsigned long long mbar;
  unsigned mph = 0;  // mbarrier phase of the next landing
  if constexpr (TMA) {
    if (tid == 0) {
      mbar_init(&mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  auto land_smem = [&](int64_t s_strip) {
    if constexpr (TMA) {
      if (tid == 0) {
        mbar_expect(&mbar, static_cast<unsigned>(RS * NT * 16));
#pragma unroll
        for (int b = 0; b < kBoxes; ++b)
          tma_load_2d(reinterpret_cast<char*>(sq) + b * kBoxRows * W * sizeof(T), &tm.y,
                      static_cast<int>(s_strip * W), SL * RPT + b * kBoxRows, &mbar);
      }
    } else if constexpr (RS > 0) {
      const T* yp = y + static_cast<int64_t>(rb + SL * RPT) * m + s_strip * W + pc;
#pragma unroll
      for (int i = 0; i < RS; ++i, yp += step) {
        if (rb + SL * (RPT + i) < n) cp_async_16(&sq[i * NT + tid], yp);
        else sq[i * NT + tid] = make_uint4(0, 0, 0, 0);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  };
  // Land the first strip: y is not written by K1 / K2.
  uint4 q[RPT];
  {
    const T* yp = y + static_cast<int64_t>(rb) * m + strip * W + pc;
#pragma unroll
    for (int i = 0; i < RPT; ++i, yp += step)
      q[i] = rb + SL * i < n ? __ldg(reinterpret_cast<const uint4*>(yp)) : make_uint4(0, 0, 0, 0);
  }
  land_smem(strip);
  pdl_wait();
  tl_begin(3);
  if (info->status != MP_OK) {
    // drain the copies already aimed at this CTA's shared memory before it
    // is released (another resident CTA may reuse it)
    if constexpr (TMA) mbar_wait(&mbar, mph);
    else if constexpr (RS > 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
    return;
  }

  auto piece = [&](int i) -> uint4 {  // i is a compile-time index after unrolling
    if (RS == 0 || i < RPT) return q[i < RPT ? i : 0];
    return sq[(i - RPT) * NT + tid];
  };
  using FP = std::conditional_t<kF32, FastPart, FastPartD>;  // fast-pass partial
  using AccT = std::conditional_t<kF32, float, double>;
  __shared__ FP wf[2][NW][W];
  __shared__ RegPart<T> wx[2][NW][W];
  const double inv_n = 1.0 / static_cast<double>(n);
  int npass = 0, nx = 0, nst = 0;
#ifdef MP_L1_CYCLES  // profiling build: per-phase SM cycles of thread 0 (slots 12..15)
  long long cyw = 0, cyp = 0, cya = 0, cyx = 0;
#endif
  // (Strips claimed from a global counter instead of the static stride:
  // 143 vs 137.6 us on config 3 -- with the stride, neighbouring strips are
  // in flight together and share the 256-byte L2 promotions of their rows.)
  for (;;) {
    ++nst;
    const int64_t cb = strip * W + pc;
    // strip column `lane` (< W): iteration state, identical in every warp;
    // the threads' own columns (pc .. pc + C4 - 1) come from these lanes by
    // shuffles (no per-thread f64 divisions)
    double ul = 0.0, td = -1.0;
    float uup = 0.0f;  // RU(u_j)
    int kp = n + 1;
    bool lv = false, ex = false, pj = false;
    unsigned kdl = 0;  // column kind: 1 feasible, 2 zero budget, 3 project
    T t1 = T(INFINITY);  // first-pass threshold
    if (lane < W) {
      const double vj = v[strip * W + lane];
      ul = DERIVE ? derive_u(*params, vj) : u[strip * W + lane];
      uup = __double2float_ru(ul);
      kdl = vj <= ul ? 1u : (ul == 0.0 ? 2u : 3u);
      pj = lv = kdl == 3u;
      if (pj) {
        // first iterate from the norm pass, nudged below the rounding of v_j,
        // and the speculative first probe (halfnormal_tau)
        td = (vj * (1.0 - 0x1p-40) - ul) * inv_n;
        t1 = round_down_to(T(0), fmax(td, static_cast<double>(halfnormal_tau(vj, ul, n))));
      }
      if (DERIVE && u_out && warp == 0) u_out[strip * W + lane] = ul;
    }
    unsigned kinds = 0;
    T thr[C4];
#pragma unroll
    for (int c = 0; c < C4; ++c) {
      const unsigned kd = __shfl_sync(0xffffffffu, kdl, pc + c);
      kinds |= kd << (2 * c);
      thr[c] = __shfl_sync(0xffffffffu, t1, pc + c);
    }
#ifdef MP_L1_CYCLES
    const long long ck0 = clock64();
#endif
    const bool any_proj = __any_sync(0xffffffffu, pj);
    if constexpr (TMA) {
      mbar_wait(&mbar, mph);
      mph ^= 1u;
    } else if constexpr (RS > 0) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }

#ifdef MP_L1_CYCLES
    const long long ck1 = clock64();
#endif
    if (any_proj) {
      bool xp = false;  // exact pass (CTA-uniform)
      for (int par = 0, it = 0; it < 4 * 1024; par ^= 1, ++it) {
        ++npass;
        nx += xp;
        // Pieces outer, columns inner: each piece (a shared-memory load for the
        // hybrid part) is read once per pass and feeds C4 independent chains;
        // every column still sums its pieces in ascending i.
        if (!xp) {
          FP a[C4];
          T th[C4];
#pragma unroll
          for (int c = 0; c < C4; ++c) {
            a[c] = {AccT(0), 0.0f};
            th[c] = thr[c];  // +inf for columns that are not (or no longer) projected
          }
#pragma unroll
          for (int i = 0; i < NPC; ++i) {
            T e[C4];
            reg_unpack<T>(piece(i), e);
#pragma unroll
            for (int c = 0; c < C4; ++c) {
              const T ab = kF32 ? fabsf(e[c]) : fabs(e[c]);
              if (ab > th[c]) {
                a[c].s += ab;
                a[c].k += 1.0f;
              }
            }
          }
          const FP wr = reg_reduce<C4, P>(a, lane);
          if (reg_writer<T, P>(lane)) wf[par][warp][reg_col<T, P>(lane)] = wr;
        } else {
          RegPart<T> a[C4];
          T th[C4];
#pragma unroll
          for (int c = 0; c < C4; ++c) {
            a[c] = {0.0, 0, T(INFINITY)};
            th[c] = thr[c];  // +inf for columns that are not (or no longer) projected
          }
#pragma unroll
          for (int i = 0; i < NPC; ++i) {
            T e[C4];
            reg_unpack<T>(piece(i), e);
#pragma unroll
            for (int c = 0; c < C4; ++c) {
              const T ab = kF32 ? fabsf(e[c]) : fabs(e[c]);
              if (ab > th[c]) {
                a[c].s += static_cast<double>(ab);
                ++a[c].k;
                a[c].mn = ab < a[c].mn ? ab : a[c].mn;
              }
            }
          }
          const RegPart<T> wr = reg_reduce<C4, P>(a, lane);
          if (reg_writer<T, P>(lane)) wx[par][warp][reg_col<T, P>(lane)] = wr;
        }
        __syncthreads();
        if (lane < W && lv) {
          // column totals over the warps, in warp order
          RegPart<T> tot;
          if (xp) {
            // a fixed pairwise tree (log2 NW dependent f64 adds instead of
            // NW - 1: the epilogue of a pass is a latency chain)
            RegPart<T> tw[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) tw[w] = wx[par][w][lane];
#pragma unroll
            for (int o = 1; o < NW; o <<= 1) {
#pragma unroll
              for (int w = 0; w + o < NW; w += 2 * o) tw[w] = rp_add(tw[w], tw[w + o]);
            }
            tot = tw[0];
          } else {
            AccT s32 = AccT(0);  // f32: <= NPC + 5 + NW f32 terms per sum
            float k32 = 0.0f;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
              const FP f = wf[par][w][lane];
              s32 += f.s;
              k32 += f.k;
            }
            tot = {static_cast<double>(s32), static_cast<int>(k32), T(INFINITY)};
          }
          if (it == 0) {
            // the speculative pass: Michelot step m1 from t1 (a lower bound of
            // tau_j whichever side of tau_j t1 lies); counts are not
            // comparable with the later passes' (t1 may exceed tau_j).  A
            // probe within 2^-5 of its own Michelot image is next to the
            // fixed point: confirm exactly from m1 at once.  Config 3 K3b:
            // 155 -> 143.6 us (2.93 passes per strip, 1.93 exact; one fast
            // step before the confirm: 145.3 us, 3.09 passes, 1.09 exact).
            if (tot.k > 0) {
              double m1;
              if constexpr (kF32) {
                const float xs = __fsub_rd(__fmul_rd(__double2float_rd(tot.s), 1.0f - 0x1p-17f), uup);
                m1 = xs > 0.0f ? static_cast<double>(__fmul_rd(xs, __frcp_rd(static_cast<float>(tot.k)))) : 0.0;
              } else {
                m1 = (tot.s * (1.0 - 0x1p-45) - ul) / static_cast<double>(tot.k);
              }
              td = fmax(td, m1);
              if (fabs(static_cast<double>(t1) - m1) <= 0x1p-5 * m1) ex = true;
            }
          } else if (tot.k == 0) {
            lv = false;  // cannot happen for 0 < u_j < v_j; keep the threshold
          } else if (xp) {
            const double tex = (tot.s - ul) / static_cast<double>(tot.k);
            if (tot.mn > round_down_to(T(0), tex)) {
              td = tex;  // the fixed point: tau_j
              lv = false;
            } else {
              td = fmax(td, tex);
              kp = tot.k;
            }
          } else {
            if constexpr (kF32) {
              // a rigorous lower bound of (S_exact - u_j) / K: the f32 sums
              // carry < (NPC + 5 + NW) * 2^-24 <= 53 * 2^-24 relative error,
              // the margin is 2^-17
              const float xs = __fsub_rd(__fmul_rd(__double2float_rd(tot.s), 1.0f - 0x1p-17f), uup);
              const float tn = xs > 0.0f ? __fmul_rd(xs, __frcp_rd(static_cast<float>(tot.k))) : 0.0f;
              td = fmax(td, static_cast<double>(tn));
            } else {
              // f64 sums of f64 data: the Michelot step, nudged below rounding
              td = fmax(td, (tot.s * (1.0 - 0x1p-45) - ul) / static_cast<double>(tot.k));
            }
            if ((kp - tot.k) * 16 <= tot.k) ex = true;  // near convergence: exact steps from here
            kp = tot.k;
          }
        }
        const T tl = lv ? round_down_to(T(0), td) : T(INFINITY);
#pragma unroll
        for (int c = 0; c < C4; ++c) thr[c] = __shfl_sync(0xffffffffu, tl, pc + c);
        const unsigned lvb = __ballot_sync(0xffffffffu, lv);
        if (lvb == 0u) break;
        xp = xp || __ballot_sync(0xffffffffu, lv && ex) != 0u;
      }
    }
#ifdef MP_L1_CYCLES
    const long long ck2 = clock64();
#endif
    if (warp == 0 && lane < W) tau_out[strip * W + lane] = pj ? td : -1.0;

    // ---- apply from registers
    bool need_store = any_proj || x != y;
#pragma unroll
    for (int c = 0; c < C4; ++c) need_store = need_store || ((kinds >> (2 * c)) & 3u) == 2u;
    need_store = __syncthreads_or(need_store);
    // PERSIST: stream the next strip into each register right after its
    // store, so its loads overlap this strip's apply
    const int64_t next = strip + gridDim.x;
    const bool more = PERSIST && next < nstrips;
    // One branch-free rule for every column kind: d = (|y| - tau_hi) - tau_lo;
    // x = d > 0 ? copysign(d, y) : (y & keep).  Feasible columns: tau = 0 and
    // keep = all ones (d = |y| exactly, zeros keep their sign: x = y);
    // zero budget: tau = +inf, keep = 0 (+0.0); projected: tau_j, keep = 0
    // (the soft threshold's +0.0, proj/src/vector_balls.cpp:42-48).
    using UT = std::conditional_t<kF32, unsigned, unsigned long long>;
    T th_hi[C4], th_lo[C4];
    UT keep[C4];
#pragma unroll
    for (int c = 0; c < C4; ++c) {
      const double tc = __shfl_sync(0xffffffffu, td, pc + c);
      const unsigned kd = (kinds >> (2 * c)) & 3u;
      keep[c] = kd == 1u ? ~UT(0) : UT(0);
      if constexpr (kF32) {
        const TauPair tq{__double2float_rn(tc), __double2float_rn(tc - static_cast<double>(__double2float_rn(tc)))};
        th_hi[c] = kd == 1u ? 0.0f : (kd == 2u ? INFINITY : tq.hi);
        th_lo[c] = kd == 3u ? tq.lo : 0.0f;
      } else {
        th_hi[c] = kd == 1u ? 0.0 : (kd == 2u ? static_cast<double>(INFINITY) : tc);
        th_lo[c] = 0.0;
      }
    }
    T* xq = x + static_cast<int64_t>(rb) * m + cb;
    const T* yn = y + static_cast<int64_t>(rb) * m + next * W + pc;
    auto shrink = [&](const uint4& qv) -> uint4 {
      T e[C4];
      reg_unpack<T>(qv, e);
#pragma unroll
      for (int c = 0; c < C4; ++c) {
        if constexpr (kF32) {
          const float dm = shrink_mag(fabsf(e[c]), TauPair{th_hi[c], th_lo[c]});
          e[c] = dm > 0.0f ? copysignf(dm, e[c]) : __uint_as_float(__float_as_uint(e[c]) & keep[c]);
        } else {
          const double dm = fabs(e[c]) - th_hi[c];
          e[c] = dm > 0.0 ? copysign(dm, e[c])
                          : __longlong_as_double(static_cast<long long>(
                                static_cast<UT>(__double_as_longlong(e[c])) & keep[c]));
        }
      }
      return reg_pack<T>(e);
    };
    // the register pieces of a TMA strip: rewritten in place, stored back to
    // back from their own registers, then the next strip's loaded over them
    auto reg_pieces = [&]() {
      if (need_store) {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          if (rb + SL * i < n) q[i] = shrink(q[i]);
        // all results live at once, each in its own registers (the compiler
        // would stage every piece through the same four otherwise)
        static_assert(!TMA || RPT <= 8, "pin_regs: up to eight pieces");
        pin_regs(q[0], q[1 % RPT], q[2 % RPT], q[3 % RPT]);
        if constexpr (RPT > 4) pin_regs(q[4 % RPT], q[5 % RPT], q[6 % RPT], q[7 % RPT]);
        pin_regs(q[0], q[1 % RPT], q[2 % RPT], q[3 % RPT]);
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          if (rb + SL * i < n) __stcs(reinterpret_cast<uint4*>(xq + static_cast<int64_t>(i) * step), q[i]);
      }
      if (more) {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          if (rb + SL * i < n) q[i] = __ldg(reinterpret_cast<const uint4*>(yn + static_cast<int64_t>(i) * step));
      }
    };
    // 256- and 512-thread strips (64 / 128 threads measured 1-2% slower)
    constexpr bool kSplit = TMA && NT >= 256;
    if constexpr (kSplit) {
      // A global store holds its source registers for hundreds of cycles while
      // the memory system is busy with the strips' TMA traffic (ncu: ~800
      // cycles of long-scoreboard stall on the next write to them, six times
      // per strip), and fence.proxy.async waits for the stores in flight.  So
      // the shared-memory pieces go first and their TMA stores are issued
      // before the register pieces touch global memory.
      if (need_store) {
#pragma unroll
        for (int i = RPT; i < NPC; ++i) {
          if (rb + SL * i >= n) break;
          sq[(i - RPT) * NT + tid] = shrink(sq[(i - RPT) * NT + tid]);  // TMA stores it
        }
      }
    } else {
      // (register-only strips measured 5-20% slower with the split order --
      // their next strip's loads would start only after all the stores -- and
      // 6-13% slower with in-place stores and the loads lagging 2-4 pieces)
#pragma unroll
      for (int i = 0; i < NPC; ++i, xq += step, yn += step) {
        if (rb + SL * i >= n) break;
        if (need_store) {
          const uint4 r = shrink(piece(i));
          if (TMA && i >= RPT) sq[(i >= RPT ? i - RPT : 0) * NT + tid] = r;  // TMA stores it
          else __stcs(reinterpret_cast<uint4*>(xq), r);
        }
        if (more) {
          if (i < RPT) q[i < RPT ? i : 0] = __ldg(reinterpret_cast<const uint4*>(yn));
          else if constexpr (RS > 0 && !TMA) cp_async_16(&sq[(i - RPT) * NT + tid], yn);
        }
      }
    }
    if constexpr (TMA) {
      // the shared-memory half goes out by TMA; once the engine has read it,
      // the next strip's half lands in the same buffer
      if (need_store) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
#ifdef MP_L1_CYCLES
      cyx += clock64() - ck2;
#endif
      // up to four store groups: each group's boxes reload as soon as the
      // engine has read them, while the later groups are still being read
      // (one group: 179 us on config 3, two or four: 173 us).  Group g is
      // boxes [g * kBoxes / kG, (g + 1) * kBoxes / kG); 64-thread strips
      // have three boxes, hence three groups.
      constexpr int kG = kBoxes < 4 ? kBoxes : 4;
      static_assert(kG >= 1, "TMA strips: at least one box");
      if (tid == 0 && need_store) {
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          for (int b = g * kBoxes / kG; b < (g + 1) * kBoxes / kG; ++b)
            tma_store_2d(&tm.x, static_cast<int>(strip * W), SL * RPT + b * kBoxRows,
                         reinterpret_cast<const char*>(sq) + b * kBoxRows * W * sizeof(T));
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if constexpr (kSplit) reg_pieces();
      if (tid == 0) {
        auto load = [&](int b0, int b1) {
          for (int b = b0; b < b1; ++b)
            tma_load_2d(reinterpret_cast<char*>(sq) + b * kBoxRows * W * sizeof(T), &tm.y,
                        static_cast<int>(next * W), SL * RPT + b * kBoxRows, &mbar);
        };
        if (more) mbar_expect(&mbar, static_cast<unsigned>(RS * NT * 16));
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          // groups still allowed in flight: kG - 1 - g (wait_group takes an immediate)
          if (need_store) {
            if (kG - 1 - g == 3) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
            else if (kG - 1 - g == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
            else if (kG - 1 - g == 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          if (more) load(g * kBoxes / kG, (g + 1) * kBoxes / kG);
        }
      }
    } else if constexpr (RS > 0) {
      if (more) {
        // rows past n of the next strip: zero pieces (none when n fills the slots)
#pragma unroll
        for (int i = 0; i < RS; ++i)
          if (rb + SL * (RPT + i) >= n) sq[i * NT + tid] = make_uint4(0, 0, 0, 0);
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
    }
#ifdef MP_L1_CYCLES
    {
      const long long ck3 = clock64();
      cyw += ck1 - ck0;
      cyp += ck2 - ck1;
      cya += ck3 - ck2;
    }
#endif
    if (!more) break;
    strip = next;
  }
  if (tid == 0 && g_mp_timeline) {  // profiling aid: passes, max per CTA, strips, exact passes (8..11)
    atomicAdd(g_mp_timeline + 8, static_cast<unsigned long long>(npass));
    atomicAdd(g_mp_timeline + 11, static_cast<unsigned long long>(nx));
    atomicMax(g_mp_timeline + 9, static_cast<unsigned long long>(npass));
    atomicAdd(g_mp_timeline + 10, static_cast<unsigned long long>(nst));
#ifdef MP_L1_CYCLES
    atomicAdd(g_mp_timeline + 12, static_cast<unsigned long long>(cyw));
    atomicAdd(g_mp_timeline + 13, static_cast<unsigned long long>(cyp));
    atomicAdd(g_mp_timeline + 14, static_cast<unsigned long long>(cya));
    atomicAdd(g_mp_timeline + 15, static_cast<unsigned long long>(cyx));
#endif
  }
  if constexpr (TMA) {
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  }
  tl_end(3);
}

// Geometry of the register path.  A CTA of NT threads (128 / 256 / 512, so
// 4 / 2 / 1 CTAs per SM by registers) holds (NT/P) * (16 + RS) rows: 16 row
// pieces per thread in registers and, for the hybrid strips (RS = 16, P = 2),
// 16 more in shared memory.  Preference: registers only with >= 2 CTAs per
// SM (several CTAs per SM overlap one CTA's per-pass barrier and reduction
// with another's pass), smallest CTA and widest P >= 2 first; then hybrid
// strips; then one 512-thread CTA per SM; P = 1 (16-byte rows, L1-line-rate
// bound) only when nothing else fits.  Measured K3b: 256x65536 207 -> 57 us;
// 1000x16384 74 -> 56; 2000x32768 240 -> 211; 4096x16384 255 -> 206 (hybrid,
// 2 CTAs per SM); 6000x8192 201 us.  P = 0 when the path does not apply.
constexpr int kRegHybridRS = 16;
// TMA strips: shared-memory pieces per thread (of 32).  RS * (NT / 2) rows
// must be whole 256-row boxes -- the mbarrier expects RS * NT * 16 bytes.
// 256 / 512 threads: 26 (config 3 K3b 172.8 -> 169.5 us vs 24); 128: 24.
constexpr int tma_rs(int nt) { return nt == 128 ? 24 : 26; }
struct RegGeom {
  int P = 0, NT = 0, RS = 0;
};
template <typename T>
inline RegGeom l1reg_geometry(int64_t n, int64_t m, int cap) {
  constexpr int C4 = 16 / sizeof(T);
  auto fits = [&](int P, int nt, int rs) {
    return (cap <= 0 || P <= cap) && n <= static_cast<int64_t>(nt / P) * (kRegRPT + rs) && m % (C4 * P) == 0;
  };
  for (int nt = 128; nt < kRegThreads; nt *= 2)  // registers only, >= 2 CTAs per SM
    for (int P = 8; P >= 2; P >>= 1)
      if (fits(P, nt, 0)) return {P, nt, 0};
  for (int nt = 128; nt <= kRegThreads; nt *= 2)  // hybrid before a lone CTA per SM
    if (fits(2, nt, kRegHybridRS)) return {2, nt, kRegHybridRS};
  for (int P = 8; P >= 2; P >>= 1)
    if (fits(P, kRegThreads, 0)) return {P, kRegThreads, 0};
  for (int nt = 128; nt <= kRegThreads; nt *= 2)
    if (fits(1, nt, 0)) return {1, nt, 0};
  return {};
}

}  // namespace mpk
