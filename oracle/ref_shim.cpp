// ref_shim.cpp -- extern "C" entry points into the UNMODIFIED reference
// library (TEST INFRASTRUCTURE / CPU BASELINE ONLY).
//
// oracle/Makefile compiles this file together with the reference sources
// where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/libmultiproj_ref.so.  No reference source is copied into the
// repo.  Used by tests/ to pin the C restatement (oracle/mp_oracle.c) and the
// golden fixtures, and by bench.py's cpu_baseline / --impl reference legs to
// time the reference's own CPU path.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <vector>

#include "multiproj/bilevel.hpp"
#include "multiproj/bench.hpp"
#include "multiproj/errors.hpp"
#include "multiproj/tensor_io.hpp"
#include "multiproj/euclidean.hpp"
#include "multiproj/multilevel.hpp"
#include "multiproj/parallel.hpp"
#include "multiproj/rng.hpp"
#include "multiproj/tensor.hpp"
#include "multiproj/vector_balls.hpp"

using namespace multiproj;

namespace {

Norm to_norm(int q) {
  return q == 0 ? Norm::L1 : (q == 1 ? Norm::L2 : Norm::Inf);
}

// 1 ValueError, 2 ShapeError, 3 ConfigError, 9 anything else.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValueError&) {
    return 1;
  } catch (const ShapeError&) {
    return 2;
  } catch (const ConfigError&) {
    return 3;
  } catch (...) {
    return 9;
  }
}

std::unique_ptr<ThreadPool> make_pool(int workers) {
  if (workers > 1) return std::make_unique<ThreadPool>(static_cast<unsigned>(workers));
  return nullptr;
}

}  // namespace

extern "C" {

int ref_bilevel(const double* y, int64_t n, int64_t m, int p, int q,
                double eta, int workers, double* x, double* budgets,
                int64_t* zero_columns) {
  return guarded([&] {
    DenseTensor t({static_cast<size_t>(n), static_cast<size_t>(m)},
                  std::vector<double>(y, y + n * m));
    auto pool = make_pool(workers);
    BilevelResult r = bilevel_project(t, to_norm(p), to_norm(q), eta, pool.get());
    std::memcpy(x, r.X.data().data(), sizeof(double) * n * m);
    std::memcpy(budgets, r.budgets.data(), sizeof(double) * m);
    *zero_columns = static_cast<int64_t>(r.zero_columns);
  });
}

// Time `reps` calls of bilevel_project on an fp32 buffer upcast once to a
// DenseTensor (as bench_one does, proj/src/bench.cpp:54-91: the timed call
// includes the API's own output allocation and copy).  Writes each call's
// seconds to times[].
int ref_time_bilevel(const float* y32, int64_t n, int64_t m, int p, int q,
                     const double* etas, int n_etas, int reps, int workers,
                     double* times) {
  return guarded([&] {
    std::vector<double> d(y32, y32 + n * m);
    DenseTensor t({static_cast<size_t>(n), static_cast<size_t>(m)}, std::move(d));
    auto pool = make_pool(workers);
    int idx = 0;
    for (int r = 0; r < reps; ++r)
      for (int e = 0; e < n_etas; ++e) {
        auto t0 = std::chrono::steady_clock::now();
        BilevelResult res = bilevel_project(t, to_norm(p), to_norm(q), etas[e], pool.get());
        auto t1 = std::chrono::steady_clock::now();
        times[idx++] = std::chrono::duration<double>(t1 - t0).count();
        (void)res;
      }
  });
}

// Host formats / generator / records (proj/src/tensor_io.cpp, rng.cpp,
// bench.cpp:200-266): the drop-in must read and write the same bytes.
int ref_write_uniform_tensor(const char* path, const int64_t* shape, int order, uint64_t seed, double lo, double hi,
                             uint64_t* checksum) {
  return guarded([&] {
    std::vector<size_t> sh(shape, shape + order);
    DenseTensor t = gen_uniform_tensor(sh, seed, lo, hi);
    write_tensor(t, path);
    *checksum = tensor_checksum(t);
  });
}

int ref_read_tensor_checksum(const char* path, uint64_t* checksum, int64_t* size) {
  return guarded([&] {
    DenseTensor t = read_tensor(path);
    *checksum = tensor_checksum(t);
    *size = static_cast<int64_t>(t.size());
  });
}

int ref_rng_stream(uint64_t seed, int count, uint64_t* raw, double* normals) {
  return guarded([&] {
    Xoshiro256pp a(seed), b(seed);
    for (int i = 0; i < count; ++i) raw[i] = a.next();
    for (int i = 0; i < count; ++i) normals[i] = b.normal();
  });
}

// Two records, one with a comma-carrying multilevel tag, through the
// reference writer.
int ref_write_records_sample(const char* path) {
  return guarded([&] {
    BenchRecord a;
    a.algorithm = "bilevel-l1inf";
    a.n = 10;
    a.m = 20;
    a.radius = 0.1;
    a.workers = 4;
    a.repetitions = 3;
    a.median_seconds = 1.0 / 3.0;
    a.achieved_norm = 0.1;
    a.zero_columns = 7;
    a.output_checksum = 0xfedcba9876543210ULL;
    BenchRecord b = a;
    b.algorithm = "multilevel:inf,inf,1";
    b.extra_dims = {3, 5};
    b.median_seconds = 2.5e-7;
    write_csv_records({a, b}, path);
  });
}

// euclid_project_l1inf (proj/src/euclidean.cpp:82-170).
int ref_euclid(const double* y, int64_t n, int64_t m, double eta, double* x, double* budgets, double* theta) {
  return guarded([&] {
    DenseTensor t({static_cast<size_t>(n), static_cast<size_t>(m)}, std::vector<double>(y, y + n * m));
    EuclidResult r = euclid_project_l1inf(t, eta);
    std::memcpy(x, r.X.data().data(), sizeof(double) * n * m);
    std::memcpy(budgets, r.sol.budgets.data(), sizeof(double) * m);
    *theta = r.sol.theta;
  });
}

// budget_oracle_grid / clip_cost (proj/src/euclidean.cpp:64-80,172-240).
int ref_budget_grid(const double* y, int64_t n, int64_t m, double eta, int64_t steps, double* budgets, double* theta) {
  return guarded([&] {
    DenseTensor t({static_cast<size_t>(n), static_cast<size_t>(m)}, std::vector<double>(y, y + n * m));
    ColumnBudgetSolution s = budget_oracle_grid(t, eta, static_cast<std::size_t>(steps));
    std::memcpy(budgets, s.budgets.data(), sizeof(double) * m);
    *theta = s.theta;
  });
}

double ref_clip_cost(const double* y, int64_t n, int64_t m, const double* budgets) {
  DenseTensor t({static_cast<size_t>(n), static_cast<size_t>(m)}, std::vector<double>(y, y + n * m));
  return clip_cost(t, std::span<const double>(budgets, static_cast<size_t>(m)));
}

int ref_multilevel(const double* t, const int64_t* shape, int order,
                   const int* levels, int depth, double eta, int workers,
                   double* x, double* chain) {
  return guarded([&] {
    std::vector<size_t> shp(shape, shape + order);
    size_t total = 1;
    for (auto d : shp) total *= d;
    DenseTensor tt(shp, std::vector<double>(t, t + total));
    NormSpec spec;
    for (int i = 0; i < depth; ++i) spec.levels.push_back(to_norm(levels[i]));
    auto pool = make_pool(workers);
    MultilevelResult r = multilevel_project_iter(tt, spec, eta, pool.get());
    std::memcpy(x, r.X.data().data(), sizeof(double) * total);
    if (chain) {
      size_t off = 0;
      for (size_t i = 0; i + 1 < r.budget_chain.size(); ++i) {
        auto d = r.budget_chain[i].data();
        std::memcpy(chain + off, d.data(), sizeof(double) * d.size());
        off += d.size();
      }
    }
  });
}

int ref_multilevel_recursive(const double* t, const int64_t* shape, int order,
                             const int* levels, int depth, double eta,
                             double* x) {
  return guarded([&] {
    std::vector<size_t> shp(shape, shape + order);
    size_t total = 1;
    for (auto d : shp) total *= d;
    DenseTensor tt(shp, std::vector<double>(t, t + total));
    NormSpec spec;
    for (int i = 0; i < depth; ++i) spec.levels.push_back(to_norm(levels[i]));
    DenseTensor r = multilevel_project(tt, spec, eta, nullptr);
    std::memcpy(x, r.data().data(), sizeof(double) * total);
  });
}

int ref_trilevel_l1infinf(const double* t, const int64_t* shape, double eta,
                          double* x) {
  return guarded([&] {
    std::vector<size_t> shp(shape, shape + 3);
    size_t total = shp[0] * shp[1] * shp[2];
    DenseTensor tt(shp, std::vector<double>(t, t + total));
    DenseTensor r = trilevel_project_l1infinf(tt, eta, nullptr);
    std::memcpy(x, r.data().data(), sizeof(double) * total);
  });
}

int ref_project_ball(const double* y, int64_t len, int q, double radius,
                     int use_sort, double* out) {
  return guarded([&] {
    std::span<const double> s(y, static_cast<size_t>(len));
    std::vector<double> r;
    if (q == 0 && use_sort) r = project_l1_sort(s, radius);
    else r = project_ball(s, to_norm(q), radius);
    std::memcpy(out, r.data(), sizeof(double) * len);
  });
}

int ref_multilevel_norm(const double* t, const int64_t* shape, int order,
                        const int* levels, int depth, double* out) {
  return guarded([&] {
    std::vector<size_t> shp(shape, shape + order);
    size_t total = 1;
    for (auto d : shp) total *= d;
    DenseTensor tt(shp, std::vector<double>(t, t + total));
    NormSpec spec;
    for (int i = 0; i < depth; ++i) spec.levels.push_back(to_norm(levels[i]));
    *out = multilevel_norm(tt, spec);
  });
}

// Reference generator (proj/src/rng.cpp): uniform(lo, hi) and normal().
void ref_gen_uniform(uint64_t seed, double lo, double hi, double* out, int64_t count) {
  Xoshiro256pp rng(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng.uniform(lo, hi);
}

void ref_gen_normal(uint64_t seed, double* out, int64_t count) {
  Xoshiro256pp rng(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng.normal();
}

void ref_gen_raw(uint64_t seed, uint64_t* out, int64_t count) {
  Xoshiro256pp rng(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng.next();
}

}  // extern "C"
