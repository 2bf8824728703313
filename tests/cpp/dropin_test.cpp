// C++ drop-in test: the reference's own C++ API (include/multiproj/*.hpp),
// linked against libmultiproj_b200.so instead of the reference library,
// checked on the reference's worked examples and invariants
// (proj/tests/test_bilevel.cpp, proj/tests/test_multilevel.cpp,
// proj/tests/test_vector_balls.cpp).  Exit status 0 iff every check passes.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include <unistd.h>

#include <filesystem>
#include <string>

#include "multiproj/bench.hpp"
#include "multiproj/bilevel.hpp"
#include "multiproj/rng.hpp"
#include "multiproj/tensor_io.hpp"
#include "multiproj/dispatch.hpp"
#include "multiproj/euclidean.hpp"
#include "multiproj/multilevel.hpp"
#include "multiproj/vector_balls.hpp"

using namespace multiproj;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);      \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static bool close(double a, double b, double tol = 1e-12) { return std::fabs(a - b) <= tol * std::max(1.0, std::fabs(b)); }
static bool bits_equal(std::span<const double> a, std::span<const double> b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}
template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  {  // identity: budgets (0.5, 0.5)
    auto r = bilevel_project_l1inf(DenseTensor({2, 2}, {1, 0, 0, 1}), 1.0);
    EXPECT(close(r.budgets[0], 0.5) && close(r.budgets[1], 0.5));
    EXPECT(close(r.X[0], 0.5) && r.X[1] == 0 && r.X[2] == 0 && close(r.X[3], 0.5));
    EXPECT(r.zero_columns == 0);
  }
  {  // a weak column is zeroed
    auto r = bilevel_project_l1inf(DenseTensor({2, 2}, {0.9, 0.1, 0.1, 0.05}), 0.6);
    EXPECT(close(r.budgets[0], 0.6) && r.budgets[1] == 0.0 && r.zero_columns == 1);
    EXPECT(close(r.X[0], 0.6) && r.X[1] == 0 && close(r.X[2], 0.1) && r.X[3] == 0);
  }
  {  // l1,1 and l1,2 worked examples
    auto a = bilevel_project(DenseTensor({2, 2}, {0.5, 0.25, 0.5, 0.25}), Norm::L1, Norm::L1, 1.0);
    EXPECT(close(a.budgets[0], 0.75) && close(a.budgets[1], 0.25));
    EXPECT(close(a.X[0], 0.375) && close(a.X[1], 0.125) && close(a.X[2], 0.375) && close(a.X[3], 0.125));
    auto b = bilevel_project(DenseTensor({2, 2}, {3, 0, 4, 0}), Norm::L1, Norm::L2, 1.0);
    EXPECT(close(b.budgets[0], 1.0) && b.budgets[1] == 0.0);
    EXPECT(close(b.X[0], 0.6) && close(b.X[2], 0.8) && b.X[1] == 0 && b.X[3] == 0);
  }
  {  // error types
    EXPECT(throws<ValueError>([] { bilevel_project(DenseTensor({2, 2}, {1, 0, 0, 1}), Norm::L1, Norm::Inf, -1.0); }));
    EXPECT(throws<ShapeError>([] { bilevel_project(DenseTensor({3}, {1, 2, 3}), Norm::L1, Norm::Inf, 1.0); }));
    EXPECT(throws<ValueError>([] { DenseTensor({2}, {1.0, NAN}); }));
    EXPECT(throws<ShapeError>([] { DenseTensor({2, 0}, {}); }));
    EXPECT(throws<ConfigError>([] { parse_norm_spec("1,3"); }));
    EXPECT(throws<ConfigError>([] { parse_norm_spec(""); }));
    EXPECT(throws<ShapeError>([] { multilevel_project(DenseTensor({2, 2}, {1, 0, 0, 1}), NormSpec{{Norm::L1}}, 1.0); }));
    EXPECT(throws<ConfigError>([] { Algorithm::parse("nope"); }));
    EXPECT(throws<ConfigError>([] { ThreadPool(0); }));
  }
  {  // random invariants: feasibility, budgets, zero count, bit-idempotence
    std::mt19937_64 g(21);
    std::uniform_real_distribution<double> U(-1, 1), R(0, 1);
    for (int it = 0; it < 100; ++it) {
      const std::size_t n = 1 + g() % 12, m = 1 + g() % 12;
      std::vector<double> d(n * m);
      for (double& v : d) v = U(g);
      DenseTensor y({n, m}, d);
      const double eta = R(g) * 1.2 * matrix_pq_norm(y, Norm::L1, Norm::Inf);
      auto r = bilevel_project_l1inf(y, eta);
      EXPECT(matrix_pq_norm(r.X, Norm::L1, Norm::Inf) <= eta * (1 + 1e-9) + 1e-15);
      DenseTensor mx = aggregate_leading_axis(r.X, Norm::Inf);
      for (std::size_t f = 0; f < m; ++f) EXPECT(mx[f] <= r.budgets[f] * (1 + 1e-9) + 1e-15);
      EXPECT(r.zero_columns == structured_sparsity(r.X, 0.0).zero_columns);
      auto r2 = bilevel_project_l1inf(r.X, eta * (1 + 1e-9));
      EXPECT(bits_equal(r.X.data(), r2.X.data()));
    }
  }
  {  // feasible input is returned bit for bit
    DenseTensor y({2, 3}, {0.1, -0.2, 0.05, 0.0, 0.1, 0.02});
    auto r = bilevel_project_l1inf(y, matrix_pq_norm(y, Norm::L1, Norm::Inf) + 1.0);
    EXPECT(bits_equal(y.data(), r.X.data()));
  }
  {  // tri-level worked example and the nested norm
    DenseTensor y({2, 1, 2}, {1, 0.2, 0.5, 0.4});
    EXPECT(close(multilevel_norm(y, parse_norm_spec("inf,inf,1")), 1.4));
    DenseTensor x = trilevel_project_l1infinf(y, 1.0);
    EXPECT(close(x[0], 0.8) && close(x[1], 0.2) && close(x[2], 0.5) && close(x[3], 0.2));
    auto it = multilevel_project_iter(y, parse_norm_spec("inf,inf,1"), 1.0);
    EXPECT(it.budget_chain.size() == 3 && bits_equal(it.budget_chain.back().data(), it.X.data()));
    EXPECT(parse_norm_spec("inf,inf,1").to_string() == "inf,inf,1");
  }
  {  // "inf,1" multilevel == bilevel l1,inf; dispatcher tags
    DenseTensor y({3, 4}, {0.3, -0.9, 0.2, 0.5, -0.4, 0.1, 0.8, -0.6, 0.7, 0.2, -0.1, 0.9});
    const double eta = 0.4 * matrix_pq_norm(y, Norm::L1, Norm::Inf);
    auto a = multilevel_project(y, parse_norm_spec("inf,1"), eta);
    auto b = bilevel_project_l1inf(y, eta);
    EXPECT(bits_equal(a.data(), b.X.data()));
    auto c = run_projection(Algorithm::parse("bilevel-l1inf"), y, eta, nullptr);
    EXPECT(bits_equal(c.data(), b.X.data()));
    EXPECT(Algorithm::parse("multilevel:inf,inf,1").tag() == "multilevel:inf,inf,1");
    auto e = run_projection(Algorithm::parse("euclid"), y, eta, nullptr);
    EXPECT(bits_equal(e.data(), euclid_project_l1inf(y, eta).X.data()));
  }
  {  // exact Euclidean l1,inf (proj/tests/test_euclidean.cpp:20-55)
    DenseTensor y({2, 2}, {1, 0.5, 1, 0});
    auto r = euclid_project_l1inf(y, 1.0);
    EXPECT(close(r.sol.theta, 1.0 / 3) && close(r.sol.budgets[0], 5.0 / 6) && close(r.sol.budgets[1], 1.0 / 6));
    const double d = frobenius_distance(y, r.X);
    EXPECT(close(d * d, 1.0 / 6));
    DenseTensor in({2, 2}, {0.3, 0.1, -0.2, 0.05});
    auto id = euclid_project_l1inf(in, 2.0);
    EXPECT(bits_equal(id.X.data(), in.data()) && id.sol.theta == 0.0);
    auto z = euclid_project_l1inf(DenseTensor({2, 2}, {1, 2, 3, 4}), 0.0);
    EXPECT(z.X.data()[0] == 0.0 && z.X.data()[3] == 0.0);
    EXPECT(throws<ValueError>([&] { euclid_project_l1inf(in, -1.0); }));
    EXPECT(throws<ShapeError>([&] { euclid_project_l1inf(DenseTensor({4}, {1, 2, 3, 4}), 1.0); }));
    // the grid oracle brackets the exact budgets (test_euclidean.cpp:57-75)
    auto g = budget_oracle_grid(y, 1.0, 10000);
    EXPECT(std::abs(g.budgets[0] - r.sol.budgets[0]) <= 2e-4 && std::abs(g.budgets[1] - r.sol.budgets[1]) <= 2e-4);
    EXPECT(d * d <= clip_cost(y, g.budgets) + 1e-9);
    EXPECT(throws<ConfigError>([&] { budget_oracle_grid(DenseTensor({1, 4}, {1, 2, 3, 4}), 1.0, 1000); }));
  }
  {  // vector balls (proj/tests/test_vector_balls.cpp worked examples)
    std::vector<double> a{1.0, 1.0}, b{0.9, 0.1}, c{3.0, 4.0}, d{0.7, -1.2};
    auto pa = project_l1_fast(a, 1.0);
    EXPECT(close(pa[0], 0.5) && close(pa[1], 0.5));
    auto pb = project_l1_sort(b, 0.6);
    EXPECT(close(pb[0], 0.6) && pb[1] == 0.0);
    auto pc = project_l2(c, 1.0);
    EXPECT(close(pc[0], 0.6) && close(pc[1], 0.8));
    auto pd = project_linf(d, 1.0);
    EXPECT(pd[0] == 0.7 && pd[1] == -1.0);
    EXPECT(throws<ValueError>([&] { project_ball(a, Norm::L1, -1.0); }));
  }
  {  // bench records and file projection (proj/tests/test_bench.cpp:20-146)
    const std::string dir = std::filesystem::temp_directory_path() / ("mp_dropin_" + std::to_string(::getpid()));
    std::filesystem::create_directories(dir);
    auto recs = run_radius_sweep({"bilevel-l1inf", "bilevel-l11", "multilevel:inf,1"}, 40, 30, {0.5, 2.0}, 5, 2, 1);
    EXPECT(recs.size() == 6);
    for (const auto& r : recs) EXPECT(r.achieved_norm <= r.radius * (1 + 1e-9) && r.repetitions == 2 && r.n == 40);
    write_csv_records(recs, dir + "/r.csv");
    auto back = read_csv_records(dir + "/r.csv");
    EXPECT(back.size() == recs.size() && back[4].algorithm == "multilevel:inf,1" &&
           back[5].output_checksum == recs[5].output_checksum && back[2].median_seconds == recs[2].median_seconds);
    auto sizes = run_size_sweep({"multilevel:inf,inf,1"}, {{6, 5, 4}}, 1.0, 9, 1, 1);
    EXPECT(sizes.size() == 1 && sizes[0].extra_dims == std::vector<std::size_t>{4});
    auto eu = run_size_sweep({"euclid", "bilevel-l12"}, {{6, 5}, {9, 3}}, 1.0, 9, 1, 1);
    EXPECT(eu.size() == 4 && eu[0].achieved_norm <= 1.0 + 1e-9 && eu[3].m == 3);
    auto sp = measure_speedup(Algorithm::parse("bilevel-l1inf"), {50, 40}, 1.0, {1, 2, 4}, 1);
    EXPECT(sp.size() == 3 && sp[0].output_checksum == sp[2].output_checksum);
    DenseTensor y = gen_uniform_matrix(20, 10, 3, -1.0, 1.0);
    write_tensor(y, dir + "/in.mlpt");
    write_tensor(y, dir + "/in.csv");
    auto rep = project_file(dir + "/in.mlpt", dir + "/out.mlpt", Algorithm::parse("bilevel-l1inf"), 1.0, 1);
    auto repc = project_file(dir + "/in.csv", dir + "/out.csv", Algorithm::parse("bilevel-l1inf"), 1.0, 1);
    DenseTensor xo = read_tensor(dir + "/out.mlpt");
    EXPECT(bits_equal(xo.data(), bilevel_project_l1inf(y, 1.0).X.data()));
    EXPECT(bits_equal(read_tensor(dir + "/out.csv").data(), xo.data()));
    EXPECT(rep.achieved_norm <= 1.0 * (1 + 1e-9) && rep.distance > 0 && repc.zero_columns == rep.zero_columns);
    EXPECT(throws<ConfigError>([&] { project_file(dir + "/in.mlpt", dir + "/o.mlpt", Algorithm::parse("multilevel:inf,inf,1"), 1.0, 1); }));
    EXPECT(throws<ConfigError>([&] { bench_one(Algorithm::parse("bilevel-l1inf"), y, 1.0, 0, 1); }));
    std::filesystem::remove_all(dir);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
