// e2e leg of bench.py through the C++ drop-in: the reference's own call
// shape, multiproj::bilevel_project(const DenseTensor&, Norm::L1, Norm::Inf,
// eta) on a host f64 DenseTensor (pageable std::vector storage, result
// returned by value -- proj/include/multiproj/bilevel.hpp:21-26), linked
// against libmultiproj_b200.so.  Every call uploads Y, runs the three
// kernels and downloads X and the budgets.
// Usage: dropin_bench <n> <m> <reps> <rel>... ; prints one JSON object.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "multiproj/bilevel.hpp"
#include "multiproj/rng.hpp"
#include "multiproj/tensor.hpp"

using namespace multiproj;

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: dropin_bench n m reps rel...\n");
    return 2;
  }
  const std::size_t n = std::strtoull(argv[1], nullptr, 10), m = std::strtoull(argv[2], nullptr, 10);
  const int reps = std::atoi(argv[3]);
  // config 2's distribution (U[-1,1), seed 2) in the drop-in's dtype
  const DenseTensor y = gen_uniform_matrix(n, m, 2, -1.0, 1.0);
  const double norm = matrix_pq_norm(y, Norm::L1, Norm::Inf);
  std::printf("{\"n\": %zu, \"m\": %zu, \"norm\": %.17g, \"radii\": [", n, m, norm);
  for (int a = 4; a < argc; ++a) {
    const double eta = std::atof(argv[a]) * norm;
    BilevelResult warm = bilevel_project(y, Norm::L1, Norm::Inf, eta);  // context, buffers
    std::size_t surv = 0;
    for (double u : warm.budgets) surv += u > 0.0;
    std::printf("%s{\"rel\": %s, \"survivors\": %zu, \"zero_columns\": %zu, \"seconds\": [", a > 4 ? ", " : "",
                argv[a], surv, warm.zero_columns);
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      BilevelResult res = bilevel_project(y, Norm::L1, Norm::Inf, eta);
      const auto t1 = std::chrono::steady_clock::now();
      if (res.X.size() != n * m) return 3;
      std::printf("%s%.9f", r ? ", " : "", std::chrono::duration<double>(t1 - t0).count());
    }
    std::printf("]}");
  }
  std::printf("]}\n");
  return 0;
}
