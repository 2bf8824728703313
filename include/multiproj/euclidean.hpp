// multiproj/euclidean.hpp -- B200 drop-in for the exact Euclidean l_{1,inf}
// projection (proj/include/multiproj/euclidean.hpp:11-37).  Same types and
// signatures; euclid_project_l1inf runs as sm_100a kernels through
// mp_euclid_project_host (column sort in shared memory, cooperative Newton
// search on the budget-sum breakpoints, l_inf clip).  clip_cost and the
// exhaustive budget_oracle_grid are the reference's host-side verification
// utilities and stay on the host.
#ifndef MULTIPROJ_EUCLIDEAN_HPP
#define MULTIPROJ_EUCLIDEAN_HPP

#include <span>
#include <vector>

#include "multiproj/tensor.hpp"

namespace multiproj {

// Per-column clip levels of the exact projection and the shared residual
// mass theta of the active columns.
struct ColumnBudgetSolution {
  std::vector<double> budgets;
  double theta;
};

struct EuclidResult {
  DenseTensor X;
  ColumnBudgetSolution sol;
};

EuclidResult euclid_project_l1inf(const DenseTensor& y, double eta);

// Exhaustive simplex grid search over budgets (m <= 3, steps >= 100).
ColumnBudgetSolution budget_oracle_grid(const DenseTensor& y, double eta, std::size_t steps);

// sum_j sum_i max(|Y_ij| - u_j, 0)^2
double clip_cost(const DenseTensor& y, std::span<const double> budgets);

}  // namespace multiproj

#endif
