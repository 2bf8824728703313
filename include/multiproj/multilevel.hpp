// multiproj/multilevel.hpp -- B200 drop-in for the multi-level projections
// (proj/include/multiproj/multilevel.hpp:11-51).
#ifndef MULTIPROJ_MULTILEVEL_HPP
#define MULTIPROJ_MULTILEVEL_HPP

#include <string>
#include <vector>

#include "multiproj/parallel.hpp"
#include "multiproj/tensor.hpp"

namespace multiproj {

// Norm levels, innermost first; "inf,1" is l_{1,inf}, "inf,inf,1" tri-level.
struct NormSpec {
  std::vector<Norm> levels;
  std::size_t depth() const { return levels.size(); }
  std::string to_string() const;
};

NormSpec parse_norm_spec(const std::string& s);  // ConfigError on bad tokens

struct MultilevelResult {
  DenseTensor X;
  // Deepest aggregate's projection first; the last entry is X itself.
  std::vector<DenseTensor> budget_chain;
};

DenseTensor multilevel_project(const DenseTensor& t, const NormSpec& nu, double eta, ThreadPool* pool = nullptr);
MultilevelResult multilevel_project_iter(const DenseTensor& t, const NormSpec& nu, double eta,
                                         ThreadPool* pool = nullptr);
DenseTensor trilevel_project_l1infinf(const DenseTensor& t, double eta, ThreadPool* pool = nullptr);
double multilevel_norm(const DenseTensor& t, const NormSpec& nu);

}  // namespace multiproj

#endif
