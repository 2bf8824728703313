// multiproj/rng.hpp -- B200 drop-in for the reference generator and payload
// checksum (proj/include/multiproj/rng.hpp:9-41).  The stream is part of the
// reference's reproducibility contract (SplitMix64-seeded xoshiro256++, top
// 53 bits per double, Box-Muller normals), so it is restated exactly; it runs
// on the host, where the reference's callers consume it.
#ifndef MULTIPROJ_RNG_HPP
#define MULTIPROJ_RNG_HPP

#include <cstdint>
#include <vector>

#include "multiproj/tensor.hpp"

namespace multiproj {

class Xoshiro256pp {
 public:
  explicit Xoshiro256pp(std::uint64_t seed);
  std::uint64_t next();
  double next_double();                  // [0, 1)
  double uniform(double lo, double hi);  // [lo, hi)
  double normal();                       // standard normal

 private:
  std::uint64_t s_[4];
  bool cached_ = false;
  double cache_ = 0.0;
};

DenseTensor gen_uniform_matrix(std::size_t n, std::size_t m, std::uint64_t seed, double lo, double hi);
DenseTensor gen_uniform_tensor(const std::vector<std::size_t>& shape, std::uint64_t seed, double lo, double hi);

// FNV-1a (64-bit) over the little-endian bytes of the payload.
std::uint64_t tensor_checksum(const DenseTensor& t);

}  // namespace multiproj

#endif
