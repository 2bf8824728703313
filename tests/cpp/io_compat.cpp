// io_compat.cpp -- host-side surface of the drop-in (tensor formats,
// generator, checksum, bench records) driven from tests/test_dropin.py and
// compared with the compiled reference (oracle/_ref).  No GPU calls.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "multiproj/bench.hpp"
#include "multiproj/errors.hpp"
#include "multiproj/rng.hpp"
#include "multiproj/tensor_io.hpp"

using namespace multiproj;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "checksum") {  // checksum <path>
      DenseTensor t = read_tensor(argv[2]);
      std::printf("%llu %zu\n", static_cast<unsigned long long>(tensor_checksum(t)), t.size());
    } else if (mode == "write") {  // write <path> <seed> <lo> <hi> dims...
      std::vector<std::size_t> shape;
      for (int k = 6; k < argc; ++k) shape.push_back(std::strtoull(argv[k], nullptr, 10));
      DenseTensor t = gen_uniform_tensor(shape, std::strtoull(argv[3], nullptr, 10), std::atof(argv[4]),
                                         std::atof(argv[5]));
      write_tensor(t, argv[2]);
      std::printf("%llu\n", static_cast<unsigned long long>(tensor_checksum(t)));
    } else if (mode == "records") {  // records <in> <out>
      auto r = read_csv_records(argv[2]);
      write_csv_records(r, argv[3]);
      std::printf("%zu\n", r.size());
    } else if (mode == "rng") {  // rng <seed> <count>
      const int count = std::atoi(argv[3]);
      Xoshiro256pp a(std::strtoull(argv[2], nullptr, 10)), b(std::strtoull(argv[2], nullptr, 10));
      for (int i = 0; i < count; ++i) std::printf("%llu\n", static_cast<unsigned long long>(a.next()));
      for (int i = 0; i < count; ++i) std::printf("%.17g\n", b.normal());
    } else {
      return 2;
    }
  } catch (const IoError& e) {
    std::printf("IoError %s\n", e.what());
    return 3;
  } catch (const ShapeError& e) {
    std::printf("ShapeError %s\n", e.what());
    return 4;
  }
  return 0;
}
