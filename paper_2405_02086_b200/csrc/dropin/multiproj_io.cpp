// multiproj_io.cpp -- the drop-in's host-side surface around the projection
// path: the reference generator and checksum (proj/src/rng.cpp), the MLPT /
// CSV tensor formats (proj/src/tensor_io.cpp) and the benchmark-record /
// file-projection API (proj/src/bench.cpp).  Projections, norms and the
// zero-group count inside go to the GPU through the drop-in; only file bytes,
// the generator stream and the record bookkeeping stay on the host.
#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <numbers>
#include <sstream>

#include "multiproj/bench.hpp"
#include "multiproj/errors.hpp"
#include "multiproj/multilevel.hpp"
#include "multiproj/rng.hpp"
#include "multiproj/tensor_io.hpp"

namespace multiproj {

static_assert(std::endian::native == std::endian::little, "MLPT files are little endian");

// ------------------------------------------------------------- generator
// SplitMix64 seeding and xoshiro256++ (proj/include/multiproj/rng.hpp:9-15).
Xoshiro256pp::Xoshiro256pp(std::uint64_t seed) {
  std::uint64_t x = seed;
  for (std::uint64_t& w : s_) {
    x += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    w = z ^ (z >> 31);
  }
}

std::uint64_t Xoshiro256pp::next() {
  const std::uint64_t out = std::rotl(s_[0] + s_[3], 23) + s_[0];
  const std::uint64_t sh = s_[1] << 17;
  s_[2] ^= s_[0];
  s_[3] ^= s_[1];
  s_[1] ^= s_[2];
  s_[0] ^= s_[3];
  s_[2] ^= sh;
  s_[3] = std::rotl(s_[3], 45);
  return out;
}

double Xoshiro256pp::next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

double Xoshiro256pp::uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }

// Box-Muller, cosine branch first, sine branch cached (proj/src/rng.cpp:49-62).
double Xoshiro256pp::normal() {
  if (cached_) {
    cached_ = false;
    return cache_;
  }
  double a = next_double();
  const double b = next_double();
  while (a <= 0.0) a = next_double();
  const double rad = std::sqrt(-2.0 * std::log(a));
  const double ang = 2.0 * std::numbers::pi * b;
  cache_ = rad * std::sin(ang);
  cached_ = true;
  return rad * std::cos(ang);
}

DenseTensor gen_uniform_tensor(const std::vector<std::size_t>& shape, std::uint64_t seed, double lo, double hi) {
  if (!(lo < hi)) throw ConfigError("uniform bounds require lo < hi");
  std::size_t count = 1;
  for (std::size_t d : shape) count *= d;
  Xoshiro256pp g(seed);
  std::vector<double> v(count);
  for (double& e : v) e = g.uniform(lo, hi);
  return DenseTensor(shape, std::move(v));
}

DenseTensor gen_uniform_matrix(std::size_t n, std::size_t m, std::uint64_t seed, double lo, double hi) {
  if (n < 1 || m < 1) throw ConfigError("matrix dims must be >= 1");
  return gen_uniform_tensor({n, m}, seed, lo, hi);
}

std::uint64_t tensor_checksum(const DenseTensor& t) {
  std::uint64_t h = 0xcbf29ce484222325ULL;  // FNV-1a offset basis
  for (double v : t.data()) {
    const std::uint64_t bits = std::bit_cast<std::uint64_t>(v);
    for (int sh = 0; sh < 64; sh += 8) h = (h ^ ((bits >> sh) & 0xffULL)) * 0x100000001b3ULL;
  }
  return h;
}

// ---------------------------------------------------------------- formats
TensorFormat format_for_path(const std::string& path) {
  const std::string ext = ".csv";
  const bool csv = path.size() >= ext.size() && path.compare(path.size() - ext.size(), ext.size(), ext) == 0;
  return csv ? TensorFormat::Csv : TensorFormat::Mlpt;
}

namespace {

std::string quoted(const std::string& p) { return "'" + p + "'"; }

template <class F>
DenseTensor as_io_error(const std::string& path, F&& make) {
  try {
    return make();
  } catch (const ValueError& e) {
    throw IoError(quoted(path) + ": " + e.what());
  } catch (const ShapeError& e) {
    throw IoError(quoted(path) + ": " + e.what());
  }
}

}  // namespace

DenseTensor read_mlpt(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open " + quoted(path) + " for reading");
  char tag[4];
  if (!f.read(tag, 4) || std::memcmp(tag, "MLPT", 4) != 0)
    throw IoError(quoted(path) + " is not an MLPT tensor file (bad magic)");
  std::uint32_t order = 0;
  if (!f.read(reinterpret_cast<char*>(&order), 4) || order == 0) throw IoError(quoted(path) + ": malformed MLPT header");
  std::vector<std::size_t> shape;
  std::size_t count = 1;
  for (std::uint32_t k = 0; k < order; ++k) {
    std::uint64_t d = 0;
    if (!f.read(reinterpret_cast<char*>(&d), 8) || d == 0) throw IoError(quoted(path) + ": malformed MLPT dimension");
    shape.push_back(static_cast<std::size_t>(d));
    count *= shape.back();
  }
  std::vector<double> payload(count);
  if (!f.read(reinterpret_cast<char*>(payload.data()), static_cast<std::streamsize>(count * sizeof(double))))
    throw IoError(quoted(path) + ": truncated MLPT payload");
  return as_io_error(path, [&] { return DenseTensor(std::move(shape), std::move(payload)); });
}

void write_mlpt(const DenseTensor& t, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open " + quoted(path) + " for writing");
  f.write("MLPT", 4);
  const std::uint32_t order = static_cast<std::uint32_t>(t.order());
  f.write(reinterpret_cast<const char*>(&order), 4);
  for (std::size_t d : t.shape()) {
    const std::uint64_t d64 = d;
    f.write(reinterpret_cast<const char*>(&d64), 8);
  }
  f.write(reinterpret_cast<const char*>(t.data().data()), static_cast<std::streamsize>(t.size() * sizeof(double)));
  if (!f) throw IoError("write failed for " + quoted(path));
}

DenseTensor read_csv_matrix(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open " + quoted(path) + " for reading");
  std::vector<double> vals;
  std::size_t rows = 0, cols = 0;
  for (std::string line; std::getline(f, line);) {
    if (line.empty()) continue;
    std::size_t here = 0;
    std::istringstream cells(line);
    for (std::string c; std::getline(cells, c, ',');) {
      try {
        vals.push_back(std::stod(c));
      } catch (const std::exception&) {
        throw IoError(quoted(path) + ": bad CSV value '" + c + "'");
      }
      ++here;
    }
    if (rows == 0) cols = here;
    else if (here != cols) throw IoError(quoted(path) + ": ragged CSV rows");
    ++rows;
  }
  if (rows == 0) throw IoError(quoted(path) + ": empty CSV");
  return as_io_error(path, [&] { return DenseTensor::matrix(rows, cols, std::move(vals)); });
}

void write_csv_matrix(const DenseTensor& t, const std::string& path) {
  if (t.order() != 2) throw ShapeError("CSV output requires an order-2 tensor");
  std::ofstream f(path);
  if (!f) throw IoError("cannot open " + quoted(path) + " for writing");
  f.precision(17);  // round-trips every double
  const std::size_t rows = t.shape()[0], cols = t.shape()[1];
  for (std::size_t i = 0; i < rows; ++i) {
    for (std::size_t j = 0; j < cols; ++j) f << (j ? "," : "") << t.data()[i * cols + j];
    f << '\n';
  }
  if (!f) throw IoError("write failed for " + quoted(path));
}

DenseTensor read_tensor(const std::string& path) {
  return format_for_path(path) == TensorFormat::Csv ? read_csv_matrix(path) : read_mlpt(path);
}

void write_tensor(const DenseTensor& t, const std::string& path) {
  if (format_for_path(path) == TensorFormat::Csv) write_csv_matrix(t, path);
  else write_mlpt(t, path);
}

// ------------------------------------------------------- bench records
namespace {

// The ball each algorithm constrains (proj/src/bench.cpp:17-30); specs are
// innermost first.
NormSpec ball_of(const Algorithm& a) {
  switch (a.kind) {
    case Algorithm::Kind::BilevelL1Inf:
    case Algorithm::Kind::Euclid: return NormSpec{{Norm::Inf, Norm::L1}};
    case Algorithm::Kind::BilevelL11: return NormSpec{{Norm::L1, Norm::L1}};
    case Algorithm::Kind::BilevelL12: return NormSpec{{Norm::L2, Norm::L1}};
    case Algorithm::Kind::Multilevel: return a.spec;
  }
  throw ConfigError("unreachable algorithm kind");
}

// #{groups whose max |x| is 0}, aggregating l_inf down to a vector (on the GPU).
std::size_t zero_groups(const DenseTensor& x) {
  DenseTensor cur = x;
  while (cur.order() > 1) cur = aggregate_leading_axis(cur, Norm::Inf);
  return static_cast<std::size_t>(std::count(cur.data().begin(), cur.data().end(), 0.0));
}

double median_of(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const std::size_t h = v.size() / 2;
  return v.size() % 2 ? v[h] : 0.5 * (v[h - 1] + v[h]);
}

std::string g17(double v) {
  std::ostringstream o;
  o.precision(17);
  o << v;
  return o.str();
}

std::string dims_text(const std::vector<std::size_t>& d) {
  std::string s;
  for (std::size_t k = 0; k < d.size(); ++k) s += (k ? "x" : "") + std::to_string(d[k]);
  return s;
}

std::vector<std::size_t> dims_parse(const std::string& s) {
  std::vector<std::size_t> d;
  std::istringstream in(s);
  for (std::string tok; std::getline(in, tok, 'x');)
    if (!tok.empty()) d.push_back(static_cast<std::size_t>(std::stoull(tok)));
  return d;
}

const char* const kRecordHeader =
    "algorithm,n,m,extra_dims,radius,workers,reps,median_seconds,achieved_norm,zero_columns,checksum";

}  // namespace

double achieved_norm(const Algorithm& algorithm, const DenseTensor& x) { return multilevel_norm(x, ball_of(algorithm)); }

BenchRecord bench_one(const Algorithm& algorithm, const DenseTensor& input, double eta, std::size_t reps,
                      unsigned workers) {
  if (reps == 0) throw ConfigError("reps must be >= 1");
  // warm-up run, also the feasibility-checked output
  const DenseTensor out = run_projection(algorithm, input, eta, nullptr);
  const double norm = achieved_norm(algorithm, out);
  if (norm > eta * (1.0 + 1e-9))
    throw ConfigError("projection output infeasible: " + std::to_string(norm) + " > " + std::to_string(eta));
  std::vector<double> secs;
  for (std::size_t r = 0; r < reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    const DenseTensor x = run_projection(algorithm, input, eta, nullptr);
    secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  BenchRecord rec;
  rec.algorithm = algorithm.tag();
  rec.n = input.shape()[0];
  rec.m = input.order() > 1 ? input.shape()[1] : 1;
  if (input.order() > 2) rec.extra_dims.assign(input.shape().begin() + 2, input.shape().end());
  rec.radius = eta;
  rec.workers = workers;
  rec.repetitions = reps;
  rec.median_seconds = median_of(std::move(secs));
  rec.achieved_norm = norm;
  rec.zero_columns = zero_groups(out);
  rec.output_checksum = tensor_checksum(out);
  return rec;
}

std::vector<BenchRecord> run_radius_sweep(const std::vector<std::string>& algorithms, std::size_t n, std::size_t m,
                                          const std::vector<double>& radii, std::uint64_t seed, std::size_t reps,
                                          unsigned workers) {
  std::vector<Algorithm> algos;
  for (const auto& a : algorithms) algos.push_back(Algorithm::parse(a));
  std::vector<BenchRecord> out;
  if (algos.empty() || radii.empty()) return out;
  const DenseTensor y = gen_uniform_matrix(n, m, seed, 0.0, 1.0);
  for (const auto& a : algos)
    for (double r : radii) out.push_back(bench_one(a, y, r, reps, workers));
  return out;
}

std::vector<BenchRecord> run_size_sweep(const std::vector<std::string>& algorithms,
                                        const std::vector<std::vector<std::size_t>>& sizes, double eta,
                                        std::uint64_t seed, std::size_t reps, unsigned workers) {
  std::vector<Algorithm> algos;
  for (const auto& a : algorithms) algos.push_back(Algorithm::parse(a));
  std::vector<BenchRecord> out;
  for (const auto& shape : sizes) {
    const DenseTensor y = gen_uniform_tensor(shape, seed, 0.0, 1.0);
    for (const auto& a : algos) out.push_back(bench_one(a, y, eta, reps, workers));
  }
  return out;
}

std::vector<BenchRecord> measure_speedup(const Algorithm& algorithm, const std::vector<std::size_t>& shape,
                                         double eta, const std::vector<unsigned>& workers, std::size_t reps,
                                         std::uint64_t seed) {
  const DenseTensor y = gen_uniform_tensor(shape, seed, 0.0, 1.0);
  std::vector<BenchRecord> out;
  for (unsigned w : workers) {
    out.push_back(bench_one(algorithm, y, eta, reps, w));
    if (out.back().output_checksum != out.front().output_checksum)
      throw ConfigError("nondeterministic output across worker counts");
  }
  return out;
}

void write_csv_records(const std::vector<BenchRecord>& records, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw IoError("cannot open " + quoted(path) + " for writing");
  f << kRecordHeader << '\n';
  for (const auto& r : records) {
    const bool q = r.algorithm.find(',') != std::string::npos;  // multilevel specs carry commas
    f << (q ? "\"" : "") << r.algorithm << (q ? "\"" : "") << ',' << r.n << ',' << r.m << ','
      << dims_text(r.extra_dims) << ',' << g17(r.radius) << ',' << r.workers << ',' << r.repetitions << ','
      << g17(r.median_seconds) << ',' << g17(r.achieved_norm) << ',' << r.zero_columns << ',' << r.output_checksum
      << '\n';
  }
  if (!f) throw IoError("write failed for " + quoted(path));
}

std::vector<BenchRecord> read_csv_records(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open " + quoted(path) + " for reading");
  std::string line;
  if (!std::getline(f, line) || line != kRecordHeader) throw IoError(quoted(path) + ": unexpected CSV header");
  std::vector<BenchRecord> out;
  while (std::getline(f, line)) {
    if (line.empty()) continue;
    std::vector<std::string> cells;
    std::size_t pos = 0;
    if (line[0] == '"') {
      const std::size_t end = line.find('"', 1);
      if (end == std::string::npos || end + 1 >= line.size() || line[end + 1] != ',')
        throw IoError(quoted(path) + ": bad quoted CSV field");
      cells.push_back(line.substr(1, end - 1));
      pos = end + 2;
    } else {
      const std::size_t c = line.find(',');
      if (c == std::string::npos) throw IoError(quoted(path) + ": bad CSV row");
      cells.push_back(line.substr(0, c));
      pos = c + 1;
    }
    std::istringstream rest(line.substr(pos));
    for (std::string c; std::getline(rest, c, ',');) cells.push_back(c);
    if (cells.size() != 11) throw IoError(quoted(path) + ": bad CSV row");
    BenchRecord r;
    try {
      r.algorithm = cells[0];
      r.n = std::stoull(cells[1]);
      r.m = std::stoull(cells[2]);
      r.extra_dims = dims_parse(cells[3]);
      r.radius = std::stod(cells[4]);
      r.workers = static_cast<unsigned>(std::stoul(cells[5]));
      r.repetitions = std::stoull(cells[6]);
      r.median_seconds = std::stod(cells[7]);
      r.achieved_norm = std::stod(cells[8]);
      r.zero_columns = std::stoull(cells[9]);
      r.output_checksum = std::stoull(cells[10]);
    } catch (const std::logic_error&) {
      throw IoError(quoted(path) + ": bad CSV row");
    }
    out.push_back(std::move(r));
  }
  return out;
}

ProjectionReport project_file(const std::string& input_path, const std::string& output_path,
                              const Algorithm& algorithm, double eta, unsigned workers) {
  const DenseTensor y = read_tensor(input_path);
  if (algorithm.kind == Algorithm::Kind::Multilevel) {
    if (algorithm.spec.depth() != y.order())
      throw ConfigError("norm spec depth " + std::to_string(algorithm.spec.depth()) +
                        " does not match tensor order " + std::to_string(y.order()));
  } else if (y.order() != 2) {
    throw ConfigError("algorithm '" + algorithm.tag() + "' requires an order-2 tensor");
  }
  const DenseTensor x = parallel_project(algorithm, y, eta, ExecConfig{workers});
  if (format_for_path(input_path) == TensorFormat::Csv) write_csv_matrix(x, output_path);
  else write_mlpt(x, output_path);
  return {achieved_norm(algorithm, x), frobenius_distance(y, x), zero_groups(x)};
}

}  // namespace multiproj
