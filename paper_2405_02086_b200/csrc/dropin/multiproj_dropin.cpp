// multiproj_dropin.cpp -- the reference's C++ API (include/multiproj/*.hpp)
// implemented over the C-ABI (include/mp_cuda.h).  Linking this library
// instead of the reference's libmultiproj gives existing C++ callers the
// sm_100a path with unchanged signatures, ownership (results by value) and
// exception types.  Every projection and every O(N) reduction goes to the
// GPU; only O(order) bookkeeping and the final scalar of a norm stay on the
// host.  No CPU fallback: a missing GPU surfaces as std::runtime_error.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <sstream>
#include <thread>

#include <sys/mman.h>

#include "mp_cuda.h"
#include "multiproj/bilevel.hpp"
#include "multiproj/dispatch.hpp"
#include "multiproj/euclidean.hpp"
#include "multiproj/multilevel.hpp"
#include "multiproj/parallel.hpp"
#include "multiproj/tensor.hpp"
#include "multiproj/vector_balls.hpp"

namespace multiproj {

namespace {

[[noreturn]] void raise(mp_status st) {
  const std::string msg = mp_last_error();
  switch (st) {
    case MP_ERR_VALUE: throw ValueError(msg);
    case MP_ERR_SHAPE: throw ShapeError(msg);
    case MP_ERR_CONFIG: throw ConfigError(msg);
    default: throw std::runtime_error("multiproj (B200): " + msg);
  }
}

void check(mp_status st) {
  if (st != MP_OK) raise(st);
}

mp_norm to_mp(Norm q) { return q == Norm::L1 ? MP_NORM_L1 : (q == Norm::L2 ? MP_NORM_L2 : MP_NORM_INF); }

void check_radius(double r) {
  if (!(r >= 0.0) || !std::isfinite(r)) throw ValueError("radius must be a finite nonnegative real");
}

std::vector<double> ball(std::span<const double> y, Norm q, double radius) {
  check_radius(radius);
  for (double v : y)
    if (!std::isfinite(v)) throw ValueError("non-finite vector entry");
  std::vector<double> out(y.begin(), y.end());
  if (!out.empty())
    check(mp_project_ball_host(nullptr, out.data(), out.data(), MP_F64, static_cast<int64_t>(out.size()), to_mp(q),
                               radius));
  return out;
}

std::vector<double> aggregate(const DenseTensor& t, Norm q) {
  std::vector<double> out(t.fiber_count());
  check(mp_aggregate_host(nullptr, t.data().data(), out.data(), MP_F64, static_cast<int64_t>(t.fiber_length()),
                          static_cast<int64_t>(t.fiber_count()), to_mp(q)));
  return out;
}

}  // namespace

// ----------------------------------------------------------------- tensor
std::string norm_name(Norm q) { return q == Norm::L1 ? "1" : (q == Norm::L2 ? "2" : "inf"); }

DenseTensor::DenseTensor(std::vector<std::size_t> shape, std::vector<double> data)
    : shape_(std::move(shape)), data_(std::move(data)) {
  if (shape_.empty()) throw ShapeError("tensor order must be >= 1");
  std::size_t total = 1;
  for (std::size_t d : shape_) {
    if (d == 0) throw ShapeError("zero dimension in shape");
    total *= d;
  }
  if (total != data_.size()) throw ShapeError("shape/data size mismatch");
  if (!std::all_of(data_.begin(), data_.end(), [](double v) { return std::isfinite(v); }))
    throw ValueError("non-finite tensor entry");
  fibers_ = data_.size() / shape_.front();
}

DenseTensor::DenseTensor(Unchecked, std::vector<std::size_t> shape, std::vector<double> data)
    : shape_(std::move(shape)), data_(std::move(data)) {
  fibers_ = data_.size() / shape_.front();
}

// Result tensors: a fresh host buffer (transparent huge pages requested
// before the first touch -- 4 KB first-touch faults cost 300 ms on an 800 MB
// result) and the unchecked constructor (the projections of finite input
// are finite; the reference copies Y without a re-check).
struct TensorFactory {
  static std::vector<double> buffer(std::size_t n) {
    std::vector<double> v;
    v.reserve(n);
    const std::size_t bytes = n * sizeof(double);
    if (bytes >= (std::size_t(8) << 20)) {
      const uintptr_t a = (reinterpret_cast<uintptr_t>(v.data()) + (std::size_t(2) << 20) - 1) &
                          ~((std::size_t(2) << 20) - 1);
      const uintptr_t e = reinterpret_cast<uintptr_t>(v.data()) + bytes;
      if (e > a) madvise(reinterpret_cast<void*>(a), e - a, MADV_HUGEPAGE);
      // First touch on several threads: the kernel clears every fresh page
      // on its fault (one thread: ~90 ms for 800 MB); the value-initialising
      // resize below then runs over resident pages.
      const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
      char* base = reinterpret_cast<char*>(v.data());
      const std::size_t slice = ((bytes + nt - 1) / nt + 4095) & ~std::size_t(4095);
      std::vector<std::thread> th;
      for (unsigned t = 0; t < nt; ++t) {
        const std::size_t b0 = std::min(bytes, t * slice), b1 = std::min(bytes, (t + 1) * slice);
        if (b1 > b0) th.emplace_back([base, b0, b1] {
          for (std::size_t o = b0; o < b1; o += 4096) *reinterpret_cast<volatile char*>(base + o) = 0;
        });
      }
      for (auto& x : th) x.join();
    }
    v.resize(n);
    return v;
  }
  static DenseTensor result(std::vector<std::size_t> shape, std::vector<double> data) {
    return DenseTensor(DenseTensor::Unchecked{}, std::move(shape), std::move(data));
  }
};

DenseTensor DenseTensor::zeros(std::vector<std::size_t> shape) {
  std::size_t total = 1;
  for (std::size_t d : shape) total *= d;
  return DenseTensor(std::move(shape), std::vector<double>(total, 0.0));
}

DenseTensor DenseTensor::matrix(std::size_t rows, std::size_t cols, std::vector<double> row_major) {
  return DenseTensor({rows, cols}, std::move(row_major));
}

DenseTensor DenseTensor::vector(std::vector<double> values) {
  const std::size_t n = values.size();
  return DenseTensor({n}, std::move(values));
}

void DenseTensor::copy_fiber(std::size_t f, std::span<double> out) const {
  for (std::size_t i = 0; i < fiber_length(); ++i) out[i] = fiber_at(f, i);
}

void DenseTensor::set_fiber(std::size_t f, std::span<const double> values) {
  for (std::size_t i = 0; i < fiber_length(); ++i) fiber_at(f, i) = values[i];
}

FiberView::FiberView(const DenseTensor& base, std::size_t fiber) : base_(&base), fiber_(fiber) {
  if (fiber >= base.fiber_count()) throw ShapeError("fiber index out of range");
}

double vector_norm(std::span<const double> v, Norm q) {
  double s = 0.0;
  for (double x : v) {
    if (!std::isfinite(x)) throw ValueError("non-finite vector entry");
    const double a = std::fabs(x);
    if (q == Norm::L1) s += a;
    else if (q == Norm::L2) s += x * x;
    else s = std::max(s, a);
  }
  return q == Norm::L2 ? std::sqrt(s) : s;
}

double matrix_pq_norm(const DenseTensor& y, Norm p, Norm q) {
  if (y.order() != 2) throw ShapeError("matrix_pq_norm requires order 2");
  return vector_norm(aggregate(y, q), p);
}

DenseTensor aggregate_leading_axis(const DenseTensor& t, Norm q) {
  if (t.order() < 2) throw ShapeError("aggregate_leading_axis requires order >= 2");
  return DenseTensor(std::vector<std::size_t>(t.shape().begin() + 1, t.shape().end()), aggregate(t, q));
}

double frobenius_distance(const DenseTensor& a, const DenseTensor& b) {
  if (!a.same_shape(b)) throw ShapeError("frobenius_distance shape mismatch");
  double s = 0.0;
  for (std::size_t k = 0; k < a.size(); ++k) s += (a[k] - b[k]) * (a[k] - b[k]);
  return std::sqrt(s);
}

SparsityCount structured_sparsity(const DenseTensor& x, double tol) {
  if (x.order() != 2) throw ShapeError("structured_sparsity requires order 2");
  const std::vector<double> mx = aggregate(x, Norm::Inf);
  const auto zeros = static_cast<std::size_t>(std::count_if(mx.begin(), mx.end(), [tol](double v) { return v <= tol; }));
  return {zeros, static_cast<double>(zeros) / static_cast<double>(x.fiber_count())};
}

// ----------------------------------------------------------- vector balls
std::vector<double> project_l1_sort(std::span<const double> y, double r) { return ball(y, Norm::L1, r); }
std::vector<double> project_l1_fast(std::span<const double> y, double r) { return ball(y, Norm::L1, r); }
std::vector<double> project_l2(std::span<const double> y, double r) { return ball(y, Norm::L2, r); }
std::vector<double> project_linf(std::span<const double> y, double r) { return ball(y, Norm::Inf, r); }
std::vector<double> project_ball(std::span<const double> y, Norm q, double r) { return ball(y, q, r); }

void project_ball_inplace(std::span<double> y, Norm q, double radius) {
  if (y.empty()) return;
  check(mp_project_ball_host(nullptr, y.data(), y.data(), MP_F64, static_cast<int64_t>(y.size()), to_mp(q), radius));
}
void project_l1_fast_inplace(std::span<double> y, double r) { project_ball_inplace(y, Norm::L1, r); }
void project_l2_inplace(std::span<double> y, double r) { project_ball_inplace(y, Norm::L2, r); }
void project_linf_inplace(std::span<double> y, double r) { project_ball_inplace(y, Norm::Inf, r); }

// ---------------------------------------------------------------- bilevel
BilevelResult bilevel_project(const DenseTensor& y, Norm p, Norm q, double eta, ThreadPool* /*pool*/) {
  if (y.order() != 2) throw ShapeError("bilevel_project requires order 2");
  check_radius(eta);
  const std::size_t n = y.fiber_length(), m = y.fiber_count();
  std::vector<double> x = TensorFactory::buffer(y.size()), budgets(m);
  int64_t zeros = 0;
  double tau = 0.0;
  // Exact zero signs: the drop-in reproduces the reference's bytes.
  check(mp_bilevel_project_host(nullptr, y.data().data(), x.data(), MP_F64, static_cast<int64_t>(n),
                                static_cast<int64_t>(m), to_mp(p), to_mp(q), eta, budgets.data(), &zeros, &tau,
                                MP_FLAG_EXACT_ZERO_SIGN));
  return BilevelResult{TensorFactory::result(y.shape(), std::move(x)), std::move(budgets),
                       static_cast<std::size_t>(zeros)};
}

BilevelResult bilevel_project_l1inf(const DenseTensor& y, double eta, ThreadPool* pool) {
  return bilevel_project(y, Norm::L1, Norm::Inf, eta, pool);
}

// ------------------------------------------------------------- multilevel
std::string NormSpec::to_string() const {
  std::ostringstream s;
  for (std::size_t i = 0; i < levels.size(); ++i) s << (i ? "," : "") << norm_name(levels[i]);
  return s.str();
}

NormSpec parse_norm_spec(const std::string& s) {
  NormSpec spec;
  std::size_t start = 0;
  for (;;) {
    const std::size_t comma = s.find(',', start);
    const std::string tok = s.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
    if (tok == "1") spec.levels.push_back(Norm::L1);
    else if (tok == "2") spec.levels.push_back(Norm::L2);
    else if (tok == "inf") spec.levels.push_back(Norm::Inf);
    else throw ConfigError("bad norm token '" + tok + "' in spec '" + s + "' (expected 1, 2 or inf)");
    if (comma == std::string::npos) return spec;
    start = comma + 1;
  }
}

namespace {

// want_chain = false lets the device take the collapsed (inf, ..., inf, p)
// path; the projected tensor is the same bit for bit.
MultilevelResult run_multilevel(const DenseTensor& t, const NormSpec& nu, double eta, bool want_chain) {
  if (nu.depth() == 0) throw ConfigError("empty norm spec");
  if (nu.depth() != t.order()) throw ShapeError("norm spec depth does not match tensor order");
  check_radius(eta);
  const int order = static_cast<int>(t.order());
  std::vector<int64_t> shape(t.shape().begin(), t.shape().end());
  std::vector<mp_norm> levels;
  for (Norm q : nu.levels) levels.push_back(to_mp(q));
  std::size_t chain_len = 0, mi = 1;
  for (int i = order - 1; i >= 1; --i) {
    mi *= t.shape()[i];
    chain_len += mi;
  }
  std::vector<double> x = TensorFactory::buffer(t.size()), chain(std::max<std::size_t>(chain_len, 1));
  check(mp_multilevel_project_host(nullptr, t.data().data(), x.data(), MP_F64, shape.data(), order, levels.data(),
                                   order, eta, want_chain ? chain.data() : nullptr, MP_FLAG_EXACT_ZERO_SIGN));
  MultilevelResult r{TensorFactory::result(t.shape(), std::move(x)), {}};
  if (!want_chain) return r;
  std::size_t off = 0;
  for (int i = order - 1; i >= 1; --i) {
    std::vector<std::size_t> sh(t.shape().begin() + i, t.shape().end());
    std::size_t sz = 1;
    for (std::size_t d : sh) sz *= d;
    r.budget_chain.push_back(TensorFactory::result(sh, std::vector<double>(chain.begin() + off, chain.begin() + off + sz)));
    off += sz;
  }
  r.budget_chain.push_back(r.X);
  return r;
}

}  // namespace

MultilevelResult multilevel_project_iter(const DenseTensor& t, const NormSpec& nu, double eta, ThreadPool* /*pool*/) {
  return run_multilevel(t, nu, eta, true);
}

DenseTensor multilevel_project(const DenseTensor& t, const NormSpec& nu, double eta, ThreadPool* /*pool*/) {
  // The recursive and iterative forms agree bit for bit in the reference
  // (proj/tests/test_multilevel.cpp:44-67); one device algorithm serves both.
  return run_multilevel(t, nu, eta, false).X;
}

DenseTensor trilevel_project_l1infinf(const DenseTensor& t, double eta, ThreadPool* /*pool*/) {
  if (t.order() != 3) throw ShapeError("trilevel_project_l1infinf requires order 3");
  return run_multilevel(t, NormSpec{{Norm::Inf, Norm::Inf, Norm::L1}}, eta, false).X;
}

double multilevel_norm(const DenseTensor& t, const NormSpec& nu) {
  if (nu.depth() != t.order()) throw ShapeError("norm spec depth does not match tensor order");
  if (nu.depth() == 1) return vector_norm(t.data(), nu.levels[0]);
  DenseTensor cur = aggregate_leading_axis(t, nu.levels[0]);
  for (std::size_t i = 1; i + 1 < nu.depth(); ++i) cur = aggregate_leading_axis(cur, nu.levels[i]);
  return vector_norm(cur.data(), nu.levels.back());
}

// ---------------------------------------------------------------- parallel
ThreadPool::ThreadPool(unsigned workers) : workers_(workers) {
  if (workers == 0) throw ConfigError("worker count must be >= 1");
}

void ThreadPool::parallel_for(std::size_t count, const std::function<void(std::size_t, std::size_t)>& body) {
  if (count == 0) return;
  const std::size_t chunk = (count + workers_ - 1) / workers_;
  std::vector<std::thread> threads;
  for (std::size_t b = chunk; b < count; b += chunk) threads.emplace_back(body, b, std::min(b + chunk, count));
  body(0, std::min(chunk, count));
  for (auto& th : threads) th.join();
}

void parallel_for(ThreadPool* pool, std::size_t count, const std::function<void(std::size_t, std::size_t)>& body) {
  if (count == 0) return;
  if (!pool || pool->workers() == 1) return body(0, count);
  pool->parallel_for(count, body);
}

unsigned default_workers() {
  const char* env = std::getenv("MULTIPROJ_WORKERS");
  const int v = env ? std::atoi(env) : 1;
  return v >= 1 ? static_cast<unsigned>(v) : 1u;
}

// ------------------------------------------------------ exact Euclidean
EuclidResult euclid_project_l1inf(const DenseTensor& y, double eta) {
  if (y.order() != 2) throw ShapeError("euclid_project_l1inf requires order 2");
  check_radius(eta);
  const std::size_t n = y.fiber_length(), m = y.fiber_count();
  std::vector<double> x = TensorFactory::buffer(y.size()), budgets(m);
  double theta = 0.0;
  check(mp_euclid_project_host(nullptr, y.data().data(), x.data(), MP_F64, static_cast<int64_t>(n),
                               static_cast<int64_t>(m), eta, budgets.data(), &theta));
  return EuclidResult{TensorFactory::result(y.shape(), std::move(x)), ColumnBudgetSolution{std::move(budgets), theta}};
}

double clip_cost(const DenseTensor& y, std::span<const double> budgets) {
  if (y.order() != 2) throw ShapeError("clip_cost requires order 2");
  const std::size_t n = y.fiber_length(), m = y.fiber_count();
  double cost = 0.0;
  for (std::size_t j = 0; j < m; ++j)
    for (std::size_t i = 0; i < n; ++i) {
      const double over = std::abs(y.data()[i * m + j]) - budgets[j];
      if (over > 0.0) cost += over * over;
    }
  return cost;
}

// The reference's verification oracle (proj/src/euclidean.cpp:172-240):
// per-column clipping-cost tables on the budget grid u = g eta / steps, then
// the cheapest split of the `steps` cells among <= 3 columns.
ColumnBudgetSolution budget_oracle_grid(const DenseTensor& y, double eta, std::size_t steps) {
  if (y.order() != 2) throw ShapeError("budget_oracle_grid requires order 2");
  const std::size_t m = y.fiber_count(), n = y.fiber_length();
  if (m > 3) throw ConfigError("budget_oracle_grid supports m <= 3 only");
  if (steps < 100) throw ConfigError("budget_oracle_grid needs steps >= 100");
  check_radius(eta);
  const auto level = [&](std::size_t g) { return eta * static_cast<double>(g) / static_cast<double>(steps); };
  std::vector<std::vector<double>> table(m, std::vector<double>(steps + 1));
  for (std::size_t j = 0; j < m; ++j)
    for (std::size_t g = 0; g <= steps; ++g) {
      double c = 0.0;
      for (std::size_t i = 0; i < n; ++i) {
        const double over = std::abs(y.data()[i * m + j]) - level(g);
        if (over > 0.0) c += over * over;
      }
      table[j][g] = c;
    }
  std::vector<std::size_t> pick(m, 0);
  if (m == 1) {
    pick[0] = steps;
  } else if (m == 2) {
    double best = INFINITY;
    for (std::size_t a = 0; a <= steps; ++a)
      if (const double c = table[0][a] + table[1][steps - a]; c < best) {
        best = c;
        pick = {a, steps - a};
      }
  } else if (m == 3) {
    double best = INFINITY;
    for (std::size_t a = 0; a <= steps; ++a) {
      if (table[0][a] >= best) continue;
      for (std::size_t b = 0; a + b <= steps; ++b)
        if (const double c = table[0][a] + table[1][b] + table[2][steps - a - b]; c < best) {
          best = c;
          pick = {a, b, steps - a - b};
        }
    }
  }
  ColumnBudgetSolution sol{std::vector<double>(m), 0.0};
  for (std::size_t j = 0; j < m; ++j) sol.budgets[j] = level(pick[j]);
  for (std::size_t j = 0; j < m; ++j) {
    if (sol.budgets[j] <= 0.0) continue;
    double r = 0.0;
    for (std::size_t i = 0; i < n; ++i) r += std::max(0.0, std::abs(y.data()[i * m + j]) - sol.budgets[j]);
    sol.theta = std::max(sol.theta, r);
  }
  return sol;
}

// ---------------------------------------------------------------- dispatch
Algorithm Algorithm::parse(const std::string& tag) {
  if (tag == "bilevel-l1inf") return {Kind::BilevelL1Inf, {}};
  if (tag == "bilevel-l11") return {Kind::BilevelL11, {}};
  if (tag == "bilevel-l12") return {Kind::BilevelL12, {}};
  if (tag == "euclid") return {Kind::Euclid, {}};
  const std::string pre = "multilevel:";
  if (tag.compare(0, pre.size(), pre) == 0) return {Kind::Multilevel, parse_norm_spec(tag.substr(pre.size()))};
  throw ConfigError("unknown algorithm tag '" + tag + "'");
}

std::string Algorithm::tag() const {
  switch (kind) {
    case Kind::BilevelL1Inf: return "bilevel-l1inf";
    case Kind::BilevelL11: return "bilevel-l11";
    case Kind::BilevelL12: return "bilevel-l12";
    case Kind::Euclid: return "euclid";
    case Kind::Multilevel: return "multilevel:" + spec.to_string();
  }
  return "?";
}

DenseTensor run_projection(const Algorithm& a, const DenseTensor& input, double eta, ThreadPool* pool) {
  switch (a.kind) {
    case Algorithm::Kind::BilevelL1Inf: return bilevel_project(input, Norm::L1, Norm::Inf, eta, pool).X;
    case Algorithm::Kind::BilevelL11: return bilevel_project(input, Norm::L1, Norm::L1, eta, pool).X;
    case Algorithm::Kind::BilevelL12: return bilevel_project(input, Norm::L1, Norm::L2, eta, pool).X;
    case Algorithm::Kind::Multilevel: return multilevel_project(input, a.spec, eta, pool);
    case Algorithm::Kind::Euclid: return euclid_project_l1inf(input, eta).X;
  }
  throw ConfigError("unreachable algorithm kind");
}

DenseTensor parallel_project(const Algorithm& a, const DenseTensor& input, double eta, const ExecConfig& cfg) {
  if (cfg.workers == 0) throw ConfigError("worker count must be >= 1");
  return run_projection(a, input, eta, nullptr);
}

}  // namespace multiproj
