// multiproj/parallel.hpp -- B200 drop-in for the reference CPU pool
// (proj/include/multiproj/parallel.hpp).  The projections themselves run on
// the GPU grid and ignore the pool argument (results never depended on the
// worker count in the reference either); the pool stays for API parity and
// for callers that use parallel_for directly.
#ifndef MULTIPROJ_PARALLEL_HPP
#define MULTIPROJ_PARALLEL_HPP

#include <cstddef>
#include <functional>

#include "multiproj/errors.hpp"

namespace multiproj {

struct ExecConfig {
  unsigned workers = 1;
};

class ThreadPool {
 public:
  explicit ThreadPool(unsigned workers);  // ConfigError when workers == 0
  ThreadPool(const ThreadPool&) = delete;
  ThreadPool& operator=(const ThreadPool&) = delete;
  unsigned workers() const { return workers_; }
  // body(begin, end) once per non-empty chunk of ceil(count / workers).
  void parallel_for(std::size_t count, const std::function<void(std::size_t, std::size_t)>& body);

 private:
  unsigned workers_;
};

void parallel_for(ThreadPool* pool, std::size_t count, const std::function<void(std::size_t, std::size_t)>& body);

// MULTIPROJ_WORKERS from the environment, default 1.
unsigned default_workers();

}  // namespace multiproj

#endif
