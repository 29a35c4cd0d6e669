// anisoq drop-in (B200): the reference's host work splitter (parallel.hpp:
// resolve_threads, parallel_for). The device paths never use it (their
// results do not depend on `threads`); it is kept for callers that split
// their own host loops the reference's way.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

namespace anisoq {

// threads <= 0: one worker per hardware thread (at least one).
inline int resolve_threads(int threads) {
  if (threads > 0) return threads;
  return std::max(1, static_cast<int>(std::thread::hardware_concurrency()));
}

// fn(begin, end) over [0, n) in chunks of `chunk` indices; chunk edges are
// fixed by n and chunk alone, so per-index results do not depend on
// `threads`. Workers claim chunks from a shared counter; the first exception
// thrown by fn is rethrown after every worker has stopped.
template <class Fn>
void parallel_for(std::size_t n, int threads, Fn&& fn, std::size_t chunk = 1024) {
  if (n == 0) return;
  const std::size_t chunks = (n + chunk - 1) / chunk;
  auto span = [&](std::size_t c, std::size_t& b, std::size_t& e) {
    b = c * chunk;
    e = std::min(n, b + chunk);
  };
  const std::size_t workers =
      std::min<std::size_t>(static_cast<std::size_t>(resolve_threads(threads)), chunks);
  if (workers <= 1) {
    for (std::size_t c = 0; c < chunks; ++c) {
      std::size_t b, e;
      span(c, b, e);
      fn(b, e);
    }
    return;
  }
  std::atomic<std::size_t> cursor{0};
  std::atomic<bool> failed{false};
  std::exception_ptr error;
  std::mutex lock;
  auto run = [&] {
    while (!failed.load(std::memory_order_relaxed)) {
      const std::size_t c = cursor.fetch_add(1);
      if (c >= chunks) break;
      std::size_t b, e;
      span(c, b, e);
      try {
        fn(b, e);
      } catch (...) {
        std::lock_guard<std::mutex> g(lock);
        if (!error) error = std::current_exception();
        failed = true;
      }
    }
  };
  std::vector<std::thread> pool;
  for (std::size_t t = 1; t < workers; ++t) pool.emplace_back(run);
  run();
  for (auto& t : pool) t.join();
  if (error) std::rethrow_exception(error);
}

}  // namespace anisoq
