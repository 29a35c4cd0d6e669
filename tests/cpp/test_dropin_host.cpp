// Host-side parts of the drop-in headers (no device calls): the reference
// generator, fvecs/ivecs I/O, Rng, VQ <-> product codebook conversions.
// Writes generated datasets to argv[1] for tests/test_cpp_dropin_gpu.py to
// compare with the reference's own generator.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "anisoq/anisoq.hpp"

using namespace anisoq;

static int fails = 0;
#define CHECK(c)                                                    \
  do {                                                              \
    if (!(c)) {                                                     \
      ++fails;                                                      \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                               \
  } while (0)

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  SyntheticParams p;
  p.centers = 6;
  p.spread = 0.25;
  p.normalize = true;
  const Dataset mix = generate_synthetic(SyntheticKind::gaussian_mixture, 200, 8, 7, p);
  const Dataset sph = generate_synthetic(SyntheticKind::uniform_sphere, 50, 5, 3);
  write_fvecs(mix, dir + "/mix.fvecs");
  write_fvecs(sph, dir + "/sphere.fvecs");
  const Dataset back = read_fvecs(dir + "/mix.fvecs");
  CHECK(back.n == 200 && back.d == 8 && back.values == mix.values);
  const std::vector<std::vector<std::int32_t>> rows{{1, 2, 3}, {}, {7}};
  write_ivecs(rows, dir + "/rows.ivecs");
  CHECK(read_ivecs(dir + "/rows.ivecs") == rows);
  Rng r(11);
  const auto s = r.sample_distinct(10, 4);
  CHECK(s.size() == 4);
  Codebook vq;
  vq.k = 3;
  vq.d = 2;
  vq.codewords = {1, 2, 3, 4, 5, 6};
  const auto pcb = to_product(vq);
  CHECK(pcb.M == 1 && pcb.k == 3 && pcb.sub_dimension == 2 && to_vq(pcb).codewords == vq.codewords);
  bool threw = false;
  try {
    ProductCodebook two;
    two.M = 2;
    (void)to_vq(two);
  } catch (const InvalidArgument&) {
    threw = true;
  }
  CHECK(threw);
  const Dataset unit = unit_normalize(back);
  CHECK(unit.normalized && unit.n == back.n);
  std::printf("dropin_host: %d failed\n", fails);
  // parallel_for: per-index results independent of the thread count, first
  // error rethrown (parallel.hpp); fnv1a64 known answers (dataset.hpp:62-70)
  {
    std::vector<double> a(100003), b(100003);
    parallel_for(a.size(), 1, [&](std::size_t lo, std::size_t hi) {
      for (auto i = lo; i < hi; ++i) a[i] = std::sqrt((double)i) * 3.0;
    });
    parallel_for(b.size(), 7, [&](std::size_t lo, std::size_t hi) {
      for (auto i = lo; i < hi; ++i) b[i] = std::sqrt((double)i) * 3.0;
    }, 333);
    CHECK(a == b);
    bool thrown = false;
    try {
      parallel_for(5000, 4, [&](std::size_t lo, std::size_t) {
        if (lo == 2048) throw InvalidArgument("boom");
      });
    } catch (const InvalidArgument&) {
      thrown = true;
    }
    CHECK(thrown);
    CHECK(detail::fnv1a64("", 0) == 0xcbf29ce484222325ull);
    CHECK(detail::fnv1a64("a", 1) == 0xaf63dc4c8601ec8cull);
  }
  return fails ? 1 : 0;
}
