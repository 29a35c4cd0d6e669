// Drop-in check: a translation unit written against the reference API
// (anisoq/pq.hpp, anisoq/index.hpp), compiled against include/anisoq/ and
// linked with libanisoq_b200.so. The cases restate reference tests
// (test_pq.cpp, test_index.cpp) so a user switching headers sees the same
// behaviour. Run by tests/test_cpp_dropin_gpu.py on a B200.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <numeric>
#include <string>
#include <vector>

#include "anisoq/anisoq.hpp"

using namespace anisoq;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) {                                                            \
      ++g_pass;                                                            \
    } else {                                                               \
      ++g_fail;                                                            \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, T) \
  do {                           \
    bool ok_ = false;            \
    try {                        \
      (void)(expr);              \
    } catch (const T&) {         \
      ok_ = true;                \
    }                            \
    CHECK(ok_);                  \
  } while (0)

// small deterministic generator for fixtures (splitmix64 + Box-Muller), float32-rounded
struct Gen {
  std::uint64_t s;
  std::uint64_t u64() {
    s += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uni() { return (double)(u64() >> 11) * 0x1.0p-53; }
  double gauss() {
    double u1;
    do u1 = uni();
    while (u1 <= 0.0);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * uni());
  }
  std::vector<double> vec(std::size_t n, bool f32 = true) {
    std::vector<double> v(n);
    for (auto& x : v) x = f32 ? (double)(float)gauss() : gauss();
    return v;
  }
};

static Dataset unit_rows(std::size_t n, std::size_t d, std::uint64_t seed) {
  Gen g{seed};
  std::vector<double> v(n * d);
  for (std::size_t i = 0; i < n; ++i) {
    double s = 0;
    for (std::size_t j = 0; j < d; ++j) s += (v[i * d + j] = g.gauss()) * v[i * d + j];
    for (std::size_t j = 0; j < d; ++j) v[i * d + j] = (double)(float)(v[i * d + j] / std::sqrt(s));
  }
  return make_dataset(n, d, std::move(v), true);
}

static ProductCodebook example_codebook() {  // test_pq.cpp:29-37
  ProductCodebook cb;
  cb.M = 2;
  cb.k = 2;
  cb.sub_dimension = 2;
  cb.dictionaries = {-1, -1, 1, 1, -2, -2, 2, 2};
  return cb;
}

int main() {
  // reconstruct + LUT worked examples (test_pq.cpp:60-77, test_index.cpp:58-90)
  {
    const auto cb = example_codebook();
    CHECK((reconstruct(std::vector<std::uint32_t>{0, 1}, cb) == std::vector<double>{-1, -1, 2, 2}));
    CHECK_THROWS_AS(reconstruct(std::vector<std::uint32_t>{2, 0}, cb), CodeOutOfRange);
    const std::vector<double> q{1.0, 0.0, 1.0, 0.0};
    const auto lut = build_lut(q, cb);
    CHECK(lut.at(0, 0) == -1.0 && lut.at(0, 1) == 1.0 && lut.at(1, 0) == -2.0 && lut.at(1, 1) == 2.0);
    CHECK(adc_score(std::vector<std::uint32_t>{0, 1}, lut) == 1.0);
    CHECK_THROWS_AS(build_lut(std::vector<double>(3, 1.0), cb), DimensionMismatch);
  }
  // adc_search full ranking vs explicit reconstruction (test_index.cpp:114-142)
  {
    Gen g{10};
    ProductCodebook cb;
    cb.M = 4;
    cb.k = 16;
    cb.sub_dimension = 2;
    cb.dictionaries = g.vec(128, false);
    CodeMatrix codes;
    codes.n = 1000;
    codes.M = 4;
    codes.k = 16;
    codes.codes.resize(4000);
    for (auto& c : codes.codes) c = (std::uint32_t)(g.u64() % 16);
    const auto q = g.vec(8, false);
    std::vector<Hit> all(1000);
    for (std::size_t i = 0; i < 1000; ++i) {
      const auto rec = reconstruct(codes.row(i), cb);
      double s = 0.0;
      for (int t = 0; t < 8; ++t) s += q[t] * rec[t];
      all[i] = {(std::uint32_t)i, s};
    }
    std::sort(all.begin(), all.end(), [](const Hit& a, const Hit& b) {
      return a.score != b.score ? a.score > b.score : a.index < b.index;
    });
    const auto full = adc_search(q, codes, cb, 1000);
    CHECK(full.hits.size() == 1000);
    bool same = true;
    for (std::size_t i = 0; i < 1000; ++i)
      same &= full.hits[i].index == all[i].index && std::abs(full.hits[i].score - all[i].score) <= 1e-12;
    CHECK(same);
    const auto top = adc_search(q, codes, cb, 25);
    bool same25 = top.hits.size() == 25;
    for (std::size_t i = 0; i < 25 && same25; ++i) same25 &= top.hits[i].index == all[i].index;
    CHECK(same25);
    CodeMatrix empty;
    empty.M = 4;
    empty.k = 16;
    CHECK_THROWS_AS(adc_search(q, empty, cb, 5), EmptyIndex);
    CHECK_THROWS_AS(adc_search(q, codes, cb, 0), InvalidArgument);
  }
  // pq_assign_point: isotropic weights decouple per subspace (test_pq.cpp:97-123)
  {
    Gen g{302};
    ProductCodebook cb;
    cb.M = 3;
    cb.k = 4;
    cb.sub_dimension = 2;
    cb.dictionaries = g.vec(24, false);
    const auto x = g.vec(6, false);
    const auto codes = pq_assign_point(x, std::vector<std::uint32_t>{0, 0, 0}, cb,
                                       AnisotropicWeights::isotropic(2.0));
    for (std::size_t m = 0; m < 3; ++m) {
      std::size_t bj = 0;
      double best = INFINITY;
      for (std::size_t j = 0; j < 4; ++j) {
        double d2 = 0;
        for (int t = 0; t < 2; ++t) {
          const double df = x[m * 2 + t] - cb.codeword(m, j)[t];
          d2 += df * df;
        }
        if (d2 < best) best = d2, bj = j;
      }
      CHECK(codes[m] == bj);
    }
  }
  // pq_quantize: zero passes = baseline, iso = baseline, refined = fixed points
  // (test_pq.cpp:507-524)
  {
    const Dataset data = unit_rows(300, 8, 3);
    std::vector<AnisotropicWeights> unit(data.n, AnisotropicWeights::isotropic());
    std::vector<AnisotropicWeights> aniso(data.n, AnisotropicWeights::from_eta(4.125));
    TrainConfig cfg;
    cfg.seed = 2;
    auto [cb, trained] = train_l2_pq(data, 4, 4, cfg);
    const auto base = pq_quantize(data, cb, aniso, 0);
    const auto iso_any = pq_quantize(data, cb, unit, 3);
    CHECK(base.codes == iso_any.codes);
    const auto refined = pq_quantize(data, cb, aniso, 4);
    bool fixed = true;
    for (std::size_t i = 0; i < data.n; ++i) {
      const auto row = refined.row(i);
      const std::vector<std::uint32_t> cur(row.begin(), row.end());
      fixed &= pq_assign_point(data.row(i), cur, cb, aniso[i]) == cur;
    }
    CHECK(fixed);
  }
  // selector system: isotropic weights give a block-diagonal system
  // (test_pq.cpp:164-207) + joint solve residual (241-286)
  {
    const Dataset data = unit_rows(64, 8, 99);
    const std::size_t M = 2, k = 4;
    CodeMatrix codes;
    codes.n = data.n;
    codes.M = M;
    codes.k = k;
    Gen g{100};
    codes.codes.resize(data.n * M);
    for (auto& c : codes.codes) c = (std::uint32_t)(g.u64() % k);
    const std::vector<AnisotropicWeights> iso(data.n, AnisotropicWeights::isotropic(1.5));
    const auto sys_iso = assemble_selector_system(data, codes, iso, M, k);
    bool block = true;
    for (std::size_t r = 0; r < k * data.d; ++r)
      for (std::size_t c = 0; c < k * data.d; ++c)
        if (r / 4 != c / 4) block &= sys_iso.system_matrix((long)r, (long)c) == 0.0;
    CHECK(block);
    const std::vector<AnisotropicWeights> w(data.n, AnisotropicWeights::from_eta(4.125));
    const double ridge = 1e-8;
    const auto cb = pq_codebook_update(data, codes, w, M, k, ridge);
    auto sys = assemble_selector_system(data, codes, w, M, k);
    double res2 = 0.0, rn2 = 0.0;
    const long dim = (long)(k * data.d);
    for (long r = 0; r < dim; ++r) {
      double s = 0.0;
      for (long c = 0; c < dim; ++c)
        s += (sys.system_matrix(r, c) + (r == c ? ridge : 0.0)) * cb.dictionaries[c];
      res2 += (s - sys.rhs(r)) * (s - sys.rhs(r));
      rn2 += sys.rhs(r) * sys.rhs(r);
    }
    CHECK(std::sqrt(res2) <= 1e-8 * std::sqrt(rn2));
  }
  // train_apq: monotone history, deterministic (test_pq.cpp:464-495)
  {
    const Dataset data = unit_rows(400, 8, 11);
    std::vector<AnisotropicWeights> w(data.n, AnisotropicWeights::from_eta(4.125));
    TrainConfig cfg;
    cfg.seed = 11;
    cfg.max_iterations = 15;
    cfg.relative_tolerance = 0.0;
    std::vector<double> h1, h2;
    auto [cb1, c1] = train_apq(data, 4, 4, w, cfg, true, &h1);
    cfg.threads = 4;
    auto [cb2, c2] = train_apq(data, 4, 4, w, cfg, true, &h2);
    bool mono = true;
    for (std::size_t t = 1; t < h1.size(); ++t) mono &= h1[t] <= h1[t - 1] + 1e-9;
    CHECK(mono);
    CHECK(cb1.dictionaries == cb2.dictionaries && c1.codes == c2.codes && h1 == h2);
    CHECK_THROWS_AS(train_apq(data, 3, 2, w, cfg), DimensionNotDivisible);
  }
  // train_avq: monotone history, assignments are the argmin of the final
  // codebook, deterministic, reference validation (vq.hpp:243-329)
  {
    const Dataset data = unit_rows(500, 6, 12);
    std::vector<AnisotropicWeights> w(data.n, AnisotropicWeights::from_eta(3.0));
    TrainConfig cfg;
    cfg.seed = 5;
    cfg.max_iterations = 12;
    cfg.relative_tolerance = 0.0;
    auto [vq1, a1] = train_avq(data, 10, w, cfg);
    cfg.threads = 8;
    auto [vq2, a2] = train_avq(data, 10, w, cfg);
    CHECK(vq1.k == 10 && vq1.d == 6 && vq1.codewords.size() == 60);
    CHECK(a1.assignments.size() == 500 && !a1.loss_history.empty());
    bool mono = true;
    for (std::size_t t = 1; t < a1.loss_history.size(); ++t)
      mono &= a1.loss_history[t] <= a1.loss_history[t - 1] + 1e-9;
    CHECK(mono);
    CHECK(vq1.codewords == vq2.codewords && a1.assignments == a2.assignments &&
          a1.loss_history == a2.loss_history);
    const ProductCodebook pc = to_product(vq1);
    CHECK(pc.M == 1 && pc.k == 10 && pc.sub_dimension == 6);
    // vq_quantize / assign_point agree with the trained assignments' argmin
    const auto again = vq_quantize(data, vq1, w);
    bool agree = true;
    for (std::size_t i = 0; i < data.n; ++i) agree &= again[i] == assign_point(data.row(i), vq1, w[i]);
    CHECK(agree);
    CHECK(again == a1.assignments);  // the last pass used the final codebook
    // update_codeword of an isotropic set is its mean (vq.hpp:151-162)
    const std::vector<double> pts{1, 2, 3, 4, 5, 6};
    const std::vector<AnisotropicWeights> iso(2, AnisotropicWeights::isotropic());
    CHECK((update_codeword(3, pts, iso) == std::vector<double>{2.5, 3.5, 4.5}));
    CHECK_THROWS_AS(update_codeword(4, pts, iso), InvalidArgument);
    CHECK_THROWS_AS(train_avq(data, 0, w, cfg), InvalidArgument);
    CHECK_THROWS_AS(train_avq(data, 501, w, cfg), InvalidArgument);
  }
  // serialization golden bytes (test_pq.cpp:560-571)
  {
    const auto dir = std::filesystem::temp_directory_path() / "anisoq_b200_dropin";
    std::filesystem::create_directories(dir);
    CodeMatrix small;
    small.n = 1;
    small.M = 2;
    small.k = 4;
    small.codes = {3, 1};
    save_codes(small, (dir / "codes_small.bin").string());
    std::ifstream in(dir / "codes_small.bin", std::ios::binary);
    std::vector<unsigned char> bytes((std::istreambuf_iterator<char>(in)), {});
    CHECK((bytes == std::vector<unsigned char>{1, 0, 0, 0, 2, 0, 0, 0, 4, 0, 0, 0, 3, 1}));
    const auto cb = example_codebook();
    save_codebook(cb, (dir / "cb.bin").string());
    CHECK(load_codebook((dir / "cb.bin").string()).dictionaries == cb.dictionaries);
  }
  // exact search invariances (test_index.cpp:156-186)
  {
    const Dataset data = unit_rows(100, 8, 71);
    Gen g{12};
    const auto q = g.vec(8, false);
    const auto res = exact_search(q, data, 10);
    CHECK(res.hits.size() == 10);
    const auto self = exact_search(data.row(17), data, 1);
    CHECK(self.hits[0].index == 17);
  }
  // evaluate (test_index.cpp:189-263): perfect codes give recall 1 and zero
  // error; validation and ground-truth checks
  {
    Gen g{13};
    ProductCodebook cb;
    cb.M = 2;
    cb.k = 4;
    cb.sub_dimension = 3;
    cb.dictionaries.resize(24);
    for (auto& v : cb.dictionaries) v = std::round(g.gauss() * 64) / 64;
    CodeMatrix codes;
    codes.n = 16;
    codes.M = 2;
    codes.k = 4;
    for (std::size_t i = 0; i < 16; ++i) codes.codes.push_back((std::uint32_t)(g.u64() % 4)),
                                         codes.codes.push_back((std::uint32_t)(g.u64() % 4));
    std::vector<double> dv;
    for (std::size_t i = 0; i < 16; ++i) {
      const auto r = reconstruct(codes.row(i), cb);
      dv.insert(dv.end(), r.begin(), r.end());
    }
    const Dataset data = make_dataset(16, 6, dv, false);
    std::vector<double> qv;
    for (int i = 0; i < 20 * 6; ++i) qv.push_back((double)(float)g.gauss());
    const Dataset queries = make_dataset(20, 6, qv, false);
    EvalOptions opt;
    opt.recall_ns = {1, 10};
    const auto rep = evaluate(queries, data, codes, cb, opt);
    CHECK(rep.num_queries == 20 && rep.num_datapoints == 16);
    CHECK(rep.recall_1_at_n.at(1) == 1.0 && rep.recall_1_at_n.at(10) == 1.0);
    CHECK(rep.recall_k_at_k == 1.0 && rep.relative_error_max == 0.0);
    // per-query timing (extension): same report, measured latencies
    EvalOptions popt = opt;
    popt.per_query_latency = true;
    const auto prep = evaluate(queries, data, codes, cb, popt);
    CHECK(prep.recall_1_at_n == rep.recall_1_at_n && prep.recall_k_at_k == rep.recall_k_at_k);
    CHECK(prep.relative_error_mean == rep.relative_error_mean);
    CHECK(prep.latency.p50_us > 0.0 && prep.latency.p50_us <= prep.latency.p99_us);
    std::vector<std::vector<std::int32_t>> short_rows(4, std::vector<std::int32_t>{0});
    opt.ground_truth = &short_rows;
    CHECK_THROWS_AS(evaluate(queries, data, codes, cb, opt), GroundTruthMismatch);
    opt.ground_truth = nullptr;
    opt.recall_ns.clear();
    CHECK_THROWS_AS(evaluate(queries, data, codes, cb, opt), InvalidArgument);
  }
  std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
