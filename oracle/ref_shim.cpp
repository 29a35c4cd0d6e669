// oracle/_ref shim — TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers (/root/reference/proj/include,
// included in place, never copied) against the Eigen-subset stand-in
// (oracle/eigen_subset) and exposes the hot-path functions over a C ABI so
// tests/ and bench.py's reference arm can call the reference itself.
// Built by oracle/Makefile into oracle/_ref/libanisoq_ref.so with the
// reference's own floating-point flag (-ffp-contract=off,
// proj/CMakeLists.txt:11-13).
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference) may load this library; the product never does.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "anisoq/anisoq.hpp"
#include "../include/anisoq_b200.h"

using namespace anisoq;

namespace {

thread_local std::string g_err;

int map_error(const Error& e) {
  const std::string w = e.what();
  static const char* names[] = {
      "InvalidArgument", "ZeroNormDatapoint", "InvalidThreshold",
      "EmptyDataset", "EmptyIndex", "DimensionMismatch",
      "DimensionNotDivisible", "CodeOutOfRange", "MalformedFile",
      "InsufficientData", "GroundTruthMismatch", "QuadratureFailure",
      "SingularSystem"};
  g_err = w;
  for (int i = 0; i < 13; ++i) {
    const std::string p = std::string(names[i]) + ": ";
    if (w.compare(0, p.size(), p) == 0) return i + 1;
  }
  return AQ_E_INVALID_ARGUMENT;
}

#define GUARD_BEGIN try {
#define GUARD_END                                    \
  }                                                  \
  catch (const Error& e) { return map_error(e); }    \
  catch (const std::exception& e) {                  \
    g_err = e.what();                                \
    return AQ_E_CUDA;                                \
  }                                                  \
  return AQ_OK;

Dataset make_ds(const double* x, std::size_t n, std::size_t d) {
  std::vector<double> v(x, x + n * d);
  return detail::make_dataset_unchecked(n, d, std::move(v));
}

ProductCodebook make_cb(const double* dict, std::size_t M, std::size_t k,
                        std::size_t sd) {
  ProductCodebook cb;
  cb.M = M;
  cb.k = k;
  cb.sub_dimension = sd;
  cb.dictionaries.assign(dict, dict + M * k * sd);
  return cb;
}

CodeMatrix make_codes(const std::uint32_t* c, std::size_t n, std::size_t M,
                      std::size_t k) {
  CodeMatrix cm;
  cm.n = n;
  cm.M = M;
  cm.k = k;
  cm.codes.assign(c, c + n * M);
  return cm;
}

std::vector<AnisotropicWeights> make_w(const double* hp, const double* ho,
                                       std::size_t n) {
  std::vector<AnisotropicWeights> w(n);
  for (std::size_t i = 0; i < n; ++i)
    w[i] = AnisotropicWeights::from_h(hp[i], ho[i]);
  return w;
}

TrainConfig make_cfg(int max_it, double tol, std::uint64_t seed, double ridge,
                     int threads, int sweep_fixed) {
  TrainConfig cfg;
  cfg.max_iterations = max_it;
  cfg.relative_tolerance = tol;
  cfg.seed = seed;
  cfg.ridge = ridge;
  cfg.threads = threads;
  cfg.sweep_to_fixed_point = sweep_fixed != 0;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_row_norms(const double* x, std::size_t n, std::size_t d,
                  double* norms) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  std::copy(ds.norms.begin(), ds.norms.end(), norms);
  GUARD_END
}

int ref_eta_limit(double t, double norm, int d, double* out) {
  GUARD_BEGIN
  *out = eta_limit(t, norm, d);
  GUARD_END
}

int ref_pq_quantize(const double* x, std::size_t n, std::size_t d,
                    const double* dict, std::size_t M, std::size_t k,
                    std::size_t sd, const double* hp, const double* ho,
                    int passes, int threads, std::uint32_t* codes_out) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const auto cb = make_cb(dict, M, k, sd);
  const auto w = make_w(hp, ho, n);
  const CodeMatrix cm = pq_quantize(ds, cb, w, passes, threads);
  std::copy(cm.codes.begin(), cm.codes.end(), codes_out);
  GUARD_END
}

int ref_pq_assign_pass(const double* x, std::size_t n, std::size_t d,
                       const double* dict, std::size_t M, std::size_t k,
                       std::size_t sd, const double* hp, const double* ho,
                       int threads, int sweep_fixed, std::uint32_t* codes,
                       double* losses) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const auto cb = make_cb(dict, M, k, sd);
  const auto w = make_w(hp, ho, n);
  CodeMatrix cm = make_codes(codes, n, M, k);
  std::vector<double> l(n, 0.0);
  detail::pq_assign_pass(ds, cb, w, threads, sweep_fixed != 0, cm, l);
  std::copy(cm.codes.begin(), cm.codes.end(), codes);
  std::copy(l.begin(), l.end(), losses);
  GUARD_END
}

int ref_pq_assign_point(const double* x, std::size_t d,
                        const std::uint32_t* cur, const double* dict,
                        std::size_t M, std::size_t k, std::size_t sd,
                        double hp, double ho, std::uint32_t* out) {
  GUARD_BEGIN
  const auto cb = make_cb(dict, M, k, sd);
  const auto w = AnisotropicWeights::from_h(hp, ho);
  const auto r = pq_assign_point(std::span<const double>(x, d),
                                 std::span<const std::uint32_t>(cur, M), cb, w);
  std::copy(r.begin(), r.end(), out);
  GUARD_END
}

int ref_pq_assign_point_order(const double* x, std::size_t d,
                              const std::uint32_t* cur, const double* dict,
                              std::size_t M, std::size_t k, std::size_t sd,
                              double hp, double ho, const std::size_t* order,
                              std::size_t order_len, std::uint32_t* out) {
  GUARD_BEGIN
  const auto cb = make_cb(dict, M, k, sd);
  const auto w = AnisotropicWeights::from_h(hp, ho);
  const auto r = pq_assign_point(std::span<const double>(x, d),
                                 std::span<const std::uint32_t>(cur, M), cb, w,
                                 std::span<const std::size_t>(order, order_len));
  std::copy(r.begin(), r.end(), out);
  GUARD_END
}

// A_out is row-major dim x dim, dim = k*d.
int ref_assemble_selector_system(const double* x, std::size_t n,
                                 std::size_t d, const std::uint32_t* codes,
                                 const double* hp, const double* ho,
                                 std::size_t M, std::size_t k, double* A_out,
                                 double* rhs_out) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const auto w = make_w(hp, ho, n);
  const CodeMatrix cm = make_codes(codes, n, M, k);
  const SelectorSystem sys = assemble_selector_system(ds, cm, w, M, k);
  const std::size_t dim = k * d;
  for (std::size_t r = 0; r < dim; ++r)
    for (std::size_t c = 0; c < dim; ++c)
      A_out[r * dim + c] = sys.system_matrix(static_cast<Eigen::Index>(r),
                                             static_cast<Eigen::Index>(c));
  std::copy(sys.rhs.data(), sys.rhs.data() + dim, rhs_out);
  GUARD_END
}

int ref_pq_codebook_update(const double* x, std::size_t n, std::size_t d,
                           const std::uint32_t* codes, const double* hp,
                           const double* ho, std::size_t M, std::size_t k,
                           double ridge, double* dict_out) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const auto w = make_w(hp, ho, n);
  const CodeMatrix cm = make_codes(codes, n, M, k);
  const auto cb = pq_codebook_update(ds, cm, w, M, k, ridge);
  std::copy(cb.dictionaries.begin(), cb.dictionaries.end(), dict_out);
  GUARD_END
}

int ref_train_l2_pq(const double* x, std::size_t n, std::size_t d,
                    std::size_t M, std::size_t k, int max_it, double tol,
                    std::uint64_t seed, int threads, double* dict_out,
                    std::uint32_t* codes_out) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const TrainConfig cfg = make_cfg(max_it, tol, seed, -1.0, threads, 0);
  auto [cb, cm] = train_l2_pq(ds, M, k, cfg);
  std::copy(cb.dictionaries.begin(), cb.dictionaries.end(), dict_out);
  std::copy(cm.codes.begin(), cm.codes.end(), codes_out);
  GUARD_END
}

// history_out must hold max_it + 1 doubles.
int ref_train_apq(const double* x, std::size_t n, std::size_t d,
                  std::size_t M, std::size_t k, const double* hp,
                  const double* ho, int max_it, double tol, std::uint64_t seed,
                  double ridge, int threads, int sweep_fixed, int warm_start,
                  double* dict_out, std::uint32_t* codes_out,
                  double* history_out, std::size_t* history_len) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const auto w = make_w(hp, ho, n);
  const TrainConfig cfg = make_cfg(max_it, tol, seed, ridge, threads, sweep_fixed);
  std::vector<double> hist;
  auto [cb, cm] = train_apq(ds, M, k, w, cfg, warm_start != 0, &hist);
  std::copy(cb.dictionaries.begin(), cb.dictionaries.end(), dict_out);
  std::copy(cm.codes.begin(), cm.codes.end(), codes_out);
  std::copy(hist.begin(), hist.end(), history_out);
  *history_len = hist.size();
  GUARD_END
}

int ref_vq_quantize(const double* x, std::size_t n, std::size_t d, const double* cw,
                    std::size_t k, const double* hp, const double* ho, int threads,
                    std::uint32_t* assign_out) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const auto w = make_w(hp, ho, n);
  Codebook cb;
  cb.k = k;
  cb.d = d;
  cb.codewords.assign(cw, cw + k * d);
  const auto a = vq_quantize(ds, cb, w, threads);
  std::copy(a.begin(), a.end(), assign_out);
  GUARD_END
}

int ref_assign_point(const double* x, std::size_t d, const double* cw, std::size_t k,
                     double hp, double ho, std::uint32_t* out) {
  GUARD_BEGIN
  Codebook cb;
  cb.k = k;
  cb.d = d;
  cb.codewords.assign(cw, cw + k * d);
  *out = static_cast<std::uint32_t>(
      assign_point(std::span<const double>(x, d), cb, AnisotropicWeights::from_h(hp, ho)));
  GUARD_END
}

int ref_update_codeword(std::size_t d, const double* pts, std::size_t m, const double* hp,
                        const double* ho, double ridge, double* out) {
  GUARD_BEGIN
  const auto w = make_w(hp, ho, m);
  const auto c = update_codeword(d, std::span<const double>(pts, m * d), w, ridge);
  std::copy(c.begin(), c.end(), out);
  GUARD_END
}

int ref_train_avq(const double* x, std::size_t n, std::size_t d, std::size_t k,
                  const double* hp, const double* ho, int max_it, double tol,
                  std::uint64_t seed, double ridge, int threads, int keep_previous,
                  double* cw_out, std::uint32_t* assign_out, double* history_out,
                  std::size_t* history_len) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const auto w = make_w(hp, ho, n);
  TrainConfig cfg = make_cfg(max_it, tol, seed, ridge, threads, 0);
  cfg.empty_partition_policy = keep_previous ? EmptyPartitionPolicy::keep_previous
                                             : EmptyPartitionPolicy::reseed_highest_loss;
  auto [cb, a] = train_avq(ds, k, w, cfg);
  std::copy(cb.codewords.begin(), cb.codewords.end(), cw_out);
  std::copy(a.assignments.begin(), a.assignments.end(), assign_out);
  std::copy(a.loss_history.begin(), a.loss_history.end(), history_out);
  *history_len = a.loss_history.size();
  GUARD_END
}

int ref_build_lut(const double* q, std::size_t d, const double* dict,
                  std::size_t M, std::size_t k, std::size_t sd,
                  double* lut_out) {
  GUARD_BEGIN
  const auto cb = make_cb(dict, M, k, sd);
  const LookupTable lut = build_lut(std::span<const double>(q, d), cb);
  std::copy(lut.partials.begin(), lut.partials.end(), lut_out);
  GUARD_END
}

// Batched adc_search, parallel over queries exactly as evaluate() runs it
// (index.hpp:251-294, chunk 16). ids/scores: nq x topn_eff.
int ref_adc_search_batch(const double* Q, std::size_t nq, std::size_t d,
                         const std::uint32_t* codes, std::size_t n,
                         std::size_t M, std::size_t codes_k,
                         const double* dict, std::size_t cbM, std::size_t k,
                         std::size_t sd, std::size_t topn, int threads,
                         std::uint32_t* ids_out, double* scores_out,
                         std::size_t* count_out) {
  GUARD_BEGIN
  const auto cb = make_cb(dict, cbM, k, sd);
  CodeMatrix cm;
  cm.n = n;
  cm.M = M;
  cm.k = codes_k;
  cm.codes.assign(codes, codes + n * M);
  const std::size_t topn_eff = std::min(topn, n);
  *count_out = topn_eff;
  parallel_for(nq, threads, [&](std::size_t b, std::size_t e) {
    for (std::size_t qi = b; qi < e; ++qi) {
      const SearchResult r =
          adc_search(std::span<const double>(Q + qi * d, d), cm, cb, topn);
      for (std::size_t t = 0; t < r.hits.size(); ++t) {
        ids_out[qi * topn_eff + t] = r.hits[t].index;
        scores_out[qi * topn_eff + t] = r.hits[t].score;
      }
    }
  }, 16);
  GUARD_END
}

// Exact-dot rerank (north_star; not in the reference): for each query the
// candidate ids are rescored with detail::dot (geometry.hpp:170-174) and the
// best `keep` kept in select_top order (index.hpp:88-112).
int ref_rerank(const double* Q, std::size_t nq, const double* x,
               std::size_t n, std::size_t d, const std::uint32_t* cand,
               std::size_t ncand, std::size_t keep, int threads,
               std::uint32_t* ids_out, double* scores_out) {
  GUARD_BEGIN
  const std::size_t keep_eff = std::min(keep, ncand);
  parallel_for(nq, threads, [&](std::size_t b, std::size_t e) {
    for (std::size_t qi = b; qi < e; ++qi) {
      const std::span<const double> q(Q + qi * d, d);
      std::vector<Hit> hits(ncand);
      for (std::size_t c = 0; c < ncand; ++c) {
        const std::uint32_t id = cand[qi * ncand + c];
        hits[c] = {id, detail::dot(q, std::span<const double>(x + id * d, d))};
      }
      std::sort(hits.begin(), hits.end(), [](const Hit& a, const Hit& b) {
        if (a.score != b.score) return a.score > b.score;
        return a.index < b.index;
      });
      for (std::size_t t = 0; t < keep_eff; ++t) {
        ids_out[qi * keep_eff + t] = hits[t].index;
        scores_out[qi * keep_eff + t] = hits[t].score;
      }
    }
  }, 16);
  (void)n;
  GUARD_END
}

int ref_exact_search_batch(const double* Q, std::size_t nq, const double* x,
                           std::size_t n, std::size_t d, std::size_t depth,
                           int threads, std::uint32_t* ids_out,
                           double* scores_out) {
  GUARD_BEGIN
  const Dataset ds = make_ds(x, n, d);
  const std::size_t depth_eff = std::min(depth, n);
  parallel_for(nq, threads, [&](std::size_t b, std::size_t e) {
    for (std::size_t qi = b; qi < e; ++qi) {
      const SearchResult r =
          exact_search(std::span<const double>(Q + qi * d, d), ds, depth);
      for (std::size_t t = 0; t < r.hits.size(); ++t) {
        ids_out[qi * depth_eff + t] = r.hits[t].index;
        scores_out[qi * depth_eff + t] = r.hits[t].score;
      }
    }
  }, 4);
  GUARD_END
}

// Reference Rng (rng.hpp:28-89) for fixtures.
int ref_rng_gaussians(std::uint64_t seed, std::size_t count, double* out) {
  Rng rng(seed);
  for (std::size_t i = 0; i < count; ++i) out[i] = rng.next_gaussian();
  return AQ_OK;
}

int ref_sample_distinct(std::uint64_t seed, std::size_t n, std::size_t k,
                        std::size_t* out) {
  Rng rng(seed);
  const auto v = rng.sample_distinct(n, k);
  std::copy(v.begin(), v.end(), out);
  return AQ_OK;
}

// generate_synthetic (dataset.hpp:244-290); values row-major n x d.
int ref_generate_synthetic(int kind, std::size_t n, std::size_t d,
                           std::uint64_t seed, std::size_t centers,
                           double spread, int normalize, double* out) {
  GUARD_BEGIN
  SyntheticParams p;
  p.centers = centers;
  p.spread = spread;
  p.normalize = normalize != 0;
  const Dataset ds = generate_synthetic(
      kind == 0 ? SyntheticKind::uniform_sphere
                : SyntheticKind::gaussian_mixture,
      n, d, seed, p);
  std::copy(ds.values.begin(), ds.values.end(), out);
  GUARD_END
}

}  // extern "C"
