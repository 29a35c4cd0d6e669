// anisoq drop-in (B200): anisotropic vector quantization API of the reference
// (vq.hpp:32-343) — Codebook, VqAssignment, TrainConfig and the public VQ
// functions (assign_point, update_codeword, train_avq, vq_quantize) with the
// reference's signatures and validation. The data-parallel work runs on the
// B200 (the M = 1 instances of the product-quantization kernels, which equal
// the VQ algorithm bit for bit: test_pq.cpp:79-95, 209-239).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "b200.hpp"
#include "dataset.hpp"
#include "error.hpp"
#include "geometry.hpp"

namespace anisoq {

// A single (M = 1) codebook (reference vq.hpp:32-43): k codewords of dimension d.
struct Codebook {
  std::size_t k = 0;
  std::size_t d = 0;
  std::vector<double> codewords;  // row-major k*d

  std::span<const double> row(std::size_t j) const { return {codewords.data() + j * d, d}; }
  std::span<double> mutable_row(std::size_t j) { return {codewords.data() + j * d, d}; }
};

// Result of train_avq (reference vq.hpp:45-50).
struct VqAssignment {
  std::vector<std::uint32_t> assignments;  // one codeword index per datapoint
  std::vector<double> loss_history;        // total loss after each assignment pass
};

enum class EmptyPartitionPolicy { reseed_highest_loss, keep_previous };

struct TrainConfig {
  int max_iterations = 100;
  double relative_tolerance = 1e-6;
  std::uint64_t seed = 0;
  EmptyPartitionPolicy empty_partition_policy = EmptyPartitionPolicy::reseed_highest_loss;
  double ridge = -1.0;
  int threads = 1;  // host knob of the reference; results never depend on it
  bool sweep_to_fixed_point = false;
};

namespace b200 {
inline aq_train_config to_c(const TrainConfig& c) {
  return aq_train_config{c.max_iterations, c.relative_tolerance, c.seed,
                         c.empty_partition_policy == EmptyPartitionPolicy::keep_previous ? 1 : 0,
                         c.ridge, c.threads, c.sweep_to_fixed_point ? 1 : 0};
}
// float64 rows in; the library stores them as float32 when exact, else float64
inline void upload(const Dataset& data, OwnedDataset& ds) {
  check(aq_dataset_upload_f64(session(), data.values.data(), data.n, data.d, &ds.p));
}
// codebook update over a resident dataset: ds, codes (n x M), per-point
// weights -> dictionaries (M k sd)
inline void codebook_update(const OwnedDataset& ds, std::size_t n, const std::uint32_t* codes,
                            std::size_t M, std::size_t k, std::size_t sd, const aq_weights* w,
                            double ridge, double* dict_out) {
  OwnedCodes cm;
  check(aq_codes_upload(session(), codes, n, M, k, &cm.p));
  OwnedCodebook cb;
  check(aq_codebook_upload(session(), nullptr, M, k, sd, &cb.p));
  check(aq_dev_pq_codebook_update(ds.p, cm.p, w, ridge, cb.p));
  check(aq_codebook_download(cb.p, dict_out));
}
}  // namespace b200

// vq.hpp:112-132: lowest-index argmin of the anisotropic loss over a VQ
// codebook — the M = 1 coordinate-descent step (bit-identical, test_pq.cpp:79-95).
inline std::size_t assign_point(std::span<const double> x, const Codebook& cb,
                                const AnisotropicWeights& w) {
  if (cb.k == 0) throw InvalidArgument("empty codebook");
  if (x.size() != cb.d) throw DimensionMismatch("datapoint dimension does not match codebook");
  const std::uint32_t cur = 0;
  std::uint32_t out = 0;
  b200::check(aq_pq_assign_point_order(b200::session(), x.data(), x.size(), &cur,
                                       cb.codewords.data(), 1, cb.k, cb.d, w.h_parallel,
                                       w.h_perpendicular, nullptr, 0, &out));
  return out;
}

// vq.hpp:139-192: closed-form codeword for a set of weighted points (the
// M = 1 branch of the device codebook update with every point in partition 0).
inline std::vector<double> update_codeword(std::size_t d, std::span<const double> points,
                                           std::span<const AnisotropicWeights> weights,
                                           double ridge = -1.0) {
  if (d == 0 || points.empty() || points.size() % d != 0)
    throw InvalidArgument("points must be a non-empty multiple of d");
  const std::size_t m = points.size() / d;
  if (weights.size() != m) throw InvalidArgument("need one weight per point");
  b200::WeightArgs wa;
  b200::make_weights(weights, wa);
  b200::OwnedDataset ds;
  b200::check(aq_dataset_upload_f64(b200::session(), points.data(), m, d, &ds.p));
  const std::vector<std::uint32_t> codes(m, 0u);
  std::vector<double> out(d);
  b200::codebook_update(ds, m, codes.data(), 1, 1, d, &wa.w, ridge, out.data());
  return out;
}

// vq.hpp:332-343: one assignment pass against a fixed VQ codebook.
inline std::vector<std::uint32_t> vq_quantize(const Dataset& data, const Codebook& cb,
                                              std::span<const AnisotropicWeights> weights,
                                              int threads = 1) {
  (void)threads;
  if (data.d != cb.d) throw DimensionMismatch("dataset dimension does not match codebook");
  if (weights.size() != data.n) throw InvalidArgument("need one AnisotropicWeights per datapoint");
  std::vector<std::uint32_t> codes(data.n, 0u);
  if (data.n == 0) return codes;
  b200::WeightArgs wa;
  b200::make_weights(weights, wa);
  if (b200::f32_exact(data.values)) {
    const std::vector<float> x = b200::to_f32(data);
    b200::check(aq_pq_assign_pass(b200::session(), x.data(), data.n, data.d,
                                  cb.codewords.data(), 1, cb.k, cb.d, &wa.w, 0, codes.data(),
                                  nullptr));
    return codes;
  }
  b200::OwnedDataset ds;
  b200::upload(data, ds);
  b200::OwnedCodebook dcb;
  b200::check(aq_codebook_upload(b200::session(), cb.codewords.data(), 1, cb.k, cb.d, &dcb.p));
  b200::OwnedCodes cm;
  b200::check(aq_codes_upload(b200::session(), codes.data(), data.n, 1, cb.k, &cm.p));
  std::uint64_t changed = 0;
  b200::check(aq_dev_pq_assign_pass(ds.p, dcb.p, &wa.w, 0, cm.p, nullptr, &changed));
  b200::check(aq_codes_download(cm.p, codes.data()));
  return codes;
}

// vq.hpp:243-329: anisotropic vector quantization (one full-dimensional
// codebook); the device trainer returns it as an M = 1 product codebook.
inline std::pair<Codebook, VqAssignment> train_avq(const Dataset& data, std::size_t k,
                                                   std::span<const AnisotropicWeights> weights,
                                                   const TrainConfig& config) {
  if (data.n == 0) throw EmptyDataset("cannot train on an empty dataset");
  if (k == 0 || k > data.n)
    throw InvalidArgument("need 1 <= k <= n (codewords come from datapoints)");
  if (weights.size() != data.n) throw InvalidArgument("need one AnisotropicWeights per datapoint");
  b200::OwnedDataset ds;
  b200::upload(data, ds);
  b200::WeightArgs wa;
  b200::make_weights(weights, wa);
  const aq_train_config cfg = b200::to_c(config);
  b200::OwnedCodebook cb;
  b200::OwnedCodes cm;
  std::vector<double> hist(static_cast<std::size_t>(std::max(config.max_iterations, 0)) + 1);
  std::size_t hl = 0;
  b200::check(aq_dev_train_avq(ds.p, k, &wa.w, &cfg, &cb.p, &cm.p, hist.data(), &hl));
  Codebook out;
  out.k = k;
  out.d = data.d;
  out.codewords.resize(k * data.d);
  b200::check(aq_codebook_download(cb.p, out.codewords.data()));
  VqAssignment a;
  a.assignments.resize(data.n);
  b200::check(aq_codes_download(cm.p, a.assignments.data()));
  a.loss_history.assign(hist.begin(), hist.begin() + hl);
  return {std::move(out), std::move(a)};
}

}  // namespace anisoq
