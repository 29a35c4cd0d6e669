// anisoq drop-in (B200): product quantization API of the reference
// (pq.hpp:36-730) — same types, names and signatures; every data-parallel
// step runs on the B200 through libanisoq_b200.so and returns results
// bit-identical to the reference's float64 CPU code.
#pragma once

#include <cstdint>
#include <cstring>
#include <fstream>
#include <span>
#include <string>
#include <utility>
#include <vector>

#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
#else
#include "eigen_dense_subset.hpp"
#endif

#include "b200.hpp"
#include "dataset.hpp"
#include "error.hpp"
#include "geometry.hpp"
#include "vq.hpp"

namespace anisoq {

struct ProductCodebook {
  std::size_t M = 0;
  std::size_t k = 0;
  std::size_t sub_dimension = 0;
  std::vector<double> dictionaries;  // (m*k + j) * sub_dimension

  std::size_t dim() const { return M * sub_dimension; }
  std::span<const double> codeword(std::size_t m, std::size_t j) const {
    return {dictionaries.data() + (m * k + j) * sub_dimension, sub_dimension};
  }
  std::span<double> mutable_codeword(std::size_t m, std::size_t j) {
    return {dictionaries.data() + (m * k + j) * sub_dimension, sub_dimension};
  }
};

struct CodeMatrix {
  std::size_t n = 0;
  std::size_t M = 0;
  std::size_t k = 0;
  std::vector<std::uint32_t> codes;  // row-major n x M

  std::span<const std::uint32_t> row(std::size_t i) const { return {codes.data() + i * M, M}; }
  std::span<std::uint32_t> mutable_row(std::size_t i) { return {codes.data() + i * M, M}; }
};

// Normal equations of the joint codebook problem (pq.hpp:69-74), Eigen-typed
// like the reference's: real Eigen when <Eigen/Dense> is on the include path,
// otherwise the dense subset the reference's callers use
// (eigen_dense_subset.hpp).
struct SelectorSystem {
  Eigen::MatrixXd system_matrix;
  Eigen::VectorXd rhs;
};

// VQ <-> M = 1 product codebook (pq.hpp:76-92)
inline ProductCodebook to_product(const Codebook& cb) {
  ProductCodebook out;
  out.M = 1;
  out.k = cb.k;
  out.sub_dimension = cb.d;
  out.dictionaries = cb.codewords;
  return out;
}
inline Codebook to_vq(const ProductCodebook& cb) {
  if (cb.M != 1) throw InvalidArgument("to_vq requires M == 1");
  Codebook out;
  out.k = cb.k;
  out.d = cb.sub_dimension;
  out.codewords = cb.dictionaries;
  return out;
}

inline std::vector<double> reconstruct(std::span<const std::uint32_t> codes_row,
                                       const ProductCodebook& cb) {
  if (codes_row.size() != cb.M) throw DimensionMismatch("need one code per subspace");
  std::vector<double> out(cb.dim());
  for (std::size_t m = 0; m < cb.M; ++m) {
    if (codes_row[m] >= cb.k)
      throw CodeOutOfRange("code " + std::to_string(codes_row[m]) + " >= k = " +
                           std::to_string(cb.k));
    const auto cw = cb.codeword(m, codes_row[m]);
    std::copy(cw.begin(), cw.end(), out.begin() + m * cb.sub_dimension);
  }
  return out;
}

namespace b200 {
inline ProductCodebook download(aq_codebook* cb, std::size_t M, std::size_t k, std::size_t sd) {
  ProductCodebook out;
  out.M = M;
  out.k = k;
  out.sub_dimension = sd;
  out.dictionaries.resize(M * k * sd);
  check(aq_codebook_download(cb, out.dictionaries.data()));
  return out;
}
inline CodeMatrix download(aq_codes* c, std::size_t n, std::size_t M, std::size_t k) {
  CodeMatrix out;
  out.n = n;
  out.M = M;
  out.k = k;
  out.codes.resize(n * M);
  check(aq_codes_download(c, out.codes.data()));
  return out;
}
}  // namespace b200

// pq.hpp:256-282
inline std::vector<std::uint32_t> pq_assign_point(std::span<const double> x,
                                                  std::span<const std::uint32_t> current_codes,
                                                  const ProductCodebook& cb,
                                                  const AnisotropicWeights& w,
                                                  std::span<const std::size_t> sweep_order = {}) {
  if (x.size() != cb.dim()) throw DimensionMismatch("datapoint dimension does not match codebook");
  if (current_codes.size() != cb.M) throw DimensionMismatch("need one current code per subspace");
  std::vector<std::uint32_t> out(cb.M);
  b200::check(aq_pq_assign_point_order(b200::session(), x.data(), x.size(),
                                       current_codes.data(), cb.dictionaries.data(), cb.M, cb.k,
                                       cb.sub_dimension, w.h_parallel, w.h_perpendicular,
                                       sweep_order.data(), sweep_order.size(), out.data()));
  return out;
}

// pq.hpp:290-343
inline SelectorSystem assemble_selector_system(const Dataset& data, const CodeMatrix& codes,
                                               std::span<const AnisotropicWeights> weights,
                                               std::size_t M, std::size_t k) {
  if (codes.n != data.n || codes.M != M)
    throw DimensionMismatch("code matrix does not match dataset");
  if (M == 0 || data.d % M != 0) throw DimensionNotDivisible("dimension not divisible by M");
  if (weights.size() != data.n) throw InvalidArgument("need one AnisotropicWeights per datapoint");
  const std::size_t dim = k * data.d;
  SelectorSystem sys;
  sys.system_matrix = Eigen::MatrixXd::Zero(static_cast<Eigen::Index>(dim),
                                            static_cast<Eigen::Index>(dim));
  sys.rhs = Eigen::VectorXd::Zero(static_cast<Eigen::Index>(dim));
  b200::OwnedDataset ds;
  b200::OwnedCodes cm;
  b200::upload(data, ds);
  b200::check(aq_codes_upload(b200::session(), codes.codes.data(), codes.n, M, k, &cm.p));
  b200::WeightArgs wa;
  b200::make_weights(weights, wa);
  // the device writes the matrix row-major; (r, c) and (c, r) are separately
  // rounded products (pq.hpp:333-336), so copy element-wise into Eigen's
  // column-major storage
  std::vector<double> a(dim * dim);
  b200::check(aq_dev_assemble_selector_system(ds.p, cm.p, &wa.w, a.data(), sys.rhs.data()));
  for (std::size_t r = 0; r < dim; ++r)
    for (std::size_t c = 0; c < dim; ++c)
      sys.system_matrix(static_cast<Eigen::Index>(r), static_cast<Eigen::Index>(c)) =
          a[r * dim + c];
  return sys;
}

// pq.hpp:356-464
inline ProductCodebook pq_codebook_update(const Dataset& data, const CodeMatrix& codes,
                                          std::span<const AnisotropicWeights> weights,
                                          std::size_t M, std::size_t k, double ridge = -1.0) {
  if (data.n == 0) throw EmptyDataset("cannot update on an empty dataset");
  if (codes.n != data.n || codes.M != M)
    throw DimensionMismatch("code matrix does not match dataset");
  if (M == 0 || data.d % M != 0) throw DimensionNotDivisible("dimension not divisible by M");
  if (weights.size() != data.n) throw InvalidArgument("need one AnisotropicWeights per datapoint");
  b200::WeightArgs wa;
  b200::make_weights(weights, wa);
  ProductCodebook cb;
  cb.M = M;
  cb.k = k;
  cb.sub_dimension = data.d / M;
  cb.dictionaries.resize(M * k * cb.sub_dimension);
  b200::OwnedDataset ds;
  b200::upload(data, ds);
  b200::codebook_update(ds, data.n, codes.codes.data(), M, k, cb.sub_dimension, &wa.w, ridge,
                        cb.dictionaries.data());
  return cb;
}

// pq.hpp:469-501
inline std::pair<ProductCodebook, CodeMatrix> train_l2_pq(const Dataset& data, std::size_t M,
                                                          std::size_t k,
                                                          const TrainConfig& config) {
  if (data.n == 0) throw EmptyDataset("cannot train on an empty dataset");
  if (M == 0 || data.d % M != 0) throw DimensionNotDivisible("dimension not divisible by M");
  if (k == 0 || k > data.n) throw InvalidArgument("need 1 <= k <= n");
  b200::OwnedDataset ds;
  b200::upload(data, ds);
  const aq_train_config cfg = b200::to_c(config);
  b200::OwnedCodebook cb;
  b200::OwnedCodes cm;
  b200::check(aq_dev_train_l2_pq(ds.p, M, k, &cfg, &cb.p, &cm.p));
  return {b200::download(cb.p, M, k, data.d / M), b200::download(cm.p, data.n, M, k)};
}

// pq.hpp:513-575
inline std::pair<ProductCodebook, CodeMatrix> train_apq(
    const Dataset& data, std::size_t M, std::size_t k, std::span<const AnisotropicWeights> weights,
    const TrainConfig& config, bool warm_start = true, std::vector<double>* loss_history = nullptr) {
  if (data.n == 0) throw EmptyDataset("cannot train on an empty dataset");
  if (M == 0 || data.d % M != 0) throw DimensionNotDivisible("dimension not divisible by M");
  if (k == 0 || k > data.n) throw InvalidArgument("need 1 <= k <= n");
  if (weights.size() != data.n) throw InvalidArgument("need one AnisotropicWeights per datapoint");
  b200::WeightArgs wa;
  b200::make_weights(weights, wa);
  const aq_train_config cfg = b200::to_c(config);
  std::vector<double> hist(static_cast<std::size_t>(std::max(config.max_iterations, 0)) + 1);
  std::size_t hl = 0;
  aq_multi* multi = b200::multi();
  if (multi && b200::f32_exact(data.values)) {  // row shards over $ANISOQ_DEVICES
    const std::vector<float> x = b200::to_f32(data);
    ProductCodebook pcb;
    pcb.M = M;
    pcb.k = k;
    pcb.sub_dimension = data.d / M;
    pcb.dictionaries.resize(k * data.d);
    CodeMatrix codes;
    codes.n = data.n;
    codes.M = M;
    codes.k = k;
    codes.codes.resize(data.n * M);
    b200::check(aq_multi_train_apq(multi, x.data(), data.n, data.d, M, k, &wa.w, &cfg,
                                   warm_start ? 1 : 0, pcb.dictionaries.data(),
                                   codes.codes.data(), hist.data(), &hl));
    if (loss_history) loss_history->insert(loss_history->end(), hist.begin(), hist.begin() + hl);
    return {std::move(pcb), std::move(codes)};
  }
  b200::OwnedDataset ds;
  b200::upload(data, ds);
  b200::OwnedCodebook cb;
  b200::OwnedCodes cm;
  b200::check(aq_dev_train_apq(ds.p, M, k, &wa.w, &cfg, warm_start ? 1 : 0, &cb.p, &cm.p,
                               hist.data(), &hl));
  if (loss_history) loss_history->insert(loss_history->end(), hist.begin(), hist.begin() + hl);
  return {b200::download(cb.p, M, k, data.d / M), b200::download(cm.p, data.n, M, k)};
}

// pq.hpp:581-612
inline CodeMatrix pq_quantize(const Dataset& data, const ProductCodebook& cb,
                              std::span<const AnisotropicWeights> weights, int passes,
                              int threads = 1) {
  (void)threads;
  if (data.d != cb.dim()) throw DimensionMismatch("dataset dimension does not match codebook");
  if (weights.size() != data.n) throw InvalidArgument("need one AnisotropicWeights per datapoint");
  if (passes < 0) throw InvalidArgument("passes must be >= 0");
  b200::WeightArgs wa;
  b200::make_weights(weights, wa);
  CodeMatrix out;
  out.n = data.n;
  out.M = cb.M;
  out.k = cb.k;
  out.codes.resize(data.n * cb.M);
  if (!b200::f32_exact(data.values)) {  // float64 rows: the resident-dataset path
    b200::OwnedDataset ds;
    b200::upload(data, ds);
    b200::OwnedCodebook dcb;
    b200::check(aq_codebook_upload(b200::session(), cb.dictionaries.data(), cb.M, cb.k,
                                   cb.sub_dimension, &dcb.p));
    b200::OwnedCodes cm;
    b200::check(aq_codes_alloc(b200::session(), data.n, cb.M, cb.k, &cm.p));
    b200::check(aq_dev_pq_quantize(ds.p, dcb.p, &wa.w, passes, cm.p));
    b200::check(aq_codes_download(cm.p, out.codes.data()));
    return out;
  }
  const std::vector<float> x = b200::to_f32(data);
  if (aq_multi* m = b200::multi()) {  // row shards over $ANISOQ_DEVICES
    b200::check(aq_multi_pq_quantize(m, x.data(), data.n, data.d, cb.dictionaries.data(), cb.M,
                                     cb.k, cb.sub_dimension, &wa.w, passes, out.codes.data()));
    return out;
  }
  b200::check(aq_pq_quantize(b200::session(), x.data(), data.n, data.d, cb.dictionaries.data(),
                             cb.M, cb.k, cb.sub_dimension, &wa.w, passes, out.codes.data()));
  return out;
}

// ---- serialization (pq.hpp:614-730 formats) --------------------------------------------
namespace detail {
inline void put_u32(std::ostream& out, std::uint32_t v) {
  out.write(reinterpret_cast<const char*>(&v), 4);
}
inline std::uint32_t get_u32(std::istream& in, const std::string& path) {
  std::uint32_t v = 0;
  if (!in.read(reinterpret_cast<char*>(&v), 4)) throw MalformedFile(path + ": truncated header");
  return v;
}
}  // namespace detail

inline void save_codebook(const ProductCodebook& cb, const std::string& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw MalformedFile("cannot open " + path + " for writing");
  out.write("AQCB", 4);
  detail::put_u32(out, 1u);
  detail::put_u32(out, (std::uint32_t)cb.M);
  detail::put_u32(out, (std::uint32_t)cb.k);
  detail::put_u32(out, (std::uint32_t)cb.dim());
  for (double v : cb.dictionaries) {
    const float f = static_cast<float>(v);
    out.write(reinterpret_cast<const char*>(&f), 4);
  }
  if (!out) throw MalformedFile("short write to " + path);
}

inline ProductCodebook load_codebook(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw MalformedFile("cannot open " + path);
  char magic[4] = {};
  if (!in.read(magic, 4) || std::memcmp(magic, "AQCB", 4) != 0)
    throw MalformedFile(path + ": bad magic");
  const std::uint32_t version = detail::get_u32(in, path);
  if (version != 1u) throw MalformedFile(path + ": unsupported version " + std::to_string(version));
  ProductCodebook cb;
  cb.M = detail::get_u32(in, path);
  cb.k = detail::get_u32(in, path);
  const std::uint32_t d = detail::get_u32(in, path);
  if (cb.M == 0 || d == 0 || d % cb.M != 0) throw MalformedFile(path + ": inconsistent shape");
  cb.sub_dimension = d / cb.M;
  cb.dictionaries.resize(static_cast<std::size_t>(cb.k) * d);
  for (double& v : cb.dictionaries) {
    float f = 0.0f;
    if (!in.read(reinterpret_cast<char*>(&f), 4))
      throw MalformedFile(path + ": truncated dictionaries");
    v = static_cast<double>(f);
  }
  return cb;
}

inline void save_codes(const CodeMatrix& cm, const std::string& path) {
  if (cm.k > 65536) throw InvalidArgument("code serialization supports k <= 65536");
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw MalformedFile("cannot open " + path + " for writing");
  detail::put_u32(out, (std::uint32_t)cm.n);
  detail::put_u32(out, (std::uint32_t)cm.M);
  detail::put_u32(out, (std::uint32_t)cm.k);
  for (std::uint32_t c : cm.codes) {
    if (cm.k <= 256) {
      const std::uint8_t b = (std::uint8_t)c;
      out.write(reinterpret_cast<const char*>(&b), 1);
    } else {
      const std::uint16_t b = (std::uint16_t)c;
      out.write(reinterpret_cast<const char*>(&b), 2);
    }
  }
  if (!out) throw MalformedFile("short write to " + path);
}

inline CodeMatrix load_codes(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw MalformedFile("cannot open " + path);
  CodeMatrix cm;
  cm.n = detail::get_u32(in, path);
  cm.M = detail::get_u32(in, path);
  cm.k = detail::get_u32(in, path);
  if (cm.M == 0) throw MalformedFile(path + ": M must be positive");
  cm.codes.resize(cm.n * cm.M);
  for (std::uint32_t& c : cm.codes) {
    if (cm.k <= 256) {
      std::uint8_t b = 0;
      if (!in.read(reinterpret_cast<char*>(&b), 1)) throw MalformedFile(path + ": truncated codes");
      c = b;
    } else {
      std::uint16_t b = 0;
      if (!in.read(reinterpret_cast<char*>(&b), 2)) throw MalformedFile(path + ": truncated codes");
      c = b;
    }
  }
  for (std::uint32_t c : cm.codes)
    if (c >= cm.k) throw CodeOutOfRange(path + ": stored code exceeds k");
  return cm;
}

}  // namespace anisoq
